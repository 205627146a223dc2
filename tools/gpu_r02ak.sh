# compute-sanitizer on the round-2 final kernels (bounded)
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 900 $CS --tool $tool --error-exitcode 9 python tools/sanitize_run.py > gpurun_out/r02ak_$tool.log 2>&1; echo $tool rc $?
  tail -3 gpurun_out/r02ak_$tool.log
done
