# Round-2 profile capture (run under gpurun), in bounded parts (each well under the gpurun limit; every
# ncu report is exported to a gzipped CSV and deleted at once so the merge-back stays small):
#   bash tools/gpu_profile_r02.sh launches | gs | others
set -x
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-profile --no-ref-precision"
full() {  # tag kernel-regex count
  timeout 500 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include timed/ \
    --kernel-name-base mangled -k regex:$2 -c $3 -o gpurun_out/r02_full_$1 -f $B > gpurun_out/r02_full_$1.log 2>&1
  ncu -i gpurun_out/r02_full_$1.ncu-rep --page raw --csv 2>/dev/null | gzip > gpurun_out/r02_full_$1.raw.csv.gz
  rm -f gpurun_out/r02_full_$1.ncu-rep
}
case "$1" in
  launches)
    timeout 600 ncu --nvtx --nvtx-include timed/ --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/r02_launches.csv $B > gpurun_out/r02_launches.log 2>&1
    gzip -f gpurun_out/r02_launches.csv ;;
  gs)  # two plain (not zero-start) colour passes
    full gs l0_gs_fast2_kernelIffLi5ELb0ELin1E 2 ;;
  others)
    full tensor tensor_stage_kernel 1
    full hsweep l0_hsweep_kernel 1 ;;
esac
rm -f gpurun_out/*.ncu-rep
du -sh gpurun_out
