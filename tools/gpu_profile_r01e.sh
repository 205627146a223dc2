# Round-1 part-e capture: ncu --set full of the lockstep-group stencil kernels (six RHSs per launch),
# the column-march tensor pass and the fused f64 element sweep, inside the timed NVTX range.
set -x
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-profile"
full() {  # name regex count
  timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include timed/ \
    --kernel-name-base mangled -k regex:$2 -c $3 -o gpurun_out/full_$1 -f $B > gpurun_out/full_$1.log 2>&1
  ncu -i gpurun_out/full_$1.ncu-rep --page raw --csv > gpurun_out/full_$1.raw.csv 2>/dev/null
  gzip -f gpurun_out/full_$1.raw.csv
}
full stencil_gs6 'stencil_gs_fast_kernelIffLb0ELi6E' 8
full stencil_apply6 'stencil_apply_fast_kernelIffLb0ELi6E' 1
full tensor_cols 'tensor_kernelIdfLb1E' 1
find gpurun_out -name '*.ncu-rep' -delete
ls -la gpurun_out | tail -12
