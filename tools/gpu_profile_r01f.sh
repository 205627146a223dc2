# Round-1 part-f capture: ncu --set full of the f32-product stencil kernels (STENCIL_F32) and the warp-per-row
# coarsest solve, inside the timed NVTX range of one bench iteration.
set -x
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-profile"
full() {  # name regex count
  timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include timed/ \
    --kernel-name-base mangled -k regex:$2 -c $3 -o gpurun_out/full_$1 -f $B > gpurun_out/full_$1.log 2>&1
  ncu -i gpurun_out/full_$1.ncu-rep --page raw --csv > gpurun_out/full_$1.raw.csv 2>/dev/null
  gzip -f gpurun_out/full_$1.raw.csv
}
full stencil_apply6f 'stencil_apply_fast_kernelIffLb0ELi6EfE' 1
full stencil_gs6f 'stencil_gs_fast_kernelIffLb0ELi6EfE' 8
full coarsest 'coarsest_kernel' 2
find gpurun_out -name '*.ncu-rep' -delete
