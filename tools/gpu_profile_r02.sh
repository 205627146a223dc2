# Round-2 profile capture (run under gpurun): launch list of one timed 512^3 bench iteration and
# ncu --set full of the top kernels inside the timed NVTX range (raw pages exported to CSV on the box).
#   bash tools/gpu_profile_r02.sh launches | full
set -x
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-profile --no-ref-precision"
full() {  # tag kernel-regex count
  timeout 1200 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include timed/ \
    --kernel-name-base mangled -k regex:$2 -c $3 -o gpurun_out/r02_full_$1 -f $B > gpurun_out/r02_full_$1.log 2>&1
  ncu -i gpurun_out/r02_full_$1.ncu-rep --page raw --csv > gpurun_out/r02_full_$1.raw.csv 2>/dev/null
  gzip -f gpurun_out/r02_full_$1.raw.csv
}
case "$1" in
  launches)
    timeout 1200 ncu --nvtx --nvtx-include timed/ --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/r02_launches.csv $B > gpurun_out/r02_launches.log 2>&1 ;;
  full)
    full gs l0_gs_fast2_kernel 16
    full tensor tensor_stage_kernel 1
    full hsweep l0_hsweep_kernel 3
    full stencil_gs stencil_gs 16
    full galerkin gal_ 3
    full oc oc_pass_kernel 2 ;;
esac
find gpurun_out -name '*.ncu-rep' -delete
du -sh gpurun_out
