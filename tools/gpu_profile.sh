# Round profile capture (run under gpurun): launch list of one timed bench iteration + ncu --set full
# of the top kernel families inside the timed NVTX range. Every report is exported to CSV on the box
# (raw metrics page) and reports over 12 MB are dropped, so the merge-back stays under gpurun's 64 MiB.
#   bash tools/gpu_profile.sh launches | part1 | part2
set -x
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-profile"
full() {  # kernel-regex count
  timeout 900 ncu --set full --clock-control none --nvtx --nvtx-include timed/ -k regex:$1 -c $2 \
    -o gpurun_out/full_$1 -f $B > gpurun_out/full_$1.log 2>&1
  ncu -i gpurun_out/full_$1.ncu-rep --page raw --csv > gpurun_out/full_$1.raw.csv 2>/dev/null
  gzip -f gpurun_out/full_$1.raw.csv
}
case "$1" in
  launches)
    timeout 900 ncu --nvtx --nvtx-include timed/ --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/launches.csv $B > gpurun_out/launches.log 2>&1 ;;
  part1)
    full l0_gs_fast2_kernel 4; full l0_sweep_kernel 1; full stencil_gs_fast_kernel 4; full l0_sweep2_kernel 1 ;;
  part2)
    full stencil_apply_fast_kernel 1; full tensor_kernel 1; full gal_stencil_fast_kernel 1
    full gal_elem_unrolled_kernel 1; full axpy_kernel 1; full sens_cached_kernel 1 ;;
  fused)
    full l0_sweep_kernel 3 ;;
  part3)  # one whole V-cycle of the GS families (pre = zero-start, post) for the per-launch traffic average
    full l0_gs_fast2_kernel 16; full stencil_gs_fast_kernel 48 ;;
esac
find gpurun_out -name '*.ncu-rep' -size +12M -delete
du -sh gpurun_out; ls -la gpurun_out
