# Round-1 part-d capture: launch list of one timed bench iteration with the sum-factorised kernels, and
# ncu --set full of the new kernels (fused / plain f64 element sweep, f32 element sweep, sum/difference
# tensor pass) plus the dominant level-0 GS pass. Raw pages exported on the box (CSV, gzip).
set -x
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-profile"
timeout 900 ncu --nvtx --nvtx-include timed/ --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_r01d.csv $B > gpurun_out/launches_r01d.log 2>&1
full() {  # name regex count
  timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include timed/ \
    --kernel-name-base mangled -k regex:$2 -c $3 -o gpurun_out/full_$1 -f $B > gpurun_out/full_$1.log 2>&1
  ncu -i gpurun_out/full_$1.ncu-rep --page raw --csv > gpurun_out/full_$1.raw.csv 2>/dev/null
  gzip -f gpurun_out/full_$1.raw.csv
}
full hsweep_fused 'l0_hsweep_kernelIfdLi2ELi8ELi2ELb1E' 1
full hsweep_defect 'l0_hsweep_kernelIfdLi2ELi8ELi2ELb0E' 1
full hsweep_f32 'l0_hsweep_kernelIffLi1E' 1
full tensor_hada 'tensor_kernelIdfLb1E' 1
full l0_gs 'l0_gs_fast2_kernel' 8
find gpurun_out -name '*.ncu-rep' -size +12M -delete
du -sh gpurun_out; ls -la gpurun_out
