# Round-2 final profile (bounded parts; ncu reports exported to gzipped CSV and deleted at once):
#   launch list of one timed 512^3 iteration, full captures of the bottom cycle, the fused macro
#   force and two level-0 GS colour passes
set -x
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-profile --no-ref-precision --no-host-staged"
full() {  # tag kernel-regex count
  timeout 500 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include timed/ \
    --kernel-name-base mangled -k regex:$2 -c $3 -o gpurun_out/r02b_full_$1 -f $B > gpurun_out/r02b_full_$1.log 2>&1
  ncu -i gpurun_out/r02b_full_$1.ncu-rep --page raw --csv 2>/dev/null | gzip > gpurun_out/r02b_full_$1.raw.csv.gz
  rm -f gpurun_out/r02b_full_$1.ncu-rep
}
timeout 600 ncu --nvtx --nvtx-include timed/ --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r02b_launches.csv $B > gpurun_out/r02b_launches.log 2>&1
gzip -f gpurun_out/r02b_launches.csv
full bottom bottom_cycle_kernel 1
full macro macro_force_sums_kernel 1
full gs l0_gs_fast2_kernelIffLi5ELb0ELin1E 2
rm -f gpurun_out/*.ncu-rep
du -sh gpurun_out
