# bulk-window element sweep without per-issue fences: tests, isolated timing, ncu of old vs bulk loader
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernel_variants.py -x -q -k "hsweep or fused_update or hadamard" > gpurun_out/r02ac_kv.log 2>&1; echo kv rc $?
tail -3 gpurun_out/r02ac_kv.log
for v in 0 1; do IHOM_HSWEEP_TMA=$v timeout 300 python tools/kernel_bench.py --reso 512 --ops l0_residual_f64,l0_defect_f64,l0_residual_f32 --reps 5 > gpurun_out/r02ac_kb$v.json 2>&1; echo kb$v rc $?; cut -c1-300 gpurun_out/r02ac_kb$v.json; done
for v in 0 1; do
  IHOM_HSWEEP_TMA=$v timeout 400 ncu --set full --clock-control none --kernel-name-base mangled -k regex:l0_hsweep_kernelIfdLi1 -c 1 -o gpurun_out/r02ac_hs$v -f python tools/kernel_bench.py --reso 512 --ops l0_residual_f64 --reps 1 > gpurun_out/r02ac_ncu$v.log 2>&1; echo ncu$v rc $?
  ncu -i gpurun_out/r02ac_hs$v.ncu-rep --page raw --csv > gpurun_out/r02ac_hs$v.raw.csv 2>/dev/null
  rm -f gpurun_out/r02ac_hs$v.ncu-rep
done
ls -la gpurun_out | grep r02ac
