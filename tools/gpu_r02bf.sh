mkdir -p gpurun_out
for v in 1 0; do IHOM_HSWEEP32=$v timeout 300 python tools/kernel_bench.py --reso 512 --ops l0_residual_f32 --reps 5 > gpurun_out/r02bf_kb$v.json 2>&1; echo hs32=$v; cut -c1-250 gpurun_out/r02bf_kb$v.json; done
