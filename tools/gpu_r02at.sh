mkdir -p gpurun_out
timeout 300 python tools/kernel_bench.py --reso 512 --ops l0_residual_f32 --reps 5 > gpurun_out/r02at_kb.json 2>&1; echo kb rc $?; cut -c1-250 gpurun_out/r02at_kb.json
