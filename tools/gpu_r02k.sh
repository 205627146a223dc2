mkdir -p gpurun_out
python tools/kernel_bench.py --reso 512 --ops l0_gs_f32 --reps 3 > gpurun_out/r02k_kb.json 2>&1
timeout 1500 python -m pytest tests/test_trajectories.py tests/test_kernel_variants.py tests/test_gpu_parity.py -m gpu -q -x --timeout 900 > gpurun_out/r02k_t_gpu.log 2>&1; echo gpu tests rc $?; tail -4 gpurun_out/r02k_t_gpu.log
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02k_bench.json 2> gpurun_out/r02k_bench.err; echo bench rc $?
