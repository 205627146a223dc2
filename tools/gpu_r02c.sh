# r02c: modal pair-thread f64 tensor: tensor/sensitivity parity + variants, trajectories, bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_kernel_variants.py tests/test_trajectories.py tests/test_coarsest.py -m gpu -q --timeout 600 > gpurun_out/r02c_t_gpu.log 2>&1; echo gpu tests rc $?; tail -8 gpurun_out/r02c_t_gpu.log
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02c_bench.json 2> gpurun_out/r02c_bench.err; echo bench rc $?; tail -3 gpurun_out/r02c_bench.err
