mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_kernel_variants.py tests/test_trajectories.py tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/r02bg.log 2>&1; echo rc $?
tail -2 gpurun_out/r02bg.log
