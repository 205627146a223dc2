mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernel_variants.py tests/test_trajectories.py -x -q -m gpu -k "bottom or rhs_pairs or traj or memory_levers" > gpurun_out/r02ap.log 2>&1; echo rc $?
tail -3 gpurun_out/r02ap.log
