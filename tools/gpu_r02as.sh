mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "runner_options or all_double" > gpurun_out/r02as.log 2>&1; echo rc $?
tail -15 gpurun_out/r02as.log
