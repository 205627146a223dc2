mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_trajectories.py tests/test_slabs.py -m gpu -q -x --timeout 900 > gpurun_out/r02m_t_gpu.log 2>&1; echo gpu tests rc $?; tail -4 gpurun_out/r02m_t_gpu.log
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02m_bench.json 2> gpurun_out/r02m_bench.err; echo bench rc $?; tail -2 gpurun_out/r02m_bench.err
