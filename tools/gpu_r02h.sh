# r02h: full GPU suite after variant cleanup + new tests; bench with and without per-family profiling.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r02h_t_gpu.log 2>&1; echo gpu tests rc $?; tail -12 gpurun_out/r02h_t_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02h_smoke.log 2>&1; echo smoke rc $?; tail -3 gpurun_out/r02h_smoke.log
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02h_bench.json 2> gpurun_out/r02h_bench.err; echo bench rc $?; tail -2 gpurun_out/r02h_bench.err
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline --no-profile > gpurun_out/r02h_bench_noprof.json 2> gpurun_out/r02h_bench_noprof.err; echo bench noprof rc $?
