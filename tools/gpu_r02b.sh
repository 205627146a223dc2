# r02b: fused stencil Galerkin + f64 mixed-mode energies: GPU tests, bench (driver command).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r02b_t_gpu.log 2>&1; echo gpu tests rc $?; tail -15 gpurun_out/r02b_t_gpu.log
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err; echo bench rc $?; tail -3 gpurun_out/r02b_bench.err
