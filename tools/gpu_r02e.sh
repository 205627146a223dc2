# r02e: staged tensor kernel + coarsest deflation: parity tests, kernel bench, bench.
mkdir -p gpurun_out
python tools/kernel_bench.py --reso 256 --ops tensor,sensitivity --reps 3 > gpurun_out/r02e_kb.json 2>&1
python tools/kernel_bench.py --reso 512 --ops tensor --reps 2 >> gpurun_out/r02e_kb.json 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_kernel_variants.py tests/test_coarsest.py -m gpu -q -x --timeout 600 > gpurun_out/r02e_t_gpu.log 2>&1; echo gpu tests rc $?; tail -8 gpurun_out/r02e_t_gpu.log
for p in 1; do timeout 600 python tools/long_run.py --reso 128 --iters 24 --project $p > gpurun_out/r02e_long128.json 2>&1; done
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02e_bench.json 2> gpurun_out/r02e_bench.err; echo bench rc $?; tail -3 gpurun_out/r02e_bench.err
