mkdir -p gpurun_out
python tools/kernel_bench.py --reso 256 --ops tensor --reps 3 > gpurun_out/r02g_kb.json 2>&1
python tools/kernel_bench.py --reso 512 --ops tensor --reps 2 >> gpurun_out/r02g_kb.json 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_kernel_variants.py -m gpu -q -x --timeout 600 -k "tensor or sensitiv or solid or laminate or 32cubed or cache" > gpurun_out/r02g_t_gpu.log 2>&1; echo gpu tests rc $?; tail -3 gpurun_out/r02g_t_gpu.log
