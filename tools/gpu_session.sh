set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernel_variants.py tests/test_gpu_parity.py -q -x --timeout 600 > gpurun_out/t_variants.log 2>&1; echo variants rc $?; tail -3 gpurun_out/t_variants.log
for v in 0 1; do IHOM_TENSOR2=$v timeout 300 python tools/kernel_bench.py --reso 512 --ops tensor --reps 3 > gpurun_out/kb_t$v.json 2>&1; done
cat gpurun_out/kb_t*.json
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc $?
