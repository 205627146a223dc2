set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernel_variants.py -q -x --timeout 600 > gpurun_out/t_variants.log 2>&1; echo variants rc $?; tail -5 gpurun_out/t_variants.log
for v in 0 1; do IHOM_GAL_UNROLLED=$v timeout 300 python tools/kernel_bench.py --reso 512 --ops set_density --reps 3 > gpurun_out/kb_gal$v.json 2>&1; done
cat gpurun_out/kb_gal*.json
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc $?
