set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernel_variants.py -q -x --timeout 300 > gpurun_out/t_variants.log 2>&1; echo variants rc $?; tail -15 gpurun_out/t_variants.log
for z in 0 1; do IHOM_ZERO_START=$z timeout 300 python tools/kernel_bench.py --reso 512 --ops vcycle_f32 --reps 3 > gpurun_out/kb_zs$z.json 2>&1; done
cat gpurun_out/kb_zs*.json
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc $?
