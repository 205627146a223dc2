set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernel_variants.py -q -x --timeout 600 > gpurun_out/t_variants.log 2>&1; echo variants rc $?; tail -3 gpurun_out/t_variants.log
for v in 0 1; do IHOM_L0_CPAIR=$v timeout 300 python tools/kernel_bench.py --reso 512 --ops l0_gs_f32,vcycle_f32 --reps 3 > gpurun_out/kb_cp$v.json 2>&1; done
cat gpurun_out/kb_cp*.json
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc $?
