set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernel_variants.py -q -x --timeout 600 > gpurun_out/t_variants.log 2>&1; echo variants rc $?; tail -3 gpurun_out/t_variants.log
timeout 300 python tools/kernel_bench.py --reso 512 --ops set_density,l0_defect_f64,l0_residual_f32,vcycle_f32 --reps 3 > gpurun_out/kb.json 2>&1
cat gpurun_out/kb.json
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc $?
