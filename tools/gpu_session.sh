set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -8
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"l0_apply_fast_kernel|stencil_gs_fast" -c 3 -o gpurun_out/prof_b python tools/kernel_bench.py --reso 256 --reps 1 --ops l0_residual_f64,l1_gs_f32 > gpurun_out/ncu_b.log 2>&1; echo ncu=$?
timeout 600 python tools/kernel_bench.py --reso 512 --reps 2 > gpurun_out/kb512.jsonl 2> gpurun_out/kb512.err; tail -3 gpurun_out/kb512.err
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench512.json 2> gpurun_out/bench512.err; tail -3 gpurun_out/bench512.err
