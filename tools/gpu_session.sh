# GPU session: parity tests, ncu captures of the level-0 kernels, isolated kernel timings, bench.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -8
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"l0_gs_kernel|l0_apply_kernel" -c 4 -o gpurun_out/prof_l0 python tools/kernel_bench.py --reso 256 --reps 1 --ops l0_gs_f32,l0_residual_f32,l0_residual_f64 > gpurun_out/ncu_l0.log 2>&1; echo ncu=$?
timeout 600 python tools/kernel_bench.py --reso 512 --reps 2 > gpurun_out/kb512.jsonl 2> gpurun_out/kb512.err; tail -3 gpurun_out/kb512.err
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench512.json 2> gpurun_out/bench512.err; tail -3 gpurun_out/bench512.err
