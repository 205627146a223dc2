set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -3
timeout 600 python tools/kernel_bench.py --reso 512 --reps 2 --ops l0_gs_f32,l0_residual_f64,l0_residual_f32,tensor,sensitivity > gpurun_out/kb512.jsonl 2> gpurun_out/kb512.err; tail -3 gpurun_out/kb512.err
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench512.json 2> gpurun_out/bench512.err; tail -3 gpurun_out/bench512.err
timeout 900 python bench.py --no-cpu-baseline --mode pcg --no-e2e > gpurun_out/bench512_pcg.json 2> gpurun_out/bench512_pcg.err; tail -3 gpurun_out/bench512_pcg.err
