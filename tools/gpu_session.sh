set -x
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"l0_residual_norm_fast|l0_gs_fast_kernel" -c 3 -o gpurun_out/prof512 python tools/kernel_bench.py --reso 512 --reps 1 --ops vcycle_f32 > gpurun_out/ncu512.log 2>&1; echo ncu=$?
timeout 600 python tools/kernel_bench.py --reso 512 --reps 2 --ops vcycle_f32,set_density > gpurun_out/kb512.jsonl 2> gpurun_out/kb512.err; tail -3 gpurun_out/kb512.err
timeout 900 python bench.py --no-cpu-baseline --mode vcycle --no-e2e > gpurun_out/bench512_vcycle.json 2> gpurun_out/bench512_vcycle.err; tail -3 gpurun_out/bench512_vcycle.err
