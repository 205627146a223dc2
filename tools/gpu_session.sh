set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -3
timeout 600 python tools/kernel_bench.py --reso 512 --reps 2 --ops l0_gs_f32,l0_gs_f64,l0_residual_f64,l0_residual_f32,vcycle_f32,set_density > gpurun_out/kb512_tile.jsonl 2> gpurun_out/kb512.err; tail -3 gpurun_out/kb512.err
IHOM_L0_KERNEL=fast timeout 600 python tools/kernel_bench.py --reso 512 --reps 2 --ops l0_gs_f32,l0_residual_f64,l0_residual_f32 > gpurun_out/kb512_fast.jsonl 2>> gpurun_out/kb512.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"l0_tile" -c 2 -o gpurun_out/prof_tile python tools/kernel_bench.py --reso 256 --reps 1 --ops l0_gs_f32,l0_residual_f32 > gpurun_out/ncu_tile.log 2>&1; echo ncu=$?
