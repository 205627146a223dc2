set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -3
for m in 1 3 4; do IHOM_RES_MINB=$m timeout 300 python tools/kernel_bench.py --reso 512 --reps 2 --ops vcycle_f32 > gpurun_out/kb512_res$m.jsonl 2>> gpurun_out/kb512.err; done
IHOM_L0_GS2=0 timeout 300 python tools/kernel_bench.py --reso 512 --reps 2 --ops l0_gs_f32 > gpurun_out/kb512_gs1.jsonl 2>> gpurun_out/kb512.err
timeout 300 python tools/kernel_bench.py --reso 512 --reps 2 --ops l0_gs_f32,set_density > gpurun_out/kb512_gs2.jsonl 2>> gpurun_out/kb512.err
tail -3 gpurun_out/kb512.err
timeout 900 python bench.py > gpurun_out/bench512.json 2> gpurun_out/bench512.err; tail -3 gpurun_out/bench512.err
