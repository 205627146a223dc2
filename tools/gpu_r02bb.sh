mkdir -p gpurun_out
for v in 2 3; do IHOM_PAIR_MINB=$v timeout 300 python tools/kernel_bench.py --reso 512 --ops l0_gs_f32 --reps 5 > gpurun_out/r02bb_kb$v.json 2>&1; echo kb$v; cut -c1-250 gpurun_out/r02bb_kb$v.json; done
