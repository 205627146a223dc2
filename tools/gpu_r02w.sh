# fused macro force + component sums: bit identity, trajectories, headline bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernel_variants.py tests/test_trajectories.py -m gpu -x -q -k "macro_sums or project_norm or traj" > gpurun_out/r02w_tests.log 2>&1; echo tests rc $?
tail -3 gpurun_out/r02w_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02w_bench.json 2> gpurun_out/r02w_bench.err; echo bench rc $?
tail -c 1500 gpurun_out/r02w_bench.json
