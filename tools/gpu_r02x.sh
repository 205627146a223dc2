# host-staged displacements (memory lever) + fused macro-force sums: tests, then the bench with its new leg
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_host_staged.py -x -q > gpurun_out/r02x_hs.log 2>&1; echo hs rc $?
tail -15 gpurun_out/r02x_hs.log
timeout 600 python -m pytest tests/test_kernel_variants.py -x -q -k "macro_sums or project_norm or fused_update" > gpurun_out/r02x_kv.log 2>&1; echo kv rc $?
tail -3 gpurun_out/r02x_kv.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02x_bench.json 2> gpurun_out/r02x_bench.err; echo bench rc $?
tail -c 600 gpurun_out/r02x_bench.json; tail -5 gpurun_out/r02x_bench.err
