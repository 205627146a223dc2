mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernel_variants.py -q -m gpu -k "memory_levers or macro_sums or project_norm" > gpurun_out/r02af.log 2>&1; echo rc $?
tail -3 gpurun_out/r02af.log
