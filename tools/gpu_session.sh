set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_kernel_variants.py -q --timeout 900 -k "memory or rhs" > gpurun_out/t_var.log 2>&1; echo var rc $?; tail -4 gpurun_out/t_var.log
