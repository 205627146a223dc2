set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_kernel_variants.py tests/test_slabs.py tests/test_ipc_slabs.py -q --timeout 900 > gpurun_out/t_var.log 2>&1; echo var rc $?; tail -5 gpurun_out/t_var.log
