# full GPU suite + smoke after the macro-sums / host-staged changes
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/ -q -m gpu -p no:cacheprovider > gpurun_out/r02am_gpu.log 2>&1; echo gpu rc $?
tail -8 gpurun_out/r02am_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02am_smoke.log 2>&1; echo smoke rc $?
tail -3 gpurun_out/r02am_smoke.log
