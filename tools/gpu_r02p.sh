# r02p: full GPU suite + smoke + the driver's bench commands (both arms)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/r02p_t_gpu.log 2>&1; echo gpu tests rc $?; tail -4 gpurun_out/r02p_t_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02p_smoke.log 2>&1; echo smoke rc $?; tail -2 gpurun_out/r02p_smoke.log
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02p_bench.json 2> gpurun_out/r02p_bench.err; echo bench rc $?; tail -2 gpurun_out/r02p_bench.err
timeout 1200 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02p_ref.json 2> gpurun_out/r02p_ref.err; echo ref rc $?; tail -2 gpurun_out/r02p_ref.err
