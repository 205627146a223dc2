set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/t_gpu.log 2>&1; echo gpu tests rc $?; tail -3 gpurun_out/t_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc $?; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc $?; tail -2 gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc $?
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-profile"
timeout 900 ncu --nvtx --nvtx-include timed/ --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01g.csv $B > gpurun_out/launches_r01g.log 2>&1; echo ncu rc $?
