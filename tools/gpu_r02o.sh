mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
timeout 1200 $S --tool memcheck --leak-check no --print-limit 20 python tools/sanitize_run.py > gpurun_out/r02o_memcheck.log 2>&1; echo memcheck rc $?; tail -4 gpurun_out/r02o_memcheck.log
timeout 1500 $S --tool racecheck --print-limit 20 python tools/sanitize_run.py > gpurun_out/r02o_racecheck.log 2>&1; echo racecheck rc $?; tail -4 gpurun_out/r02o_racecheck.log
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "coarse_level or transfer or density_expr or four_plane" > gpurun_out/r02o_t.log 2>&1; echo tests rc $?; tail -3 gpurun_out/r02o_t.log
timeout 2400 python tools/cpu_baseline_512.py > gpurun_out/r02o_cpu512.json 2>&1; echo cpu512 rc $?; tail -1 gpurun_out/r02o_cpu512.json
