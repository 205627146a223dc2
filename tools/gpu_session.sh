set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu 2>&1 | tail -15
timeout 300 python bench.py --reso 128 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench128.json 2> gpurun_out/bench128.err; tail -3 gpurun_out/bench128.err
timeout 900 python bench.py > gpurun_out/bench512.json 2> gpurun_out/bench512.err; tail -3 gpurun_out/bench512.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches256.csv python bench.py --reso 256 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu1=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"l0_gs_kernel|stencil_gs_kernel|l0_apply_kernel|tensor_kernel|gal_elem" -s 40 -c 8 -o gpurun_out/prof256 python bench.py --reso 256 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu2=$?
ls -la gpurun_out
