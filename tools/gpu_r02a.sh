# r02a: coarsest fix validation on the B200 -- long runs (projected vs reference operator),
# GPU tests, the driver's bench command in both arms.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a_smi.txt 2>&1; nproc >> gpurun_out/r02a_smi.txt; free -g >> gpurun_out/r02a_smi.txt
for p in 1 0; do timeout 600 python tools/long_run.py --reso 128 --iters 40 --project $p > gpurun_out/r02a_long128_p$p.json 2>&1; echo long128 p$p rc $?; done
timeout 900 python tools/long_run.py --reso 256 --iters 30 --vol 0.3 --obj bulk > gpurun_out/r02a_long256_bulk.json 2>&1; echo long256 rc $?
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err; echo bench rc $?; tail -3 gpurun_out/r02a_bench.err
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/r02a_t_gpu.log 2>&1; echo gpu tests rc $?; tail -5 gpurun_out/r02a_t_gpu.log
timeout 1200 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02a_ref.json 2> gpurun_out/r02a_ref.err; echo ref rc $?; tail -3 gpurun_out/r02a_ref.err
