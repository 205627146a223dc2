set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_slabs.py tests/test_ipc_slabs.py tests/test_kernel_variants.py -q -x --timeout 900 > gpurun_out/t_slab.log 2>&1; echo slab rc $?; tail -3 gpurun_out/t_slab.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --same-device --reso 256 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo bench2 rc $?; tail -3 gpurun_out/bench2.err; head -c 600 gpurun_out/bench2.json
