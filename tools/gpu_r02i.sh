# r02i: multi-process slab paths (IPC fabric with bounded neighbour barriers) + torchrun bench on one device.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_ipc_slabs.py tests/test_slabs.py -m gpu -q --timeout 900 > gpurun_out/r02i_t_gpu.log 2>&1; echo slab tests rc $?; tail -6 gpurun_out/r02i_t_gpu.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --same-device --reso 128 --steps 3 --warmup 3 > gpurun_out/r02i_bench2.json 2> gpurun_out/r02i_bench2.err; echo bench2 rc $?; tail -2 gpurun_out/r02i_bench2.err
