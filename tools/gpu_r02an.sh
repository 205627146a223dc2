# the 2-rank z-slab bench path at full size (512^3), both ranks on one B200 (--same-device): functionality
# of the N=2 configuration the driver scales over (time-sliced contexts: not a timing)
mkdir -p gpurun_out
IHOM_FABRIC_TIMEOUT_S=300 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --same-device --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r02an_n2.json 2> gpurun_out/r02an_n2.err; echo n2 rc $?
tail -c 1500 gpurun_out/r02an_n2.json; tail -5 gpurun_out/r02an_n2.err
