mkdir -p gpurun_out
timeout 1500 python tools/host_staged_1024.py 1024 1024 512 4 > gpurun_out/r02bc_1024.json 2> gpurun_out/r02bc_1024.err; echo p1024 rc $?
cat gpurun_out/r02bc_1024.json; tail -3 gpurun_out/r02bc_1024.err
