# host-staged: tests + the 1024x1024x512 per-GPU proxy with design updates between iterations
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_host_staged.py tests/test_capi.py -x -q -m gpu > gpurun_out/r02z_hs.log 2>&1; echo hs rc $?
tail -4 gpurun_out/r02z_hs.log
timeout 1500 python tools/host_staged_1024.py 1024 1024 512 4 > gpurun_out/r02z_1024.json 2> gpurun_out/r02z_1024.err; echo p1024 rc $?
cat gpurun_out/r02z_1024.json; tail -5 gpurun_out/r02z_1024.err
