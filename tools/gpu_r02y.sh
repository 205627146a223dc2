# host-staged displacements: tests, bench leg, and the 1024x1024x512 per-GPU proxy
mkdir -p gpurun_out
free -g | head -2; nproc
timeout 900 python -m pytest tests/test_host_staged.py -x -q > gpurun_out/r02y_hs.log 2>&1; echo hs rc $?
tail -15 gpurun_out/r02y_hs.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-ref-precision > gpurun_out/r02y_bench.json 2> gpurun_out/r02y_bench.err; echo bench rc $?
python -c "
import json;d=json.loads(open('gpurun_out/r02y_bench.json').read().strip().splitlines()[-1])
print(d['value'],d['e2e'],d['hbm_used_gb_per_gpu'],d.get('host_staged'))"
tail -3 gpurun_out/r02y_bench.err
timeout 1200 python tools/host_staged_1024.py 1024 1024 512 3 > gpurun_out/r02y_1024.json 2> gpurun_out/r02y_1024.err; echo p1024 rc $?
cat gpurun_out/r02y_1024.json; tail -5 gpurun_out/r02y_1024.err
