mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_host_staged.py tests/test_ipc_slabs.py -x -q -m gpu > gpurun_out/r02ar_t.log 2>&1; echo t rc $?
tail -2 gpurun_out/r02ar_t.log
timeout 900 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-ref-precision --no-e2e > gpurun_out/r02ar_bench.json 2> gpurun_out/r02ar_bench.err; echo bench rc $?
python -c "
import json;d=json.loads(open('gpurun_out/r02ar_bench.json').read().strip().splitlines()[-1]);print(d['host_staged'])"
