# host-staged: tests (one domain, local slabs, IPC slabs) + bench leg
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_host_staged.py tests/test_ipc_slabs.py -x -q -m gpu > gpurun_out/r02aa_hs.log 2>&1; echo hs rc $?
tail -4 gpurun_out/r02aa_hs.log
timeout 900 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-ref-precision --no-e2e > gpurun_out/r02aa_bench.json 2> gpurun_out/r02aa_bench.err; echo bench rc $?
python -c "
import json;d=json.loads(open('gpurun_out/r02aa_bench.json').read().strip().splitlines()[-1])
print(d['value'],d['hbm_used_gb_per_gpu'],d.get('host_staged'))"
tail -3 gpurun_out/r02aa_bench.err
