mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_slabs.py -x -q -m gpu -k "filter or slab" > gpurun_out/r02bh_t.log 2>&1; echo t rc $?
tail -3 gpurun_out/r02bh_t.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-ref-precision --no-host-staged > gpurun_out/r02bh_bench.json 2> gpurun_out/r02bh_bench.err; echo bench rc $?
python -c "
import json;d=json.loads(open('gpurun_out/r02bh_bench.json').read().strip().splitlines()[-1])
k=d['kernels'];print(d['value'],d['e2e']['value'],k['filter'])"
