# colour-pair level-0 GS: bitwise tests (bounded), isolated timing, bench
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernel_variants.py -x -q -m gpu -k "gs_pair or zero_start or fused_update" > gpurun_out/r02az_t.log 2>&1; echo t rc $?
tail -3 gpurun_out/r02az_t.log
for v in 0 1; do IHOM_GS_PAIR=$v timeout 300 python tools/kernel_bench.py --reso 512 --ops l0_gs_f32 --reps 5 > gpurun_out/r02az_kb$v.json 2>&1; echo kb$v; cut -c1-250 gpurun_out/r02az_kb$v.json; done
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-ref-precision --no-host-staged > gpurun_out/r02az_bench.json 2> gpurun_out/r02az_bench.err; echo bench rc $?
python -c "
import json;d=json.loads(open('gpurun_out/r02az_bench.json').read().strip().splitlines()[-1])
k=d['kernels'];print(d['value'],d['e2e']['value'],d['gpu_launches']/40,d['roofline'],k['l0_gs_f32'])"
