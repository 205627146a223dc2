# element-sweep windows as bulk copies: bitwise tests, isolated kernel timing (old loader vs bulk), bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernel_variants.py -x -q -k "hsweep or fused_update or hadamard" > gpurun_out/r02ab_kv.log 2>&1; echo kv rc $?
tail -4 gpurun_out/r02ab_kv.log
for v in 0 1; do IHOM_HSWEEP_TMA=$v timeout 300 python tools/kernel_bench.py --reso 512 --ops l0_residual_f64,l0_defect_f64,l0_residual_f32 --reps 5 > gpurun_out/r02ab_kb$v.json 2>&1; echo kb$v rc $?; cat gpurun_out/r02ab_kb$v.json | cut -c1-400; done
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-ref-precision --no-host-staged > gpurun_out/r02ab_bench.json 2> gpurun_out/r02ab_bench.err; echo bench rc $?
python -c "
import json;d=json.loads(open('gpurun_out/r02ab_bench.json').read().strip().splitlines()[-1])
print(d['value'],d['e2e']['value'],d['roofline']['frac'],{k:d['kernels'][k] for k in ['l0_residual_f64','l0_residual_f32','l0_gs_f32']})"
tail -3 gpurun_out/r02ab_bench.err
