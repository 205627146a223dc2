# f64 element sweep with 16-row CTAs (HS_BY64=16) vs 8-row
mkdir -p gpurun_out
for v in 8 16; do IHOM_HS_BY64=$v timeout 300 python tools/kernel_bench.py --reso 512 --ops l0_residual_f64,l0_defect_f64 --reps 5 > gpurun_out/r02ag_kb$v.json 2>&1; echo kb$v rc $?; cut -c1-250 gpurun_out/r02ag_kb$v.json; done
IHOM_HS_BY64=16 timeout 900 python -m pytest tests/test_kernel_variants.py tests/test_trajectories.py -x -q -m gpu -k "hadamard or fused_update or traj" > gpurun_out/r02ag_t.log 2>&1; echo t rc $?; tail -2 gpurun_out/r02ag_t.log
IHOM_HS_BY64=16 timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-ref-precision --no-host-staged > gpurun_out/r02ag_bench.json 2> gpurun_out/r02ag_bench.err; echo bench rc $?
python -c "
import json;d=json.loads(open('gpurun_out/r02ag_bench.json').read().strip().splitlines()[-1])
k=d['kernels'];print(d['value'],d['e2e']['value'],k['l0_residual_f64'],d['cycles_per_iteration'][:6])"
