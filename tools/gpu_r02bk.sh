# same-box A/B: u += e folded into the f64 defect sweep (FUSED_UPDATE=1, default) vs a separate axpy
mkdir -p gpurun_out
for v in 1 0 1 0; do IHOM_FUSED_UPDATE=$v timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-ref-precision --no-host-staged > gpurun_out/r02bk_$v.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/r02bk_$v.json').read().strip().splitlines()[-1]);k=d['kernels'];print('FUSED_UPDATE=$v',d['value'],d['e2e']['value'],k['l0_residual_f64']['ms']/40,k.get('vector',{}).get('ms',0)/40)"; done
