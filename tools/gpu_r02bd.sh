# same-box A/B of the colour-pair GS (bench defaults minus the side legs)
mkdir -p gpurun_out
for v in 0 1 0 1; do IHOM_GS_PAIR=$v timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-ref-precision --no-host-staged > gpurun_out/r02bd_$v.json 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/r02bd_$v.json').read().strip().splitlines()[-1]);print('GS_PAIR=$v',d['value'],d['e2e']['value'],d['gpu_launches']/40,d['roofline']['frac'])"; done
