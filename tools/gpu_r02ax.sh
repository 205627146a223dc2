# profiler overhead: the same bench with and without the per-family CUDA-event profiler
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-ref-precision --no-host-staged > gpurun_out/r02ax_prof.json 2>/dev/null; echo a rc $?
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-ref-precision --no-host-staged --no-profile > gpurun_out/r02ax_noprof.json 2>/dev/null; echo b rc $?
for f in prof noprof; do python -c "
import json;d=json.loads(open('gpurun_out/r02ax_$f.json').read().strip().splitlines()[-1]);print('$f',d['value'],d['e2e']['value'])"; done
