# fused macro force with per-block partials: tests + bench (profiled families)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernel_variants.py tests/test_trajectories.py tests/test_host_staged.py -x -q -k "macro_sums or project_norm or traj or host_staged" > gpurun_out/r02ad_kv.log 2>&1; echo kv rc $?
tail -3 gpurun_out/r02ad_kv.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-ref-precision --no-host-staged > gpurun_out/r02ad_bench.json 2> gpurun_out/r02ad_bench.err; echo bench rc $?
python -c "
import json;d=json.loads(open('gpurun_out/r02ad_bench.json').read().strip().splitlines()[-1])
k=d['kernels'];print(d['value'],d['e2e']['value'],d['roofline']['frac'],k['macro_force'],k['reduce'],d['gpu_launches'])"
tail -3 gpurun_out/r02ad_bench.err
