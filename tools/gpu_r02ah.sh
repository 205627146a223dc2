# bottom cycle (cooperative launch): bitwise tests under a short timeout first, then bench
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernel_variants.py -x -q -m gpu -k "bottom_cycle" > gpurun_out/r02ah_t.log 2>&1; echo t rc $?
tail -5 gpurun_out/r02ah_t.log
timeout 900 python -m pytest tests/test_kernel_variants.py tests/test_trajectories.py -x -q -m gpu -k "rhs_pairs or traj or memory_levers" > gpurun_out/r02ah_t2.log 2>&1; echo t2 rc $?
tail -3 gpurun_out/r02ah_t2.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-ref-precision --no-host-staged > gpurun_out/r02ah_bench.json 2> gpurun_out/r02ah_bench.err; echo bench rc $?
python -c "
import json;d=json.loads(open('gpurun_out/r02ah_bench.json').read().strip().splitlines()[-1])
k=d['kernels'];print(d['value'],d['e2e']['value'],d['gpu_launches'],d['gpu_launches']/40,{x:k.get(x) for x in ['bottom_cycle','coarse_gs_f32','coarsest','l2_gs_f32']})"
tail -3 gpurun_out/r02ah_bench.err
