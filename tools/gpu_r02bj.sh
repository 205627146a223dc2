mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_trajectories.py -x -q -m gpu -k "oc or traj" > gpurun_out/r02bj_t.log 2>&1; echo t rc $?
tail -2 gpurun_out/r02bj_t.log
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-ref-precision --no-host-staged > gpurun_out/r02bj_bench.json 2> gpurun_out/r02bj_bench.err; echo bench rc $?
python -c "
import json;d=json.loads(open('gpurun_out/r02bj_bench.json').read().strip().splitlines()[-1])
k=d['kernels'];print(d['value'],k['oc_trial'])"
