set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_kernel_variants.py tests/test_gpu_parity.py -q --timeout 900 > gpurun_out/t_gpu.log 2>&1; echo tests rc $?; tail -3 gpurun_out/t_gpu.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc $?
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench.json"))
print(d["value"], d["e2e"]["value"], d.get("cycles_per_iteration"), d["objective"], d["kernels"]["vector"], d["kernels"]["reduce"])
PY
