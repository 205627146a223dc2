set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/t_gpu.log 2>&1; echo gpu tests rc $?; tail -5 gpurun_out/t_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc $?; tail -2 gpurun_out/bench.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench.json"))
print(d["value"], d["e2e"]["value"], d.get("cycles_per_iteration"), d.get("objective"), d["hbm_used_gb_per_gpu"], d.get("cpu_baseline"))
for k, v in list(d["kernels"].items())[:14]: print("  ", k, round(v["ms"] / 8, 2), v["launches"] / 8, v["GB/s"])
PY
