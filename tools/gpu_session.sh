set -x
mkdir -p gpurun_out
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo rc $?
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench.json"))
print(d["value"], d["e2e"]["value"], d.get("cycles_per_iteration"))
for k, v in d["kernels"].items():
    if k.startswith("l1") or k.startswith("l2") or k.startswith("coarse"): print("  ", k, round(v["ms"] / 8, 2), v["launches"] / 8, v["GB/s"])
PY
timeout 1500 python -m pytest tests/test_slabs.py -q --timeout 900 -k "256" > gpurun_out/t_slab.log 2>&1; echo slab rc $?; tail -2 gpurun_out/t_slab.log
