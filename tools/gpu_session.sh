set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernel_variants.py -q -x --timeout 600 -k "rhs_pairs" > gpurun_out/t_pairs.log 2>&1; echo pairs rc $?; tail -25 gpurun_out/t_pairs.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc $?; tail -3 gpurun_out/bench.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench.json"))
print(d["value"], d["e2e"]["value"], d["cycles_per_iteration"], d["objective"])
for k, v in list(d["kernels"].items())[:12]: print(k, round(v["ms"] / 8, 2), v["launches"] // 8, v["GB/s"])
PY
