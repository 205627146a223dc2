set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernel_variants.py -q -x --timeout 600 -k "fused or sweep_level0 or energy" > gpurun_out/t_variants.log 2>&1; echo variants rc $?; tail -5 gpurun_out/t_variants.log
timeout 900 python -m pytest tests/test_slabs.py tests/test_ipc_slabs.py tests/test_gpu_parity.py -q -x --timeout 600 > gpurun_out/t_slabs.log 2>&1; echo slabs rc $?; tail -3 gpurun_out/t_slabs.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc $?
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench.json"))
print(d["value"], d["e2e"]["value"], d["cycles_per_iteration"], d["objective"], d.get("hbm_used_gb_per_gpu"))
for k, v in list(d["kernels"].items())[:8]: print(k, round(v["ms"] / 8, 2), v["launches"] // 8, v["GB/s"])
PY
