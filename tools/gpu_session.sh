set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_kernel_variants.py -q -x --timeout 900 -k "stream" > gpurun_out/t_var.log 2>&1; echo var rc $?; tail -3 gpurun_out/t_var.log
for k in 0 1; do IHOM_STENCIL_STREAM=$k timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_st$k.json 2> gpurun_out/bench_st$k.err; echo rc $?
python - $k <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/bench_st{sys.argv[1]}.json"))
print(sys.argv[1], d["value"], d["e2e"]["value"], d.get("cycles_per_iteration"), d["objective"])
for k, v in d["kernels"].items():
    if k.startswith("l1") or k.startswith("l2"): print("  ", k, round(v["ms"] / 8, 2), v["launches"] / 8, v["GB/s"])
PY
done
