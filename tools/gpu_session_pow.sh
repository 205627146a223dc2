set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/t_gpu.log 2>&1; echo gpu tests rc $?; tail -3 gpurun_out/t_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc $?; tail -2 gpurun_out/smoke.log
for k in 0 1; do IHOM_POW_INT=$k timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_pw$k.json 2> gpurun_out/bench_pw$k.err; echo rc $?
python - $k <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/bench_pw{sys.argv[1]}.json"))
print(sys.argv[1], d["value"], d["e2e"]["value"], d.get("cycles_per_iteration"), d["objective"], d["kernels"]["pow"])
PY
done
