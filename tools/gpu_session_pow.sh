set -x
mkdir -p gpurun_out
for k in 0 1; do IHOM_FILTER_NZ=$k timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_slabs.py -q --timeout 900 -k "filter or slab" > gpurun_out/t_f$k.log 2>&1; echo t $k rc $?; tail -1 gpurun_out/t_f$k.log; done
for k in 0 1; do IHOM_FILTER_NZ=$k timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_f$k.json 2> gpurun_out/bench_f$k.err; echo rc $?
python - $k <<'PY'
import json, sys
d = json.load(open(f"gpurun_out/bench_f{sys.argv[1]}.json"))
print(sys.argv[1], d["value"], d.get("cycles_per_iteration"), d["objective"], d["kernels"]["filter"])
PY
done
