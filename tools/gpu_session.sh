set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 600 -k "level0_apply" > gpurun_out/t_par.log 2>&1; echo par rc $?; tail -3 gpurun_out/t_par.log
timeout 900 python -m pytest tests/test_kernel_variants.py -q -x --timeout 600 -k "hadamard" > gpurun_out/t_var.log 2>&1; echo var rc $?; tail -3 gpurun_out/t_var.log
for k in 0 1; do IHOM_HSWEEP=$k IHOM_HSWEEP32=$k timeout 600 python tools/kernel_bench.py --reso 512 --ops l0_defect_f64,l0_residual_f64,l0_residual_f32 --reps 3; done > gpurun_out/kb.log 2>&1; grep -v "^+" gpurun_out/kb.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc $?; tail -3 gpurun_out/bench.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench.json"))
print(d["value"], d["e2e"]["value"], d.get("cycles_per_iteration"), d.get("objective"), d.get("roofline"))
for k, v in list(d["kernels"].items())[:14]: print(k, round(v["ms"] / 8, 2), v["launches"] / 8, v["GB/s"])
PY
