set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernel_variants.py -q -x --timeout 600 > gpurun_out/t_variants.log 2>&1; echo variants rc $?; tail -3 gpurun_out/t_variants.log
for v in 32768 4096; do IHOM_WARP_VMAX=$v timeout 300 python tools/kernel_bench.py --reso 512 --ops vcycle_f32 --reps 3 > gpurun_out/kb_wv$v.json 2>&1; done
for v in 2 3; do IHOM_SWEEP64_MINB=$v timeout 300 python tools/kernel_bench.py --reso 512 --ops vcycle_f32 --reps 3 > gpurun_out/kb_s64_$v.json 2>&1; done
python - <<'PY'
import json
for f in ["kb_wv32768","kb_wv4096","kb_s64_2","kb_s64_3"]:
    d=json.loads(open(f"gpurun_out/{f}.json").read().splitlines()[-1])["families"]
    print(f, {k: v["ms_per_launch"] for k, v in d.items() if k in ("coarse_gs_f32","coarse_residual_f32","l0_residual_f64","l2_gs_f32")})
PY
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc $?
