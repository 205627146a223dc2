set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernel_variants.py -q -x --timeout 600 -k column > gpurun_out/t_col.log 2>&1; echo col rc $?; tail -3 gpurun_out/t_col.log
for v in 0 2 4 8; do IHOM_GS_COL=$v timeout 300 python tools/kernel_bench.py --reso 512 --ops l0_gs_f32,vcycle_f32 --reps 3 > gpurun_out/kb_col$v.json 2>&1; done
python - <<'PY'
import json
for v in (0, 2, 4, 8):
    ls = open(f"gpurun_out/kb_col{v}.json").read().splitlines()
    a = json.loads(ls[0])["families"]["l0_gs_f32"]["ms_per_launch"]; b = json.loads(ls[1])["families"]["l0_gs_f32"]["ms_per_launch"]
    print("GS_COL", v, "pass", a, "vcycle avg", b)
PY
bash tools/gpu_profile.sh fused
