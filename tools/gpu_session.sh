set -x
mkdir -p gpurun_out
for v in 4096 512 64; do IHOM_WARP_VMAX=$v timeout 300 python tools/kernel_bench.py --reso 512 --ops vcycle_f32 --reps 3 > gpurun_out/kb_wv$v.json 2>&1; done
python - <<'PY'
import json
for f in ["kb_wv4096","kb_wv512","kb_wv64"]:
    d=json.loads(open(f"gpurun_out/{f}.json").read().splitlines()[-1])["families"]
    print(f, {k: (v["ms_per_launch"], v["launches"]) for k, v in d.items() if k in ("coarse_gs_f32","coarse_residual_f32","prolong","restrict")})
PY
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc $?
bash tools/gpu_profile.sh part2
