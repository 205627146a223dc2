"""Per-family table (ms / iteration, launches / iteration, algorithmic GB/s) from a bench.py JSON line.
python tools/bench_table.py gpurun_out/bench.json"""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
it = d["steps"] * d.get("iterations_per_step", 1)
tot = sum(v["ms"] for v in d["kernels"].values())
print(f"value {d['value']} s/iteration, e2e {d.get('e2e', {}).get('value')}, roofline {d['roofline']['kernel']} "
      f"frac {d['roofline']['frac']}, launches/iteration {d['gpu_launches'] / it:.0f}, kernel sum {tot / it:.1f} ms, "
      f"clocks {d['clocks']}")
print("| family | ms / iter | launches / iter | share | GB/s (algorithmic) |")
print("|---|---|---|---|---|")
for k, v in d["kernels"].items():
    print(f"| {k} | {v['ms'] / it:.2f} | {v['launches'] / it:.1f} | {v['share']:.3f} | {v['GB/s']} |")
