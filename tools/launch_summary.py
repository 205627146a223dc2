"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into a markdown table.

python tools/launch_summary.py gpurun_out/launches.csv profiles/ncu_<round>_launches.md --title "..."
Groups launches by kernel (template arguments kept, parameter list dropped) and reports launches,
total / average device time and the share of the summed kernel time.
"""
import argparse
import csv
import io
import re


def short(name):
    name = re.sub(r"^void ", "", name)
    depth, out = 0, []
    for ch in name:  # drop the parameter list, keep template arguments
        if ch == "(" and depth == 0:
            break
        depth += ch == "<"
        depth -= ch == ">"
        out.append(ch)
    return "".join(out).replace("ihomgpu::", "")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("out")
    ap.add_argument("--title", default="")
    ap.add_argument("--command", default="")
    a = ap.parse_args()
    text = open(a.csv).read()
    start = text.index('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    agg = {}
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        ms = float(r["Metric Value"]) * {"ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(r["Metric Unit"], 1e-6)
        k = short(r["Kernel Name"])
        n, t = agg.get(k, (0, 0.0))
        agg[k] = (n + 1, t + ms)
    total = sum(t for _, t in agg.values())
    nl = sum(n for n, _ in agg.values())
    lines = [f"# {a.title}", ""]
    if a.command:
        lines += [f"Command (GPU box): `{a.command}`", ""]
    lines += ["ncu serialises launches and runs them cold-cache, so absolute times sit above the in-bench CUDA-event",
              "times; the kernel SHARES are what the bench's `kernels` table must agree with.", "",
              f"Total launches: {nl}; summed kernel time {total:.1f} ms.", "",
              "| kernel | launches | total ms | share | avg ms |", "|---|---|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| {k} | {n} | {t:.2f} | {t / total:.3f} | {t / n:.4f} |")
    open(a.out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:40]))


if __name__ == "__main__":
    main()
