"""Summarise an ncu report (--set full; .ncu-rep or its exported raw page .csv[.gz]) into profiles/: per-kernel duration, DRAM
bytes, throughput %, occupancy, issue activity and top stall reasons.

python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/ncu_r01_<name>.md [--json profiles/ncu_traffic.json --family l0_gs_f32=l0_tile_kernel]
"""
import argparse
import csv
import io
import json
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("launch__registers_per_thread", "regs"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1 %"),
]


def to_bytes(v, unit):
    f = float(v)
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def to_ms(v, unit):
    f = float(v)
    return f * {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}.get(unit, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    ap.add_argument("--json")
    ap.add_argument("--family", action="append", default=[], help="family=kernel-substring")
    ap.add_argument("--title", default="")
    a = ap.parse_args()
    if a.rep.endswith(".csv.gz") or a.rep.endswith(".csv"):  # raw page exported on the GPU box
        import gzip
        raw = (gzip.open(a.rep, "rt") if a.rep.endswith(".gz") else open(a.rep)).read()
    else:
        raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    idx = {m: hdr.index(m) for m, _ in METRICS if m in hdr}
    kname = hdr.index("Kernel Name")
    grid = hdr.index("Grid Size") if "Grid Size" in hdr else None
    lines = [f"# ncu summary: {a.title or a.rep}", "", "| kernel | grid | " + " | ".join(n for _, n in METRICS if _ in idx) + " |",
             "|---" * (2 + len(idx)) + "|"]
    per_kernel = {}
    for r in rows[2:]:
        name = r[kname]
        cells = []
        for m, n in METRICS:
            if m not in idx:
                continue
            v, u = r[idx[m]], units[idx[m]]
            if "bytes" in m:
                cells.append(f"{to_bytes(v, u) / 1e6:.1f} MB")
            elif m == "gpu__time_duration.sum":
                cells.append(f"{to_ms(v, u):.3f} ms")
            else:
                cells.append(v)
        lines.append(f"| {name[:70]} | {r[grid] if grid is not None else ''} | " + " | ".join(cells) + " |")
        rd = to_bytes(r[idx["dram__bytes_read.sum"]], units[idx["dram__bytes_read.sum"]])
        wr = to_bytes(r[idx["dram__bytes_write.sum"]], units[idx["dram__bytes_write.sum"]])
        per_kernel.setdefault(name, []).append(rd + wr)
    stall_cols = [(i, h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""))
                  for i, h in enumerate(hdr)
                  if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")]
    if stall_cols:
        lines += ["", "## warp stalls per issued instruction (top 5, first launch of each kernel)", ""]
        seen = set()
        for r in rows[2:]:
            if r[kname] in seen:
                continue
            seen.add(r[kname])
            vals = sorted(((float(r[i]), n) for i, n in stall_cols if r[i] not in ("", "n/a") and n != "selected"),
                          reverse=True)[:5]
            lines.append(f"* `{r[kname][:60]}`: " + ", ".join(f"{n} {v:.2f}" for v, n in vals))
    open(a.out, "w").write("\n".join(lines) + "\n")
    if a.json:
        try:
            cur = json.load(open(a.json))
        except Exception:
            cur = {}
        for spec in a.family:
            fam, sub = spec.split("=", 1)
            vals = [v for k, vs in per_kernel.items() if sub in k for v in vs]
            if vals:
                cur[fam] = sum(vals) / len(vals)
        json.dump(cur, open(a.json, "w"), indent=1)
    print(open(a.out).read()[:3000])


if __name__ == "__main__":
    main()
