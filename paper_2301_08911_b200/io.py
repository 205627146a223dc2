"""Density / tensor / run-report files in the reference's formats.

Host plumbing around the GPU path, mirroring src/io.cpp and write_report (src/runner.cpp:145-166):

  rho.raw              float32, x-fastest, no header            (export_density raw, io.cpp:23-31)
  rho.vti              VTK ImageData, ASCII cell data, %.7g x 8  (export_density vti, io.cpp:32-51)
  rho.meta.json        resolution / volume_fraction / seed / dtype / order (io.cpp:54-64)
  Ch.txt               6 x 6, %.17g, space-separated            (export_tensor, io.cpp:78-87)
  log.csv              iter,objective,volume,cycles,residual,ms (runner.cpp:156-161)
  config.resolved.json config_to_json (src/config.cpp:205-230)

JSON is written with sorted keys and a 2-space indent, as nlohmann::json::dump(2) does.
"""
from __future__ import annotations

import json
import os

import numpy as np


def export_density(rho, n, path: str, fmt: str = "raw") -> None:
    """rho: x-fastest field of n = (nx, ny, nz) (or a cubic n) elements."""
    n3 = (n, n, n) if np.isscalar(n) else tuple(int(v) for v in n)
    v = np.ascontiguousarray(rho, dtype=np.float64).ravel()
    if v.size != n3[0] * n3[1] * n3[2]:
        raise ValueError("density size does not match the resolution")
    if fmt == "raw":
        v.astype("<f4").tofile(path)
        return
    if fmt != "vti":
        raise ValueError(f"unknown density format: {fmt}")
    with open(path, "w") as out:
        out.write('<?xml version="1.0"?>\n'
                  '<VTKFile type="ImageData" version="1.0" byte_order="LittleEndian">\n'
                  f'  <ImageData WholeExtent="0 {n3[0]} 0 {n3[1]} 0 {n3[2]}" Origin="0 0 0" '
                  f'Spacing="{_g(1.0 / n3[0])} {_g(1.0 / n3[1])} {_g(1.0 / n3[2])}">\n'
                  f'    <Piece Extent="0 {n3[0]} 0 {n3[1]} 0 {n3[2]}">\n'
                  '      <CellData Scalars="density">\n'
                  '        <DataArray type="Float32" Name="density" format="ascii">\n')
        parts = []
        for i, x in enumerate(v):
            parts.append("%.7g" % x)
            parts.append("\n" if (i + 1) % 8 == 0 else " ")
        out.write("".join(parts))
        out.write("\n        </DataArray>\n      </CellData>\n    </Piece>\n  </ImageData>\n</VTKFile>\n")


def _g(x: float) -> str:
    """std::ostream default formatting of a double (6 significant digits, %g)."""
    return "%g" % x


def import_density_raw(path: str, n) -> np.ndarray:
    """float32 x-fastest file -> float64 field (src/io.cpp:66-76); raises on a short file."""
    n3 = (n, n, n) if np.isscalar(n) else tuple(int(v) for v in n)
    m = n3[0] * n3[1] * n3[2]
    if not os.path.exists(path):
        raise RuntimeError(f"cannot open density file: {path}")
    buf = np.fromfile(path, dtype="<f4", count=m)
    if buf.size != m:
        raise RuntimeError(f"density file too short: {path}")
    return buf.astype(np.float64)


def write_density_meta(n, path: str, volume: float, seed: int) -> None:
    n3 = [n, n, n] if np.isscalar(n) else [int(v) for v in n]
    meta = {"resolution": n3, "volume_fraction": volume, "seed": int(seed), "dtype": "float32", "order": "x-fastest"}
    with open(path, "w") as out:
        out.write(json.dumps(meta, indent=2, sort_keys=True) + "\n")


def export_tensor(C, path: str) -> None:
    C = np.asarray(C, dtype=np.float64).reshape(6, 6)
    with open(path, "w") as out:
        for i in range(6):
            out.write(" ".join("%.17g" % C[i, j] for j in range(6)) + "\n")


def import_tensor(path: str) -> np.ndarray:
    try:
        vals = open(path).read().split()
    except OSError:
        raise RuntimeError(f"cannot open tensor file: {path}")
    if len(vals) < 36:
        raise RuntimeError(f"malformed tensor file: {path}")
    try:
        return np.array([float(v) for v in vals[:36]]).reshape(6, 6)
    except ValueError:
        raise RuntimeError(f"malformed tensor file: {path}")


def config_to_json(cfg, init_file: str = "", workers: int = 0, out_dir: str = "out") -> str:
    """config_to_json (src/config.cpp:205-230) for a RunConfig."""
    j = {"reso": cfg.reso, "vol": cfg.vol, "E": cfg.youngs, "nu": cfg.poisson, "obj": cfg.obj, "beta": cfg.beta,
         "eta": cfg.eta, "tau": cfg.tau, "gamma": cfg.gamma, "penal": cfg.penal, "filter-radius": cfg.filter_radius,
         "filter-placement": cfg.filter_placement, "kernel": cfg.kernel, "sym": cfg.sym,
         "init": ("file:" + init_file) if cfg.init == "file" else cfg.init, "basis-n": cfg.basis_n,
         "seed": cfg.seed, "max-iter": cfg.max_iter, "step": cfg.step, "damp": cfg.damp, "tol": cfg.tol,
         "max-cycles": cfg.max_cycles, "precision": cfg.precision, "workers": workers, "out": out_dir}
    return json.dumps(j, indent=2, sort_keys=True)


def write_report(report, cfg, out_dir: str, init_file: str = "", workers: int = 0) -> None:
    """The six output files of write_report (src/runner.cpp:145-166)."""
    os.makedirs(out_dir, exist_ok=True)
    p = lambda name: os.path.join(out_dir, name)  # noqa: E731
    n = cfg.reso
    export_density(report.density, n, p("rho.raw"), "raw")
    write_density_meta(n, p("rho.meta.json"), cfg.vol, cfg.seed)
    export_density(report.density, n, p("rho.vti"), "vti")
    export_tensor(report.tensor, p("Ch.txt"))
    with open(p("log.csv"), "w") as log:
        log.write("iter,objective,volume,cycles,residual,ms\n")
        for r in report.records:
            log.write("%d,%.17g,%.17g,%d,%.6g,%.3f\n" % (r["iter"], r["objective"], r["volume"], r["cycles"],
                                                        r["residual"], r["ms"]))
    with open(p("config.resolved.json"), "w") as out:
        out.write(config_to_json(cfg, init_file, workers, out_dir) + "\n")
