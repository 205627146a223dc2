"""Command line with the reference's flags and outputs (tools/main.cpp, src/config.cpp).

    python -m paper_2301_08911_b200.cli [--config file.json] [--key value ...] [--solver-mode M] [--device D]

The same keys, types and validation as parse_config (src/config.cpp:141-203): a JSON config file
first, flags on top (``--key value`` or ``--key=value``); unknown keys, malformed numbers and
out-of-range values raise. ``--init file:<path>`` starts from a float32 raw density. Outputs go to
``--out`` (default ./out): rho.raw, rho.meta.json, rho.vti, Ch.txt, log.csv, config.resolved.json.
``--workers`` is accepted for compatibility (no host worker pool on the GPU path). Two flags of
this build: ``--solver-mode vcycle|mixed_defect|pcg`` and ``--device``.
"""
from __future__ import annotations

import json
import sys

from . import PRECISION, SOLVER_MODE, RunConfig, run_optimization
from .io import import_density_raw, write_report

OBJECTIVES = ("bulk", "shear", "npr-relaxed", "npr-log")
SYMMETRIES = ("none", "reflect3", "reflect6", "rotate3")
KERNELS = ("linear", "spline4")
PLACEMENTS = ("density", "sensitivity")
STRINGS = {"obj", "kernel", "sym", "init", "out", "precision", "filter-placement", "solver-mode"}
INTS = {"reso", "basis-n", "seed", "max-iter", "max-cycles", "workers", "device"}
FLOATS = {"vol", "E", "nu", "beta", "eta", "tau", "gamma", "penal", "filter-radius", "step", "damp", "tol"}

USAGE = __doc__


class Options:
    """RunConfig + the fields the GPU RunConfig does not carry (init file, workers, out dir)."""

    def __init__(self):
        self.cfg = RunConfig(reso=64)
        self.init_file = ""
        self.workers = 0
        self.out_dir = "out"


def _lookup(choices, v, what):
    if v not in choices:
        raise ValueError(f"unknown {what}: {v}")
    return v


def _apply(o: Options, key: str, v) -> None:
    c = o.cfg
    simple = {"reso": "reso", "vol": "vol", "E": "youngs", "nu": "poisson", "beta": "beta", "eta": "eta",
              "tau": "tau", "gamma": "gamma", "penal": "penal", "filter-radius": "filter_radius",
              "basis-n": "basis_n", "seed": "seed", "max-iter": "max_iter", "step": "step", "damp": "damp",
              "tol": "tol", "max-cycles": "max_cycles", "device": "device"}
    if key in simple:
        setattr(c, simple[key], int(v) if key in INTS else float(v))
    elif key == "obj":
        c.obj = _lookup(OBJECTIVES, v, "objective")
    elif key == "kernel":
        c.kernel = _lookup(KERNELS, v, "kernel")
    elif key == "sym":
        c.sym = _lookup(SYMMETRIES, v, "symmetry")
    elif key == "filter-placement":
        c.filter_placement = _lookup(PLACEMENTS, v, "filter placement")
    elif key == "precision":
        c.precision = _lookup(("mixed", "double"), v, "precision")
    elif key == "solver-mode":
        c.solver_mode = _lookup(tuple(k for k in SOLVER_MODE), v, "solver mode")
    elif key == "init":
        if v in ("constant", "trig"):
            c.init = v
        elif v.startswith("file:"):
            if not v[5:]:
                raise ValueError("init file path is empty")
            c.init, o.init_file = "file", v[5:]
        else:
            raise ValueError(f"unknown init: {v} (constant | trig | file:<path>)")
    elif key == "workers":
        o.workers = int(v)
    elif key == "out":
        o.out_dir = str(v)
    else:
        raise ValueError(f"unknown config key: {key}")


def _validate(o: Options) -> None:  # src/config.cpp:61-78
    c = o.cfg
    checks = [(c.reso >= 4, "reso must be >= 4"), (0.0 < c.vol <= 1.0, "vol must lie in (0, 1]"),
              (c.youngs > 0.0, "E must be positive"), (-1.0 < c.poisson < 0.5, "nu must lie in (-1, 0.5)"),
              (c.penal >= 1.0, "penal must be >= 1"), (c.filter_radius >= 0.0, "filter-radius must be >= 0"),
              (c.max_iter >= 1, "max-iter must be >= 1"), (0.0 < c.step < 1.0, "step must lie in (0, 1)"),
              (0.0 < c.damp <= 1.0, "damp must lie in (0, 1]"), (c.tol > 0.0, "tol must be positive"),
              (c.max_cycles >= 1, "max-cycles must be >= 1"), (1 <= c.basis_n <= 8, "basis-n must lie in [1, 8]"),
              (o.workers >= 0, "workers must be >= 0")]
    for ok, msg in checks:
        if not ok:
            raise ValueError(msg)


def parse_config(argv) -> Options:
    """parse_config (src/config.cpp:141-203): config file first, then flags."""
    flags = {}
    i = 0
    while i < len(argv):
        a = argv[i]
        if not a.startswith("--"):
            raise ValueError(f"unexpected argument: {a}")
        a = a[2:]
        if "=" in a:
            a, value = a.split("=", 1)
        else:
            if i + 1 >= len(argv):
                raise ValueError(f"missing value for --{a}")
            i += 1
            value = argv[i]
        flags[a] = value
        i += 1
    o = Options()
    if "config" in flags:
        try:
            j = json.load(open(flags.pop("config")))
        except OSError as e:
            raise ValueError(f"cannot open config file: {e.filename}")
        for k, v in j.items():
            _apply(o, k, v)
    for k, v in flags.items():
        if k in STRINGS:
            _apply(o, k, v)
        elif k in INTS:
            try:
                iv = int(v)
            except ValueError:
                raise ValueError(f"invalid integer for --{k}: {v}")
            _apply(o, k, iv)
        elif k in FLOATS:
            try:
                fv = float(v)
            except ValueError:
                raise ValueError(f"invalid number for --{k}: {v}")
            _apply(o, k, fv)
        else:
            raise ValueError(f"unknown config key: {k}")
    _validate(o)
    assert o.cfg.precision in PRECISION
    return o


def main(argv=None) -> int:
    argv = sys.argv[1:] if argv is None else argv
    if any(a in ("--help", "-h") for a in argv):
        print(USAGE)
        return 0
    try:
        o = parse_config(argv)
        c = o.cfg
        print(f"grid {c.reso}^3  vol {c.vol:.3f}  obj {c.obj}  sym {c.sym}  precision {c.precision}  "
              f"solver {c.solver_mode}  device {c.device}")
        init = import_density_raw(o.init_file, c.reso) if c.init == "file" else None

        def observer(it, prev, nxt, C, rec):
            if it % 10 == 0:
                print(f"iter {rec['iter']:4d}  f {rec['objective']:.6g}  vol {rec['volume']:.4f}  "
                      f"cycles {rec['cycles']}  resid {rec['residual']:.3g}  {rec['ms']:.0f} ms")
            return True
        rep = run_optimization(c, observer, init_rho=init)
        write_report(rep, c, o.out_dir, o.init_file, o.workers)
        last = rep.records[-1]
        state = "converged" if rep.converged else (
            "solver failure (partial report written)" if rep.solver_failed else "stopped at max-iter")
        print(f"{state} after {len(rep.records)} iterations: f = {last['objective']:.8g}, "
              f"volume = {last['volume']:.5f}, poisson estimate = {rep.poisson_est:.4f}")
        if rep.init_fallback:
            print("warning: trig init bisection fell back to a constant field")
        if rep.oc_warning:
            print("warning: OC volume bisection hit its bracket")
        return 2 if rep.solver_failed else 0
    except Exception as e:  # noqa: BLE001 - the reference prints and exits 1
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
