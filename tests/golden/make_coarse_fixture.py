"""Generates tests/golden/coarse_fail_npr128.npz: the coarsest-level (4^3, 192x192) operator and
load at which the reference algorithm's coarsest solve throws "coarsest operator is singular beyond
translations" (src/multigrid.cpp:446-447) on BASELINE configs[3]'s workload at 128^3 (npr-relaxed,
vol 0.2, mixed precision, reference defaults) -- iteration ~14 of the oracle loop.

It runs the oracle (oracle/, the CPU restatement) with the reference's unprojected operator
(set_coarse_project(False)) and the failure dump enabled; ~8 min on 8 cores.
    python tests/golden/make_coarse_fixture.py
"""
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402


def main():
    dump = os.path.join(tempfile.mkdtemp(), "coarse_fail.bin")
    oracle.set_coarse_project(False)
    oracle.set_coarse_dump(dump)
    try:
        oracle.run(reso=128, vol=0.2, obj="npr-relaxed", max_iter=30, mixed=True)
        raise SystemExit("the unprojected oracle loop did not fail; no fixture written")
    except oracle.OracleError as e:
        print("oracle failed as the reference does:", e)
    finally:
        oracle.set_coarse_dump(None)
        oracle.set_coarse_project(True)
    nv, n = np.fromfile(dump, dtype=np.int64, count=2)
    d = np.fromfile(dump, dtype=np.float64)[2:]
    raw, f = d[: n * n].reshape(n, n), d[n * n:]
    out = os.path.join(ROOT, "tests", "golden", "coarse_fail_npr128.npz")
    np.savez_compressed(out, raw=raw, f=f, nv=nv)
    print("wrote", out, raw.shape)


if __name__ == "__main__":
    main()
