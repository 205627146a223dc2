"""Output files and the command line, after tests/test_io.cpp and
tests/test_config.cpp of the reference: byte layouts, round trips, JSON keys, flag parsing."""
import json
import os

import numpy as np
import pytest

from paper_2301_08911_b200 import io as pio
from paper_2301_08911_b200.cli import main, parse_config


def test_raw_export_constant_field_bytes(tmp_path):  # test_io.cpp:29-43
    p = tmp_path / "rho.raw"
    pio.export_density(np.full(64, 0.5), 4, str(p), "raw")
    b = p.read_bytes()
    assert len(b) == 256
    assert b == bytes([0x00, 0x00, 0x00, 0x3F]) * 64


def test_raw_round_trip_bit_exact(tmp_path):  # test_io.cpp:45-54
    f = np.random.default_rng(3).uniform(0, 1, 216).astype(np.float32).astype(np.float64)
    p = str(tmp_path / "r.raw")
    pio.export_density(f, (6, 6, 6), p, "raw")
    np.testing.assert_array_equal(pio.import_density_raw(p, (6, 6, 6)), f)
    with pytest.raises(RuntimeError):
        pio.import_density_raw(p, 8)  # too short
    with pytest.raises(RuntimeError):
        pio.import_density_raw(str(tmp_path / "missing.raw"), 4)


def test_vti_extents_and_cell_count(tmp_path):  # test_io.cpp:56-75
    f = np.random.default_rng(5).uniform(0, 1, 4 * 6 * 8)
    p = tmp_path / "rho.vti"
    pio.export_density(f, (4, 6, 8), str(p), "vti")
    text = p.read_text()
    assert 'WholeExtent="0 4 0 6 0 8"' in text and 'Piece Extent="0 4 0 6 0 8"' in text
    assert 'Spacing="0.25 0.166667 0.125"' in text
    body = text.split('format="ascii">\n')[1].split("\n        </DataArray>")[0]
    vals = body.split()
    assert len(vals) == f.size
    np.testing.assert_allclose([float(v) for v in vals], f, rtol=1e-6)
    assert body.count("\n") == f.size // 8


def test_tensor_round_trip_and_format(tmp_path):
    C = np.random.default_rng(7).normal(size=(6, 6)) * 1e5
    p = str(tmp_path / "Ch.txt")
    pio.export_tensor(C, p)
    lines = open(p).read().splitlines()
    assert len(lines) == 6 and all(len(line.split(" ")) == 6 for line in lines)
    np.testing.assert_array_equal(pio.import_tensor(p), C)  # %.17g round-trips a double exactly
    open(p, "w").write("1 2 3\n")
    with pytest.raises(RuntimeError):
        pio.import_tensor(p)


def test_meta_json(tmp_path):
    p = tmp_path / "rho.meta.json"
    pio.write_density_meta(8, str(p), 0.25, 11)
    j = json.loads(p.read_text())
    assert j == {"resolution": [8, 8, 8], "volume_fraction": 0.25, "seed": 11, "dtype": "float32",
                 "order": "x-fastest"}


def test_parse_config_flags_file_and_validation(tmp_path):
    o = parse_config(["--reso", "32", "--vol=0.2", "--obj", "npr-relaxed", "--sym", "reflect3",
                      "--init", "file:/x/rho.raw", "--out", str(tmp_path)])
    assert (o.cfg.reso, o.cfg.vol, o.cfg.obj, o.cfg.sym, o.cfg.init, o.init_file) == \
        (32, 0.2, "npr-relaxed", "reflect3", "file", "/x/rho.raw")
    cfgfile = tmp_path / "c.json"
    cfgfile.write_text(json.dumps({"reso": 16, "obj": "shear", "tol": 1e-3}))
    o = parse_config(["--config", str(cfgfile), "--reso", "24"])  # flags override the file
    assert (o.cfg.reso, o.cfg.obj, o.cfg.tol) == (24, "shear", 1e-3)
    for bad in (["--reso", "3"], ["--vol", "0"], ["--nu", "0.5"], ["--obj", "stiff"], ["--reso", "x"],
                ["--tol", "1e-2x"], ["--bogus", "1"], ["reso"], ["--reso"], ["--init", "file:"],
                ["--basis-n", "9"], ["--step", "1"]):
        with pytest.raises(ValueError):
            parse_config(bad)


def test_cli_errors_exit_1(capsys):
    assert main(["--reso", "2"]) == 1
    assert "error: reso must be >= 4" in capsys.readouterr().err
    assert main(["--help"]) == 0


@pytest.mark.gpu
def test_cli_end_to_end_writes_reference_outputs(tmp_path, orc):
    out = tmp_path / "out"
    rc = main(["--reso", "16", "--vol", "0.3", "--obj", "bulk", "--max-iter", "2", "--out", str(out)])
    assert rc == 0
    for name in ("rho.raw", "rho.meta.json", "rho.vti", "Ch.txt", "log.csv", "config.resolved.json"):
        assert (out / name).exists(), name
    rows = (out / "log.csv").read_text().splitlines()
    assert rows[0] == "iter,objective,volume,cycles,residual,ms" and len(rows) == 3
    recs, rho_o, _ = orc.run(reso=16, vol=0.3, obj="bulk", max_iter=2, mixed=True)
    obj = [float(r.split(",")[1]) for r in rows[1:]]
    for a, ro in zip(obj, recs):
        assert abs(a - ro["objective"]) <= 1e-4 * abs(ro["objective"])
    rho = pio.import_density_raw(str(out / "rho.raw"), 16)
    assert np.max(np.abs(rho - rho_o)) < 1e-3
    cfg = json.loads((out / "config.resolved.json").read_text())
    assert cfg["reso"] == 16 and cfg["obj"] == "bulk" and cfg["out"] == str(out)
    # restart from the written design (init file:)
    out2 = tmp_path / "out2"
    assert main(["--reso", "16", "--vol", "0.3", "--max-iter", "1", "--init", f"file:{out}/rho.raw",
                 "--out", str(out2)]) == 0
