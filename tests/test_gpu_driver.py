"""The experiment driver on the device path vs runs of the reference's own driver
(cli.py cmd_run, recorded by tests/golden/make_golden.py): same exit code, the
same manifest/row keys, per-point status, iterations within +-1 and the history
CSV columns (scalar V-cycles exact, r_P rtol 1e-6, r_true rtol 1e-5)."""

from __future__ import annotations

import json

import numpy as np
import pytest

from conftest import arr, cases

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("e", cases("driver"), ids=lambda e: e["name"])
def test_driver_matches_reference_runs(e, tmp_path):
    from paper_1308_4605_b200 import driver as D
    cfgf = tmp_path / "cfg.json"
    cfgf.write_text(json.dumps(e["config"]))
    out = tmp_path / "out"
    assert D.main(["run", "--config", str(cfgf), "--out", str(out)]) == e["exit_code"]
    man = json.loads((out / "manifest.json").read_text())
    assert sorted(man) == e["manifest_keys"]
    assert man["command"] == "run" and man["prng"] == "philox4x64-10"
    for ref, got in zip(e["runs"], man["runs"]):
        assert sorted(got) == e["row_keys"]
        for k in ("index", "file", "sweep_point", "seed", "status"):
            assert got[k] == ref[k], k
        assert abs(got["iterations"] - ref["iterations"]) <= 1
        text = (out / got["file"]).read_text().splitlines()
        assert text[0] == D.CSV_HEADER
        mine = np.array([[float(v) for v in ln.split(",")] for ln in text[1:]])
        want = arr(e["name"], f"run{ref['index']}")
        k = min(len(mine), len(want))
        assert np.array_equal(mine[:k, [0, 1, 4]], want[:k, [0, 1, 4]])
        assert np.allclose(mine[:k, 2], want[:k, 2], rtol=1e-6)
        assert np.allclose(mine[:k, 3], want[:k, 3], rtol=1e-5, atol=1e-12 * np.nan_to_num(want[0, 3]),
                           equal_nan=True)


def _golden_driver():
    from conftest import GOLD
    return json.loads((GOLD / "golden_driver.json").read_text())


def test_mg_bench_matches_reference(tmp_path):
    """``mg-bench`` (cli.py:391-452) on the device vs the reference driver's CSV:
    same rows (solver, sweeps, cycle), residual norms rtol 1e-9."""
    from paper_1308_4605_b200 import driver as D
    g = _golden_driver()["mg_bench"]
    cfgf = tmp_path / "cfg.json"
    cfgf.write_text(json.dumps(g["config"]))
    assert D.main(["mg-bench", "--config", str(cfgf), "--out", str(tmp_path)]) == g["exit_code"]
    got = (tmp_path / "mg_bench.csv").read_text().splitlines()
    want = g["csv"].splitlines()
    assert got[0] == want[0] == D.MG_CSV_HEADER and len(got) == len(want)
    for a, b in zip(got[1:], want[1:]):
        fa, fb = a.split(","), b.split(",")
        assert fa[:3] == fb[:3]
        assert np.allclose([float(x) for x in fa[3:]], [float(x) for x in fb[3:]], rtol=1e-9, atol=1e-300)
    man = json.loads((tmp_path / "manifest.json").read_text())
    assert man["command"] == "mg-bench" and man["runs"] == [{"file": "mg_bench.csv"}]


@pytest.mark.parametrize("k", [0, 1])
def test_spectrum_matches_reference(k, tmp_path):
    """``spectrum`` (cli.py:455-482; spectrum.py) on the device: eigenvalues at
    1e-9 of the largest, identical counts and histogram."""
    from paper_1308_4605_b200 import driver as D
    g = _golden_driver()["spectrum"][k]
    cfgf = tmp_path / "cfg.json"
    cfgf.write_text(json.dumps(g["config"]))
    assert D.main(["spectrum", "--config", str(cfgf), "--out", str(tmp_path)]) == g["exit_code"]
    rep = json.loads((tmp_path / "spectrum.json").read_text())
    ref = g["report"]
    lam, lr = np.array(rep["eigenvalues"]), np.array(ref["eigenvalues"])
    assert lam.shape == lr.shape
    assert np.abs(lam - lr).max() <= 1e-9 * np.abs(lr).max()
    for key in ("which", "n_dof", "n_eigenvalues", "zero_multiplicity", "nonpositive_count"):
        assert rep[key] == ref[key], key
    assert rep["frac_near_unit"] == pytest.approx(ref["frac_near_unit"], abs=0.02)


def test_exact_subsolver_preset_matches_reference(tmp_path):
    """The ``constant-periodic-steady`` preset's solver (P1 with dense exact
    subsolvers, device-factorised) at 16^2: one iteration, as the reference."""
    from paper_1308_4605_b200 import driver as D
    g = _golden_driver()["exact_run"]
    cfgf = tmp_path / "cfg.json"
    cfgf.write_text(json.dumps(g["config"]))
    assert D.main(["run", "--config", str(cfgf), "--out", str(tmp_path)]) == g["exit_code"]
    man = json.loads((tmp_path / "manifest.json").read_text())
    assert man["runs"][0]["iterations"] == g["iterations"]
    got = np.array([[float(v) for v in ln.split(",")] for ln in (tmp_path / man["runs"][0]["file"]).read_text().splitlines()[1:]])
    want = np.array([[float(v) for v in ln.split(",")] for ln in g["csv"].splitlines()[1:]])
    assert np.array_equal(got[:, [0, 1, 4]], want[:, [0, 1, 4]])
    assert np.allclose(got[0, 2:4], want[0, 2:4], rtol=1e-9)
    assert got[-1, 2] <= 1e-10 * got[0, 2]


def test_presets_run_on_device(tmp_path):
    """Every preset runs end to end on the device (the fig presets at their
    default size; fig6 reduced by a sweep override to keep the test short)."""
    from paper_1308_4605_b200 import driver as D
    for name in ("fig1-mg-sweeps", "fig7-spectrum", "constant-periodic-steady", "bubble-2d", "fig3-restarts"):
        cmd = D.PRESETS[name]["command"]
        assert D.main([cmd, "--preset", name, "--out", str(tmp_path / name)]) == 0, name
        assert (tmp_path / name / "manifest.json").exists()


def test_run_jobs_parallel_matches_serial(tmp_path):
    """``run --jobs 2`` (worker processes sharing the GPU, cli.py:376-378)
    writes the same histories as the serial run."""
    from paper_1308_4605_b200 import driver as D
    cfg = {"problem": {"kind": "bubble", "dim": 2, "cells": 32, "bc": "no_slip", "seed": 3},
           "solver": {"gmres": {"restart": 10, "rtol": 1e-9}},
           "sweep": {"solver.precond.kind": ["P1", "P2", "P3"]}}
    cfgf = tmp_path / "cfg.json"
    cfgf.write_text(json.dumps(cfg))
    assert D.main(["run", "--config", str(cfgf), "--out", str(tmp_path / "s")]) == 0
    assert D.main(["run", "--config", str(cfgf), "--out", str(tmp_path / "p"), "--jobs", "2"]) == 0
    for i in range(3):
        a = (tmp_path / "s" / f"run_{i:03d}.csv").read_text()
        b = (tmp_path / "p" / f"run_{i:03d}.csv").read_text()
        assert a == b
