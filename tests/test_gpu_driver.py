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
