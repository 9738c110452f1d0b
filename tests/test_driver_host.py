"""Experiment driver host logic (no GPU): config schema, sweep expansion and the
no-partial-output rule of the reference driver (cli.py:131-142, 263-289, 361-372),
checked against the reference driver's own runs recorded in tests/golden."""

from __future__ import annotations

import json

import pytest

from conftest import cases


@pytest.mark.parametrize("e", cases("driver"), ids=lambda e: e["name"])
def test_sweep_expansion_matches_reference(e):
    from paper_1308_4605_b200 import driver as D
    pts = D.sweep_points(json.loads(json.dumps(e["config"])))
    assert [p["_sweep_point"] for p in pts] == [r["sweep_point"] for r in e["runs"]]
    for p in pts:
        D.check_keys(p)
        D.problem_spec(p["problem"])
        D.make_solver(p.get("solver", {}))


def test_bad_configs_exit_2_without_outputs(tmp_path, capsys):
    from paper_1308_4605_b200 import driver as D
    bad = [
        {"problem": {"cels": 8}},                                     # typo'd key
        {"problem": {"cells": 7}},                                    # odd cells
        {"problem": {"bc": "wall"}},                                  # unknown bc
        {"solver": {"precond": {"kind": "P9"}}},                      # unknown preconditioner
        {"solver": {"device": "cpu"}},                                # device path only
        {"solver": {"precond": {"exact_subsolvers": True}}},          # dense study path
        {"sweep": {"problem.cells": []}},                             # empty sweep list
        {"problem": {"beta": -1.0}},
        {"problem": {"kind": "bubble", "bubble": {"r_mu": 0.5}}},      # contrast < 1
    ]
    for i, cfg in enumerate(bad):
        f = tmp_path / f"c{i}.json"
        f.write_text(json.dumps(cfg))
        out = tmp_path / f"out{i}"
        assert D.main(["run", "--config", str(f), "--out", str(out)]) == 2, cfg
        assert not out.exists()
    assert "error:" in capsys.readouterr().err
    assert D.main(["run", "--config", str(tmp_path / "missing.json"), "--out", str(tmp_path / "o")]) == 2


def test_history_csv_format():
    from paper_1308_4605_b200 import driver as D
    from paper_1308_4605_b200.krylov import ConvergenceHistory
    h = ConvergenceHistory()
    h.add(0, 3, 1.5, 2.25, False)
    h.add(1, 6, 0.1, float("nan"), True)
    assert D.history_csv(h) == (D.CSV_HEADER + "\n0,3,1.5,2.25,0\n1,6,0.1,nan,1\n")
