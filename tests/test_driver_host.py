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
        {"problem": {"cells": 128}, "solver": {"precond": {"exact_subsolvers": True}}},  # dense cap
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


def test_presets_and_paper_scale(capsys):
    """The reference's nine presets (cli.py:494-598), --paper-scale (:621-623)
    and the preset/subcommand consistency check (:659-662)."""
    import argparse
    from paper_1308_4605_b200 import driver as D
    assert sorted(D.PRESETS) == ["bubble-2d", "constant-periodic-steady", "fig1-mg-sweeps", "fig2-vcycles",
                                 "fig3-restarts", "fig4-precond-compare", "fig5-cfl", "fig6-scaling",
                                 "fig7-spectrum"]
    assert D.main(["presets", "list"]) == 0
    assert "fig7-spectrum" in capsys.readouterr().out
    ns = lambda **k: argparse.Namespace(**{"config": None, "preset": None, "paper_scale": False, **k})
    cmd, cfg = D.load_config(ns(preset="fig4-precond-compare"))
    assert cmd == "run" and cfg["problem"]["cells"] == 128
    cmd, cfg = D.load_config(ns(preset="fig4-precond-compare", paper_scale=True))
    assert cfg["problem"]["cells"] == 512
    assert D.PRESETS["fig4-precond-compare"]["config"]["problem"]["cells"] == 128  # preset not mutated
    for name, p in D.PRESETS.items():
        cmd, cfg = D.load_config(ns(preset=name))
        D.check_keys(cfg)
        for pt in D.sweep_points(cfg):
            D.problem_spec(pt["problem"])
            if cmd == "run":
                D.make_solver(pt.get("solver", {}))
    with pytest.raises(D.ConfigError):
        D.load_config(ns())
    assert D.main(["mg-bench", "--preset", "fig4-precond-compare"]) == 2  # preset of another subcommand
    assert D.main(["run", "--preset", "nope"]) == 2
