"""Goldens for the driver's mg-bench / spectrum / exact-subsolver paths, made by
the REFERENCE's own driver (``stokesmg.cli``):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_driver.py

* ``mg-bench`` (cli.py:391-452) on a small constant-coefficient no-slip grid,
  both targets, sweeps 1 and 2: the mg_bench.csv rows;
* ``spectrum`` (cli.py:455-482) of the fig7 preset (16^2 bubble, precondS)
  and of M on an 8^2 grid: the eigenvalues and the report statistics;
* ``run`` of the ``constant-periodic-steady`` preset (P1 with exact dense
  subsolvers) at 16^2: the history CSV.

Stored in ``tests/golden/golden_driver.json`` (small; text).
"""

from __future__ import annotations

import json
import pathlib
import sys
import tempfile

REF = pathlib.Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))

from stokesmg import cli  # noqa: E402

OUT = pathlib.Path(__file__).resolve().parent

MG_CFG = {"problem": {"kind": "constant", "dim": 2, "cells": 32, "bc": "no_slip", "beta": "inf", "seed": 4},
          "mg_bench": {"target": "both", "sweeps": [1, 2], "max_cycles": 8, "rtol": 1e-12}}
SPEC_CFGS = [
    {"problem": {"kind": "bubble", "dim": 2, "cells": 16, "bc": "no_slip", "beta": "inf", "seed": 0},
     "spectrum": {"which": "precondS"}},
    {"problem": {"kind": "bubble", "dim": 2, "cells": 8, "bc": "periodic", "beta": 1.0, "seed": 2},
     "spectrum": {"which": "M"}},
]
EXACT_CFG = {"problem": {"kind": "constant", "dim": 2, "cells": 16, "bc": "periodic", "beta": "inf", "seed": 0},
             "solver": {"precond": {"kind": "P1", "exact_subsolvers": True}, "gmres": {"rtol": 1e-10, "max_iters": 10}}}


def main():
    out = {}
    with tempfile.TemporaryDirectory() as d:
        rc = cli.cmd_mg_bench(json.loads(json.dumps(MG_CFG)), d)
        out["mg_bench"] = {"config": MG_CFG, "exit_code": rc,
                           "csv": (pathlib.Path(d) / "mg_bench.csv").read_text()}
    out["spectrum"] = []
    for cfg in SPEC_CFGS:
        with tempfile.TemporaryDirectory() as d:
            rc = cli.cmd_spectrum(json.loads(json.dumps(cfg)), d)
            rep = json.loads((pathlib.Path(d) / "spectrum.json").read_text())
            out["spectrum"].append({"config": cfg, "exit_code": rc, "report": rep})
    with tempfile.TemporaryDirectory() as d:
        rc = cli.cmd_run(json.loads(json.dumps(EXACT_CFG)), d, 1, None)
        man = json.loads((pathlib.Path(d) / "manifest.json").read_text())
        out["exact_run"] = {"config": EXACT_CFG, "exit_code": rc,
                            "csv": (pathlib.Path(d) / man["runs"][0]["file"]).read_text(),
                            "iterations": man["runs"][0]["iterations"]}
    (OUT / "golden_driver.json").write_text(json.dumps(out, indent=1))
    print("mg rows", out["mg_bench"]["csv"].count("\n"), "spectra", len(out["spectrum"]),
          "exact its", out["exact_run"]["iterations"])


if __name__ == "__main__":
    main()
