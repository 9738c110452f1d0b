"""The reference's ``stokesmg.cli`` names on the device driver.

``paper_1308_4605_b200.driver`` implements the reference CLI's subcommands
(``run``, ``mg-bench``, ``spectrum``, ``presets``; ``cli.py:332-623``) on the
B200 path; this module re-exports it under the names the reference's own
``tests/test_cli.py`` and user scripts import (``cli.py:75, 118-330``), so
``python -m paper_1308_4605_b200.cli ...`` and ``from stokesmg.cli import main``
(through ``tools/ref_shim.py``) drive the device solver unchanged.
"""

from __future__ import annotations

import sys

from .driver import (CSV_HEADER, PRESETS, ConfigError, check_keys, main, make_grid, make_problem, make_solver,
                     sweep_points)

# reference spellings (cli.py): validate_keys :121, build_grid :139, build_problem :182,
# build_solver :226, expand_sweep :262
validate_keys = check_keys
build_grid = make_grid
build_problem = make_problem
build_solver = make_solver
expand_sweep = sweep_points

__all__ = ["CSV_HEADER", "PRESETS", "ConfigError", "build_grid", "build_problem", "build_solver", "expand_sweep",
           "main", "validate_keys"]

if __name__ == "__main__":
    sys.exit(main())
