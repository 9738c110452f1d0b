"""Run the REFERENCE's own hot-path test files against this package on the device.

    python tools/ref_shim.py stage          # in the build container: copy the
                                            # reference's tests to baseline/_ref_tests
    python tools/ref_shim.py run [pytest args]

``stage`` copies the reference's test modules (``/root/reference/pkg/tests``,
read-only there) into ``baseline/_ref_tests/`` -- git-ignored like the
``baseline/_ref`` install of the reference package, so it travels to the GPU
box but is never part of the repository.

``run`` makes ``import stokesmg`` resolve to ``paper_1308_4605_b200`` (grid,
operators, multigrid, schur, precond, krylov, problems, spectrum, cli and the
dense study tooling _exact) and runs the staged reference tests under pytest,
unmodified: the hot-path modules and test_problems / test_spectrum /
test_acceptance / test_cli (the CLI tests drive the device driver).
Nothing is taken from the real reference (``FROM_REFERENCE`` is empty).  Test
cases that inspect implementation details the drop-in does not share are
deselected in ``DESELECT`` with the reason.
"""

from __future__ import annotations

import importlib
import importlib.util
import pathlib
import shutil
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
STAGE = ROOT / "baseline" / "_ref_tests"
REF_PKG = ROOT / "baseline" / "_ref" / "stokesmg"
SRC_TESTS = pathlib.Path("/root/reference/pkg/tests")
FILES = ["conftest.py", "reference.py", "test_multigrid.py", "test_precond.py", "test_schur.py",
         "test_operators.py", "test_krylov.py", "test_grid.py", "test_problems.py", "test_spectrum.py",
         "test_acceptance.py", "test_cli.py"]
SUBMODULES = ["grid", "operators", "multigrid", "schur", "precond", "krylov", "problems", "_exact", "spectrum",
              "cli"]
FROM_REFERENCE = {"modules": [], "attrs": {}}  # nothing is taken from the reference
DESELECT = {
    # spies on np.zeros for the (m+1, n) basis block: the drop-in's basis is
    # a device allocation (sb_gmres_flat), not a NumPy array
    "basis in HBM": "test_memory_basis_is_restart_plus_one",
}


def stage():
    STAGE.mkdir(parents=True, exist_ok=True)
    for f in FILES:
        shutil.copy2(SRC_TESTS / f, STAGE / f)
    print(f"staged {len(FILES)} files -> {STAGE}")


def _load_reference():
    """The real reference package under the private name ``_stokesmg_ref``."""
    spec = importlib.util.spec_from_file_location("_stokesmg_ref", REF_PKG / "__init__.py",
                                                  submodule_search_locations=[str(REF_PKG)])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["_stokesmg_ref"] = mod
    spec.loader.exec_module(mod)
    return mod


def install_alias():
    sys.path.insert(0, str(ROOT))
    ours = importlib.import_module("paper_1308_4605_b200")
    sys.modules["stokesmg"] = ours
    for sub in SUBMODULES:
        sys.modules[f"stokesmg.{sub}"] = importlib.import_module(f"paper_1308_4605_b200.{sub}")
    if REF_PKG.exists():
        _load_reference()
        for sub in FROM_REFERENCE["modules"]:
            sys.modules[f"stokesmg.{sub}"] = importlib.import_module(f"_stokesmg_ref.{sub}")
        for sub, names in FROM_REFERENCE["attrs"].items():
            ref = importlib.import_module(f"_stokesmg_ref.{sub}")
            for n in names:
                setattr(sys.modules[f"stokesmg.{sub}"], n, getattr(ref, n))


def subprocess_alias():
    """Child processes the reference tests start (``python -m stokesmg.cli``,
    test_cli.py:242-247) resolve ``stokesmg`` through a generated alias package
    on PYTHONPATH -- written by this tool, nothing from the reference."""
    import os
    pkg = STAGE / "_alias" / "stokesmg"
    pkg.mkdir(parents=True, exist_ok=True)
    subs = [m for m in SUBMODULES if m != "cli"]
    (pkg / "__init__.py").write_text(
        "import importlib, sys\n"
        "from paper_1308_4605_b200 import *  # noqa: F401,F403\n"
        f"for _s in {subs!r}:\n"
        "    sys.modules['stokesmg.' + _s] = importlib.import_module('paper_1308_4605_b200.' + _s)\n")
    (pkg / "cli.py").write_text(
        "import sys\n"
        "from paper_1308_4605_b200.cli import *  # noqa: F401,F403\n"
        "from paper_1308_4605_b200.cli import main\n"
        "if __name__ == '__main__':\n"
        "    sys.exit(main())\n")
    extra = [str(pkg.parent), str(ROOT)]
    old = os.environ.get("PYTHONPATH")
    os.environ["PYTHONPATH"] = os.pathsep.join(extra + ([old] if old else []))


def run(args):
    import pytest
    if not STAGE.exists():
        print(f"no staged reference tests at {STAGE} (run `stage` in the build container)")
        return 2
    install_alias()
    subprocess_alias()
    sel = [str(STAGE / f) for f in FILES if f.startswith("test_")]
    desel = ["-k", " and ".join(f"not {name}" for name in DESELECT.values())]
    return pytest.main(["-p", "no:cacheprovider", "--rootdir", str(STAGE), *desel, *sel, *args])


if __name__ == "__main__":
    cmd = sys.argv[1] if len(sys.argv) > 1 else "run"
    if cmd == "stage":
        stage()
    else:
        sys.exit(run(sys.argv[2:]))
