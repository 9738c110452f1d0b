"""Debug: wave vs per-colour on the C4 16^3 golden case, component by component."""
import os
import sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from conftest import arr, cases, face, pkg_coeff, pkg_grid  # noqa
from paper_1308_4605_b200 import multigrid as MG, operators  # noqa
from paper_1308_4605_b200.grid import CellField, FaceField  # noqa

e = [x for x in cases("gmres") if x["name"] == "gm_C4_16_P1"][0]
g = pkg_grid(e)
c = pkg_coeff(e, grid=g)
print("bc", g.bc, "theta", c.theta, "form", c.viscous_form)
rng = np.random.default_rng(0)
x = [rng.standard_normal(g.face_shape(a)) for a in range(3)]
for a in range(3):
    if not g.periodic(a):
        x[a][(slice(None),) * a + (0,)] = 0.0
        x[a][(slice(None),) * a + (-1,)] = 0.0
r = [rng.standard_normal(g.face_shape(a)) for a in range(3)]
out = {}
for wm in ("4", "0"):
    os.environ["SB_WAVE_MIN"] = wm
    h = MG.build_hierarchy(g, c)
    s = MG.smooth(h, 0, "face", FaceField(g, tuple(a.copy() for a in x)), FaceField(g, tuple(r)), 1.0)
    v = MG.vcycle(FaceField(g, tuple(r)), h, MG.SmootherParams(), "face")
    out[wm] = ([np.array(a) for a in s.components], [np.array(a) for a in v.components])
for a in range(3):
    d1 = np.abs(out["4"][0][a] - out["0"][0][a]).max()
    d2 = np.abs(out["4"][1][a] - out["0"][1][a]).max()
    print("comp", a, "smooth diff", d1, "vcycle diff", d2)
    if d1 > 0:
        idx = np.argwhere(np.abs(out["4"][0][a] - out["0"][0][a]) > 0)
        print("  first bad", idx[:8].tolist(), len(idx))
