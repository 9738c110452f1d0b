"""Host side of the inhomogeneous-wall API (no GPU): the BoundaryValues container
(operators.py:224-264) and boundary_lift (operators.py:471-481) against the
reference's golden vectors, plus the reference's shape check
(test_operators.py:597-601)."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import arr, cases, golden_bvals, pkg_grid


@pytest.mark.parametrize("e", cases("affine"), ids=lambda e: e["name"])
def test_boundary_lift_vs_golden(e):
    from paper_1308_4605_b200.operators import BoundaryValues, boundary_lift
    g = pkg_grid(e)
    normal, tang = golden_bvals(e)
    lift = boundary_lift(BoundaryValues(g, normal, tang))
    for a in range(g.dim):
        assert np.array_equal(lift.components[a], arr(e["name"], f"lift{a}"))


def test_boundary_value_shape_checked():
    from paper_1308_4605_b200.grid import NO_SLIP, GridSpec
    from paper_1308_4605_b200.operators import BoundaryValues
    g = GridSpec((4, 4), 0.25, ((NO_SLIP, NO_SLIP), (NO_SLIP, NO_SLIP)))
    with pytest.raises(ValueError, match="shape"):
        BoundaryValues(g, {(0, 0): np.zeros(3)}, {}).normal_values(0, 0)
    with pytest.raises(ValueError, match="shape"):
        BoundaryValues(g, {}, {(0, 0, 1): np.zeros(4)}).tangential_values(0, 0, 1)
    assert BoundaryValues.zeros(g).tangential_values(1, 1, 0).shape == (5,)
