"""GPU visible fraction (visibility.py:46-115) against the reference's own
outputs (tests/golden/visibility.npz, grid 64, 16 scenes / 1132 pairs).  The
value is an integer count of grid^2 sample points, so the bar is bitwise:
the device takes the yaw's cos / sin from the host libm and follows numpy's
(OpenBLAS) operation order in the corner and projection products."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_visibility_matches_reference(golden, cuda_dev):
    from paper_2601_10819_b200 import ops

    g = golden("visibility")
    k = 0
    while f"K{k}" in g:
        cams = ops.Cameras(g[f"K{k}"], g[f"R{k}"], g[f"t{k}"], device=cuda_dev)
        vis, behind = ops.visibility(cams, g[f"wh{k}"], g[f"obj{k}"], grid=64)
        vis, behind = vis.cpu().numpy(), behind.cpu().numpy()
        np.testing.assert_array_equal(behind, g[f"behind{k}"])
        # counts / 4096 are exact in f32: compare the integer counts
        np.testing.assert_array_equal(np.rint(vis.astype(np.float64) * 4096), np.rint(g[f"vis{k}"] * 4096), str(k))
        k += 1
    assert k == 16


def test_visibility_argument_errors(cuda_dev):
    from paper_2601_10819_b200 import ops

    cams = ops.Cameras([[100, 100, 64, 64]], np.eye(3).reshape(1, 9), [[0, 0, 0]], device=cuda_dev)
    with pytest.raises(ValueError):
        ops.visibility(cams, [[128, 128]], np.zeros((1, 7)), grid=1)
    vis, behind = ops.visibility(cams, [[128, 128]], [[0, 0, -5, 1, 1, 1, 0]], grid=8)
    assert bool(behind[0, 0]) and float(vis[0, 0]) == 0.0
    vis, _ = ops.visibility(cams, [[128, 128]], [[0, 0, 10, 1, 1, 1, 0]], grid=8)
    assert float(vis[0, 0]) == 1.0  # fully inside the image, no blockers
