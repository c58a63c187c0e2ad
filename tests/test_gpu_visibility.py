"""GPU visible fraction (visibility.py:46-115) against the reference's own
outputs (tests/golden/visibility.npz, grid 64).  The count is an integer of
grid^2 sample points; f64 projection rounding may move a sample lying on a
rect edge, so the bar is two points (2/4096) per pair, flags exact."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_visibility_matches_reference(golden, cuda_dev):
    from paper_2601_10819_b200 import ops

    g = golden("visibility")
    k = 0
    worst = 0.0
    while f"K{k}" in g:
        cams = ops.Cameras(g[f"K{k}"], g[f"R{k}"], g[f"t{k}"], device=cuda_dev)
        n_cams = g[f"K{k}"].shape[0]
        vis, behind = ops.visibility(cams, [[640, 480]] * n_cams, g[f"obj{k}"], grid=64)
        vis, behind = vis.cpu().numpy(), behind.cpu().numpy()
        np.testing.assert_array_equal(behind, g[f"behind{k}"])
        worst = max(worst, float(np.abs(vis - g[f"vis{k}"]).max()))
        k += 1
    assert k == 4
    assert worst <= 2.0 / 4096


def test_visibility_argument_errors(cuda_dev):
    from paper_2601_10819_b200 import ops

    cams = ops.Cameras([[100, 100, 64, 64]], np.eye(3).reshape(1, 9), [[0, 0, 0]], device=cuda_dev)
    with pytest.raises(ValueError):
        ops.visibility(cams, [[128, 128]], np.zeros((1, 7)), grid=1)
    vis, behind = ops.visibility(cams, [[128, 128]], [[0, 0, -5, 1, 1, 1, 0]], grid=8)
    assert bool(behind[0, 0]) and float(vis[0, 0]) == 0.0
    vis, _ = ops.visibility(cams, [[128, 128]], [[0, 0, 10, 1, 1, 1, 0]], grid=8)
    assert float(vis[0, 0]) == 1.0  # fully inside the image, no blockers
