"""The bench's per-case CPU reference legs (bench.py ``_cpu_ref_dense`` /
``_cpu_ref_oae``) run the UNMODIFIED reference from ``baseline/_ref``; here,
on small Sparse4D-layout inputs, they must reproduce the oracle: the
reference's ``msda_optimized(FULL)`` per channel group byte for byte against
the C oracle's dense restatement (SURVEY §8(c) "Groups G", "Dense Sparse4D
layout"), and the reference's OAE pooling (oae.py:81-164) against the numpy
oracle to 1e-12.  Skipped when the reference is not installed.
"""

import numpy as np
import pytest

import bench
from oracle import msda_oracle as mo
from tools import sparse4d_cases as s4

pytestmark = pytest.mark.skipif(bench.reference_features() is None, reason="baseline/_ref not installed")


def _scene(rng, cams, channels, levels=((16, 44), (8, 22), (4, 11), (2, 6))):
    tiles, r = [], 0
    for _ in range(cams):
        for h, w in levels:
            tiles.append((r, h, w))
            r += h * w
    table = rng.uniform(-1, 1, (r, channels)).astype(np.float32)
    shape = np.array([[list(x) for x in levels]] * cams, dtype=np.int32)
    return table, tiles, shape


@pytest.mark.parametrize("groups,channels", [(8, 256), (1, 64), (4, 64)])
def test_dense_reference_leg_matches_c_oracle(c_oracle, groups, channels):
    rng = np.random.default_rng(groups * 100 + channels)
    cams, q_n, p_n, levels = 3, 11, 5, 4
    table, tiles, shape = _scene(rng, cams, channels)
    loc = rng.uniform(-0.05, 1.05, (1, q_n, p_n, cams, 2)).astype(np.float32)  # some samples off the grid
    w = rng.uniform(0, 1, (1, q_n, p_n, cams, levels, groups)).astype(np.float32)
    ref = c_oracle.msda_dense_groups_c(table, tiles, shape, loc, w, levels, normalize=False)
    res = bench._cpu_ref_dense(table, tiles, shape, loc, w, ref)
    assert res["kind"] == "reference" and res["bitwise_equal_to_oracle"]


def test_oae_reference_leg_matches_numpy_oracle():
    rng = np.random.default_rng(7)
    cams, channels, q_n = 4, 32, 5
    strides = [4.0, 8.0, 16.0, 32.0]
    levels = [(64, 176), (32, 88), (16, 44), (8, 22)]
    table, tiles, _ = _scene(rng, cams, channels, levels)
    K, R, T = s4.ring(cams)
    anchors = np.zeros((q_n, 10))
    anchors[:, :2] = rng.uniform(-4, 4, (q_n, 2))
    anchors[:, 2] = 0.9
    anchors[:, 3:6] = (0.6, 0.6, 1.8)
    anchors[:, 6] = rng.uniform(-np.pi, np.pi, q_n)
    offs = rng.uniform(-1, 1, (6, 3))
    desc = rng.standard_normal((q_n, channels))
    vis = rng.uniform(0, 1, (q_n, cams))
    vis[2] = 1e-5  # all occluded: the memory fallback
    mem = rng.standard_normal((q_n, channels))
    mem /= np.linalg.norm(mem, axis=1, keepdims=True)
    emb = []
    for q in range(q_n):
        kps = mo.keypoints(anchors[q], offs)
        views = [mo.extract_view(table, tiles, 4, c, strides, K[c], R[c], T[c], kps, desc[q]) for c in range(cams)]
        emb.append(mo.fuse(views, vis[q], mem[q])[0])
    res = bench._cpu_ref_oae(table, tiles, K, R, T, strides, anchors, offs, desc, vis, mem, np.array(emb), nq=q_n)
    assert res["kind"] == "reference" and res["gpu_max_abs_err_on_sample"] <= 1e-12
