"""Seeded input generators shared by the tests and tests/golden/make_golden.py.

They restate the reference test generators so the same seeds produce the
same inputs: ``make_pyramids`` / ``make_plan`` (reference
pkg/tests/test_features.py:21-56) and ``tiny_workload`` (criterion 1,
pkg/tests/test_acceptance.py:56-91).  Grids are returned as
``{(cam, level): (H, W, C) float32}`` and plans as per-query tuple lists
``(cam, level, u, v, w)``.
"""

from __future__ import annotations

import numpy as np


def make_pyramids(rng, n_cams=2, n_levels=2, channels=4, size_lo=3, size_hi=9):
    grids, strides = {}, []
    for cam in range(n_cams):
        stride = 4.0
        for lvl in range(n_levels):
            h = int(rng.integers(size_lo, size_hi))
            w = int(rng.integers(size_lo, size_hi))
            grids[(cam, lvl)] = rng.standard_normal((h, w, channels)).astype(np.float32)
            if cam == 0:
                strides.append(stride)
            stride *= 2.0
    return grids, strides


def make_plan(rng, grids, n_queries, samples_lo=1, samples_hi=9, margin=2.0):
    keys = list(grids)
    per_query = []
    for _ in range(n_queries):
        samples = []
        for _ in range(int(rng.integers(samples_lo, samples_hi))):
            cam, lvl = keys[int(rng.integers(0, len(keys)))]
            h, w, _ = grids[(cam, lvl)].shape
            samples.append((cam, lvl, float(rng.uniform(-margin, w - 1 + margin)),
                            float(rng.uniform(-margin, h - 1 + margin)), float(rng.uniform(0.05, 1.0))))
        per_query.append(samples)
    return per_query


def tiny_workload(rng):
    n_cams = int(rng.integers(1, 3))
    n_levels = int(rng.integers(1, 3))
    channels = int(rng.integers(1, 3)) * 2
    grids, shapes = {}, {}
    for cam in range(n_cams):
        for lvl in range(n_levels):
            h = int(rng.integers(2, 5))
            w = int(rng.integers(2, 5))
            grids[(cam, lvl)] = rng.uniform(-1.0, 1.0, size=(h, w, channels)).astype(np.float32)
            shapes[(cam, lvl)] = (h, w)
    per_query = []
    for _ in range(int(rng.integers(1, 4))):
        samples = []
        for _ in range(int(rng.integers(1, 7))):
            cam = int(rng.integers(0, n_cams))
            lvl = int(rng.integers(0, n_levels))
            h, w = shapes[(cam, lvl)]
            samples.append((cam, lvl, float(rng.uniform(-1.0, w)), float(rng.uniform(-1.0, h)),
                            float(rng.uniform(0.05, 1.0))))
        per_query.append(samples)
    return grids, n_cams, n_levels, per_query


def make_dense(rng, bs=1, n_q=5, n_p=3, cams=2, n_levels=2, groups=2, channels=8, size_lo=3, size_hi=9,
               loc_lo=-0.1, loc_hi=1.1):
    """Sparse4D-layout inputs: grids, spatial_shape [cams, L, 2], locations, weights."""
    grids = {}
    shape = np.zeros((cams, n_levels, 2), dtype=np.int32)
    for c in range(cams):
        for lvl in range(n_levels):
            h = int(rng.integers(size_lo, size_hi))
            w = int(rng.integers(size_lo, size_hi))
            grids[(c, lvl)] = rng.uniform(-1.0, 1.0, size=(h, w, channels)).astype(np.float32)
            shape[c, lvl] = (h, w)
    loc = rng.uniform(loc_lo, loc_hi, size=(bs, n_q, n_p, cams, 2)).astype(np.float32)
    logits = rng.standard_normal((bs, n_q, n_p * cams * n_levels, groups))
    e = np.exp(logits - logits.max(axis=2, keepdims=True))
    wts = (e / e.sum(axis=2, keepdims=True)).reshape(bs, n_q, n_p, cams, n_levels, groups).astype(np.float32)
    return grids, shape, loc, wts


def bilinear_inputs(rng, n_grids=4, n_coords=200):
    """Grids and (u, v) cell coordinates for bilinear_sample fixtures: random
    coordinates over [-2, W+1] x [-2, H+1], exact integers (cell centres),
    the last row/column, halves, and values just outside the grid."""
    grids, coords = [], []
    for k in range(n_grids):
        h, w, c = int(rng.integers(2, 12)), int(rng.integers(2, 12)), 2 * int(rng.integers(1, 40))
        grid = rng.standard_normal((h, w, c)).astype(np.float32)
        if k == 0:
            grid[0, 0] = -0.0  # signed zeros in the grid
        us = rng.uniform(-2.0, w + 1.0, n_coords).astype(np.float32)
        vs = rng.uniform(-2.0, h + 1.0, n_coords).astype(np.float32)
        special_u = np.array([0, w - 1, w - 1, -1, -0.5, w - 0.5, 0.5, -1e-7, w - 1 + 1e-6, 3.0], np.float32)
        special_v = np.array([0, h - 1, 0, -1, -0.5, h - 0.5, 0.5, -1e-7, h - 1 + 1e-6, -0.0], np.float32)
        grids.append(grid)
        coords.append((np.concatenate([us, special_u]), np.concatenate([vs, special_v])))
    return grids, coords


def per_query_hash(per_query) -> str:
    import hashlib

    h = hashlib.sha256()
    for samples in per_query:
        h.update(np.array([len(samples)], dtype=np.int64).tobytes())
        for c, m, u, v, w in samples:
            h.update(np.array([c, m], dtype=np.int32).tobytes())
            h.update(np.array([u, v, w], dtype=np.float64).tobytes())
    return h.hexdigest()
