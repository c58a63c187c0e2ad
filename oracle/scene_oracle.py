"""CPU oracle for the two SURVEY §8(f) components either side of the MSDA path:
feature painting (the producer of the pyramids MSDA reads) and the tracker's
association cost (the consumer of the pooled embeddings).

TEST INFRASTRUCTURE ONLY: imported by tests/ (and never by the product
package).  Every function restates the reference with numpy, in the
reference's own operation order, and cites the lines it follows (paths
relative to /root/reference/pkg/src/mvtrack3d/).  Pinned against outputs of
the real reference: tests/golden/paint.npz and tests/golden/assoc.npz
(tests/golden/make_golden.py), checked by tests/test_oracle_golden.py.
"""

from __future__ import annotations

import hashlib
import math

import numpy as np

# --------------------------------------------------------------------------
# rng.py:19-30 — substream(seed, *labels)


def _label_to_int(label) -> int:
    """rng.py:19-24: ints masked to 64 bits, strings -> BLAKE2b-64 little endian."""
    if isinstance(label, (int, np.integer)):
        return int(label) & 0xFFFFFFFFFFFFFFFF
    if isinstance(label, str):
        return int.from_bytes(hashlib.blake2b(label.encode("utf-8"), digest_size=8).digest(), "little")
    raise TypeError(f"labels must be int or str, got {type(label).__name__}")


def substream(seed: int, *labels) -> np.random.Generator:
    """rng.py:26-30: numpy PCG64 seeded by SeedSequence([seed, *labels])."""
    entropy = [int(seed) & 0xFFFFFFFFFFFFFFFF] + [_label_to_int(x) for x in labels]
    return np.random.default_rng(np.random.SeedSequence(entropy))


def paint_background(seed, frame, cam_id, level, sigma, shape):
    """simulator.py:256-257: the f64 Gaussian background of one grid."""
    return substream(seed, "paint", frame, cam_id, level).normal(0.0, sigma, size=shape)


def identity_signature(seed, identity, dim):
    """simulator.py:191-195: unit-norm standard-normal appearance vector."""
    raw = substream(seed, "signature", identity).standard_normal(dim)
    return raw / np.linalg.norm(raw)


# --------------------------------------------------------------------------
# geometry.py:50-53, 162-182, 195-204; visibility.py:46-65


def rot_z(yaw):
    c, s = math.cos(yaw), math.sin(yaw)
    return np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])


def box_corners(state):
    """geometry.py:195-204; state = (x, y, z, w, l, h, yaw)."""
    x, y, z, w, l, h, yaw = (float(v) for v in state[:7])
    signs = np.array([[(i >> b) & 1 for b in range(3)] for i in range(8)], dtype=float) * 2.0 - 1.0
    local = signs * np.array([l / 2.0, w / 2.0, h / 2.0])
    return local @ rot_z(yaw).T + np.array([x, y, z])


def projected_rect(K, R, t, state, eps=1e-6):
    """visibility.py:46-65 (corners behind the camera skipped, geometry.py:162-182).

    Returns (u_min, u_max, v_min, v_max, mean_depth) or None (fully behind)."""
    R = np.asarray(R, dtype=float).reshape(3, 3)
    t = np.asarray(t, dtype=float).reshape(3)
    us, vs, ds = [], [], []
    for corner in box_corners(state):
        p = R @ np.asarray(corner, dtype=float).reshape(3) + t
        d = p[2]
        if d <= eps:
            continue
        us.append(float(K[0] * p[0] / d + K[2]))
        vs.append(float(K[1] * p[1] / d + K[3]))
        ds.append(float(d))
    if not us:
        return None
    return (min(us), max(us), min(vs), max(vs), float(np.mean(ds)))


def visible_fraction(K, R, t, width, height, objects, target, grid=64):
    """visibility.py:68-115 for one (camera, target object): (value, fully_behind)."""
    rect = projected_rect(K, R, t, objects[target])
    if rect is None:
        return 0.0, True
    blockers = []
    for o, obj in enumerate(objects):
        if o == target:
            continue
        br = projected_rect(K, R, t, obj)
        if br is not None and br[4] < rect[4]:
            blockers.append(br)
    steps = (np.arange(grid, dtype=float) + 0.5) / grid
    us = rect[0] + steps * (rect[1] - rect[0])
    vs = rect[2] + steps * (rect[3] - rect[2])
    uu, vv = np.meshgrid(us, vs)
    visible = (uu >= 0.0) & (uu < width) & (vv >= 0.0) & (vv < height)
    for br in blockers:
        visible &= ~((br[0] <= uu) & (uu <= br[1]) & (br[2] <= vv) & (vv <= br[3]))
    return float(np.count_nonzero(visible)) / float(grid * grid), False


def paint_grid(K, R, t, image_wh, stride, entities, signatures, background):
    """simulator.py:249-289 for one (camera, level) grid.

    entities: states [n, 7], moving objects first then occluders (the order
    _paint_grid builds `rects` in); signatures: list aligned with entities,
    None for occluders.  background: f64 (H, W, C).  Returns f32 (H, W, C)."""
    height, width = background.shape[:2]
    values = background.copy()
    rects = []
    for st, sig in zip(entities, signatures):
        r = projected_rect(K, R, t, st)
        if r is not None:
            rects.append((r, sig))
    if rects:
        uu = (np.arange(width, dtype=float) + 0.5) * stride
        vv = (np.arange(height, dtype=float) + 0.5) * stride
        uu, vv = np.meshgrid(uu, vv)
        best = np.full((height, width), np.inf)
        winner = np.full((height, width), -1, dtype=np.int64)
        for idx, (r, _) in enumerate(rects):
            inside = (r[0] <= uu) & (uu <= r[1]) & (r[2] <= vv) & (vv <= r[3]) & (r[4] < best)
            best[inside] = r[4]
            winner[inside] = idx
        for idx, (_, sig) in enumerate(rects):
            if sig is None:
                continue
            mask = winner == idx
            if mask.any():
                values[mask] += sig
    return values.astype(np.float32)


def grid_dims(image_wh, stride):
    """simulator.py:252-253: ceil(H / stride) x ceil(W / stride)."""
    return int(math.ceil(image_wh[1] / stride)), int(math.ceil(image_wh[0] / stride))


# --------------------------------------------------------------------------
# tracker.py:105-142 — the association cost matrices (the Hungarian solve
# itself, scipy.optimize.linear_sum_assignment, is not restated)

INADMISSIBLE = 1e9  # tracker.py _INADMISSIBLE


def _pairwise_sum(a):
    """numpy's float64 add.reduce on a contiguous row (pairwise_sum of
    numpy/_core/src/umath/loops_utils.h.src): sequential below 8 elements,
    8 running partial sums combined as ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7))
    up to 128, then the remainder sequentially; halves above 128."""
    n = len(a)
    if n < 8:
        res = 0.0
        for x in a:
            res = res + float(x)
        return res
    if n <= 128:
        r = [float(x) for x in a[:8]]
        i = 8
        while i < n - (n % 8):
            for j in range(8):
                r[j] = r[j] + float(a[i + j])
            i += 8
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        while i < n:
            res = res + float(a[i])
            i += 1
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return _pairwise_sum(a[:n2]) + _pairwise_sum(a[n2:])


def norm_rows(diff):
    """np.linalg.norm(diff, axis=-1) for real f64 (linalg: sqrt(add.reduce(x*x)))."""
    sq = diff * diff
    flat = sq.reshape(-1, sq.shape[-1])
    return np.sqrt(np.array([_pairwise_sum(row) for row in flat])).reshape(sq.shape[:-1])


def association_cost(q_centers, d_centers, q_emb, d_emb, gate_radius, alpha_emb, alpha_geo):
    """tracker.py:119-128: (cost, solver_cost, admissible), all [n_q, n_d]."""
    q_centers = np.asarray(q_centers, dtype=float)
    d_centers = np.asarray(d_centers, dtype=float)
    q_emb = np.asarray(q_emb, dtype=float)
    d_emb = np.asarray(d_emb, dtype=float)
    geo = norm_rows(q_centers[:, None, :] - d_centers[None, :, :])
    emb = norm_rows(q_emb[:, None, :] - d_emb[None, :, :])
    admissible = geo <= gate_radius
    gate = gate_radius if np.isfinite(gate_radius) else 1.0
    cost = alpha_emb * emb + alpha_geo * geo / gate
    return cost, np.where(admissible, cost, INADMISSIBLE), admissible
