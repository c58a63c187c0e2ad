"""TEST INFRASTRUCTURE ONLY — numpy restatement of the reference MSDA path.

Every function cites the reference line range it restates (paths relative to
``/root/reference/pkg/src/mvtrack3d/``).  Only ``tests/``, ``__graft_entry__``
(smoke check) and ``bench.py`` (cpu_baseline / ``--impl reference``) may use
this module; the product package never imports it.

Data layout used throughout (the same layout the GPU consumes, so the oracle
also checks the layout mapping):

* ``table``   — feature rows ``[R, C]``: every (camera, level) grid
  ``(H, W, C)`` row-major, concatenated camera-major then level-minor.
* ``tiles``   — per tile ``t = cam * n_levels + level``: ``(start_row, H, W)``.
* CSR plan    — ``offsets`` int64[Q+1], ``cam`` int32[S] (dense camera
  index, ascending camera id), ``lvl`` int32[S], ``u``/``v``/``w`` f32[S].

Parity: pinned against fixtures produced by the real reference
(``tests/golden/make_golden.py`` → ``tests/test_oracle_golden.py``).
"""

from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np

F32 = np.float32
F16 = np.float16
_ONE = np.float32(1.0)


# --------------------------------------------------------------------------
# layout helpers


def pack_grids(grids: dict, n_cams: int, n_levels: int, dtype=np.float32):
    """(cam, level) -> (H, W, C) grids  →  (table [R, C], tiles list).

    Layout of ``FeatureGrid.values`` (features.py:54-80) concatenated in
    camera-id then level order (the order ``_check_plan_targets`` and the
    canonical sort see, features.py:222-238, 261-263).
    """
    rows, tiles, start = [], [], 0
    for cam in range(n_cams):
        for lvl in range(n_levels):
            g = np.ascontiguousarray(grids[(cam, lvl)])
            h, w, c = g.shape
            rows.append(g.reshape(h * w, c))
            tiles.append((start, h, w))
            start += h * w
    return np.concatenate(rows, axis=0).astype(dtype, copy=False), tiles


def csr_from_per_query(per_query):
    """Per-query tuple lists → CSR arrays (SamplePlan.__init__, features.py:122-141)."""
    counts = [len(s) for s in per_query]
    offsets = np.zeros(len(counts) + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    flat = [t for s in per_query for t in s]
    cam = np.array([t[0] for t in flat], dtype=np.int32)
    lvl = np.array([t[1] for t in flat], dtype=np.int32)
    u = np.array([t[2] for t in flat], dtype=np.float32)
    v = np.array([t[3] for t in flat], dtype=np.float32)
    w = np.array([t[4] for t in flat], dtype=np.float32)
    return offsets, cam, lvl, u, v, w


# --------------------------------------------------------------------------
# scalar semantics (msda_reference)


def canonical_order(cam, lvl, u, v, w):
    """Per-query visiting order: lexicographic (camera, level, v, u, weight).

    Restates features.py:261-263 (np.lexsort, last key primary, stable).
    """
    return np.lexsort((w, u, v, lvl, cam))


def bilinear_f32(table, tile, u, v):
    """Zero-padded bilinear lookup, float32, fixed expression tree.

    Restates features.py:184-219: floor, fractional parts, four f32 products,
    ``((c00*w00 + c10*w10) + (c01*w01 + c11*w11))``; neighbours outside
    ``[0, W-1] x [0, H-1]`` read as zero.
    """
    start, h, w = tile
    uu, vv = F32(u), F32(v)
    x0f, y0f = np.floor(uu), np.floor(vv)
    fu, fv = uu - x0f, vv - y0f
    omu, omv = _ONE - fu, _ONE - fv
    wts = (omu * omv, fu * omv, omu * fv, fu * fv)
    zero = np.zeros(table.shape[1], dtype=np.float32)

    def cell(yf, xf):
        if 0.0 <= xf <= w - 1 and 0.0 <= yf <= h - 1:
            return table[start + int(yf) * w + int(xf)].astype(np.float32)
        return zero

    c = (cell(y0f, x0f), cell(y0f, x0f + 1), cell(y0f + 1, x0f), cell(y0f + 1, x0f + 1))
    return (c[0] * wts[0] + c[1] * wts[1]) + (c[2] * wts[2] + c[3] * wts[3])


def check_targets(tiles, n_levels, cam, lvl):
    """Unknown camera / missing level → ValueError (features.py:231-238)."""
    n_cams = len(tiles) // n_levels
    if cam.size and (cam.min() < 0 or cam.max() >= n_cams or lvl.min() < 0 or lvl.max() >= n_levels):
        raise ValueError("plan references an unknown camera or a missing level")


def msda_exact(table, tiles, n_levels, offsets, cam, lvl, u, v, w, normalize=True):
    """Scalar MSDA in canonical order, all float32.

    Restates ``msda_reference`` (features.py:241-276): per query, canonical
    lexsort, sequential f32 weight sum (zero → ValueError), then
    ``acc += (w / wsum) * bilinear`` in that order.  Empty queries give a
    zero row and ``empty=True``.
    """
    check_targets(tiles, n_levels, cam, lvl)
    q_n = len(offsets) - 1
    c_n = table.shape[1]
    out = np.zeros((q_n, c_n), dtype=np.float32)
    empty = np.zeros(q_n, dtype=bool)
    for q in range(q_n):
        lo, hi = int(offsets[q]), int(offsets[q + 1])
        if lo == hi:
            empty[q] = True
            continue
        order = lo + canonical_order(cam[lo:hi], lvl[lo:hi], u[lo:hi], v[lo:hi], w[lo:hi])
        wsum = F32(0.0)
        if normalize:
            for s in order:
                wsum = F32(wsum + w[s])
            if wsum == F32(0.0):
                raise ValueError(f"query {q}: plan weights sum to zero, cannot renormalize")
        acc = np.zeros(c_n, dtype=np.float32)
        for s in order:
            vec = bilinear_f32(table, tiles[cam[s] * n_levels + lvl[s]], u[s], v[s])
            ws = F32(w[s] / wsum) if normalize else w[s]
            acc = acc + ws * vec
        out[q] = acc
    return out, empty


# --------------------------------------------------------------------------
# tile-grouped batched semantics (msda_optimized, FULL and PACKED_HALF)


def normalized_weights(offsets, cam, lvl, u, v, w):
    """Per-query f32 sums in canonical order, then w / sum (features.py:279-288)."""
    q_n = len(offsets) - 1
    qidx = np.repeat(np.arange(q_n, dtype=np.int64), np.diff(offsets))
    order = np.lexsort((w, u, v, lvl, cam, qidx))
    sums = np.zeros(q_n, dtype=np.float32)
    np.add.at(sums, qidx[order], w[order])
    bad = (sums == 0.0) & (np.diff(offsets) > 0)
    if bad.any():
        raise ValueError(f"query {int(np.nonzero(bad)[0][0])}: plan weights sum to zero, cannot renormalize")
    return w / sums[qidx], qidx


def _tiled_range(table, tiles, n_levels, offsets, cam, lvl, u, v, wn, qidx, q_lo, q_hi, dtype):
    """Tile-major pass over queries [q_lo, q_hi) (features.py:362-416).

    Samples are ordered (camera, level) first, then per query (v, u, weight);
    each tile's samples are interpolated in the compute dtype with the fixed
    add tree, scaled by the sample weight and scatter-added sequentially
    (``np.add.at``) — for one query that is the canonical order again.
    """
    c_n = table.shape[1]
    s_lo, s_hi = int(offsets[q_lo]), int(offsets[q_hi])
    n_q = q_hi - q_lo
    acc = np.zeros((n_q, c_n), dtype=dtype)
    if s_hi == s_lo:
        return acc.astype(np.float32)
    sl = slice(s_lo, s_hi)
    c_, l_, u_, v_, w_, q_ = cam[sl], lvl[sl], u[sl], v[sl], wn[sl], qidx[sl] - q_lo
    order = np.lexsort((w_, u_, v_, q_, l_, c_))
    c_, l_, u_, v_, w_, q_ = (a[order] for a in (c_, l_, u_, v_, w_, q_))
    cut = np.nonzero((np.diff(c_) != 0) | (np.diff(l_) != 0))[0] + 1
    starts = np.concatenate(([0], cut))
    ends = np.concatenate((cut, [len(c_)]))
    for a, b in zip(starts, ends):
        start, h, w = tiles[int(c_[a]) * n_levels + int(l_[a])]
        grid = table[start:start + h * w].astype(dtype, copy=False).reshape(h, w, c_n)
        uu, vv = u_[a:b], v_[a:b]
        x0f, y0f = np.floor(uu), np.floor(vv)
        fu, fv = uu - x0f, vv - y0f
        omu, omv = _ONE - fu, _ONE - fv
        iw = np.stack([omu * omv, fu * omv, omu * fv, fu * fv]).astype(dtype, copy=False)
        inx0 = (x0f >= 0.0) & (x0f <= w - 1)
        inx1 = (x0f >= -1.0) & (x0f <= w - 2)
        iny0 = (y0f >= 0.0) & (y0f <= h - 1)
        iny1 = (y0f >= -1.0) & (y0f <= h - 2)
        xi0 = np.clip(x0f, 0, w - 1).astype(np.int64)
        xi1 = np.clip(x0f + 1.0, 0, w - 1).astype(np.int64)
        yi0 = np.clip(y0f, 0, h - 1).astype(np.int64)
        yi1 = np.clip(y0f + 1.0, 0, h - 1).astype(np.int64)
        terms = []
        for k, (yy, xx, m) in enumerate(
            ((yi0, xi0, inx0 & iny0), (yi0, xi1, inx1 & iny0), (yi1, xi0, inx0 & iny1), (yi1, xi1, inx1 & iny1))
        ):
            g = grid[yy, xx]
            g[~m] = 0
            terms.append(g * iw[k][:, None])
        t = (terms[0] + terms[1]) + (terms[2] + terms[3])
        t = t * w_[a:b].astype(dtype)[:, None]
        np.add.at(acc, q_[a:b], t)
    return acc.astype(np.float32)


def msda_tiled(table, tiles, n_levels, offsets, cam, lvl, u, v, w, precision="full", normalize=True, workers=1):
    """Batched MSDA (restates ``msda_optimized``, features.py:419-467).

    ``precision="full"`` is bit-identical to :func:`msda_exact`;
    ``precision="half"`` stores features as float16 and interpolates /
    accumulates in float16 (PACKED_HALF).  ``workers`` splits queries over
    threads without changing any output bit.
    """
    check_targets(tiles, n_levels, cam, lvl)
    if table.shape[1] % 2:
        raise ValueError("odd channel count")
    dtype = {"full": np.float32, "half": np.float16}[precision]
    if normalize:
        wn, qidx = normalized_weights(offsets, cam, lvl, u, v, w)
    else:
        wn = w
        qidx = np.repeat(np.arange(len(offsets) - 1, dtype=np.int64), np.diff(offsets))
    q_n = len(offsets) - 1
    empty = np.diff(offsets) == 0
    workers = max(1, int(workers))
    if workers == 1 or q_n < 2 * workers:
        return _tiled_range(table, tiles, n_levels, offsets, cam, lvl, u, v, wn, qidx, 0, q_n, dtype), empty
    bounds = np.linspace(0, q_n, workers + 1, dtype=np.int64)
    out = np.zeros((q_n, table.shape[1]), dtype=np.float32)
    with ThreadPoolExecutor(max_workers=workers) as pool:
        futs = {
            (int(a), int(b)): pool.submit(
                _tiled_range, table, tiles, n_levels, offsets, cam, lvl, u, v, wn, qidx, int(a), int(b), dtype
            )
            for a, b in zip(bounds[:-1], bounds[1:])
            if b > a
        }
        for (a, b), f in futs.items():
            out[a:b] = f.result()
    return out, empty


# --------------------------------------------------------------------------
# Sparse4D dense layout with channel groups


def dense_to_csr(spatial_shape, sampling_location, weights, group, n_levels):
    """Dense Sparse4D inputs → CSR plan for one channel group.

    ``sampling_location`` [bs, Q, P, cams, 2] normalized (x, y) shared across
    levels; ``weights`` [bs, Q, P, cams, L, G].  Level cell coordinates use
    the reference convention ``cell = pixel/stride - 0.5``
    (features.py:20-24, 45-47) with ``pixel/stride = loc * W_l`` computed as
    ``f32(f32(x * W_l) - 0.5)``.  Queries are the flattened (b, q) pairs.
    """
    bs, q_n, p_n, cams, _ = sampling_location.shape
    rows = []
    for b in range(bs):
        for q in range(q_n):
            for p in range(p_n):
                for c in range(cams):
                    x, y = sampling_location[b, q, p, c]
                    for lvl in range(n_levels):
                        h, w = spatial_shape[c, lvl]
                        uu = F32(F32(F32(x) * F32(w)) - F32(0.5))
                        vv = F32(F32(F32(y) * F32(h)) - F32(0.5))
                        rows.append((b * q_n + q, c, lvl, uu, vv, weights[b, q, p, c, lvl, group]))
    qi = np.array([r[0] for r in rows], dtype=np.int64)
    offsets = np.zeros(bs * q_n + 1, dtype=np.int64)
    np.cumsum(np.bincount(qi, minlength=bs * q_n), out=offsets[1:])
    order = np.argsort(qi, kind="stable")
    pick = lambda k, dt: np.array([rows[i][k] for i in order], dtype=dt)  # noqa: E731
    return offsets, pick(1, np.int32), pick(2, np.int32), pick(3, np.float32), pick(4, np.float32), pick(5, np.float32)


def dense_to_csr_vectorized(spatial_shape, sampling_location, weights, group):
    """``dense_to_csr`` vectorised (full BASELINE sizes): the same samples in
    the same per-query order (point, camera, level) with the same f32 cell
    arithmetic ``f32(f32(x * W_l) - 0.5)`` (features.py:20-24, 45-47)."""
    bs, q_n, p_n, cams, _ = sampling_location.shape
    n_levels = spatial_shape.shape[1]
    W = spatial_shape[:, :, 1].astype(F32)[None, None, None]  # [1, 1, 1, cams, L]
    H = spatial_shape[:, :, 0].astype(F32)[None, None, None]
    u = (sampling_location[..., 0:1].astype(F32) * W).astype(F32) - F32(0.5)
    v = (sampling_location[..., 1:2].astype(F32) * H).astype(F32) - F32(0.5)
    cam = np.broadcast_to(np.arange(cams, dtype=np.int32)[None, None, None, :, None], u.shape)
    lvl = np.broadcast_to(np.arange(n_levels, dtype=np.int32)[None, None, None, None, :], u.shape)
    per_q = p_n * cams * n_levels
    offsets = np.arange(bs * q_n + 1, dtype=np.int64) * per_q
    return (offsets, cam.reshape(-1).copy(), lvl.reshape(-1).copy(), u.astype(F32).reshape(-1),
            v.astype(F32).reshape(-1), np.ascontiguousarray(weights[..., group], dtype=F32).reshape(-1))


def msda_dense_groups(table, tiles, spatial_shape, sampling_location, weights, n_levels, normalize=False):
    """Group oracle: group g's channel slice aggregated with weights[..., g].

    ``out[:, g*C/G:(g+1)*C/G] = msda_exact(table[:, slice], plan_g)``.
    """
    g_n = weights.shape[-1]
    c_n = table.shape[1]
    cg = c_n // g_n
    bs, q_n = sampling_location.shape[:2]
    out = np.zeros((bs * q_n, c_n), dtype=np.float32)
    for g in range(g_n):
        offs, cam, lvl, u, v, w = dense_to_csr(spatial_shape, sampling_location, weights, g, n_levels)
        sub = np.ascontiguousarray(table[:, g * cg:(g + 1) * cg]).astype(np.float32)
        out[:, g * cg:(g + 1) * cg], _ = msda_exact(sub, tiles, n_levels, offs, cam, lvl, u, v, w, normalize)
    return out.reshape(bs, q_n, c_n)


# --------------------------------------------------------------------------
# keypoints and projection (geometry.py)


def rot_z(yaw):
    """geometry.py:49-52."""
    c, s = math.cos(yaw), math.sin(yaw)
    return np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])


def keypoints(anchor, offsets):
    """7 fixed + learned keypoints, float64 (geometry.py:207-247).

    ``anchor`` = (x, y, z, w, l, h, yaw, ...); fixed = centre + the six face
    centres ``±half`` along local axes rotated by yaw; learned =
    ``centre + R(yaw) @ (offset * (l/2, w/2, h/2))``.
    """
    x, y, z, w, l, h, yaw = (float(a) for a in anchor[:7])
    R = rot_z(yaw)
    half = np.array([l / 2.0, w / 2.0, h / 2.0])
    centre = np.array([x, y, z])
    dirs = np.array([[1, 0, 0], [-1, 0, 0], [0, 1, 0], [0, -1, 0], [0, 0, 1], [0, 0, -1]], dtype=float)
    pts = [centre, *((dirs * half) @ R.T + centre)]
    if offsets is not None and len(offsets):
        pts += list((np.asarray(offsets, dtype=float) * half) @ R.T + centre)
    return np.array(pts)


def project(K, R, t, point, eps=1e-6):
    """Pinhole projection (geometry.py:162-182); None when depth <= eps."""
    fx, fy, cx, cy = K
    p = np.asarray(R, dtype=float) @ np.asarray(point, dtype=float) + np.asarray(t, dtype=float)
    if p[2] <= eps:
        return None
    return fx * p[0] / p[2] + cx, fy * p[1] / p[2] + cy, p[2]


def projection_plan(anchors, learned_offsets, cams, strides, level_shapes, dt=0.0):
    """Anchors + cameras → CSR plan + weights-free sample list (float64 math).

    Composition of generate_keypoints → motion_compensate (geometry.py:250-255,
    shift by velocity·dt) → project_point (behind-camera samples dropped) →
    pixel_to_cell per level stride (features.py:45-47).  Returns per-query
    tuples (cam, level, u_cell, v_cell, p_index).
    """
    out = []
    for a in anchors:
        kps = keypoints(a, learned_offsets)
        vel = np.array([a[7], a[8], a[9]], dtype=float) if len(a) >= 10 else np.zeros(3)
        kps = kps + vel * dt
        samples = []
        for ci, (K, R, t) in enumerate(cams):
            for p, pt in enumerate(kps):
                pr = project(K, R, t, pt)
                if pr is None:
                    continue
                for lvl, s in enumerate(strides):
                    samples.append((ci, lvl, pr[0] / s - 0.5, pr[1] / s - 0.5, p))
        out.append(samples)
    return out


# --------------------------------------------------------------------------
# occlusion-aware embedding (oae.py)


def bilinear_f64_table(table, tile, u, v):
    """Float64 zero-padded bilinear (the OAE level reads, oae.py:108-111, in f64)."""
    start, h, w = tile
    x0, y0 = math.floor(u), math.floor(v)
    fu, fv = u - x0, v - y0
    out = np.zeros(table.shape[1])
    for yi, wy in ((y0, 1.0 - fv), (y0 + 1, fv)):
        for xi, wx in ((x0, 1.0 - fu), (x0 + 1, fu)):
            if 0 <= xi < w and 0 <= yi < h:
                out += wx * wy * table[start + yi * w + xi].astype(np.float64)
    return out


def extract_view(table, tiles, n_levels, cam_index, strides, K, R, t, kps, descriptor):
    """Per-camera keypoint feature g(.) (oae.py:81-122).

    Behind-camera keypoints are skipped; each survivor is read at every level
    (f32 bilinear, features.py:184-219) and averaged over levels in f64;
    softmax(desc·g_k/√D) weights the keypoint vectors.  Returns (vec, valid).
    """
    dim = len(descriptor)
    vecs = []
    for pt in kps:
        pr = project(K, R, t, pt)
        if pr is None:
            continue
        lv = [
            bilinear_f32(table, tiles[cam_index * n_levels + m], pr[0] / s - 0.5, pr[1] / s - 0.5).astype(np.float64)
            for m, s in enumerate(strides)
        ]
        vecs.append(np.mean(np.asarray(lv), axis=0))
    if not vecs:
        return np.zeros(dim), False
    mat = np.asarray(vecs)
    sc = mat @ np.asarray(descriptor, dtype=float) / np.sqrt(dim)
    sc -= sc.max()
    e = np.exp(sc)
    e /= e.sum()
    return e @ mat, True


def fuse(per_view, vis, memory, floor=1e-3):
    """Visibility-weighted fusion + L2 normalise, memory fallback (oae.py:125-164).

    Returns (embedding, all_occluded).
    """
    wts = [float(v) if ok else 0.0 for (vec, ok), v in zip(per_view, vis)]
    total = float(np.sum(wts))
    if not total > floor:
        return np.asarray(memory, dtype=float), True
    acc = np.zeros_like(np.asarray(per_view[0][0], dtype=float))
    for wv, (vec, _) in zip(wts, per_view):
        acc += wv * np.asarray(vec, dtype=float)
    raw = acc / total
    n = np.linalg.norm(raw)
    if n < 1e-12 or not np.isfinite(n):
        raise ValueError("cannot normalize a zero or non-finite vector")
    return raw / n, False


def msda_project_groups(table, tiles, anchors, offsets, K, R, T, strides, wts, n_levels, normalize, dt):
    """Fused projection oracle: generate_keypoints ->
    motion_compensate -> project_point (behind-camera samples leave the plan)
    -> pixel_to_cell per level -> msda_reference per channel group."""
    bs, q_n = anchors.shape[:2]
    g_n = wts.shape[-1]
    c_n = table.shape[1]
    cg = c_n // g_n
    out = np.zeros((bs * q_n, c_n), dtype=np.float32)
    cams = list(zip(K, R, T))
    for b in range(bs):
        plans = projection_plan(anchors[b].astype(np.float64), offsets.astype(np.float64), cams, strides,
                                   None, dt=dt)
        for q, samples in enumerate(plans):
            for g in range(g_n):
                pq = [(c, m, np.float32(u), np.float32(v), wts[b, q, p, c, m, g]) for c, m, u, v, p in samples]
                offs, cam, lvl, uu, vv, ww = csr_from_per_query([pq])
                sub = np.ascontiguousarray(table[:, g * cg:(g + 1) * cg])
                if len(pq):
                    r, _ = msda_exact(sub, tiles, n_levels, offs, cam, lvl, uu, vv, ww, normalize)
                    out[b * q_n + q, g * cg:(g + 1) * cg] = r[0]
    return out.reshape(bs, q_n, c_n)
