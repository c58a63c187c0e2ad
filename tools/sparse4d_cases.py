"""Synthetic Sparse4D-layout workloads shared by bench.py (the driver's clock)
and tools/bench_paths.py (builder sweeps).

Inputs per SURVEY §8(d): features U[-1, 1) channel-last (device RNG, cast to
the storage dtype), sampling_location U[0, 1)^2 per (b, q, p, cam) shared
across levels, weights softmax over (P * cams * L) of N(0, 1) logits per
(b, q, g), G = 8.  Level shapes: cfg1/3/4 = 256x704 at strides 4-32
(64x176 .. 8x22), cfg2 = 1080p at strides 4-32 with ceil (simulator.py:252-253).
"""

from __future__ import annotations

import math

import numpy as np
import torch

CFG1_LEVELS = [(64, 176), (32, 88), (16, 44), (8, 22)]
CFG2_LEVELS = [(270, 480), (135, 240), (68, 120), (34, 60)]
L2_BYTES = 126 * 1024 * 1024


def make_feats(cams, levels, C, dtype, dev, bs=1, seed=0):
    from paper_2601_10819_b200 import ops

    rows = cams * sum(h * w for h, w in levels)
    g = torch.Generator(device=dev).manual_seed(seed)
    table = (torch.rand((bs, rows, C), generator=g, device=dev) * 2 - 1).to(dtype)
    shape = torch.tensor([[list(lv) for lv in levels]] * cams, dtype=torch.int32)
    start, r = [], 0
    for _ in range(cams):
        s = []
        for h, w in levels:
            s.append(r)
            r += h * w
        start.append(s)
    return ops.DeviceFeatures(table, shape, torch.tensor(start, dtype=torch.int64))


def make_dense_inputs(bs, Q, P, cams, L, G, dev, seed=1):
    g = torch.Generator(device=dev).manual_seed(seed)
    loc = torch.rand((bs, Q, P, cams, 2), generator=g, device=dev)
    logits = torch.randn((bs, Q, P * cams * L, G), generator=g, device=dev)
    w = torch.softmax(logits, dim=2).reshape(bs, Q, P, cams, L, G).contiguous()
    return loc, w


def staged_fine_levels(levels, dtype):
    """The dense FAST split the library makes (csrc/msda_staged.cu
    dense_staged_fine_levels): 4 levels whose levels 2-3 of every camera fit
    120 KB as 128-B row slices padded to 64-row TMA boxes -> the gather moves
    levels 0-1 from L2, levels 2-3 come from shared memory (any storage
    dtype).  Returns 2, or None when the anchor-major gather takes every level."""
    if len(levels) != 4:
        return None
    stage = sum((h * w + 63) // 64 * 64 * 128 for h, w in levels[2:])
    return 2 if stage <= 120 * 1024 else None


def touched_bytes(feats, loc, esize, per_level=False):
    """(unique in-bounds corner cells x C x esize, every in-grid corner row the
    gather moves L2 -> SM x C x esize) of a dense sampling;
    ``per_level`` adds the gathered bytes of each level."""
    shape = feats.spatial_shape.long()
    start = feats.scale_start_index
    bs, Q, P, cams, _ = loc.shape
    L = shape.shape[1]
    idx = []
    lv_moved = [0] * L
    for c in range(cams):
        for m in range(L):
            H, W = int(shape[c, m, 0]), int(shape[c, m, 1])
            u = loc[:, :, :, c, 0] * W - 0.5
            v = loc[:, :, :, c, 1] * H - 0.5
            x0, y0 = torch.floor(u).long(), torch.floor(v).long()
            for dy in (0, 1):
                for dx in (0, 1):
                    x, y = x0 + dx, y0 + dy
                    ok = (x >= 0) & (x < W) & (y >= 0) & (y < H)
                    b = torch.arange(bs, device=loc.device).view(bs, 1, 1).expand_as(x)
                    idx.append((b * feats.table.shape[1] + int(start[c, m]) + y * W + x)[ok])
                    lv_moved[m] += int(idx[-1].numel()) * feats.channels * esize
    rows = torch.cat(idx)
    res = torch.unique(rows).numel() * feats.channels * esize, rows.numel() * feats.channels * esize
    return (*res, lv_moved) if per_level else res


def algorithmic_bytes(feats, loc, w, esize):
    """SURVEY §8(d) dense figure: touched feature bytes + locations + weights + f32 output."""
    tb, moved, lv = touched_bytes(feats, loc, esize, per_level=True)
    bs, Q = loc.shape[:2]
    total = tb + loc.numel() * 4 + w.numel() * 4 + bs * Q * feats.channels * 4
    return {"touched_feature_bytes": int(tb), "input_bytes": int(loc.numel() * 4 + w.numel() * 4),
            "output_bytes": int(bs * Q * feats.channels * 4), "total": int(total), "gathered_corner_bytes": int(moved),
            "gathered_corner_bytes_per_level": [int(x) for x in lv]}


def host_view(feats):
    """Batch item 0 of the table as f32 numpy (f16/bf16 widen exactly) + the
    oracle's tile list [(start, H, W)] in (camera, level) order."""
    table = feats.table[0].float().cpu().numpy()
    shape = feats.spatial_shape.cpu().numpy()
    start = feats.scale_start_index.cpu().numpy()
    cams, L = shape.shape[:2]
    tiles = [(int(start[c, m]), int(shape[c, m, 0]), int(shape[c, m, 1])) for c in range(cams) for m in range(L)]
    return table, tiles, shape


def ring(cams, radius=12.0, height=4.0, focal=300.0, size=(704, 256)):
    """Cameras on a ring looking at (0, 0, 0.9) (camera_looking_at, geometry.py:258-290, restated):
    K [cams, 4] (fx, fy, cx, cy), R [cams, 3, 3], t [cams, 3] (SURVEY §8(d) projection runs)."""
    Ks, Rs, ts = [], [], []
    for i in range(cams):
        ang = 2 * math.pi * i / cams
        pos = np.array([radius * math.cos(ang), radius * math.sin(ang), height])
        z = np.array([0.0, 0.0, 0.9]) - pos
        z /= np.linalg.norm(z)
        x = np.cross(z, [0.0, 0.0, 1.0])
        x /= np.linalg.norm(x)
        y = np.cross(z, x)
        R = np.vstack([x, y, z])
        Ks.append([focal, focal, size[0] / 2, size[1] / 2])
        Rs.append(R)
        ts.append(-R @ pos)
    return np.array(Ks), np.array(Rs), np.array(ts)


def anchors_for(Q, dev, seed=2):
    """Anchors uniform in x, y in [-4, 4] m, z = 0.9, (w, l, h) = (0.6, 0.6, 1.8), yaw U(-pi, pi)."""
    g = torch.Generator(device="cpu").manual_seed(seed)
    a = torch.zeros((Q, 10))
    a[:, 0:2] = torch.rand((Q, 2), generator=g) * 8 - 4
    a[:, 2] = 0.9
    a[:, 3:6] = torch.tensor([0.6, 0.6, 1.8])
    a[:, 6] = torch.rand(Q, generator=g) * 2 * math.pi - math.pi
    return a.to(dev)
