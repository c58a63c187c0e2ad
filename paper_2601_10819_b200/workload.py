"""Deterministic synthetic MSDA workloads, byte-identical to the reference's.

``BenchWorkload`` / ``generate_workload`` restate the reference bench
generator (``mvtrack3d/bench.py:26-113``) and ``substream`` restates
``mvtrack3d/rng.py:26-29`` so that the GPU path and the reference CPU path
see exactly the same inputs (pinned by the SHA-256 ``checksum``, which covers
the same bytes in the same order as the reference's).

The generated pyramid is written straight into the channel-last concatenated
table the kernels consume (``[sum_{cam,level} H*W, C]``, camera-major then
level-minor — the layout of ``FeatureGrid.values`` stacked, features.py:54-80),
optionally into a caller-provided (e.g. pinned) host buffer.
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np


def _label_to_int(label) -> int:
    if isinstance(label, (int, np.integer)):
        return int(label) & 0xFFFFFFFFFFFFFFFF
    if isinstance(label, str):
        return int.from_bytes(hashlib.blake2b(label.encode("utf-8"), digest_size=8).digest(), "little")
    raise TypeError(f"substream labels must be int or str, got {type(label).__name__}")


def substream(seed: int, *labels) -> np.random.Generator:
    """Independent PCG64 stream from ``seed`` and a label path (rng.py:26-29)."""
    entropy = [int(seed) & 0xFFFFFFFFFFFFFFFF] + [_label_to_int(x) for x in labels]
    return np.random.default_rng(np.random.SeedSequence(entropy))


@dataclass(frozen=True)
class BenchWorkload:
    """Workload descriptor; field names and defaults of bench.py:26-38."""

    cameras: int = 6
    levels: int = 4
    channels: int = 256
    queries: int = 900
    points_per_query: int = 13
    level0_size: tuple = (64, 64)
    repetitions: int = 3
    seed: int = 0
    fps_targets: tuple = (30.0,)

    def to_dict(self) -> dict:
        return {
            "schema_version": 1,
            "cameras": self.cameras,
            "levels": self.levels,
            "channels": self.channels,
            "queries": self.queries,
            "points_per_query": self.points_per_query,
            "level0_size": list(self.level0_size),
            "repetitions": self.repetitions,
            "seed": self.seed,
            "fps_targets": list(self.fps_targets),
        }

    def level_dims(self):
        """(H, W) per level: ``max(1, size >> m)`` (bench.py:80-81)."""
        return [(max(1, self.level0_size[0] >> m), max(1, self.level0_size[1] >> m)) for m in range(self.levels)]

    def strides(self):
        """Level strides ``8 * 2**m`` (bench.py:84)."""
        return [8.0 * 2 ** m for m in range(self.levels)]

    @property
    def num_rows(self) -> int:
        return self.cameras * sum(h * w for h, w in self.level_dims())

    @property
    def num_samples(self) -> int:
        return self.queries * self.cameras * self.levels * self.points_per_query


@dataclass
class GeneratedWorkload:
    """Materialized inputs: packed feature table + CSR plan (+ checksum)."""

    workload: BenchWorkload
    table: np.ndarray          # [R, C] float32, channel-last concatenated
    tile_start: np.ndarray     # int64 [cams*levels]
    spatial_shape: np.ndarray  # int32 [cams, levels, 2] (H, W)
    strides: list
    offsets: np.ndarray        # int64 [Q+1]
    camera_ids: np.ndarray     # int32 [S]
    levels: np.ndarray         # int32 [S]
    us: np.ndarray             # float32 [S]
    vs: np.ndarray
    weights: np.ndarray
    checksum: str

    @property
    def tiles(self):
        n_l = self.spatial_shape.shape[1]
        return [(int(self.tile_start[t]), int(self.spatial_shape[t // n_l, t % n_l, 0]),
                 int(self.spatial_shape[t // n_l, t % n_l, 1])) for t in range(len(self.tile_start))]


def generate_workload(workload: BenchWorkload, table_out: np.ndarray | None = None) -> GeneratedWorkload:
    """Materialize the reference bench workload (bench.py:65-113), same bytes.

    Every query samples ``points_per_query`` locations in each level of each
    camera; features are U[-1, 1), coordinates U(-1, W) / U(-1, H) cells per
    level, weights U(0.01, 1).  The plan is already grouped by query (the
    reference's stable ``argsort`` by query index is the identity here).
    """
    wl = workload
    rng = substream(wl.seed, "bench", "inputs")
    digest = hashlib.sha256()
    dims = wl.level_dims()
    n_rows = wl.num_rows
    if table_out is None:
        table = np.empty((n_rows, wl.channels), dtype=np.float32)
    else:
        table = table_out
        if table.shape != (n_rows, wl.channels) or table.dtype != np.float32:
            raise ValueError("table_out has the wrong shape or dtype")
    tile_start = np.zeros(wl.cameras * wl.levels, dtype=np.int64)
    row = 0
    for cam in range(wl.cameras):
        for m, (h, w) in enumerate(dims):
            vals = rng.uniform(-1.0, 1.0, (h, w, wl.channels)).astype(np.float32)
            digest.update(vals.tobytes())
            table[row:row + h * w] = vals.reshape(h * w, wl.channels)
            tile_start[cam * wl.levels + m] = row
            row += h * w
    per_q = wl.cameras * wl.levels * wl.points_per_query
    n = wl.queries * per_q
    cams = np.tile(np.repeat(np.arange(wl.cameras, dtype=np.int32), wl.levels * wl.points_per_query), wl.queries)
    lvls = np.tile(np.tile(np.repeat(np.arange(wl.levels, dtype=np.int32), wl.points_per_query), wl.cameras),
                   wl.queries)
    heights = np.array([d[0] for d in dims], dtype=np.float64)
    widths = np.array([d[1] for d in dims], dtype=np.float64)
    us = rng.uniform(-1.0, widths[lvls], n).astype(np.float32)
    vs = rng.uniform(-1.0, heights[lvls], n).astype(np.float32)
    ws = rng.uniform(0.01, 1.0, n).astype(np.float32)
    for arr in (us, vs, ws):
        digest.update(arr.tobytes())
    offsets = np.arange(wl.queries + 1, dtype=np.int64) * per_q
    shape = np.array([[d for d in dims]] * wl.cameras, dtype=np.int32).reshape(wl.cameras, wl.levels, 2)
    return GeneratedWorkload(wl, table, tile_start, shape, wl.strides(), offsets, cams, lvls, us, vs, ws,
                             "sha256:" + digest.hexdigest())
