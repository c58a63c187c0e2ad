"""Multi-GPU drivers: one process per GPU, torch.distributed for the plumbing.

Two partitionings:

* **Stream-sharded** (``shard_streams``): independent camera-stream batches
  (scenes) are dealt round-robin to ranks; each rank owns its scenes'
  features, anchors and weights end to end.  No data-path collective.
* **Camera-sharded** (``CameraShardedAggregation``): one scene's cameras are
  split into contiguous ranges, each rank aggregates over its own cameras
  (un-normalised partial numerator ``[bs, Q, C]`` plus, when normalising,
  the partial per-(anchor, group) weight sums ``[bs, Q, G]``), and the
  partials are summed with one all-reduce (NCCL over NVLink on GPUs; any
  backend works).  The cross-rank summation order differs from the
  reference's sequential order, so this mode is tolerance parity only.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import torch
import torch.distributed as dist


def camera_range(n_cams: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced camera range [lo, hi) of ``rank``."""
    base, extra = divmod(n_cams, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_streams(n_scenes: int, rank: int, world: int) -> list[int]:
    """Scenes (independent stream batches) owned by ``rank``, round-robin."""
    return list(range(rank, n_scenes, world))


@dataclass
class CameraShardedAggregation:
    """Sparse4D deformable aggregation of one scene with cameras across ranks.

    ``local_fn(loc, weights)`` aggregates this rank's cameras without
    normalisation and returns ``[bs, Q, C]`` float32 — or ``(out, weight_sums
    [bs, Q, G])``.  On GPUs it is the C-ABI ``msda_dense_partial`` bound to
    the rank's feature table and ``normalize_fn`` is ``msda_dense_normalize``
    (see :meth:`for_device_features`), so no arithmetic runs outside the
    library; the CPU tests pass a numpy stand-in and fall back to torch.
    """

    n_cams: int
    local_fn: Callable
    group: object = None
    normalize_fn: Callable | None = None

    def __post_init__(self):
        self.rank = dist.get_rank(self.group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(self.group) if dist.is_initialized() else 1
        self.cam_lo, self.cam_hi = camera_range(self.n_cams, self.rank, self.world)

    def __call__(self, sampling_location, weights, normalize: bool = False, local_inputs: bool = False):
        """sampling_location [bs, Q, P, cams, 2], weights [bs, Q, P, cams, L, G]
        for ALL cameras (each rank slices its own) or, with ``local_inputs``,
        already restricted to this rank's camera range; returns [bs, Q, C]."""
        if local_inputs:
            loc, wts = sampling_location, weights
        else:
            loc = sampling_location[:, :, :, self.cam_lo:self.cam_hi].contiguous()
            wts = weights[:, :, :, self.cam_lo:self.cam_hi].contiguous()
        res = self.local_fn(loc, wts)
        part, wsum = res if isinstance(res, tuple) else (res, None)
        bs, q_n, c_n = part.shape
        g_n = weights.shape[-1]
        if normalize:
            if wsum is None:  # CPU stand-in: the weight sums of this rank's cameras
                wsum = wts.sum(dim=(2, 3, 4), dtype=torch.float32).to(part.device)  # [bs, Q, G]
            # one all-reduce of [bs*Q, C + G]: numerators and weight sums together
            buf = torch.cat([part.reshape(bs * q_n, c_n), wsum.reshape(bs * q_n, g_n)], dim=1)
        else:
            buf = part.reshape(bs * q_n, c_n)
        if self.world > 1:
            dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=self.group)
        if not normalize:
            return buf.reshape(bs, q_n, c_n)
        out = buf[:, :c_n].contiguous()
        ws = buf[:, c_n:].contiguous()
        if self.normalize_fn is not None:
            return self.normalize_fn(out, ws).reshape(bs, q_n, c_n)
        if bool((ws == 0).any()):
            raise ValueError("an anchor's weights sum to zero, cannot renormalize")
        return (out.reshape(bs, q_n, g_n, c_n // g_n) / ws.reshape(bs, q_n, g_n, 1)).reshape(bs, q_n, c_n)

    @classmethod
    def for_device_features(cls, n_cams, local_feats, precision="fast", group=None):
        """Bind to this rank's ``ops.DeviceFeatures`` (its camera range only)."""
        from . import ops

        def local(loc, wts):
            return ops.deformable_aggregation_partial(local_feats, loc, wts, precision=precision)

        return cls(n_cams, local, group, ops.normalize_groups)


def init_from_env(backend: str | None = None):
    """Initialise the default process group from torchrun's environment.

    Uses NCCL with the rank's GPU when CUDA is available, gloo otherwise.
    """
    import os

    if dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29511")
    if backend is None:
        backend = "nccl" if torch.cuda.is_available() else "gloo"
    if backend == "nccl":
        local = int(os.environ.get("LOCAL_RANK", 0))
        torch.cuda.set_device(local)
        dist.init_process_group(backend, rank=rank, world_size=world, device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend, rank=rank, world_size=world)
    return rank, world
