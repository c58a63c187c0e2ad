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
  backend works) — or, with ``transport="peer"``, pushed straight into every
  rank's symmetric buffer over NVLink and normalised by one waiting kernel
  (``PeerExchange``, csrc/peer.cu).  The cross-rank summation order differs
  from the reference's sequential order, so this mode is tolerance parity
  only.
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


class PeerExchange:
    """Symmetric peer-memory buffers for the camera-sharded all-reduce
    (C ABI ``msda_peer_*``): every rank allocates one buffer, the CUDA-IPC
    handles are exchanged with an object all-gather over ``group`` (any
    backend), and each call pushes this rank's partial into every rank's
    buffer over NVLink and normalises — no NCCL on the data path.

    ``rows`` = bs * Q, ``channels`` = C, ``groups`` = G are fixed per
    instance; the epoch counter advances once per call on every rank (all
    ranks must call in lockstep, as with any collective)."""

    def __init__(self, rows: int, channels: int, groups: int, device, group=None):
        import ctypes

        from . import _lib as L
        from .errors import raise_for_status

        self._L = L
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        if self.world > 8:
            raise ValueError("peer exchange supports up to 8 ranks (one NVSwitch domain)")
        self.rows, self.channels, self.groups = int(rows), int(channels), int(groups)
        self.device = torch.device(device)
        lib = L.lib()
        with torch.cuda.device(self.device):
            nbytes = lib.msda_peer_buffer_size(self.rows, self.channels, self.groups)
            own = ctypes.c_void_p()
            raise_for_status(lib.msda_peer_alloc(nbytes, ctypes.byref(own)), -1, "msda_peer_alloc")
            self._own = own.value
            handle = ctypes.create_string_buffer(64)
            raise_for_status(lib.msda_ipc_handle(self._own, handle), -1, "msda_ipc_handle")
            handles = [None] * self.world
            if self.world > 1:
                dist.all_gather_object(handles, handle.raw, group=group)
            else:
                handles = [handle.raw]
            self._opened = []
            ptrs = []
            for r, h in enumerate(handles):
                if r == self.rank:
                    ptrs.append(self._own)
                    continue
                p = ctypes.c_void_p()
                raise_for_status(lib.msda_ipc_open(ctypes.create_string_buffer(h, 64), ctypes.byref(p)), -1,
                                 "msda_ipc_open")
                self._opened.append(p.value)
                ptrs.append(p.value)
            self._ptrs = (ctypes.c_void_p * self.world)(*ptrs)
            self._status = torch.zeros(64, dtype=torch.int32, device=self.device)
            torch.cuda.synchronize(self.device)
        if self.world > 1:
            dist.barrier(group=group)  # every buffer zeroed and mapped before the first epoch
        self.epoch = 0

    def allreduce_normalize(self, num, weight_sums, normalize: bool, out=None, weight_sums_out=None,
                            check: bool = True):
        """num [rows, C] f32 and weight_sums [rows, G] f32 (this rank's
        partials, on this rank's device) -> out [rows, C] = sum over ranks,
        divided per group by the summed weights when ``normalize``."""
        from .errors import raise_for_status

        num = num.reshape(self.rows, self.channels).contiguous()
        ws = weight_sums.reshape(self.rows, self.groups).contiguous() if weight_sums is not None else None
        if out is None:
            out = torch.empty((self.rows, self.channels), dtype=torch.float32, device=self.device)
        self.epoch += 1
        stream = torch.cuda.current_stream(self.device).cuda_stream
        code = self._L.lib().msda_peer_allreduce_normalize(
            num.data_ptr(), ws.data_ptr() if ws is not None else None, self._ptrs, self.world, self.rank,
            self.epoch & 0xFFFFFFFF, self.rows, self.channels, self.groups, int(bool(normalize)), out.data_ptr(),
            weight_sums_out.data_ptr() if weight_sums_out is not None else None, self._status.data_ptr(), stream)
        raise_for_status(code, -1, "msda_peer_allreduce_normalize")
        if check:
            st = self._status.cpu()
            raise_for_status(int(st[0]), int(st[2]) if int(st[0]) else -1, "msda_peer_allreduce_normalize")
        return out

    def close(self):
        lib = self._L.lib()
        if self._own is None:
            return
        torch.cuda.synchronize(self.device)
        if self.world > 1:
            dist.barrier(group=self.group)  # no peer still reads or adds into our buffer
        for p in self._opened:
            lib.msda_ipc_close(p)
        lib.msda_peer_free(self._own)
        self._own = None


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
    transport: str = "collective"  # or "peer": PeerExchange over NVLink (GPU ranks, <= 8)

    def __post_init__(self):
        if self.transport not in ("collective", "peer"):
            raise ValueError(f"unknown transport {self.transport!r}")
        self._peer = None
        self.rank = dist.get_rank(self.group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(self.group) if dist.is_initialized() else 1
        self.cam_lo, self.cam_hi = camera_range(self.n_cams, self.rank, self.world)

    def __call__(self, sampling_location, weights, normalize: bool = False, local_inputs: bool = False,
                 check: bool = True):
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
        if self.transport == "peer":
            if wsum is None:
                wsum = wts.sum(dim=(2, 3, 4), dtype=torch.float32).to(part.device)
            px = self._peer
            if px is None or (px.rows, px.channels, px.groups) != (bs * q_n, c_n, g_n):
                if px is not None:
                    px.close()
                px = self._peer = PeerExchange(bs * q_n, c_n, g_n, part.device, self.group)
            return px.allreduce_normalize(part, wsum, normalize, check=check).reshape(bs, q_n, c_n)
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
    def for_device_features(cls, n_cams, local_feats, precision="fast", group=None, transport="collective"):
        """Bind to this rank's ``ops.DeviceFeatures`` (its camera range only);
        ``transport="peer"`` replaces the all-reduce + normalise launches with
        the peer-memory exchange (``PeerExchange``)."""
        from . import ops

        def local(loc, wts):
            return ops.deformable_aggregation_partial(local_feats, loc, wts, precision=precision)

        return cls(n_cams, local, group, ops.normalize_groups, transport)

    def close(self):
        if self._peer is not None:
            self._peer.close()
            self._peer = None


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
