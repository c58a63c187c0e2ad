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

    Device path (:meth:`for_device_features`): ``partial_into(loc, weights,
    num, wsum)`` is the C-ABI ``msda_dense_partial`` writing this rank's
    un-normalised numerators ``num [bs*Q, C]`` and per-(anchor, group)
    weight sums ``wsum [bs*Q, G]`` straight into two views of ONE contiguous
    buffer ``[bs*Q*C | bs*Q*G]``, so a single all-reduce sums both (no
    staging copy), then ``normalize_fn`` (``msda_dense_normalize``) divides in
    place — no arithmetic outside the library.  :meth:`capture` records
    partial kernels + NCCL all-reduce + normalisation as one CUDA graph.

    CPU tests pass ``local_fn(loc, weights)`` returning ``[bs, Q, C]`` (or
    ``(out, weight_sums)``), copied into the same buffer, with a torch
    normalisation fallback.
    """

    n_cams: int
    local_fn: Callable | None = None
    group: object = None
    normalize_fn: Callable | None = None
    transport: str = "collective"  # or "peer": PeerExchange over NVLink (GPU ranks, <= 8)
    partial_into: Callable | None = None

    def __post_init__(self):
        if self.transport not in ("collective", "peer"):
            raise ValueError(f"unknown transport {self.transport!r}")
        if self.local_fn is None and self.partial_into is None:
            raise ValueError("local_fn or partial_into is required")
        self._peer = None
        self._buf = None
        self.rank = dist.get_rank(self.group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(self.group) if dist.is_initialized() else 1
        self.cam_lo, self.cam_hi = camera_range(self.n_cams, self.rank, self.world)

    def _packed(self, rows, c_n, g_n, device):
        n = rows * (c_n + g_n)
        if self._buf is None or self._buf.numel() != n or self._buf.device != torch.device(device):
            self._buf = torch.empty(n, dtype=torch.float32, device=device)
        return self._buf, self._buf[:rows * c_n].view(rows, c_n), self._buf[rows * c_n:].view(rows, g_n)

    def __call__(self, sampling_location, weights, normalize: bool = False, local_inputs: bool = False,
                 check: bool = True):
        """sampling_location [bs, Q, P, cams, 2], weights [bs, Q, P, cams, L, G]
        for ALL cameras (each rank slices its own) or, with ``local_inputs``,
        already restricted to this rank's camera range; returns [bs, Q, C]."""
        out = self._run(sampling_location, weights, normalize, local_inputs, check)
        return out.clone()

    def _run(self, sampling_location, weights, normalize, local_inputs, check=True):
        if local_inputs:
            loc, wts = sampling_location, weights
        else:
            loc = sampling_location[:, :, :, self.cam_lo:self.cam_hi].contiguous()
            wts = weights[:, :, :, self.cam_lo:self.cam_hi].contiguous()
        bs, q_n = int(loc.shape[0]), int(loc.shape[1])
        g_n = int(weights.shape[-1])
        rows = bs * q_n
        if self.partial_into is not None:
            c_n = self.channels
            buf, num, wsum = self._packed(rows, c_n, g_n, loc.device)
            self.partial_into(loc, wts, num, wsum)
        else:  # CPU stand-in
            res = self.local_fn(loc, wts)
            part, ws_ = res if isinstance(res, tuple) else (res, None)
            c_n = int(part.shape[-1])
            buf, num, wsum = self._packed(rows, c_n, g_n, part.device)
            num.copy_(part.reshape(rows, c_n))
            if ws_ is None:  # the weight sums of this rank's cameras
                ws_ = wts.sum(dim=(2, 3, 4), dtype=torch.float32)
            wsum.copy_(ws_.reshape(rows, g_n))
        if self.transport == "peer":
            px = self._peer
            if px is None or (px.rows, px.channels, px.groups) != (rows, c_n, g_n):
                if px is not None:
                    px.close()
                px = self._peer = PeerExchange(rows, c_n, g_n, num.device, self.group)
            return px.allreduce_normalize(num, wsum, normalize, check=check).reshape(bs, q_n, c_n)
        if self.world > 1:  # one all-reduce of the numerators (+ the weight sums when normalising)
            dist.all_reduce(buf if normalize else num.view(-1), op=dist.ReduceOp.SUM, group=self.group)
        if not normalize:
            return num.reshape(bs, q_n, c_n)
        if self.normalize_fn is not None:
            return self.normalize_fn(num, wsum, check=check).reshape(bs, q_n, c_n)
        if bool((wsum == 0).any()):
            raise ValueError("an anchor's weights sum to zero, cannot renormalize")
        return (num.reshape(rows, g_n, c_n // g_n) / wsum.reshape(rows, g_n, 1)).reshape(bs, q_n, c_n)

    def capture(self, sampling_location, weights, normalize: bool = False, local_inputs: bool = True):
        """One call — partial kernels, NCCL all-reduce, normalisation —
        captured as a CUDA graph over the given (static) input tensors: write
        new inputs into them and ``replay()``.  Returns (graph, out): ``out``
        [bs, Q, C] is the graph's output buffer, rewritten by every replay."""
        if self.partial_into is None or self.transport != "collective":
            raise ValueError("capture needs the device path and the collective transport")
        self._run(sampling_location, weights, normalize, local_inputs, check=True)  # warm-up: comm, workspace
        torch.cuda.synchronize(sampling_location.device)
        side = torch.cuda.Stream(sampling_location.device)
        side.wait_stream(torch.cuda.current_stream(sampling_location.device))
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=side):
            out = self._run(sampling_location, weights, normalize, local_inputs, check=False)
        torch.cuda.current_stream(sampling_location.device).wait_stream(side)
        return graph, out

    @classmethod
    def for_device_features(cls, n_cams, local_feats, precision="fast", group=None, transport="collective"):
        """Bind to this rank's ``ops.DeviceFeatures`` (its camera range only);
        ``transport="peer"`` replaces the all-reduce + normalise launches with
        the peer-memory exchange (``PeerExchange``)."""
        from . import ops

        agg = cls(n_cams, None, group, ops.normalize_groups, transport, lambda *a: None)
        agg.bind_features(local_feats, precision)
        return agg

    def bind_features(self, local_feats, precision="fast"):
        """(Re)bind the device path to this rank's feature table (a new frame)."""
        from . import ops

        def partial_into(loc, wts, num, wsum):
            ops.deformable_aggregation_partial(local_feats, loc, wts, precision=precision, out=num, weight_sums=wsum)

        self.partial_into = partial_into
        self.channels = local_feats.channels

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
