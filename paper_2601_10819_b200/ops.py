"""Device-tensor API over the C ABI (torch supplies memory and streams only).

All arithmetic happens in ``libmsda_b200.so``; these wrappers validate
shapes, pass raw device pointers and the current CUDA stream, and map the
C-ABI status back to the reference's exceptions.

Entry points
------------
``DeviceFeatures``          the channel-last multi-camera multi-level table
``msda_csr``                CSR plan (reference SamplePlan) → out [Q, C], empty [Q]
``deformable_aggregation``  Sparse4D API (mc_ms_feat, spatial_shape,
                            scale_start_index, sampling_location, weights)
``msda_dense_project``      dense path with keypoint projection fused in
``oae_pool``                occlusion-aware embedding pooling
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L
from .errors import raise_for_status

_DTYPES = {torch.float32: L.MSDA_F32, torch.float16: L.MSDA_F16, torch.bfloat16: L.MSDA_BF16}
_PREC = {"exact": L.MSDA_EXACT, "exact_half": L.MSDA_EXACT_HALF, "fast": L.MSDA_FAST, "fast_h2": L.MSDA_FAST_H2}


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _stream(device):
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


class _Workspace:
    """Grow-only per-(device, stream) workspace, reused across calls."""

    def __init__(self):
        self._bufs = {}

    def get(self, device, nbytes):
        key = (device.index, torch.cuda.current_stream(device).cuda_stream)
        buf = self._bufs.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)
            self._bufs[key] = buf
        return buf


WORKSPACE = _Workspace()


def precision_code(precision) -> int:
    if isinstance(precision, int):
        return precision
    try:
        return _PREC[str(precision)]
    except KeyError:
        raise ValueError(f"unknown precision mode: {precision!r}") from None


_CONST_CACHE: dict = {}


def _small_const(values, dtype, dev, shape):
    """Small per-call constants (level strides, learned keypoint offsets)
    given as host lists/arrays: uploaded once per distinct value set and
    device, then reused — a host→device copy from pageable memory would
    synchronise every call.  Device tensors pass through untouched."""
    if isinstance(values, torch.Tensor) and values.device == dev:
        return values.to(dtype).reshape(shape).contiguous()
    np_dtype = {torch.float64: np.float64, torch.float32: np.float32, torch.int32: np.int32,
                torch.int64: np.int64}[dtype]
    arr = np.ascontiguousarray(np.asarray(values.cpu() if isinstance(values, torch.Tensor) else values,
                                          dtype=np_dtype))
    key = (arr.tobytes(), arr.shape, str(dtype), str(dev))
    hit = _CONST_CACHE.get(key)
    if hit is None:
        if len(_CONST_CACHE) > 256:
            _CONST_CACHE.clear()
        hit = torch.from_numpy(arr).to(device=dev, dtype=dtype).reshape(shape).contiguous()
        _CONST_CACHE[key] = hit
    return hit


@dataclass
class DeviceFeatures:
    """Feature table resident in HBM.

    ``table``: [R, C] or [B, R, C] (f32 / f16 / bf16), rows = every (camera,
    level) grid (H, W, C) row-major, camera-major then level-minor.
    ``spatial_shape``: int32 [cams, L, 2] (H, W); ``scale_start_index``:
    int64 [cams, L] first row of each grid.
    """

    table: torch.Tensor
    spatial_shape: torch.Tensor
    scale_start_index: torch.Tensor

    def __post_init__(self):
        if self.table.dim() == 2:
            self.table = self.table.unsqueeze(0)
        if self.table.dim() != 3 or not self.table.is_cuda or not self.table.is_contiguous():
            raise ValueError("table must be a contiguous CUDA tensor [R, C] or [B, R, C]")
        if self.table.dtype not in _DTYPES:
            raise ValueError(f"unsupported feature dtype {self.table.dtype}")
        dev = self.table.device
        # host-side shape tables (a per-call deformable_aggregation argument in
        # Sparse4D) are uploaded once per value set, not copied every call
        self.spatial_shape = _small_const(self.spatial_shape, torch.int32, dev, tuple(self.spatial_shape.shape))
        self.scale_start_index = _small_const(self.scale_start_index, torch.int64, dev,
                                              tuple(self.scale_start_index.shape))
        if self.spatial_shape.dim() != 3 or self.spatial_shape.shape[2] != 2:
            raise ValueError("spatial_shape must be [cams, levels, 2]")
        if tuple(self.scale_start_index.shape) != tuple(self.spatial_shape.shape[:2]):
            raise ValueError("scale_start_index must be [cams, levels]")
        # host copy of the level shapes (C ABI spatial_shape_host): the call
        # picks its on-chip staging plan without a device read
        self._shape_host = np.ascontiguousarray(self.spatial_shape.cpu().numpy(), dtype=np.int32)
    @property
    def n_cams(self):
        return int(self.spatial_shape.shape[0])

    @property
    def n_levels(self):
        return int(self.spatial_shape.shape[1])

    @property
    def channels(self):
        return int(self.table.shape[2])

    def descriptor(self) -> L.Features:
        return L.Features(_ptr(self.table), _DTYPES[self.table.dtype], int(self.table.shape[0]), self.n_cams,
                          self.n_levels, self.channels, 0, int(self.table.shape[1]), _ptr(self.spatial_shape),
                          _ptr(self.scale_start_index), ctypes.c_void_p(self._shape_host.ctypes.data))

    @classmethod
    def from_grids(cls, grids, device="cuda", dtype=torch.float32):
        """Pack ``[[grid(H, W, C) per level] per camera]`` (numpy or torch)."""
        rows, shape, start, r = [], [], [], 0
        for cam in grids:
            shape.append([])
            start.append([])
            for g in cam:
                g = torch.as_tensor(g)
                h, w, c = g.shape
                rows.append(g.reshape(h * w, c))
                shape[-1].append([h, w])
                start[-1].append(r)
                r += h * w
        table = torch.cat(rows, 0).to(device=device, dtype=dtype).contiguous()
        return cls(table, torch.tensor(shape, dtype=torch.int32), torch.tensor(start, dtype=torch.int64))


def _check_call(code, ws, device, check, what):
    if code != L.MSDA_OK:
        raise_for_status(code, -1, what)
    if check:
        st, det = ctypes.c_int32(0), ctypes.c_int64(-1)
        rc = L.lib().msda_read_status(_ptr(ws), _stream(device), ctypes.byref(st), ctypes.byref(det))
        if rc != L.MSDA_OK:
            raise_for_status(rc, -1, what)
        raise_for_status(st.value, det.value, what)


def msda_csr(feats: DeviceFeatures, offsets, camera_index, level, u, v, weight, precision="exact",
             normalize=True, out=None, empty=None, check=True, stages=3):
    """CSR-plan MSDA on device (``msda_reference`` / ``msda_optimized`` math).

    ``camera_index`` is the dense camera index (ascending camera id).  With
    ``check`` the call synchronises and raises the reference exception for
    data-dependent errors; without it the call is fully asynchronous.
    """
    dev = feats.table.device
    q_n = int(offsets.numel()) - 1
    s_n = int(u.numel())
    c_n = feats.channels
    if out is None:
        out = torch.empty((q_n, c_n), dtype=torch.float32, device=dev)
    if empty is None:
        empty = torch.empty((q_n,), dtype=torch.uint8, device=dev)
    lib = L.lib()
    nbytes = lib.msda_csr_workspace_size(q_n, s_n, c_n)
    ws = WORKSPACE.get(dev, nbytes)
    plan = L.CsrPlan(q_n, s_n, _ptr(offsets), _ptr(camera_index), _ptr(level), _ptr(u), _ptr(v), _ptr(weight))
    fd = feats.descriptor()
    code = lib.msda_csr_stages(ctypes.byref(fd), ctypes.byref(plan), precision_code(precision),
                               int(bool(normalize)), _ptr(out), _ptr(empty), _ptr(ws), ws.numel(), _stream(dev),
                               int(stages))
    _check_call(code, ws, dev, check, "msda_csr")
    return out, empty


def deformable_aggregation(mc_ms_feat, spatial_shape, scale_start_index, sampling_location, weights,
                           precision="fast", normalize=False, out=None, check=False):
    """Sparse4D ``deformable_aggregation`` (BASELINE north_star API).

    mc_ms_feat [bs, R, C] (f32/f16/bf16), spatial_shape [cams, L, 2],
    scale_start_index [cams, L], sampling_location [bs, Q, P, cams, 2]
    (normalized x, y), weights [bs, Q, P, cams, L, G]  →  out [bs, Q, C] f32.
    Sampling follows the reference convention (cell = loc*W - 0.5, zero
    padding, features.py:20-24, 184-219).
    """
    feats = mc_ms_feat if isinstance(mc_ms_feat, DeviceFeatures) else DeviceFeatures(
        mc_ms_feat.contiguous(), spatial_shape, scale_start_index)
    dev = feats.table.device
    bs, q_n, p_n, cams, two = sampling_location.shape
    if two != 2 or cams != feats.n_cams:
        raise ValueError("sampling_location must be [bs, Q, P, cams, 2]")
    g_n = int(weights.shape[-1])
    if tuple(weights.shape) != (bs, q_n, p_n, cams, feats.n_levels, g_n):
        raise ValueError("weights must be [bs, Q, P, cams, levels, groups]")
    if bs != feats.table.shape[0]:
        raise ValueError("batch of mc_ms_feat and sampling_location differ")
    loc = sampling_location.to(torch.float32).contiguous()
    wts = weights.to(torch.float32).contiguous()
    if out is None:
        out = torch.empty((bs, q_n, feats.channels), dtype=torch.float32, device=dev)
    lib = L.lib()
    nbytes = lib.msda_dense_workspace_size(bs, q_n, p_n, cams, feats.n_levels, g_n, feats.channels)
    ws = WORKSPACE.get(dev, nbytes)
    fd = feats.descriptor()
    code = lib.msda_dense(ctypes.byref(fd), q_n, p_n, g_n, _ptr(loc), _ptr(wts), precision_code(precision),
                          int(bool(normalize)), _ptr(out), _ptr(ws), ws.numel(), _stream(dev))
    _check_call(code, ws, dev, check, "deformable_aggregation")
    return out


class Cameras:
    """Pinhole cameras on device in float64 (CameraModel, geometry.py:56-97)."""

    def __init__(self, K, R, t, device="cuda"):
        self.K = torch.as_tensor(K, dtype=torch.float64).reshape(-1, 4).to(device).contiguous()
        self.R = torch.as_tensor(R, dtype=torch.float64).reshape(-1, 9).to(device).contiguous()
        self.t = torch.as_tensor(t, dtype=torch.float64).reshape(-1, 3).to(device).contiguous()
        if not (self.K.shape[0] == self.R.shape[0] == self.t.shape[0]):
            raise ValueError("K, R, t must describe the same number of cameras")

    def descriptor(self) -> L.Cameras:
        return L.Cameras(_ptr(self.K), _ptr(self.R), _ptr(self.t))

    @classmethod
    def from_models(cls, cams, device="cuda"):
        """From objects with focal_x/focal_y/principal_x/principal_y/rotation/translation."""
        import numpy as np

        K = np.array([[c.focal_x, c.focal_y, c.principal_x, c.principal_y] for c in cams], dtype=np.float64)
        R = np.array([np.asarray(c.rotation, dtype=np.float64).reshape(9) for c in cams])
        t = np.array([np.asarray(c.translation, dtype=np.float64).reshape(3) for c in cams])
        return cls(K, R, t, device)


def deformable_aggregation_partial(feats: DeviceFeatures, sampling_location, weights, precision="fast", out=None,
                                   weight_sums=None):
    """Un-normalised FAST aggregation of ``feats``' cameras plus the
    per-(query, group) weight sums: the partials a camera-sharded rank
    all-reduces (C ABI ``msda_dense_partial``).  Returns (out [bs, Q, C],
    weight_sums [bs, Q, G]); ``out`` / ``weight_sums`` may be given (e.g. two
    views of one buffer that a single all-reduce then sums)."""
    dev = feats.table.device
    loc = sampling_location.to(device=dev, dtype=torch.float32).contiguous()
    wts = weights.to(device=dev, dtype=torch.float32).contiguous()
    bs, q_n, p_n = int(loc.shape[0]), int(loc.shape[1]), int(loc.shape[2])
    g_n = int(wts.shape[-1])
    if tuple(loc.shape) != (bs, q_n, p_n, feats.n_cams, 2) or tuple(wts.shape) != (
            bs, q_n, p_n, feats.n_cams, feats.n_levels, g_n):
        raise ValueError("sampling_location [bs, Q, P, cams, 2] and weights [bs, Q, P, cams, L, G] expected")
    if bs != feats.table.shape[0]:  # the C ABI takes the batch from the feature descriptor
        raise ValueError("batch of the feature table and sampling_location differ")
    if out is None:
        out = torch.empty((bs, q_n, feats.channels), dtype=torch.float32, device=dev)
    if weight_sums is None:
        weight_sums = torch.empty((bs, q_n, g_n), dtype=torch.float32, device=dev)
    if (out.numel() != bs * q_n * feats.channels or weight_sums.numel() != bs * q_n * g_n or not out.is_contiguous()
            or not weight_sums.is_contiguous() or out.dtype != torch.float32 or weight_sums.dtype != torch.float32):
        raise ValueError("out [bs, Q, C] and weight_sums [bs, Q, G] must be contiguous float32")
    wsum = weight_sums
    lib = L.lib()
    ws = WORKSPACE.get(dev, lib.msda_dense_workspace_size(bs, q_n, p_n, feats.n_cams, feats.n_levels, g_n,
                                                          feats.channels))
    fd = feats.descriptor()
    code = lib.msda_dense_partial(ctypes.byref(fd), q_n, p_n, g_n, _ptr(loc), _ptr(wts), precision_code(precision),
                                  _ptr(out), _ptr(wsum), _ptr(ws), ws.numel(), _stream(dev))
    if code != L.MSDA_OK:
        raise_for_status(code, -1, "deformable_aggregation_partial")
    return out.reshape(bs, q_n, feats.channels), wsum.reshape(bs, q_n, g_n)


def normalize_groups(out, weight_sums, check=True):
    """In place: out[..., c] /= weight_sums[..., c // (C / G)] (C ABI
    ``msda_dense_normalize``); a zero sum raises the reference's ValueError."""
    dev = out.device
    c_n, g_n = int(out.shape[-1]), int(weight_sums.shape[-1])
    n_q = out.numel() // c_n
    if not out.is_contiguous() or not weight_sums.is_contiguous() or weight_sums.numel() != n_q * g_n:
        raise ValueError("contiguous out [..., C] and weight_sums [..., G] expected")
    ws = WORKSPACE.get(dev, 256)
    code = L.lib().msda_dense_normalize(_ptr(out), _ptr(weight_sums), n_q, c_n, g_n, _ptr(ws), _stream(dev))
    _check_call(code, ws, dev, check, "normalize_groups")
    return out


def msda_dense_project(feats: DeviceFeatures, anchors, learned_offsets, cameras: Cameras, strides, weights, dt=0.0,
                       precision="fast", normalize=False, out=None, check=False):
    """Dense MSDA with keypoint generation + projection fused into the kernel.

    anchors [bs, Q, 10] (x, y, z, w, l, h, yaw, vx, vy, vz); learned_offsets
    [n_learned, 3]; strides [L] pixel strides; weights [bs, Q, 7+n_learned,
    cams, L, G].  Behind-camera keypoints leave the plan.
    """
    dev = feats.table.device
    anchors = anchors.to(device=dev, dtype=torch.float32).contiguous()
    bs, q_n, ten = anchors.shape
    if ten != 10 or bs != feats.table.shape[0]:
        raise ValueError("anchors must be [bs, Q, 10] with bs == feature batch")
    offs = _small_const(learned_offsets, torch.float32, dev, (-1, 3))
    n_learned = int(offs.shape[0])
    p_n = 7 + n_learned
    strides = _small_const(strides, torch.float32, dev, (-1,))
    if strides.numel() != feats.n_levels:
        raise ValueError("one stride per level")
    wts = weights.to(device=dev, dtype=torch.float32).contiguous()
    g_n = int(wts.shape[-1])
    if tuple(wts.shape) != (bs, q_n, p_n, feats.n_cams, feats.n_levels, g_n):
        raise ValueError("weights must be [bs, Q, 7 + n_learned, cams, levels, groups]")
    if cameras.K.shape[0] != feats.n_cams:
        raise ValueError("camera count differs from the feature table")
    if out is None:
        out = torch.empty((bs, q_n, feats.channels), dtype=torch.float32, device=dev)
    lib = L.lib()
    nbytes = lib.msda_dense_workspace_size(bs, q_n, p_n, feats.n_cams, feats.n_levels, g_n, feats.channels)
    ws = WORKSPACE.get(dev, nbytes)
    fd, cd = feats.descriptor(), cameras.descriptor()
    code = lib.msda_dense_project(ctypes.byref(fd), q_n, _ptr(anchors), n_learned, _ptr(offs), ctypes.byref(cd),
                                  _ptr(strides), float(dt), g_n, _ptr(wts), precision_code(precision),
                                  int(bool(normalize)), _ptr(out), _ptr(ws), ws.numel(), _stream(dev))
    _check_call(code, ws, dev, check, "msda_dense_project")
    return out


def oae_pool(feats: DeviceFeatures, anchors, learned_offsets, cameras: Cameras, strides, descriptors, visibility,
             memory, check=True):
    """Occlusion-aware embedding pooling (oae.py:81-164) for Q queries.

    Returns (embeddings [Q, C] f32 unit-norm, all_occluded [Q] bool).
    """
    from .errors import ChannelMismatch

    dev = feats.table.device
    if feats.table.shape[0] != 1:
        raise ValueError("oae_pool takes a single-scene feature table")
    anchors = anchors.to(device=dev, dtype=torch.float32).reshape(-1, 10).contiguous()
    q_n = int(anchors.shape[0])
    desc = descriptors.to(device=dev, dtype=torch.float32).contiguous()
    if desc.dim() != 2 or desc.shape[0] != q_n:
        raise ValueError("descriptors must be [Q, D]")
    if desc.shape[1] != feats.channels:
        raise ChannelMismatch(f"pyramid has C={feats.channels} but descriptor has D={desc.shape[1]}")
    vis = visibility.to(device=dev, dtype=torch.float32).contiguous()
    mem = memory.to(device=dev, dtype=torch.float32).contiguous()
    if tuple(vis.shape) != (q_n, feats.n_cams) or tuple(mem.shape) != (q_n, feats.channels):
        raise ValueError("visibility must be [Q, cams] and memory [Q, C]")
    offs = _small_const(learned_offsets, torch.float32, dev, (-1, 3))
    strides = _small_const(strides, torch.float32, dev, (-1,))
    out = torch.empty((q_n, feats.channels), dtype=torch.float32, device=dev)
    occl = torch.empty((q_n,), dtype=torch.uint8, device=dev)
    lib = L.lib()
    ws = WORKSPACE.get(dev, lib.msda_oae_workspace_size(q_n, feats.n_cams, feats.channels))
    fd, cd = feats.descriptor(), cameras.descriptor()
    code = lib.msda_oae_pool(ctypes.byref(fd), q_n, _ptr(anchors), int(offs.shape[0]), _ptr(offs), ctypes.byref(cd),
                             _ptr(strides), _ptr(desc), _ptr(vis), _ptr(mem), _ptr(out), _ptr(occl), _ptr(ws),
                             ws.numel(), _stream(dev))
    _check_call(code, ws, dev, check, "oae_pool")
    return out, occl.bool()


def _boxes_with_trig(boxes):
    """[n, 7] (x, y, z, w, l, h, yaw) -> [n, 9] f64 with cos(yaw), sin(yaw)
    from Python's math module: the values rot_z uses (geometry.py:50-53), so
    the device corner arithmetic sees the reference's bits (C ABI contract)."""
    import math

    b = np.asarray(boxes.cpu() if isinstance(boxes, torch.Tensor) else boxes, dtype=np.float64).reshape(-1, 7)
    trig = np.array([[math.cos(y), math.sin(y)] for y in b[:, 6]], dtype=np.float64).reshape(-1, 2)
    return torch.from_numpy(np.ascontiguousarray(np.concatenate([b, trig], axis=1)))


def visibility(cameras: Cameras, image_wh, objects, grid: int = 64):
    """Visible fraction of every object in every camera (visibility.py:46-115).

    ``objects`` [n, 7] (x, y, z, w, l, h, yaw); ``image_wh`` [cams, 2].
    Returns (visibility [cams, n] f32, fully_behind [cams, n] bool).
    """
    dev = cameras.K.device
    obj = _boxes_with_trig(objects).to(dev).contiguous()
    wh = torch.as_tensor(image_wh, dtype=torch.int32).reshape(-1, 2).to(dev).contiguous()
    n_cams, n_obj = int(cameras.K.shape[0]), int(obj.shape[0])
    if wh.shape[0] != n_cams:
        raise ValueError("one image size per camera")
    if grid < 2:
        raise ValueError("grid must be at least 2")
    vis = torch.empty((n_cams, n_obj), dtype=torch.float32, device=dev)
    behind = torch.empty((n_cams, n_obj), dtype=torch.uint8, device=dev)
    lib = L.lib()
    ws = WORKSPACE.get(dev, lib.msda_visibility_workspace_size(n_cams, n_obj))
    cd = cameras.descriptor()
    code = lib.msda_visibility(ctypes.byref(cd), _ptr(wh), n_cams, _ptr(obj), n_obj, int(grid), _ptr(vis),
                               _ptr(behind), _ptr(ws), ws.numel(), _stream(dev))
    if code != L.MSDA_OK:
        raise_for_status(code, -1, "visibility")
    return vis, behind.bool()


class PaintScene:
    """A scene prepared for feature painting (simulator.py:249-289): cameras,
    level grids (ceil(image / stride), simulator.py:252-253), the table
    layout, entity boxes and signatures resident on device.  ``run`` paints
    one frame into the channel-last table the MSDA path reads.

    ``entities`` [n_objects + n_occluders, 7] f64 (x, y, z, w, l, h, yaw):
    moving objects first (``signatures`` [n_objects, C] f64), then occluders.
    """

    def __init__(self, cameras: Cameras, image_wh, strides, channels, entities, n_objects, signatures=None):
        import math

        dev = cameras.K.device
        wh = np.asarray(image_wh, dtype=np.int64).reshape(-1, 2)
        n_cams = int(cameras.K.shape[0])
        if wh.shape[0] != n_cams:
            raise ValueError("one image size per camera")
        if channels <= 0 or channels % 4:
            raise ValueError("channels must be a positive multiple of 4")
        st = [float(x) for x in np.asarray(strides, dtype=np.float64).reshape(-1)]
        n_levels = len(st)
        shape = np.array([[[int(math.ceil(h / s)), int(math.ceil(w / s))] for s in st] for w, h in wh],
                         dtype=np.int32)
        start = np.zeros((n_cams, n_levels), dtype=np.int64)
        rows = 0
        for c in range(n_cams):
            for m in range(n_levels):
                start[c, m] = rows
                rows += int(shape[c, m, 0] * shape[c, m, 1])
        self.ent = _boxes_with_trig(entities).to(dev).contiguous()
        n_ent = int(self.ent.shape[0])
        if not 0 <= n_objects <= n_ent:
            raise ValueError("n_objects must be within the entity count")
        self.sig = None
        if n_objects:
            self.sig = torch.as_tensor(np.asarray(signatures, dtype=np.float64)).to(dev).contiguous()
            if tuple(self.sig.shape) != (n_objects, channels):
                raise ValueError("signatures must be [n_objects, channels]")
        self.cameras, self.device = cameras, dev
        self.n_cams, self.n_levels, self.channels, self.rows = n_cams, n_levels, int(channels), rows
        self.n_objects, self.n_ent = int(n_objects), n_ent
        self.shape_host = torch.from_numpy(np.ascontiguousarray(shape))
        self.start_host = torch.from_numpy(start)
        self.d_shape = self.shape_host.to(dev)
        self.d_start = self.start_host.to(dev)
        self.d_strides = torch.tensor(st, dtype=torch.float64, device=dev)
        self.ws = torch.empty(max(256, int(L.lib().msda_paint_workspace_size(n_cams, n_ent))), dtype=torch.uint8,
                              device=dev)

    def run(self, background=None, sigma=0.01, seed=0, frame=0, dtype=torch.float32, out=None):
        """Paint one frame.  ``background``: f64 [rows, C] (the reference's
        numpy draw gives a bit-identical table) or None for a device Philox
        N(0, sigma) draw keyed by (seed, frame).  Returns ``DeviceFeatures``."""
        bg = None
        if background is not None:
            bg = torch.as_tensor(background, dtype=torch.float64).to(self.device).contiguous()
            if tuple(bg.shape) != (self.rows, self.channels):
                raise ValueError(f"background must be [{self.rows}, {self.channels}]")
        if out is None:
            out = torch.empty((self.rows, self.channels), dtype=dtype, device=self.device)
        elif tuple(out.shape) != (self.rows, self.channels) or not out.is_contiguous():
            raise ValueError("out must be a contiguous [rows, C] tensor")
        cd = self.cameras.descriptor()
        code = L.lib().msda_paint(ctypes.byref(cd), self.n_cams, self.n_levels, _ptr(self.d_strides),
                                  _ptr(self.d_shape), _ptr(self.shape_host), _ptr(self.d_start), self.channels,
                                  _ptr(self.ent), self.n_objects, self.n_ent - self.n_objects, _ptr(self.sig),
                                  _ptr(bg), float(sigma), int(seed) & 0xFFFFFFFFFFFFFFFF, int(frame),
                                  _DTYPES[out.dtype], _ptr(out), _ptr(self.ws), self.ws.numel(),
                                  _stream(self.device))
        if code != L.MSDA_OK:
            raise_for_status(code, -1, "paint")
        return DeviceFeatures(out, self.shape_host, self.start_host)


def paint(cameras: Cameras, image_wh, strides, channels, entities, n_objects, signatures=None, background=None,
          sigma=0.01, seed=0, frame=0, dtype=torch.float32):
    """One-shot ``PaintScene(...).run(...)``: the painted channel-last table
    (``DeviceFeatures``) of every camera's pyramid."""
    return PaintScene(cameras, image_wh, strides, channels, entities, n_objects, signatures).run(
        background, sigma, seed, frame, dtype)


def association_cost(q_centers, d_centers, q_embeddings, d_embeddings, gate_radius=2.0, alpha_emb=1.0,
                     alpha_geo=1.0, device=None):
    """The tracker's association cost matrices (tracker.py:119-128) on device,
    f64 and bit-identical to the reference's numpy.

    Returns (cost, solver_cost, admissible) [n_q, n_d]."""
    if device is None:
        device = q_embeddings.device if torch.is_tensor(q_embeddings) else torch.device("cuda")
    t = lambda a, n: torch.as_tensor(a, dtype=torch.float64).to(device).reshape(-1, n).contiguous()  # noqa: E731
    qe = torch.as_tensor(q_embeddings, dtype=torch.float64).to(device).contiguous()
    de = torch.as_tensor(d_embeddings, dtype=torch.float64).to(device).contiguous()
    if qe.dim() != 2 or de.dim() != 2 or qe.shape[1] != de.shape[1]:
        raise ValueError("embeddings must be [n, D] with one D")
    n_q, n_d, dim = int(qe.shape[0]), int(de.shape[0]), int(qe.shape[1])
    qc, dc = t(q_centers, 3), t(d_centers, 3)
    if qc.shape[0] != n_q or dc.shape[0] != n_d:
        raise ValueError("one centre per query / detection")
    cost = torch.empty((n_q, n_d), dtype=torch.float64, device=device)
    solver = torch.empty_like(cost)
    adm = torch.empty((n_q, n_d), dtype=torch.uint8, device=device)
    code = L.lib().msda_assoc_cost(_ptr(qc), _ptr(dc), _ptr(qe), _ptr(de), n_q, n_d, dim, float(gate_radius),
                                   float(alpha_emb), float(alpha_geo), _ptr(cost), _ptr(solver), _ptr(adm),
                                   _stream(device))
    if code != L.MSDA_OK:
        raise_for_status(code, -1, "association_cost")
    return cost, solver, adm.bool()

