"""FPYR pyramid container → device feature table.

The container (reference simulator.py:481-545, docs/formats.md:54-74):
``b"FPYR" | u32 version=1 | u32 n_frames | u32 n_cameras | u32 n_levels |
u32 channels``, then per camera (ascending id) ``u32 id`` and per level
``f32 stride, u32 H, u32 W``, then the payload frame-major, camera-major,
level-major, each grid ``H*W*C`` little-endian f32 in ``(H, W, C)`` order.

A frame's payload is therefore *exactly* the channel-last concatenated
feature table the kernels consume (rows camera-major then level-minor), so
loading a frame onto the GPU is one contiguous host→device copy of a
memory-mapped file region — no repacking.  ``FpyrReader.upload`` page-locks
the mapping once and DMAs each frame straight from it, asynchronously on the
caller's stream (or stages through a pinned buffer when the mapping cannot
be registered).

``read_pyramid_sequence`` / ``write_pyramid_sequence`` mirror the reference
functions (same format, same ValueErrors for bad magic, unknown version,
truncation and trailing bytes).
"""

from __future__ import annotations

import mmap
import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np

MAGIC = b"FPYR"
VERSION = 1


@dataclass(frozen=True)
class FpyrHeader:
    n_frames: int
    n_cameras: int
    n_levels: int
    channels: int
    camera_ids: tuple
    strides: tuple       # [cam][level] float
    shapes: tuple        # [cam][level] (H, W)
    payload_offset: int

    @property
    def rows(self) -> int:
        return sum(h * w for cam in self.shapes for h, w in cam)

    @property
    def frame_bytes(self) -> int:
        return self.rows * self.channels * 4

    def spatial_shape(self) -> np.ndarray:
        return np.asarray(self.shapes, dtype=np.int32).reshape(self.n_cameras, self.n_levels, 2)

    def scale_start_index(self) -> np.ndarray:
        sizes = self.spatial_shape().prod(axis=2).reshape(-1)
        start = np.zeros_like(sizes, dtype=np.int64)
        np.cumsum(sizes[:-1], out=start[1:])
        return start.reshape(self.n_cameras, self.n_levels)


def read_header(buf) -> FpyrHeader:
    """Parse and validate the header of an FPYR byte buffer / mmap."""
    if len(buf) < 24 or bytes(buf[:4]) != MAGIC:
        raise ValueError(f"not a pyramid container (magic {bytes(buf[:4])!r})")
    version, n_frames, n_cameras, n_levels, channels = struct.unpack_from("<5I", buf, 4)
    if version != VERSION:
        raise ValueError(f"unsupported container version {version}")
    pos = 24
    ids, strides, shapes = [], [], []
    for _ in range(n_cameras):
        if pos + 4 + 12 * n_levels > len(buf):
            raise ValueError("truncated pyramid container")
        (cam_id,) = struct.unpack_from("<I", buf, pos)
        pos += 4
        st, sh = [], []
        for _ in range(n_levels):
            s, h, w = struct.unpack_from("<fII", buf, pos)
            pos += 12
            st.append(float(s))
            sh.append((int(h), int(w)))
        ids.append(int(cam_id))
        strides.append(tuple(st))
        shapes.append(tuple(sh))
    hdr = FpyrHeader(n_frames, n_cameras, n_levels, channels, tuple(ids), tuple(strides), tuple(shapes), pos)
    total = pos + n_frames * hdr.frame_bytes
    if len(buf) < total:
        raise ValueError("truncated pyramid container")
    if len(buf) > total:
        raise ValueError("trailing bytes after pyramid container payload")
    return hdr


class FpyrReader:
    """Memory-mapped FPYR file with zero-copy frame views and GPU upload.

    ``pin=True``: on the first upload the whole mapping is page-locked
    (``msda_host_register``, read-only), so each frame goes to the device as
    one DMA straight from the page cache; if the range cannot be registered
    the upload stages through a pinned buffer (one host memcpy per frame)."""

    def __init__(self, path, pin: bool = True):
        self.path = Path(path)
        self._fh = open(self.path, "rb")
        size = self.path.stat().st_size
        # a private (copy-on-write) mapping when pinning: the driver page-locks
        # those, not read-only shared file mappings (measured on the B200 box)
        access = mmap.ACCESS_COPY if pin else mmap.ACCESS_READ
        self._mm = mmap.mmap(self._fh.fileno(), 0, access=access) if size else b""
        self.header = read_header(self._mm)
        self._staging = None
        self._pin = pin
        self._registered = None  # base address of the registered mapping
        self._base = None  # numpy view of the whole mapping (keeps the address)

    @property
    def registered(self) -> bool:
        return self._registered is not None

    def _register(self):
        import ctypes

        from . import _lib as L

        if not self._pin or self._registered is not None or not isinstance(self._mm, mmap.mmap):
            return
        self._pin = False  # one attempt
        self._base = np.frombuffer(self._mm, dtype=np.uint8)
        addr = self._base.ctypes.data
        if L.lib().msda_host_register(ctypes.c_void_p(addr), self._base.nbytes, 0) == L.MSDA_OK:
            self._registered = addr

    def close(self):
        if self._registered is not None:
            import ctypes

            import torch

            from . import _lib as L

            torch.cuda.synchronize()  # no copy may still read the mapping
            L.lib().msda_host_unregister(ctypes.c_void_p(self._registered))
            self._registered = None
        self._base = None
        if isinstance(self._mm, mmap.mmap):
            self._mm.close()
        self._fh.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __len__(self):
        return self.header.n_frames

    def frame_table(self, frame: int) -> np.ndarray:
        """Frame ``frame`` as a read-only ``[rows, C]`` float32 view (no copy)."""
        h = self.header
        if not 0 <= frame < h.n_frames:
            raise IndexError(f"frame {frame} out of range")
        off = h.payload_offset + frame * h.frame_bytes
        view = np.frombuffer(self._mm, dtype="<f4", count=h.rows * h.channels, offset=off).reshape(
            h.rows, h.channels)
        view.flags.writeable = False  # frames are immutable (features.py:67), whatever the mapping mode
        return view

    def upload(self, frame: int, device="cuda", out=None, dtype=None, stream=None):
        """Copy one frame into a device table and wrap it as ``ops.DeviceFeatures``.

        The file region goes through a pinned staging buffer (one memcpy on the
        host) and one asynchronous H2D copy on ``stream``.
        """
        import torch

        from .ops import DeviceFeatures

        h = self.header
        src = self.frame_table(frame)
        stream = stream or torch.cuda.current_stream(device)
        self._register()
        if out is None:
            out = torch.empty(src.shape, dtype=torch.float32, device=device)
        if self._registered is not None:  # one DMA from the page-locked mapping
            import warnings

            with warnings.catch_warnings():  # read-only view: the copy only reads it
                warnings.simplefilter("ignore", UserWarning)
                host = torch.from_numpy(src)
            with torch.cuda.stream(stream):
                out.copy_(host, non_blocking=True)
        else:
            if self._staging is None or self._staging.shape != src.shape:
                self._staging = torch.empty(src.shape, dtype=torch.float32, pin_memory=True)
            stream.synchronize()  # the staging buffer may still feed a previous copy
            self._staging.numpy()[...] = src
            with torch.cuda.stream(stream):
                out.copy_(self._staging, non_blocking=True)
        with torch.cuda.stream(stream):
            table = out if dtype in (None, torch.float32) else out.to(dtype)
        return DeviceFeatures(table, torch.from_numpy(h.spatial_shape()), torch.from_numpy(h.scale_start_index()))


def write_pyramid_sequence(path, pyramid_frames) -> None:
    """Write frames (dicts camera_id → pyramid with ``levels`` of (stride,
    values)) in the FPYR layout (reference simulator.py:494-513)."""
    if not pyramid_frames:
        raise ValueError("no frames to write")
    first = pyramid_frames[0]
    cam_ids = sorted(first)
    n_levels = len(first[cam_ids[0]].levels)
    channels = first[cam_ids[0]].channels
    with open(path, "wb") as fh:
        fh.write(MAGIC)
        fh.write(struct.pack("<5I", VERSION, len(pyramid_frames), len(cam_ids), n_levels, channels))
        for cam_id in cam_ids:
            fh.write(struct.pack("<I", cam_id))
            for grid in first[cam_id].levels:
                fh.write(struct.pack("<fII", grid.stride, grid.height, grid.width))
        for frame in pyramid_frames:
            if sorted(frame) != cam_ids:
                raise ValueError("camera set differs between frames")
            for cam_id in cam_ids:
                for grid in frame[cam_id].levels:
                    fh.write(np.ascontiguousarray(grid.values, dtype="<f4").tobytes())


def read_pyramid_sequence(path) -> list:
    """Frames as dicts camera_id → FeaturePyramid (reference simulator.py:516-545)."""
    from .features import FeatureGrid, FeaturePyramid

    with FpyrReader(path) as rd:
        h = rd.header
        frames = []
        for f in range(h.n_frames):
            table = rd.frame_table(f)
            frame, row = {}, 0
            for ci, cam_id in enumerate(h.camera_ids):
                grids = []
                for (hh, ww), st in zip(h.shapes[ci], h.strides[ci]):
                    vals = np.array(table[row:row + hh * ww]).reshape(hh, ww, h.channels)
                    grids.append(FeatureGrid(stride=st, values=vals))
                    row += hh * ww
                frame[cam_id] = FeaturePyramid(camera_id=cam_id, levels=grids)
            frames.append(frame)
            del table  # release the mmap view before the reader closes
    return frames
