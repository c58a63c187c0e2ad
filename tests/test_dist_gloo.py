"""Multi-process (world_size 2, gloo, CPU) tests of the sharding drivers.

The per-rank compute is the numpy oracle here (tests may use it as the
checker's stand-in for the GPU kernel); what is under test is the host
logic: camera ranges, slicing, the all-reduce of partial numerators and
weight sums, and the renormalisation.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import helpers
from oracle import msda_oracle as mo


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, normalize, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    from paper_2601_10819_b200.dist import CameraShardedAggregation, camera_range

    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(77)
    cams, n_levels, groups, channels = 5, 2, 4, 16
    grids, shape, loc, wts = helpers.make_dense(rng, bs=2, n_q=6, n_p=4, cams=cams, n_levels=n_levels,
                                                groups=groups, channels=channels)
    lo, hi = camera_range(cams, rank, world)
    local = {(c - lo, m): g for (c, m), g in grids.items() if lo <= c < hi}
    table, tiles = mo.pack_grids(local, hi - lo, n_levels)

    def local_fn(l_loc, l_wts):
        return torch.from_numpy(mo.msda_dense_groups(table, tiles, shape[lo:hi], l_loc.numpy(), l_wts.numpy(),
                                                     n_levels, normalize=False))

    agg = CameraShardedAggregation(cams, local_fn)
    out = agg(torch.from_numpy(loc), torch.from_numpy(wts), normalize=normalize).numpy()
    if rank == 0:
        full, ftiles = mo.pack_grids(grids, cams, n_levels)
        ref = mo.msda_dense_groups(full, ftiles, shape, loc, wts, n_levels, normalize=normalize)
        q.put(float(np.abs(out - ref).max() / np.abs(ref).max()))
    dist.destroy_process_group()


@pytest.mark.parametrize("normalize", [False, True])
def test_camera_sharded_matches_single_scene(normalize):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, normalize, q)) for r in range(2)]
    for p in procs:
        p.start()
    err = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert err <= 1e-5


def test_camera_range_partition():
    from paper_2601_10819_b200.dist import camera_range, shard_streams

    for n in (1, 5, 16, 512):
        for world in (1, 2, 3, 8):
            ranges = [camera_range(n, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            sizes = [b - a for a, b in ranges]
            assert max(sizes) - min(sizes) <= 1
    assert shard_streams(16, 1, 8) == [1, 9]


def test_camera_sharded_transport_validation():
    """Only the all-reduce ("collective") and peer-memory ("peer") transports exist."""
    import pytest

    from paper_2601_10819_b200.dist import CameraShardedAggregation

    with pytest.raises(ValueError, match="unknown transport"):
        CameraShardedAggregation(4, lambda loc, w: None, transport="nvshmem")
    agg = CameraShardedAggregation(4, lambda loc, w: None)
    assert agg.transport == "collective" and agg.world == 1 and (agg.cam_lo, agg.cam_hi) == (0, 4)
    agg.close()  # no peer buffers: a no-op
