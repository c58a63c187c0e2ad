"""Camera-sharded all-reduce over peer memory (csrc/peer.cu, dist.PeerExchange).

The production setting is one process per GPU with the partials pushed over
NVLink; the GPU box of this suite has one GPU, so two processes share it: the
CUDA-IPC mapping, the float4 remote adds, the system-scope arrival counters,
the epoch double-buffering and the normalising wait are all exercised for
real, only the link differs.  Each rank aggregates its camera range with
msda_dense_partial; the peer result must equal the one-call normalised
aggregation of all cameras (tolerance: the cross-rank order differs) on
several consecutive epochs, without normalisation too, and a zero weight
sum must raise on every rank.
"""

import os
import socket
import sys
import traceback

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _scene(seed, cams, bs=2, q_n=10):
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import helpers

    rng = np.random.default_rng(seed)
    return helpers.make_dense(rng, bs=bs, n_q=q_n, n_p=13, cams=cams, n_levels=4, groups=8, channels=256,
                              size_lo=6, size_hi=24)


def _worker(rank, world, port, cams, result_dir):
    try:
        sys.path.insert(0, ROOT)
        import torch
        import torch.distributed as dist

        from oracle import msda_oracle as mo
        from paper_2601_10819_b200 import ops
        from paper_2601_10819_b200.dist import CameraShardedAggregation, camera_range

        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        lo, hi = camera_range(cams, rank, world)
        errs = []
        agg = None
        for epoch, seed in enumerate((41, 42, 43)):
            grids, shape, loc, wts = _scene(seed, cams)
            # this rank's cameras only, in the channel-last table layout
            local = {(c - lo, m): g for (c, m), g in grids.items() if lo <= c < hi}
            table, tiles = mo.pack_grids(local, hi - lo, 4)
            start = np.array([t[0] for t in tiles], dtype=np.int64).reshape(hi - lo, 4)
            tt = torch.from_numpy(np.ascontiguousarray(np.broadcast_to(table, (2,) + table.shape))).to(dev)
            feats = ops.DeviceFeatures(tt, torch.from_numpy(np.ascontiguousarray(shape[lo:hi])),
                                       torch.from_numpy(start))
            if agg is None:
                agg = CameraShardedAggregation.for_device_features(cams, feats, transport="peer")
            else:
                agg.bind_features(feats)
            t = lambda a: torch.from_numpy(a).to(dev)  # noqa: E731
            full_table, full_tiles = mo.pack_grids(grids, cams, 4)
            for normalize in (True, False):
                out = agg(t(loc), t(wts), normalize=normalize).cpu().numpy()
                ref = mo.msda_dense_groups(full_table, full_tiles, shape, loc, wts, 4, normalize=normalize)
                errs.append(float(np.abs(out - ref).max() / np.abs(ref).max()))
        zero = wts.copy()
        zero[1, 3, :, :, :, 2] = 0.0
        raised = False
        try:
            agg(t(loc), t(zero), normalize=True)
        except ValueError as e:
            raised = "sum to zero" in str(e)
        agg.close()
        dist.destroy_process_group()
        with open(os.path.join(result_dir, f"rank{rank}.txt"), "w") as f:
            f.write(f"{max(errs)} {int(raised)} {agg.world}\n")
    except Exception:
        with open(os.path.join(result_dir, f"rank{rank}.txt"), "w") as f:
            f.write("ERROR\n" + traceback.format_exc())


@pytest.mark.parametrize("world,cams", [(2, 5), (3, 7)])
def test_peer_allreduce_two_processes_one_gpu(cuda_dev, tmp_path, world, cams):
    import torch.multiprocessing as mp

    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_worker, args=(r, world, port, cams, str(tmp_path))) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        if p.is_alive():
            p.kill()
            pytest.fail("peer exchange worker hung")
    for r in range(world):
        txt = (tmp_path / f"rank{r}.txt").read_text()
        assert not txt.startswith("ERROR"), txt
        err, raised, w = txt.split()
        assert float(err) <= 1e-4, (r, err)
        assert raised == "1" and int(w) == world
