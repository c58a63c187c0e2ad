"""FPYR container mirror (reference simulator.py:481-545): byte-identical
writer, reader equal to the reference-written fixture, reference error
behaviour; the GPU upload is one contiguous copy into the feature table."""

import io

import numpy as np
import pytest

from paper_2601_10819_b200 import features as F
from paper_2601_10819_b200 import fpyr


def _frames():
    rng = np.random.default_rng(47)
    frames = []
    for _ in range(3):
        frame = {}
        for cam in (7, 2):
            lv = [F.FeatureGrid(stride=8.0 * 2 ** m, values=rng.standard_normal((5 - m, 6 - m, 4)).astype(np.float32))
                  for m in range(2)]
            frame[cam] = F.FeaturePyramid(cam, lv)
        frames.append(frame)
    return frames


def test_writer_is_byte_identical_to_reference(golden, tmp_path):
    path = tmp_path / "pyr.bin"
    fpyr.write_pyramid_sequence(path, _frames())
    assert path.read_bytes() == golden("fpyr")["blob"].tobytes()


def test_reader_matches_frames_and_table_layout(golden, tmp_path):
    path = tmp_path / "pyr.bin"
    path.write_bytes(golden("fpyr")["blob"].tobytes())
    frames = _frames()
    loaded = fpyr.read_pyramid_sequence(path)
    assert len(loaded) == 3
    for fa, fb in zip(frames, loaded):
        assert sorted(fa) == sorted(fb)
        for cam in fa:
            for ga, gb in zip(fa[cam].levels, fb[cam].levels):
                assert ga.stride == gb.stride
                np.testing.assert_array_equal(ga.values, gb.values)
    with fpyr.FpyrReader(path) as rd:
        h = rd.header
        assert h.camera_ids == (2, 7) and h.channels == 4 and h.n_levels == 2
        t = rd.frame_table(1)
        rows = np.concatenate([frames[1][c].levels[m].values.reshape(-1, 4) for c in (2, 7) for m in range(2)])
        np.testing.assert_array_equal(t, rows)  # payload == channel-last concatenated table
        assert list(h.scale_start_index().reshape(-1)) == [0, 30, 50, 80]
        del t


def test_reader_errors(golden, tmp_path):
    blob = golden("fpyr")["blob"].tobytes()
    for name, data in (("magic", b"JUNK" + blob[4:]), ("cut", blob[:-7]), ("long", blob + b"\x00\x00"),
                       ("version", blob[:4] + b"\x02" + blob[5:]), ("tiny", b"FP")):
        p = tmp_path / f"{name}.bin"
        p.write_bytes(data)
        with pytest.raises(ValueError):
            fpyr.read_pyramid_sequence(p)


@pytest.mark.gpu
@pytest.mark.parametrize("pin", [True, False])
def test_upload_frame_to_device(golden, tmp_path, cuda_dev, pin):
    """pin=True: the mapping is page-locked and each frame is one DMA from it;
    pin=False: staged through a pinned buffer.  Same bytes either way, every
    frame, in any order."""
    path = tmp_path / "pyr.bin"
    path.write_bytes(golden("fpyr")["blob"].tobytes())
    with fpyr.FpyrReader(path, pin=pin) as rd:
        for frame in (2, 0, 1, 2):
            feats = rd.upload(frame, device=cuda_dev)
            host = rd.frame_table(frame).copy()
            np.testing.assert_array_equal(feats.table[0].cpu().numpy(), host)
        assert feats.spatial_shape.cpu().tolist() == [[[5, 6], [4, 5]], [[5, 6], [4, 5]]]
        assert rd.registered == pin
