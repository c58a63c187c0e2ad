"""bench-msda harness mirror (reference bench.py / cli.py): schema validation
on the CPU, the report and CLI on the GPU (test_cli.py:307-330 shape)."""

import json

import pytest

from paper_2601_10819_b200 import harness
from paper_2601_10819_b200.workload import BenchWorkload


def test_workload_schema_fail_closed():
    assert harness.workload_from_dict({"schema_version": 1}) == BenchWorkload()
    doc = BenchWorkload(cameras=2, level0_size=(8, 8)).to_dict()
    assert harness.workload_from_dict(doc) == BenchWorkload(cameras=2, level0_size=(8, 8))
    for bad in ({"schema_version": 2}, {"schema_version": 1, "camras": 2}, {"schema_version": 1, "cameras": 0},
                {"schema_version": 1, "channels": 1.5}, {"schema_version": 1, "level0_size": [8]},
                {"schema_version": 1, "fps_targets": [0]}, {"schema_version": 1, "cameras": True}, []):
        with pytest.raises(ValueError):
            harness.workload_from_dict(bad)


def test_zero_repetitions_skips_measurement():
    report = harness.bench_msda(BenchWorkload(cameras=2, levels=2, channels=8, queries=16, points_per_query=4,
                                              level0_size=(8, 8), repetitions=0))
    assert report["measured"] is False and "speedup" not in report


def test_cli_rejects_bad_config(tmp_path, capsys):
    cfg = tmp_path / "bad.json"
    cfg.write_text('{"schema_version": 1, "bogus": 3}')
    assert harness.main(["bench-msda", "--config", str(cfg), "--out-dir", str(tmp_path)]) == 1
    cfg.write_text("{not json")
    assert harness.main(["bench-msda", "--config", str(cfg), "--out-dir", str(tmp_path)]) == 1
    assert harness.main([]) == 1


@pytest.mark.gpu
def test_cli_bench_msda_tiny_workload(tmp_path, capsys, cuda_dev):
    cfg = tmp_path / "bench.json"
    cfg.write_text(json.dumps({"schema_version": 1, "cameras": 2, "levels": 2, "channels": 8, "queries": 16,
                               "points_per_query": 4, "level0_size": [8, 8], "repetitions": 1}))
    out_dir = tmp_path / "bench_out"
    assert harness.main(["bench-msda", "--config", str(cfg), "--out-dir", str(out_dir)]) == 0
    assert "speedup" in capsys.readouterr().out
    report = json.loads((out_dir / "bench.json").read_text())
    assert report["measured"] is True and report["mode"] == "full"
    assert report["workload"]["queries"] == 16 and "30" in report["cameras_at_fps"]
    assert report["input_checksum"].startswith("sha256:")
    assert (out_dir / "manifest.json").exists()
