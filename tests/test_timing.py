"""Stage timing harness (bench.py drop-in): CSV format and recorders."""

import pytest

from paper_2112_10258_b200 import timing


def test_csv_roundtrip_and_format(tmp_path):
    rows = [timing.StageTiming("convolution", 0, 1, 1, 32, 1234.5678901234),
            timing.StageTiming("orient", -1, -1, 1, 32, 7.0)]
    p = tmp_path / "t.csv"
    timing.emit_csv(rows, p)
    assert p.read_text().splitlines() == ["stage,octave,level,workers,chunk,wall_micros",
                                          "convolution,0,1,1,32,1234.56789", "orient,-1,-1,1,32,7"]
    back = timing.read_csv(p)
    assert [(r.stage, r.octave, r.level, r.workers, r.chunk) for r in back] == [
        (r.stage, r.octave, r.level, r.workers, r.chunk) for r in rows]


def test_host_recorder():
    rec = timing.StageRecorder(workers=2, chunk=8)
    with rec.stage("dog", 1, 2):
        pass
    (s,) = rec.samples
    assert (s.stage, s.octave, s.level, s.workers, s.chunk) == ("dog", 1, 2, 2, 8) and s.wall_micros >= 0


@pytest.mark.gpu
def test_time_pipeline_device_clock():
    import numpy as np

    import paper_2112_10258_b200 as vk
    from paper_2112_10258_b200 import synthetic

    vol = vk.Volume(synthetic.random_blob_phantom((40, 44, 36), np.random.default_rng(7), n_blobs=10, margin=6))
    for dev in (False, True):
        summ = timing.time_pipeline(vol, vk.PipelineConfig(), repeats=2, device_clock=dev)
        stages = {m.stage for m in summ.means}
        assert {"convolution", "orient", "descriptor"} <= stages, stages
        assert all(m.wall_micros >= 0 for m in summ.means) and summ.total_mean_micros > 0
