"""ThroughputReport mirror (evaluate.py:83-125), restating the cases of the
reference's TestThroughput (pkg/tests/test_evaluate.py:124-150) and its
evaluation-arithmetic acceptance criterion (test_acceptance.py:214-219)."""
import json

import numpy as np
import pytest

from paper_2403_16438_b200.pipeline import MIN_STAGE_SECONDS, ThroughputReport, throughput_report


def test_arithmetic_against_real_time():
    # 10,000 frames in 5.5 + 6.9 + 0.1 s = 800 frames/s; 741 frames/s real time -> 1.08
    rep = throughput_report(10_000, {"motion": 5.5, "segment": 6.9, "trace": 0.1}, target_fps=741.0)
    assert isinstance(rep, ThroughputReport)
    assert rep.total_seconds == pytest.approx(12.5)
    assert rep.effective_fps == pytest.approx(800.0)
    assert rep.realtime_ratio == pytest.approx(1.08, abs=0.01)


def test_tiny_totals_clamp_to_one_millisecond():
    rep = throughput_report(100, {"motion": 1e-9})
    assert MIN_STAGE_SECONDS == 1e-3
    assert rep.total_seconds == MIN_STAGE_SECONDS
    assert np.isfinite(rep.effective_fps) and rep.effective_fps == pytest.approx(1e5)


def test_explicit_total_for_overlapped_stages():
    rep = throughput_report(100, {"a": 1.0, "b": 1.0}, total_seconds=1.5)
    assert rep.total_seconds == 1.5
    assert rep.stage_seconds == {"a": 1.0, "b": 1.0}


def test_without_target_rate():
    rep = throughput_report(100, {"a": 1.0})
    assert rep.realtime_ratio is None and rep.target_fps is None
    assert rep.effective_fps == pytest.approx(100.0)


def test_json_fields_and_round_trip():
    stages = {"motion": 0.5}
    rep = throughput_report(50, stages, target_fps=100.0)
    stages["motion"] = 9.0  # the report keeps its own copy
    d = json.loads(rep.to_json())
    assert list(d) == ["stage_seconds", "total_seconds", "frames", "effective_fps", "target_fps", "realtime_ratio"]
    assert d["frames"] == 50 and d["stage_seconds"] == {"motion": 0.5}
    assert d["realtime_ratio"] == pytest.approx(1.0)
