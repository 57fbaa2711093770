"""Host pieces around the profiling step: the UtilMonitor sampler
(Table 1) and the out-of-memory backoff (SPEC on_failure).
The backoff values are SPEC's worked examples; the guarded round that
uses them runs on the GPU (tests/test_gpu_parity.py::test_oom_backoff_guarded)."""
import time

import numpy as np
import pytest

import paper_2207_01053_b200 as pb
from paper_2207_01053_b200.monitor import UtilMonitor, failed_client, oom_backoff


def _profiles(peaks):
    p = np.zeros(len(peaks), dtype=pb.PROFILE_DT)
    for i, pk in enumerate(peaks):
        p[i] = (i + 1, pk, 10, 100, 5, 50, 40, 1, 0)
    return p


def test_oom_backoff_spec_examples():
    # S:459 "vram 2000, backoff 2.0 -> 4000"; "vram 8000, backoff 2.0, device 11264 -> 11264 (clamped)";
    # S:461 "non-failed client unaffected"
    p = _profiles([2000, 8000, 3000])
    q = oom_backoff(p, 1, 2.0)
    assert int(q[0]["peak_bytes"]) == 4000
    q = oom_backoff(p, 2, 2.0, max_bytes=11264)
    assert int(q[1]["peak_bytes"]) == 11264
    assert int(q[0]["peak_bytes"]) == 2000 and int(q[2]["peak_bytes"]) == 3000
    # the failed client's measured fields are cleared, the input is not modified
    assert int(q[1]["step_ns"]) == int(q[1]["train_ns"]) == int(q[1]["sm_ns"]) == 0
    assert int(p[1]["peak_bytes"]) == 8000 and int(p[1]["step_ns"]) == 5
    with pytest.raises(KeyError):
        oom_backoff(p, 99)


def test_failed_client_parses_library_messages():
    assert failed_client("PLAN: run_round: client 17: slot 512 < HWM 1024") == 17
    assert failed_client("no client here") is None


def test_util_monitor_samples_process():
    m = UtilMonitor(interval=0.05)
    m.start()
    t0 = time.perf_counter()
    x = 0.0
    while time.perf_counter() - t0 < 0.3:  # some CPU work in the window
        x += sum(i * i for i in range(1000))
    s = m.stop()
    assert s["samples"] >= 4
    assert s["ram_bytes_peak"] > 0 and s["cpu_pct_peak"] >= 0
    assert s["cpu_time_s"] > 0
