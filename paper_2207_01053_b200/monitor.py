"""Host-side pieces around the profiling step: the paper's
UtilMonitor sampler and the out-of-memory failure path.

* ``UtilMonitor`` — a ``threading.Thread`` that samples the process's CPU load,
  RAM, CPU time and the GPU's compute utilisation and memory every 0.7 s
  (Table 1 and the paragraph after it: psutil for the
  process, nvidia-smi via gputil for the GPU; here psutil and NVML).  All
  clients of a GPU run inside the same process and the same grouped kernels,
  so these are per-process figures; the per-client VRAM and CUDA_time of
  Table 1 come exactly from the library (``protea_profile.peak_bytes``,
  ``train_ns``, ``sm_ns``).
* ``oom_backoff`` / ``Simulation.run_round_guarded`` — SPEC's ``on_failure``
  (S:454-462): a client whose allocation proved too small gets its memory
  estimate multiplied by the backoff factor (clamped to the device capacity),
  its measured fields cleared, and the round is re-planned.  With exact
  high-water marks this only triggers when a caller plans from a stale or
  hand-made profile; the library rejects such a plan before any device work
  (``PROTEA_ERR_PLAN``: slot < HWM), so no client state is lost.
"""
from __future__ import annotations

import re
import threading
import time

import numpy as np

try:  # optional: NVML through nvidia-ml-py
    import pynvml as _nvml
except Exception:  # pragma: no cover - image without the package
    _nvml = None

try:
    import psutil as _psutil
except Exception:  # pragma: no cover
    _psutil = None


class UtilMonitor(threading.Thread):
    """Samples CPU %, RSS, CPU time, GPU % and GPU memory every ``interval`` s until ``stop()``."""

    def __init__(self, device: int = 0, interval: float = 0.7):
        super().__init__(daemon=True)
        self.interval = interval
        self.samples = []
        self._lock = threading.Lock()
        self._stop_ev = threading.Event()
        self._proc = _psutil.Process() if _psutil else None
        self._gpu = None
        if _nvml is not None:
            try:
                _nvml.nvmlInit()
                self._gpu = _nvml.nvmlDeviceGetHandleByIndex(device)
            except Exception:
                self._gpu = None
        if self._proc is not None:
            self._proc.cpu_percent(None)  # prime the interval counter

    def _sample(self):
        s = {"t": time.perf_counter()}
        if self._proc is not None:
            ct = self._proc.cpu_times()
            s.update(cpu_pct=self._proc.cpu_percent(None), ram_bytes=self._proc.memory_info().rss,
                     cpu_time_s=ct.user + ct.system)
        if self._gpu is not None:
            try:
                u = _nvml.nvmlDeviceGetUtilizationRates(self._gpu)
                m = _nvml.nvmlDeviceGetMemoryInfo(self._gpu)
                s.update(gpu_pct=float(u.gpu), vram_used_bytes=int(m.used), vram_total_bytes=int(m.total))
            except Exception:
                pass
        with self._lock:
            self.samples.append(s)

    def run(self):
        while not self._stop_ev.is_set():
            self._sample()
            self._stop_ev.wait(self.interval)

    def stop(self) -> dict:
        self._stop_ev.set()
        if self.is_alive():
            self.join()
        self._sample()  # closing sample: CPU time and counters at the end of the window
        return self.summary()

    def summary(self) -> dict:
        with self._lock:
            ss = list(self.samples)
        out = {"samples": len(ss), "interval_s": self.interval}
        for key in ("cpu_pct", "ram_bytes", "gpu_pct", "vram_used_bytes"):
            v = [s[key] for s in ss if key in s]
            if v:
                out[key + "_mean"] = float(np.mean(v))
                out[key + "_peak"] = float(np.max(v))
        ct = [s["cpu_time_s"] for s in ss if "cpu_time_s" in s]
        if len(ct) >= 2:
            out["cpu_time_s"] = ct[-1] - ct[0]
        return out


def oom_backoff(profiles, client_id: int, factor: float = 2.0, max_bytes: int | None = None):
    """SPEC on_failure: copy of ``profiles`` where client ``client_id``'s peak_bytes is
    multiplied by ``factor`` (clamped to ``max_bytes``) and its measured fields are cleared."""
    p = np.array(profiles, copy=True)
    sel = p["client_id"] == client_id
    if not sel.any():
        raise KeyError(f"client {client_id} not in the profiles")
    peak = np.ceil(p["peak_bytes"][sel].astype(np.float64) * factor).astype(np.uint64)
    if max_bytes is not None:
        peak = np.minimum(peak, np.uint64(max_bytes))
    p["peak_bytes"][sel] = peak
    for f in ("step_ns", "train_ns", "sm_ns"):
        p[f][sel] = 0
    return p


_CLIENT_RE = re.compile(r"client (-?\d+)")


def failed_client(message: str):
    """Client id named by a library error message (protea_last_error names the offending client)."""
    m = _CLIENT_RE.search(message)
    return int(m.group(1)) if m else None
