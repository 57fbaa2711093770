"""Full-size parity at the north-star bars, teacher forced (GPU).

The bench's own workload (BASELINE.json configs[1]: 100 CNN-1x clients, 500
samples, B in {8,16,32,64}, E = 2, all co-resident on one GPU, heavy and light
lock-step iterations, deferred side-stream work) runs once with two traced
clients: the B = 8 client (126 steps, it spans every iteration of the round)
and a B = 64 client (16 steps, all in the heavy iterations).  For every one of
their steps the oracle takes one step from the GPU's weights (tests/
teacher_forced.py) taking the GPU's ReLU / max-pool decisions of that step where
they are valid (within rounding of its own: oracle.sgd.forced_*, the rule for
"several correct results"), and the per-step update must agree at BASELINE.json
north_star's bars: rel-L2 <= 1e-5 in the fp32 verification mode against the
float64 oracle; in bf16 mode <= 1e-3 against the oracle's bf16 emulation
 and <= 1e-2 against plain float64.  Config 5 (ResNet-8,
500 clients) is checked the same way on three sampled clients."""
import json
import os

import numpy as np
import pytest

import synth
from tests.teacher_forced import bench_round_with_trace, gpu_weights, oracle_updates, per_step_rel

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REPORT = os.path.join(ROOT, "gpurun_out", "teacher_forced.jsonl")


@pytest.fixture(scope="module")
def torch():
    t = pytest.importorskip("torch")
    if not t.cuda.is_available():
        pytest.skip("no GPU")
    return t


def _report(rec):
    os.makedirs(os.path.dirname(REPORT), exist_ok=True)
    with open(REPORT, "a") as f:
        f.write(json.dumps(rec) + "\n")


def _check(wl, precision, trace_ids, bars, tag):
    """bars: [(emulate_bf16, decision tolerance, per-step bar)]."""
    elem = 4 if precision == 0 else 2
    snaps, st, _ = bench_round_with_trace(wl, precision, trace_ids)
    for cid in trace_ids:
        w = gpu_weights(wl, cid, snaps[cid], elem)
        for emulate, tol, bar in bars:
            upd, forced = oracle_updates(wl, cid, snaps[cid], elem, emulate_bf16=emulate, tol=tol)
            tot, layers = per_step_rel(wl, cid, w, upd)
            vs = "bf16emu" if emulate else "f64"
            _report({"test": tag, "client": int(cid), "steps": int(len(tot)), "vs": vs, "bar": bar,
                     "decision_tol": tol, "forced_decisions": forced,
                     "max": float(tot.max()), "median": float(np.median(tot)),
                     "layers_max": {k: float(v.max()) for k, v in layers.items()},
                     "layers_median": {k: float(np.median(v)) for k, v in layers.items()},
                     "iterations": int(st["iterations"])})
            assert tot.max() <= bar, (tag, cid, vs, float(tot.max()), int(np.argmax(tot)))


def test_config2_full_fp32_every_step(torch):
    wl = synth.build_workload(2)
    _check(wl, 0, [0, 3], [(False, 1e-5, 1e-5)], "config2_fp32")


def test_config2_full_bf16_every_step(torch):
    wl = synth.build_workload(2)
    _check(wl, 1, [0, 3], [(True, 1e-3, 1e-3), (False, 5e-2, 1e-2)], "config2_bf16")


def test_config5_full_bf16_sampled_clients(torch):
    wl = synth.build_workload(5)
    steps = {c.id: synth_steps(c) for c in wl.clients}
    longest = max(steps, key=lambda i: (steps[i], -i))
    b64 = next(c.id for c in wl.clients if c.batch == 64 and c.n > 64)
    ragged = next(c.id for c in wl.clients if c.batch == 16 and c.n % 16 and c.id not in (longest, b64))
    _check(wl, 1, [longest, b64, ragged], [(True, 1e-3, 1e-3), (False, 5e-2, 1e-2)], "config5_bf16")


def synth_steps(c):
    return c.epochs * -(-c.n // c.batch)
