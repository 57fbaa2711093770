"""Batches above 64 rows (GPU): PAPER.md §4.3 gives a third of the clients each batch 32, 1024
and 2048.  Such a batch runs as micro-clients of <= 64 rows that step from the same weights; a merge
kernel forms w + sum_m (b_m / |beta|) (w_m - w) = w - lr * (mean gradient over the whole batch)
(DESIGN.md §5).  Parity against the float64 oracle at the north-star bars, ragged batches where some
micro-clients hold no rows, the observed high-water mark of the split slot, and the paper's B = 1024."""
import dataclasses

import numpy as np
import pytest

import synth
from oracle import profiler as opf
from tests.gpu_helpers import gpu_run, oracle_run, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    t = pytest.importorskip("torch")
    if not t.cuda.is_available():
        pytest.skip("no GPU")
    return t


def _wl(config, sizes_batches, epochs=1, k=None):
    """A config's model / data recipe with explicit (n, B) per client."""
    wl = synth.build_workload(config, n_clients=300 if config == 5 else len(sizes_batches), samples=8,
                              k=len(sizes_batches) if config == 5 else None)
    tmpl = synth.class_templates(wl.shape, wl.classes, wl.seed)
    wl.clients = [dataclasses.replace(c, n=n, batch=B, epochs=epochs)
                  for c, (n, B) in zip(wl.clients, sizes_batches)]
    wl.shards = {c.id: synth.make_shard(tmpl, c.n, c.id, wl.seed) for c in wl.clients}
    return wl


# (n, B): 2 micros; 3 micros with a 22-row last one and a ragged second batch (50 rows: micros 1, 2 idle);
# an ordinary client beside them
CASES = [(200, 128), (200, 150), (40, 16)]


@pytest.mark.parametrize("config", [2, 5])
def test_big_batch_fp32_vs_oracle(torch, config):
    wl = _wl(config, CASES, epochs=2)
    got, ex = gpu_run(wl)
    ref = oracle_run(wl)
    assert rel_l2(got[4], ref[4]) <= 1e-5
    assert rel_l2(got[4] - ex["g0"][4], ref[4] - ex["g0"][4]) <= 1e-4


@pytest.mark.parametrize("config", [2, 5])
def test_big_batch_bf16_vs_oracle(torch, config):
    wl = _wl(config, CASES, epochs=2)
    got, _ = gpu_run(wl, precision=1)
    ref = oracle_run(wl)
    assert rel_l2(got[4], ref[4]) <= 1e-2


def test_big_batch_bf16_teacher_forced(torch):
    """Every step of the micro-split clients against the bf16-emulating oracle (per-step bar 1e-3)."""
    from tests.teacher_forced import bench_round_with_trace, gpu_weights, oracle_updates, per_step_rel
    wl = _wl(2, CASES, epochs=2)
    ids = [c.id for c in wl.clients]
    snaps, _, _ = bench_round_with_trace(wl, 1, ids)
    for cid in ids:
        upd, _ = oracle_updates(wl, cid, snaps[cid], 2, emulate_bf16=True, tol=1e-3)
        tot, _ = per_step_rel(wl, cid, gpu_weights(wl, cid, snaps[cid], 2), upd)
        assert tot.max() <= 1e-3, (cid, float(tot.max()))


def test_big_batch_observed_hwm(torch):
    from paper_2207_01053_b200.sim import Simulation
    for config, prec in ((2, 1), (2, 0), (5, 1)):
        wl = _wl(config, CASES)
        sim = Simulation(precision=prec, arena_bytes=1 << 30)
        mid = sim.register_model(wl.model, 4, 10, 32, 32, 3)
        sim.register_shards([(c.id, *wl.shards[c.id]) for c in wl.clients])
        prof = sim.profile(sim.clients([(c.id, mid, c.batch, c.epochs) for c in wl.clients]))
        eb = 4 if prec == 0 else 2
        for p, c in zip(prof, wl.clients):
            assert int(p["peak_bytes"]) == opf.hwm_bytes(c.model, 4, 10, c.batch, c.n, c.epochs, eb), (config, c)
        sim.close()


def test_paper_batch_1024(torch):
    """One client with the paper's batch of 1024, n = 1024, one step: 16 micro-clients."""
    wl = _wl(2, [(1024, 1024)])
    got, _ = gpu_run(wl)
    ref = oracle_run(wl)
    assert rel_l2(got[4], ref[4]) <= 1e-5
    got16, _ = gpu_run(wl, precision=1)
    assert rel_l2(got16[4], ref[4]) <= 1e-2
