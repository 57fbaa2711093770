"""Observed arena high-water marks (GPU).

PAPER.md Table 1 "VRAM" and get_properties() ("How much
VRAM is the training making use of?") are read as the per-client peak
(reading R2).  The library OBSERVES it: the client's slot is poisoned, the
client runs, and the highest byte that differs from the poison is its
high-water mark.  These tests check the observation against the hand-pinned
slot-layout formula (oracle.profiler.hwm_bytes, tests/golden/hwm.json) and
that no kernel writes outside its client's slot."""
import numpy as np
import pytest

import synth
from oracle import profiler as opf

pytestmark = pytest.mark.gpu

POISON = 0xA5


@pytest.fixture(scope="module")
def torch():
    t = pytest.importorskip("torch")
    if not t.cuda.is_available():
        pytest.skip("no GPU")
    return t


def _sim(wl, precision, arena=1 << 30, widths=(4,)):
    from paper_2207_01053_b200.sim import Simulation
    H, W, C = synth.INPUT_SHAPE[wl.model]
    sim = Simulation(precision=precision, arena_bytes=arena)
    mids = {w: sim.register_model(synth.LIB_ARCH[wl.model], w, wl.classes, H, W, C) for w in widths}
    sim.register_shards([(c.id, *wl.shards[c.id]) for c in wl.clients])
    clients = sim.clients([(c.id, mids[c.width_q], c.batch, c.epochs) for c in wl.clients])
    return sim, clients


CASES = [  # (config, build kwargs, precision, widths)
    (1, dict(n_clients=4, samples=20), 0, (4,)),
    (1, dict(n_clients=4, samples=20), 1, (4,)),
    (2, dict(n_clients=8, samples=70), 0, (4,)),
    (2, dict(n_clients=8, samples=70), 1, (4,)),
    (4, dict(n_clients=300, k=12, samples=70), 1, (1, 2, 4)),
    (5, dict(n_clients=300, k=8, samples=70), 1, (4,)),
    (5, dict(n_clients=300, k=8, samples=70), 0, (4,)),
    (6, dict(n_clients=300, k=6, samples=70), 1, (4,)),
    (7, dict(n_clients=4, samples=20), 1, (4,)),
    (7, dict(n_clients=4, samples=20), 0, (4,)),
]


@pytest.mark.parametrize("config,kw,precision,widths", CASES)
def test_probe_observed_hwm_equals_layout(torch, config, kw, precision, widths):
    """protea_profile_clients' observed peak == the pinned layout formula for every client with n_k >= B_k
    (a client whose every batch is partial may leave the tail of its last buffers untouched: <=)."""
    wl = synth.build_workload(config, **kw)
    sim, clients = _sim(wl, precision, widths=widths)
    prof = sim.profile(clients)
    eb = 4 if precision == 0 else 2
    bad = []
    for p, c in zip(prof, wl.clients):
        want = opf.hwm_bytes(c.model, c.width_q, c.classes, c.batch, c.n, c.epochs, eb)  # (CNN28 / RESNET18 ids)
        got = int(p["peak_bytes"])
        if (c.n >= c.batch and got != want) or got > want:
            bad.append((c.id, c.width_q, c.batch, c.n, got, want))
    sim.close()
    assert not bad, bad


def test_round_observed_hwm_and_no_write_outside_slots(torch):
    """A bf16 config-2 round and a config-5 round with observe_hwm: the whole arena is poisoned first, slots
    are planned with a 10 % margin (so every slot ends in an unused tail); afterwards every byte outside
    [offset, offset + HWM) of every slot is still poison, and measured.peak_bytes (the observation over
    the client's whole lifetime) equals the layout formula."""
    for config, kw in ((2, dict(n_clients=12, samples=40)), (5, dict(n_clients=300, k=10, samples=70))):
        wl = synth.build_workload(config, **kw)
        sim, clients = _sim(wl, 1)
        prof = sim.profile(clients)
        plan, _ = sim.plan(prof, margin_permille=1100)
        sim.arena.fill_(POISON)
        g = torch.tensor(synth.init_weights(wl.model), device="cuda")
        _, (st, meas) = sim.run_round(clients, plan, g, lr=0.05, seed=wl.seed, measured=True, observe_hwm=True)
        arena = sim.arena.cpu().numpy()
        touched = np.zeros(arena.size, dtype=bool)
        byid = {int(p["client_id"]): int(p["peak_bytes"]) for p in meas}
        for a, c in zip(plan, wl.clients):
            off, slot = int(a["offset"]), int(a["slot"])
            hw = byid[c.id]
            assert hw == opf.hwm_bytes(c.model, c.width_q, c.classes, c.batch, c.n, c.epochs, 2) or \
                (c.n < c.batch and hw <= slot), (config, c.id, hw)
            assert slot >= hw
            touched[off:off + hw] = True
        outside = arena[~touched]
        assert outside.size > 0 and np.all(outside == POISON), (config, int(np.sum(outside != POISON)))
        sim.close()


def test_probe_guard_detects_nothing_and_oom_when_arena_small(torch):
    wl = synth.build_workload(2, n_clients=2, samples=16)
    eb = 2
    need = max(opf.hwm_bytes(c.model, 4, 10, c.batch, c.n, c.epochs, eb) for c in wl.clients)
    import paper_2207_01053_b200 as pb
    sim, clients = _sim(wl, 1, arena=need + 1024)  # a slot fits, slot + 4 KiB guard does not
    with pytest.raises(pb.ProteaError) as e:
        sim.profile(clients)
    assert e.value.name == "OOM"
    sim.close()


def test_resnet8_small_shard_observed_hwm_equals_layout(torch):
    """ResNet-8 clients whose shard is smaller than their batch (b = n < B: every batch is the whole shard)
    and ragged ones: the whole-image weight-gradient splits (common.h r8_split_cap, a balanced partition)
    touch every reserved partial, so the OBSERVED mark equals the layout exactly -- a plan from observed
    profiles must never undersize the slot run_round validates against (bench.py feeds them back)."""
    import dataclasses
    wl = synth.build_workload(5, n_clients=300, k=6, samples=70)
    shapes = [(5, 16), (9, 32), (13, 16), (7, 64), (21, 32), (45, 16)]  # (n, B)
    tmpl = synth.class_templates(wl.shape, wl.classes, wl.seed)
    wl.clients = [dataclasses.replace(c, n=n, batch=b, epochs=1) for c, (n, b) in zip(wl.clients, shapes)]
    wl.shards = {c.id: synth.make_shard(tmpl, c.n, c.id, wl.seed) for c in wl.clients}
    sim, clients = _sim(wl, 1)
    prof = sim.profile(clients)
    plan, _ = sim.plan(prof, margin_permille=1100)
    g = torch.tensor(synth.init_weights(wl.model), device="cuda")
    _, (st, meas) = sim.run_round(clients, plan, g, lr=0.05, seed=wl.seed, measured=True, observe_hwm=True)
    bad = []
    for p, c in zip(meas, wl.clients):
        want = opf.hwm_bytes(c.model, c.width_q, c.classes, c.batch, c.n, c.epochs, 2)
        if int(p["peak_bytes"]) != want:
            bad.append((c.id, c.n, c.batch, int(p["peak_bytes"]), want))
    for p, c in zip(prof, wl.clients):  # the one-step probe observes the same marks
        want = opf.hwm_bytes(c.model, c.width_q, c.classes, c.batch, c.n, c.epochs, 2)
        if int(p["peak_bytes"]) != want:
            bad.append(("probe", c.id, c.n, c.batch, int(p["peak_bytes"]), want))
    sim.close()
    assert not bad, bad
