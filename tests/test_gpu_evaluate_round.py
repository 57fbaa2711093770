"""Evaluate round (GPU): PAPER.md P:238 (configure_evaluate / aggregate_evaluate after aggregation) on each
client's validation split (P:302, 10 % of its data; synth.make_val_shard).  The library runs the training
path's forward kernels (bf16: tcgen05 for the CNN and ResNet-8; fp32: SIMT) over all clients in
lock-step, then a classifier head; oracle/evaluate.py is the reference.  Loss sums per client within the
precision's bar; the number correct exactly, except for samples whose oracle top-2 logit margin is
within the forward pass's rounding (an argmax decided by rounding: both answers are valid)."""
import dataclasses

import numpy as np
import pytest

import synth
from oracle import evaluate as oev
from tests.gpu_helpers import arch_of, gpu_run, shape_of, widths_of

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    t = pytest.importorskip("torch")
    if not t.cuda.is_available():
        pytest.skip("no GPU")
    return t


def _margin_count(w, c, x, y, tol):
    """samples whose oracle top-2 margin is below tol x the logit scale (their argmax may go either way)."""
    H, W, C = shape_of(c.model)
    z = oev.logits(w, c.model, c.width_q, c.classes, x.reshape(-1, H, W, C))
    s = np.sort(z, axis=1)
    return int(np.sum(s[:, -1] - s[:, -2] <= tol * max(1.0, np.max(np.abs(z)))))


CASES = [(1, dict(n_clients=6, samples=90)), (4, dict(k=9, samples=60)), (5, dict(n_clients=300, k=6, samples=80)),
         (2, dict(n_clients=3, samples=700)),  # config 2: 78 validation rows -> two micro-clients
         (6, dict(n_clients=200, k=5, samples=120)),  # FEMNIST-shaped CNN, 62 classes
         (7, dict(n_clients=3, samples=40))]  # ResNet-18 (GroupNorm)


@pytest.mark.parametrize("precision", [0, 1])
@pytest.mark.parametrize("config,kw", CASES)
def test_evaluate_round_vs_oracle(torch, config, kw, precision):
    from paper_2207_01053_b200.sim import Simulation, concat_globals
    wl = synth.build_workload(config, epochs=1, **kw)
    widths = widths_of(wl)
    tmpl = synth.class_templates(wl.shape, wl.classes, wl.seed)
    val = {c.id: synth.make_val_shard(tmpl, c.n, c.id, wl.seed) for c in wl.clients}
    trained, _ = gpu_run(wl, precision=0)  # a trained global model (one fp32 round) to evaluate
    sim = Simulation(precision=precision, arena_bytes=1 << 30)
    H, W, C = shape_of(wl.model)
    mids = {q: sim.register_model(arch_of(wl.model), q, wl.classes, H, W, C) for q in widths}
    sim.register_val_shards([(c.id, *val[c.id]) for c in wl.clients])
    clients = sim.clients([(c.id, mids[c.width_q], c.batch, c.epochs) for c in wl.clients])
    g = torch.tensor(concat_globals([trained[q] for q in widths]), device="cuda")
    per, tot = sim.evaluate_round(clients, g)
    ref, rtot = oev.evaluate_round(wl.clients, val, {q: trained[q].astype(np.float64) for q in widths})
    loss_tol, dec_tol = (1e-5, 1e-5) if precision == 0 else (2e-2, 5e-2)
    for p, c in zip(per, wl.clients):
        rl, rc, rn = ref[c.id]
        assert int(p["n"]) == rn == synth.val_size(c.n)
        assert abs(float(p["loss_sum"]) - rl) <= loss_tol * max(abs(rl), 1e-3), (c.id, float(p["loss_sum"]), rl)
        free = _margin_count(trained[c.width_q].astype(np.float64), c, *val[c.id], dec_tol)
        assert abs(int(p["correct"]) - rc) <= free, (c.id, int(p["correct"]), rc, free)
    assert tot[2] == rtot[2] and abs(tot[0] - rtot[0]) <= loss_tol * abs(rtot[0])
    sim.close()


def test_evaluate_round_errors(torch):
    import paper_2207_01053_b200 as pb
    from paper_2207_01053_b200.sim import Simulation
    wl = synth.build_workload(2, n_clients=2, samples=20)
    sim = Simulation(precision=1, arena_bytes=1 << 28)
    mid = sim.register_model(wl.model, 4, 10, 32, 32, 3)
    clients = sim.clients([(c.id, mid, c.batch, c.epochs) for c in wl.clients])
    g = torch.tensor(synth.init_weights(wl.model), device="cuda")
    with pytest.raises(pb.ProteaError) as e:  # no validation split registered
        sim.evaluate_round(clients, g)
    assert e.value.name == "INVALID"
    tmpl = synth.class_templates(wl.shape, wl.classes, wl.seed)
    sim.register_val_shards([(c.id, *synth.make_val_shard(tmpl, c.n, c.id, wl.seed)) for c in wl.clients])
    with pytest.raises(pb.ProteaError) as e:
        sim.evaluate_round(clients, g[:-1])
    assert e.value.name == "DIM"
    per, tot = sim.evaluate_round(clients, g)
    assert tot[2] == sum(synth.val_size(c.n) for c in wl.clients)
    sim.close()
