"""K7 cross-rank exchange and the run_round validation contract (GPU).

SURVEY §8(e): the only exchange of a round is the sum over ranks of the per-GPU
FedAvg partials sum_{k in g} n_k (w_k - w_g); its deterministic form gathers
the partials and reduces them in rank order.  protea_run_round with a
communicator runs ncclAllGather + the rank-ordered finalise kernel; the same
kernel is reachable without NCCL through protea_round_finalize_ordered, so
the multi-rank result is pinned here on one GPU against a host rank-ordered
fp64 sum (bitwise), and the communicator path itself runs with a one-rank
NCCL communicator (bitwise equal to the communicator-free round)."""
import numpy as np
import pytest

import synth
from tests.gpu_helpers import gpu_run

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    t = pytest.importorskip("torch")
    if not t.cuda.is_available():
        pytest.skip("no GPU")
    return t


def _rank_partials(torch, wl, world, precision=0):
    """Virtual ranks on one GPU: rank r runs only its planned clients (partial_only) -> fp64 partials."""
    import paper_2207_01053_b200 as pb
    from paper_2207_01053_b200.sim import Simulation
    w0 = torch.tensor(synth.init_weights(wl.model), device="cuda")
    parts, sims = [], []
    for rank in range(world):
        sim = Simulation(precision=precision, arena_bytes=1 << 30, rank=rank, world=world)
        mid = sim.register_model(wl.model, 4, 10, 32, 32, 3)
        sim.register_shards([(c.id, *wl.shards[c.id]) for c in wl.clients])
        cl = sim.clients([(c.id, mid, c.batch, c.epochs) for c in wl.clients])
        plan, _ = sim.plan(sim.profile(cl), caps=[1 << 30] * world)
        sim.run_round(cl, plan, w0, torch.empty_like(w0), lr=0.05, seed=wl.seed, rnd=0, partial_only=True)
        part = torch.empty(w0.numel(), dtype=torch.float64, device="cuda")
        pb.protea_round_partial(sim.ctx, part)
        parts.append(part)
        sims.append(sim)
    return w0, torch.stack(parts), sims


def test_rank_ordered_finalise_bitwise(torch):
    """protea_round_finalize_ordered == host fp64 ((p0 + p1) + p2) + p3, then w_g + acc / N rounded once
    (reading R20), bit for bit; and it differs from a different summation order only by rounding."""
    import paper_2207_01053_b200 as pb
    wl = synth.build_workload(3, k=12, samples=10, epochs=1)
    world = 4
    w0, parts, sims = _rank_partials(torch, wl, world)
    out = torch.empty_like(w0)
    pb.protea_round_finalize_ordered(sims[0].ctx, parts, w0, out)
    P = parts.cpu().numpy()
    acc = P[0].copy()
    for r in range(1, world):
        acc = acc + P[r]
    N = float(sum(c.n for c in wl.clients))
    ref = (w0.cpu().numpy().astype(np.float64) + acc / N).astype(np.float32)
    assert np.array_equal(out.cpu().numpy().view(np.int32), ref.view(np.int32))
    # host-side partials give the same bits (device or host pointer)
    out2 = torch.empty_like(w0)
    pb.protea_round_finalize_ordered(sims[0].ctx, parts.cpu(), w0.cpu(), out2)
    assert torch.equal(out, out2)
    # the single-rank round on the same clients agrees to <= 1 ulp (fp64 accumulation, other order)
    one, _ = gpu_run(wl)
    ulp = np.abs(out.cpu().numpy().view(np.int32).astype(np.int64) - one[4].view(np.int32).astype(np.int64))
    assert ulp.max() <= 1
    with pytest.raises(pb.ProteaError) as e:
        pb.protea_round_finalize_ordered(sims[0].ctx, parts[:, :-1].contiguous(), w0[:-1], out[:-1])
    assert e.value.name == "DIM"
    for s in sims:
        s.close()


def test_one_rank_communicator_path_bitwise(torch):
    """run_round with an NCCL communicator (world = 1): plan agreement + error-flag exchange + ncclAllGather
    + the rank-ordered finalise; bitwise equal to the communicator-free round."""
    from paper_2207_01053_b200.sim import Simulation
    wl = synth.build_workload(2, n_clients=4, samples=16, epochs=1)
    ref, _ = gpu_run(wl, precision=1)
    nid = torch.cuda.nccl.unique_id()
    sim = Simulation(precision=1, arena_bytes=1 << 30, rank=0, world=1, nccl_id=nid)
    got, _ = gpu_run(wl, precision=1, sim=sim)
    assert np.array_equal(got[4].view(np.int32), ref[4].view(np.int32))


def test_validation_errors(torch):
    """labels outside [0, classes) and a model with another input size are rejected before any
    device work (INVALID), in run_round and in profile_clients."""
    import paper_2207_01053_b200 as pb
    from paper_2207_01053_b200.sim import Simulation
    wl = synth.build_workload(2, n_clients=2, samples=8, epochs=1)
    sim = Simulation(precision=1, arena_bytes=1 << 28)
    mid = sim.register_model(synth.MODEL_CNN, 4, 10, 32, 32, 3)
    with pytest.raises(pb.ProteaError) as e:  # MLP (784-byte examples) beside a 3072-byte CNN
        sim.register_model(synth.MODEL_MLP, 4, 10, 28, 28, 1)
    assert e.value.name == "INVALID"
    x, y = wl.shards[wl.clients[0].id]
    y_bad = y.copy()
    y_bad[3] = 10
    sim.register_shards([(wl.clients[0].id, x, y_bad), (wl.clients[1].id, *wl.shards[wl.clients[1].id])])
    cl = sim.clients([(c.id, mid, c.batch, c.epochs) for c in wl.clients])
    with pytest.raises(pb.ProteaError) as e:
        sim.profile(cl)
    assert e.value.name == "INVALID" and "label" in str(e.value)
    foot = np.zeros(len(cl), dtype=pb.PROFILE_DT)
    for i, c in enumerate(wl.clients):
        pk, st, fl = pb.protea_client_footprint(pb.MODEL_CNN, 4, 10, 32, 32, 3, c.n, c.batch, c.epochs, 1)
        foot[i] = (c.id, pk, st, fl, 0, 0, 0, 1, 0)
    plan, _ = sim.plan(foot)
    g = torch.tensor(synth.init_weights(wl.model), device="cuda")
    with pytest.raises(pb.ProteaError) as e:
        sim.run_round(cl, plan, g)
    assert e.value.name == "INVALID" and "label" in str(e.value)
    y_neg = y.copy()
    y_neg[0] = -1
    sim.register_shards([(wl.clients[0].id, x, y_neg)])
    with pytest.raises(pb.ProteaError) as e:
        sim.run_round(cl, plan, g)
    assert e.value.name == "INVALID"
    sim.register_shards([(wl.clients[0].id, x, y)])  # valid again: the round runs
    sim.run_round(cl, plan, g)
    sim.close()
