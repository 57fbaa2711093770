"""HeteroFL-style overlapping-width aggregation on the GPU (protea_heterofl_*) against the oracle
(oracle/fedavg.py heterofl_*, pinned in tests/test_oracle_heterofl.py)."""
import numpy as np
import pytest

from oracle import fedavg as fa
from oracle import sgd

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2207_01053_b200.sim import Simulation
    sim = Simulation(arena_bytes=1 << 20)
    yield torch, sim
    sim.close()


@pytest.mark.parametrize("q", [1, 2, 4])
def test_extract_bitwise(env, q):
    import paper_2207_01053_b200 as pb
    torch, sim = env
    g = np.random.default_rng(q).standard_normal(sgd.n_params(sgd.CNN, 4)).astype(np.float32)
    got = pb.protea_heterofl_extract(sim.ctx, torch.tensor(g, device="cuda"), q).cpu().numpy()
    assert np.array_equal(got, fa.heterofl_extract(g, q))


@pytest.mark.parametrize("classes", [10, 62])
def test_aggregate_vs_oracle(env, classes):
    import paper_2207_01053_b200 as pb
    torch, sim = env
    rng = np.random.default_rng(classes)
    g = rng.standard_normal(sgd.n_params(sgd.CNN, 4, classes)).astype(np.float32)
    qs, n = [1, 2, 4, 1, 2], [5, 1, 9, 30, 2]
    ws = [rng.standard_normal(sgd.n_params(sgd.CNN, q, classes)).astype(np.float32) for q in qs]
    got = pb.protea_heterofl_aggregate(sim.ctx, torch.tensor(g, device="cuda"),
                                       [torch.tensor(w, device="cuda") for w in ws], qs, n, classes=classes)
    ref = fa.heterofl_aggregate(g, ws, qs, n, classes).astype(np.float32)
    ulp = np.abs(got.cpu().numpy().view(np.int32).astype(np.int64) - ref.view(np.int32).astype(np.int64))
    assert ulp.max() <= 1


def test_aggregate_errors(env):
    import paper_2207_01053_b200 as pb
    torch, sim = env
    g = torch.zeros(sgd.n_params(sgd.CNN, 4), device="cuda")
    w1 = torch.zeros(sgd.n_params(sgd.CNN, 1), device="cuda")
    for args, name in [(([], [], []), "EMPTY"), (([w1], [3], [1]), "INVALID"), (([w1], [1], [0]), "INVALID")]:
        with pytest.raises(pb.ProteaError) as e:
            pb.protea_heterofl_aggregate(sim.ctx, g, *args)
        assert e.value.name == name
