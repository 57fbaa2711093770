"""Oracle pins for the HeteroFL-style overlapping-width aggregation (R23).

The flat index map is checked against an independent path (per-layer tensor slicing of the unpacked
full model, re-packed at the sub-model width), and the aggregation against vanilla FedAvg (all clients
full width), its fixed point (clients that did not move) and a per-element brute force."""
import numpy as np
import pytest

from oracle import fedavg as fa
from oracle import sgd


def _slice_submodel(full_flat, q, classes=10):
    p = sgd.unpack(np.asarray(full_flat, dtype=np.float64), sgd.CNN, 4, classes)
    c1, c2, f = sgd.cnn_channels(q)
    c2f = sgd.cnn_channels(4)[1]
    sub = {"conv1.W": p["conv1.W"][:c1], "conv1.b": p["conv1.b"][:c1],
           "conv2.W": p["conv2.W"][:c2, :, :, :c1], "conv2.b": p["conv2.b"][:c2],
           "fc1.W": p["fc1.W"].reshape(-1, 8, 8, c2f)[:f, :, :, :c2].reshape(f, 64 * c2), "fc1.b": p["fc1.b"][:f],
           "fc2.W": p["fc2.W"][:, :f], "fc2.b": p["fc2.b"]}
    return sgd.pack(sub, sgd.CNN, q, classes)


@pytest.mark.parametrize("q", [1, 2, 4])
def test_extract_equals_tensor_slicing(q):
    g = np.random.default_rng(q).standard_normal(sgd.n_params(sgd.CNN, 4))
    assert np.array_equal(fa.heterofl_extract(g, q), _slice_submodel(g, q))


def test_full_width_clients_equal_vanilla_fedavg():
    rng = np.random.default_rng(5)
    g = rng.standard_normal(sgd.n_params(sgd.CNN, 4))
    ws = [rng.standard_normal(g.size) for _ in range(3)]
    n = [7, 1, 30]
    np.testing.assert_allclose(fa.heterofl_aggregate(g, ws, [4, 4, 4], n), fa.fedavg(ws, n), rtol=1e-13, atol=1e-15)


def test_unmoved_clients_are_a_fixed_point():
    g = np.random.default_rng(6).standard_normal(sgd.n_params(sgd.CNN, 4))
    qs = [1, 2, 1, 4, 2]
    out = fa.heterofl_aggregate(g, [fa.heterofl_extract(g, q) for q in qs], qs, [3, 1, 4, 1, 5])
    np.testing.assert_allclose(out, g, rtol=1e-14, atol=1e-15)


def test_elements_brute_force():
    rng = np.random.default_rng(7)
    P = sgd.n_params(sgd.CNN, 4)
    g = rng.standard_normal(P)
    qs, n = [1, 2, 2, 4], [2, 3, 5, 7]
    ws = [rng.standard_normal(sgd.n_params(sgd.CNN, q)) for q in qs]
    out = fa.heterofl_aggregate(g, ws, qs, n)
    maps = [fa.heterofl_index_map(q) for q in qs]
    inv = [dict(zip(m.tolist(), range(m.size))) for m in maps]
    for i in rng.choice(P, 400, replace=False).tolist() + [0, P - 1]:
        num = den = 0.0
        for k in range(4):
            if i in inv[k]:
                num += n[k] * ws[k][inv[k][i]]
                den += n[k]
        ref = g[i] if den == 0 else num / den
        assert abs(out[i] - ref) <= 1e-12 * max(1.0, abs(ref))
    # width-1 elements are held by every client, elements only the width-4 client holds keep its value
    only4 = np.setdiff1d(maps[3], maps[2])
    np.testing.assert_allclose(out[only4], ws[3][only4], rtol=1e-15, atol=0)


def test_errors():
    g = np.zeros(sgd.n_params(sgd.CNN, 4))
    w1 = np.zeros(sgd.n_params(sgd.CNN, 1))
    for args, code in [(([], [], []), "EMPTY"), (([w1], [3], [1]), "INVALID"), (([w1], [1], [0]), "INVALID"),
                       (([w1], [2], [1]), "DIM")]:
        with pytest.raises(fa.FedAvgError) as e:
            fa.heterofl_aggregate(g, *args)
        assert e.value.code == code
