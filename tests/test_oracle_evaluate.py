"""Pins of oracle/evaluate.py (forward-only client evaluation).

* logits equal an independently written torch float64 model (tests/test_oracle_sgd.torch_forward);
* loss_sum / n equals the training loss of oracle/sgd.loss_and_grad on the same batch (mean CE);
* all-zero weights give logits 0: loss_sum = n ln C and every prediction is class 0 (first maximum)."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import synth  # noqa: E402
from oracle import evaluate as oev  # noqa: E402
from oracle import sgd  # noqa: E402
from tests.test_oracle_sgd import torch_forward  # noqa: E402


def _data(model, n, seed, classes=10):
    rng = np.random.default_rng(seed)
    shape = (28, 28, 1) if model == sgd.MLP else (32, 32, 3)
    x = rng.integers(0, 256, size=(n,) + shape, dtype=np.uint8)
    y = rng.integers(0, classes, size=n)
    return x, y


@pytest.mark.parametrize("model,wq", [(sgd.MLP, 4), (sgd.CNN, 1), (sgd.CNN, 4), (sgd.RESNET8, 4)])
def test_logits_vs_torch(model, wq):
    w = synth.init_weights(model, wq, 10, seed=3).astype(np.float64)
    x, _ = _data(model, 5, 1)
    z = oev.logits(w, model, wq, 10, x)
    zt = torch_forward(model, wq, 10, torch.tensor(w), torch.tensor(x / 255.0)).numpy()
    assert np.max(np.abs(z - zt)) <= 1e-12 * max(1.0, np.max(np.abs(zt)))


@pytest.mark.parametrize("model", [sgd.MLP, sgd.CNN, sgd.RESNET8])
def test_loss_equals_training_loss(model):
    w = synth.init_weights(model, 4, 10, seed=5).astype(np.float64)
    x, y = _data(model, 7, 2)
    loss_sum, correct, n = oev.evaluate(w, model, 4, 10, x, y)
    lt, _ = sgd.loss_and_grad(sgd.unpack(w, model, 4, 10), model, x / 255.0, y)
    assert n == 7 and 0 <= correct <= 7
    assert abs(loss_sum / n - lt) <= 1e-12


def test_zero_weights_closed_form():
    w = np.zeros(sgd.n_params(sgd.CNN, 1, 10))
    x, y = _data(sgd.CNN, 6, 4)
    loss_sum, correct, n = oev.evaluate(w, sgd.CNN, 1, 10, x, y)
    assert abs(loss_sum - 6 * math.log(10)) <= 1e-12
    assert correct == int(np.sum(y == 0))


def test_evaluate_round_is_the_per_client_sum():
    """evaluate_round = each client's evaluate() on its own split with its group's weights; totals = sums."""
    wl = synth.build_workload(4, k=6, samples=20)
    tmpl = synth.class_templates(wl.shape, wl.classes, wl.seed)
    val = {c.id: synth.make_val_shard(tmpl, c.n, c.id, wl.seed) for c in wl.clients}
    g = {q: synth.init_weights(sgd.CNN, q, 10, seed=q).astype(np.float64) for q in (1, 2, 4)}
    per, tot = oev.evaluate_round(wl.clients, val, g)
    for c in wl.clients:
        x, y = val[c.id]
        assert per[c.id] == oev.evaluate(g[c.width_q], sgd.CNN, c.width_q, 10, x.reshape(-1, 32, 32, 3), y)
        assert per[c.id][2] == synth.val_size(c.n) == max(1, round(c.n / 9))
    assert tot[2] == sum(v[2] for v in per.values()) and tot[1] == sum(v[1] for v in per.values())


def test_resnet18_logits_vs_torch():
    from tests.test_oracle_sgd import torch_resnet18
    w = synth.init_weights(sgd.RESNET18, 4, 10, seed=3).astype(np.float64)
    x, _ = _data(sgd.RESNET18, 2, 1)
    z = oev.logits(w, sgd.RESNET18, 4, 10, x)
    zt = torch_resnet18(torch.tensor(w), torch.tensor(x / 255.0)).numpy()
    assert np.max(np.abs(z - zt)) <= 1e-11 * max(1.0, np.max(np.abs(zt)))
