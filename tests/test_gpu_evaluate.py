"""protea_evaluate (forward-only client evaluation on a validation
split) against oracle/evaluate.py on the same seeded inputs: loss sum within
the fp32 tolerance, accuracy exact except where the oracle's top-2 logit margin is
below the fp32 rounding of the forward pass (an argmax decided by rounding)."""
import numpy as np
import pytest

import synth
from oracle import evaluate as oev

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    t = pytest.importorskip("torch")
    if not t.cuda.is_available():
        pytest.skip("no GPU")
    return t


def _val_split(model, n, seed, classes=10):
    shape = synth.FEMNIST if model == synth.MODEL_MLP else synth.CIFAR
    x, y = synth.make_shard(synth.class_templates(shape, classes, seed), n, 7, seed)
    return x.reshape(n, shape["H"], shape["W"], shape["C"]), y


@pytest.mark.parametrize("model,wq,n", [(synth.MODEL_CNN, 4, 45), (synth.MODEL_CNN, 1, 150),
                                        (synth.MODEL_CNN, 2, 64), (synth.MODEL_MLP, 4, 130)])
def test_evaluate_matches_oracle(torch, model, wq, n):
    import paper_2207_01053_b200 as pb
    from paper_2207_01053_b200.sim import Simulation
    H, W, C = (28, 28, 1) if model == synth.MODEL_MLP else (32, 32, 3)
    x, y = _val_split(model, n, 3)
    w = synth.init_weights(model, wq, 10, seed=11)
    sim = Simulation(precision=pb.PREC_FP32, arena_bytes=1 << 26)
    mid = sim.register_model(model, wq, 10, H, W, C)
    loss, correct, cnt = sim.evaluate(mid, torch.tensor(w, device="cuda"), x, y)
    loss_h, correct_h, _ = sim.evaluate(mid, w.astype(np.float32), x, y)  # host weights, same result
    sim.close()
    ref_loss, ref_correct, ref_n = oev.evaluate(w, model, wq, 10, x, y)
    assert cnt == ref_n == n
    assert abs(loss - ref_loss) <= 1e-5 * abs(ref_loss)
    assert loss_h == loss and correct_h == correct
    z = np.sort(oev.logits(w, model, wq, 10, x), axis=1)
    near = int(np.sum(z[:, -1] - z[:, -2] < 1e-4 * np.maximum(1.0, np.abs(z[:, -1]))))
    assert abs(correct - ref_correct) <= near


def test_evaluate_errors(torch):
    import paper_2207_01053_b200 as pb
    from paper_2207_01053_b200.sim import Simulation
    sim = Simulation(precision=pb.PREC_FP32, arena_bytes=1 << 26)
    mid = sim.register_model(synth.MODEL_CNN, 4, 10, 32, 32, 3)
    rid = sim.register_model(synth.MODEL_RESNET8, 4, 10, 32, 32, 3)
    x, y = _val_split(synth.MODEL_CNN, 8, 1)
    w = synth.init_weights(synth.MODEL_CNN, 4, 10).astype(np.float32)
    with pytest.raises(pb.ProteaError) as e:
        sim.evaluate(mid, w, x[:0], y[:0])
    assert e.value.name == "INVALID"
    bad = y.copy()
    bad[3] = 10
    with pytest.raises(pb.ProteaError) as e:
        sim.evaluate(mid, w, x, bad)
    assert e.value.name == "INVALID" and "sample 3" in str(e.value)
    wr = synth.init_weights(synth.MODEL_RESNET8, 4, 10).astype(np.float32)
    with pytest.raises(pb.ProteaError) as e:
        sim.evaluate(rid, wr, x, y)
    assert e.value.name == "INVALID"
    sim.close()
