"""Pins for oracle/sgd.py and oracle/round.py.

- torch CPU float64 autograd of the same models (a library reference, not the
  oracle retyped): gradients <= 1e-12 relative; a torch.optim.SGD loop over
  the same batches reproduces local_sgd;
- central finite differences of the loss: <= 1e-6 relative;
- closed forms: zero logits -> loss ln C, dz rows sum to 0; lr = 0 -> identity;
- FedSGD identity (E=1, B_k=n_k, all clients sampled): the FedAvg round equals
  one full-batch GD step on the pooled data (pins the n_k weighting and the
  mean-over-batch loss convention, SURVEY §8(c).2 pin iv);
- K = 1: the round equals that client's local SGD.
"""
import math

import numpy as np
import pytest

import synth
from oracle import round as orr
from oracle import sgd
from oracle.splitmix import epoch_perm

torch = pytest.importorskip("torch")
F = torch.nn.functional


def torch_forward(model, wq, classes, w, xb):
    """Independent torch float64 model of the same architectures (NHWC in)."""
    p = {}
    off = 0
    for name, ws, bs in sgd.layer_shapes(model, wq, classes):
        nw, nb = int(np.prod(ws)), int(np.prod(bs))
        p[name + ".W"] = w[off:off + nw].view(ws)
        off += nw
        p[name + ".b"] = w[off:off + nb].view(bs)
        off += nb
    n = xb.shape[0]
    if model == sgd.MLP:
        h = F.relu(F.linear(xb.reshape(n, -1), p["fc1.W"], p["fc1.b"]))
        return F.linear(h, p["fc2.W"], p["fc2.b"])
    x = xb.permute(0, 3, 1, 2)

    def cw(name):
        return p[name + ".W"].permute(0, 3, 1, 2)

    if model in (sgd.CNN, sgd.CNN28):
        x = F.max_pool2d(F.relu(F.conv2d(x, cw("conv1"), p["conv1.b"], padding=2)), 2)
        x = F.max_pool2d(F.relu(F.conv2d(x, cw("conv2"), p["conv2.b"], padding=2)), 2)
        x = x.permute(0, 2, 3, 1).reshape(n, -1)
        x = F.relu(F.linear(x, p["fc1.W"], p["fc1.b"]))
        return F.linear(x, p["fc2.W"], p["fc2.b"])
    x = F.relu(F.conv2d(x, cw("conv0"), p["conv0.b"], padding=1))
    for blk, s in (("b1", 1), ("b2", 2), ("b3", 2)):
        o = F.relu(F.conv2d(x, cw(blk + "a"), p[blk + "a.b"], stride=s, padding=1))
        o = F.conv2d(o, cw(blk + "b"), p[blk + "b.b"], padding=1)
        if s == 1:
            sc = x
        else:
            sub = x[:, :, ::2, ::2]
            sc = F.pad(sub, (0, 0, 0, 0, 0, o.shape[1] - sub.shape[1]))
        x = F.relu(o + sc)
    x = x.mean(dim=(2, 3))
    return F.linear(x, p["fc.W"], p["fc.b"])


def torch_grad(model, wq, classes, w, xb, yb):
    wt = torch.tensor(w, dtype=torch.float64, requires_grad=True)
    z = torch_forward(model, wq, classes, wt, torch.tensor(xb, dtype=torch.float64))
    loss = F.cross_entropy(z, torch.tensor(yb, dtype=torch.long))
    loss.backward()
    return float(loss.detach()), wt.grad.numpy()


CASES = [(sgd.MLP, 4, 5), (sgd.CNN, 1, 3), (sgd.CNN, 4, 2), (sgd.RESNET8, 4, 2), (sgd.CNN28, 2, 3)]


def _batch(model, nb, seed=0, classes=10):
    rng = np.random.default_rng(seed)
    H, W, C = sgd.input_shape(model)
    x = rng.integers(0, 256, size=(nb, H, W, C)).astype(np.float64) / 255.0
    y = rng.integers(0, classes, size=nb)
    return x, y


@pytest.mark.parametrize("model,wq,nb", CASES)
def test_grad_vs_torch_f64(model, wq, nb):
    w = synth.init_weights(model, wq, 10, seed=1).astype(np.float64)
    x, y = _batch(model, nb)
    loss, g = sgd.flat_loss_and_grad(w, model, wq, 10, x, y)
    tl, tg = torch_grad(model, wq, 10, w, x, y)
    assert abs(loss - tl) <= 1e-12 * abs(tl)
    assert np.linalg.norm(g - tg) <= 1e-12 * np.linalg.norm(tg)


@pytest.mark.parametrize("model,wq,nb", [(sgd.MLP, 4, 3), (sgd.CNN, 1, 2), (sgd.RESNET8, 4, 2), (sgd.CNN28, 1, 2)])
def test_grad_finite_differences(model, wq, nb):
    w = synth.init_weights(model, wq, 10, seed=2).astype(np.float64)
    x, y = _batch(model, nb, seed=3)
    _, g = sgd.flat_loss_and_grad(w, model, wq, 10, x, y)
    rng = np.random.default_rng(4)
    # coordinates with large gradients from every layer + random ones
    idx = list(rng.choice(w.size, 12, replace=False)) + list(np.argsort(-np.abs(g))[:12])
    h = 1e-6
    for i in idx:
        wp, wm = w.copy(), w.copy()
        wp[i] += h
        wm[i] -= h
        fd = (sgd.flat_loss_and_grad(wp, model, wq, 10, x, y)[0] - sgd.flat_loss_and_grad(wm, model, wq, 10, x, y)[0]) / (2 * h)
        assert abs(fd - g[i]) <= 1e-6 * max(1e-3, np.abs(g).max()), (i, fd, g[i])


def test_zero_logits_closed_form():
    for C in (2, 10, 62):
        loss, dz = sgd.softmax_ce(np.zeros((4, C)), np.array([0, 1, 1, C - 1]))
        assert abs(loss - math.log(C)) < 1e-15
        assert np.allclose(dz.sum(axis=1), 0.0, atol=1e-15)
        assert np.allclose(dz[0, 0], (1.0 / C - 1.0) / 4)


def test_pool_first_max_tiebreak():
    r = np.array([[[[1.0], [1.0]], [[1.0], [0.5]]]])  # one 2x2 window, ties at q=0,1,2
    p, a = sgd.pool2_fwd(r)
    assert p[0, 0, 0, 0] == 1.0 and a[0, 0, 0, 0] == 0
    r = np.array([[[[0.0], [2.0]], [[2.0], [0.5]]]])
    p, a = sgd.pool2_fwd(r)
    assert a[0, 0, 0, 0] == 1
    d = sgd.pool2_bwd(np.array([[[[3.0]]]]), a, r.shape)
    assert d[0, 0, 1, 0] == 3.0 and d.sum() == 3.0


def test_lr_zero_identity():
    wl = synth.build_workload(1, n_clients=2, samples=12)
    c = wl.clients[0]
    w0 = synth.init_weights(wl.model)
    x, y = wl.shards[c.id]
    w, _ = sgd.local_sgd(w0, c.model, 4, 10, x, y, 5, 2, 0.0, 0, 0, c.id)
    assert np.array_equal(w, w0.astype(np.float64))


@pytest.mark.parametrize("model,wq", [(sgd.MLP, 4), (sgd.CNN, 1)])
def test_local_sgd_vs_torch_optim_loop(model, wq):
    """A torch.optim.SGD loop over the same (pinned) permutation and batches,
    partial last batch kept, reproduces oracle local_sgd to 1e-11."""
    n, B, E, lr = 11, 4, 2, 0.05
    rng = np.random.default_rng(8)
    H, W, C = sgd.input_shape(model)
    x = rng.integers(0, 256, size=(n, H * W * C)).astype(np.uint8)
    y = rng.integers(0, 10, size=n).astype(np.int32)
    w0 = synth.init_weights(model, wq, 10, seed=5)
    w_or, _ = sgd.local_sgd(w0, model, wq, 10, x, y, B, E, lr, 9, 2, 31)
    wt = torch.tensor(w0.astype(np.float64), requires_grad=True)
    opt = torch.optim.SGD([wt], lr=lr)
    xf = torch.tensor(x.reshape(n, H, W, C).astype(np.float64) / 255.0)
    steps = 0
    for e in range(E):
        perm = epoch_perm(n, 9, 2, 31, e)
        for j in range(0, n, B):
            idx = perm[j:j + B]
            opt.zero_grad()
            z = torch_forward(model, wq, 10, wt, xf[idx])
            F.cross_entropy(z, torch.tensor(y[idx], dtype=torch.long)).backward()
            opt.step()
            steps += 1
    assert steps == E * math.ceil(n / B)
    wt = wt.detach().numpy()
    assert np.linalg.norm(w_or - wt) <= 1e-11 * np.linalg.norm(wt)


def test_fedsgd_identity():
    # E=1, B_k = n_k, every client: FedAvg round == w - lr * grad of mean loss on pooled data.
    wl = synth.build_workload(2, n_clients=3, samples=5, epochs=1)
    for c in wl.clients:
        c.batch = c.n
    w0 = synth.init_weights(wl.model, 4, 10, seed=2)
    lr = 0.1
    new = orr.run_round(wl.clients, wl.shards, {4: w0}, lr, 0, 0)[4]
    xs = np.concatenate([wl.shards[c.id][0] for c in wl.clients]).reshape(-1, 32, 32, 3) / 255.0
    ys = np.concatenate([wl.shards[c.id][1] for c in wl.clients])
    _, g = torch_grad(sgd.CNN, 4, 10, w0.astype(np.float64), xs, ys)
    ref = w0.astype(np.float64) - lr * g
    assert np.linalg.norm(new - ref) <= 1e-12 * np.linalg.norm(ref)


def test_round_k1_equals_client_sgd():
    wl = synth.build_workload(1, n_clients=1, samples=23)
    c = wl.clients[0]
    w0 = synth.init_weights(wl.model)
    new = orr.run_round(wl.clients, wl.shards, {4: w0}, 0.05, 4, 1)[4]
    w, _ = sgd.local_sgd(w0, c.model, 4, 10, *wl.shards[c.id], c.batch, c.epochs, 0.05, 4, 1, c.id)
    # n*w/n rounds at most once per element
    assert np.all(np.abs(new - w) <= 2.3e-16 * np.abs(w))


def test_round_groups_keep_unsampled():
    wl = synth.build_workload(4, k=2, samples=3, epochs=1)
    gw = {wq: synth.init_weights(sgd.CNN, wq, 10) for wq in (1, 2, 4)}
    new = orr.run_round(wl.clients, wl.shards, gw, 0.05, 0, 0)
    present = {c.width_q for c in wl.clients}
    for wq in (1, 2, 4):
        if wq not in present:
            assert np.array_equal(new[wq], gw[wq].astype(np.float64))
        else:
            assert not np.array_equal(new[wq], gw[wq].astype(np.float64))


def test_synth_shapes_and_param_segments():
    for model, wq in ((sgd.MLP, 4), (sgd.CNN, 1), (sgd.CNN, 2), (sgd.CNN, 4), (sgd.RESNET8, 4)):
        assert synth.init_weights(model, wq).size == sgd.n_params(model, wq)
    s = synth.dirichlet_sizes(1000, 50000, 0.5, seed=0)
    assert s.sum() == 50000 and s.min() >= 1


def torch_resnet18(w, xb, classes=10):
    """Independent torch float64 ResNet-18 with GroupNorm (R26): conv(bias) -> GN -> ReLU, basic blocks with
    identity / option-A shortcuts, GAP, FC."""
    p, off = {}, 0
    for name, ws, bs in sgd.layer_shapes(sgd.RESNET18, 4, classes):
        nw, nb = int(np.prod(ws)), int(np.prod(bs))
        p[name + ".W"] = w[off:off + nw].view(ws)
        off += nw
        p[name + ".b"] = w[off:off + nb].view(bs)
        off += nb
    x = xb.permute(0, 3, 1, 2)

    def conv(x, name, s):
        return F.conv2d(x, p[name + ".W"].permute(0, 3, 1, 2), p[name + ".b"], stride=s, padding=1)

    def gn(x, name):
        return F.group_norm(x, 2, p[name + ".W"], p[name + ".b"], eps=1e-5)

    x = F.relu(gn(conv(x, "conv0", 1), "gn0"))
    cin = 64
    for s, c in enumerate((64, 128, 256, 512)):
        for b in range(2):
            name, st = f"s{s + 1}b{b}", (2 if (s > 0 and b == 0) else 1)
            o = F.relu(gn(conv(x, name + "a", st), name + "ga"))
            o = gn(conv(o, name + "b", 1), name + "gb")
            if st == 1 and cin == c:
                sc = x
            else:
                sub = x[:, :, ::2, ::2]
                sc = F.pad(sub, (0, 0, 0, 0, 0, c - cin))
            x = F.relu(o + sc)
            cin = c
    return F.linear(x.mean(dim=(2, 3)), p["fc.W"], p["fc.b"])


def test_resnet18_gn_grad_vs_torch_f64():
    w = synth.init_weights(sgd.RESNET18, 4, 10, seed=2).astype(np.float64)
    x, y = _batch(sgd.RESNET18, 2)
    loss, g = sgd.flat_loss_and_grad(w, sgd.RESNET18, 4, 10, x, y)
    wt = torch.tensor(w, requires_grad=True)
    lt = F.cross_entropy(torch_resnet18(wt, torch.tensor(x)), torch.tensor(y))
    lt.backward()
    assert abs(loss - lt.item()) <= 1e-12 * abs(lt.item())
    assert np.linalg.norm(g - wt.grad.numpy()) <= 1e-10 * np.linalg.norm(wt.grad.numpy())


def test_gn_closed_forms():
    """GroupNorm: per (sample, group) zero mean / unit variance before the affine; gamma = 0 gives beta;
    its backward kills a constant shift of the input (the normalisation removes it)."""
    rng = np.random.default_rng(0)
    z = rng.normal(size=(3, 4, 4, 8)) * 3 + 1
    out, (xh, rstd, G) = sgd.gn_fwd(z, np.ones(8), np.zeros(8))
    xg = xh.reshape(3, 4, 4, 2, 4)
    assert np.allclose(xg.mean(axis=(1, 2, 4)), 0, atol=1e-12) and np.allclose(xg.var(axis=(1, 2, 4)), 1, atol=1e-4)
    out0, _ = sgd.gn_fwd(z, np.zeros(8), np.arange(8.0))
    assert np.allclose(out0, np.broadcast_to(np.arange(8.0), z.shape))
    dz, dgam, dbet = sgd.gn_bwd(np.ones_like(z), np.full(8, 1.7), sgd.gn_fwd(z, np.ones(8), np.zeros(8))[1])
    assert np.allclose(dz, 0, atol=1e-10) and np.allclose(dbet, 48) and np.allclose(dgam.reshape(2, 4).sum(1), 0, atol=1e-10)
