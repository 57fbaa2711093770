"""Client evaluation (forward only), float64 — oracle, test infrastructure only.

SURVEY §8(f).3: each client evaluates the global model on its held-out
validation split (§4.1: the clients' data is split into training
and validation sets; the evaluate round follows aggregation, §3.3).
For a model w and samples (x, y):

    loss_sum = sum_i [ logsumexp(z_i) - z_i[y_i] ]      (z_i = the model's logits)
    correct  = #{ i : argmax_c z_i[c] == y_i }           (first maximum on ties)

The forward pass is the one of oracle/sgd.py (readings R10/R11); evaluate_round applies it
per client to its validation split (the aggregate is the sum over clients: the example-weighted mean
loss and the accuracy follow by dividing by the total n).
"""
import numpy as np

from . import sgd


def logits(w, model, width_q, classes, x_u8):
    """x_u8 [n, H, W, C] u8 -> logits [n, classes] (float64)."""
    p = sgd.unpack(np.asarray(w, dtype=np.float64), model, width_q, classes)
    xb = np.asarray(x_u8, dtype=np.float64) / 255.0
    nb = xb.shape[0]
    if model == sgd.MLP:
        h1 = sgd.relu(xb.reshape(nb, -1) @ p["fc1.W"].T + p["fc1.b"])
        return h1 @ p["fc2.W"].T + p["fc2.b"]
    if model in (sgd.CNN, sgd.CNN28):
        z1, _ = sgd.conv_fwd(xb, p["conv1.W"], p["conv1.b"], 1, 2)
        a1, _ = sgd.pool2_fwd(sgd.relu(z1))
        z2, _ = sgd.conv_fwd(a1, p["conv2.W"], p["conv2.b"], 1, 2)
        a2, _ = sgd.pool2_fwd(sgd.relu(z2))
        h = sgd.relu(a2.reshape(nb, -1) @ p["fc1.W"].T + p["fc1.b"])
        return h @ p["fc2.W"].T + p["fc2.b"]
    if model == sgd.RESNET18:  # R26: conv (bias) -> GroupNorm -> ReLU, 8 basic blocks, GAP, fc
        a = sgd.relu(sgd.gn_fwd(sgd.conv_fwd(xb, p["conv0.W"], p["conv0.b"], 1, 1)[0], p["gn0.W"], p["gn0.b"])[0])
        for name, cin, cout, stride in sgd.resnet18_blocks():
            za, _ = sgd.conv_fwd(a, p[name + "a.W"], p[name + "a.b"], stride, 1)
            ra = sgd.relu(sgd.gn_fwd(za, p[name + "ga.W"], p[name + "ga.b"])[0])
            zb, _ = sgd.conv_fwd(ra, p[name + "b.W"], p[name + "b.b"], 1, 1)
            sc = a if (stride == 1 and cin == cout) else sgd.option_a(a, cout)
            a = sgd.relu(sgd.gn_fwd(zb, p[name + "gb.W"], p[name + "gb.b"])[0] + sc)
        return a.mean(axis=(1, 2)) @ p["fc.W"].T + p["fc.b"]
    if model == sgd.RESNET8:  # conv0, three basic blocks (option-A shortcut), global average pool, fc
        z0, _ = sgd.conv_fwd(xb, p["conv0.W"], p["conv0.b"], 1, 1)
        a = sgd.relu(z0)
        for blk, stride in (("b1", 1), ("b2", 2), ("b3", 2)):
            za, _ = sgd.conv_fwd(a, p[blk + "a.W"], p[blk + "a.b"], stride, 1)
            zb, _ = sgd.conv_fwd(sgd.relu(za), p[blk + "b.W"], p[blk + "b.b"], 1, 1)
            if stride == 1:
                sc = a
            else:
                sub = a[:, ::2, ::2, :]
                sc = np.zeros(sub.shape[:3] + (zb.shape[3],))
                sc[..., :sub.shape[3]] = sub
            a = sgd.relu(zb + sc)
        return a.mean(axis=(1, 2)) @ p["fc.W"].T + p["fc.b"]
    raise ValueError(model)


def evaluate(w, model, width_q, classes, x_u8, y):
    """-> (loss_sum, correct, n) of the model w on (x, y)."""
    z = logits(w, model, width_q, classes, x_u8)
    y = np.asarray(y, dtype=np.int64)
    m = z.max(axis=1)
    lse = np.log(np.exp(z - m[:, None]).sum(axis=1)) + m
    loss_sum = float(np.sum(lse - z[np.arange(len(y)), y]))
    correct = int(np.sum(np.argmax(z, axis=1) == y))  # numpy argmax = first maximum
    return loss_sum, correct, len(y)


def evaluate_round(clients, val_shards, global_w):
    """PAPER.md P:238 (configure_evaluate / aggregate_evaluate) with P:302's validation split: every client
    evaluates its shape group's global weights on its own validation data.  clients: objects with id,
    model, width_q, classes; val_shards: id -> (x u8 [n, D], y); global_w: width_q -> weights.
    Returns ({id: (loss_sum, correct, n)}, (sum loss_sum, sum correct, sum n))."""
    per = {}
    for c in clients:
        x, y = val_shards[c.id]
        H, W, C = sgd.input_shape(c.model)
        per[c.id] = evaluate(global_w[c.width_q], c.model, c.width_q, c.classes, x.reshape(-1, H, W, C), y)
    tot = (sum(v[0] for v in per.values()), sum(v[1] for v in per.values()), sum(v[2] for v in per.values()))
    return per, tot
