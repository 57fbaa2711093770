"""Discrete decisions of the CNN step (ReLU masks, 2x2 max-pool argmax) along the float64 oracle's
trajectory of one client: the smallest margins (|z| / scale of the layer, top-1 minus top-2 of a pool
window / scale).  Margins near fp32 rounding (~1e-7) mean an fp32 (or bf16) path can take a different
decision than float64 at that step, after which the trajectories separate (full-size parity)."""
import dataclasses
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402
from oracle import sgd  # noqa: E402
from oracle.splitmix import epoch_perm  # noqa: E402


def margins(p, xb):
    z1, _ = sgd.conv_fwd(xb, p["conv1.W"], p["conv1.b"], 1, 2)
    a1, _ = sgd.pool2_fwd(sgd.relu(z1))
    z2, _ = sgd.conv_fwd(a1, p["conv2.W"], p["conv2.b"], 1, 2)
    out = []
    for z in (z1, z2):
        s = np.abs(z).max()
        r = np.maximum(z, 0)
        nb, H, W, C = r.shape
        w = r.reshape(nb, H // 2, 2, W // 2, 2, C).transpose(0, 1, 3, 5, 2, 4).reshape(-1, 4)
        w = np.sort(w, axis=1)
        pos = w[:, 3] > 0
        gap = (w[pos, 3] - w[pos, 2]).min() / s if pos.any() else np.inf
        out.append((np.abs(z[z != 0]).min() / s, gap))
    return out


def main():
    wl = synth.build_workload(2)
    c = dataclasses.replace(wl.clients[3], n=64, batch=8, epochs=1)
    tmpl = synth.class_templates(wl.shape, wl.classes, wl.seed)
    x, y = synth.make_shard(tmpl, c.n, c.id, wl.seed)
    xf = x.reshape(c.n, 32, 32, 3).astype(np.float64) / 255.0
    w = synth.init_weights(wl.model).astype(np.float64)
    perm = epoch_perm(c.n, wl.seed, 0, c.id, 0)
    for j in range(math.ceil(c.n / c.batch)):
        idx = perm[j * c.batch:(j + 1) * c.batch]
        p = sgd.unpack(w, sgd.CNN, 4, 10)
        (m1, g1), (m2, g2) = margins(p, xf[idx])
        print(f"step {j}: conv1 min|z|/max {m1:.1e} pool gap {g1:.1e} | conv2 min|z|/max {m2:.1e} pool gap {g2:.1e}")
        _, gflat = sgd.flat_loss_and_grad(w, sgd.CNN, 4, 10, xf[idx], y[idx])
        w = w - wl.lr * gflat


if __name__ == "__main__":
    main()
