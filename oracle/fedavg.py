"""Vanilla FedAvg (oracle; test infrastructure only).

PAPER.md P:234 (§3.3): ResourceAwareFedAvg "enhances the vanilla Federated
Averaging (FedAvg) [McMahan et al., P:83] strategy"; aggregate_fit
"aggregates them to generate a new global model".  McMahan's FedAvg weights
client k by n_k, its number of training examples (reading R1).

    w' = sum_k n_k w_k / sum_k n_k          (exact definition, float64)

Errors mirror SPEC.md [strategy] fedavg_aggregate: empty -> EMPTY, any n_k <= 0
-> INVALID, sum n = 0 -> ZERO_WEIGHT, dimension mismatch -> DIM.
"""
from __future__ import annotations

import numpy as np


class FedAvgError(ValueError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def fedavg(params, num_examples):
    if len(params) == 0:
        raise FedAvgError("EMPTY", "no results to aggregate")
    if len(params) != len(num_examples):
        raise FedAvgError("INVALID", "params / num_examples length mismatch")
    dim = np.asarray(params[0]).size
    for k, (w, n) in enumerate(zip(params, num_examples)):
        if np.asarray(w).size != dim:
            raise FedAvgError("DIM", f"client {k}: dimension {np.asarray(w).size} != {dim}")
        if int(n) <= 0:
            raise FedAvgError("INVALID", f"client {k}: num_examples {n} <= 0")
    total = sum(int(n) for n in num_examples)
    if total == 0:
        raise FedAvgError("ZERO_WEIGHT", "zero total weight")
    acc = np.zeros(dim, dtype=np.float64)
    for w, n in zip(params, num_examples):
        acc += float(n) * np.asarray(w, dtype=np.float64).ravel()
    return acc / float(total)


# ---------------------------------------------------------------------------
# HeteroFL-style overlapping-width aggregation (reading R23).
# The global model is the full-width CNN (width_q = 4).  A width-q client trains the sub-model made
# of the FIRST channels of every hidden dimension: conv1 out [:C1(q)]; conv2 out [:C2(q)], in
# [:C1(q)]; fc1 out [:F(q)], in = for each of the 8x8 pooled positions the first C2(q) channels (NHWC
# flattening p * C2 + c); fc2 in [:F(q)] (all classes); biases of the kept outputs.  Aggregation:
# every global element becomes the n_k-weighted mean over the clients whose sub-model holds it
# (reading R1 weights), elements no client holds keep the global value.
# ---------------------------------------------------------------------------
def heterofl_index_map(width_q, classes=10):
    """Global flat index of every element of the width-q CNN sub-model, in the sub-model's flat order."""
    from .sgd import CNN, cnn_channels, layer_shapes
    c1, c2, f = cnn_channels(width_q)
    c2_full = cnn_channels(4)[1]
    base, off = {}, 0
    for name, ws, bs in layer_shapes(CNN, 4, classes):
        nw, nb = int(np.prod(ws)), int(np.prod(bs))
        base[name] = (np.arange(nw).reshape(ws) + off, np.arange(nb) + off + nw)
        off += nw + nb
    keep_out = {"conv1": c1, "conv2": c2, "fc1": f, "fc2": classes}
    idx = []
    for name, ws, bs in layer_shapes(CNN, width_q, classes):
        W, b = base[name]
        if name == "conv1":
            Ws = W[:c1]
        elif name == "conv2":
            Ws = W[:c2, :, :, :c1]
        elif name == "fc1":
            Ws = W.reshape(W.shape[0], 64, c2_full)[:f, :, :c2].reshape(f, 64 * c2)
        else:
            Ws = W[:, :f]
        idx.append(Ws.ravel())
        idx.append(b[:keep_out[name]])
    return np.concatenate(idx)


def heterofl_extract(global_full, width_q, classes=10):
    """The width-q sub-model of the full-width global weights (what a width-q client starts from)."""
    return np.asarray(global_full)[heterofl_index_map(width_q, classes)]


def heterofl_aggregate(global_full, params, width_q, num_examples, classes=10):
    """n_k-weighted mean per global element over the clients holding it (float64)."""
    from .sgd import CNN, n_params
    if len(params) == 0:
        raise FedAvgError("EMPTY", "no results to aggregate")
    g = np.asarray(global_full, dtype=np.float64).ravel()
    if g.size != n_params(CNN, 4, classes):
        raise FedAvgError("DIM", "global model is not the full-width CNN")
    num = np.zeros_like(g)
    den = np.zeros_like(g)
    for k, (w, q, n) in enumerate(zip(params, width_q, num_examples)):
        if q not in (1, 2, 4):
            raise FedAvgError("INVALID", f"client {k}: width_q {q} not in (1, 2, 4)")
        if int(n) <= 0:
            raise FedAvgError("INVALID", f"client {k}: num_examples {n} <= 0")
        w = np.asarray(w, dtype=np.float64).ravel()
        if w.size != n_params(CNN, q, classes):
            raise FedAvgError("DIM", f"client {k}: dimension {w.size} != {n_params(CNN, q, classes)}")
        m = heterofl_index_map(q, classes)
        num[m] += float(n) * w
        den[m] += float(n)
    out = g.copy()
    held = den > 0
    out[held] = num[held] / den[held]
    return out
