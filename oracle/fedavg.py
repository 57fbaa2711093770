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
