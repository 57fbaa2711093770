"""One federated round (oracle; test infrastructure only).

PAPER.md §3.3: configure_fit selects the clients (the sampled id list
is an input here) and aggregate_fit "aggregates them to generate a new global
model".  Each sampled client runs its local SGD (oracle/sgd.py) starting from
the global weights of its shape group; FedAvg (oracle/fedavg.py) then runs
independently per shape group (BASELINE.json configs[3] "FedAvg over
shared-shape subsets", reading R12).  A group with no sampled client
keeps its weights.
"""
from __future__ import annotations

from concurrent.futures import ProcessPoolExecutor

import numpy as np

from .fedavg import fedavg
from .sgd import local_sgd


def _client_job(args):
    (w0, model, width_q, classes, x, y, batch, epochs, lr, seed, rnd, cid, shuffle, max_steps, emul) = args
    w, losses = local_sgd(w0, model, width_q, classes, x, y, batch, epochs, lr, seed, rnd, cid,
                          shuffle=shuffle, max_steps=max_steps, emulate_bf16=emul)
    return w, losses


def run_round(clients, shards, global_w, lr, seed, rnd, shuffle=True, workers=0, return_clients=False,
              emulate_bf16=False):
    """clients: objects with id, n, batch, epochs, model, width_q, classes.
    global_w: dict width_q -> float array.  Returns dict width_q -> float64 array."""
    jobs = []
    for c in clients:
        x, y = shards[c.id]
        jobs.append((global_w[c.width_q], c.model, c.width_q, c.classes, x, y, c.batch, c.epochs,
                     lr, seed, rnd, c.id, shuffle, None, emulate_bf16))
    if workers and workers > 1:
        with ProcessPoolExecutor(max_workers=workers) as ex:
            results = list(ex.map(_client_job, jobs))
    else:
        results = [_client_job(j) for j in jobs]
    new = {}
    for wq, w in global_w.items():
        members = [(r[0], c.n) for c, r in zip(clients, results) if c.width_q == wq]
        if members:
            new[wq] = fedavg([m[0] for m in members], [m[1] for m in members])
        else:
            new[wq] = np.asarray(w, dtype=np.float64).copy()
    if return_clients:
        return new, {c.id: r for c, r in zip(clients, results)}
    return new
