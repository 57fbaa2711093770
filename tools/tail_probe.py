"""Per-iteration op cost in the lock-step tail vs the full cohort (config 2, bf16).

Runs three rounds and prints per-op device time per lock-step iteration:
  full   — all 100 clients (the bench round),
  tail   — only the 25 B=8 clients (126 iterations of 200 rows: the tail's shape),
  heavy  — 100 clients, E=1, n = 7 B each: 7 iterations of all 3000 rows.
"""
import dataclasses
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2207_01053_b200 as pb  # noqa: E402
from paper_2207_01053_b200.sim import Simulation  # noqa: E402


def run(wl, ids, label):
    sim = Simulation(precision=pb.PREC_BF16, arena_bytes=4 << 30)
    mid = sim.register_model(pb.MODEL_CNN, 4, 10, 32, 32, 3)
    cl = [c for c in wl.clients if c.id in ids]
    sim.register_shards([(c.id, *wl.shards[c.id]) for c in cl])
    clients = sim.clients([(c.id, mid, c.batch, c.epochs) for c in cl])
    foot = np.zeros(len(cl), dtype=pb.PROFILE_DT)
    for i, c in enumerate(cl):
        pk, st, fl = pb.protea_client_footprint(pb.MODEL_CNN, 4, 10, 32, 32, 3, c.n, c.batch, c.epochs, pb.PREC_BF16)
        foot[i] = (c.id, pk, st, fl, 0, 0, 0, 1, 0)
    plan, mk = pb.protea_plan(foot, [4 << 30])
    g = torch.tensor(synth.init_weights(wl.model), device=sim.device)
    out = torch.empty_like(g)
    sim.run_round(clients, plan, g, out, lr=wl.lr, seed=wl.seed, rnd=0)
    _, st = sim.run_round(clients, plan, out, g, lr=wl.lr, seed=wl.seed, rnd=1, time_ops=0xFFFFFFFF)
    _, st2 = sim.run_round(clients, plan, g, out, lr=wl.lr, seed=wl.seed, rnd=2)
    it = int(mk[0])
    ops = {pb.OPC_NAMES[i]: float(st["op_ns"][i]) / it / 1e3 for i in range(len(pb.OPC_NAMES)) if st["op_ns"][i] > 0}
    sim.close()
    return {"label": label, "clients": len(cl), "iterations": it, "round_ms": st2["round_ns"] / 1e6,
            "us_per_iter": st2["round_ns"] / 1e3 / it, "op_us_per_iter": {k: round(v, 1) for k, v in ops.items()}}


def main():
    wl = synth.build_workload(2)
    res = [run(wl, {c.id for c in wl.clients}, "full"),
           run(wl, {c.id for c in wl.clients if c.batch == 8}, "tail (B=8 only)")]
    # heavy: every client does 7 full batches (E=1, n = 7 B): 7 iterations of all 3000 rows
    hv = synth.build_workload(2)
    hv.clients = [dataclasses.replace(c, n=7 * c.batch, epochs=1) for c in hv.clients]
    hv.shards = {c.id: (hv.shards[c.id][0][:c.n], hv.shards[c.id][1][:c.n]) for c in hv.clients}
    res.append(run(hv, {c.id for c in hv.clients}, "heavy (100 clients x 7 full batches)"))
    for r in res:
        print(json.dumps(r))


if __name__ == "__main__":
    main()
