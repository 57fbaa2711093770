"""Round time and client-steps/s of every BASELINE.json config on B200, at the
per-GPU share of a G-GPU plan for G = 1, 2, 4, 8.

Only one GPU is available here, so a G-GPU round is measured rank by rank:
rank r's clients of the G-GPU plan (protea_plan, LPT by FLOPs + FIFO
first-fit) run as a `partial_only` round in a rank-r context on the one GPU,
and the G-GPU round time is the max over ranks of those device times (CUDA
events inside protea_run_round).  The one thing not measured is the NCCL fp64
sum of the FedAvg partials (P doubles: 17 MB for CNN-1x, ~20 us over NVLink).

Precision: bf16 (tensor-core CNN path; MLP and ResNet-8 run their SIMT kernels
on bf16 storage).  Output: one JSON line per (config, G) on stdout.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2207_01053_b200 as pb  # noqa: E402
from paper_2207_01053_b200.sim import Simulation, concat_globals  # noqa: E402

CASES = [  # (label, config, kwargs for synth.build_workload)
    ("config1 MLP 10 clients", 1, {}),
    ("config2 CNN-1x 100 clients", 2, {}),
    ("config3 Dirichlet K=10", 3, {"k": 10}),
    ("config3 Dirichlet K=100", 3, {"k": 100}),
    ("config4 widths 1/4,1/2,1 K=100", 4, {}),
    ("config5 ResNet-8 K=500", 5, {}),
]


def shape_of(model):
    return (28, 28, 1) if model == synth.MODEL_MLP else (32, 32, 3)


def run_case(label, cfg, kw, gpus, prec, reps):
    wl = synth.build_workload(cfg, **kw)
    H, W, C = shape_of(wl.model)
    widths = sorted({c.width_q for c in wl.clients})
    foot = np.zeros(len(wl.clients), dtype=pb.PROFILE_DT)
    for i, c in enumerate(wl.clients):
        pk, st, fl = pb.protea_client_footprint(wl.model, c.width_q, wl.classes, H, W, C, c.n, c.batch, c.epochs, prec)
        foot[i] = (c.id, pk, st, fl, 0, 0, 0, 1, 0)
    steps = int(foot["steps"].sum())
    flops = int(foot["flops"].sum())
    g0 = {w: synth.init_weights(wl.model, w, wl.classes, seed=0) for w in widths}
    out = []
    for G in gpus:
        cap = int(foot["peak_bytes"].sum() * 1.25) + (64 << 20)
        plan, mk = pb.protea_plan(foot, [cap] * G)
        per_rank = []
        for r in range(G):
            mine = [c for c, a in zip(wl.clients, plan) if int(a["gpu"]) == r]
            if not mine:
                per_rank.append(0.0)
                continue
            sim = Simulation(precision=prec, arena_bytes=cap, rank=r, world=G)
            mids = {w: sim.register_model(wl.model, w, wl.classes, H, W, C) for w in widths}
            sim.register_shards([(c.id, *wl.shards[c.id]) for c in wl.clients])  # n_k of every client (FedAvg N)
            clients = sim.clients([(c.id, mids[c.width_q], c.batch, c.epochs) for c in wl.clients])
            g = torch.tensor(concat_globals([g0[w] for w in widths]), device=sim.device)
            o = torch.empty_like(g)
            best = None
            for k in range(reps + 1):  # round 0 warms up (tensor maps, attributes)
                _, st = sim.run_round(clients, plan, g, o, lr=wl.lr, seed=wl.seed, rnd=k, partial_only=(G > 1))
                if k and (best is None or st["round_ns"] < best):
                    best = st["round_ns"]
            per_rank.append(best / 1e6)
            sim.close()
            torch.cuda.empty_cache()
        ms = max(per_rank)
        rec = {"case": label, "config": cfg, "gpus": G, "clients": len(wl.clients), "client_steps": steps,
               "max_local_steps": int(foot["steps"].max()), "round_ms": ms, "rank_ms": per_rank,
               "client_steps_per_s": steps / (ms / 1e3), "tflops": flops / (ms / 1e3) / 1e12,
               "plan_makespan_steps": [int(x) for x in mk], "precision": "bf16" if prec == pb.PREC_BF16 else "fp32"}
        print(json.dumps(rec), flush=True)
        out.append(rec)
    return out


def main():
    prec = pb.PREC_FP32 if "fp32" in sys.argv else pb.PREC_BF16
    only = [a for a in sys.argv[1:] if a.isdigit()]
    gpus = (1, 2, 4, 8)
    t0 = time.time()
    for label, cfg, kw in CASES:
        if only and str(cfg) not in only:
            continue
        run_case(label, cfg, kw, gpus, prec, reps=2)
    print(json.dumps({"wall_s": time.time() - t0}), file=sys.stderr)


if __name__ == "__main__":
    main()
