"""Per-op device time of one round of config 3 or 4 (1 GPU, bf16): python tools/config_probe.py 4"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2207_01053_b200 as pb  # noqa: E402
from paper_2207_01053_b200.sim import Simulation, concat_globals  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
wl = synth.build_workload(cfg)
widths = sorted({c.width_q for c in wl.clients})
sim = Simulation(precision=pb.PREC_BF16, arena_bytes=4 << 30)
mids = {w: sim.register_model(wl.model, w, 10, 32, 32, 3) for w in widths}
sim.register_shards([(c.id, *wl.shards[c.id]) for c in wl.clients])
cl = sim.clients([(c.id, mids[c.width_q], c.batch, c.epochs) for c in wl.clients])
plan, mk = sim.plan(sim.profile(cl))
g = torch.tensor(concat_globals([synth.init_weights(wl.model, w, 10, seed=0) for w in widths]), device="cuda")
o = torch.empty_like(g)
for r in range(2):
    sim.run_round(cl, plan, g, o, lr=wl.lr, seed=wl.seed, rnd=r)
_, st = sim.run_round(cl, plan, g, o, lr=wl.lr, seed=wl.seed, rnd=3, time_ops=0xFFFFFFFF, serialize=True)
_, st2 = sim.run_round(cl, plan, g, o, lr=wl.lr, seed=wl.seed, rnd=4)
print(json.dumps({"config": cfg, "round_ms": st2["round_ns"] / 1e6, "iterations": int(mk[0]),
                  "launches": st2["kernel_launches"], "widths": {w: sum(c.width_q == w for c in wl.clients) for w in widths},
                  "op_ms": {pb.OPC_NAMES[i]: round(st["op_ns"][i] / 1e6, 2) for i in range(pb.N_OPC) if st["op_ns"][i]}}))
sim.close()
