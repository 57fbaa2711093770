import json, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch, synth
import paper_2207_01053_b200 as pb
from paper_2207_01053_b200.sim import Simulation
for prec in (pb.PREC_BF16, pb.PREC_FP32):
    wl = synth.build_workload(1)
    sim = Simulation(precision=prec, arena_bytes=256 << 20)
    mid = sim.register_model(wl.model, 4, 10, 28, 28, 1)
    sim.register_shards([(c.id, *wl.shards[c.id]) for c in wl.clients])
    cl = sim.clients([(c.id, mid, c.batch, c.epochs) for c in wl.clients])
    plan, mk = sim.plan(sim.profile(cl))
    g = torch.tensor(synth.init_weights(wl.model), device="cuda"); o = torch.empty_like(g)
    for r in range(3): sim.run_round(cl, plan, g, o, lr=0.05, seed=1, rnd=r)
    _, st = sim.run_round(cl, plan, g, o, lr=0.05, seed=1, rnd=5, time_ops=0xFFFFFFFF, serialize=True)
    _, st2 = sim.run_round(cl, plan, g, o, lr=0.05, seed=1, rnd=6)
    print(json.dumps({"prec": prec, "round_ms": st2["round_ns"]/1e6, "launches": st2["kernel_launches"],
        "op_us": {pb.OPC_NAMES[i]: round(st["op_ns"][i]/1e3, 1) for i in range(pb.N_OPC) if st["op_ns"][i]}}))
    sim.close()
