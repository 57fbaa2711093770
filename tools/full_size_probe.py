import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch, synth
import paper_2207_01053_b200 as pb
from paper_2207_01053_b200.sim import Simulation
from oracle import round as orr
from tests.gpu_helpers import rel_l2
wl = synth.build_workload(2)
w0 = synth.init_weights(wl.model)
for sample in ({0}, {3}, {0, 3}):
    ref = orr.run_round([c for c in wl.clients if c.id in sample], wl.shards, {4: w0}, wl.lr, wl.seed, 0, workers=2)[4]
    for prec in (0, 1):
        sim = Simulation(precision=prec, arena_bytes=4 << 30)
        mid = sim.register_model(wl.model, 4, 10, 32, 32, 3)
        cl = [c for c in wl.clients if c.id in sample]
        sim.register_shards([(c.id, *wl.shards[c.id]) for c in cl])
        clients = sim.clients([(c.id, mid, c.batch, c.epochs) for c in cl])
        plan, _ = sim.plan(sim.profile(clients))
        g, st = sim.run_round(clients, plan, torch.tensor(w0, device="cuda"), lr=wl.lr, seed=wl.seed)
        got = g.cpu().numpy().astype(np.float64)
        print(sorted(sample), "fp32" if prec == 0 else "bf16", "rel-L2 weights %.3e update %.3e" % (rel_l2(got, ref), rel_l2(got - w0, ref - w0)), flush=True)
        sim.close()
