import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch, synth
import paper_2207_01053_b200 as pb
from paper_2207_01053_b200.sim import Simulation, concat_globals
for cfg, kw, prec in ((5, dict(n_clients=50, k=3, samples=20), 1), (1, dict(n_clients=3, samples=23), 1),
                      (2, dict(n_clients=4, samples=30, epochs=1), 1), (4, dict(k=6, samples=20, epochs=1), 1)):
    wl = synth.build_workload(cfg, **kw)
    H, W, C = (28, 28, 1) if wl.model == synth.MODEL_MLP else (32, 32, 3)
    widths = sorted({c.width_q for c in wl.clients})
    sim = Simulation(precision=prec, arena_bytes=512 << 20)
    mids = {w: sim.register_model(wl.model, w, 10, H, W, C) for w in widths}
    sim.register_shards([(c.id, *wl.shards[c.id]) for c in wl.clients])
    cl = sim.clients([(c.id, mids[c.width_q], c.batch, c.epochs) for c in wl.clients])
    plan, _ = sim.plan(sim.profile(cl))
    g = torch.tensor(concat_globals([synth.init_weights(wl.model, w, 10, seed=0) for w in widths]), device="cuda")
    out, st = sim.run_round(cl, plan, g, lr=0.05, seed=1)
    torch.cuda.synchronize()
    print("config", cfg, "ok", float(out.abs().sum()))
    sim.close()
sim = Simulation(arena_bytes=1 << 20)
from oracle import sgd
gf = torch.randn(sgd.n_params(sgd.CNN, 4), device="cuda")
subs = [pb.protea_heterofl_extract(sim.ctx, gf, q) for q in (1, 2, 4)]
o = pb.protea_heterofl_aggregate(sim.ctx, gf, subs, [1, 2, 4], [3, 4, 5])
torch.cuda.synchronize(); print("heterofl ok", float((o - gf).abs().max()))
sim.close()
