"""Small rounds of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck):
bf16 rounds of configs 1, 2 (incl. a batch > 64 split into micro-clients), 4 and 5, an fp32 round of
config 2, an evaluate round, and the HeteroFL kernels.  Usage (GPU box):
  compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2207_01053_b200 as pb  # noqa: E402
import synth  # noqa: E402
from paper_2207_01053_b200.sim import Simulation, concat_globals  # noqa: E402

for cfg, kw, prec in ((5, dict(n_clients=50, k=3, samples=20), 1), (1, dict(n_clients=3, samples=23), 1),
                      (2, dict(n_clients=4, samples=30, epochs=1), 1), (2, dict(n_clients=3, samples=90, epochs=1), 0),
                      (2, dict(n_clients=3, samples=90, epochs=1), 1), (4, dict(k=6, samples=20, epochs=1), 1)):
    wl = synth.build_workload(cfg, **kw)
    if cfg == 2 and kw["samples"] == 90:  # one client with a batch of 80 rows: two micro-clients
        wl.clients[0] = dataclasses.replace(wl.clients[0], batch=80)
    H, W, C = (28, 28, 1) if wl.model == synth.MODEL_MLP else (32, 32, 3)
    widths = sorted({c.width_q for c in wl.clients})
    sim = Simulation(precision=prec, arena_bytes=512 << 20)
    mids = {w: sim.register_model(wl.model, w, 10, H, W, C) for w in widths}
    sim.register_shards([(c.id, *wl.shards[c.id]) for c in wl.clients])
    cl = sim.clients([(c.id, mids[c.width_q], c.batch, c.epochs) for c in wl.clients])
    plan, _ = sim.plan(sim.profile(cl))
    g = torch.tensor(concat_globals([synth.init_weights(wl.model, w, 10, seed=0) for w in widths]), device="cuda")
    out, st = sim.run_round(cl, plan, g, lr=0.05, seed=1, observe_hwm=True)
    tmpl = synth.class_templates(wl.shape, wl.classes, wl.seed)
    sim.register_val_shards([(c.id, *synth.make_val_shard(tmpl, c.n, c.id, wl.seed)) for c in wl.clients])
    per, tot = sim.evaluate_round(cl, out)
    torch.cuda.synchronize()
    print("config", cfg, "prec", prec, "ok", float(out.abs().sum()), tot, flush=True)
    sim.close()
sim = Simulation(arena_bytes=1 << 20)
gf = torch.randn(2156490, device="cuda")  # CNN-1x parameters
subs = [pb.protea_heterofl_extract(sim.ctx, gf, q) for q in (1, 2, 4)]
o = pb.protea_heterofl_aggregate(sim.ctx, gf, subs, [1, 2, 4], [3, 4, 5])
torch.cuda.synchronize()
print("heterofl ok", float((o - gf).abs().max()))
sim.close()
