"""Host-side cost of one bench round (config 5 or 2): protea_plan wall time, run_round wall time, and
the library's device round time (round_ns, CUDA events from the start of run_round)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2207_01053_b200 as pb  # noqa: E402
import synth  # noqa: E402
from paper_2207_01053_b200.sim import Simulation  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
wl = bench.workload(1, cfg, "strong" if cfg != 2 else "weak")
foot = np.zeros(len(wl.clients), dtype=pb.PROFILE_DT)
for i, c in enumerate(wl.clients):
    pk, st, fl = pb.protea_client_footprint(wl.model, 4, 10, 32, 32, 3, c.n, c.batch, c.epochs, pb.PREC_BF16)
    foot[i] = (c.id, pk, st, fl, 0, 0, 0, 1, 0)
caps = [int(sum(int(f["peak_bytes"]) for f in foot) * 1.25) + (256 << 20)]
sim = Simulation(precision=pb.PREC_BF16, arena_bytes=caps[0])
mid = sim.register_model(wl.model, 4, 10, 32, 32, 3)
tmpl = synth.class_templates(wl.shape, wl.classes, wl.seed)
sim.register_shards([(c.id, *synth.make_shard(tmpl, c.n, c.id, wl.seed)) for c in wl.clients])
cl = sim.clients([(c.id, mid, c.batch, c.epochs) for c in wl.clients])
g = torch.tensor(synth.init_weights(wl.model), device=sim.device)
g2 = torch.empty_like(g)
for k in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan, _ = pb.protea_plan(foot, caps)
    t1 = time.perf_counter()
    _, (st, meas) = sim.run_round(cl, plan, g, g2, lr=wl.lr, seed=wl.seed, rnd=k, measured=True)
    t2 = time.perf_counter()
    g, g2 = g2, g
    print(f"config{cfg} round {k}: plan {1e3 * (t1 - t0):.2f} ms, run_round wall {1e3 * (t2 - t1):.2f} ms, "
          f"round_ns {st['round_ns'] / 1e6:.2f} ms, launches {st['kernel_launches']}")
