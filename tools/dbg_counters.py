"""Read the PROTEA_DBG kernel cycle counters over one config-2 round (build with PROTEA_DBG=1)."""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2207_01053_b200 as pb  # noqa: E402
from paper_2207_01053_b200.sim import Simulation  # noqa: E402

lib = ctypes.CDLL(os.path.join(ROOT, "paper_2207_01053_b200", "libprotea.so"))
lib.protea_debug_counters.argtypes = [ctypes.POINTER(ctypes.c_uint64), ctypes.c_int]
wl = synth.build_workload(2)
if "heavy" in sys.argv:  # every client 7 full batches, E=1: 7 iterations of all 3000 rows
    import dataclasses
    wl.clients = [dataclasses.replace(c, n=7 * c.batch, epochs=1) for c in wl.clients]
    wl.shards = {c.id: (wl.shards[c.id][0][:c.n], wl.shards[c.id][1][:c.n]) for c in wl.clients}
sim = Simulation(precision=pb.PREC_BF16, arena_bytes=4 << 30)
mid = sim.register_model(pb.MODEL_CNN, 4, 10, 32, 32, 3)
sim.register_shards([(c.id, *wl.shards[c.id]) for c in wl.clients])
clients = sim.clients([(c.id, mid, c.batch, c.epochs) for c in wl.clients])
foot = np.zeros(len(wl.clients), dtype=pb.PROFILE_DT)
for i, c in enumerate(wl.clients):
    pk, st, fl = pb.protea_client_footprint(pb.MODEL_CNN, 4, 10, 32, 32, 3, c.n, c.batch, c.epochs, pb.PREC_BF16)
    foot[i] = (c.id, pk, st, fl, 0, 0, 0, 1, 0)
plan, _ = pb.protea_plan(foot, [4 << 30])
g = torch.tensor(synth.init_weights(wl.model), device=sim.device)
out = torch.empty_like(g)
buf = (ctypes.c_uint64 * 64)()
sim.run_round(clients, plan, g, out, lr=wl.lr, seed=wl.seed, rnd=0)
torch.cuda.synchronize()
lib.protea_debug_counters(buf, 1)
sim.run_round(clients, plan, out, g, lr=wl.lr, seed=wl.seed, rnd=1)
torch.cuda.synchronize()
lib.protea_debug_counters(buf, 0)
names = ["prod_wait_empty", "prod_issue", "mma_wait_acc_empty", "mma_wait_full", "mma_issue", "epi_wait_acc_full",
         "epi_drain", "epi_finish", "cta_ns_total", "split_reduce(c2w)"]
for base, label in ((0, "conv2 wgrad halo"), (16, "conv2 fwd halo"), (32, "conv2 dgrad halo"), (48, "conv1 fwd quad")):
    print("==", label)
    for i, n in enumerate(names):
        nm = n if not (base and i == 5) else "epi_total(wait+work)"
        if base and i == 6:
            nm = "mma_wait_weights"
        if base and i == 7:
            nm = "first_tile_done_ns"
        v = buf[base + i] / 148 / 1e6
        print(f"  {nm:22s} {v:10.3f} " + ("Mcyc per CTA" if (i < 8 and not (base and i == 7)) else "ms per CTA"))
