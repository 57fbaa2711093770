"""One config-2 round (args: [fp32] [tail]) (bf16, 1 GPU) bracketed by cudaProfilerStart/Stop, for ncu
captures of steady-state (all-clients-active) launches:

  ncu --profile-from-start off -k regex:NAME --launch-skip S --launch-count C \
      python tools/prof_round.py

The warm-up round (outside the profiled range) pays one-time setup (tensor maps,
attributes); the probe of bench.py is not run.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2207_01053_b200 as pb  # noqa: E402
from paper_2207_01053_b200.sim import Simulation  # noqa: E402


def main():
    args = sys.argv[1:]
    prec = pb.PREC_FP32 if "fp32" in args else pb.PREC_BF16
    wl = synth.build_workload(2)
    if "tail" in args:  # only the B=8 clients: the shape of the lock-step tail
        wl.clients = [c for c in wl.clients if c.batch == 8]
    sim = Simulation(precision=prec, arena_bytes=4 << 30)
    mid = sim.register_model(pb.MODEL_CNN, 4, 10, 32, 32, 3)
    sim.register_shards([(c.id, *wl.shards[c.id]) for c in wl.clients])
    clients = sim.clients([(c.id, mid, c.batch, c.epochs) for c in wl.clients])
    foot = np.zeros(len(wl.clients), dtype=pb.PROFILE_DT)
    for i, c in enumerate(wl.clients):
        pk, st, fl = pb.protea_client_footprint(pb.MODEL_CNN, 4, 10, 32, 32, 3, c.n, c.batch, c.epochs, prec)
        foot[i] = (c.id, pk, st, fl, 0, 0, 0, 1, 0)
    plan, _ = pb.protea_plan(foot, [4 << 30])
    g = torch.tensor(synth.init_weights(wl.model), device=sim.device)
    out = torch.empty_like(g)
    sim.run_round(clients, plan, g, out, lr=wl.lr, seed=wl.seed, rnd=0)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    sim.run_round(clients, plan, out, g, lr=wl.lr, seed=wl.seed, rnd=1)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    sim.close()


if __name__ == "__main__":
    main()
