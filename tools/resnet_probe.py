"""Per-op device time of one config-5 round (ResNet-8, K=500, bf16 storage, 1 GPU)."""
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


def main():
    prec = pb.PREC_FP32 if "fp32" in sys.argv else pb.PREC_BF16
    wl = synth.build_workload(5)
    sim = Simulation(precision=prec, arena_bytes=8 << 30)
    mid = sim.register_model(wl.model, 4, 10, 32, 32, 3)
    sim.register_shards([(c.id, *wl.shards[c.id]) for c in wl.clients])
    clients = sim.clients([(c.id, mid, c.batch, c.epochs) for c in wl.clients])
    foot = np.zeros(len(wl.clients), dtype=pb.PROFILE_DT)
    for i, c in enumerate(wl.clients):
        pk, st, fl = pb.protea_client_footprint(wl.model, 4, 10, 32, 32, 3, c.n, c.batch, c.epochs, prec)
        foot[i] = (c.id, pk, st, fl, 0, 0, 0, 1, 0)
    plan, mk = pb.protea_plan(foot, [8 << 30])
    g = torch.tensor(synth.init_weights(wl.model), device=sim.device)
    out = torch.empty_like(g)
    sim.run_round(clients, plan, g, out, lr=wl.lr, seed=wl.seed, rnd=0)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    _, st = sim.run_round(clients, plan, out, g, lr=wl.lr, seed=wl.seed, rnd=1, time_ops=0xFFFFFFFF, serialize=True)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    _, st2 = sim.run_round(clients, plan, g, out, lr=wl.lr, seed=wl.seed, rnd=2)
    ops = {pb.OPC_NAMES[i]: round(float(st["op_ns"][i]) / 1e6, 2) for i in range(len(pb.OPC_NAMES)) if st["op_ns"][i] > 0}
    print(json.dumps({"round_ms": st2["round_ns"] / 1e6, "iterations": int(mk[0]), "op_ms": ops,
                      "op_tflops": {pb.OPC_NAMES[i]: round(float(st["op_flops"][i]) / max(1, float(st["op_ns"][i])) / 1e3, 2)
                                    for i in range(len(pb.OPC_NAMES)) if st["op_ns"][i] > 0}}))
    sim.close()


if __name__ == "__main__":
    main()
