"""Paper-analogue arms on B200: round time of the
profile-driven packing (PROFILED: slots from the exact arena HWM)
against the paper's "original setup" (STATIC: one client per whole GPU, run
sequentially), for the shapes of the paper's experiments:

  Exp I: homogeneous clients, pool 100, clients/round 10 -> 100
  Exp II: heterogeneous batch sizes, one third each
                      (paper 32/1024/2048; here 8/32/64, the library's range)
  Exp III: Exp II under an emulated capacity small enough
                      that memory packing binds (256 MiB for 14-24 MiB slots,
                      the paper's 11 GiB GTX 1080 Ti scaled to our footprints):
                      STATIC (one client per GPU), FIXED (a uniform fraction
                      sized for the largest client, as a fixed Ray num_gpus
                      would give: max_active = C // max HWM) and PROFILED
                      (exact HWM slots, FIFO first-fit); with the mean
                      allocated fraction of C over the lock-step iterations.

Workload: CNN-1x on synthetic CIFAR-shaped data, 500 samples/client, E=1,
bf16 tensor-core mode.  Output: one JSON document (stdout) with per-arm round
time (CUDA events), client-steps/s, achieved TFLOP/s and the speed-up, beside
the paper's 1.56x / 1.66x on GTX 1080 Ti (context only, not comparable).
"""
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


def run_arm(sim, mid, wl, ids, policy, reps=2, caps=None, max_active=0):
    clients = sim.clients([(c.id, mid, c.batch, c.epochs) for c in wl.clients if c.id in ids])
    prof = sim.profile(clients)
    plan, mk = sim.plan(prof, caps=caps, policy=policy, max_active=max_active)
    g = torch.tensor(synth.init_weights(synth.MODEL_CNN), device="cuda")
    out = torch.empty_like(g)
    sim.run_round(clients, plan, g, out, lr=0.05, seed=1, rnd=0)  # warm-up
    best = None
    for r in range(reps):
        _, st = sim.run_round(clients, plan, g, out, lr=0.05, seed=1, rnd=r + 1)
        best = st if best is None or st["round_ns"] < best["round_ns"] else best
    steps = int(sum(int(p["steps"]) for p in prof))
    flops = int(sum(int(p["flops"]) for p in prof))
    ms = best["round_ns"] / 1e6
    T = int(mk[0])
    live = np.zeros(T)
    conc = np.zeros(T)
    for a in plan:
        live[int(a["admit"]):int(a["release"])] += int(a["slot"])
        conc[int(a["admit"]):int(a["release"])] += 1
    cap = (caps or [sim.arena.numel()])[0]
    return {"round_ms": ms, "iterations": T, "client_steps": steps,
            "client_steps_per_s": steps / (ms / 1e3), "tflops": flops / (ms / 1e3) / 1e12,
            "kernel_launches": best["kernel_launches"], "mean_allocated_frac": float(live.mean() / cap),
            "peak_concurrent_clients": int(conc.max())}


def main():
    res = {"hardware": torch.cuda.get_device_name(0), "precision": "bf16", "model": "CNN-1x, CIFAR-shaped synthetic",
           "samples_per_client": 500, "epochs": 1,
           "paper_context": {"exp1_cifar_speedup": 1.56, "exp1_femnist_speedup": 2.35, "exp2_speedup": 1.66,
                             "gpu_util_gain": 2.6, "hardware": "GTX 1080 Ti (paper P:304); not comparable"},
           "exp1": [], "exp2": []}
    pool = 100
    wl = synth.build_workload(2, n_clients=pool, samples=500, epochs=1)
    for c in wl.clients:
        c.batch = 32
    sim = Simulation(precision=pb.PREC_BF16, arena_bytes=8 << 30)
    mid = sim.register_model(pb.MODEL_CNN, 4, 10, 32, 32, 3)
    sim.register_shards([(c.id, *wl.shards[c.id]) for c in wl.clients])
    for k in (10, 20, 50, 100):
        ids = set(int(i) for i in synth.sample_clients(pool, k, seed=3, rnd=0))
        prof = run_arm(sim, mid, wl, ids, pb.POLICY_PROFILED)
        stat = run_arm(sim, mid, wl, ids, pb.POLICY_STATIC, reps=1)
        res["exp1"].append({"clients_per_round": k, "profiled": prof, "static": stat,
                            "speedup": stat["round_ms"] / prof["round_ms"]})
        print(json.dumps(res["exp1"][-1]), file=sys.stderr, flush=True)
    sim.close()
    # Exp II: one third each at batch 8 / 32 / 64
    wl2 = synth.build_workload(2, n_clients=pool, samples=500, epochs=1)
    for c in wl2.clients:
        c.batch = (8, 32, 64)[c.id % 3]
    sim = Simulation(precision=pb.PREC_BF16, arena_bytes=8 << 30)
    mid = sim.register_model(pb.MODEL_CNN, 4, 10, 32, 32, 3)
    sim.register_shards([(c.id, *wl2.shards[c.id]) for c in wl2.clients])
    for k in (30, 99):
        ids = set(int(i) for i in synth.sample_clients(pool, k, seed=4, rnd=0))
        prof = run_arm(sim, mid, wl2, ids, pb.POLICY_PROFILED)
        stat = run_arm(sim, mid, wl2, ids, pb.POLICY_STATIC, reps=1)
        res["exp2"].append({"clients_per_round": k, "batches": [8, 32, 64], "profiled": prof, "static": stat,
                            "speedup": stat["round_ms"] / prof["round_ms"]})
        print(json.dumps(res["exp2"][-1]), file=sys.stderr, flush=True)
    # Exp III: the same heterogeneous cohort under a capacity where memory binds
    cap = 256 << 20
    ids = set(int(i) for i in synth.sample_clients(pool, 99, seed=4, rnd=0))
    cl = [c for c in wl2.clients if c.id in ids]
    max_hwm = max(pb.protea_client_footprint(pb.MODEL_CNN, 4, 10, 32, 32, 3, c.n, c.batch, c.epochs, pb.PREC_BF16)[0]
                  for c in cl)
    arms = {}
    sim.close()
    sim = Simulation(precision=pb.PREC_BF16, arena_bytes=8 << 30)
    mid = sim.register_model(pb.MODEL_CNN, 4, 10, 32, 32, 3)
    sim.register_shards([(c.id, *wl2.shards[c.id]) for c in wl2.clients])
    arms["static"] = run_arm(sim, mid, wl2, ids, pb.POLICY_STATIC, reps=1, caps=[cap])
    arms["fixed"] = run_arm(sim, mid, wl2, ids, pb.POLICY_PROFILED, caps=[cap], max_active=int(cap // max_hwm))
    arms["profiled"] = run_arm(sim, mid, wl2, ids, pb.POLICY_PROFILED, caps=[cap])
    res["exp3"] = {"capacity_bytes": cap, "max_hwm_bytes": int(max_hwm), "fixed_max_active": int(cap // max_hwm),
                   "batches": [8, 32, 64], "clients_per_round": 99, **arms,
                   "speedup_vs_static": arms["static"]["round_ms"] / arms["profiled"]["round_ms"],
                   "speedup_vs_fixed": arms["fixed"]["round_ms"] / arms["profiled"]["round_ms"]}
    print(json.dumps(res["exp3"]), file=sys.stderr, flush=True)
    sim.close()
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
