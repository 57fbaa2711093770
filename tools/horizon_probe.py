"""fp32 verify mode vs the float64 oracle for one config-2 client as the local horizon grows
(n samples, B, E): localises where a long-horizon deviation starts."""
import dataclasses
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from oracle import round as orr  # noqa: E402
from paper_2207_01053_b200.sim import Simulation  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def main():
    wl = synth.build_workload(2)
    w0 = synth.init_weights(wl.model)
    base = wl.clients[3]  # B = 64
    tmpl = synth.class_templates(wl.shape, wl.classes, wl.seed)
    for n, B, E, shuffle in ((64, 64, 1, True), (128, 64, 1, True), (500, 64, 1, True), (500, 64, 1, False),
                             (500, 64, 2, True), (64, 8, 1, True), (500, 8, 1, False)):
        c = dataclasses.replace(base, n=n, batch=B, epochs=E)
        shards = {c.id: synth.make_shard(tmpl, n, c.id, wl.seed)}
        ref = orr.run_round([c], shards, {4: w0}, wl.lr, wl.seed, 0, shuffle=shuffle)[4]
        sim = Simulation(precision=0, arena_bytes=1 << 30)
        mid = sim.register_model(wl.model, 4, 10, 32, 32, 3)
        sim.register_shards([(c.id, *shards[c.id])])
        cl = sim.clients([(c.id, mid, c.batch, c.epochs)])
        plan, _ = sim.plan(sim.profile(cl))
        g, _ = sim.run_round(cl, plan, torch.tensor(w0, device="cuda"), lr=wl.lr, seed=wl.seed, shuffle=shuffle)
        got = g.cpu().numpy().astype(np.float64)
        sim.close()
        print(f"n={n} B={B} E={E} shuffle={shuffle}: weights {rel(got, ref):.2e} update {rel(got - w0, ref - w0):.2e}",
              flush=True)


if __name__ == "__main__":
    main()
