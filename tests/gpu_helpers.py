"""Shared helpers for the -m gpu tests: run a synth workload through the C ABI
and through the oracle on the same seeded inputs."""
import numpy as np

import synth
from oracle import round as orr


def shape_of(model):
    return synth.INPUT_SHAPE[model]


def arch_of(model):
    """the library's arch id of a harness model (MODEL_CNN28 = the CNN arch on a 28x28x1 input)"""
    return synth.LIB_ARCH[model]


def widths_of(wl, all_widths=False):
    if all_widths and wl.model == synth.MODEL_CNN:
        return [1, 2, 4]
    return sorted({c.width_q for c in wl.clients})


def init_globals(wl, widths, seed=0):
    return {wq: synth.init_weights(wl.model, wq, wl.classes, seed=seed) for wq in widths}


def gpu_run(wl, rounds=1, precision=0, lr=0.05, arena_bytes=None, shuffle=True, all_widths=False, caps=None,
            policy=0, order=0, max_active=0, init_seed=0, sim=None, return_sim=False):
    import torch
    from paper_2207_01053_b200.sim import Simulation, concat_globals
    widths = widths_of(wl, all_widths)
    H, W, C = shape_of(wl.model)
    if sim is None:
        sim = Simulation(precision=precision, arena_bytes=arena_bytes or (1 << 30))
    mids = {wq: sim.register_model(arch_of(wl.model), wq, wl.classes, H, W, C) for wq in widths}
    sim.register_shards([(c.id, wl.shards[c.id][0], wl.shards[c.id][1]) for c in wl.clients])
    clients = sim.clients([(c.id, mids[c.width_q], c.batch, c.epochs) for c in wl.clients])
    prof = sim.profile(clients)
    plan, mk = sim.plan(prof, caps=caps, policy=policy, order=order, max_active=max_active)
    g0 = init_globals(wl, widths, init_seed)
    g = torch.tensor(concat_globals([g0[w] for w in widths]), device="cuda")
    stats = []
    for r in range(rounds):
        g, st = sim.run_round(clients, plan, g, lr=lr, seed=wl.seed, rnd=r, shuffle=shuffle)
        stats.append(st)
    out = g.cpu().numpy()
    res, off = {}, 0
    for w in widths:
        n = g0[w].size
        res[w] = out[off:off + n]
        off += n
    extra = dict(prof=prof, plan=plan, makespans=mk, stats=stats, g0=g0)
    if return_sim:
        extra["sim"] = sim
    else:
        sim.close()
    return res, extra


def oracle_run(wl, rounds=1, lr=0.05, shuffle=True, all_widths=False, init_seed=0, g0=None, workers=0,
               emulate_bf16=False):
    widths = widths_of(wl, all_widths)
    g = {w: v.astype(np.float64) for w, v in (g0 or init_globals(wl, widths, init_seed)).items()}
    for r in range(rounds):
        g = orr.run_round(wl.clients, wl.shards, g, lr, wl.seed, r, shuffle=shuffle, workers=workers,
                          emulate_bf16=emulate_bf16)
    return g


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))
