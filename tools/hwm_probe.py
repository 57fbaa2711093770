"""Which slot buffers does one local step touch?  protea_profile_clients leaves its observation probe in
the arena (slots back to back in client order, each followed by a 4 KiB guard); this reads the arena and
reports, per client and per buffer of the layout (oracle.profiler.slot_layout), the touched fraction and
the highest touched byte.  Usage: python tools/hwm_probe.py  (GPU)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import synth  # noqa: E402
from oracle.profiler import align256, slot_layout  # noqa: E402
from paper_2207_01053_b200.sim import Simulation  # noqa: E402

POISON = 0xA5
cases = [(1, dict(n_clients=4, samples=20), 1, (4,)), (1, dict(n_clients=4, samples=20), 0, (4,)),
         (2, dict(n_clients=4, samples=70), 1, (4,)), (2, dict(n_clients=4, samples=70), 0, (4,)),
         (4, dict(n_clients=300, k=12, samples=70), 1, (1, 2, 4)), (5, dict(n_clients=300, k=8, samples=70), 1, (4,)),
         (5, dict(n_clients=300, k=8, samples=70), 0, (4,))]
for config, kw, prec, widths in cases:
    wl = synth.build_workload(config, **kw)
    H, W, C = (28, 28, 1) if wl.model == synth.MODEL_MLP else (32, 32, 3)
    sim = Simulation(precision=prec, arena_bytes=1 << 30)
    mids = {w: sim.register_model(wl.model, w, 10, H, W, C) for w in widths}
    sim.register_shards([(c.id, *wl.shards[c.id]) for c in wl.clients])
    clients = sim.clients([(c.id, mids[c.width_q], c.batch, c.epochs) for c in wl.clients])
    prof = sim.profile(clients)
    arena = sim.arena.cpu().numpy()
    eb = 4 if prec == 0 else 2
    off = 0
    for c, p in zip(wl.clients, prof):
        lay = slot_layout(c.model, c.width_q, 10, c.batch, c.n, c.epochs, eb)
        need = sum(align256(s) for _, s in lay)
        rep = {}
        o = off
        for name, size in lay:
            seg = arena[o:o + size] != POISON
            hi = int(np.nonzero(seg)[0].max()) + 1 if seg.any() else 0
            if hi < size:
                rep[name] = {"bytes": size, "touched": int(seg.sum()), "highest": hi}
            o += align256(size)
        print(json.dumps({"config": config, "prec": eb, "id": c.id, "B": c.batch, "n": c.n, "wq": c.width_q,
                          "observed": int(p["peak_bytes"]), "layout": need, "untouched_tails": rep}))
        off += need + 4096
    sim.close()
