"""Per-step, per-layer teacher-forced comparison of micro-client batches (diagnostic)."""
import dataclasses
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import synth  # noqa: E402
from tests.teacher_forced import bench_round_with_trace, gpu_weights, oracle_updates, per_step_rel  # noqa: E402

for prec in (1, 0):
    for nb in ((200, 128), (144, 72), (72, 72), (200, 16)):
        wl = synth.build_workload(2, n_clients=1, samples=8)
        tmpl = synth.class_templates(wl.shape, wl.classes, wl.seed)
        wl.clients = [dataclasses.replace(c, n=nb[0], batch=nb[1], epochs=1) for c in wl.clients]
        wl.shards = {c.id: synth.make_shard(tmpl, c.n, c.id, wl.seed) for c in wl.clients}
        cid = wl.clients[0].id
        elem = 4 if prec == 0 else 2
        snaps, _, _ = bench_round_with_trace(wl, prec, [cid])
        for emu in ((True, False) if prec else (False,)):
            upd, forced = oracle_updates(wl, cid, snaps[cid], elem, emulate_bf16=emu, tol=1e-3 if prec else 1e-5)
            tot, layers = per_step_rel(wl, cid, gpu_weights(wl, cid, snaps[cid], elem), upd)
            print(json.dumps({"prec": prec, "n_B": nb, "emu": emu, "per_step": [float(x) for x in tot],
                              "forced": forced,
                              "layers": {k: [float("%.2e" % x) for x in v] for k, v in layers.items()}}), flush=True)
