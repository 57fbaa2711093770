"""FEMNIST-shaped CNN (28x28x1, 62 classes): teacher-forced per-step updates vs the oracle (diagnostic)."""
import dataclasses
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import synth  # noqa: E402
from tests.teacher_forced import bench_round_with_trace, gpu_weights, oracle_updates, per_step_rel  # noqa: E402

for prec in (0, 1):
    for n, B, E in ((40, 16, 2), (70, 8, 1), (100, 64, 1)):
        wl = synth.build_workload(6, n_clients=20, k=1, samples=8, epochs=1)
        tmpl = synth.class_templates(wl.shape, wl.classes, wl.seed)
        wl.clients = [dataclasses.replace(c, n=n, batch=B, epochs=E) for c in wl.clients]
        wl.shards = {c.id: synth.make_shard(tmpl, c.n, c.id, wl.seed) for c in wl.clients}
        cid = wl.clients[0].id
        elem = 4 if prec == 0 else 2
        snaps, _, _ = bench_round_with_trace(wl, prec, [cid])
        for emu, tol in (((False, 1e-5),) if prec == 0 else ((True, 1e-3), (False, 5e-2))):
            try:
                upd, forced = oracle_updates(wl, cid, snaps[cid], elem, emulate_bf16=emu, tol=tol)
            except Exception as ex:  # noqa: BLE001
                print(json.dumps({"prec": prec, "n_B_E": [n, B, E], "emu": emu, "error": str(ex)[:300]}), flush=True)
                continue
            tot, layers = per_step_rel(wl, cid, gpu_weights(wl, cid, snaps[cid], elem), upd)
            print(json.dumps({"prec": prec, "n_B_E": [n, B, E], "emu": emu, "per_step": ["%.1e" % x for x in tot],
                              "forced": {k: v for k, v in forced.items() if v},
                              "layers": {k: float("%.2e" % max(v)) for k, v in layers.items()}}), flush=True)
