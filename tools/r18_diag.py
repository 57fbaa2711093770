"""ResNet-18-GN: per-layer one-step update vs the float64 oracle (diagnostic)."""
import dataclasses
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import synth  # noqa: E402
from oracle import sgd  # noqa: E402
from tests.gpu_helpers import gpu_run, oracle_run  # noqa: E402

for prec in (0,):
    for n, B in ((2, 2), (4, 4)):
        wl = synth.build_workload(7, n_clients=1, samples=6, epochs=1)
        tmpl = synth.class_templates(wl.shape, wl.classes, wl.seed)
        wl.clients = [dataclasses.replace(c, n=n, batch=B) for c in wl.clients]
        wl.shards = {c.id: synth.make_shard(tmpl, c.n, c.id, wl.seed) for c in wl.clients}
        got, ex = gpu_run(wl, precision=prec)
        ref = oracle_run(wl)
        g0 = ex["g0"][4].astype(np.float64)
        dg, dr = got[4] - g0, ref[4] - g0
        out, off = {}, 0
        for name, ws, bs in sgd.layer_shapes(sgd.RESNET18, 4, 10):
            for part, shp in (("W", ws), ("b", bs)):
                k = int(np.prod(shp))
                a, b = dg[off:off + k], dr[off:off + k]
                out[f"{name}.{part}"] = "%.1e/%.1e" % (np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30), np.linalg.norm(b))
                off += k
        print(json.dumps({"prec": prec, "n": n, "B": B, "total": float(np.linalg.norm(dg - dr) / np.linalg.norm(dr)),
                          "layers": out}), flush=True)
