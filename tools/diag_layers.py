"""Per-layer diagnostic: rel-L2 of the round update (GPU vs float64 oracle), fp32 and bf16 modes."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import synth
from oracle import sgd
from tests.gpu_helpers import gpu_run, oracle_run

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
wl = synth.build_workload(cfg, n_clients=8, samples=45) if cfg == 2 else synth.build_workload(cfg)
ref64 = oracle_run(wl)
refem = oracle_run(wl, emulate_bf16=True)
for prec, ref, tag in ((0, ref64, "f64"), (1, ref64, "f64"), (1, refem, "bf16-emul")):
    got, ex = gpu_run(wl, precision=prec)
    for w in got:
        g0 = ex["g0"][w].astype(np.float64)
        dg, dr = got[w] - g0, ref[w] - g0
        off = 0
        out = []
        for name, ws, bs in sgd.layer_shapes(wl.model, w, 10):
            for part, shp in (("W", ws), ("b", bs)):
                n = int(np.prod(shp))
                a, b = dg[off:off + n], dr[off:off + n]
                out.append(f"{name}.{part}:{np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30):.2e}")
                off += n
        print("prec", prec, "vs", tag, "width", w, "total", np.linalg.norm(dg - dr) / np.linalg.norm(dr), " ".join(out))
