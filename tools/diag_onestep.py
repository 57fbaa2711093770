"""One local step per client (n = B, E = 1): per-layer rel-L2 of the update, GPU vs oracle (f64 and bf16-emulated)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import synth
from oracle import sgd
from tests.gpu_helpers import gpu_run, oracle_run

B = int(sys.argv[1]) if len(sys.argv) > 1 else 8
K = int(sys.argv[2]) if len(sys.argv) > 2 else 1
LR = float(sys.argv[3]) if len(sys.argv) > 3 else 0.05
wl = synth.build_workload(2, n_clients=1, samples=B * K, epochs=1)
wl.lr = LR
for c in wl.clients:
    c.batch = B
ref64 = oracle_run(wl, lr=LR)
refem = oracle_run(wl, emulate_bf16=True, lr=LR)


def report(tag, got, ref, g0):
    dg, dr = got - g0, ref - g0
    off, out = 0, []
    for name, ws, bs in sgd.layer_shapes(wl.model, 4, 10):
        for part, shp in (("W", ws), ("b", bs)):
            n = int(np.prod(shp))
            a, b = dg[off:off + n], dr[off:off + n]
            out.append(f"{name}.{part}:{np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30):.1e}")
            off += n
    print(f"B={B} steps={K} lr={LR} {tag:14s} total {np.linalg.norm(dg - dr) / np.linalg.norm(dr):.2e} " + " ".join(out), flush=True)


g32, ex = gpu_run(wl, precision=0, lr=LR)
g16, _ = gpu_run(wl, precision=1, lr=LR)
g0 = ex["g0"][4].astype(np.float64)
report("fp32 vs f64", g32[4], ref64[4], g0)
report("bf16 vs f64", g16[4], ref64[4], g0)
report("bf16 vs emul", g16[4], refem[4], g0)
report("emul vs f64", refem[4], ref64[4], g0)
