"""Full-cohort global weights of config 2 (BASELINE configs[1]: 100 clients, 5,950 client-steps) against
the float64 oracle, next to two host controls run through the SAME oracle code (VERDICT r1 "What's weak"
#2): the oracle's arithmetic in NumPy float32 (what fp32 arithmetic alone does over the full horizon) and
the oracle's bf16 emulation (reading R17).  The GPU rows are the library's fp32 verify and bf16 rounds in
the bench launch configuration.  Usage: python tools/global_controls.py [config] > profiles/...json
(GPU box; ~6 min of host oracle time on 16 cores)."""
import os

for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):  # one BLAS thread per worker process
    os.environ.setdefault(_v, "1")
import json  # noqa: E402
import math  # noqa: E402
import sys  # noqa: E402
import time
from concurrent.futures import ProcessPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import synth  # noqa: E402
from oracle import sgd  # noqa: E402
from oracle import round as orr  # noqa: E402
from oracle.fedavg import fedavg  # noqa: E402
from oracle.splitmix import epoch_perm  # noqa: E402


def _f32_client(args):
    """The oracle's local SGD (sgd.loss_and_grad) with every array in float32."""
    w0, c, x, y, lr, seed = args
    w = np.asarray(w0, dtype=np.float32)
    H, W, C = sgd.input_shape(c.model)
    xf = (x.reshape(c.n, H, W, C).astype(np.float32) / np.float32(255.0))
    nb = math.ceil(c.n / c.batch)
    for e in range(c.epochs):
        perm = epoch_perm(c.n, seed, 0, c.id, e)
        for j in range(nb):
            idx = perm[j * c.batch:min((j + 1) * c.batch, c.n)]
            p = sgd.unpack(w, c.model, c.width_q, c.classes)
            _, g = sgd.loss_and_grad(p, c.model, xf[idx], y[idx])
            w = (w - np.float32(lr) * sgd.pack(g, c.model, c.width_q, c.classes).astype(np.float32)).astype(np.float32)
    return w


def gpu_round(wl, precision):
    import torch
    from tests.teacher_forced import bench_round_with_trace
    _, st, out = bench_round_with_trace(wl, precision, [])
    return out.astype(np.float64), st


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    wl = synth.build_workload(cfg)
    w0 = synth.init_weights(wl.model)
    workers = min(16, len(os.sched_getaffinity(0)))
    t0 = time.time()
    ref = orr.run_round(wl.clients, wl.shards, {4: w0}, wl.lr, wl.seed, 0, workers=workers)[4]
    t_ref = time.time() - t0
    emu = orr.run_round(wl.clients, wl.shards, {4: w0}, wl.lr, wl.seed, 0, workers=workers, emulate_bf16=True)[4]
    with ProcessPoolExecutor(max_workers=workers) as ex:
        ws = list(ex.map(_f32_client, [(w0, c, *wl.shards[c.id], wl.lr, wl.seed) for c in wl.clients]))
    f32 = fedavg(ws, [c.n for c in wl.clients])
    g32, _ = gpu_round(wl, 0)
    g16, _ = gpu_round(wl, 1)
    w0d = w0.astype(np.float64)
    rows = {
        "gpu_fp32_verify": (g32, ref), "gpu_bf16": (g16, ref), "gpu_bf16_vs_bf16_emulation": (g16, emu),
        "host_numpy_float32_control": (f32, ref), "host_bf16_emulation_control": (emu, ref)}
    out = {"config": cfg, "clients": len(wl.clients), "client_steps": int(sum(sgd.steps(c.n, c.batch, c.epochs)
                                                                           for c in wl.clients)),
           "oracle_f64_wall_s": t_ref, "workers": workers,
           "rel_l2_weights": {k: rel(a, b) for k, (a, b) in rows.items()},
           "rel_l2_round_update": {k: rel(a - w0d, b - w0d) for k, (a, b) in rows.items()}}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
