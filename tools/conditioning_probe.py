"""Conditioning of the local-SGD iteration (oracle only, float64): how far the federated result of
one config-2 client moves when the initial weights move by one fp32 rounding (relative 2^-24).
Explains why no finite-precision path can meet a fixed rel-L2 bar against float64 over long local
horizons (126 steps at B = 8), while short horizons agree (full-size parity)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402
from oracle import round as orr  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def main():
    wl = synth.build_workload(2)
    w0 = synth.init_weights(wl.model).astype(np.float64)
    rng = np.random.default_rng(0)
    w1 = w0 * (1.0 + 2.0 ** -24 * rng.choice([-1.0, 1.0], w0.size))
    for cid in (int(a) for a in (sys.argv[1:] or ["0", "3"])):
        cl = [c for c in wl.clients if c.id == cid]
        t = time.time()
        a = orr.run_round(cl, wl.shards, {4: w0}, wl.lr, wl.seed, 0)[4]
        b = orr.run_round(cl, wl.shards, {4: w1}, wl.lr, wl.seed, 0)[4]
        print(f"client {cid} (B={cl[0].batch}, {cl[0].epochs * -(-cl[0].n // cl[0].batch)} steps): input perturbation "
              f"{rel(w1, w0):.2e} -> result rel-L2 {rel(b, a):.2e}, update rel-L2 {rel(b - w1, a - w0):.2e} "
              f"({time.time() - t:.0f} s)", flush=True)


if __name__ == "__main__":
    main()
