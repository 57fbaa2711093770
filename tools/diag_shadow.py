"""After a bf16 round, read the client slot back from the arena and check the
bf16 weight shadow == bf16(fp32 master) for conv2 / fc1."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
from oracle import sgd, profiler as pf
from tests.gpu_helpers import gpu_run

wl = synth.build_workload(2, n_clients=1, samples=16, epochs=1)
for c in wl.clients:
    c.batch = 8
got, ex = gpu_run(wl, precision=1, return_sim=True)
sim = ex["sim"]
a = ex["plan"][0]
P = sgd.n_params(sgd.CNN, 4)
c = wl.clients[0]
lay = pf.slot_layout(sgd.CNN, 4, 10, c.batch, c.n, c.epochs, 2)
off = {}
o = 0
for name, sz in lay:
    off[name] = o
    o += pf.align256(sz)
slot = sim.arena[int(a["offset"]):int(a["offset"]) + o].cpu().numpy()
master = slot[off["params"]:off["params"] + 4 * P].view(np.float32)
shadow = slot[off["wsh"]:off["wsh"] + 2 * P].view(np.uint16)
mb = sgd.bf16(master.astype(np.float64)).astype(np.float32).view(np.uint32) >> 16
p = 0
for name, ws, bs in sgd.layer_shapes(sgd.CNN, 4, 10):
    for part, shp in (("W", ws), ("b", bs)):
        n = int(np.prod(shp))
        bad = np.count_nonzero(mb[p:p + n] != shadow[p:p + n])
        print(f"{name}.{part}: {bad}/{n} shadow != bf16(master); master-vs-final-global max diff {np.abs(master[p:p+n]-got[4][p:p+n]).max():.3e}")
        p += n
