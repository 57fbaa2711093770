"""Teacher-forced per-step parity helpers (GPU runs; the oracle steps on the host).

A full-size client's trajectory separates from the float64 oracle over a long
horizon through discrete decisions (ReLU masks, max-pool argmaxes) whose
margins fall below fp32 / bf16 rounding (DESIGN.md §3 "Full-size parity").
Teacher forcing removes the horizon: the library snapshots a traced client's
fp32 weights after every local step of the round it really runs
(protea_round_opts.trace_*), and for every step s the oracle takes ONE step
from the GPU's w_s on the same batch (the SplitMix64 permutation, reading
R10).  The per-step update w_{s+1} - w_s is then compared with the oracle's
-lr * grad(w_s) at the north-star bars."""
from __future__ import annotations

import math
import multiprocessing as mp

import numpy as np

import synth
from oracle import sgd
from oracle.splitmix import epoch_perm

_JOB = {}


def slot_offsets(c, elem):
    """{buffer: (byte offset, bytes)} of client c's slot (oracle.profiler.slot_layout, pinned by
    tests/golden/hwm.json; buffers in slot order, each aligned to 256 B)."""
    from oracle.profiler import align256, slot_layout
    off, out = 0, {}
    for name, size in slot_layout(c.model, c.width_q, c.classes, c.batch, c.n, c.epochs, elem):
        out[name] = (off, size)
        off += align256(size)
    return out


def _act(raw, off, size, elem, shape):
    b = raw[off:off + size]
    if elem == 4:
        v = b.view(np.float32)
    else:  # bf16 -> fp32 exactly
        v = (b.view(np.uint16).astype(np.uint32) << 16).view(np.float32)
    return v.astype(np.float64).reshape(shape)


def master_weights(c, raw, elem):
    """The fp32 master weights at the start of a slot snapshot.  bf16-mode CNN: fc1's W is stored as 16-bit
    halves, per row f and 128-block of k1: 128 upper halves then 128 lower halves (DESIGN.md §5 "split
    planes")."""
    P = sgd.n_params(c.model, c.width_q, c.classes)
    w = raw[:4 * P].copy().view(np.float32)
    if elem == 2 and c.model == sgd.CNN:  # (the tcgen05 path; CNN28 runs SIMT kernels on plain fp32)
        c1, c2, f = sgd.cnn_channels(c.width_q)
        off = (c1 * 75 + c1) + (c2 * 25 * c1 + c2)
        nw = f * 64 * c2
        K1 = nw // f
        blocks = raw[4 * off:4 * (off + nw)].view(np.uint16).reshape(f, K1 // 128, 2, 128)
        u = (blocks[:, :, 0, :].astype(np.uint32) << 16) | blocks[:, :, 1, :].astype(np.uint32)
        w[off:off + nw] = u.reshape(-1).view(np.float32)
    return w


def decode_snapshot(c, raw, elem, rows):
    """(fp32 weights, GPU decisions of the step that produced the snapshot) from one slot snapshot.  A
    batch of more than 64 rows runs as micro-clients (slots of <= 64 rows back to back):
    the decisions are concatenated over them, the weights are micro 0's (the merged ones)."""
    from oracle.profiler import MICRO_ROWS, hwm_bytes
    b = min(c.batch, c.n)
    if b > MICRO_ROWS:
        import dataclasses
        parts, off, w = [], 0, None
        for r0 in range(0, b, MICRO_ROWS):
            cap = min(MICRO_ROWS, b - r0)
            cm = dataclasses.replace(c, batch=cap)
            size = hwm_bytes(c.model, c.width_q, c.classes, cap, c.n, c.epochs, elem)
            wm, dm = decode_snapshot(cm, raw[off:off + size], elem, max(0, min(cap, rows - r0)))
            w = wm if w is None else w
            parts.append(dm)
            off += size
        return w, {k: np.concatenate([d[k] for d in parts]) for k in parts[0]}
    lay = slot_offsets(c, elem)
    w = master_weights(c, raw, elem)
    B = b  # per-row buffers hold min(B, n) rows (slot layout)
    dec = {}
    if c.model == sgd.MLP:
        o, n = lay["h1"]
        dec["h1"] = _act(raw, o, n, elem, (B, 64))[:rows]
    elif c.model in (sgd.CNN, sgd.CNN28):
        c1, c2, f = sgd.cnn_channels(c.width_q)
        s1, s2 = (16, 8) if c.model == sgd.CNN else (14, 7)
        for k, shp in (("a1", (B, s1, s1, c1)), ("a2", (B, s2, s2, c2)), ("h", (B, f))):
            o, n = lay[k]
            dec[k] = _act(raw, o, n, elem, shp)[:rows]
        for k, shp in (("i1", (B, s1, s1, c1)), ("i2", (B, s2, s2, c2))):
            o, n = lay[k]
            dec[k] = raw[o:o + n].astype(np.int64).reshape(shp)[:rows]
    elif c.model == sgd.RESNET18:  # y_l: the activation after GroupNorm (+ shortcut) and ReLU of conv layer l
        from oracle.profiler import conv_layers
        hw = [h for h, _, _ in conv_layers(sgd.RESNET18)]
        co = [ch for _, ch, _ in conv_layers(sgd.RESNET18)]
        for l in range(17):
            key = "a0" if l == 0 else (f"r{(l - 1) // 2}" if l % 2 == 1 else f"o{(l - 2) // 2}")
            side = int(round(hw[l] ** 0.5))
            o, n = lay[f"y{l}"]
            dec[key] = _act(raw, o, n, elem, (B, side, side, co[l]))[:rows]
    else:
        for k, shp in (("a0", (B, 32, 32, 16)), ("r1", (B, 32, 32, 16)), ("o1", (B, 32, 32, 16)),
                       ("r2", (B, 16, 16, 32)), ("o2", (B, 16, 16, 32)), ("r3", (B, 8, 8, 64)),
                       ("o3", (B, 8, 8, 64))):
            o, n = lay[k]
            dec[k] = _act(raw, o, n, elem, shp)[:rows]
    return w, dec


def bench_round_with_trace(wl, precision, trace_ids, lr=None, rnd=0):
    """Run wl's whole cohort as bench.py does (footprint profiles, one GPU, every client admitted at t=0,
    default launch configuration) and return {id: slot snapshots uint8 [S_k + 1, H_k]} and the round
    stats (H_k = the client's footprint peak_bytes)."""
    import torch

    import paper_2207_01053_b200 as pb
    from paper_2207_01053_b200.sim import Simulation
    lr = wl.lr if lr is None else lr
    arch = synth.LIB_ARCH[wl.model]
    H, W, C = synth.INPUT_SHAPE[wl.model]
    foot = np.zeros(len(wl.clients), dtype=pb.PROFILE_DT)
    for i, c in enumerate(wl.clients):
        pk, st, fl = pb.protea_client_footprint(arch, c.width_q, c.classes, H, W, C, c.n, c.batch, c.epochs,
                                                precision)
        foot[i] = (c.id, pk, st, fl, 0, 0, 0, 1, 0)
    arena = int(sum(int(f["peak_bytes"]) for f in foot) * 1.25) + (256 << 20)
    sim = Simulation(precision=precision, arena_bytes=arena)
    mid = sim.register_model(arch, 4, wl.classes, H, W, C)
    sim.register_shards([(c.id, *wl.shards[c.id]) for c in wl.clients])
    clients = sim.clients([(c.id, mid, c.batch, c.epochs) for c in wl.clients])
    plan, _ = pb.protea_plan(foot, [arena])
    byid = {c.id: c for c in wl.clients}
    hk = {int(f["client_id"]): int(f["peak_bytes"]) for f in foot}
    bufs = {cid: torch.empty((sgd.steps(byid[cid].n, byid[cid].batch, byid[cid].epochs) + 1) * hk[cid],
                             dtype=torch.uint8, device=sim.device) for cid in trace_ids}
    g = torch.tensor(synth.init_weights(wl.model, 4, wl.classes), device=sim.device)
    out, st = sim.run_round(clients, plan, g, lr=lr, seed=wl.seed, rnd=rnd, trace=bufs)
    snaps = {cid: b.view(-1, hk[cid]).cpu().numpy() for cid, b in bufs.items()}
    sim.close()
    return snaps, st, out.cpu().numpy()


def _step(args):
    s, emulate, tol = args
    j = _JOB
    c = j["client"]
    x, y = j["shard"]
    n = c.n
    nb = math.ceil(n / c.batch)
    e, b = divmod(s, nb)
    perm = epoch_perm(n, j["seed"], j["rnd"], c.id, e)
    idx = perm[b * c.batch:min((b + 1) * c.batch, n)]
    H, W, C = sgd.input_shape(c.model)
    xb = x[idx].reshape(len(idx), H, W, C).astype(np.float64) / 255.0
    w, _ = decode_snapshot(c, j["snaps"][s], j["elem"], len(idx))
    dec = None
    if tol is not None:  # the GPU's decisions of step s live in snapshot s + 1
        _, dec = decode_snapshot(c, j["snaps"][s + 1], j["elem"], len(idx))
    _, gr = sgd.flat_loss_and_grad(w.astype(np.float64), c.model, c.width_q, c.classes, xb, y[idx], emulate,
                                   dec, tol or 0.0)
    return -j["lr"] * gr, (dec or {}).get("_forced", {})


def oracle_updates(wl, cid, snaps, elem, emulate_bf16=False, tol=None, lr=None, rnd=0, workers=None):
    """[S_k, P] float64: the oracle's update of each step s from the GPU's snapshot s (tol: take the GPU's
    ReLU / pool decisions where valid within tol, oracle.sgd.forced_*), and the forced-decision counts."""
    c = next(c for c in wl.clients if c.id == cid)
    _JOB.update(client=c, shard=wl.shards[cid], snaps=snaps, seed=wl.seed, rnd=rnd, elem=elem,
                lr=wl.lr if lr is None else lr)
    S = snaps.shape[0] - 1
    workers = workers or min(16, len(__import__("os").sched_getaffinity(0)))
    with mp.get_context("fork").Pool(workers) as pool:
        res = pool.map(_step, [(s, emulate_bf16, tol) for s in range(S)], chunksize=1)
    forced = {}
    for _, f in res:
        for k, v in f.items():
            forced[k] = forced.get(k, 0) + v
    return np.stack([r[0] for r in res]), forced


def gpu_weights(wl, cid, snaps, elem):
    c = next(c for c in wl.clients if c.id == cid)
    return np.stack([master_weights(c, s, elem) for s in snaps])


def per_step_rel(wl, cid, wsnaps, upd_oracle):
    """Per step: rel-L2 of the GPU update (weights s+1 - s) vs the oracle's, overall and per layer.
    Both sides hold the step's result as fp32 master weights (reading R17), so the oracle's new weights
    w_s - lr g are rounded to fp32 once, as the GPU's SGD epilogue rounds them; the norm of the
    unrounded oracle update is the denominator."""
    c = next(c for c in wl.clients if c.id == cid)
    w0 = wsnaps[:-1].astype(np.float64)
    d_gpu = wsnaps[1:].astype(np.float64) - w0
    d_or32 = (w0 + upd_oracle).astype(np.float32).astype(np.float64) - w0
    tot = np.linalg.norm(d_gpu - d_or32, axis=1) / np.linalg.norm(upd_oracle, axis=1)
    layers = {}
    off = 0
    for name, ws, bs in sgd.layer_shapes(c.model, c.width_q, c.classes):
        for part, shp in (("W", ws), ("b", bs)):
            n = int(np.prod(shp))
            a, b, u = d_gpu[:, off:off + n], d_or32[:, off:off + n], upd_oracle[:, off:off + n]
            layers[f"{name}.{part}"] = np.linalg.norm(a - b, axis=1) / np.maximum(np.linalg.norm(u, axis=1), 1e-300)
            off += n
    return tot, layers
