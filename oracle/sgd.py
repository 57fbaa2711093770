"""Local SGD of one client, float64 (oracle; test infrastructure only).

PAPER.md never states the local training recipe: clients "finish training"
(§3.2), ResNet-18 / LEAF CNN are named (§4.1) and batch sizes vary
per client (§4.3).  The recipe below is DESIGN.md reading R10 (SURVEY
§8(c).2), followed step by step:

 1. x = u8 / 255.
 2. epoch permutation pi_{k,e} (oracle/splitmix.py); `shuffle=False` = identity.
 3. batch j = pi[jB, min((j+1)B, n)), the last partial batch kept.
 4. forward: conv kxk zero-pad "same" (stride s), ReLU y=max(x,0) with
    ReLU'(0)=0, max-pool 2x2/2 whose backward routes to the FIRST maximum in
    row-major window order (strict >), FC y = x W^T + b.
 5. loss = mean over the actual batch |beta| of CE(softmax(z), y), softmax
    stabilised by the row max; dz = (softmax - onehot)/|beta|.
 6. backward per layer in reverse: dX = dY W with the pre-update W,
    dW = dY^T X, db = sum_rows dY; no dX for layer 1.
 7. plain SGD W <- W - lr dW, b <- b - lr db (no momentum / weight decay).
 8. repeat for E epochs; the client returns (w_k, n_k).

Models (reading R11):
  MLP 784-64-10;
  CNN-w: conv5x5 3->32w, ReLU, pool2; conv5x5 32w->64w, ReLU, pool2;
         FC 64w*64 -> 512w, ReLU; FC 512w -> classes;
  ResNet-8 (He et al. 6n+2, n=1): conv3x3 3->16, ReLU; 3 basic blocks
         (16, 32, 64 channels; stride 2 at blocks 2,3; option-A shortcut =
         subsample x[:, ::2, ::2] and zero-pad the new channels at the END);
         global average pool; FC 64 -> classes.  Conv biases, no BatchNorm.

Layouts: activations NHWC; conv weights [Cout, k, k, Cin]; FC weights
[out, in]; the CNN's FC1 input is the NHWC flatten of [8, 8, C2].  Flat
parameter order: per layer W then b, layers in forward order.

Convolution here is written as an explicit im2col + matmul (a library matmul
used as one step); pooling and its backward are written out per window.
"""
from __future__ import annotations

import math

import numpy as np

from .splitmix import epoch_perm

MLP, CNN, RESNET8, CNN28, RESNET18 = 0, 1, 2, 3, 4  # CNN28: the CNN-w family on a 28x28x1 (FEMNIST-shaped)
# input; RESNET18: the paper's CIFAR model with GroupNorm (reading R26)
GN_GROUPS, GN_EPS = 2, 1e-5


def resnet18_blocks():
    """[(block name, cin, cout, stride)] of the 8 basic blocks (4 stages x 2, 64 / 128 / 256 / 512 channels,
    stride 2 at the first block of stages 2-4)."""
    out, cin = [], 64
    for s, c in enumerate((64, 128, 256, 512)):
        for b in range(2):
            out.append((f"s{s + 1}b{b}", cin, c, 2 if (s > 0 and b == 0) else 1))
            cin = c
    return out


# ---------------------------------------------------------------------------
# model tables (the oracle's own copy)
# ---------------------------------------------------------------------------
def cnn_channels(width_q):
    w = width_q / 4.0
    return int(round(32 * w)), int(round(64 * w)), int(round(512 * w))


def layer_shapes(model, width_q=4, classes=10):
    """List of (name, W shape, b shape)."""
    if model == MLP:
        return [("fc1", (64, 784), (64,)), ("fc2", (classes, 64), (classes,))]
    if model in (CNN, CNN28):
        c1, c2, f = cnn_channels(width_q)
        cin, pooled = (3, 64) if model == CNN else (1, 49)  # 32x32x3 -> 8x8 after two pools; 28x28x1 -> 7x7
        return [("conv1", (c1, 5, 5, cin), (c1,)), ("conv2", (c2, 5, 5, c1), (c2,)),
                ("fc1", (f, pooled * c2), (f,)), ("fc2", (classes, f), (classes,))]
    if model == RESNET18:  # conv W / b, then the following GroupNorm's gamma / beta as a (C,), (C,) pair
        out = [("conv0", (64, 3, 3, 3), (64,)), ("gn0", (64,), (64,))]
        for name, cin, cout, _ in resnet18_blocks():
            out += [(name + "a", (cout, 3, 3, cin), (cout,)), (name + "ga", (cout,), (cout,)),
                    (name + "b", (cout, 3, 3, cout), (cout,)), (name + "gb", (cout,), (cout,))]
        return out + [("fc", (classes, 512), (classes,))]
    if model == RESNET8:
        return [("conv0", (16, 3, 3, 3), (16,)),
                ("b1a", (16, 3, 3, 16), (16,)), ("b1b", (16, 3, 3, 16), (16,)),
                ("b2a", (32, 3, 3, 16), (32,)), ("b2b", (32, 3, 3, 32), (32,)),
                ("b3a", (64, 3, 3, 32), (64,)), ("b3b", (64, 3, 3, 64), (64,)),
                ("fc", (classes, 64), (classes,))]
    raise ValueError(model)


def n_params(model, width_q=4, classes=10):
    return sum(int(np.prod(w)) + int(np.prod(b)) for _, w, b in layer_shapes(model, width_q, classes))


def unpack(flat, model, width_q=4, classes=10):
    p, off = {}, 0
    for name, ws, bs in layer_shapes(model, width_q, classes):
        nw, nb = int(np.prod(ws)), int(np.prod(bs))
        p[name + ".W"] = flat[off:off + nw].reshape(ws)
        off += nw
        p[name + ".b"] = flat[off:off + nb].reshape(bs)
        off += nb
    assert off == flat.size
    return p


def pack(p, model, width_q=4, classes=10):
    return np.concatenate([np.concatenate([p[n + ".W"].ravel(), p[n + ".b"].ravel()])
                           for n, _, _ in layer_shapes(model, width_q, classes)])


def input_shape(model):
    return (28, 28, 1) if model in (MLP, CNN28) else (32, 32, 3)  # RESNET18, RESNET8, CNN: CIFAR-shaped


# ---------------------------------------------------------------------------
# layer primitives
# ---------------------------------------------------------------------------
def im2col(x, k, stride, pad):
    """x [n,H,W,C] -> cols [n,Ho,Wo,k,k,C] with zero padding."""
    n, H, W, C = x.shape
    Ho = (H + 2 * pad - k) // stride + 1
    Wo = (W + 2 * pad - k) // stride + 1
    xp = np.zeros((n, H + 2 * pad, W + 2 * pad, C), dtype=x.dtype)
    xp[:, pad:pad + H, pad:pad + W, :] = x
    cols = np.empty((n, Ho, Wo, k, k, C), dtype=x.dtype)
    for ky in range(k):
        for kx in range(k):
            cols[:, :, :, ky, kx, :] = xp[:, ky:ky + stride * Ho:stride, kx:kx + stride * Wo:stride, :]
    return cols


def col2im(dcols, x_shape, k, stride, pad):
    """Adjoint of im2col: scatter-add dcols [n,Ho,Wo,k,k,C] into dx [n,H,W,C]."""
    n, H, W, C = x_shape
    Ho, Wo = dcols.shape[1], dcols.shape[2]
    dxp = np.zeros((n, H + 2 * pad, W + 2 * pad, C), dtype=dcols.dtype)
    for ky in range(k):
        for kx in range(k):
            dxp[:, ky:ky + stride * Ho:stride, kx:kx + stride * Wo:stride, :] += dcols[:, :, :, ky, kx, :]
    return dxp[:, pad:pad + H, pad:pad + W, :]


def conv_fwd(x, Wt, b, stride, pad):
    co, k = Wt.shape[0], Wt.shape[1]
    cols = im2col(x, k, stride, pad)
    n, Ho, Wo = cols.shape[:3]
    z = cols.reshape(n * Ho * Wo, -1) @ Wt.reshape(co, -1).T + b
    return z.reshape(n, Ho, Wo, co), cols


def conv_bwd(dz, x_shape, cols, Wt, stride, pad, need_dx):
    co, k = Wt.shape[0], Wt.shape[1]
    dzm = dz.reshape(-1, co)
    dW = (dzm.T @ cols.reshape(dzm.shape[0], -1)).reshape(Wt.shape)
    db = dzm.sum(axis=0)
    dx = None
    if need_dx:
        dcols = (dzm @ Wt.reshape(co, -1)).reshape(cols.shape)
        dx = col2im(dcols, x_shape, k, stride, pad)
    return dW, db, dx


def relu(z):
    return np.maximum(z, 0.0)


def pool2_fwd(r):
    """2x2/2 max pool of r [n,H,W,C]; returns (pooled, argmax q in 0..3).
    Window order q = 2*dy + dx (row-major); the first maximum wins (strict >)."""
    n, H, W, C = r.shape
    win = [r[:, dy::2, dx::2, :] for dy in (0, 1) for dx in (0, 1)]
    best = win[0].copy()
    arg = np.zeros(best.shape, dtype=np.int64)
    for q in (1, 2, 3):
        upd = win[q] > best
        best = np.where(upd, win[q], best)
        arg = np.where(upd, q, arg)
    return best, arg


def pool2_bwd(dp, arg, shape):
    dr = np.zeros(shape, dtype=dp.dtype)
    for q in range(4):
        dy, dx = divmod(q, 2)
        dr[:, dy::2, dx::2, :] = np.where(arg == q, dp, 0.0)
    return dr


# ---------------------------------------------------------------------------
# forced decisions (teacher-forced parity; tests/teacher_forced.py)
# ---------------------------------------------------------------------------
# A ReLU mask or a 2x2 max-pool argmax is a discrete decision taken from floating-point values.  Where
# the candidates lie within rounding of each other both choices are correct results of the method, and
# the one the GPU took depends on its summation order ("Full-size parity").  With
# `decisions` the oracle takes the GPU's choice, but only after checking that it is VALID: the forced
# choice must be within `tol` x (the layer's max |value|) of the oracle's own.  Anything else raises.
class ForcedDecisionError(AssertionError):
    pass


def _tol_check(name, bad, slack, scale, tol):
    if np.any(bad & (slack > tol * scale)):
        worst = float(np.max(np.where(bad, slack, 0.0)) / scale)
        raise ForcedDecisionError(f"{name}: GPU decision off by {worst:.3e} of the layer scale (tol {tol:.1e})")


def forced_relu_mask(name, z, gpu_pos, tol, rep):
    """mask = gpu_pos (the GPU's stored activation > 0), valid where it differs from z > 0 only if |z| is
    within tol of zero."""
    own = z > 0
    diff = own != gpu_pos
    _tol_check(name, diff, np.abs(z), max(float(np.max(np.abs(z))), 1e-300), tol)
    rep[name] = rep.get(name, 0) + int(diff.sum())
    return gpu_pos


def forced_pool(name, z, gpu_arg, gpu_pos, tol, rep):
    """2x2/2 max pool of relu(z) with the GPU's argmax where its pooled value is positive: the forced
    element must be within tol of the window max, and the ReLU decision of the pooled value (the GPU's
    pooled value > 0) within tol of zero.  Returns (pooled value, argmax, mask = pooled > 0)."""
    best, arg = pool2_fwd(relu(z))
    win = np.stack([z[:, dy::2, dx::2, :] for dy in (0, 1) for dx in (0, 1)])  # pre-activation windows
    ga = np.where(gpu_pos, gpu_arg, arg)
    pre = np.take_along_axis(win, ga[None], axis=0)[0]
    diff = ga != arg
    _tol_check(name + ".argmax", diff, best - relu(pre), max(float(np.max(np.abs(z))), 1e-300), tol)
    rep[name + ".argmax"] = rep.get(name + ".argmax", 0) + int(diff.sum())
    # ReLU of the pooled value: the forced element's pre-activation where the GPU kept it, else the window max
    mask = forced_relu_mask(name + ".relu", np.where(gpu_pos, pre, win.max(axis=0)), gpu_pos, tol, rep)
    return np.where(mask, relu(pre), 0.0), ga, mask


def gn_fwd(z, gamma, beta, groups=GN_GROUPS, eps=GN_EPS):
    """GroupNorm (Wu & He 2018) of z [n, H, W, C]: per sample and group of C / groups channels, x^ = (z - mean)
    / sqrt(var + eps) over (H, W, channels of the group), then gamma_c x^ + beta_c.  Returns (out, cache)."""
    n, H, W, C = z.shape
    zg = z.reshape(n, H, W, groups, C // groups)
    mu = zg.mean(axis=(1, 2, 4), keepdims=True)
    var = ((zg - mu) ** 2).mean(axis=(1, 2, 4), keepdims=True)
    rstd = 1.0 / np.sqrt(var + eps)
    xh = ((zg - mu) * rstd).reshape(n, H, W, C)
    return xh * gamma + beta, (xh, rstd, groups)


def gn_bwd(dy, gamma, cache):
    """Gradients of GroupNorm: (dz, dgamma, dbeta) from dy = d(out)."""
    xh, rstd, groups = cache
    n, H, W, C = dy.shape
    dbeta = dy.sum(axis=(0, 1, 2))
    dgamma = (dy * xh).sum(axis=(0, 1, 2))
    dxh = (dy * gamma).reshape(n, H, W, groups, C // groups)
    xg = xh.reshape(n, H, W, groups, C // groups)
    dz = rstd * (dxh - dxh.mean(axis=(1, 2, 4), keepdims=True) - xg * (dxh * xg).mean(axis=(1, 2, 4), keepdims=True))
    return dz.reshape(n, H, W, C), dgamma, dbeta


def option_a(a, cout):
    """Option-A shortcut: the input subsampled at even pixels with zero channels appended (R11)."""
    sub = a[:, ::2, ::2, :]
    sc = np.zeros(sub.shape[:3] + (cout,))
    sc[..., :sub.shape[3]] = sub
    return sc


def softmax_ce(z, y):
    """Mean CE over the batch and dz = (softmax - onehot)/|beta|."""
    nb = z.shape[0]
    m = z.max(axis=1, keepdims=True)
    e = np.exp(z - m)
    s = e.sum(axis=1, keepdims=True)
    p = e / s
    loss = float(np.mean(np.log(s[:, 0]) + m[:, 0] - z[np.arange(nb), y]))
    dz = p.copy()
    dz[np.arange(nb), y] -= 1.0
    return loss, dz / nb


# ---------------------------------------------------------------------------
# per-model loss + gradient
# ---------------------------------------------------------------------------
def bf16(x):
    """Round to the nearest bfloat16 (ties to even) through float32, returned as float64.

    Used only by the bf16-EMULATION mode (reading R17):
    the CUDA bf16 path stores activations / gradient operands and the tensor-core
    weight shadow in bf16 and accumulates in fp32."""
    f = np.asarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    r = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000  # RNE on the upper 16 bits (finite, inf: exact)
    r = np.where(np.isnan(f), 0x7FC00000, r)          # NaN -> the canonical quiet NaN (IEEE: stays NaN)
    return r.astype(np.uint32).view(np.float32).astype(np.float64)


def bf16_rz(x):
    """The upper 16 bits of the float32 value (round toward zero to bfloat16), as float64.

    The CUDA bf16 mode keeps the CNN's fc1 weights as the fp32 master split into two 16-bit planes and
    feeds the tensor cores the high plane (reading R17): this is that operand."""
    f = np.asarray(x, dtype=np.float32)
    u = f.view(np.uint32) & np.uint32(0xFFFF0000)
    return u.view(np.float32).astype(np.float64)


def loss_and_grad(p, model, xb, yb, emulate_bf16=False, decisions=None, tol=0.0):
    """xb float64 [nb, H, W, C] in [0,1]; returns (loss, grads dict).

    emulate_bf16: round to bf16 exactly where the CUDA bf16 mode stores bf16
    (pooled / hidden activations, dh, the pre-activation gradients dz, and the
    conv2 weights read by the tensor cores; the fc1 weights are truncated to their upper
    16 bits, bf16_rz, the operand the split-plane master gives; ResNet-8: every stored
    activation and gradient, the staged input and every conv's weights); everything else
    float64.

    decisions (teacher-forced parity only; None = the oracle's own decisions): the GPU's ReLU masks and
    pool argmaxes of this step, taken where valid within `tol` (forced_relu_mask / forced_pool); keys
    MLP "h1"; CNN "a1", "i1", "a2", "i2", "h"; ResNet-8 "a0", "r1", "o1", "r2", "o2", "r3", "o3" (the
    GPU's stored activations, > 0 = the mask; i1 / i2 its argmaxes).  The number of decisions that
    differed from the oracle's own is added to decisions["_forced"]."""
    q = bf16 if emulate_bf16 else (lambda v: v)
    dec = decisions
    rep = dec.setdefault("_forced", {}) if dec is not None else None
    g = {}
    nb = xb.shape[0]
    if model == MLP:
        x = xb.reshape(nb, -1)
        z1 = x @ p["fc1.W"].T + p["fc1.b"]
        h1 = q(relu(z1))
        m1 = h1 > 0 if dec is None else forced_relu_mask("h1", z1, dec["h1"] > 0, tol, rep)
        h1 = np.where(m1, h1, 0.0)
        z2 = h1 @ p["fc2.W"].T + p["fc2.b"]
        loss, dz2 = softmax_ce(z2, yb)
        g["fc2.W"], g["fc2.b"] = dz2.T @ h1, dz2.sum(0)
        dh1 = dz2 @ p["fc2.W"]
        dz1 = dh1 * m1
        g["fc1.b"] = dz1.sum(0)
        g["fc1.W"] = q(dz1).T @ x
        return loss, g
    if model in (CNN, CNN28):
        if model == CNN:  # tcgen05 path: bf16 weight / input operands
            W2q = q(p["conv2.W"])
            W3q = bf16_rz(p["fc1.W"]) if emulate_bf16 else p["fc1.W"]  # fc1: the hi plane of the fp32 master
            W1q, xq = q(p["conv1.W"]), q(xb)
        else:  # CNN28 runs the SIMT kernels on bf16 storage: fp32 weights and input, bf16 stored tensors
            W1q, W2q, W3q, xq = p["conv1.W"], p["conv2.W"], p["fc1.W"], xb
        z1, cols1 = conv_fwd(xq, W1q, p["conv1.b"], 1, 2)
        if dec is None:
            a1, arg1 = pool2_fwd(relu(z1))
            m1 = a1 > 0
        else:
            a1, arg1, m1 = forced_pool("pool1", z1, dec["i1"], dec["a1"] > 0, tol, rep)
        a1 = q(a1)
        z2, cols2 = conv_fwd(a1, W2q, p["conv2.b"], 1, 2)
        if dec is None:
            a2, arg2 = pool2_fwd(relu(z2))
            m2 = a2 > 0
        else:
            a2, arg2, m2 = forced_pool("pool2", z2, dec["i2"], dec["a2"] > 0, tol, rep)
        a2 = q(a2)
        f = a2.reshape(nb, -1)
        z3 = f @ W3q.T + p["fc1.b"]
        h = q(relu(z3))
        m3 = h > 0 if dec is None else forced_relu_mask("h", z3, dec["h"] > 0, tol, rep)
        h = np.where(m3, h, 0.0)
        z4 = h @ p["fc2.W"].T + p["fc2.b"]
        loss, dz4 = softmax_ce(z4, yb)
        g["fc2.W"], g["fc2.b"] = dz4.T @ h, dz4.sum(0)
        dz3 = (dz4 @ p["fc2.W"]) * m3
        g["fc1.b"] = dz3.sum(0)
        dz3 = q(dz3)
        g["fc1.W"] = dz3.T @ f
        da2 = (dz3 @ W3q).reshape(a2.shape)
        dz2 = q(pool2_bwd(da2 * m2, arg2, z2.shape))
        g["conv2.W"], g["conv2.b"], da1 = conv_bwd(dz2, a1.shape, cols2, W2q, 1, 2, True)
        dz1 = q(pool2_bwd(da1 * m1, arg1, z1.shape))
        g["conv1.W"], g["conv1.b"], _ = conv_bwd(dz1, xb.shape, cols1, W1q, 1, 2, False)
        return loss, g
    if model == RESNET18:
        # R26: conv (bias) -> GroupNorm -> ReLU; basic blocks out = ReLU(GN(conv(ReLU(GN(conv(a))))) + sc(a)),
        # sc = identity or option A; GAP over the 4x4 map; FC.  The SIMT path (both modes) stores every conv
        # output z, every activation and every gradient tensor in the mode's storage type (emulate_bf16:
        # rounded there), weights and GroupNorm statistics in fp32.
        def rmask(name, v):
            return v > 0 if dec is None else forced_relu_mask(name, v, dec[name] > 0, tol, rep)

        z0, cols0 = conv_fwd(xb, p["conv0.W"], p["conv0.b"], 1, 1)
        z0 = q(z0)
        y0, gc0 = gn_fwd(z0, p["gn0.W"], p["gn0.b"])
        m0 = rmask("a0", y0)
        a = q(np.where(m0, y0, 0.0))
        caches = []
        for bi, (name, cin, cout, stride) in enumerate(resnet18_blocks()):
            za, colsa = conv_fwd(a, p[name + "a.W"], p[name + "a.b"], stride, 1)
            za = q(za)
            ya, gca = gn_fwd(za, p[name + "ga.W"], p[name + "ga.b"])
            ma = rmask(f"r{bi}", ya)
            ra = q(np.where(ma, ya, 0.0))
            zb, colsb = conv_fwd(ra, p[name + "b.W"], p[name + "b.b"], 1, 1)
            zb = q(zb)
            nb_, gcb = gn_fwd(zb, p[name + "gb.W"], p[name + "gb.b"])
            sc = a if (stride == 1 and cin == cout) else option_a(a, cout)
            s = nb_ + sc
            ms = rmask(f"o{bi}", s)
            out = q(np.where(ms, s, 0.0))
            caches.append((name, cin, cout, stride, a, colsa, gca, ma, ra, colsb, gcb, ms))
            a = out
        gap = a.mean(axis=(1, 2))
        z = gap @ p["fc.W"].T + p["fc.b"]
        loss, dz = softmax_ce(z, yb)
        g["fc.W"], g["fc.b"] = dz.T @ gap, dz.sum(0)
        dgap = dz @ p["fc.W"]
        HW = a.shape[1] * a.shape[2]
        dout = q(np.broadcast_to(dgap[:, None, None, :] / HW, a.shape).copy())
        for name, cin, cout, stride, a_in, colsa, gca, ma, ra, colsb, gcb, ms in reversed(caches):
            gs = q(dout * ms)  # gradient of the block output's pre-ReLU sum: GN-b's output and the shortcut
            dzb, g[name + "gb.W"], g[name + "gb.b"] = gn_bwd(gs, p[name + "gb.W"], gcb)
            dzb = q(dzb)
            g[name + "b.W"], g[name + "b.b"], dra = conv_bwd(dzb, ra.shape, colsb, p[name + "b.W"], 1, 1, True)
            dra = q(dra)
            dza, g[name + "ga.W"], g[name + "ga.b"] = gn_bwd(dra * ma, p[name + "ga.W"], gca)
            dza = q(dza)
            g[name + "a.W"], g[name + "a.b"], da_in = conv_bwd(dza, a_in.shape, colsa, p[name + "a.W"], stride, 1, True)
            if stride == 1 and cin == cout:
                da_in = da_in + gs
            else:
                da_in[:, ::2, ::2, :] += gs[..., :cin]
            dout = q(da_in)
        dz0, g["gn0.W"], g["gn0.b"] = gn_bwd(dout * m0, p["gn0.W"], gc0)
        dz0 = q(dz0)
        g["conv0.W"], g["conv0.b"], _ = conv_bwd(dz0, xb.shape, cols0, p["conv0.W"], 1, 1, False)
        return loss, g
    if model == RESNET8:
        # emulate_bf16: the staged input, the stored activations (a0, each block's ra and output), the
        # stored gradients (each block's ds and dza, dz0) and every conv's weights (tensor-core shadow)
        def rmask(name, z):  # the ReLU decision of a stored activation (own, or the GPU's where valid)
            return z > 0 if dec is None else forced_relu_mask(name, z, dec[name] > 0, tol, rep)

        z0, cols0 = conv_fwd(q(xb), q(p["conv0.W"]), p["conv0.b"], 1, 1)
        m0 = rmask("a0", z0)
        a0 = q(np.where(m0, relu(z0), 0.0))
        caches = []
        a = a0
        for bi, (blk, stride) in enumerate((("b1", 1), ("b2", 2), ("b3", 2))):
            Wa, Wb = q(p[blk + "a.W"]), q(p[blk + "b.W"])
            za, colsa = conv_fwd(a, Wa, p[blk + "a.b"], stride, 1)
            ma = rmask(f"r{bi + 1}", za)
            ra = q(np.where(ma, relu(za), 0.0))
            zb, colsb = conv_fwd(ra, Wb, p[blk + "b.b"], 1, 1)
            cout = zb.shape[3]
            if stride == 1 and a.shape[3] == cout:
                sc = a
            else:
                sub = a[:, ::2, ::2, :]
                sc = np.zeros(sub.shape[:3] + (cout,))
                sc[..., :sub.shape[3]] = sub
            s = zb + sc
            ms = rmask(f"o{bi + 1}", s)
            out = q(np.where(ms, relu(s), 0.0))
            caches.append((blk, stride, a, ma, colsa, ra, colsb, ms, Wa, Wb))
            a = out
        gap = a.mean(axis=(1, 2))
        z = gap @ p["fc.W"].T + p["fc.b"]
        loss, dz = softmax_ce(z, yb)
        g["fc.W"], g["fc.b"] = dz.T @ gap, dz.sum(0)
        dgap = dz @ p["fc.W"]
        HW = a.shape[1] * a.shape[2]
        dout = np.broadcast_to(dgap[:, None, None, :] / HW, a.shape).copy()
        for blk, stride, a_in, ma, colsa, ra, colsb, ms, Wa, Wb in reversed(caches):
            ds = q(dout * ms)
            g[blk + "b.W"], g[blk + "b.b"], dra = conv_bwd(ds, ra.shape, colsb, Wb, 1, 1, True)
            dza = q(dra * ma)
            g[blk + "a.W"], g[blk + "a.b"], da_in = conv_bwd(dza, a_in.shape, colsa, Wa, stride, 1, True)
            if stride == 1 and a_in.shape[3] == ds.shape[3]:
                da_in = da_in + ds
            else:
                da_in[:, ::2, ::2, :] += ds[..., :a_in.shape[3]]
            dout = da_in
        dz0 = q(dout * m0)
        g["conv0.W"], g["conv0.b"], _ = conv_bwd(dz0, xb.shape, cols0, p["conv0.W"], 1, 1, False)
        return loss, g
    raise ValueError(model)


def flat_loss_and_grad(w, model, width_q, classes, xb, yb, emulate_bf16=False, decisions=None, tol=0.0):
    p = unpack(np.asarray(w, dtype=np.float64), model, width_q, classes)
    loss, g = loss_and_grad(p, model, xb, yb, emulate_bf16, decisions, tol)
    return loss, pack(g, model, width_q, classes)


# ---------------------------------------------------------------------------
# local SGD
# ---------------------------------------------------------------------------
def steps(n, batch, epochs):
    return epochs * math.ceil(n / batch)


def local_sgd(w0, model, width_q, classes, x_u8, y, batch, epochs, lr, seed, rnd, client_id,
              shuffle=True, max_steps=None, emulate_bf16=False):
    """Run one client's local SGD; returns (w_k float64, losses list)."""
    w = np.array(w0, dtype=np.float64)
    n = x_u8.shape[0]
    H, W, C = input_shape(model)
    xf = x_u8.reshape(n, H, W, C).astype(np.float64) / 255.0
    nbat = math.ceil(n / batch)
    losses = []
    done = 0
    for e in range(epochs):
        perm = epoch_perm(n, seed, rnd, client_id, e) if shuffle else list(range(n))
        for j in range(nbat):
            if max_steps is not None and done >= max_steps:
                return w, losses
            idx = perm[j * batch:min((j + 1) * batch, n)]
            loss, gflat = flat_loss_and_grad(w, model, width_q, classes, xf[idx], y[idx], emulate_bf16)
            w = w - lr * gflat
            losses.append(loss)
            done += 1
    return w, losses
