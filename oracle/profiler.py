"""Per-client profile estimates (oracle; test infrastructure only).

PAPER.md Table 1 (§2.2) lists the metrics Protea's UtilMonitor
tracks; the hot path keeps VRAM (-> exact peak device bytes of the client's
arena slot) and CUDA_time (-> device-timed training time, a measurement:
"parity unpinned").  P:217 (§3.3): get_properties() reports "does this client
use a GPU? How much VRAM is the training making use of? ... How long did it
take to do the training".  Eq. (1) (§3.4):

    num_gpus = vram_measured_for_single_worker / total_vram_in_system

Definitions (DESIGN.md "Profiler" table; readings R2, R3, R21):
  S_k      = E * ceil(n_k / B_k)
  FLOPs_k  = E * n_k * f(model, w),   f = 2 * (fwd MACs + wgrad MACs + dgrad
             MACs without the first layer's dgrad), per sample
  HWM_k    = sum of align256(buffer bytes) over the slot layout below (the
             arena is a bump allocator; nothing is freed inside a round)
  q_k      = ceil(1024 * slot_k / sum_g C_g)   (Eq. (1) in units of 1/1024,
             rounded up: SPEC D-7)
"""
from __future__ import annotations

import math

from .sgd import MLP, CNN, CNN28, RESNET8, RESNET18, cnn_channels, n_params, resnet18_blocks

ALIGN = 256


def align256(x: int) -> int:
    return (x + ALIGN - 1) // ALIGN * ALIGN


def local_steps(n: int, batch: int, epochs: int) -> int:
    return epochs * math.ceil(n / batch)


def macs_per_sample(model, width_q=4, classes=10):
    """[(layer, MACs of one forward pass for one sample)] in forward order."""
    if model == MLP:
        return [("fc1", 784 * 64), ("fc2", 64 * classes)]
    if model == CNN:
        c1, c2, f = cnn_channels(width_q)
        return [("conv1", 32 * 32 * c1 * 5 * 5 * 3),
                ("conv2", 16 * 16 * c2 * 5 * 5 * c1),
                ("fc1", 64 * c2 * f),
                ("fc2", f * classes)]
    if model == CNN28:
        c1, c2, f = cnn_channels(width_q)
        return [("conv1", 28 * 28 * c1 * 5 * 5 * 1),
                ("conv2", 14 * 14 * c2 * 5 * 5 * c1),
                ("fc1", 49 * c2 * f),
                ("fc2", f * classes)]
    if model == RESNET18:  # GroupNorm layers do no multiply-accumulates
        out, hw = [("conv0", 32 * 32 * 64 * 9 * 3)], 32
        for name, cin, cout, stride in resnet18_blocks():
            hw //= stride
            out += [(name + "a", hw * hw * cout * 9 * cin), (name + "b", hw * hw * cout * 9 * cout)]
        return out + [("fc", 512 * classes)]
    if model == RESNET8:
        return [("conv0", 32 * 32 * 16 * 9 * 3),
                ("b1a", 32 * 32 * 16 * 9 * 16), ("b1b", 32 * 32 * 16 * 9 * 16),
                ("b2a", 16 * 16 * 32 * 9 * 16), ("b2b", 16 * 16 * 32 * 9 * 32),
                ("b3a", 8 * 8 * 64 * 9 * 32), ("b3b", 8 * 8 * 64 * 9 * 64),
                ("fc", 64 * classes)]
    raise ValueError(model)


def flops_per_sample(model, width_q=4, classes=10) -> int:
    layers = macs_per_sample(model, width_q, classes)
    fwd = sum(m for _, m in layers)
    wgrad = fwd
    dgrad = sum(m for _, m in layers[1:])
    return 2 * (fwd + wgrad + dgrad)


def client_flops(n, epochs, model, width_q=4, classes=10) -> int:
    return epochs * n * flops_per_sample(model, width_q, classes)


WGRAD_CHUNK_PX = 2048  # pixels reduced by one split of a conv weight-gradient GEMM


def conv_layers(model, width_q=4):
    """[(Hout*Wout, cout, k*k*cin)] of every conv layer (for the wgrad split buffer)."""
    if model == CNN:
        c1, c2, _ = cnn_channels(width_q)
        return [(1024, c1, 25 * 3), (256, c2, 25 * c1)]
    if model == CNN28:
        c1, c2, _ = cnn_channels(width_q)
        return [(784, c1, 25 * 1), (196, c2, 25 * c1)]
    if model == RESNET18:
        out, hw = [(1024, 64, 27)], 32
        for _, cin, cout, stride in resnet18_blocks():
            hw //= stride
            out += [(hw * hw, cout, 9 * cin), (hw * hw, cout, 9 * cout)]
        return out
    if model == RESNET8:
        return [(1024, 16, 27), (1024, 16, 144), (1024, 16, 144), (256, 32, 144), (256, 32, 288),
                (64, 64, 288), (64, 64, 576)]
    return []


def resnet8_wgrad_splits(hw, b):
    """Weight-gradient splits of a ResNet-8 conv with an hw-pixel output map for a slot of b rows (DESIGN.md
    §5): 2-image splits at 32x32; at 16x16 / 8x8 the larger of the 2048-pixel split count and
    min(4, ceil(b / 2)) (never fewer than ~4 splits for small batches; non-decreasing in b).  Each split
    then holds ceil(b / splits) whole images."""
    if hw == 1024:
        return math.ceil(b / 2)
    return max(math.ceil(b * hw / WGRAD_CHUNK_PX), min(4, math.ceil(b / 2)))


def slot_layout(model, width_q, classes, batch, n, epochs, elem_bytes):
    """[(buffer, bytes)] of one client's arena slot.

    elem_bytes = 4 in fp32-verify mode, 2 in bf16 mode (activation storage; in
    bf16 mode the slot also holds a bf16 shadow copy of the weights).
    b = min(batch, n): a batch holds at most that many rows,
    and per-row buffers are sized for it.
    wsp = split-K partials of the conv weight gradients: each conv layer's
    reduction over b*Hout*Wout pixels is cut into ceil(b*Hout*Wout / 2048)
    splits (ResNet-8: resnet8_wgrad_splits), each
    holding cout rows of K+1 fp32 partials (the +1 is the bias column); see the
    branches below for which layers keep partials where.
    """
    b, e = min(batch, n), elem_bytes  # a batch holds min(B, n) rows
    P = n_params(model, width_q, classes)
    out = [("params", 4 * P), ("perm", 4 * epochs * n), ("stats", 64)]
    if e == 2 and model != RESNET18:
        out.append(("wsh", 2 * P))  # bf16 shadow weights read by the tensor-core GEMMs
    if model == MLP:
        out += [("h1", b * 64 * e), ("dz1", b * 64 * e)]
    elif model in (CNN, CNN28):
        c1, c2, f = cnn_channels(width_q)
        hw = 1024 if model == CNN else 784  # conv1 map; conv2 map hw / 4; pool-2 output hw / 16
        out += [("a1", b * hw // 4 * c1 * e), ("i1", b * hw // 4 * c1),
                ("a2", b * hw // 16 * c2 * e), ("i2", b * hw // 16 * c2),
                ("h", b * f * e), ("dh", b * f * e),
                ("dz2", b * hw // 4 * c2 * e), ("dz1", b * hw * c1 * e)]
        if e == 2 and model == CNN:  # bf16 tcgen05 mode: input staged for the tensor cores + conv1 weight shadow
            # (6x6 window taps x 4 pool positions x C1 x 8 padded channels, bf16)
            out += [("xs", b * 36 * 36 * 8 * 2), ("w1q", 36 * 4 * c1 * 8 * 2)]
    elif model == RESNET18:  # per conv layer its output z and activation y, then GN stats, gradients
        convs = conv_layers(model)
        out += [(f"z{i}", b * hw * co * e) for i, (hw, co, _) in enumerate(convs)]
        out += [(f"y{i}", b * hw * co * e) for i, (hw, co, _) in enumerate(convs)]
        out += [("gnstats", b * 17 * 2 * 2 * 4), ("gx", b * 65536 * e), ("gy", b * 65536 * e),
                ("gz", b * 65536 * e), ("gnp", b * 2 * 512 * 4)]
    elif model == RESNET8:
        out += [("a0", b * 1024 * 16 * e),
                ("r1", b * 1024 * 16 * e), ("o1", b * 1024 * 16 * e),
                ("r2", b * 256 * 32 * e), ("o2", b * 256 * 32 * e),
                ("r3", b * 64 * 64 * e), ("o3", b * 64 * 64 * e),
                ("dgap", b * 64 * 4),
                ("g0", b * 1024 * 16 * e), ("g1", b * 1024 * 16 * e), ("g2", b * 1024 * 16 * e)]
        if e == 2:  # bf16 mode: conv0 weight shadow padded to 8 input channels [16][9][8] (tensor cores)
            out.append(("w0p", 16 * 9 * 8 * 2))
            out.append(("xs", b * 1024 * 8 * 2))  # conv0 input staged as [b][32][32][8] bf16
    else:
        raise ValueError(model)
    convs = conv_layers(model, width_q)
    splits = [math.ceil(b * hw / WGRAD_CHUNK_PX) for hw, _, _ in convs]
    if model == RESNET8:
        splits = [resnet8_wgrad_splits(hw, b) for hw, _, _ in convs]
    ceil4 = lambda k: -(-k // 4) * 4  # noqa: E731
    if model == RESNET18:  # one region reused layer by layer (reduced right after each wgrad), pitch K+1
        out.append(("wsp", max(4 * s * co * (K + 1) for s, (_, co, K) in zip(splits, convs))))
    elif model == RESNET8:
        # a region per layer, all seven kept until the step's single merged SGD reduce; regions placed at
        # row pitch ceil4(K+1), the last layer's rows written at pitch K+1 (its last row ends the slot)
        wsp = sum(s * co * ceil4(K + 1) for s, (_, co, K) in zip(splits[:-1], convs[:-1]))
        wsp += splits[-1] * convs[-1][1] * (convs[-1][2] + 1)
        out.append(("wsp", 4 * wsp))
    elif model == CNN and e == 2 and width_q == 4:
        # width 1, bf16: conv1's partials reuse dz2; conv2's partials (pitch ceil4(K+1)) exist only when
        # a client's rows need more than one split
        _, co, K = convs[1]
        if splits[1] > 1:
            out.append(("wsp", 4 * splits[1] * co * ceil4(K + 1)))
    elif convs:
        # one region reused layer by layer (max), rows at pitch K+1
        out.append(("wsp", max(4 * s * co * (K + 1) for s, (_, co, K) in zip(splits, convs))))
    return out


MICRO_ROWS = 64  # a batch of more rows runs as micro-clients of <= 64 rows (DESIGN.md §5 "batches > 64")


def hwm_bytes(model, width_q, classes, batch, n, epochs, elem_bytes) -> int:
    """Sum of align256(buffer) over the slot; a batch of b = min(B, n) > 64 rows holds ceil(b / 64) slots of
    min(64, rest) rows back to back plus the fp32 merge weights (4P bytes)."""
    b = min(batch, n)
    if b <= MICRO_ROWS:
        return sum(align256(sz) for _, sz in slot_layout(model, width_q, classes, batch, n, epochs, elem_bytes))
    tot = sum(hwm_bytes(model, width_q, classes, min(MICRO_ROWS, b - r0), n, epochs, elem_bytes)
              for r0 in range(0, b, MICRO_ROWS))
    return tot + align256(4 * n_params(model, width_q, classes))


def eq1_q1024(slot_bytes: int, total_capacity: int) -> int:
    """Eq. (1) as an integer count of 1/1024 GPU (rounded up, SPEC D-7)."""
    if total_capacity <= 0:
        raise ValueError("no GPU capacity")
    return -(-1024 * slot_bytes // total_capacity)
