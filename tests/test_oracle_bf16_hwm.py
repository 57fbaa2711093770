"""Pins of the two oracle parts VERDICT r1 found unpinned (CPU only).

1. ``oracle.sgd.bf16`` (the bf16-emulation rounding, reading R17:
   "conversions RNE") against torch's float32 -> bfloat16 conversion, bit for
   bit, on >= 10^6 values covering ties, subnormals, the overflow edge, inf
   and NaN; and ``emulate_bf16`` with the rounding replaced by the identity is
   bit-identical to the float64 path (so the emulation changes nothing but
   the rounding points).
2. ``oracle.profiler.slot_layout`` / ``hwm_bytes`` against hand-derived
   per-buffer sizes (tests/golden/hwm.json, written from DESIGN.md §5), and
   the SURVEY §8(c).3 examples reconciled line by line."""
import json
import os

import numpy as np
import pytest

from oracle import profiler as pf
from oracle import sgd

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "hwm.json")))


def _torch_bf16_bits(f32):
    import torch
    t = torch.from_numpy(np.ascontiguousarray(f32, dtype=np.float32)).to(torch.bfloat16)
    return t.view(torch.int16).numpy().view(np.uint16)


def _oracle_bf16_bits(f32):
    r = sgd.bf16(f32).astype(np.float32)
    return (r.view(np.uint32) >> 16).astype(np.uint16)


def test_bf16_rne_matches_torch_bitwise():
    rng = np.random.default_rng(0)
    # 1) uniformly random bit patterns: every exponent incl. subnormals (exp 0), inf / NaN (exp 255)
    u = rng.integers(0, 2**32, size=1_000_000, dtype=np.uint64).astype(np.uint32)
    # 2) exact ties (low half 0x8000) with even and odd kept bit, and the neighbours of a tie
    hi = rng.integers(0, 2**16, size=50_000, dtype=np.uint64).astype(np.uint32) << 16
    ties = np.concatenate([hi | 0x8000, hi | 0x7FFF, hi | 0x8001, hi, hi | 0xFFFF])
    # 3) hand-picked edges: +-0, the smallest subnormals, bf16 max and the overflow boundary, inf, NaNs
    edges = np.array([0x00000000, 0x80000000, 0x00000001, 0x00008000, 0x00018000, 0x007FFFFF, 0x00800000,
                      0x7F7F0000, 0x7F7F7FFF, 0x7F7F8000, 0x7F7FFFFF, 0xFF7F8000, 0x7F800000, 0xFF800000,
                      0x7FC00000, 0x7F800001, 0xFFFFFFFF, 0x7FFFFFFF, 0x3F808000, 0x3F818000], dtype=np.uint32)
    bits = np.concatenate([u, ties, edges])
    f = bits.view(np.float32)
    got, ref = _oracle_bf16_bits(f), _torch_bf16_bits(f)
    nan = np.isnan(f)
    assert np.array_equal(got[~nan], ref[~nan])
    # NaN stays NaN (exponent all ones, mantissa non-zero)
    assert np.all((got[nan] & 0x7F80) == 0x7F80) and np.all((got[nan] & 0x007F) != 0)
    assert nan.sum() > 1000 and (np.abs(f) < np.float32(1.18e-38)).sum() > 1000  # both classes exercised
    # closed forms: 1 + 2^-8 is a tie between 1 and 1 + 2^-7 -> even (1); 1 + 3*2^-8 -> 1 + 2^-6
    assert sgd.bf16(np.float32(1 + 2**-8)) == 1.0
    assert sgd.bf16(np.float32(1 + 3 * 2**-8)) == 1 + 2**-6


def test_bf16_rz_is_the_upper_half():
    """bf16_rz (the fc1 split-plane operand) = the float32's upper 16 bits: torch's int32 view masked,
    the value's magnitude never grows, and (hi << 16 | lo) rebuilds every float32 exactly."""
    import torch
    rng = np.random.default_rng(3)
    bits = rng.integers(0, 2**32, size=1_000_000, dtype=np.uint64).astype(np.uint32)
    f = bits.view(np.float32)
    got = sgd.bf16_rz(f).astype(np.float32).view(np.uint32)
    ref = (torch.from_numpy(bits.view(np.int32)) & torch.tensor(-65536, dtype=torch.int32)).numpy().view(np.uint32)
    fin = np.isfinite(f)
    assert np.array_equal(got[fin], ref[fin])
    assert np.all(np.abs(sgd.bf16_rz(f[fin])) <= np.abs(f[fin].astype(np.float64)))
    hi, lo = (bits >> 16).astype(np.uint32), (bits & 0xFFFF).astype(np.uint32)
    assert np.array_equal(((hi << 16) | lo), bits)


def _tiny_inputs(model, nb, seed):
    rng = np.random.default_rng(seed)
    H, W, C = sgd.input_shape(model)
    x = rng.integers(0, 256, size=(nb, H, W, C)).astype(np.float64) / 255.0
    y = rng.integers(0, 10, size=nb)
    return x, y


@pytest.mark.parametrize("model,width_q", [(sgd.MLP, 4), (sgd.CNN, 1), (sgd.CNN, 4), (sgd.RESNET8, 4)])
def test_emulate_bf16_with_identity_rounding_is_the_f64_path(monkeypatch, model, width_q):
    rng = np.random.default_rng(1)
    P = sgd.n_params(model, width_q, 10)
    w = rng.uniform(-0.1, 0.1, size=P)
    x, y = _tiny_inputs(model, 3, 2)
    l0, g0 = sgd.flat_loss_and_grad(w, model, width_q, 10, x, y, emulate_bf16=False)
    monkeypatch.setattr(sgd, "bf16", lambda v: v)
    monkeypatch.setattr(sgd, "bf16_rz", lambda v: v)
    l1, g1 = sgd.flat_loss_and_grad(w, model, width_q, 10, x, y, emulate_bf16=True)
    assert l0 == l1 and np.array_equal(g0, g1)
    monkeypatch.undo()
    # and with the real rounding the emulation does move the gradient (the rounding points are live)
    _, g2 = sgd.flat_loss_and_grad(w, model, width_q, 10, x, y, emulate_bf16=True)
    assert not np.array_equal(g0, g2)


def _ev(expr):
    return int(eval(expr, {"__builtins__": {}}, {"max": max}))


@pytest.mark.parametrize("case", GOLD["cases"], ids=[c["name"] for c in GOLD["cases"]])
def test_slot_layout_matches_hand_derived_buffers(case):
    lay = pf.slot_layout(case["model"], case["width_q"], case["classes"], case["batch"], case["n"], case["epochs"],
                         case["elem"])
    want = [(name, _ev(expr)) for name, expr in case["buffers"]]
    assert [(k, int(v)) for k, v in lay] == want
    total = sum(pf.align256(v) for _, v in want)
    assert total == case["total"]
    assert pf.hwm_bytes(case["model"], case["width_q"], case["classes"], case["batch"], case["n"], case["epochs"],
                        case["elem"]) == case["total"]


@pytest.mark.parametrize("item", GOLD["survey_reconciliation"]["items"], ids=lambda i: i["case"])
def test_survey_hwm_examples_reconciled(item):
    """The survey's printed example follows from its own generic formula, and survey - removed + added
    (per buffer, each aligned) is the built layout's total."""
    a = pf.align256
    survey = sum(a(_ev(e)) for _, e in item["survey_buffers"])
    if "survey_value" in item:
        assert survey == item["survey_value"]
    else:
        assert round(survey / 2**20, 2) == item["survey_value_mib"]
    removed = sum(a(_ev(e)) for _, e, _why in item["removed"])
    added = sum(a(_ev(e)) for _, e, _why in item["added"])
    case = next(c for c in GOLD["cases"] if c["name"] == item["case"])
    assert survey - removed + added == case["total"]
    # every removed buffer is one of the survey's, every added one is in the built layout
    assert {n for n, _, _ in item["removed"]} <= {n for n, _ in item["survey_buffers"]}
    assert {n for n, _, _ in item["added"]} <= {n for n, _ in case["buffers"]}


def test_resnet8_wgrad_split_rule():
    """oracle.profiler.resnet8_wgrad_splits: every split holds whole images and at most 2048
    output pixels; 32x32 layers use 2-image splits; 16x16 / 8x8 layers use at least min(4, ceil(b / 2))
    splits; the count never decreases with b (so the footprint stays monotone in the batch, reading R13);
    and b = 64 gives the hand-derived split counts of tests/golden/hwm.json (32 / 8 / 4)."""
    import math
    for hw in (1024, 256, 64):
        prev = 0
        for b in range(1, 65):
            s = pf.resnet8_wgrad_splits(hw, b)
            assert s >= prev
            prev = s
            ips = math.ceil(b / s)  # images in the largest split of a balanced partition
            assert ips * hw <= pf.WGRAD_CHUNK_PX, (hw, b, s)
            assert s <= b
            if hw == 1024:
                assert s == math.ceil(b / 2)
            else:
                assert s >= min(4, math.ceil(b / 2))
    assert [pf.resnet8_wgrad_splits(hw, 64) for hw in (1024, 256, 64)] == [32, 8, 4]
