"""CPU tests of the C-ABI library (no GPU): symbols, the host planner and the
footprint formulas, each compared with the independent oracle."""
import json
import os
import random
import re

import numpy as np
import pytest

import paper_2207_01053_b200 as pb
from oracle import planner as pl
from oracle import profiler as pf
from oracle import sgd

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    import glob
    hdr = "".join(open(f).read() for f in glob.glob(os.path.join(ROOT, "include", "*.h")))
    declared = set(re.findall(r"\b(protea_[a-z_0-9]+)\s*\(", hdr))
    assert declared == set(pb.EXPORTS)
    for name in declared:
        assert hasattr(pb._lib, name), name


def _profiles(rows):
    a = np.zeros(len(rows), dtype=pb.PROFILE_DT)
    for i, (cid, peak, steps, flops) in enumerate(rows):
        a[i]["client_id"], a[i]["peak_bytes"], a[i]["steps"], a[i]["flops"] = cid, peak, steps, flops
    return a


def _as_tuples(assign):
    return [(int(a["client_id"]), int(a["gpu"]), int(a["offset"]), int(a["slot"]), int(a["admit"]),
             int(a["release"]), int(a["q1024"])) for a in assign]


def _oracle_tuples(assign):
    return [(a["id"], a["gpu"], a["offset"], a["slot"], a["admit"], a["release"], a["q1024"]) for a in assign]


def test_plan_bit_exact_golden():
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "planner_golden.json")))
    u = g["unit_bytes"]
    for case, orders in ((g["lpt_case"], (("asc_id", 0), ("desc_steps", 1))), (g["spec_fifo_case"], (("asc_id", 0),))):
        rows = [(c[0], c[1] * u, c[2], c[3]) for c in case["clients"]]
        caps = [c * u for c in case["caps_units"]]
        for key, order in orders:
            a, mk = pb.protea_plan(_profiles(rows), caps, order=order)
            for t in _as_tuples(a):
                e = case[key][str(t[0])]
                assert (t[1], t[2] // u, t[3] // u, t[4], t[5]) == tuple(e)
            assert list(mk) == case["makespans"]


def test_plan_bit_exact_vs_oracle_random():
    rng = random.Random(2024)
    for trial in range(1500):
        G = rng.randint(1, 8)
        caps = [rng.randint(1, 64) * 256 * rng.choice([1, 3, 1000]) for _ in range(G)]
        n = rng.randint(1, 40)
        ids = rng.sample(range(10 ** 7), n)
        rows = [(ids[i], rng.randint(1, min(caps)), rng.randint(1, 20), rng.choice([1, 5, rng.randint(1, 10 ** 9)]))
                for i in range(n)]
        policy = rng.choice([0, 0, 1])
        order = rng.choice([0, 1])
        margin = rng.choice([1000, 1100, 1337])
        ma = rng.choice([0, 0, 1, 4])
        try:
            ref = pl.plan([dict(id=r[0], peak_bytes=r[1], steps=r[2], flops=r[3]) for r in rows], caps,
                          policy=policy, order=order, margin_permille=margin, max_active=ma)
        except pl.PlanError as e:
            with pytest.raises(pb.ProteaError) as ee:
                pb.protea_plan(_profiles(rows), caps, policy, order, margin, ma)
            assert ee.value.name == e.code
            continue
        a, mk = pb.protea_plan(_profiles(rows), caps, policy, order, margin, ma)
        assert _as_tuples(a) == _oracle_tuples(ref[0])
        assert list(mk) == ref[1]


def test_plan_errors():
    with pytest.raises(pb.ProteaError) as e:
        pb.protea_plan(_profiles([(1, 10, 1, 1), (1, 10, 1, 1)]), [4096])
    assert e.value.name == "INVALID"
    with pytest.raises(pb.ProteaError) as e:
        pb.protea_plan(_profiles([(1, 5000, 1, 1)]), [4096])
    assert e.value.name == "NO_CAPACITY"
    with pytest.raises(pb.ProteaError) as e:
        pb.protea_plan(_profiles([(1, 100, 1, 1)]), [4096], margin_permille=999)
    assert e.value.name == "INVALID"


def test_plan_float_trap_scenario_a():
    MiB = 1 << 20
    rows = [(i, 2600 * MiB, 10, 1) for i in range(100)]
    a, mk = pb.protea_plan(_profiles(rows), [11264 * MiB], margin_permille=1100)
    assert int(a[0]["slot"]) == 2860 * MiB and list(mk) == [340]
    assert int(a[0]["q1024"]) == -(-1024 * 2860 // 11264)
    _, mk = pb.protea_plan(_profiles(rows), [11264 * MiB], policy=pb.POLICY_STATIC)
    assert list(mk) == [1000]


MODELS = [(pb.MODEL_MLP, 4, 28, 28, 1), (pb.MODEL_CNN, 1, 32, 32, 3), (pb.MODEL_CNN, 2, 32, 32, 3),
          (pb.MODEL_CNN, 4, 32, 32, 3), (pb.MODEL_RESNET8, 4, 32, 32, 3), (pb.MODEL_CNN, 4, 28, 28, 1),
          (pb.MODEL_CNN, 1, 28, 28, 1), (3, 4, 32, 32, 3)]  # 3 = PROTEA_MODEL_RESNET18


@pytest.mark.parametrize("arch,wq,H,W,C", MODELS)
def test_footprint_matches_oracle(arch, wq, H, W, C):
    rng = random.Random(arch * 10 + wq)
    for _ in range(60):
        n, e = rng.randint(1, 2500), rng.randint(1, 3)
        b = rng.randint(1, 64) if rng.random() < 0.6 else rng.choice([65, 100, 128, 500, 1024, 2048])
        for prec, eb in ((pb.PREC_FP32, 4), (pb.PREC_BF16, 2)):
            om = sgd.CNN28 if (arch, H) == (pb.MODEL_CNN, 28) else sgd.RESNET18 if arch == 3 else arch
            peak, steps, flops = pb.protea_client_footprint(arch, wq, 10, H, W, C, n, b, e, prec)
            assert peak == pf.hwm_bytes(om, wq, 10, b, n, e, eb)
            assert steps == pf.local_steps(n, b, e)
            assert flops == pf.client_flops(n, e, om, wq)


def test_footprint_rejects_bad_models():
    with pytest.raises(pb.ProteaError):
        pb.protea_client_footprint(pb.MODEL_CNN, 3, 10, 32, 32, 3, 10, 8, 1)
    with pytest.raises(pb.ProteaError):
        pb.protea_client_footprint(pb.MODEL_MLP, 4, 10, 32, 32, 3, 10, 8, 1)
    with pytest.raises(pb.ProteaError):
        pb.protea_client_footprint(pb.MODEL_CNN, 4, 10, 32, 32, 3, 0, 8, 1)
