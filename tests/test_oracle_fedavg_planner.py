"""Pins for oracle/fedavg.py, oracle/planner.py, oracle/profiler.py, oracle/splitmix.py.

Each check ties the oracle to something other than itself: SPEC/paper worked
examples (tests/golden/*.json, cited there), exact rational brute force,
closed forms and invariants.
"""
import itertools
import json
import math
import os
import random
from fractions import Fraction

import numpy as np
import pytest

from oracle import fedavg as fa
from oracle import planner as pl
from oracle import profiler as pf
from oracle import sgd
from oracle import splitmix as sm

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# --------------------------------------------------------------------------- splitmix
def test_splitmix64_published_vector():
    # Published SplitMix64 output for seed 0 (Vigna's reference implementation).
    assert sm.splitmix64_stream(0, 3) == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_epoch_perm_is_permutation_and_deterministic():
    for n in (1, 2, 7, 50, 333):
        p = sm.epoch_perm(n, 3, 1, 17, 0)
        assert sorted(p) == list(range(n))
        assert p == sm.epoch_perm(n, 3, 1, 17, 0)
    assert sm.epoch_perm(50, 3, 1, 17, 0) != sm.epoch_perm(50, 3, 1, 17, 1)
    assert sm.epoch_perm(50, 3, 1, 17, 0) != sm.epoch_perm(50, 3, 1, 18, 0)


# --------------------------------------------------------------------------- fedavg
def test_fedavg_spec_examples():
    for ex in load("spec_examples.json")["fedavg"]:
        out = fa.fedavg([np.array(p) for p in ex["params"]], ex["n"])
        assert np.array_equal(out, np.array(ex["expect"]))


def test_fedavg_errors():
    with pytest.raises(fa.FedAvgError) as e:
        fa.fedavg([], [])
    assert e.value.code == "EMPTY"
    with pytest.raises(fa.FedAvgError) as e:
        fa.fedavg([np.ones(2), np.ones(3)], [1, 1])
    assert e.value.code == "DIM"
    with pytest.raises(fa.FedAvgError) as e:
        fa.fedavg([np.ones(2)], [0])
    assert e.value.code == "INVALID"


def test_fedavg_bruteforce_exact_rational():
    # agreement with a brute-force weighted mean within 1e-12
    # on 200 random instances; here the brute force is exact rational arithmetic.
    rng = random.Random(7)
    for _ in range(200):
        K, D = rng.randint(1, 10), rng.randint(1, 32)
        ws = [[rng.uniform(-10, 10) for _ in range(D)] for _ in range(K)]
        ns = [rng.randint(1, 1000) for _ in range(K)]
        out = fa.fedavg([np.array(w) for w in ws], ns)
        N = sum(ns)
        for d in range(D):
            exact = sum(Fraction(ws[k][d]) * ns[k] for k in range(K)) / N
            assert abs(out[d] - float(exact)) <= 1e-12 * max(1.0, abs(float(exact)))


def test_fedavg_invariances():
    rng = np.random.default_rng(1)
    ws = [rng.normal(size=9) for _ in range(5)]
    ns = [3, 1, 4, 1, 5]
    base = fa.fedavg(ws, ns)
    perm = [4, 2, 0, 3, 1]
    assert np.allclose(fa.fedavg([ws[i] for i in perm], [ns[i] for i in perm]), base, rtol=1e-14, atol=1e-15)
    assert np.allclose(fa.fedavg(ws, [7 * n for n in ns]), base, rtol=1e-14, atol=1e-15)
    same = rng.normal(size=9)
    assert np.allclose(fa.fedavg([same] * 4, [1, 2, 3, 4]), same, rtol=1e-15)
    v = [rng.normal(size=9) for _ in range(5)]
    lhs = fa.fedavg([2.0 * a + 3.0 * b for a, b in zip(ws, v)], ns)
    assert np.allclose(lhs, 2.0 * base + 3.0 * fa.fedavg(v, ns), rtol=1e-13, atol=1e-13)


# --------------------------------------------------------------------------- profiler
def test_param_counts_match_baseline():
    # SURVEY §8(a) / BASELINE.json configs: P = 50,890 / 2,156,490 / 541,162 / 136,314 / 75,050
    assert sgd.n_params(sgd.MLP) == 50890
    assert sgd.n_params(sgd.CNN, 4) == 2156490
    assert sgd.n_params(sgd.CNN, 2) == 541162
    assert sgd.n_params(sgd.CNN, 1) == 136314
    assert sgd.n_params(sgd.RESNET8) == 75050


def test_flops_per_sample_constants():
    # SURVEY §8(c).3 table (independently derived there)
    assert pf.flops_per_sample(sgd.MLP) == 204544
    assert pf.flops_per_sample(sgd.CNN, 4) == 101087232
    assert pf.flops_per_sample(sgd.CNN, 2) == 27737088
    assert pf.flops_per_sample(sgd.CNN, 1) == 8166912
    assert pf.flops_per_sample(sgd.RESNET8) == 72552192
    assert pf.flops_per_sample(sgd.CNN28, 4, 62) == 72544256  # "CNN-1x FEMNIST, 62 classes"


def test_flops_vs_torch_module_count():
    torch = pytest.importorskip("torch")
    nn = torch.nn

    def count(model_layers, x_shape):
        macs = []
        x = torch.zeros((1,) + x_shape)
        for lay in model_layers:
            y = lay(x)
            if isinstance(lay, nn.Conv2d):
                macs.append(y.numel() * lay.in_channels * lay.kernel_size[0] * lay.kernel_size[1])
            elif isinstance(lay, nn.Linear):
                macs.append(y.numel() * lay.in_features)
            x = y
        return macs

    for wq in (1, 2, 4):
        c1, c2, f = sgd.cnn_channels(wq)
        layers = [nn.Conv2d(3, c1, 5, padding=2), nn.ReLU(), nn.MaxPool2d(2),
                  nn.Conv2d(c1, c2, 5, padding=2), nn.ReLU(), nn.MaxPool2d(2), nn.Flatten(),
                  nn.Linear(64 * c2, f), nn.ReLU(), nn.Linear(f, 10)]
        m = count(layers, (3, 32, 32))
        expect = 2 * (2 * sum(m) + sum(m[1:]))
        assert pf.flops_per_sample(sgd.CNN, wq) == expect
        layers = [nn.Conv2d(1, c1, 5, padding=2), nn.ReLU(), nn.MaxPool2d(2),  # the FEMNIST-shaped CNN
                  nn.Conv2d(c1, c2, 5, padding=2), nn.ReLU(), nn.MaxPool2d(2), nn.Flatten(),
                  nn.Linear(49 * c2, f), nn.ReLU(), nn.Linear(f, 62)]
        m = count(layers, (1, 28, 28))
        assert pf.flops_per_sample(sgd.CNN28, wq, 62) == 2 * (2 * sum(m) + sum(m[1:]))
        assert sgd.n_params(sgd.CNN28, wq, 62) == sum(p.numel() for p in nn.Sequential(*layers).parameters())


def test_local_steps_closed_form():
    assert pf.local_steps(500, 8, 2) == 126
    assert pf.local_steps(500, 64, 2) == 16
    assert pf.local_steps(50, 10, 1) == 5
    assert pf.local_steps(1, 64, 2) == 2


def test_hwm_monotone():
    for model, wqs in ((sgd.MLP, (4,)), (sgd.CNN, (1, 2, 4)), (sgd.RESNET8, (4,))):
        for e in (2, 4):
            for wq in wqs:
                h = [pf.hwm_bytes(model, wq, 10, b, 500, 2, e) for b in (8, 16, 32, 64)]
                assert all(a < b for a, b in zip(h, h[1:]))
                hb = [pf.hwm_bytes(model, wq, 10, b, 500, 2, e) for b in range(1, 80)]
                assert all(a <= b for a, b in zip(hb, hb[1:]))
        if model == sgd.CNN:
            for b in (8, 64):
                hw = [pf.hwm_bytes(model, wq, 10, b, 500, 2, 2) for wq in (1, 2, 4)]
                assert hw[0] < hw[1] < hw[2]
    # every buffer aligned to 256 B
    assert pf.hwm_bytes(sgd.CNN, 4, 10, 8, 500, 2, 4) % 256 == 0


def test_eq1_examples():
    g = load("spec_examples.json")
    for ex in g["eq1"]:
        assert pf.eq1_q1024(ex["vram"], ex["total"]) == ex["q1024"]


# --------------------------------------------------------------------------- planner
def _clients(rows, unit):
    return [dict(id=i, peak_bytes=s * unit, steps=st, flops=w) for i, s, st, w in rows]


def _check(assign, exp, unit):
    for a in assign:
        e = exp[str(a["id"])]
        assert (a["gpu"], a["offset"] // unit, a["slot"] // unit, a["admit"], a["release"]) == tuple(e)


def test_planner_golden_lpt():
    g = load("planner_golden.json")
    u = g["unit_bytes"]
    case = g["lpt_case"]
    caps = [c * u for c in case["caps_units"]]
    for order, key in ((pl.ASC_ID, "asc_id"), (pl.DESC_STEPS, "desc_steps")):
        assign, mk = pl.plan(_clients(case["clients"], u), caps, order=order)
        _check(assign, case[key], u)
        assert mk == case["makespans"]


def test_planner_spec_fifo():
    g = load("planner_golden.json")
    u = g["unit_bytes"]
    case = g["spec_fifo_case"]
    assign, mk = pl.plan(_clients(case["clients"], u), [c * u for c in case["caps_units"]])
    _check(assign, case["asc_id"], u)
    assert mk == case["makespans"]


def test_planner_scenario_a_and_float_trap():
    s = load("spec_examples.json")["scenario_a"]
    MiB = 1 << 20
    cl = [dict(id=i, peak_bytes=s["hwm_mib"] * MiB, steps=s["steps"], flops=1) for i in range(s["n"])]
    caps = [s["cap_mib"] * MiB]
    a, mk = pl.plan(cl, caps, margin_permille=s["margin_permille"])
    assert a[0]["slot"] == s["slot_mib"] * MiB
    assert mk == [s["profiled_makespan"]]
    _, mk = pl.plan(cl, caps, policy=pl.STATIC)
    assert mk == [s["static_makespan"]]
    # the float trap of SURVEY finding 5: ceil(2600 * 1.10) is 2861 in IEEE double
    assert math.ceil(2600 * 1.10) == 2861
    assert -(-2600 * 1100 // 1000) == 2860


def test_planner_homogeneous_closed_form():
    rng = random.Random(3)
    for _ in range(200):
        n, C, slot, S = rng.randint(1, 40), rng.randint(1, 50), rng.randint(1, 20), rng.randint(1, 9)
        if slot > C:
            continue
        ma = rng.choice([0, 1, 2, 5])
        cl = [dict(id=i, peak_bytes=slot * 256, steps=S, flops=5) for i in range(n)]
        _, mk = pl.plan(cl, [C * 256], max_active=ma)
        k = C // slot if ma == 0 else min(C // slot, ma)
        assert mk == [math.ceil(n / k) * S]


def _invariants(clients, caps, assign, mk, order, max_active, policy=pl.PROFILED):
    by = {a["id"]: a for a in assign}
    # I1 every client exactly once
    assert sorted(by) == sorted(c["id"] for c in clients) and len(assign) == len(clients)
    steps = {c["id"]: c["steps"] for c in clients}
    for g, C in enumerate(caps):
        mine = [a for a in assign if a["gpu"] == g]
        for a in mine:
            # I4 release - admit = S
            assert a["release"] - a["admit"] == steps[a["id"]]
            assert 0 <= a["offset"] and a["offset"] + a["slot"] <= C
        # I2 live slots disjoint at every step
        T = max([a["release"] for a in mine], default=0)
        for t in range(T):
            live = sorted((a["offset"], a["offset"] + a["slot"]) for a in mine if a["admit"] <= t < a["release"])
            for (o1, e1), (o2, e2) in zip(live, live[1:]):
                assert e1 <= o2
            if max_active:
                assert len(live) <= max_active
        # I3 admit non-decreasing along queue order
        if order == pl.ASC_ID:
            q = sorted(mine, key=lambda a: a["id"])
        else:
            q = sorted(mine, key=lambda a: (-steps[a["id"]], a["id"]))
        adm = [a["admit"] for a in q]
        assert adm == sorted(adm)
        assert mk[g] == T


def test_planner_invariants_random():
    rng = random.Random(11)
    for trial in range(1000):
        G = rng.randint(1, 4)
        caps = [rng.randint(4, 40) * 256 for _ in range(G)]
        n = rng.randint(1, 25)
        clients = [dict(id=rng.randint(0, 10 ** 6) * 1000 + i, peak_bytes=rng.randint(1, min(caps) // 256) * 256 - rng.randint(0, 255),
                        steps=rng.randint(1, 12), flops=rng.randint(1, 100)) for i in range(n)]
        order = rng.choice([pl.ASC_ID, pl.DESC_STEPS])
        ma = rng.choice([0, 0, 1, 3])
        a, mk = pl.plan(clients, caps, order=order, max_active=ma)
        _invariants(clients, caps, a, mk, order, ma)
        # I7 determinism
        assert pl.plan(clients, caps, order=order, max_active=ma) == (a, mk)


def test_planner_errors():
    with pytest.raises(pl.PlanError) as e:
        pl.plan([dict(id=1, peak_bytes=10, steps=1, flops=1)] * 2, [1024])
    assert e.value.code == "INVALID"
    with pytest.raises(pl.PlanError) as e:
        pl.plan([dict(id=1, peak_bytes=2000, steps=1, flops=1)], [1024])
    assert e.value.code == "NO_CAPACITY"


def test_planner_lpt_graham_bound_bruteforce():
    # Graham (1969): LPT max load <= (4/3 - 1/(3G)) OPT; OPT by enumerating all G^n partitions.
    rng = random.Random(5)
    for _ in range(150):
        G, n = rng.randint(2, 3), rng.randint(2, 7)
        W = [rng.randint(1, 50) for _ in range(n)]
        clients = [dict(id=i, peak_bytes=256, steps=1, flops=W[i]) for i in range(n)]
        a, _ = pl.plan(clients, [256 * 64] * G)
        load = [0] * G
        for x in a:
            load[x["gpu"]] += W[x["id"]]
        opt = min(max(sum(W[i] for i in range(n) if part[i] == g) for g in range(G))
                  for part in itertools.product(range(G), repeat=n))
        assert max(load) * 3 * G <= (4 * G - 1) * opt


def test_planner_makespan_bounds_bruteforce():
    # Single GPU: makespan >= the best over all n! admission orders of the same
    # greedy first-fit list scheduler, and within [max S, sum S].
    rng = random.Random(9)
    for _ in range(60):
        n = rng.randint(1, 6)
        C = rng.randint(4, 12) * 256
        rows = [(i, rng.randint(1, C // 256), rng.randint(1, 5), 1) for i in range(n)]
        cl = _clients(rows, 256)
        _, mk = pl.plan(cl, [C])
        best = min(pl.plan([dict(c, id=j) for j, c in enumerate(p)], [C])[1][0]
                   for p in itertools.permutations(cl))
        assert best <= mk[0] <= sum(r[2] for r in rows)
        assert mk[0] >= max(r[2] for r in rows)
        area = sum(r[1] * 256 * r[2] for r in rows)
        assert mk[0] * C >= area
