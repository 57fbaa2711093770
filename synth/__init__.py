"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NONE of the method's arithmetic (no SGD, no FedAvg, no
profiler formula, no packing rule).  It only draws the random inputs that both
sides consume, so that a parity test can hand the *same* bytes to
`oracle/` and to the C-ABI library:

* per-client data shards (u8 images + int32 labels) shaped like FEMNIST
  (28x28x1) or CIFAR-10 (32x32x3), NHWC;
* Dirichlet(0.5)-skewed shard sizes (BASELINE.json configs[2..4]);
* initial fp32 global weights U(+-1/sqrt(fan_in)) for each model;
* the sampled client ids of a round (uniform without replacement, sorted).

The recipe is stated in DESIGN.md "Input recipe";
the parameter-segment table below is the *generator's* own copy of the model
shapes (needed to draw U(+-1/sqrt(fan_in)) per tensor) and is independent of
the oracle's and the library's layouts; a parity test fails if they diverge.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# ---------------------------------------------------------------------------
# Dataset shapes (§4.1: FEMNIST 28x28 grey, 62 classes;
# CIFAR-10 32x32 RGB, 10 classes).
# ---------------------------------------------------------------------------
FEMNIST = dict(H=28, W=28, C=1)
CIFAR = dict(H=32, W=32, C=3)

MODEL_MLP, MODEL_CNN, MODEL_RESNET8, MODEL_CNN28, MODEL_RESNET18 = 0, 1, 2, 3, 4
MODEL_NAMES = {MODEL_MLP: "mlp", MODEL_CNN: "cnn", MODEL_RESNET8: "resnet8", MODEL_CNN28: "cnn28",
               MODEL_RESNET18: "resnet18"}
# the library's arch and input shape of each harness model (MODEL_CNN28 = the CNN-w family on the
# FEMNIST-shaped 28x28x1 input of the paper's LEAF experiment; the library's arch CNN at 28x28x1)
LIB_ARCH = {MODEL_MLP: 0, MODEL_CNN: 1, MODEL_RESNET8: 2, MODEL_CNN28: 1, MODEL_RESNET18: 3}
INPUT_SHAPE = {MODEL_MLP: (28, 28, 1), MODEL_CNN: (32, 32, 3), MODEL_RESNET8: (32, 32, 3), MODEL_CNN28: (28, 28, 1),
               MODEL_RESNET18: (32, 32, 3)}


def width_channels(width_q: int) -> tuple[int, int, int]:
    """CNN-w channel counts for width w = width_q/4 (w in {1/4, 1/2, 1})."""
    return 8 * width_q, 16 * width_q, 128 * width_q


def param_segments(model: int, width_q: int = 4, classes: int = 10):
    """[(n_elements, fan_in)] per tensor in flat-parameter order (W then b per layer)."""
    segs = []

    def fc(nin, nout):
        segs.append((nout * nin, nin))
        segs.append((nout, nin))

    def conv(k, cin, cout):
        segs.append((cout * k * k * cin, k * k * cin))
        segs.append((cout, k * k * cin))

    if model == MODEL_MLP:
        fc(784, 64)
        fc(64, classes)
    elif model in (MODEL_CNN, MODEL_CNN28):
        c1, c2, f = width_channels(width_q)
        cin, pooled = (3, 64) if model == MODEL_CNN else (1, 49)
        conv(5, cin, c1)
        conv(5, c1, c2)
        fc(pooled * c2, f)
        fc(f, classes)
    elif model == MODEL_RESNET18:  # conv W, b, then GroupNorm gamma = 1, beta = 0 (fan_in 0: constants)
        def gn(c):
            segs.append((c, -1))
            segs.append((c, 0))
        conv(3, 3, 64)
        gn(64)
        cin = 64
        for s_, c in enumerate((64, 128, 256, 512)):
            for _b in range(2):
                conv(3, cin, c)
                gn(c)
                conv(3, c, c)
                gn(c)
                cin = c
        fc(512, classes)
    elif model == MODEL_RESNET8:
        conv(3, 3, 16)
        conv(3, 16, 16)
        conv(3, 16, 16)
        conv(3, 16, 32)
        conv(3, 32, 32)
        conv(3, 32, 64)
        conv(3, 64, 64)
        fc(64, classes)
    else:
        raise ValueError(model)
    return segs


def init_weights(model: int, width_q: int = 4, classes: int = 10, seed: int = 0) -> np.ndarray:
    """Initial global weights, fp32, U(+-1/sqrt(fan_in)) per tensor."""
    rng = np.random.Generator(np.random.PCG64([0x1A17, seed, model, width_q, classes]))
    out = []
    for n, fan_in in param_segments(model, width_q, classes):
        if fan_in <= 0:  # GroupNorm gamma (-1) = 1, beta (0) = 0
            out.append(np.full(n, 1.0 if fan_in < 0 else 0.0))
            continue
        bound = 1.0 / math.sqrt(fan_in)
        out.append(rng.uniform(-bound, bound, size=n))
    return np.concatenate(out).astype(np.float32)


# ---------------------------------------------------------------------------
# Shard sizes
# ---------------------------------------------------------------------------
def dirichlet_sizes(n_clients: int, total: int, alpha: float = 0.5, seed: int = 0) -> np.ndarray:
    """n_k = 1 + floor(p_k (T - N)), p ~ Dir(alpha), then largest-remainder
    top-up (ties to the lower id) so that sum(n_k) == T."""
    if total < n_clients:
        raise ValueError("total < n_clients")
    rng = np.random.Generator(np.random.PCG64([0xD1C7, seed, n_clients, total]))
    p = rng.dirichlet(np.full(n_clients, alpha))
    extra = total - n_clients
    share = p * extra
    base = np.floor(share).astype(np.int64)
    rem = share - base
    left = extra - int(base.sum())
    # largest remainder first, ties -> lower id (stable sort on -rem)
    order = np.argsort(-rem, kind="stable")
    base[order[:left]] += 1
    sizes = base + 1
    assert int(sizes.sum()) == total
    return sizes


# ---------------------------------------------------------------------------
# Data
# ---------------------------------------------------------------------------
def class_templates(shape: dict, classes: int, seed: int = 0) -> np.ndarray:
    D = shape["H"] * shape["W"] * shape["C"]
    rng = np.random.Generator(np.random.PCG64([0x7E3, seed, D, classes]))
    return rng.integers(0, 256, size=(classes, D)).astype(np.float64)


def make_shard(templates: np.ndarray, n: int, client_id: int, seed: int = 0):
    """x = clip(round(T_y + 32 N(0,1)), 0, 255) as u8 [n, D] (NHWC flattened), y int32 [n]."""
    classes, D = templates.shape
    rng = np.random.Generator(np.random.PCG64([0x5A4D, seed, client_id]))
    y = rng.integers(0, classes, size=n).astype(np.int32)
    x = np.clip(np.rint(templates[y] + 32.0 * rng.standard_normal((n, D))), 0, 255).astype(np.uint8)
    return x, y


def val_size(n_train: int) -> int:
    """Validation split of a client with n_train training examples: 10 % of its data, the
    configs' shard sizes being the training part (SURVEY §8(c).1 ambiguities): round(n_train / 9), >= 1."""
    return max(1, int(round(n_train / 9)))


def make_val_shard(templates: np.ndarray, n_train: int, client_id: int, seed: int = 0):
    """The client's validation split: same class templates and noise model as its training shard, its own
    PCG64 stream."""
    n = val_size(n_train)
    classes, D = templates.shape
    rng = np.random.Generator(np.random.PCG64([0x5A56, seed, client_id]))
    y = rng.integers(0, classes, size=n).astype(np.int32)
    x = np.clip(np.rint(templates[y] + 32.0 * rng.standard_normal((n, D))), 0, 255).astype(np.uint8)
    return x, y


def sample_clients(pool: int, k: int, seed: int, rnd: int) -> np.ndarray:
    """Uniform sample without replacement, sorted ascending (SPEC D-14)."""
    if k > pool:
        raise ValueError("k > pool")
    rng = np.random.Generator(np.random.PCG64([0x5A3F, seed, rnd]))
    return np.sort(rng.choice(pool, size=k, replace=False)).astype(np.int64)


# ---------------------------------------------------------------------------
# Config presets (BASELINE.json configs)
# ---------------------------------------------------------------------------
@dataclass
class Client:
    id: int
    n: int
    batch: int
    epochs: int
    model: int
    width_q: int = 4  # width = width_q / 4
    classes: int = 10


@dataclass
class Workload:
    name: str
    model: int
    shape: dict
    classes: int
    clients: list  # list[Client] (the sampled cohort, ascending id)
    lr: float = 0.05
    seed: int = 0
    rounds: int = 1
    shards: dict = field(default_factory=dict)  # id -> (x u8 [n,D], y int32 [n])

    @property
    def D(self):
        return self.shape["H"] * self.shape["W"] * self.shape["C"]

    def widths(self):
        return sorted({c.width_q for c in self.clients})


BATCHES = (8, 16, 32, 64)
WIDTHS_Q = (1, 2, 4)  # 0.25x, 0.5x, 1x


def build_workload(config: int, *, k=None, n_clients=None, samples=None, epochs=None,
                   shards=True, seed=None, rounds=None) -> Workload:
    """Build one of BASELINE.json configs 1..5 (optionally shrunk for parity tests).

    config 1: 10 clients MLP 784-64-10, 50 samples, E=1, B=10, 3 rounds.
    config 2: 100 clients CNN-1x CIFAR, 500 samples, B=(8,16,32,64)[id%4], E=2.
    config 3: pool 1000 Dirichlet(0.5) over 50,000 samples, CNN-1x, K sampled (10|100).
    config 4: pool 1000 Dirichlet, widths (1/4,1/2,1)[id%3], K=100.
    config 5: pool 10,000 Dirichlet over 500,000, ResNet-8, K=500.
    """
    seed = (config if seed is None else seed)
    if config == 1:
        model, shape, classes = MODEL_MLP, FEMNIST, 10
        n_pool = n_clients or 10
        sizes = np.full(n_pool, samples or 50)
        ids = np.arange(n_pool) if k is None else sample_clients(n_pool, k, seed, 0)
        mk = lambda i: Client(int(i), int(sizes[i]), 10, epochs or 1, model, 4, classes)
        rounds = rounds or 3
    elif config == 2:
        model, shape, classes = MODEL_CNN, CIFAR, 10
        n_pool = n_clients or 100
        sizes = np.full(n_pool, samples or 500)
        ids = np.arange(n_pool) if k is None else sample_clients(n_pool, k, seed, 0)
        mk = lambda i: Client(int(i), int(sizes[i]), BATCHES[i % 4], epochs or 2, model, 4, classes)
    elif config in (3, 4):
        model, shape, classes = MODEL_CNN, CIFAR, 10
        n_pool = n_clients or 1000
        sizes = dirichlet_sizes(n_pool, (samples or 50) * n_pool, 0.5, seed=0)
        ids = sample_clients(n_pool, k or 100, seed, 0)
        if config == 3:
            mk = lambda i: Client(int(i), int(sizes[i]), BATCHES[i % 4], epochs or 2, model, 4, classes)
        else:
            mk = lambda i: Client(int(i), int(sizes[i]), BATCHES[i % 4], epochs or 2, model,
                                  WIDTHS_Q[i % 3], classes)
    elif config == 5:
        model, shape, classes = MODEL_RESNET8, CIFAR, 10
        n_pool = n_clients or 10000
        sizes = dirichlet_sizes(n_pool, (samples or 50) * n_pool, 0.5, seed=0)
        ids = sample_clients(n_pool, k or 500, seed, 0)
        mk = lambda i: Client(int(i), int(sizes[i]), BATCHES[i % 4], epochs or 2, model, 4, classes)
    elif config == 7:  # the paper's CIFAR experiment model: ResNet-18 (GroupNorm, R26), pool 100
        model, shape, classes = MODEL_RESNET18, CIFAR, 10
        n_pool = n_clients or 100
        sizes = np.full(n_pool, samples or 500)
        ids = np.arange(n_pool) if k is None else sample_clients(n_pool, k, seed, 0)
        mk = lambda i: Client(int(i), int(sizes[i]), BATCHES[i % 4], epochs or 1, model, 4, classes)
    elif config == 6:  # the paper's FEMNIST experiment shape: 3597 writers, 62 classes, 28x28x1
        model, shape, classes = MODEL_CNN28, FEMNIST, 62
        n_pool = n_clients or 3597
        sizes = dirichlet_sizes(n_pool, (samples or 226) * n_pool, 0.5, seed=0)
        ids = sample_clients(n_pool, k or 100, seed, 0)
        mk = lambda i: Client(int(i), int(sizes[i]), BATCHES[i % 4], epochs or 1, model, 4, classes)
    else:
        raise ValueError(config)
    wl = Workload(name=f"config{config}", model=model, shape=shape, classes=classes,
                  clients=[mk(int(i)) for i in ids], seed=seed, rounds=rounds or 1)
    if shards:
        tmpl = class_templates(shape, classes, seed)
        for c in wl.clients:
            wl.shards[c.id] = make_shard(tmpl, c.n, c.id, seed)
    return wl
