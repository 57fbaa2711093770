"""Thin Python binding of libprotea.so (include/protea.h), argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; this module only
converts numpy / torch objects to the C structs and pointers the ABI takes.
There is no CPU fallback: importing the package fails loudly if the shared
library is missing (build it with `python paper_2207_01053_b200/build.py` or
`__graft_entry__.build()`).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libprotea.so")
if not os.path.exists(LIB_PATH):
    raise ImportError(f"libprotea.so not built at {LIB_PATH}: run __graft_entry__.build()")
_lib = ctypes.CDLL(LIB_PATH)

# status codes (protea_status)
OK, ERR_INVALID, ERR_EMPTY, ERR_ZERO_WEIGHT, ERR_DIM, ERR_NO_CAPACITY, ERR_PLAN, ERR_OOM, ERR_CUDA, ERR_NCCL = range(10)
STATUS_NAMES = {0: "OK", 1: "INVALID", 2: "EMPTY", 3: "ZERO_WEIGHT", 4: "DIM", 5: "NO_CAPACITY", 6: "PLAN", 7: "OOM",
                8: "CUDA", 9: "NCCL"}
MODEL_MLP, MODEL_CNN, MODEL_RESNET8, MODEL_RESNET18 = 0, 1, 2, 3
PREC_FP32, PREC_BF16 = 0, 1
POLICY_PROFILED, POLICY_STATIC = 0, 1
ORDER_ASC_ID, ORDER_DESC_STEPS = 0, 1

EXPORTS = ["protea_init", "protea_finalize", "protea_last_error", "protea_register_model", "protea_register_shards",
           "protea_profile_clients", "protea_plan", "protea_run_round", "protea_fedavg", "protea_client_footprint",
           "protea_selftest_gemm", "protea_round_partial", "protea_round_finalize", "protea_plan_hash",
           "protea_round_finalize_ordered", "protea_register_val_shards", "protea_evaluate_round",
           "protea_evaluate", "protea_heterofl_extract", "protea_heterofl_aggregate"]


class ProteaError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.name = STATUS_NAMES.get(code, str(code))


# ---------------------------------------------------------------------------
# C structs
# ---------------------------------------------------------------------------
class InitOpts(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("rank", ctypes.c_int32), ("world", ctypes.c_int32),
                ("precision", ctypes.c_int32), ("nccl_id", ctypes.c_void_p), ("arena", ctypes.c_void_p),
                ("arena_bytes", ctypes.c_uint64), ("stream", ctypes.c_void_p)]


class ModelDesc(ctypes.Structure):
    _fields_ = [("arch", ctypes.c_int32), ("width_q", ctypes.c_int32), ("classes", ctypes.c_int32),
                ("H", ctypes.c_int32), ("W", ctypes.c_int32), ("C", ctypes.c_int32)]


class Cluster(ctypes.Structure):
    _fields_ = [("n_gpus", ctypes.c_uint32), ("reserved", ctypes.c_uint32), ("capacity", ctypes.c_void_p)]


class PlanOpts(ctypes.Structure):
    _fields_ = [("policy", ctypes.c_int32), ("order", ctypes.c_int32), ("margin_permille", ctypes.c_uint32),
                ("max_active", ctypes.c_uint32)]


N_OPC = 32
# op classes that run on tcgen05 tensor cores in bf16 mode (CNN); the others use SIMT fp32 math
TC_OPS_BUILT = {"conv1_fwd": True, "conv2_fwd": True, "fc1_fwd": True, "fc1_dgrad": True, "fc1_wgrad": True,
                "conv2_dgrad": True, "conv2_wgrad": True, "conv1_wgrad": True, "resnet_fwd": True,
                "resnet_dgrad": True, "resnet_wgrad": True}
OPC_NAMES = ["conv1_fwd", "conv2_fwd", "fc1_fwd", "head", "fc1_dgrad", "fc1_wgrad", "conv2_dgrad", "conv2_wgrad",
             "conv2_reduce", "conv1_wgrad", "conv1_reduce", "mlp_fc1_fwd", "mlp_head", "mlp_fc1_wgrad", "admit",
             "fedavg", "stage_x", "resnet_fwd", "resnet_head", "resnet_dgrad", "resnet_wgrad",
             "resnet_reduce", "eval_head"] + [f"op{i}" for i in range(23, 32)]


class RoundOpts(ctypes.Structure):
    _fields_ = [("lr", ctypes.c_float), ("seed", ctypes.c_uint32), ("round", ctypes.c_uint32),
                ("shuffle", ctypes.c_int32), ("time_ops", ctypes.c_uint32), ("partial_only", ctypes.c_uint32),
                ("serialize", ctypes.c_uint32), ("observe_hwm", ctypes.c_uint32), ("n_trace", ctypes.c_uint32),
                ("trace_ids", ctypes.c_void_p), ("trace_bufs", ctypes.c_void_p)]


class RoundStats(ctypes.Structure):
    _fields_ = [("round_ns", ctypes.c_uint64), ("iterations", ctypes.c_uint64), ("client_steps", ctypes.c_uint64),
                ("kernel_launches", ctypes.c_uint64), ("flops", ctypes.c_uint64), ("loss_sum", ctypes.c_double),
                ("op_ns", ctypes.c_uint64 * N_OPC), ("op_launches", ctypes.c_uint64 * N_OPC),
                ("op_flops", ctypes.c_uint64 * N_OPC), ("op_bytes", ctypes.c_uint64 * N_OPC),
                ("op_timed_launches", ctypes.c_uint64 * N_OPC), ("op_timed_flops", ctypes.c_uint64 * N_OPC),
                ("op_timed_bytes", ctypes.c_uint64 * N_OPC)]

    def as_dict(self):
        d = {}
        for k, _ in self._fields_:
            v = getattr(self, k)
            d[k] = list(v) if k.startswith("op_") else v
        return d


SHARD_DT = np.dtype([("client_id", "<i8"), ("n", "<i8"), ("x", "<u8"), ("y", "<u8")], align=True)
CLIENT_DT = np.dtype([("client_id", "<i8"), ("model_id", "<i4"), ("batch", "<i4"), ("epochs", "<i4"),
                      ("reserved", "<i4")], align=True)
PROFILE_DT = np.dtype([("client_id", "<i8"), ("peak_bytes", "<u8"), ("steps", "<u8"), ("flops", "<u8"),
                       ("step_ns", "<u8"), ("train_ns", "<u8"), ("sm_ns", "<u8"), ("uses_gpu", "<u4"),
                       ("reserved", "<u4")], align=True)
ASSIGN_DT = np.dtype([("client_id", "<i8"), ("gpu", "<i4"), ("q1024", "<u4"), ("offset", "<u8"), ("slot", "<u8"),
                      ("admit", "<u8"), ("release", "<u8")], align=True)
assert SHARD_DT.itemsize == 32 and CLIENT_DT.itemsize == 24 and PROFILE_DT.itemsize == 64 and ASSIGN_DT.itemsize == 48

_vp, _sz = ctypes.c_void_p, ctypes.c_size_t
_lib.protea_init.argtypes = [ctypes.POINTER(InitOpts), ctypes.POINTER(ctypes.c_void_p)]
_lib.protea_finalize.argtypes = [_vp]
_lib.protea_finalize.restype = None
_lib.protea_last_error.argtypes = [_vp]
_lib.protea_last_error.restype = ctypes.c_char_p
_lib.protea_register_model.argtypes = [_vp, ctypes.POINTER(ModelDesc), ctypes.POINTER(ctypes.c_int32),
                                       ctypes.POINTER(ctypes.c_uint64)]
_lib.protea_register_shards.argtypes = [_vp, _vp, _sz]
_lib.protea_profile_clients.argtypes = [_vp, _vp, _sz, _vp]
_lib.protea_plan.argtypes = [_vp, _sz, ctypes.POINTER(Cluster), ctypes.POINTER(PlanOpts), _vp, _vp]
_lib.protea_run_round.argtypes = [_vp, ctypes.POINTER(RoundOpts), _vp, _sz, _vp, _vp, _vp, _sz, _vp,
                                  ctypes.POINTER(RoundStats)]
_lib.protea_fedavg.argtypes = [_vp, _vp, _vp, _sz, _sz, _vp]
_lib.protea_client_footprint.argtypes = [ctypes.POINTER(ModelDesc), ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                         ctypes.c_int32, ctypes.POINTER(ctypes.c_uint64),
                                         ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64)]
_lib.protea_round_partial.argtypes = [_vp, _vp, _sz]
_lib.protea_round_finalize.argtypes = [_vp, _vp, _vp, _vp, _sz]
_lib.protea_round_finalize_ordered.argtypes = [_vp, _vp, ctypes.c_int32, _vp, _vp, _sz]
_lib.protea_register_val_shards.argtypes = [_vp, _vp, _sz]
_lib.protea_evaluate_round.argtypes = [_vp, _vp, _sz, _vp, _sz, _vp, _vp]
_lib.protea_selftest_gemm.argtypes = [_vp, _vp, _vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32]
for _f in EXPORTS:
    if _f not in ("protea_finalize", "protea_last_error", "protea_plan_hash"):
        getattr(_lib, _f).restype = ctypes.c_int
_lib.protea_plan_hash.argtypes = [_vp, _sz, _vp]
_lib.protea_evaluate.argtypes = [_vp, ctypes.c_int32, _vp, _vp, _vp, ctypes.c_int64, _vp]
_lib.protea_plan_hash.restype = ctypes.c_uint64
_lib.protea_heterofl_extract.argtypes = [_vp, ctypes.c_int32, _vp, ctypes.c_int32, _vp]
_lib.protea_heterofl_aggregate.argtypes = [_vp, ctypes.c_int32, _vp, _vp, _vp, _vp, _sz, _vp]


def _check(code, ctx=None):
    if code != OK:
        msg = _lib.protea_last_error(ctx)
        raise ProteaError(code, msg.decode() if msg else "")


def _ptr(a):
    """data pointer of a numpy array or torch tensor (or an int)."""
    if a is None:
        return None
    if isinstance(a, int):
        return a
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data


# ---------------------------------------------------------------------------
# ABI calls (same names as include/protea.h)
# ---------------------------------------------------------------------------
def protea_init(device=0, rank=0, world=1, precision=PREC_FP32, arena=None, arena_bytes=0, stream=None,
                nccl_id=None):
    """arena: device tensor (uint8) or pointer; stream: torch.cuda.Stream, cudaStream_t int, or None."""
    if stream is not None and hasattr(stream, "cuda_stream"):
        stream = stream.cuda_stream
    nid = None
    if nccl_id is not None:
        buf = (ctypes.c_uint8 * 128).from_buffer_copy(bytes(nccl_id))
        nid = ctypes.addressof(buf)
    if arena is not None and hasattr(arena, "numel") and not arena_bytes:
        arena_bytes = arena.numel() * arena.element_size()
    o = InitOpts(device, rank, world, precision, nid, _ptr(arena), arena_bytes, stream)
    ctx = ctypes.c_void_p()
    _check(_lib.protea_init(ctypes.byref(o), ctypes.byref(ctx)))
    return ctx


def protea_finalize(ctx):
    _lib.protea_finalize(ctx)


def protea_last_error(ctx=None):
    m = _lib.protea_last_error(ctx)
    return m.decode() if m else ""


def protea_register_model(ctx, arch, width_q=4, classes=10, H=32, W=32, C=3):
    d = ModelDesc(arch, width_q, classes, H, W, C)
    mid, npar = ctypes.c_int32(), ctypes.c_uint64()
    _check(_lib.protea_register_model(ctx, ctypes.byref(d), ctypes.byref(mid), ctypes.byref(npar)), ctx)
    return mid.value, npar.value


def _shard_records(shards):
    keep = []
    rec = np.zeros(len(shards), dtype=SHARD_DT)
    for i, (cid, x, y) in enumerate(shards):
        x = np.ascontiguousarray(x, dtype=np.uint8)
        y = np.ascontiguousarray(y, dtype=np.int32)
        keep += [x, y]
        rec[i] = (cid, y.shape[0], x.ctypes.data, y.ctypes.data)
    return rec, keep


def protea_register_shards(ctx, shards):
    """shards: iterable of (client_id, x u8 [n, D], y int32 [n]) host arrays."""
    rec, keep = _shard_records(shards)
    _check(_lib.protea_register_shards(ctx, rec.ctypes.data, len(rec)), ctx)


def protea_register_val_shards(ctx, shards):
    """Validation splits, same records as protea_register_shards."""
    rec, keep = _shard_records(shards)
    _check(_lib.protea_register_val_shards(ctx, rec.ctypes.data, len(rec)), ctx)


def protea_evaluate_round(ctx, clients, global_w):
    """Every client evaluates its group's global weights (float32 tensor/array, host or device, all groups
    concatenated) on its validation split.  Returns (per-client EVAL_DT records, (loss_sum, correct, n))."""
    n_params = global_w.numel() if hasattr(global_w, "numel") else global_w.size
    per = np.zeros(len(clients), dtype=EVAL_DT)
    tot = EvalResult()
    _check(_lib.protea_evaluate_round(ctx, clients.ctypes.data, len(clients), _ptr(global_w), n_params,
                                      per.ctypes.data, ctypes.byref(tot)), ctx)
    return per, (tot.loss_sum, int(tot.correct), int(tot.n))


def clients_array(rows):
    """rows: iterable of (client_id, model_id, batch, epochs) -> CLIENT_DT array."""
    rows = list(rows)
    a = np.zeros(len(rows), dtype=CLIENT_DT)
    for i, (cid, mid, b, e) in enumerate(rows):
        a[i] = (cid, mid, b, e, 0)
    return a


def protea_profile_clients(ctx, clients):
    out = np.zeros(len(clients), dtype=PROFILE_DT)
    _check(_lib.protea_profile_clients(ctx, clients.ctypes.data, len(clients), out.ctypes.data), ctx)
    return out


def protea_plan(profiles, caps, policy=POLICY_PROFILED, order=ORDER_ASC_ID, margin_permille=1000, max_active=0):
    profiles = np.ascontiguousarray(profiles, dtype=PROFILE_DT)
    caps = np.ascontiguousarray(caps, dtype=np.uint64)
    cl = Cluster(len(caps), 0, caps.ctypes.data)
    po = PlanOpts(policy, order, margin_permille, max_active)
    out = np.zeros(len(profiles), dtype=ASSIGN_DT)
    mk = np.zeros(len(caps), dtype=np.uint64)
    _check(_lib.protea_plan(profiles.ctypes.data, len(profiles), ctypes.byref(cl), ctypes.byref(po),
                            out.ctypes.data, mk.ctypes.data))
    return out, mk


EVAL_DT = np.dtype([("loss_sum", np.float64), ("correct", np.uint64), ("n", np.uint64)])


class EvalResult(ctypes.Structure):
    _fields_ = [("loss_sum", ctypes.c_double), ("correct", ctypes.c_uint64), ("n", ctypes.c_uint64)]


def protea_evaluate(ctx, model_id, weights, x, y):
    """Evaluate model `model_id` with `weights` (float32 tensor/array, host or device) on u8 samples x
    [n, H, W, C] and int32 labels y (host).  Returns (loss_sum, correct, n)."""
    x = np.ascontiguousarray(x, dtype=np.uint8)
    y = np.ascontiguousarray(y, dtype=np.int32)
    r = EvalResult()
    _check(_lib.protea_evaluate(ctx, model_id, _ptr(weights), x.ctypes.data, y.ctypes.data, len(y),
                                ctypes.byref(r)), ctx)
    return r.loss_sum, int(r.correct), int(r.n)


def protea_plan_hash(clients, plan):
    """64-bit hash of a round's client list and plan (run_round compares it across ranks when world > 1)."""
    clients = np.ascontiguousarray(clients, dtype=CLIENT_DT)
    plan = np.ascontiguousarray(plan, dtype=ASSIGN_DT)
    assert len(clients) == len(plan)
    return int(_lib.protea_plan_hash(clients.ctypes.data, len(clients), plan.ctypes.data))


def protea_run_round(ctx, clients, plan, global_in, global_out, lr=0.05, seed=0, rnd=0, shuffle=True,
                     measured=False, time_ops=0, partial_only=False, serialize=False, observe_hwm=False,
                     trace=None):
    """global_in / global_out: float32 torch tensors (cuda or cpu) or numpy arrays.
    trace: {client_id: device uint8 tensor of (S_k + 1) * footprint peak_bytes} slot snapshots per local step."""
    trace = trace or {}
    tids = np.array(list(trace.keys()), dtype=np.int64)
    tbufs = np.array([_ptr(t) for t in trace.values()], dtype=np.uint64)
    o = RoundOpts(lr, seed, rnd, 1 if shuffle else 0, time_ops, 1 if partial_only else 0, 1 if serialize else 0,
                  1 if observe_hwm else 0, len(tids), tids.ctypes.data if len(tids) else None,
                  tbufs.ctypes.data if len(tids) else None)
    st = RoundStats()
    n_params = global_in.numel() if hasattr(global_in, "numel") else global_in.size
    meas = np.zeros(len(clients), dtype=PROFILE_DT) if measured else None
    _check(_lib.protea_run_round(ctx, ctypes.byref(o), clients.ctypes.data, len(clients),
                                 np.ascontiguousarray(plan, dtype=ASSIGN_DT).ctypes.data, _ptr(global_in),
                                 _ptr(global_out), n_params, meas.ctypes.data if measured else None,
                                 ctypes.byref(st)), ctx)
    return (st.as_dict(), meas) if measured else st.as_dict()


def protea_round_partial(ctx, dst):
    """dst: float64 tensor / array of n_params (device or host)."""
    n = dst.numel() if hasattr(dst, "numel") else dst.size
    _check(_lib.protea_round_partial(ctx, _ptr(dst), n), ctx)


def protea_round_finalize(ctx, acc_sum, global_in, global_out):
    n = global_in.numel() if hasattr(global_in, "numel") else global_in.size
    _check(_lib.protea_round_finalize(ctx, _ptr(acc_sum), _ptr(global_in), _ptr(global_out), n), ctx)


def protea_round_finalize_ordered(ctx, partials, global_in, global_out):
    """partials: float64 [nparts, n_params] tensor / array (device or host), ranks in order."""
    n = global_in.numel() if hasattr(global_in, "numel") else global_in.size
    nparts = partials.shape[0]
    assert tuple(partials.shape) == (nparts, n)
    _check(_lib.protea_round_finalize_ordered(ctx, _ptr(partials), int(nparts), _ptr(global_in), _ptr(global_out), n),
           ctx)


def protea_fedavg(ctx, params, num_examples, out):
    """params: list of device float32 tensors (same length); out: device tensor."""
    ptrs = np.array([p.data_ptr() for p in params], dtype=np.uint64)
    ns = np.ascontiguousarray(num_examples, dtype=np.int64)
    dim = out.numel()
    _check(_lib.protea_fedavg(ctx, ptrs.ctypes.data, ns.ctypes.data, len(params), dim, out.data_ptr()), ctx)


def protea_client_footprint(arch, width_q, classes, H, W, C, n, batch, epochs, precision=PREC_FP32):
    d = ModelDesc(arch, width_q, classes, H, W, C)
    pb, st, fl = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    _check(_lib.protea_client_footprint(ctypes.byref(d), n, batch, epochs, precision, ctypes.byref(pb),
                                        ctypes.byref(st), ctypes.byref(fl)))
    return pb.value, st.value, fl.value


def protea_selftest_gemm(A, B, D, M, N, K, mn_major=False):
    """include/protea_selftest.h: D = A B^T on the library's tcgen05 core (device tensors)."""
    _check(_lib.protea_selftest_gemm(A.data_ptr(), B.data_ptr(), D.data_ptr(), M, N, K, 1 if mn_major else 0))


def protea_heterofl_extract(ctx, global_full, width_q, classes=10):
    """Width-q sub-model (new device tensor) of the full-width CNN weights (HeteroFL, R23)."""
    import torch
    q = int(width_q)
    c1, c2, f = 8 * q, 16 * q, 128 * q
    out = torch.empty(c1 * 75 + c1 + c2 * 25 * c1 + c2 + f * 64 * c2 + f + classes * f + classes,
                      dtype=torch.float32, device=global_full.device)
    _check(_lib.protea_heterofl_extract(ctx, int(classes), global_full.data_ptr(), q, out.data_ptr()), ctx)
    return out


def protea_heterofl_aggregate(ctx, global_full, params, widths, num_examples, out=None, classes=10):
    """n_k-weighted per-element mean over the clients whose width-q sub-model holds the element; the
    rest keeps global_full (device tensors; HeteroFL, R23)."""
    import torch
    out = torch.empty_like(global_full) if out is None else out
    n = len(params)
    ptrs = (ctypes.c_void_p * max(n, 1))(*[p.data_ptr() for p in params])
    wq = np.asarray(widths, dtype=np.int32)
    ne = np.asarray(num_examples, dtype=np.int64)
    _check(_lib.protea_heterofl_aggregate(ctx, int(classes), global_full.data_ptr(), ptrs, wq.ctypes.data,
                                          ne.ctypes.data, n, out.data_ptr()), ctx)
    return out
