#!/usr/bin/env python
"""Benchmark of the Protea hot path (BASELINE.json metric: client local-steps/sec).

One bench "step" = one federated round of the whole hot path:
A1 round setup (sampled cohort, host), A4 protea_plan (host, integer), and
protea_run_round = A2 every client's local SGD epochs + A3 in-run profiles +
A5 FedAvg (+ the NCCL sum when N > 1).  The N=1 workload is BASELINE.json
configs[1] ("config2"): 100 clients, CNN-1x on CIFAR-shaped synthetic data,
500 samples each, B in {8,16,32,64} (id mod 4), 2 local epochs -> 5,950
client-steps per round.  For N > 1 every GPU gets another 100 such clients
(weak scaling, LPT partition by FLOPs, one NCCL all-gather of the fp64 FedAvg
partials + a rank-ordered sum per round).

--config 3|5 --scaling strong runs the north-star target instead: ONE round of
the config's cohort (config 3: K = 100 of a 1000-client Dirichlet(0.5) pool,
CNN-1x; config 5: K = 500 of a 10,000-client Dirichlet pool, ResNet-8) split
over the N GPUs by the profile-driven LPT packing (strong scaling: total work
fixed).  --config 2 --scaling strong splits config 2's 100 clients.

Launch: python bench.py [--gpus N --steps K --warmup W] [--config 2|3|5] [--scaling weak|strong]
        [--impl reference]   (N > 1 under torchrun; rank 0 prints one JSON line)
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "client_local_steps_per_sec"
UNIT = "client-steps/s"
CLIENTS_PER_GPU = 100


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return dict(hbm=float(p["hbm_gbs"]), bf16=float(p["bf16_tflops"]), bf16_sus=float(p["bf16_tflops_sustained"]),
                    sm_max_mhz=float(p.get("sm_max_mhz", 1965.0)), src="measured (MEASURED_PEAKS.json)")
    except Exception:
        return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, sm_max_mhz=1965.0,
                    src="fallback (B200_PROFILING.md)")


# fp32 SIMT peak: 148 SMs x 128 FP32 lanes x 2 FLOP/FMA x SM clock
def fp32_alu_peak_tflops(mhz):
    return 148 * 128 * 2 * mhz * 1e6 / 1e12


def workload(world, config=2, scaling="weak"):
    if config == 2:
        return synth.build_workload(2, n_clients=CLIENTS_PER_GPU * (world if scaling == "weak" else 1), shards=False)
    if config == 3:
        return synth.build_workload(3, k=100 * (world if scaling == "weak" else 1), shards=False)
    if config == 5:
        return synth.build_workload(5, k=500 * (world if scaling == "weak" else 1), shards=False)
    raise ValueError(f"bench: config {config} not supported (2, 3, 5)")


ALGO_NOTE = {"fc1_wgrad": "SURVEY §8(d): 8 B per fc1 weight per client-step (fp32 master read + write) + dh / a2 reads",
             "resnet_fwd": "2 x useful MACs of the 3x3 convs of the launch's rows (implicit GEMM)",
             "resnet_dgrad": "2 x useful MACs of the 3x3 input-gradient convs", "resnet_wgrad": "2 x useful MACs "
             "of the 3x3 weight-gradient GEMMs"}
ARCH_NAME = {synth.MODEL_CNN: "CNN-1x (P=2,156,490)", synth.MODEL_RESNET8: "ResNet-8 (P=75,050)"}


# ---------------------------------------------------------------------------
# nvidia-smi clock sampler (rank 0, during the timed region)
# ---------------------------------------------------------------------------
class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.samples = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                self.samples.append(parts)

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=2)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[5 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# oracle (CPU) baseline: bounded sample of the same workload on the host cores
# ---------------------------------------------------------------------------
_ORACLE_JOB = {}


def _oracle_worker_init():
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass


def _oracle_client(i):
    from oracle.sgd import local_sgd
    j = _ORACLE_JOB
    c = j["clients"][i]
    x, y = j["shards"][c.id]
    t0 = time.perf_counter()
    _, losses = local_sgd(j["w0"], c.model, c.width_q, c.classes, x, y, c.batch, c.epochs, j["lr"], j["seed"], 0,
                          c.id, max_steps=j["steps"][i])
    return len(losses), time.perf_counter() - t0


def oracle_sample(wl, frac=0.05, cores=None):
    """Run the first ceil(frac * S_k) local steps of every client on a process
    pool of `cores` workers (one task per client, BLAS threads pinned to 1).
    Returns (client-steps done, wall seconds, cores)."""
    import multiprocessing as mp
    from oracle.profiler import local_steps
    cores = cores or len(os.sched_getaffinity(0))
    tmpl = synth.class_templates(wl.shape, wl.classes, wl.seed)
    shards = {c.id: synth.make_shard(tmpl, c.n, c.id, wl.seed) for c in wl.clients}
    _ORACLE_JOB.update(clients=wl.clients, shards=shards, w0=synth.init_weights(wl.model).astype(np.float64),
                       lr=wl.lr, seed=wl.seed,
                       steps=[max(1, math.ceil(frac * local_steps(c.n, c.batch, c.epochs))) for c in wl.clients])
    ctx = mp.get_context("fork")
    t0 = time.perf_counter()
    with ctx.Pool(cores, initializer=_oracle_worker_init) as pool:
        res = pool.map(_oracle_client, range(len(wl.clients)), chunksize=1)
    wall = time.perf_counter() - t0
    return sum(r[0] for r in res), wall, cores


# ---------------------------------------------------------------------------
# reference arm: the oracle as it stands, timed on host cores
# ---------------------------------------------------------------------------
def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    wl = workload(1, args.config, args.scaling)
    frac = 0.02 if args.config == 2 else 0.01
    oracle_sample(wl, frac=0.005)  # warm the pool / imports (not timed)
    for _ in range(max(0, args.warmup - 1)):
        oracle_sample(wl, frac=0.005)
    steps = 0
    wall = 0.0
    cores = None
    for _ in range(args.steps):
        s, w, cores = oracle_sample(wl, frac=frac)
        steps += s
        wall += w
    value = steps / wall
    sample = (f"first ceil({frac}*S_k) local steps of each of the {len(wl.clients)} config{args.config} clients per "
              f"bench step ({steps // args.steps} client-steps/step), float64 numpy oracle, {cores} processes")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wall / args.steps,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_block(wl, 1, "f64", args.config, args.scaling),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def config_block(wl, world, dtype, config=2, scaling="weak"):
    steps = [c.epochs * -(-c.n // c.batch) for c in wl.clients]  # S_k = E ceil(n_k / B_k)
    what = {2: "config2 (BASELINE.json configs[1]): CNN-1x (P=2,156,490) on synthetic CIFAR-shaped u8 data, "
               "500 samples/client, B=(8,16,32,64)[id%4], E=2, lr=0.05",
            3: "config3 (BASELINE.json configs[2]): K=100 of a 1000-client Dirichlet(0.5) pool (50,000 samples), "
               "CNN-1x, B=(8,16,32,64)[id%4], E=2, lr=0.05",
            5: "config5 (BASELINE.json configs[4]): K=500 of a 10,000-client Dirichlet(0.5) pool (500,000 samples), "
               "ResNet-8 (P=75,050), B=(8,16,32,64)[id%4], E=2, lr=0.05"}[config]
    per = f"{len(wl.clients) // world} clients/GPU" if scaling == "weak" else f"{len(wl.clients)} clients over {world} GPU(s)"
    return {"workload": f"{what}; {per}",
            "clients_total": len(wl.clients), "client_steps_per_round": int(sum(steps)),
            "max_local_steps": int(max(steps)), "precision": dtype,
            "l2": "no flush: per-GPU resident inputs (u8 shards + per-client fp32 weights and activations) exceed "
                  "the 126 MB L2" if config != 5 else "no flush: per-GPU resident shards (1.5 MB..) + client "
                  "slots (500 x 3-19 MB) exceed the 126 MB L2",
            "parallelism": f"clients partitioned over {world} GPU(s) by LPT on FLOPs; NCCL all-gather of the fp64 "
                           "FedAvg partials + rank-ordered sum" if world > 1
                           else "1 GPU, all clients co-resident (lock-step grouped kernels)"}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default="bf16", choices=["fp32", "bf16"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--config", type=int, default=2, choices=[2, 3, 5])
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--observe-hwm", type=int, default=1,
                    help="timed rounds observe each client's arena high-water mark (A3 profile -> next plan)")
    args = ap.parse_args()
    if args.impl == "reference":
        return reference_arm(args)

    import torch
    import torch.distributed as dist

    import paper_2207_01053_b200 as pb
    from paper_2207_01053_b200.sim import Simulation

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    prec = pb.PREC_FP32 if args.precision == "fp32" else pb.PREC_BF16
    dtype = "f32" if prec == pb.PREC_FP32 else "bf16"
    eb = 4 if prec == pb.PREC_FP32 else 2

    wl = workload(world, args.config, args.scaling)
    arch = wl.model
    # A4 inputs on every rank from the pure host footprint (identical on all ranks)
    foot = np.zeros(len(wl.clients), dtype=pb.PROFILE_DT)
    for i, c in enumerate(wl.clients):
        pk, st, fl = pb.protea_client_footprint(arch, 4, 10, 32, 32, 3, c.n, c.batch, c.epochs, prec)
        foot[i] = (c.id, pk, st, fl, 0, 0, 0, 1, 0)
    arena_bytes = int(sum(int(f["peak_bytes"]) for f in foot) // world * 1.25) + (256 << 20)
    caps = [arena_bytes] * world
    plan0, _ = pb.protea_plan(foot, caps)
    mine = [c for c, a in zip(wl.clients, plan0) if int(a["gpu"]) == rank]

    nccl_id = None
    if world > 1:
        obj = [torch.cuda.nccl.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    sim = Simulation(device=local, precision=prec, arena_bytes=arena_bytes, rank=rank, world=world, nccl_id=nccl_id)
    mid = sim.register_model(arch, 4, 10, 32, 32, 3)
    tmpl = synth.class_templates(wl.shape, wl.classes, wl.seed)
    # every rank holds every sampled client's shard (HBM is ample; run_round takes n_k of all
    # clients from the registry for the FedAvg denominator); the e2e timing re-sends only this rank's shards
    all_shards = {c.id: synth.make_shard(tmpl, c.n, c.id, wl.seed) for c in wl.clients}
    shards = {c.id: all_shards[c.id] for c in mine}
    sim.register_shards([(c.id, *all_shards[c.id]) for c in wl.clients])
    all_clients = sim.clients([(c.id, mid, c.batch, c.epochs) for c in wl.clients])
    my_clients = sim.clients([(c.id, mid, c.batch, c.epochs) for c in mine])

    # A3 cold start: probe profiles of this rank's shape classes (reported, not timed)
    t0 = time.perf_counter()
    probe = sim.profile(my_clients)
    probe_s = time.perf_counter() - t0
    profiles = foot.copy()

    g = torch.tensor(synth.init_weights(wl.model), device=sim.device)
    g2 = torch.empty_like(g)
    stream = sim.stream
    round_steps = sum(int(f["steps"]) for f in foot)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # warm-up rounds; the first one times every op class to pick the dominant kernel
    rnd = 0
    dominant, op_stats = None, None
    for w in range(args.warmup):
        plan, _ = pb.protea_plan(profiles, caps)
        # the first warm-up round runs serialised (no side-stream overlap) with every op class timed: the
        # per-op shares of that round are the ones a serialised ncu launch list of this command shows
        _, st = sim.run_round(all_clients, plan, g, g2, lr=wl.lr, seed=wl.seed, rnd=rnd,
                              time_ops=(0xFFFFFFFF if w == 0 else 0), serialize=(w == 0))
        g, g2 = g2, g
        rnd += 1
        if w == 0:
            op_stats = st
            dominant = int(np.argmax(st["op_ns"]))
    if dominant is None:
        dominant = 7

    # ---- timed region (device time, CUDA events on the library's stream)
    clocks = ClockSampler(local) if rank == 0 else None
    from paper_2207_01053_b200.monitor import UtilMonitor  # paper's UtilMonitor analogue (host side)
    umon = UtilMonitor(device=local, interval=0.1) if rank == 0 else None
    barrier()
    if clocks:
        clocks.start()
    if umon:
        umon.start()
    launches = 0
    dom_ns = dom_fl = dom_by = dom_n = 0
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    host_t0 = time.perf_counter()
    for k in range(args.steps):
        ev[k][0].record(stream)
        plan, _ = pb.protea_plan(profiles, caps)                     # A4
        # the dominant op's launches are bracketed by CUDA events in the LAST timed round only: on config 5
        # (~630 ResNet wgrad launches per round) event records in every round cost ~15 % of the round
        instrument = k == args.steps - 1
        _, (st, meas) = sim.run_round(all_clients, plan, g, g2, lr=wl.lr, seed=wl.seed, rnd=rnd,
                                      measured=True, time_ops=(1 << dominant) if instrument else 0,
                                      observe_hwm=bool(args.observe_hwm))  # A2 + A3 + A5
        ev[k][1].record(stream)
        g, g2 = g2, g
        rnd += 1
        launches += st["kernel_launches"]
        dom_ns += st["op_ns"][dominant]
        # the timed launches and their work (fc1 wgrad launches deferred to the side stream in light
        # iterations run concurrently with other kernels and are not timed)
        dom_fl += st["op_timed_flops"][dominant]
        dom_by += st["op_timed_bytes"][dominant]
        dom_n += st["op_timed_launches"][dominant]
        if world == 1:  # A3 -> next A4: the latest in-run profile replaces the previous one (reading R7)
            profiles = meas  # (N > 1: each rank observes only its own clients; the plan keeps the footprints)
            # a client whose every batch is partial (n < B) may leave the tail of its last buffers untouched, so
            # its observed mark can sit below the slot layout run_round validates against: plan at least that
            profiles["peak_bytes"] = np.maximum(profiles["peak_bytes"], foot["peak_bytes"])
    barrier()
    host_s = time.perf_counter() - host_t0
    clk = clocks.stop() if clocks else None
    host_mon = umon.stop() if umon else None
    dev_ms = sum(a.elapsed_time(b) for a, b in ev)
    t = torch.tensor([dev_ms], dtype=torch.float64, device=sim.device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dev_ms = float(t.item())
    ms_per_step = dev_ms / args.steps
    value = round_steps / (ms_per_step / 1e3)

    # ---- roofline of the dominant kernel (achieved per launch from the live events)
    pk = peaks()
    timing_src = "timed rounds (CUDA events on the launching stream)"
    if dom_n == 0 and op_stats is not None and op_stats["op_launches"][dominant]:
        # every launch of the op ran deferred on the side stream in the timed rounds (PROTEA_OVERLAP_ROWS):
        # take the serialised warm-up round's launches of it instead
        dom_n = int(op_stats["op_launches"][dominant])
        dom_ns, dom_fl, dom_by = op_stats["op_ns"][dominant], op_stats["op_flops"][dominant], op_stats["op_bytes"][dominant]
        timing_src = "serialised warm-up round (every timed-round launch was deferred to the side stream)"
    avg_ns = max(dom_ns / max(1, dom_n), 1.0)
    fl_per = dom_fl / max(1, dom_n)
    by_per = dom_by / max(1, dom_n)
    alu_peak = fp32_alu_peak_tflops(pk["sm_max_mhz"])
    ridge = alu_peak * 1e12 / (pk["hbm"] * 1e9)
    # which op classes run on tcgen05 in bf16 mode (the rest are SIMT fp32 math)
    tc_ops = {"conv1_fwd", "conv2_fwd", "fc1_fwd", "fc1_dgrad", "fc1_wgrad", "conv2_dgrad", "conv2_wgrad",
              "conv1_wgrad", "resnet_fwd", "resnet_dgrad", "resnet_wgrad"} if prec == pb.PREC_BF16 else set()
    on_tc = pb.OPC_NAMES[dominant] in tc_ops and pb.TC_OPS_BUILT.get(pb.OPC_NAMES[dominant], False)
    if fl_per / max(by_per, 1) >= ridge:
        bound, achieved, peak, unit = ("tensor", fl_per / avg_ns / 1e3, pk["bf16_sus"], "TFLOP/s") if on_tc \
            else ("alu", fl_per / avg_ns / 1e3, alu_peak, "TFLOP/s")
    else:
        bound, achieved, peak, unit = "hbm", by_per / avg_ns, pk["hbm"], "GB/s"
    traffic = None
    tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tf):  # DRAM bytes of this op from the committed ncu launch list of the same command
        try:
            rec = json.load(open(tf)).get(pb.OPC_NAMES[dominant], {}).get(dtype, {})
            # the ncu list covers every launch of the op in the round, `achieved` only the timed ones: scale
            # the timed launches' algorithmic bytes by the round's measured DRAM / algorithmic byte ratio
            algo_round = float(st["op_bytes"][dominant])
            if rec and algo_round > 0:
                traffic = by_per * rec["dram_bytes_per_launch"] * rec["launches"] / algo_round
        except Exception:
            traffic = None
    # bf16 mode keeps fc1's fp32 master as two 16-bit planes (the upper plane is the tensor-core operand of
    # fc1 fwd / dgrad), so fc1 wgrad moves exactly SURVEY §8(d)'s 8 B per weight: no
    # implementation bytes beyond the algorithmic ones (round 1 wrote a separate 2 B bf16 shadow)
    impl = ({"note": "fp32 master as hi/lo 16-bit planes: no shadow write; actual bytes = algorithmic bytes"}
            if pb.OPC_NAMES[dominant] == "fc1_wgrad" and prec == pb.PREC_BF16 else None)
    roof = {"kernel": pb.OPC_NAMES[dominant], "bound": bound, "achieved": achieved, "peak": peak, "unit": unit,
            "frac": achieved / peak, "traffic": traffic, "algorithmic": ALGO_NOTE.get(pb.OPC_NAMES[dominant], "engine op_work: "
            "operands read once, results written once"), "implementation_extra": impl,
            "peak_src": pk["src"] if bound != "alu" else f"derived: 148 SM x 128 FP32 lanes x 2 x {pk['sm_max_mhz']:.0f} MHz",
            "per_launch": {"flops": fl_per, "bytes": by_per, "avg_ns": avg_ns, "launches": dom_n, "source": timing_src},
            "share_of_step": dom_ns / (ms_per_step * 1e6) if world == 1 else None,  # (one instrumented round)
            "share_of_step_serialized": (op_stats["op_ns"][dominant] / max(1, op_stats["round_ns"])) if op_stats else None}

    # ---- e2e: through the public API with HOST buffers (H2D of shards + global weights, D2H of the result)
    e2e = None
    if not args.no_e2e:
        pin_g = torch.tensor(synth.init_weights(wl.model)).pin_memory()
        pin_o = torch.empty_like(pin_g).pin_memory()
        pinned = {cid: (torch.from_numpy(x).pin_memory(), torch.from_numpy(y).pin_memory())
                  for cid, (x, y) in shards.items()}
        h2d = sum(int(x.numel()) + 4 * int(y.numel()) for x, y in pinned.values()) + 4 * g.numel()
        d2h = 4 * g.numel() + 8
        barrier()
        t0 = time.perf_counter()
        for k in range(args.steps):
            pb.protea_register_shards(sim.ctx, [(cid, x.numpy(), y.numpy()) for cid, (x, y) in pinned.items()])
            plan, _ = pb.protea_plan(profiles, caps)
            sim.run_round(all_clients, plan, pin_g, pin_o, lr=wl.lr, seed=wl.seed, rnd=rnd)
            pin_g, pin_o = pin_o, pin_g
            rnd += 1
        barrier()
        e2e_s = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=sim.device)
        if world > 1:
            dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
        e2e = {"value": round_steps * args.steps / float(e2e_s.item()), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}

    # ---- CPU oracle baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        frac = 0.05 if args.config == 2 else 0.02
        s, w, cores = oracle_sample(wl, frac=frac)
        cpu = {"value": s / w, "unit": UNIT, "cores": cores, "kind": "oracle",
               "sample": f"first ceil({frac}*S_k) local steps of each of the {len(wl.clients)} config{args.config} "
                         f"clients ({s} client-steps, {w:.1f} s wall), float64 numpy oracle, one client per process"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": args.scaling, "vs_baseline": None, "dtype": dtype, "data": "synthetic",
                "config": config_block(wl, world, dtype, args.config, args.scaling),
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
                "clocks": clk,
                "detail": {"round_tflops": sum(int(f["flops"]) for f in foot) / (ms_per_step / 1e3) / 1e12,
                           "iterations_per_round": int(st["iterations"]), "host_wall_s": host_s,
                           "probe_s": probe_s, "util_monitor": host_mon, "probe_step_ns": sorted({int(p["step_ns"]) for p in probe}),
                           "op_ms_warmup": {pb.OPC_NAMES[i]: op_stats["op_ns"][i] / 1e6 for i in range(pb.N_OPC)
                                            if op_stats and op_stats["op_ns"][i]},
                           # every op class of the serialised warm-up round against both roofs (tensor-pipe and
                           # HBM utilisation = achieved algorithmic FLOP/s, bytes/s over the measured peaks)
                           "op_util_warmup": {pb.OPC_NAMES[i]: {
                               "ms": op_stats["op_ns"][i] / 1e6,
                               "tflops": op_stats["op_flops"][i] / op_stats["op_ns"][i] / 1e3,
                               "gbs": op_stats["op_bytes"][i] / op_stats["op_ns"][i],
                               "tensor_frac": op_stats["op_flops"][i] / op_stats["op_ns"][i] / 1e3 / pk["bf16_sus"],
                               "hbm_frac": op_stats["op_bytes"][i] / op_stats["op_ns"][i] / pk["hbm"]}
                               for i in range(pb.N_OPC) if op_stats and op_stats["op_ns"][i]},
                           "loss_mean_last_round": st["loss_sum"] / max(1, st["client_steps"])}}
        print(json.dumps(line), flush=True)
    sim.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
