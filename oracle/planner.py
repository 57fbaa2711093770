"""Profile-driven packing of clients onto GPU memory slots (oracle; test infra only).

PAPER.md §3.2: the Virtual Client Engine (1) reads each client's
resources, (2) assigns them, (3) "Ray will schedule the clients in the round in
a FIFO fashion with as many clients running concurrently as the available
system resources can hold", (4) "once a client has finished training, the
resources get freed and another client in the round will be spawned".
§3.4 Eq. (1) turns the measured VRAM into the resource request.
§5: memory does not predict compute -> the multi-GPU split balances
FLOP work (reading R5).

Algorithm (SURVEY §8(c).4, step by step; integer arithmetic only):

 0. validate: duplicate id -> INVALID; slot_k = align256(ceil(peak_k *
    margin_permille / 1000)); slot_k > max_g C_g -> NO_CAPACITY.  Policy
    STATIC (the paper's "original setup", one client per whole GPU):
    slot_k := C_g of the GPU it is placed on.
 1. partition (LPT): sort by (W_k desc, id asc); give each client to the GPU
    with minimal (load_g, g) among GPUs with C_g >= slot_k; load_g += W_k.
 2. per GPU, admission replay in integer step time: queue ordered ASC_ID
    (paper FIFO) or DESC_STEPS (S_k desc, id asc); free list {[0, C_g)}; t=0;
    loop: admit heads while |A| < max_active and the head fits the lowest-
    offset free gap (strict head-of-line blocking, SPEC D-6); stop if nothing
    is active and the queue is empty; else t = min release, release every
    client with release == t in ascending id, coalescing gaps.
 3. output per client (ascending id): gpu, offset, slot, admit, release,
    q1024 = ceil(1024 slot / sum C); per GPU makespan = max release.
"""
from __future__ import annotations

ALIGN = 256
ASC_ID, DESC_STEPS = 0, 1
PROFILED, STATIC = 0, 1


class PlanError(ValueError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def align_up(x, a=ALIGN):
    return (x + a - 1) // a * a


def plan(clients, caps, policy=PROFILED, order=ASC_ID, margin_permille=1000, max_active=0):
    """clients: list of dicts with id, peak_bytes, steps, flops.  caps: [C_g].

    Returns (assignments sorted by id: list of dicts, makespans list)."""
    G = len(caps)
    if G == 0 or any(c <= 0 for c in caps):
        raise PlanError("INVALID", "cluster needs >= 1 GPU with capacity > 0")
    if margin_permille < 1000:
        raise PlanError("INVALID", "margin_permille < 1000")
    if len(clients) == 0:
        raise PlanError("INVALID", "no clients")
    seen = set()
    for c in clients:
        if c["id"] in seen:
            raise PlanError("INVALID", f"duplicate client id {c['id']}")
        seen.add(c["id"])
        if c["steps"] <= 0 or c["peak_bytes"] <= 0:
            raise PlanError("INVALID", f"client {c['id']}: steps/peak_bytes must be > 0")
    total_cap = sum(caps)
    maxcap = max(caps)
    slot = {}
    for c in clients:
        s = align_up(-(-c["peak_bytes"] * margin_permille // 1000))
        if s > maxcap:
            raise PlanError("NO_CAPACITY", f"client {c['id']}: slot {s} exceeds every GPU")
        slot[c["id"]] = s

    # 1. LPT partition
    load = [0] * G
    members = [[] for _ in range(G)]
    for c in sorted(clients, key=lambda c: (-c["flops"], c["id"])):
        best = None
        for g in range(G):
            if caps[g] >= slot[c["id"]] and (best is None or load[g] < load[best]):
                best = g
        load[best] += c["flops"]
        members[best].append(c)

    # 2. per-GPU admission replay
    out = {}
    makespans = [0] * G
    for g in range(G):
        C = caps[g]
        if order == ASC_ID:
            queue = sorted(members[g], key=lambda c: c["id"])
        else:
            queue = sorted(members[g], key=lambda c: (-c["steps"], c["id"]))
        free = [[0, C]]  # sorted, coalesced [offset, length]
        active = {}  # id -> (offset, slot, release)
        t = 0
        qi = 0
        while True:
            while qi < len(queue) and (max_active <= 0 or len(active) < max_active):
                h = queue[qi]
                s = C if policy == STATIC else slot[h["id"]]
                gap = next((i for i, (o, ln) in enumerate(free) if ln >= s), None)
                if gap is None:
                    break
                o, ln = free[gap]
                if ln == s:
                    free.pop(gap)
                else:
                    free[gap] = [o + s, ln - s]
                active[h["id"]] = (o, s, t + h["steps"])
                out[h["id"]] = dict(id=h["id"], gpu=g, offset=o, slot=s, admit=t,
                                    release=t + h["steps"], q1024=-(-1024 * s // total_cap))
                qi += 1
            if not active and qi == len(queue):
                break
            if not active:
                raise PlanError("PLAN", "head client can never be admitted")
            t = min(r for (_, _, r) in active.values())
            for cid in sorted(k for k, v in active.items() if v[2] == t):
                o, s, _ = active.pop(cid)
                free.append([o, s])
                free.sort()
                merged = []
                for fo, fl in free:
                    if merged and merged[-1][0] + merged[-1][1] == fo:
                        merged[-1][1] += fl
                    else:
                        merged.append([fo, fl])
                free = merged
        makespans[g] = max((out[c["id"]]["release"] for c in members[g]), default=0)
        assert free == [[0, C]]
    return [out[k] for k in sorted(out)], makespans
