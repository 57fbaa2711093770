"""World-size-2 CPU tests (gloo) of the N>1 host logic: every rank computes the
identical integer plan from the same profiles (LPT partition by FLOPs, reading
R5), runs only its own clients, and the per-rank FedAvg partials
sum_k n_k (w_k - w_g) summed across ranks and finalised as w_g + acc / N equal
the single-process FedAvg.  Local SGD here is the oracle's (test
infrastructure); the GPU path runs the same decomposition through
protea_run_round(partial_only) + protea_round_finalize (tests/test_gpu_parity.py)
and through NCCL in bench.py under torchrun."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synth
        import paper_2207_01053_b200 as pb
        from oracle import sgd

        wl = synth.build_workload(3, k=12, samples=6, epochs=1)
        prof = np.zeros(len(wl.clients), dtype=pb.PROFILE_DT)
        for i, c in enumerate(wl.clients):
            pk, st, fl = pb.protea_client_footprint(pb.MODEL_CNN, 4, 10, 32, 32, 3, c.n, c.batch, c.epochs, 0)
            prof[i] = (c.id, pk, st, fl, 0, 0, 0, 1, 0)
        plan, mk = pb.protea_plan(prof, [1 << 30] * world)
        # plan agreement: identical bytes on every rank
        h = torch.tensor(np.frombuffer(plan.tobytes(), dtype=np.uint8).astype(np.int64))
        hs = [torch.zeros_like(h) for _ in range(world)]
        dist.all_gather(hs, h)
        same = all(torch.equal(hs[0], x) for x in hs)
        # the library's agreement check (protea_run_round, world > 1): max over ranks of (h, ~h) == (h, ~h)
        cl = pb.clients_array([(c.id, 0, c.batch, c.epochs) for c in wl.clients])
        ph = pb.protea_plan_hash(cl, plan)
        hv = torch.tensor([ph >> 1, (~ph & (2**64 - 1)) >> 1], dtype=torch.int64)  # int64-safe halves
        dist.all_reduce(hv, op=dist.ReduceOp.MAX)
        agree = int(hv[0]) == ph >> 1 and int(hv[1]) == (~ph & (2**64 - 1)) >> 1
        bad = plan.copy()
        if rank == 1:
            bad[0]["admit"] += 1  # a rank with a different plan
        bh = pb.protea_plan_hash(cl, bad)
        bv = torch.tensor([bh >> 1, (~bh & (2**64 - 1)) >> 1], dtype=torch.int64)
        dist.all_reduce(bv, op=dist.ReduceOp.MAX)
        disagree = not (int(bv[0]) == bh >> 1 and int(bv[1]) == (~bh & (2**64 - 1)) >> 1)
        same = same and agree and disagree
        mine = [c for c, a in zip(wl.clients, plan) if int(a["gpu"]) == rank]
        w0 = synth.init_weights(wl.model).astype(np.float64)
        acc = np.zeros_like(w0)
        for c in mine:
            wk, _ = sgd.local_sgd(w0, c.model, 4, 10, *wl.shards[c.id], c.batch, c.epochs, 0.05, wl.seed, 0, c.id)
            acc += c.n * (wk - w0)
        t = torch.tensor(acc)
        dist.all_reduce(t)
        N = sum(c.n for c in wl.clients)
        q.put((rank, same, [c.id for c in mine], (w0 + t.numpy() / N)))
    finally:
        dist.destroy_process_group()


def test_two_rank_plan_and_fedavg_decomposition():
    import synth
    from oracle import round as orr
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert all(r[1] for r in res)
    ids0, ids1 = set(res[0][2]), set(res[1][2])
    assert ids0 and ids1 and not (ids0 & ids1)
    wl = synth.build_workload(3, k=12, samples=6, epochs=1)
    assert ids0 | ids1 == {c.id for c in wl.clients}
    ref = orr.run_round(wl.clients, wl.shards, {4: synth.init_weights(wl.model)}, 0.05, wl.seed, 0)[4]
    for r in res:
        assert np.linalg.norm(r[3] - ref) <= 1e-13 * np.linalg.norm(ref)
    assert np.array_equal(res[0][3], res[1][3])
