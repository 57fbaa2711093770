"""Convenience wrapper sequencing the C-ABI calls of one rank (marshalling only).

PyTorch provides the device memory (the arena block and global-weight
tensors) and the stream; every computation happens inside libprotea.so.
"""
from __future__ import annotations

import numpy as np

from . import (PREC_FP32, POLICY_PROFILED, ORDER_ASC_ID, clients_array, protea_evaluate, protea_evaluate_round,
               protea_finalize, protea_init, protea_plan, protea_profile_clients, protea_register_model,
               protea_register_shards, protea_register_val_shards, protea_run_round)


class Simulation:
    """One rank's context: arena (torch uint8 block) + stream + registered models/shards."""

    def __init__(self, device=0, precision=PREC_FP32, arena_bytes=1 << 30, rank=0, world=1, nccl_id=None,
                 stream=None):
        import torch
        self.torch = torch
        self.device = torch.device("cuda", device)
        self.arena = torch.empty(int(arena_bytes), dtype=torch.uint8, device=self.device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.precision = precision
        self.ctx = protea_init(device=device, rank=rank, world=world, precision=precision, arena=self.arena,
                               arena_bytes=int(arena_bytes), stream=self.stream, nccl_id=nccl_id)
        self.models = []  # (model_id, n_params, offset)
        self.n_params = 0

    def register_model(self, arch, width_q=4, classes=10, H=32, W=32, C=3):
        mid, npar = protea_register_model(self.ctx, arch, width_q, classes, H, W, C)
        self.models.append((mid, npar, self.n_params))
        self.n_params += npar
        return mid

    def register_shards(self, shards):
        protea_register_shards(self.ctx, shards)

    def register_val_shards(self, shards):
        protea_register_val_shards(self.ctx, shards)

    def evaluate_round(self, clients, global_w):
        """Evaluate round: per-client (loss_sum, correct, n) records and their totals."""
        return protea_evaluate_round(self.ctx, clients, global_w)

    @staticmethod
    def clients(rows):
        return clients_array(rows)

    def profile(self, clients):
        return protea_profile_clients(self.ctx, clients)

    def plan(self, profiles, caps=None, policy=POLICY_PROFILED, order=ORDER_ASC_ID, margin_permille=1000,
             max_active=0):
        caps = [self.arena.numel()] if caps is None else caps
        return protea_plan(profiles, caps, policy, order, margin_permille, max_active)

    def run_round(self, clients, plan, global_in, global_out=None, lr=0.05, seed=0, rnd=0, shuffle=True,
                  measured=False, time_ops=0, partial_only=False, serialize=False, observe_hwm=False, trace=None):
        if global_out is None:
            global_out = self.torch.empty_like(global_in)
        r = protea_run_round(self.ctx, clients, plan, global_in, global_out, lr, seed, rnd, shuffle, measured,
                             time_ops, partial_only, serialize, observe_hwm, trace)
        return global_out, r

    def evaluate(self, model_id, weights, x, y):
        """Forward-only evaluation (loss_sum, correct, n) of `weights` of model `model_id` on (x, y)."""
        return protea_evaluate(self.ctx, model_id, weights, x, y)

    def run_round_guarded(self, clients, profiles, global_in, global_out=None, caps=None, policy=POLICY_PROFILED,
                          max_retries=8, backoff=2.0, **kw):
        """Plan from ``profiles`` and run; if the library rejects the plan because a client's slot is smaller
        than its high-water mark (stale or hand-made profile), apply the SPEC out-of-memory backoff to that
        client (peak x ``backoff``, clamped to the capacity) and re-plan.  Returns (out, stats, profiles)."""
        from . import ERR_OOM, ERR_PLAN, ProteaError
        from .monitor import failed_client, oom_backoff
        caps = [self.arena.numel()] if caps is None else caps
        for _ in range(max_retries + 1):
            plan, _mk = self.plan(profiles, caps=caps, policy=policy)
            try:
                out, st = self.run_round(clients, plan, global_in, global_out, **kw)
                return out, st, profiles
            except ProteaError as e:
                cid = failed_client(str(e))
                if e.code not in (ERR_OOM, ERR_PLAN) or cid is None or "HWM" not in str(e):
                    raise
                profiles = oom_backoff(profiles, cid, backoff, max(caps))
        raise RuntimeError("run_round_guarded: out-of-memory backoff did not converge")

    def close(self):
        if self.ctx is not None:
            protea_finalize(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def concat_globals(arrays):
    return np.concatenate([np.asarray(a, dtype=np.float32) for a in arrays])
