"""Plain, slow, obviously-correct CPU oracle for the Protea hot path.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s `cpu_baseline` / `--impl reference` legs may import anything
under `oracle/`.  The product path (`paper_2207_01053_b200`, the C-ABI
library) never imports, links or executes it, and it shares no code with it.

What it computes (PAPER.md = /root/reference/PAPER.md, line numbers "P:n"):

* `fedavg`   — vanilla FedAvg, w' = sum_k n_k w_k / sum_k n_k
               (§3.3 "vanilla Federated Averaging (FedAvg)", McMahan P:83).
* `sgd`      — each client's local SGD epochs in float64 ("finished
               training", P:304 models; recipe = DESIGN.md reading R10).
* `profiler` — per-client profile: S_k, FLOPs_k, exact arena HWM, Eq. (1)
               ratio (Table 1 VRAM / CUDA_time; Eq. (1)).
* `planner`  — profile-driven packing: LPT partition across GPUs, then the
               VCE's FIFO admission "with as many clients running concurrently
               as the available system resources can hold" (§3.2 (3)-(4)).
* `round`    — one federated round: local SGD for every sampled client, then
               FedAvg per shape group (§3.3 configure_fit / aggregate_fit).
* `evaluate` — forward-only evaluation of a model on a client's validation
               split: loss sum and first-max accuracy (§4.1).

Everything is float64 numpy (floating point) or Python ints (integers).
Pins (tests/test_oracle_*.py) tie each function to something other than
itself: closed forms, the paper's / SPEC's worked examples, brute force,
finite differences and torch-CPU float64 autograd.  Device time is the only
profile field with "parity unpinned" (it is a measurement).
"""
