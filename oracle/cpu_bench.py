"""CPU baseline timing of the ACCO round — TEST/BENCH INFRASTRUCTURE ONLY.

Times the fp64 oracle port (numpy, all host threads through BLAS) on a bounded
sample of the bench workload: one micro-batch fwd/bwd of B sequences, plus one
ACCO optimizer phase pair (estimate on a transient state + commit) over all Psi
parameters, composed into tokens/s for an update of 2 micro-batches
(k = 1, one worker): tokens/s = 2*B*T / (2*t_microbatch + t_phases).
Called only by bench.py's cpu_baseline leg and `--impl reference` arm.
"""
from __future__ import annotations

import os
import time

import numpy as np

from . import accosim_oracle as O
from . import gpt_oracle as G


def blas_threads() -> int:
    """Threads numpy's BLAS actually runs with (the cores the CPU arm uses)."""
    try:
        from threadpoolctl import threadpool_info

        n = [i.get("num_threads", 0) for i in threadpool_info() if i.get("user_api") == "blas"]
        if n:
            return int(max(n))
    except Exception:  # noqa: BLE001
        pass
    return os.cpu_count() or 1


def acco_round_sample(cfg: G.GPTConfig, batch: int = 1, seed: int = 1):
    """One ACCO update (k = 1, one worker): the estimate-stage and main-stage
    micro-batches (each B sequences, fwd + bwd, both timed) and the estimate /
    commit optimizer phases over all Psi parameters. Returns dict(t_microbatch
    (mean of the two), t_phases, tokens_per_s, cores, sample)."""
    th = G.default_theta0(cfg, seed)
    tok = G.dataset(cfg)
    ocfg = O.OptimizerConfig(kind="adamw", learning_rate=6e-4, weight_decay=0.1, adam_beta2=0.95,
                             scheduler="cosine", total_steps=100)
    st = O.OptimizerState.for_range(ocfg, 0, th.shape[0])
    t_start = time.perf_counter()
    idx = O.sample_indices(O.derive(seed, 0, 0, 1, 0), batch, cfg.n_samples)  # bootstrap / estimate stage
    t0 = time.perf_counter()
    loss, g_est = G.loss_and_grad(cfg, th, tok[idx])
    t_mb0 = time.perf_counter() - t0
    t0 = time.perf_counter()
    _, est = O.opt_step(st.copy(), th, g_est, ocfg)      # estimate phase (transient state)
    t_ph = time.perf_counter() - t0
    idx = O.sample_indices(O.derive(seed, 0, 0, 2, 0), batch, cfg.n_samples)  # main stage
    t0 = time.perf_counter()
    _, g_main = G.loss_and_grad(cfg, th, tok[idx])
    t_mb1 = time.perf_counter() - t0
    t0 = time.perf_counter()
    st, th = O.opt_step(st, th, (g_main * batch + g_est * batch) * (1.0 / (2 * batch)), ocfg)  # commit phase
    t_ph += time.perf_counter() - t0
    total = time.perf_counter() - t_start
    tokens = 2 * batch * cfg.seq_len
    return {"t_microbatch_s": 0.5 * (t_mb0 + t_mb1), "t_phases_s": t_ph, "tokens_per_s": tokens / total,
            "loss": loss, "cores": blas_threads(),
            "sample": f"1 ACCO update (k=1, 1 worker) at B={batch} seq x {cfg.seq_len} tokens: 2 micro-batch "
                      f"fwd/bwd + estimate/commit AdamW over {th.shape[0]} params, fp64 numpy (BLAS threads)"}
