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


def acco_round_sample(cfg: G.GPTConfig, batch: int = 1, seed: int = 1):
    """Returns dict(t_microbatch, t_phases, tokens_per_s, sample)."""
    th = G.default_theta0(cfg, seed)
    tok = G.dataset(cfg)
    idx = O.sample_indices(O.derive(seed, 0, 0, 2, 0), batch, cfg.n_samples)
    t0 = time.perf_counter()
    loss, g = G.loss_and_grad(cfg, th, tok[idx])
    t_mb = time.perf_counter() - t0
    ocfg = O.OptimizerConfig(kind="adamw", learning_rate=6e-4, weight_decay=0.1, adam_beta2=0.95,
                             scheduler="cosine", total_steps=100)
    st = O.OptimizerState.for_range(ocfg, 0, th.shape[0])
    t0 = time.perf_counter()
    mean = g * (1.0 / batch)
    _, est = O.opt_step(st.copy(), th, mean, ocfg)      # estimate (transient)
    mean2 = (g + g) * (1.0 / (2 * batch))
    st, th = O.opt_step(st, th, mean2, ocfg)             # commit
    t_ph = time.perf_counter() - t0
    tokens = 2 * batch * cfg.seq_len
    return {"t_microbatch_s": t_mb, "t_phases_s": t_ph, "tokens_per_s": tokens / (2 * t_mb + t_ph),
            "loss": loss, "cores": os.cpu_count(),
            "sample": f"1 ACCO update (k=1, 1 worker) at B={batch} seq x {cfg.seq_len} tokens: 2 micro-batch "
                      f"fwd/bwd (timed once, x2) + estimate/commit AdamW over {th.shape[0]} params, fp64 numpy"}
