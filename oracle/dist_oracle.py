"""Per-rank (one process per worker) restatement of the ACCO round over
torch.distributed — TEST INFRASTRUCTURE ONLY.

This is the decomposition the B200 engine runs in NCCL mode
(paper_2406_02613_b200/csrc/engine.cu, Trainer::launch_phase), restated in
fp64 on CPU so the multi-process host logic can be tested with the gloo
backend (world size 2) on a machine without GPUs:

* each rank computes only its own worker's stage bundles (protocols.cpp:554-600);
* counts all-reduce (collectives.cpp:48-53);
* reduce-scatter of the **owner-padded** send buffer (chunk = ceil(dim/N),
  chunk w = shard_partition range w + zero pad) — NCCL needs equal counts;
* the rank's own shard: estimate on a transient state copy / commit on the
  persistent state (protocols.cpp:647-670), then all-gather + unpack.

With two ranks the gloo sums a+b are bitwise equal to the reference's
ascending-worker fold, so the result must equal the single-process oracle
(accosim_oracle.run_acco) bitwise.
"""
from __future__ import annotations

import math
from dataclasses import replace

import numpy as np

from . import accosim_oracle as O


def padded_layout(dim: int, n: int):
    ranges = O.shard_partition(dim, n)
    chunk = math.ceil(dim / n) if n else 0
    return ranges, chunk


def pack(flat: np.ndarray, ranges, chunk: int) -> np.ndarray:
    out = np.zeros(chunk * len(ranges))
    for w, (lo, hi) in enumerate(ranges):
        out[w * chunk:w * chunk + (hi - lo)] = flat[lo:hi]
    return out


def unpack(padded: np.ndarray, ranges, chunk: int, dim: int) -> np.ndarray:
    out = np.zeros(dim)
    for w, (lo, hi) in enumerate(ranges):
        out[lo:hi] = padded[w * chunk:w * chunk + (hi - lo)]
    return out


def run_acco_rank(dist, grad_fn, theta0: np.ndarray, cfg: O.OptimizerConfig, sim: O.SimConfig, t_updates: int,
                  schedule=None):
    """ACCO on this rank (rank = worker id). Returns (theta_history, estimate_history)."""
    import torch

    rank, world = dist.get_rank(), dist.get_world_size()
    assert world == sim.n_workers
    if cfg.total_steps == 0:
        cfg = replace(cfg, total_steps=t_updates)
    if schedule is None:
        schedule = O.floor_schedule(t_updates, world, sim.n_grad_accumulation)
    dim = theta0.shape[0]
    ranges, chunk = padded_layout(dim, world)
    lo, hi = ranges[rank]
    state = O.OptimizerState.for_range(cfg, lo, hi)
    theta = np.array(theta0, dtype=np.float64, copy=True)
    estimate = theta.copy()
    th_hist, est_hist = [theta.copy()], [estimate.copy()]

    def counts_ar(n):
        t = torch.tensor([n], dtype=torch.int64)
        dist.all_reduce(t)
        return int(t.item())

    def rs(grad_sum):
        buf = torch.from_numpy(pack(grad_sum, ranges, chunk))
        dist.all_reduce(buf)  # gloo: reduce-scatter as all-reduce + owner slice
        return buf.numpy()[rank * chunk:rank * chunk + (hi - lo)].copy()

    def ag(shard):
        mine = torch.zeros(chunk, dtype=torch.float64)
        mine[:hi - lo] = torch.from_numpy(shard)
        parts = [torch.zeros(chunk, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, mine)
        return unpack(torch.cat(parts).numpy(), ranges, chunk, dim)

    def stage(params, rnd, tag, k):
        b = O.Bundle()
        for j in range(k):
            g, n, _ = grad_fn(params, O.make_batch_stream(sim, rnd, tag, rank, j))
            b.add(g, n)
        return b

    for t in range(t_updates):
        mb_est, mb_main = schedule[t]
        # phase 2t: estimate
        b = stage(theta0, 0, O.TAG_INIT, 1) if t == 0 else stage(estimate, t, O.TAG_ESTIMATE, mb_est[rank])
        total_est = counts_ar(b.samples)
        g_est = rs(b.grad_sum)
        _, est_shard = O.opt_step(state.copy(), theta[lo:hi], g_est * (1.0 / float(total_est)), cfg)
        estimate = ag(est_shard)
        # phase 2t+1: commit
        b = stage(theta, t, O.TAG_MAIN, mb_main[rank])
        total = counts_ar(b.samples)
        g = rs(b.grad_sum)
        state, new_shard = O.opt_step(state, theta[lo:hi], (g + g_est) * (1.0 / float(total + total_est)), cfg)
        theta = ag(new_shard)
        th_hist.append(theta.copy())
        est_hist.append(estimate.copy())
    return th_hist, est_hist
