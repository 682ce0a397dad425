"""World-size-2 gloo test (CPU) of the multi-process ACCO decomposition the
B200 engine uses in NCCL mode: per-rank stages, counts all-reduce, owner-padded
reduce-scatter, per-shard estimate/commit, all-gather — checked bitwise against
the single-process oracle (itself bitwise equal to the reference)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import accosim_oracle as O
from oracle import dist_oracle as D


def _problem(dim=7, seed=3):
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((dim, dim))
    a = q @ q.T / dim + np.eye(dim)
    b = rng.standard_normal(dim)
    return a, b


def _grad_fn(a, b, sigma=0.3):
    def f(theta, stream):
        s = O.Stream(stream)
        g = a @ theta - b + sigma * np.array([s.gaussian() for _ in range(len(b))])
        return g, 4, 0.0
    return f


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, dim, kind, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a, b = _problem(dim)
    cfg = O.OptimizerConfig(kind=kind, learning_rate=0.05, weight_decay=0.01, adam_beta2=0.95, scheduler="cosine")
    sim = O.SimConfig(n_workers=world, batch_size=4, n_grad_accumulation=2, master_seed=9)
    sched = [([1] * world, [2, 3][:world])] + [([2, 1][:world], [3, 2][:world])] * 4
    th, est = D.run_acco_rank(dist, _grad_fn(a, b), np.ones(dim), cfg, sim, 5, schedule=sched)
    np.save(os.path.join(out_dir, f"th{rank}.npy"), np.array(th))
    np.save(os.path.join(out_dir, f"est{rank}.npy"), np.array(est))
    dist.destroy_process_group()


@pytest.mark.parametrize("dim,kind", [(7, "adamw"), (8, "sgd"), (1, "adam")])
def test_two_rank_acco_matches_single_process_oracle(tmp_path, dim, kind):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), dim, kind, str(tmp_path)), nprocs=world, join=True)
    a, b = _problem(dim)
    cfg = O.OptimizerConfig(kind=kind, learning_rate=0.05, weight_decay=0.01, adam_beta2=0.95, scheduler="cosine")
    sim = O.SimConfig(n_workers=world, batch_size=4, n_grad_accumulation=2, master_seed=9)
    sched = [([1] * world, [2, 3])] + [([2, 1], [3, 2])] * 4
    ref = O.run_acco(_grad_fn(a, b), np.ones(dim), cfg, sim, 5, schedule=sched)
    for r in range(world):
        th = np.load(tmp_path / f"th{r}.npy")
        est = np.load(tmp_path / f"est{r}.npy")
        for t in range(6):  # every rank holds identical replicas, equal to the oracle bitwise
            assert th[t].tolist() == ref.theta_history[t].tolist(), (r, t)
            assert est[t].tolist() == ref.estimate_history[t].tolist(), (r, t)


def test_owner_padded_layout_roundtrip():
    for dim, n in [(7, 2), (10, 3), (17, 5), (3, 4), (437760, 2), (124439808 % 1000 + 1, 8)]:
        ranges, chunk = D.padded_layout(dim, n)
        x = np.arange(dim, dtype=np.float64) + 1
        p = D.pack(x, ranges, chunk)
        assert p.shape == (chunk * n,)
        assert np.array_equal(D.unpack(p, ranges, chunk, dim), x)
        for w, (lo, hi) in enumerate(ranges):  # padding is zero, owner chunk = its range
            assert np.all(p[w * chunk + (hi - lo):(w + 1) * chunk] == 0)
            assert np.array_equal(p[w * chunk:w * chunk + hi - lo], x[lo:hi])
