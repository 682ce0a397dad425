"""Peer fabric at world size 2 and 3 on the one GPU gpurun provides: one
process per rank (all on device 0) exchange CUDA-IPC handles over gloo and run
the ACCO / ZeRO-1 comm phases through the fused fold + AdamW + replica-store
kernel, with the cross-process device-flag counts and barriers — the
multi-rank path of the N-GPU NVLink deployment, minus NVLink. Every rank's
parameter history must match the fp64 oracle's 2-worker run (rel <= 1e-5 per
update) and the two ranks' replicas must agree bitwise. The runs enable the
debug replica check (check_replicas: hashes of both replicas exchanged and
compared after every comm phase, the reference's check_replicas,
protocols.cpp:208-212); a corrupted replica must fail every rank with the
reference's logic_error."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MINI = dict(vocab=64, d_model=32, n_layer=2, n_head=2, seq_len=16, n_samples=32, data_seed=3)

WORKER = r'''
import os, sys
import numpy as np
sys.path.insert(0, os.environ["ROOT"])
rank, world, port, method, out, vocab = (int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4], sys.argv[5],
                                         int(sys.argv[6]))
hetero = len(sys.argv) > 7 and sys.argv[7] == "hetero"
import torch
import torch.distributed as dist
torch.cuda.set_device(0)
dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
from paper_2406_02613_b200 import api
MINI = dict(vocab=vocab, d_model=32, n_layer=2, n_head=2, seq_len=16, n_samples=32, data_seed=3)
peer = api.PeerComm(rank=rank, world=world, device=0)
opt = api.OptimizerConfig(kind="adamw", learning_rate=6e-4, weight_decay=0.1, adam_beta2=0.95, scheduler="cosine")
if hetero:  # rank 0 is 4x slower; the adaptive schedule lets the fast rank accumulate more
    sim = api.SimConfig(n_workers=world, batch_size=4, n_grad_accumulation=1, master_seed=7, eval_every=1,
                        schedule="adaptive", worker_multipliers=[4.0] + [1.0] * (world - 1))
else:
    sim = api.SimConfig(n_workers=world, batch_size=4, n_grad_accumulation=2, master_seed=7, eval_every=1,
                        check_replicas=True)
try:
    tr = api.run_protocol(method, api.LMConfig(**MINI, precision="fp32", max_batch=4), opt, sim, 3, comm=peer)
except api.LogicError as e:
    print("LOGIC_ERROR", e, flush=True)
    sys.exit(5)
np.save(os.path.join(out, f"th{rank}.npy"), np.array(tr.theta_history))
np.save(os.path.join(out, f"est{rank}.npy"), np.array(tr.estimate_history))
np.save(os.path.join(out, f"samples{rank}.npy"), np.array([r.samples_cum for r in tr.records]))
np.save(os.path.join(out, f"counts{rank}.npy"), np.array([[r.mb_estimate, r.mb_main] for r in tr.records]))
dist.destroy_process_group()
print("rank", rank, "ok", flush=True)
'''


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("method,world,vocab", [("acco", 2, 64), ("zero1", 2, 64), ("dpu", 2, 64), ("wp", 2, 64),
                                                ("acco", 3, 63)])  # world 3, Psi = 28000: ragged shards
def test_peer_fabric_multi_rank_one_gpu(cuda, tmp_path, method, world, vocab):
    from oracle import accosim_oracle as O
    from oracle import gpt_oracle as G

    port = str(_free_port())
    env = dict(os.environ, ROOT=ROOT)
    procs = [subprocess.Popen([sys.executable, "-c", WORKER, str(r), str(world), port, method, str(tmp_path), str(vocab)],
                              env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True) for r in range(world)]
    outs = []
    try:
        for p in procs:
            outs.append(p.communicate(timeout=240)[0])
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    for p, o in zip(procs, outs):
        assert p.returncode == 0, o[-3000:]
    th = [np.load(tmp_path / f"th{r}.npy") for r in range(world)]
    for r in range(1, world):
        assert np.array_equal(th[0], th[r])  # every rank holds the same replica
    gc = G.GPTConfig(**{**MINI, "vocab": vocab})
    prob = G.LMProblem(gc)
    th0 = G.default_theta0(gc, 7).astype(np.float32).astype(np.float64)
    ocfg = O.OptimizerConfig(kind="adamw", learning_rate=6e-4, weight_decay=0.1, adam_beta2=0.95,
                             scheduler="cosine")
    ref = O.run_method(method, (lambda t, s: prob.stochastic_grad(t, s, 4)), th0, ocfg, O.SimConfig(world, 4, 2, False, 7),
                       3, eval_fn=prob.value_and_grad)
    for t in range(3):
        a, b = th[0][t + 1], ref.theta_history[t + 1]
        assert np.linalg.norm(a - b) / np.linalg.norm(b) <= 1e-5, t
    assert list(np.load(tmp_path / "samples0.npy")) == [r.samples_cum for r in ref.records]


def test_peer_fabric_heterogeneous_adaptive_two_ranks(cuda, tmp_path):
    """The paper's heterogeneous setting on the multi-rank path: rank 0 is 4x
    slower (HeterogeneityProfile multiplier -> measured throttle), the adaptive
    schedule decides each stage's length from live phase completion, and the
    per-rank counts logged by the run, replayed on the fp64 oracle, reproduce
    every rank's parameter trajectory."""
    from oracle import accosim_oracle as O
    from oracle import gpt_oracle as G

    world, vocab, T = 2, 64, 3
    port = str(_free_port())
    env = dict(os.environ, ROOT=ROOT)
    procs = [subprocess.Popen([sys.executable, "-c", WORKER, str(r), str(world), port, "acco", str(tmp_path), str(vocab),
                               "hetero"], env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
             for r in range(world)]
    outs = []
    try:
        for p in procs:
            outs.append(p.communicate(timeout=240)[0])
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    for p, o in zip(procs, outs):
        assert p.returncode == 0, o[-3000:]
    th = [np.load(tmp_path / f"th{r}.npy") for r in range(world)]
    assert np.array_equal(th[0], th[1])
    cnt = [np.load(tmp_path / f"counts{r}.npy") for r in range(world)]  # per rank: [T][2][its own count]
    sched = [([int(cnt[w][t][0][0]) for w in range(world)], [int(cnt[w][t][1][0]) for w in range(world)])
             for t in range(T)]
    assert all(k >= 1 for est, main in sched for k in est + main)
    gc = G.GPTConfig(**{**MINI, "vocab": vocab})
    prob = G.LMProblem(gc)
    th0 = G.default_theta0(gc, 7).astype(np.float32).astype(np.float64)
    ocfg = O.OptimizerConfig(kind="adamw", learning_rate=6e-4, weight_decay=0.1, adam_beta2=0.95,
                             scheduler="cosine")
    ref = O.run_acco((lambda t, s: prob.stochastic_grad(t, s, 4)), th0, ocfg, O.SimConfig(world, 4, 1, False, 7), T,
                     schedule=sched, eval_fn=prob.value_and_grad)
    for t in range(T):
        a, b = th[0][t + 1], ref.theta_history[t + 1]
        assert np.linalg.norm(a - b) / np.linalg.norm(b) <= 1e-5, (t, sched)


def test_replica_check_catches_a_corrupted_rank(cuda, tmp_path):
    """ACCO_DEBUG_CORRUPT=1,1: rank 1 perturbs its theta replica after comm
    phase 1; the replica hashes disagree and BOTH ranks fail with
    "protocol: parameter divergence across workers" (no hang)."""
    world = 2
    port = str(_free_port())
    env = dict(os.environ, ROOT=ROOT, ACCO_DEBUG_CORRUPT="1,1")
    procs = [subprocess.Popen([sys.executable, "-c", WORKER, str(r), str(world), port, "acco", str(tmp_path), "64"],
                              env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True) for r in range(world)]
    outs = []
    try:
        for p in procs:
            outs.append(p.communicate(timeout=240)[0])
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    for p, o in zip(procs, outs):
        assert p.returncode == 5, o[-3000:]
        assert "parameter divergence across workers" in o
