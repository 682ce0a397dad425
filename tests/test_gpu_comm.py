"""NCCL-mode engine and fabric helpers on one B200.

gpurun provides one GPU, so the NCCL communicator has world size 1 — the same
code path as N>1 (counts AR, RS into the shard, per-shard K6/K7, in-place AG)
minus the peer traffic. The multi-rank decomposition itself is covered on CPU
by tests/test_dist_gloo.py (world size 2)."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist

from oracle import accosim_oracle as O
from oracle import dist_oracle as D
from oracle import gpt_oracle as G
from paper_2406_02613_b200 import _lib, api

pytestmark = pytest.mark.gpu

MINI = dict(vocab=64, d_model=32, n_layer=2, n_head=2, seq_len=16, n_samples=32, data_seed=3)


def _s():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


@pytest.mark.parametrize("dim,n", [(10, 3), (17, 5), (3, 4), (437761, 8), (1001, 2)])
def test_pack_unpack_padded_match_layout(cuda, dim, n):
    ranges, chunk = D.padded_layout(dim, n)
    x = torch.arange(dim, dtype=torch.float32, device=cuda) + 1
    pad = torch.full((chunk * n,), -7.0, device=cuda)
    _lib.call("acco_pack_padded", C.c_void_p(x.data_ptr()), C.c_void_p(pad.data_ptr()), dim, n, _s())
    torch.cuda.synchronize()
    ref = D.pack(x.cpu().double().numpy(), ranges, chunk)
    assert np.array_equal(pad.cpu().double().numpy(), ref)
    for dt, dcode in ((torch.float32, _lib.DTYPE_F32), (torch.bfloat16, _lib.DTYPE_BF16)):
        back = torch.zeros(dim, dtype=dt, device=cuda)
        src = pad.to(dt)
        _lib.call("acco_unpack_padded", C.c_void_p(src.data_ptr()), C.c_void_p(back.data_ptr()), dim, n, dcode,
                  _s())
        torch.cuda.synchronize()
        assert torch.equal(back, x.to(dt))


@pytest.fixture(scope="module")
def nccl_comm(cuda):
    if not dist.is_initialized():
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    return api.Comm(rank=0, world=1, device=0)


def test_nccl_collectives_world1(cuda, nccl_comm):
    h = nccl_comm.handle
    x = torch.randn(1000, device=cuda)
    y = torch.empty_like(x)
    _lib.call("acco_reduce_scatter_f32", h, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), 1000, _s())
    cnt = torch.tensor([5], dtype=torch.int64, device=cuda)
    tot = torch.zeros(1, dtype=torch.int64, device=cuda)
    _lib.call("acco_all_reduce_i64", h, C.c_void_p(cnt.data_ptr()), C.c_void_p(tot.data_ptr()), 1, _s())
    z = torch.empty(1000, dtype=torch.bfloat16, device=cuda)
    xb = x.to(torch.bfloat16)
    _lib.call("acco_all_gather", h, C.c_void_p(xb.data_ptr()), C.c_void_p(z.data_ptr()), 1000, _lib.DTYPE_BF16, _s())
    torch.cuda.synchronize()
    assert torch.equal(y, x) and tot.item() == 5 and torch.equal(z, xb)
    assert _lib.lib().acco_comm_size(h) == 1 and _lib.lib().acco_comm_rank(h) == 0


@pytest.mark.parametrize("method", ["acco", "zero1", "ddp", "dpu", "wp"])
def test_engine_nccl_mode_matches_oracle(cuda, nccl_comm, method):
    opt = api.OptimizerConfig(kind="adamw", learning_rate=6e-4, weight_decay=0.1, adam_beta2=0.95,
                              scheduler="cosine")
    sim = api.SimConfig(n_workers=1, batch_size=4, n_grad_accumulation=2, master_seed=7)
    tr = api.run_protocol(method, api.LMConfig(**MINI, precision="fp32", max_batch=4), opt, sim, 4,
                          comm=nccl_comm)
    gc = G.GPTConfig(**MINI)
    prob = G.LMProblem(gc)
    th0 = G.default_theta0(gc, 7).astype(np.float32).astype(np.float64)
    ocfg = O.OptimizerConfig(**{k: getattr(opt, k) for k in O.OptimizerConfig.__dataclass_fields__})
    osim = O.SimConfig(1, 4, 2, False, 7)
    fn = (lambda th, s: prob.stochastic_grad(th, s, 4))
    ref = O.run_method(method, fn, th0, ocfg, osim, 4, eval_fn=prob.value_and_grad)
    for t in range(4):
        a, b = tr.theta_history[t + 1], ref.theta_history[t + 1]
        assert np.linalg.norm(a - b) / np.linalg.norm(b) <= 1e-5
        assert tr.records[t].samples_cum == ref.records[t].samples_cum
        assert abs(tr.records[t].loss - ref.records[t].loss) <= 1e-5 * abs(ref.records[t].loss)


@pytest.mark.parametrize("method", ["acco", "zero1", "dpu", "wp"])
def test_engine_peer_fabric_matches_oracle(cuda, method):
    """Peer fabric (one fused fold + optimizer + replica-store kernel per comm
    phase, device flags for counts and phase barriers) at world size 1: the
    same protocol code path as N GPUs on NVLink, with this rank as its own peer."""
    peer = api.PeerComm(rank=0, world=1, device=0)
    opt = api.OptimizerConfig(kind="adamw", learning_rate=6e-4, weight_decay=0.1, adam_beta2=0.95,
                              scheduler="cosine")
    sim = api.SimConfig(n_workers=1, batch_size=4, n_grad_accumulation=2, master_seed=7, eval_every=1)
    tr = api.run_protocol(method, api.LMConfig(**MINI, precision="fp32", max_batch=4), opt, sim, 4, comm=peer)
    gc = G.GPTConfig(**MINI)
    prob = G.LMProblem(gc)
    th0 = G.default_theta0(gc, 7).astype(np.float32).astype(np.float64)
    ocfg = O.OptimizerConfig(**{k: getattr(opt, k) for k in O.OptimizerConfig.__dataclass_fields__})
    osim = O.SimConfig(1, 4, 2, False, 7)
    ref = O.run_method(method, (lambda th, s: prob.stochastic_grad(th, s, 4)), th0, ocfg, osim, 4,
                       eval_fn=prob.value_and_grad)
    for t in range(4):
        a, b = tr.theta_history[t + 1], ref.theta_history[t + 1]
        assert np.linalg.norm(a - b) / np.linalg.norm(b) <= 1e-5
        e, f = tr.estimate_history[t + 1], ref.estimate_history[t + 1]
        assert np.linalg.norm(e - f) / np.linalg.norm(f) <= 1e-5
        assert tr.records[t].samples_cum == ref.records[t].samples_cum
        assert abs(tr.records[t].loss - ref.records[t].loss) <= 1e-5 * abs(ref.records[t].loss)
    kinds = {iv.kind for iv in tr.timeline if iv.stream == "comm"}
    assert "optimizer" in kinds


def test_peer_fabric_rejects_ddp(cuda):
    peer = api.PeerComm(rank=0, world=1, device=0)
    with pytest.raises(api.InvalidArgument):
        api.Trainer("ddp", api.Model(api.LMConfig(**MINI, precision="fp32", max_batch=4)),
                    api.OptimizerConfig(kind="sgd", learning_rate=0.1), api.SimConfig(n_workers=1, batch_size=4),
                    peer)


def test_engine_nccl_replica_check(cuda, nccl_comm):
    """Debug replica check on the NCCL path: both replicas hashed after every
    comm phase, hashes all-gathered over NCCL (8 B each) and compared."""
    opt = api.OptimizerConfig(kind="adamw", learning_rate=6e-4, weight_decay=0.1, adam_beta2=0.95)
    sim = api.SimConfig(n_workers=1, batch_size=4, master_seed=7, check_replicas=True)
    tr = api.run_protocol("acco", api.LMConfig(**MINI, precision="bf16", max_batch=4), opt, sim, 3, comm=nccl_comm)
    assert len(tr.records) == 3 and not tr.diverged


def test_nccl_stuck_phase_fails_instead_of_hanging(cuda, nccl_comm, monkeypatch):
    """Failure detection on the NCCL path (the reference's deadlock detection,
    protocols.cpp:476-482): a comm phase that makes no progress — here a 3 s
    spin on the comm stream standing in for a dead peer — trips the
    ACCO_NCCL_TIMEOUT_S watchdog, which aborts the communicator and raises
    (code 4) instead of blocking forever. A fresh communicator is used: an
    aborted one is unusable."""
    uid = (C.c_ubyte * 128)()
    _lib.call("acco_comm_unique_id", uid)
    h = C.c_void_p()
    _lib.call("acco_comm_init_rank", 1, 0, uid, 0, C.byref(h))

    class _C:
        handle, rank, world = h, 0, 1

    monkeypatch.setenv("ACCO_NCCL_TIMEOUT_S", "1")
    opt = api.OptimizerConfig(kind="adamw", learning_rate=6e-4)
    sim = api.SimConfig(n_workers=1, batch_size=2, master_seed=7, eval_every=0, comm_delay_ns=3e9)
    import time
    t0 = time.time()
    with pytest.raises(_lib.AccoError, match="no progress") as e:
        api.run_protocol("acco", api.LMConfig(**MINI, precision="bf16", max_batch=2), opt, sim, 1, comm=_C())
    assert e.value.code == 4 and time.time() - t0 < 30
    torch.cuda.synchronize()
    _lib.lib().acco_comm_destroy(h)
