"""K6 (estimate) / K7 (commit) fused optimizer kernels vs the fp64 oracle
restatement of opt_step (proj/src/optim.cpp:50-92), itself pinned bitwise to
the reference (tests/test_oracle_golden.py). fp32 tolerance: rel <= 1e-5
(norm-wise), SURVEY.md §7."""
import ctypes as C
import json
import os

import numpy as np
import pytest
import torch

from oracle import accosim_oracle as O
from paper_2406_02613_b200 import _lib

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _cfg(d):
    k = {"sgd": 0, "adam": 1, "adamw": 2}[d["kind"]]
    return _lib.OptCfg(k, d["learning_rate"], d["adam_beta1"], d["adam_beta2"], d["adam_eps"], d["weight_decay"],
                       1 if d["scheduler"] == "cosine" else 0, d["n_warmup_steps"], d["total_steps"],
                       d["cosine_min_factor"])


def _p(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)


def _state(theta, n, dev):
    th = torch.tensor(theta, dtype=torch.float32, device=dev)
    m = torch.zeros(n, device=dev)
    v = torch.zeros(n, device=dev)
    st = _lib.ShardState(0, th.data_ptr(), m.data_ptr(), v.data_ptr(), 0, n)
    return st, th, m, v


def test_commit_matches_opt_step_golden(cuda):
    """Persistent commit over the reference's 6-step trajectories, all optimizer kinds."""
    for c in json.load(open(os.path.join(GOLD, "optim.json"))):
        cfg = _cfg(c["cfg"])
        n = len(c["theta0"])
        st, th, m, v = _state(c["theta0"], n, cuda)
        total = torch.tensor([1], dtype=torch.int64, device=cuda)
        for s, g in enumerate(c["grads"]):
            gd = torch.tensor(g, dtype=torch.float32, device=cuda)
            out = torch.empty(n, device=cuda)
            _lib.call("acco_opt_commit", C.byref(cfg), C.byref(st), _p(gd), None, _p(total), None, _p(out),
                      _lib.DTYPE_F32, None, _stream())
            torch.cuda.synchronize()
            assert st.step == s + 1
            assert _rel(th.cpu().numpy(), c["thetas"][s]) < 1e-6
            assert torch.equal(out, th)
            if c["cfg"]["kind"] != "sgd":
                assert _rel(m.cpu().numpy(), c["m"][s]) < 1e-6
                assert _rel(v.cpu().numpy(), c["v"][s]) < 1e-6


@pytest.mark.parametrize("kind", ["sgd", "adam", "adamw"])
@pytest.mark.parametrize("n", [1, 7, 1_000_003])
def test_estimate_commit_pair_vs_oracle(cuda, kind, n):
    """One ACCO round on a shard: estimate (transient) then commit with the
    retained estimate-phase sum, totals read from device memory."""
    rng = np.random.default_rng(n)
    cfg_o = O.OptimizerConfig(kind=kind, learning_rate=0.01 if kind != "sgd" else 0.1, weight_decay=0.05,
                              adam_beta2=0.95, scheduler="cosine", total_steps=10)
    cfg = _cfg(cfg_o.__dict__)
    theta = rng.standard_normal(n).astype(np.float32).astype(np.float64)
    st, th, m, v = _state(theta, n, cuda)
    ost = O.OptimizerState.for_range(cfg_o, 0, n)
    oth = theta.copy()
    for rnd in range(3):
        g_est = rng.standard_normal(n).astype(np.float32).astype(np.float64) * 8
        g_main = rng.standard_normal(n).astype(np.float32).astype(np.float64) * 8
        n_est, n_main = 8 + rnd, 16
        tot = torch.tensor([n_est, n_main], dtype=torch.int64, device=cuda)
        ge = torch.tensor(g_est, dtype=torch.float32, device=cuda)
        gm = torch.tensor(g_main, dtype=torch.float32, device=cuda)
        est_out = torch.empty(n, dtype=torch.bfloat16, device=cuda)
        m0, v0 = m.clone(), v.clone()
        _lib.call("acco_opt_estimate", C.byref(cfg), C.byref(st), _p(ge), _p(tot[0:1]), _p(est_out),
                  _lib.DTYPE_BF16, None, _stream())
        torch.cuda.synchronize()
        assert torch.equal(m, m0) and torch.equal(v, v0) and st.step == rnd  # transient
        _, o_est = O.opt_step(ost, oth, g_est * (1.0 / n_est), cfg_o)
        assert _rel(est_out.float().cpu().numpy(), o_est) < 4e-3  # bf16 payload
        out = torch.empty(n, device=cuda)
        _lib.call("acco_opt_commit", C.byref(cfg), C.byref(st), _p(gm), _p(ge), _p(tot[1:2]), _p(tot[0:1]),
                  _p(out), _lib.DTYPE_F32, None, _stream())
        torch.cuda.synchronize()
        ost, oth = O.opt_step(ost, oth, (g_main + g_est) * (1.0 / (n_est + n_main)), cfg_o)
        assert st.step == rnd + 1
        assert _rel(th.cpu().numpy(), oth) < 1e-6


def test_nonfinite_flag_and_empty_shard(cuda):
    cfg = _cfg(O.OptimizerConfig(kind="adamw", learning_rate=0.1).__dict__)
    n = 1000
    st, th, m, v = _state(np.ones(n), n, cuda)
    g = torch.zeros(n, device=cuda)
    g[500] = float("inf")
    flag = torch.zeros(1, dtype=torch.int32, device=cuda)
    tot = torch.tensor([4], dtype=torch.int64, device=cuda)
    _lib.call("acco_opt_commit", C.byref(cfg), C.byref(st), _p(g), None, _p(tot), None, None, _lib.DTYPE_F32,
              _p(flag), _stream())
    torch.cuda.synchronize()
    # bit 0: non-finite input (opt_step's invalid_argument); bit 1: non-finite new parameter
    assert flag.item() & 1
    flag.zero_()
    g.zero_()
    st2, th2, m2, v2 = _state(np.ones(n), n, cuda)  # (the commit above wrote non-finite theta into st)
    _lib.call("acco_opt_commit", C.byref(cfg), C.byref(st2), _p(g), None, _p(tot), None, None, _lib.DTYPE_F32,
              _p(flag), _stream())
    torch.cuda.synchronize()
    assert flag.item() == 0
    # empty trailing shard is a no-op (proj/tests/test_optim.cpp:168-181)
    st0 = _lib.ShardState(0, 0, 0, 0, 5, 5)
    _lib.call("acco_opt_commit", C.byref(cfg), C.byref(st0), None, None, _p(tot), None, None, _lib.DTYPE_F32,
              None, _stream())
    with pytest.raises(_lib.InvalidArgument):
        bad = _cfg(O.OptimizerConfig(kind="adamw", learning_rate=0.0).__dict__)
        _lib.call("acco_opt_estimate", C.byref(bad), C.byref(st), _p(g), _p(tot), _p(th), _lib.DTYPE_F32, None,
                  _stream())
