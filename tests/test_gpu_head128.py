"""Head size 128 (Llama-7B/8B-class attention geometry) on the tcgen05 flash
attention kernels (csrc/attn_tc.cu: fa_fwd_tc2<128>, fa_bwd_dq_tc<128>,
fa_bwd_dkv_tc<128>) and on the fp32 SIMT parity path (attn_simt.cu).

fp32 mode: gradient rel <= 1e-5 vs the fp64 oracle (oracle/gpt_oracle.py).
bf16 mode: per-tensor gradient rel <= 5e-2 vs the oracle, loss rel <= 1e-2;
tcgen05 vs the SIMT kernels on the same bf16 model (ACCO_ATTN_LEGACY) rel <=
2e-2; the dynamic work queue is bitwise equal to the static LPT tables."""
import ctypes as C

import numpy as np
import pytest
import torch

from oracle import accosim_oracle as O
from oracle import gpt_oracle as G
from paper_2406_02613_b200 import _lib, api

pytestmark = pytest.mark.gpu


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)


def _grad(model, params_t, seed, B, dev):
    g = torch.zeros(model.dim, device=dev)
    loss = torch.zeros(1, dtype=torch.float64, device=dev)
    _lib.call("acco_model_stochastic_grad", model.handle, C.c_void_p(params_t.data_ptr()), C.c_uint64(seed), B,
              C.c_void_p(g.data_ptr()), C.c_void_p(loss.data_ptr()),
              C.c_void_p(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    return g.double().cpu().numpy(), loss.item()


def _cfg(arch, seq, n_layer=2, hkv=None):
    c = dict(vocab=128, d_model=256, n_layer=n_layer, n_head=2, seq_len=seq, n_samples=16, data_seed=4)
    if arch == "llama":
        c.update(arch="llama", n_kv_head=hkv or 1, d_ff=320)
    return c


@pytest.fixture
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch.device("cuda:0")


@pytest.mark.parametrize("arch", ["gpt2", "llama"])
def test_head128_fp32_matches_oracle(cuda, arch):
    c = _cfg(arch, 40, n_layer=1)
    B = 2
    m = api.Model(api.LMConfig(**c, precision="fp32", max_batch=B))
    gc = G.GPTConfig(**c)
    th = G.default_theta0(gc, 3) + 0.05 * np.random.default_rng(1).standard_normal(m.dim)
    seed = O.derive(3, 0, 1, 2, 0)
    g, loss_sum = _grad(m, torch.tensor(th, dtype=torch.float32).to(cuda), seed, B, cuda)
    og, _, ol = G.LMProblem(gc).stochastic_grad(th.astype(np.float32).astype(np.float64), seed, B)
    assert abs(loss_sum / B - ol) <= 1e-6 * abs(ol)
    assert _rel(g, og * B) <= 1e-5


@pytest.mark.parametrize("arch,seq,hkv", [("gpt2", 128, None), ("gpt2", 200, None), ("llama", 256, 1),
                                          ("llama", 136, 2)])
def test_head128_bf16_per_tensor(cuda, arch, seq, hkv):
    c = _cfg(arch, seq, hkv=hkv)
    B = 2
    m = api.Model(api.LMConfig(**c, precision="bf16", max_batch=B))
    gc = G.GPTConfig(**c)
    rng = np.random.default_rng(2)
    th = (G.default_theta0(gc, 3) + 0.05 * rng.standard_normal(m.dim)).astype(np.float32)
    th_bf = torch.tensor(th).to(torch.bfloat16)
    seed = O.derive(4, 1, 0, 2, 0)
    g, loss_sum = _grad(m, th_bf.to(cuda), seed, B, cuda)
    og, _, ol = G.LMProblem(gc).stochastic_grad(th_bf.float().double().numpy(), seed, B)
    og = og * B
    assert abs(loss_sum / B - ol) <= 1e-2 * abs(ol)
    for name, shape, _, off in G.param_layout(gc):
        n = int(np.prod(shape))
        if n < 1024:
            continue
        assert _rel(g[off:off + n], og[off:off + n]) <= 5e-2, name


@pytest.mark.parametrize("arch,seq", [("gpt2", 384), ("gpt2", 1024), ("llama", 320), ("llama", 1000)])
def test_head128_tcgen05_matches_simt(cuda, arch, seq, monkeypatch):
    c = _cfg(arch, seq, n_layer=1, hkv=2)
    c["n_samples"] = 8
    m = api.Model(api.LMConfig(**c, precision="bf16", max_batch=2))
    gc = G.GPTConfig(**c)
    rng = np.random.default_rng(5)
    th = torch.tensor(G.default_theta0(gc, 3) + 0.05 * rng.standard_normal(m.dim)).to(torch.bfloat16).to(cuda)
    seed = O.derive(6, 0, 0, 2, 0)
    g_tc, l_tc = _grad(m, th, seed, 2, cuda)
    monkeypatch.setenv("ACCO_ATTN_LEGACY", "1")
    g_simt, l_simt = _grad(m, th, seed, 2, cuda)
    assert abs(l_tc - l_simt) <= 2e-3 * abs(l_simt)
    assert _rel(g_tc, g_simt) <= 2e-2


@pytest.mark.parametrize("arch", ["gpt2", "llama"])
def test_head128_dynamic_queue_matches_static(cuda, arch, monkeypatch):
    c = _cfg(arch, 512, hkv=1)
    c["n_samples"] = 8
    m = api.Model(api.LMConfig(**c, precision="bf16", max_batch=3))
    gc = G.GPTConfig(**c)
    th = torch.tensor(G.default_theta0(gc, 2)).to(torch.bfloat16).to(cuda)
    seed = O.derive(4, 0, 0, 3, 0)
    monkeypatch.setenv("ACCO_ATTN_STATIC", "1")
    g_s, l_s = _grad(m, th, seed, 3, cuda)
    monkeypatch.delenv("ACCO_ATTN_STATIC")
    monkeypatch.setenv("ACCO_ATTN_DYNAMIC", "1")
    for _ in range(2):
        g_d, l_d = _grad(m, th, seed, 3, cuda)
        assert l_d == l_s
        assert np.array_equal(g_d, g_s)
