"""Llama-family LM plugin (BASELINE.json config C4: RMSNorm, RoPE, grouped-query
attention, SwiGLU, untied head) vs the fp64 oracle (oracle/gpt_oracle.py,
arch="llama", pinned by finite differences and torch float64 autograd in
tests/test_gpt_oracle.py).

fp32 mode: gradient rel <= 1e-5 (norm-wise), loss rel <= 1e-6; dataset, theta0
and token indexing bit-exact. bf16 mode (tcgen05 GEMMs + tcgen05 GQA flash
attention): per-tensor gradient rel <= 5e-2, loss rel <= 1e-2 (bf16 rounding of
activations/weights, not a precision claim). An ACCO run (2 virtual workers)
matches the oracle's run_acco per update with theta rel <= 1e-5."""
import ctypes as C

import numpy as np
import pytest
import torch

from oracle import accosim_oracle as O
from oracle import gpt_oracle as G
from paper_2406_02613_b200 import _lib, api

pytestmark = pytest.mark.gpu

CFGS = {
    # hd 8, 2 query heads per KV head
    "tiny": dict(vocab=64, d_model=32, n_layer=2, n_head=4, n_kv_head=2, d_ff=48, seq_len=16, n_samples=32,
                 data_seed=3, arch="llama"),
    # hd 32, one KV head for 4 query heads (MQA), ragged sequence length
    "mqa": dict(vocab=96, d_model=128, n_layer=2, n_head=4, n_kv_head=1, d_ff=200, seq_len=40, n_samples=16,
                data_seed=5, arch="llama"),
    # no grouping (n_kv_head = n_head)
    "mha": dict(vocab=80, d_model=64, n_layer=1, n_head=2, n_kv_head=2, d_ff=96, seq_len=24, n_samples=16,
                data_seed=7, arch="llama"),
}


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


@pytest.mark.parametrize("name", list(CFGS))
def test_llama_dataset_theta0_bitexact(cuda, name):
    c = CFGS[name]
    m = api.Model(api.LMConfig(**c, precision="fp32", max_batch=4))
    gc = G.GPTConfig(**c)
    assert m.dim == G.param_count(gc)
    assert np.array_equal(m.dataset(), G.dataset(gc))
    assert np.array_equal(m.default_theta0(11), G.default_theta0(gc, 11).astype(np.float32))


@pytest.mark.parametrize("name", list(CFGS))
def test_llama_fp32_gradient_matches_oracle(cuda, name):
    c = CFGS[name]
    B = 3
    m = api.Model(api.LMConfig(**c, precision="fp32", max_batch=B))
    gc = G.GPTConfig(**c)
    rng = np.random.default_rng(0)
    th = (G.default_theta0(gc, 5) + 0.05 * rng.standard_normal(m.dim)).astype(np.float32)
    seed = O.derive(5, 1, 2, 2, 0)
    g, loss_sum = _grad(m, torch.tensor(th, device=cuda), seed, B, cuda)
    og, n, ol = G.LMProblem(gc).stochastic_grad(th.astype(np.float64), seed, B)
    assert n == B
    assert abs(loss_sum / B - ol) <= 1e-6 * abs(ol)
    og = og * B
    assert _rel(g, og) <= 1e-5
    for pname, shape, _, off in G.param_layout(gc):  # every tensor, incl. the norms and the untied head
        k = int(np.prod(shape))
        assert _rel(g[off:off + k], og[off:off + k]) <= 1e-4, pname


def test_llama_acco_run_matches_oracle(cuda):
    """ACCO with 2 virtual workers on the Llama plugin: every stage's first
    micro-batch overwrites the accumulator (untied embedding rows included)."""
    c = CFGS["tiny"]
    opt = api.OptimizerConfig(kind="adamw", learning_rate=1e-3, weight_decay=0.1, adam_beta2=0.95,
                              scheduler="cosine")
    sim = api.SimConfig(n_workers=2, batch_size=3, n_grad_accumulation=2, master_seed=4)
    tr = api.run_protocol("acco", api.LMConfig(**c, precision="fp32", max_batch=3), opt, sim, 3)
    gc = G.GPTConfig(**c)
    prob = G.LMProblem(gc)
    th0 = G.default_theta0(gc, 4).astype(np.float32).astype(np.float64)
    ref = O.run_acco(lambda th, s: prob.stochastic_grad(th, s, 3), th0,
                     O.OptimizerConfig(kind="adamw", learning_rate=1e-3, weight_decay=0.1, adam_beta2=0.95,
                                       scheduler="cosine"),
                     O.SimConfig(2, 3, 2, False, 4), 3, eval_fn=prob.value_and_grad)
    for t in range(3):
        assert _rel(tr.theta_history[t + 1], ref.theta_history[t + 1]) <= 1e-5
        assert tr.records[t].samples_cum == ref.records[t].samples_cum
        assert abs(tr.records[t].loss - ref.records[t].loss) <= 1e-5 * abs(ref.records[t].loss)


@pytest.mark.parametrize("seq,hkv", [(128, 2), (200, 1), (256, 4)])
def test_llama_bf16_tcgen05_gqa_per_tensor(cuda, seq, hkv):
    """hd 64 routes attention to the tcgen05 flash kernels with grouped KV
    heads; check every weight tensor's gradient separately."""
    c = dict(vocab=128, d_model=256, n_layer=2, n_head=4, n_kv_head=hkv, d_ff=320, seq_len=seq, n_samples=16,
             data_seed=4, arch="llama")
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


@pytest.mark.parametrize("seq", [128, 320])
def test_tcgen05_gqa_matches_simt(cuda, seq, monkeypatch):
    """Same bf16 Llama gradient with the tcgen05 GQA flash kernels vs the SIMT
    ones (ACCO_ATTN_LEGACY; the mma.sync path is MHA-only, so GQA falls to
    SIMT): agreement at bf16 rounding."""
    c = dict(vocab=128, d_model=256, n_layer=1, n_head=4, n_kv_head=2, d_ff=256, seq_len=seq, n_samples=8,
             data_seed=6, arch="llama")
    m = api.Model(api.LMConfig(**c, precision="bf16", max_batch=2))
    gc = G.GPTConfig(**c)
    # (moderate weights: at 10x init the bf16 model is chaotic — loss ~80 —
    # and both paths sit ~100% away from fp64, tools/diag/gqa_diag.py)
    rng = np.random.default_rng(5)
    th = torch.tensor(G.default_theta0(gc, 3) + 0.05 * rng.standard_normal(m.dim)).to(torch.bfloat16).to(cuda)
    seed = O.derive(6, 0, 0, 2, 0)
    g_tc, l_tc = _grad(m, th, seed, 2, cuda)
    monkeypatch.setenv("ACCO_ATTN_LEGACY", "1")
    g_simt, l_simt = _grad(m, th, seed, 2, cuda)
    assert abs(l_tc - l_simt) <= 2e-3 * abs(l_simt)
    assert _rel(g_tc, g_simt) <= 2e-2


def test_llama_config_validation(cuda):
    with pytest.raises(_lib.InvalidArgument):  # 4 heads cannot share 3 KV heads
        api.Model(api.LMConfig(vocab=64, d_model=32, n_layer=1, n_head=4, n_kv_head=3, seq_len=8, n_samples=4,
                               arch="llama"))
    with pytest.raises(_lib.InvalidArgument):  # d_ff must keep TMA 16-byte strides
        api.Model(api.LMConfig(vocab=64, d_model=32, n_layer=1, n_head=4, d_ff=30, seq_len=8, n_samples=4,
                               arch="llama"))


def test_swiglu_fused_epilogue_matches_unfused(cuda, monkeypatch):
    """d_ff % 128 == 0 routes the gate|up GEMM to the fused SwiGLU epilogue
    (tcgen05 path); it must reproduce the separate GEMM + SwiGLU kernel."""
    c = dict(vocab=128, d_model=256, n_layer=2, n_head=4, n_kv_head=2, d_ff=384, seq_len=128, n_samples=8,
             data_seed=6, arch="llama")
    m = api.Model(api.LMConfig(**c, precision="bf16", max_batch=2))
    gc = G.GPTConfig(**c)
    rng = np.random.default_rng(7)
    th = torch.tensor(G.default_theta0(gc, 3) + 0.05 * rng.standard_normal(m.dim)).to(torch.bfloat16).to(cuda)
    seed = O.derive(6, 0, 0, 2, 0)
    g_f, l_f = _grad(m, th, seed, 2, cuda)
    monkeypatch.setenv("ACCO_NO_SWIGLU_FUSION", "1")
    g_u, l_u = _grad(m, th, seed, 2, cuda)
    og, _, ol = G.LMProblem(gc).stochastic_grad(th.float().cpu().double().numpy(), seed, 2)
    assert abs(l_f - ol * 2) <= 1e-2 * abs(ol * 2)
    assert _rel(g_f, og * 2) <= 5e-2
    assert _rel(g_f, g_u) <= 2e-2


def test_swiglu_cta_pair_tiles_match(cuda, monkeypatch):
    """The fused SwiGLU GEMM on CTA-pair tiles (the default: the leader stages
    the gate rows, its peer the matching up rows) gives the same result as the
    single-CTA tiles (ACCO_GEMM_NO_CG2=1; same per-element accumulation
    order), and so does the DSwiGLU backward on pair tiles (ACCO_DSWIGLU_CG2=1)."""
    c = dict(vocab=128, d_model=256, n_layer=2, n_head=4, n_kv_head=2, d_ff=384, seq_len=128, n_samples=8,
             data_seed=6, arch="llama")
    m = api.Model(api.LMConfig(**c, precision="bf16", max_batch=2))
    gc = G.GPTConfig(**c)
    th = torch.tensor(G.default_theta0(gc, 3)).to(torch.bfloat16).to(cuda)
    seed = O.derive(6, 0, 0, 2, 0)
    g1, l1 = _grad(m, th, seed, 2, cuda)
    monkeypatch.setenv("ACCO_GEMM_NO_CG2", "1")
    g2, l2 = _grad(m, th, seed, 2, cuda)
    monkeypatch.delenv("ACCO_GEMM_NO_CG2")
    monkeypatch.setenv("ACCO_DSWIGLU_CG2", "1")
    g3, l3 = _grad(m, th, seed, 2, cuda)
    assert l1 == l2 == l3
    # (the other GEMMs' tile choice differs under ACCO_GEMM_NO_CG2, which can
    # change split-K orders: compare within fp32 accumulation noise there)
    assert np.allclose(g1, g2, rtol=0, atol=1e-6 * np.abs(g1).max())
    assert np.array_equal(g1, g3) or np.allclose(g1, g3, rtol=0, atol=1e-6 * np.abs(g1).max())
