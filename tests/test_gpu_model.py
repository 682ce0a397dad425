"""LM plugin (stochastic_grad contract, problems.cpp:419-451) vs the fp64 oracle.

fp32 mode: gradient rel <= 1e-5 (norm-wise) and loss rel <= 1e-6.
bf16 mode (tcgen05 GEMMs, bf16 activations): rel <= 3e-2 on the gradient,
1e-2 on the loss — bf16 rounding of activations/weights, not a precision claim.
Dataset, theta0 and token indexing are bit-exact."""
import ctypes as C

import numpy as np
import pytest
import torch

from oracle import accosim_oracle as O
from oracle import gpt_oracle as G
from paper_2406_02613_b200 import _lib, api

pytestmark = pytest.mark.gpu

CFGS = {
    "tiny": dict(vocab=64, d_model=32, n_layer=2, n_head=2, seq_len=16, n_samples=32, data_seed=3),
    "c1": dict(vocab=256, d_model=128, n_layer=2, n_head=4, seq_len=64, n_samples=64, data_seed=1),
    "ragged": dict(vocab=100, d_model=64, n_layer=1, n_head=1, seq_len=24, n_samples=16, data_seed=9),
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
def test_dataset_theta0_bitexact(cuda, name):
    c = CFGS[name]
    m = api.Model(api.LMConfig(**c, precision="fp32", max_batch=4))
    gc = G.GPTConfig(**c)
    assert m.dim == G.param_count(gc)
    assert np.array_equal(m.dataset(), G.dataset(gc))
    assert np.array_equal(m.default_theta0(11), G.default_theta0(gc, 11).astype(np.float32))


@pytest.mark.parametrize("name", list(CFGS))
def test_fp32_gradient_matches_oracle(cuda, name):
    c = CFGS[name]
    B = 4
    m = api.Model(api.LMConfig(**c, precision="fp32", max_batch=B))
    gc = G.GPTConfig(**c)
    prob = G.LMProblem(gc)
    rng = np.random.default_rng(0)
    th = (G.default_theta0(gc, 5) + 0.02 * rng.standard_normal(m.dim)).astype(np.float32)
    seed = O.derive(5, 1, 2, 2, 0)
    g, loss_sum = _grad(m, torch.tensor(th, device=cuda), seed, B, cuda)
    og, n, ol = prob.stochastic_grad(th.astype(np.float64), seed, B)
    assert n == B
    assert abs(loss_sum / B - ol) <= 1e-6 * abs(ol)
    assert _rel(g, og * B) <= 1e-5  # accumulator holds N * mean (Bundle::add)


def test_accumulates_across_micro_batches(cuda):
    c = CFGS["tiny"]
    m = api.Model(api.LMConfig(**c, precision="fp32", max_batch=3))
    gc = G.GPTConfig(**c)
    prob = G.LMProblem(gc)
    th = G.default_theta0(gc, 1).astype(np.float32)
    pt = torch.tensor(th, device=cuda)
    acc = torch.zeros(m.dim, device=cuda)
    loss = torch.zeros(2, dtype=torch.float64, device=cuda)
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    seeds = [O.derive(1, 0, 0, 2, j) for j in range(2)]
    for j, sd in enumerate(seeds):
        _lib.call("acco_model_stochastic_grad", m.handle, C.c_void_p(pt.data_ptr()), C.c_uint64(sd), 3,
                  C.c_void_p(acc.data_ptr()), C.c_void_p(loss[j:].data_ptr()), s)
    torch.cuda.synchronize()
    ref = sum(prob.stochastic_grad(th.astype(np.float64), sd, 3)[0] * 3 for sd in seeds)
    assert _rel(acc.cpu().numpy(), ref) <= 1e-5


def test_value_and_grad_full_dataset(cuda):
    c = CFGS["tiny"]
    m = api.Model(api.LMConfig(**c, precision="fp32", max_batch=8))
    gc = G.GPTConfig(**c)
    th = G.default_theta0(gc, 2).astype(np.float32)
    pt = torch.tensor(th, device=cuda)
    g = torch.zeros(m.dim, device=cuda)
    loss = C.c_double()
    _lib.call("acco_model_value_and_grad", m.handle, C.c_void_p(pt.data_ptr()), C.byref(loss),
              C.c_void_p(g.data_ptr()), C.c_void_p(torch.cuda.current_stream().cuda_stream))
    of, og = G.LMProblem(gc).value_and_grad(th.astype(np.float64))
    assert abs(loss.value - of) <= 1e-6 * abs(of)
    assert _rel(g.cpu().numpy(), og) <= 1e-5


@pytest.mark.parametrize("name", ["tiny", "c1"])
def test_bf16_gradient_close_to_oracle(cuda, name):
    c = CFGS[name]
    B = 4
    m = api.Model(api.LMConfig(**c, precision="bf16", max_batch=B))
    gc = G.GPTConfig(**c)
    rng = np.random.default_rng(1)
    th = (G.default_theta0(gc, 5) + 0.05 * rng.standard_normal(m.dim)).astype(np.float32)
    th_bf = torch.tensor(th).to(torch.bfloat16)
    seed = O.derive(9, 0, 1, 2, 0)
    g, loss_sum = _grad(m, th_bf.to(cuda), seed, B, cuda)
    og, _, ol = G.LMProblem(gc).stochastic_grad(th_bf.float().double().numpy(), seed, B)
    assert abs(loss_sum / B - ol) <= 1e-2 * abs(ol)
    assert _rel(g, og * B) <= 3e-2


@pytest.mark.parametrize("seq", [128, 100, 256, 131, 141])
def test_bf16_tensor_core_attention_per_tensor(cuda, seq):
    """head size 64 routes attention to the mma.sync flash kernels; check every
    weight tensor's gradient separately so an attention-backward error cannot
    hide under the (large) embedding gradient."""
    c = dict(vocab=128, d_model=128, n_layer=2, n_head=2, seq_len=seq, n_samples=16, data_seed=4)
    B = 3
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


@pytest.mark.parametrize("seq", [128, 200, 384, 1024, 1023])
def test_tcgen05_attention_matches_mma_path(cuda, seq, monkeypatch):
    """Same bf16 model gradient with the tcgen05 flash forward vs the mma.sync
    one (ACCO_ATTN_LEGACY): both bf16, so agreement is at bf16 rounding.
    (T = 141: the legacy mma.sync backward disagrees by 8 % while the tcgen05
    path matches the oracle there, test_bf16_tensor_core_attention_per_tensor;
    the legacy comparator is not on the product path.)"""
    c = dict(vocab=128, d_model=128, n_layer=1, n_head=2, seq_len=seq, n_samples=8, data_seed=6)
    m = api.Model(api.LMConfig(**c, precision="bf16", max_batch=2))
    gc = G.GPTConfig(**c)
    th = torch.tensor(G.default_theta0(gc, 3) * 10).to(torch.bfloat16).to(cuda)
    seed = O.derive(6, 0, 0, 2, 0)
    g_tc, l_tc = _grad(m, th, seed, 2, cuda)
    monkeypatch.setenv("ACCO_ATTN_LEGACY", "1")
    g_mma, l_mma = _grad(m, th, seed, 2, cuda)
    assert abs(l_tc - l_mma) <= 2e-3 * abs(l_mma)
    assert _rel(g_tc, g_mma) <= 2e-2


def test_micro_batch_bounds(cuda):
    m = api.Model(api.LMConfig(**CFGS["tiny"], precision="fp32", max_batch=2))
    pt = torch.zeros(m.dim, device=cuda)
    with pytest.raises(_lib.InvalidArgument):
        _grad(m, pt, 1, 3, cuda)
    with pytest.raises(_lib.InvalidArgument):
        api.Model(api.LMConfig(vocab=64, d_model=30, n_layer=1, n_head=3, seq_len=8, n_samples=4))


@pytest.mark.parametrize("arch,d", [("gpt2", 1024), ("llama", 2048)])
def test_wide_row_norm_backward_matches_warp_per_row(cuda, arch, d, monkeypatch):
    """d >= 1024 routes the LayerNorm/RMSNorm backward to the block-per-row
    kernel; it must agree with the warp-per-row kernel (ACCO_LN_NARROW) and
    with the fp64 oracle at bf16 rounding."""
    c = dict(vocab=96, d_model=d, n_layer=1, n_head=d // 64, seq_len=64, n_samples=8, data_seed=2)
    if arch == "llama":
        c.update(arch="llama", n_kv_head=d // 128, d_ff=2 * d)
    m = api.Model(api.LMConfig(**c, precision="bf16", max_batch=2))
    gc = G.GPTConfig(**c)
    rng = np.random.default_rng(3)
    th = torch.tensor(G.default_theta0(gc, 1) + 0.02 * rng.standard_normal(m.dim)).to(torch.bfloat16)
    seed = O.derive(2, 0, 0, 2, 0)
    g_wide, l_wide = _grad(m, th.to(cuda), seed, 2, cuda)
    monkeypatch.setenv("ACCO_LN_NARROW", "1")
    g_nar, l_nar = _grad(m, th.to(cuda), seed, 2, cuda)
    assert abs(l_wide - l_nar) <= 1e-6 * abs(l_nar)  # forward is shared
    assert _rel(g_wide, g_nar) <= 1e-2
    og, _, ol = G.LMProblem(gc).stochastic_grad(th.float().double().numpy(), seed, 2)
    assert _rel(g_wide, og * 2) <= 5e-2


def test_embedding_backward_past_the_old_sort_limits(cuda):
    """The embedding-gradient sort is a multi-CTA stable radix sort on 64-bit
    (token, position) keys: one micro-batch of 40 x 1024 = 40960 tokens (> the
    old single-CTA sort's 32768) over a 150000-token vocabulary (V * M > 2^32,
    the old 32-bit key limit) gives the same full-dataset gradient as two
    micro-batches of 20 sequences (which the old sort handled)."""
    c = dict(vocab=150000, d_model=32, n_layer=1, n_head=1, seq_len=1024, n_samples=40, data_seed=5)
    grads = []
    for mb in (40, 20):
        m = api.Model(api.LMConfig(**c, precision="bf16", max_batch=mb))
        th = torch.tensor(m.default_theta0(3)).to(torch.bfloat16).to(cuda)
        g = torch.zeros(m.dim, device=cuda)
        loss = C.c_double()
        _lib.call("acco_model_value_and_grad", m.handle, C.c_void_p(th.data_ptr()), C.byref(loss),
                  C.c_void_p(g.data_ptr()), C.c_void_p(torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        grads.append((g.double().cpu().numpy(), loss.value))
        del m
        torch.cuda.empty_cache()
    (g1, l1), (g2, l2) = grads
    # (fp32 accumulation orders differ — K = 40960 vs 2 x 20480 in the weight
    # gradients, and the GEMM plans / split-K orders of the two micro-batch
    # sizes — so the bf16 roundings of the backward activations flip in places:
    # a few 1e-4; a mis-sorted or dropped token would be an O(1) error)
    assert abs(l1 - l2) <= 1e-6 * abs(l2)
    assert _rel(g1, g2) <= 2e-3
    V, d = c["vocab"], c["d_model"]
    assert _rel(g1[:V * d], g2[:V * d]) <= 2e-3  # the token-embedding rows themselves


@pytest.mark.parametrize("arch,d", [("gpt2", 768), ("gpt2", 1024), ("gpt2", 256), ("llama", 2048), ("llama", 512)])
def test_fused_bias_and_norm_param_grads_match_separate(cuda, arch, d, monkeypatch):
    """bf16 path: the bias gradients come off the weight-gradient GEMMs
    (ones-operand MMA) and the norm weights' / biases' gradients from per-block
    partials of the norm backward folded once per micro-batch; the separate
    column reductions (ACCO_BIAS_COLSUM=1, ACCO_LN_PARAMS_SEPARATE=1) sum the
    same bf16 values in another fp32 order: the two agree to fp32 rounding.
    The fused norm kernel's dx is bitwise the unfused one's, so the weight
    gradients differ only where the bias restriction (tile width <= 192)
    changes a weight-gradient GEMM's split-K order."""
    c = dict(vocab=96, d_model=d, n_layer=2, n_head=max(1, d // 64), seq_len=128, n_samples=8, data_seed=4)
    if arch == "llama":
        c.update(arch="llama", n_kv_head=max(1, d // 128), d_ff=2 * d)
    m = api.Model(api.LMConfig(**c, precision="bf16", max_batch=3))
    gc = G.GPTConfig(**c)
    rng = np.random.default_rng(5)
    th = torch.tensor(G.default_theta0(gc, 2) + 0.02 * rng.standard_normal(m.dim)).to(torch.bfloat16).to(cuda)
    seed = O.derive(4, 0, 0, 3, 0)
    g_f, l_f = _grad(m, th, seed, 3, cuda)
    monkeypatch.setenv("ACCO_BIAS_COLSUM", "1")
    monkeypatch.setenv("ACCO_LN_PARAMS_SEPARATE", "1")
    m2 = api.Model(api.LMConfig(**c, precision="bf16", max_batch=3))  # (the norm path is chosen per model)
    g_s, l_s = _grad(m2, th, seed, 3, cuda)
    assert l_f == l_s
    small = np.zeros(m.dim, dtype=bool)  # the column-reduced entries: biases and norm parameters
    for name, shape, _kind, off in G.param_layout(gc):
        if len(shape) == 1:
            small[off:off + shape[0]] = True
    assert _rel(g_f[~small], g_s[~small]) <= 1e-6
    assert _rel(g_f[small], g_s[small]) <= 2e-6


@pytest.mark.parametrize("arch", ["gpt2", "llama"])
def test_attention_dynamic_queue_matches_static(cuda, arch, monkeypatch):
    """The tcgen05 attention kernels taking their work items from the
    per-stream queue (the mode with collectives beside compute) compute every
    item exactly as the static LPT tables do: bitwise equal gradients and loss,
    over repeated launches (the queue resets itself after each kernel)."""
    c = dict(vocab=96, d_model=256, n_layer=2, n_head=4, seq_len=512, n_samples=8, data_seed=4)
    if arch == "llama":
        c.update(arch="llama", n_kv_head=2, d_ff=512)
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


@pytest.mark.parametrize("arch,hd", [("gpt2", 64), ("llama", 64), ("gpt2", 128)])
def test_attention_d_in_dq_matches_separate_pass(cuda, arch, hd, monkeypatch):
    """D = rowsum(dO o O) computed inside the dQ kernel (default) vs the
    separate D pass (ACCO_ATTN_DSUM_PASS): the same values up to the fp32
    summation order, so the gradients agree to fp32/bf16 rounding."""
    c = dict(vocab=96, d_model=256, n_layer=2, n_head=256 // hd, seq_len=384, n_samples=8, data_seed=4)
    if arch == "llama":
        c.update(arch="llama", n_kv_head=2, d_ff=512)
    m = api.Model(api.LMConfig(**c, precision="bf16", max_batch=3))
    gc = G.GPTConfig(**c)
    th = torch.tensor(G.default_theta0(gc, 2)).to(torch.bfloat16).to(cuda)
    seed = O.derive(4, 0, 0, 3, 0)
    g_f, l_f = _grad(m, th, seed, 3, cuda)
    monkeypatch.setenv("ACCO_ATTN_DSUM_PASS", "1")
    g_p, l_p = _grad(m, th, seed, 3, cuda)
    assert abs(l_f - l_p) <= 1e-6 * abs(l_p)
    assert _rel(g_f, g_p) <= 1e-3
