"""Pin the fp64 LM gradient oracle (the reference has no LM):
central finite differences (problems.cpp:453-472 pattern, <= 1e-4 as in
test_problems.cpp:92-109) and an independent torch float64 autograd model."""
import math

import numpy as np
import pytest
import torch

from oracle import accosim_oracle as O
from oracle import gpt_oracle as G

TINY = G.GPTConfig(vocab=32, d_model=16, n_layer=2, n_head=2, seq_len=8, n_samples=16, data_seed=3)


def test_c1_param_count():
    c1 = G.GPTConfig(vocab=256, d_model=128, n_layer=2, n_head=4, seq_len=64)
    assert G.param_count(c1) == 437_760
    gpt2s = G.GPTConfig(vocab=50257, d_model=768, n_layer=12, n_head=12, seq_len=1024)
    assert G.param_count(gpt2s) == 124_439_808  # GPT-2 small
    gpt2m = G.GPTConfig(vocab=50257, d_model=1024, n_layer=24, n_head=16, seq_len=1024)
    assert G.param_count(gpt2m) == 354_823_168  # GPT-2 medium


def test_dataset_is_deterministic_markov():
    tok = G.dataset(TINY)
    assert tok.shape == (16, 9)
    assert tok.min() >= 0 and tok.max() < 32
    assert np.array_equal(tok, G.dataset(TINY))
    # first token of sequence 0 is Stream(derive(seed, 0xda7a, 0)).below(V)
    assert tok[0, 0] == O.Stream(O.derive(3, 0xDA7A, 0)).below(32)


def test_theta0_layout_and_stats():
    th = G.default_theta0(TINY, 7)
    P = G.unpack(TINY, th)
    assert np.all(P["h.0.ln_1.weight"] == 1.0) and np.all(P["h.1.mlp.c_fc.bias"] == 0.0)
    w = P["h.0.attn.c_attn.weight"]
    assert abs(w.std() - 0.02) < 0.004 and np.abs(w).max() <= 0.02 * math.sqrt(3) + 1e-12
    # first drawn element = (0.02*sqrt3)*(2u-1) with u the first uniform01 of the key stream
    u = O.Stream(O.derive(7, 0x7E7A0)).uniform01()
    assert th[0] == (0.02 * G.SQRT3) * (2.0 * u - 1.0)


def test_finite_differences():
    rng = np.random.default_rng(0)
    th = G.default_theta0(TINY, 1) + 0.05 * rng.standard_normal(G.param_count(TINY))
    tok = G.dataset(TINY)[:4]
    f, g = G.loss_and_grad(TINY, th, tok)
    eps = 1e-6
    worst = 0.0
    for j in rng.choice(th.size, 200, replace=False):
        p = th.copy(); p[j] += eps
        m = th.copy(); m[j] -= eps
        num = (G.loss_and_grad(TINY, p, tok, False)[0] - G.loss_and_grad(TINY, m, tok, False)[0]) / (2 * eps)
        worst = max(worst, abs(num - g[j]) / max(1.0, abs(num), abs(g[j])))
    assert worst <= 1e-4


def _torch_loss(cfg, theta, tok):
    P = {n: t for n, t in zip([n for n, *_ in G.param_layout(cfg)],
                              torch.split(theta, [int(np.prod(s)) for _, s, _, _ in G.param_layout(cfg)]))}
    P = {n: P[n].reshape(s) for n, s, _, _ in G.param_layout(cfg)}
    B, T, d, H = tok.shape[0], cfg.seq_len, cfg.d_model, cfg.n_head
    xi, yt = tok[:, :T], tok[:, 1:]
    x = P["wte"][xi] + P["wpe"][:T]
    for l in range(cfg.n_layer):
        p = f"h.{l}."
        h = torch.nn.functional.layer_norm(x, (d,), P[p + "ln_1.weight"], P[p + "ln_1.bias"], 1e-5)
        q, k, v = (h @ P[p + "attn.c_attn.weight"].T + P[p + "attn.c_attn.bias"]).split(d, -1)
        q, k, v = (t.reshape(B, T, H, d // H).transpose(1, 2) for t in (q, k, v))
        y = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True)
        x = x + y.transpose(1, 2).reshape(B, T, d) @ P[p + "attn.c_proj.weight"].T + P[p + "attn.c_proj.bias"]
        h2 = torch.nn.functional.layer_norm(x, (d,), P[p + "ln_2.weight"], P[p + "ln_2.bias"], 1e-5)
        u = torch.nn.functional.gelu(h2 @ P[p + "mlp.c_fc.weight"].T + P[p + "mlp.c_fc.bias"], approximate="tanh")
        x = x + u @ P[p + "mlp.c_proj.weight"].T + P[p + "mlp.c_proj.bias"]
    hf = torch.nn.functional.layer_norm(x, (d,), P["ln_f.weight"], P["ln_f.bias"], 1e-5)
    logits = hf @ P["wte"].T
    nll = torch.nn.functional.cross_entropy(logits.reshape(-1, cfg.vocab), yt.reshape(-1), reduction="none")
    return nll.reshape(B, T).mean(1).mean()


def test_matches_torch_float64_autograd():
    cfg = G.GPTConfig(vocab=64, d_model=32, n_layer=2, n_head=4, seq_len=16, n_samples=8, data_seed=5)
    th = G.default_theta0(cfg, 2) * 5.0
    tok = G.dataset(cfg)
    f, g = G.loss_and_grad(cfg, th, tok)
    t = torch.tensor(th, dtype=torch.float64, requires_grad=True)
    ft = _torch_loss(cfg, t, torch.tensor(tok))
    (gt,) = torch.autograd.grad(ft, t)
    assert abs(f - ft.item()) <= 1e-12 * abs(f)
    assert np.linalg.norm(g - gt.numpy()) <= 1e-10 * np.linalg.norm(g)


def test_lm_problem_contract():
    p = G.LMProblem(TINY)
    th = G.default_theta0(TINY, 1)
    seed = O.derive(1, 0, 0, 2, 0)
    g, n, loss = p.stochastic_grad(th, seed, 4)
    idx = O.sample_indices(seed, 4, TINY.n_samples)
    l2, g2 = G.loss_and_grad(TINY, th, p.tokens[idx])
    assert n == 4 and loss == l2 and np.array_equal(g, g2)
    f, gf = p.value_and_grad(th)
    assert abs(f - math.log(32)) < 0.05  # near-uniform predictions at init


# ---------------------------------------------------------------- Llama family (C4)
LLAMA = G.GPTConfig(vocab=48, d_model=32, n_layer=2, n_head=4, seq_len=12, n_samples=8, data_seed=4,
                    arch="llama", n_kv_head=2, d_ff=40)


def _torch_llama_loss(cfg, theta, tok):
    lay = G.param_layout(cfg)
    P = {n: t.reshape(s) for (n, s, _, _), t in zip(lay, torch.split(theta, [int(np.prod(s)) for _, s, _, _ in lay]))}
    B, T, d, H, Hk, F = tok.shape[0], cfg.seq_len, cfg.d_model, cfg.n_head, cfg.kv_heads, cfg.ffn
    hd = d // H
    cos, sin = (torch.tensor(a) for a in G.rope_table(cfg))

    def rms(x, w):
        return x * torch.rsqrt((x * x).mean(-1, keepdim=True) + 1e-5) * w

    def rope(x):  # [B, h, T, hd]
        x1, x2 = x[..., :hd // 2], x[..., hd // 2:]
        return torch.cat([x1 * cos - x2 * sin, x2 * cos + x1 * sin], -1)

    xi, yt = tok[:, :T], tok[:, 1:]
    x = P["wte"][xi]
    for l in range(cfg.n_layer):
        p = f"layers.{l}."
        qkv = rms(x, P[p + "attention_norm.weight"]) @ P[p + "attention.wqkv"].T
        q, k, v = qkv.split([H * hd, Hk * hd, Hk * hd], -1)
        q = rope(q.reshape(B, T, H, hd).transpose(1, 2))
        k = rope(k.reshape(B, T, Hk, hd).transpose(1, 2))
        v = v.reshape(B, T, Hk, hd).transpose(1, 2)
        y = torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True, enable_gqa=True)
        x = x + y.transpose(1, 2).reshape(B, T, H * hd) @ P[p + "attention.wo"].T
        g, u = (rms(x, P[p + "ffn_norm.weight"]) @ P[p + "feed_forward.w_gate_up"].T).split(F, -1)
        x = x + (torch.nn.functional.silu(g) * u) @ P[p + "feed_forward.w_down"].T
    logits = rms(x, P["norm.weight"]) @ P["output.weight"].T
    nll = torch.nn.functional.cross_entropy(logits.reshape(-1, cfg.vocab), yt.reshape(-1), reduction="none")
    return nll.reshape(B, T).mean(1).mean()


def test_llama_param_count_c4():
    # TinyLlama-1.1B shape (Llama-style ~1.1B, GQA, SwiGLU)
    c4 = G.GPTConfig(vocab=32000, d_model=2048, n_layer=22, n_head=32, seq_len=2048, arch="llama",
                     n_kv_head=4, d_ff=5632)
    assert G.param_count(c4) == 1_100_048_384
    names = [n for n, *_ in G.param_layout(LLAMA)]
    assert names[:4] == ["wte", "layers.0.attention_norm.weight", "layers.0.attention.wqkv", "layers.0.attention.wo"]
    assert names[-2:] == ["norm.weight", "output.weight"]


def test_llama_matches_torch_float64_autograd():
    th = G.default_theta0(LLAMA, 2) * 5.0
    tok = G.dataset(LLAMA)
    f, g = G.loss_and_grad(LLAMA, th, tok)
    t = torch.tensor(th, dtype=torch.float64, requires_grad=True)
    ft = _torch_llama_loss(LLAMA, t, torch.tensor(tok))
    (gt,) = torch.autograd.grad(ft, t)
    assert abs(f - ft.item()) <= 1e-12 * abs(f)
    assert np.linalg.norm(g - gt.numpy()) <= 1e-10 * np.linalg.norm(g)


def test_llama_finite_differences():
    rng = np.random.default_rng(1)
    th = G.default_theta0(LLAMA, 1) + 0.05 * rng.standard_normal(G.param_count(LLAMA))
    tok = G.dataset(LLAMA)[:3]
    f, g = G.loss_and_grad(LLAMA, th, tok)
    eps = 1e-6
    worst = 0.0
    for j in rng.choice(th.size, 150, replace=False):
        p = th.copy(); p[j] += eps
        m = th.copy(); m[j] -= eps
        num = (G.loss_and_grad(LLAMA, p, tok, False)[0] - G.loss_and_grad(LLAMA, m, tok, False)[0]) / (2 * eps)
        worst = max(worst, abs(num - g[j]) / max(1.0, abs(num), abs(g[j])))
    assert worst <= 1e-4
