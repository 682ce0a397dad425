"""fp64 numpy GPT-style LM gradient oracle — TEST INFRASTRUCTURE ONLY.

The reference (accosim) has no language model: BASELINE.json's "tiny GPT-style
LM" is new. This module defines it once, for both the oracle and the B200
plugin (paper_2406_02613_b200/csrc/lm_*.cu implements the same definition):

* Problem contract: ``stochastic_grad(theta, MicroBatch)`` of
  /root/reference/proj/src/problems.cpp:419-451 — B sample indices drawn with
  replacement by ``Stream(batch.stream).below(n_samples)`` (:442-444); one
  sample = one sequence of seq_len+1 tokens; its loss = mean token
  cross-entropy; GradResult.gradient = mean over the B sequences.
* Data: a seeded Markov chain over the vocabulary (integer-only, bit-exact):
  succ[v] = Stream(derive(seed, 0x5eed, V)).below(V) for v = 0..V-1;
  sequence s uses Stream(derive(seed, 0xda7a, s)): x0 = below(V), then per
  position r = next_u64(); x = succ[x] if r & 3 else (r >> 2) % V.
* Model: GPT-2 block (pre-LN, causal MHA, tanh-GELU MLP 4d, final LN, LM head
  tied to wte, learned positions). Flat parameter order = ``param_layout``.
* Llama family (``arch="llama"``, BASELINE.json config C4):
  pre-RMSNorm blocks (eps 1e-5, weight only), fused q|k|v projection with
  grouped-query attention (n_kv_head KV heads; query head h reads KV head
  h // (n_head / n_kv_head)), rotary embeddings on q and k (rotate-half
  pairing (i, i + hd/2), angle t * rope_base^(-2i/hd)), SwiGLU MLP with a
  fused gate|up projection (rows [0, F) gate, [F, 2F) up; a = silu(gate) * up),
  no biases, no learned positions, untied LM head ``output.weight``.
* theta0: Stream(derive(master_seed, 0x7e7a0)) — the default_theta0 key of
  problems.cpp:474-488 — uniform with std 0.02 (c_proj: 0.02/sqrt(2L)):
  value = (std*sqrt(3)) * (2u - 1), one draw per element in flat order;
  LN weights 1, biases 0 (no draws). Exact arithmetic, so GPU and oracle agree
  bit-for-bit on theta0.

Pinned by a central finite-difference check (pattern of problems.cpp:453-472,
threshold of test_problems.cpp:92-109) and torch float64 autograd, in
tests/test_gpt_oracle.py ("parity pinned by construction").
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import List, Tuple

import numpy as np

from .accosim_oracle import derive, stream_u64_block, uniform01_block

SQRT3 = 1.7320508075688772
LN_EPS = 1e-5


@dataclass(frozen=True)
class GPTConfig:
    vocab: int = 256
    d_model: int = 128
    n_layer: int = 2
    n_head: int = 4
    seq_len: int = 64
    n_samples: int = 256
    data_seed: int = 1
    arch: str = "gpt2"       # "gpt2" | "llama"
    n_kv_head: int = 0       # llama: KV heads (0 -> n_head)
    d_ff: int = 0            # llama: SwiGLU hidden size (0 -> 4 * d_model)
    rope_base: float = 10000.0

    @property
    def kv_heads(self) -> int:
        return self.n_kv_head or self.n_head

    @property
    def ffn(self) -> int:
        return self.d_ff or 4 * self.d_model


# (name, shape, init-kind); kinds: "w" std .02, "wp" std .02/sqrt(2L), "one", "zero"
def param_layout(cfg: GPTConfig) -> List[Tuple[str, tuple, str, int]]:
    d, V, T = cfg.d_model, cfg.vocab, cfg.seq_len
    if cfg.arch == "llama":
        hd = d // cfg.n_head
        nqkv = (cfg.n_head + 2 * cfg.kv_heads) * hd
        F = cfg.ffn
        specs = [("wte", (V, d), "w")]
        for l in range(cfg.n_layer):
            p = f"layers.{l}."
            specs += [
                (p + "attention_norm.weight", (d,), "one"),
                (p + "attention.wqkv", (nqkv, d), "w"),
                (p + "attention.wo", (d, cfg.n_head * hd), "wp"),
                (p + "ffn_norm.weight", (d,), "one"),
                (p + "feed_forward.w_gate_up", (2 * F, d), "w"),
                (p + "feed_forward.w_down", (d, F), "wp"),
            ]
        specs += [("norm.weight", (d,), "one"), ("output.weight", (V, d), "w")]
        out, off = [], 0
        for name, shape, kind in specs:
            out.append((name, shape, kind, off))
            off += int(np.prod(shape))
        return out
    specs = [("wte", (V, d), "w"), ("wpe", (T, d), "w")]
    for l in range(cfg.n_layer):
        p = f"h.{l}."
        specs += [
            (p + "ln_1.weight", (d,), "one"), (p + "ln_1.bias", (d,), "zero"),
            (p + "attn.c_attn.weight", (3 * d, d), "w"), (p + "attn.c_attn.bias", (3 * d,), "zero"),
            (p + "attn.c_proj.weight", (d, d), "wp"), (p + "attn.c_proj.bias", (d,), "zero"),
            (p + "ln_2.weight", (d,), "one"), (p + "ln_2.bias", (d,), "zero"),
            (p + "mlp.c_fc.weight", (4 * d, d), "w"), (p + "mlp.c_fc.bias", (4 * d,), "zero"),
            (p + "mlp.c_proj.weight", (d, 4 * d), "wp"), (p + "mlp.c_proj.bias", (d,), "zero"),
        ]
    specs += [("ln_f.weight", (d,), "one"), ("ln_f.bias", (d,), "zero")]
    out, off = [], 0
    for name, shape, kind in specs:
        out.append((name, shape, kind, off))
        off += int(np.prod(shape))
    return out


def param_count(cfg: GPTConfig) -> int:
    name, shape, _, off = param_layout(cfg)[-1]
    return off + int(np.prod(shape))


def unpack(cfg: GPTConfig, theta: np.ndarray) -> dict:
    return {n: theta[o:o + int(np.prod(s))].reshape(s) for n, s, _, o in param_layout(cfg)}


def dataset(cfg: GPTConfig) -> np.ndarray:
    V, T = cfg.vocab, cfg.seq_len
    succ = (stream_u64_block(derive(cfg.data_seed, 0x5EED, V), 0, V) % np.uint64(V)).astype(np.int64)
    U = np.stack([stream_u64_block(derive(cfg.data_seed, 0xDA7A, s), 0, T + 1) for s in range(cfg.n_samples)])
    tok = np.empty((cfg.n_samples, T + 1), dtype=np.int64)
    x = (U[:, 0] % np.uint64(V)).astype(np.int64)
    tok[:, 0] = x
    for t in range(1, T + 1):
        r = U[:, t]
        jump = ((r >> np.uint64(2)) % np.uint64(V)).astype(np.int64)
        x = np.where((r & np.uint64(3)) != 0, succ[x], jump)
        tok[:, t] = x
    return tok


def default_theta0(cfg: GPTConfig, master_seed: int) -> np.ndarray:
    key = derive(master_seed, 0x7E7A0)
    theta = np.zeros(param_count(cfg))
    k = 0
    for name, shape, kind, off in param_layout(cfg):
        n = int(np.prod(shape))
        if kind == "one":
            theta[off:off + n] = 1.0
        elif kind in ("w", "wp"):
            std = 0.02 if kind == "w" else 0.02 / math.sqrt(2.0 * cfg.n_layer)
            a = std * SQRT3
            theta[off:off + n] = a * (2.0 * uniform01_block(key, k, n) - 1.0)
            k += n
    return theta


# ------------------------------------------------------------------ forward/backward


def _gelu(x):
    k0, k1 = 0.7978845608028654, 0.044715
    t = np.tanh(k0 * (x + k1 * x * x * x))
    return 0.5 * x * (1.0 + t), t


def _dgelu(x, t):
    k0, k1 = 0.7978845608028654, 0.044715
    return 0.5 * (1.0 + t) + 0.5 * x * (1.0 - t * t) * k0 * (1.0 + 3.0 * k1 * x * x)


def _ln(x, g, b):
    mu = x.mean(-1, keepdims=True)
    xc = x - mu
    var = (xc * xc).mean(-1, keepdims=True)
    rstd = 1.0 / np.sqrt(var + LN_EPS)
    xh = xc * rstd
    return xh * g + b, (xh, rstd)


def _ln_bwd(dy, g, cache):
    xh, rstd = cache
    dxh = dy * g
    dx = rstd * (dxh - dxh.mean(-1, keepdims=True) - xh * (dxh * xh).mean(-1, keepdims=True))
    dg = (dy * xh).reshape(-1, xh.shape[-1]).sum(0)
    db = dy.reshape(-1, dy.shape[-1]).sum(0)
    return dx, dg, db


def _rms(x, g):
    rstd = 1.0 / np.sqrt((x * x).mean(-1, keepdims=True) + LN_EPS)
    xh = x * rstd
    return xh * g, (xh, rstd)


def _rms_bwd(dy, g, cache):
    xh, rstd = cache
    dxh = dy * g
    dx = rstd * (dxh - xh * (dxh * xh).mean(-1, keepdims=True))
    dg = (dy * xh).reshape(-1, xh.shape[-1]).sum(0)
    return dx, dg


def rope_table(cfg: GPTConfig):
    """cos/sin [T, hd/2] of angle t * base^(-2i/hd) (fp64; the GPU reads the
    same table rounded to fp32)."""
    hd = cfg.d_model // cfg.n_head
    i = np.arange(hd // 2, dtype=np.float64)
    inv = cfg.rope_base ** (-2.0 * i / hd)
    ang = np.arange(cfg.seq_len, dtype=np.float64)[:, None] * inv[None, :]
    return np.cos(ang), np.sin(ang)


def _rope(x, cos, sin):  # x [..., T, hd]
    h2 = x.shape[-1] // 2
    x1, x2 = x[..., :h2], x[..., h2:]
    return np.concatenate([x1 * cos - x2 * sin, x2 * cos + x1 * sin], -1)


def _rope_bwd(dy, cos, sin):
    h2 = dy.shape[-1] // 2
    d1, d2 = dy[..., :h2], dy[..., h2:]
    return np.concatenate([d1 * cos + d2 * sin, d2 * cos - d1 * sin], -1)


def _ce(cfg, logits, yt):
    mx = logits.max(-1, keepdims=True)
    z = logits - mx
    lse = np.log(np.exp(z).sum(-1, keepdims=True))
    logp = z - lse
    nll = -np.take_along_axis(logp, yt[..., None], -1)[..., 0]
    B, T = yt.shape
    dlog = np.exp(logp)
    np.put_along_axis(dlog, yt[..., None], np.take_along_axis(dlog, yt[..., None], -1) - 1.0, -1)
    dlog /= float(T * B)
    return float(nll.mean(1).mean(0)), dlog


def _llama_loss_and_grad(cfg: GPTConfig, theta: np.ndarray, tokens: np.ndarray, need_grad: bool):
    P = unpack(cfg, theta)
    B, T = tokens.shape[0], cfg.seq_len
    d, H, Hk, F = cfg.d_model, cfg.n_head, cfg.kv_heads, cfg.ffn
    hd = d // H
    G_ = H // Hk
    cos, sin = rope_table(cfg)
    xi, yt = tokens[:, :T], tokens[:, 1:T + 1]
    x = P["wte"][xi]
    mask = np.triu(np.ones((T, T), dtype=bool), 1)
    scale = 1.0 / math.sqrt(hd)
    caches = []
    for l in range(cfg.n_layer):
        p = f"layers.{l}."
        h, c1 = _rms(x, P[p + "attention_norm.weight"])
        qkv = h @ P[p + "attention.wqkv"].T
        q = qkv[..., :H * hd].reshape(B, T, H, hd).transpose(0, 2, 1, 3)
        k = qkv[..., H * hd:(H + Hk) * hd].reshape(B, T, Hk, hd).transpose(0, 2, 1, 3)
        v = qkv[..., (H + Hk) * hd:].reshape(B, T, Hk, hd).transpose(0, 2, 1, 3)
        q, k = _rope(q, cos, sin), _rope(k, cos, sin)
        kr, vr = np.repeat(k, G_, axis=1), np.repeat(v, G_, axis=1)
        s = (q @ kr.transpose(0, 1, 3, 2)) * scale
        s = np.where(mask, -np.inf, s)
        s = s - s.max(-1, keepdims=True)
        e = np.exp(s)
        att = e / e.sum(-1, keepdims=True)
        y = (att @ vr).transpose(0, 2, 1, 3).reshape(B, T, H * hd)
        x = x + y @ P[p + "attention.wo"].T
        h2, c2 = _rms(x, P[p + "ffn_norm.weight"])
        gu = h2 @ P[p + "feed_forward.w_gate_up"].T
        g, u = gu[..., :F], gu[..., F:]
        sg = 1.0 / (1.0 + np.exp(-g))
        a = g * sg * u
        x = x + a @ P[p + "feed_forward.w_down"].T
        caches.append((h, c1, q, kr, vr, att, y, h2, c2, g, u, sg, a))
    hf, cf = _rms(x, P["norm.weight"])
    logits = hf @ P["output.weight"].T
    loss, dlog = _ce(cfg, logits, yt)
    if not need_grad:
        return loss, None
    Gd = {n: np.zeros(s) for n, s, _, _ in param_layout(cfg)}
    Gd["output.weight"] += dlog.reshape(-1, cfg.vocab).T @ hf.reshape(-1, d)
    dx, Gd["norm.weight"] = _rms_bwd(dlog @ P["output.weight"], P["norm.weight"], cf)
    for l in reversed(range(cfg.n_layer)):
        p = f"layers.{l}."
        h, c1, q, kr, vr, att, y, h2, c2, g, u, sg, a = caches[l]
        Gd[p + "feed_forward.w_down"] += dx.reshape(-1, d).T @ a.reshape(-1, F)
        da = dx @ P[p + "feed_forward.w_down"]
        dg = da * u * sg * (1.0 + g * (1.0 - sg))
        du = da * g * sg
        dgu = np.concatenate([dg, du], -1)
        Gd[p + "feed_forward.w_gate_up"] += dgu.reshape(-1, 2 * F).T @ h2.reshape(-1, d)
        ddx, dw = _rms_bwd(dgu @ P[p + "feed_forward.w_gate_up"], P[p + "ffn_norm.weight"], c2)
        Gd[p + "ffn_norm.weight"] += dw
        dx = dx + ddx
        Gd[p + "attention.wo"] += dx.reshape(-1, d).T @ y.reshape(-1, H * hd)
        dy = (dx @ P[p + "attention.wo"]).reshape(B, T, H, hd).transpose(0, 2, 1, 3)
        dvr = att.transpose(0, 1, 3, 2) @ dy
        datt = dy @ vr.transpose(0, 1, 3, 2)
        ds = att * (datt - (datt * att).sum(-1, keepdims=True))
        dq = (ds @ kr) * scale
        dkr = (ds.transpose(0, 1, 3, 2) @ q) * scale
        dk = dkr.reshape(B, Hk, G_, T, hd).sum(2)
        dv = dvr.reshape(B, Hk, G_, T, hd).sum(2)
        dq, dk = _rope_bwd(dq, cos, sin), _rope_bwd(dk, cos, sin)
        dqkv = np.concatenate([t.transpose(0, 2, 1, 3).reshape(B, T, -1) for t in (dq, dk, dv)], -1)
        Gd[p + "attention.wqkv"] += dqkv.reshape(-1, dqkv.shape[-1]).T @ h.reshape(-1, d)
        ddx, dw = _rms_bwd(dqkv @ P[p + "attention.wqkv"], P[p + "attention_norm.weight"], c1)
        Gd[p + "attention_norm.weight"] += dw
        dx = dx + ddx
    np.add.at(Gd["wte"], xi.reshape(-1), dx.reshape(-1, d))
    grad = np.concatenate([Gd[n].reshape(-1) for n, _, _, _ in param_layout(cfg)])
    return loss, grad


def loss_and_grad(cfg: GPTConfig, theta: np.ndarray, tokens: np.ndarray, need_grad: bool = True):
    """Mean over the batch of per-sequence mean token CE, and its gradient
    (= GradResult.gradient, the per-sample mean). tokens: [B, seq_len+1]."""
    if cfg.arch == "llama":
        return _llama_loss_and_grad(cfg, theta, tokens, need_grad)
    P = unpack(cfg, theta)
    B, T = tokens.shape[0], cfg.seq_len
    d, H = cfg.d_model, cfg.n_head
    hd = d // H
    xi, yt = tokens[:, :T], tokens[:, 1:T + 1]
    x = P["wte"][xi] + P["wpe"][None, :T]
    mask = np.triu(np.ones((T, T), dtype=bool), 1)
    scale = 1.0 / math.sqrt(hd)
    caches = []
    for l in range(cfg.n_layer):
        p = f"h.{l}."
        h, c1 = _ln(x, P[p + "ln_1.weight"], P[p + "ln_1.bias"])
        qkv = h @ P[p + "attn.c_attn.weight"].T + P[p + "attn.c_attn.bias"]
        q, k, v = (qkv[..., i * d:(i + 1) * d].reshape(B, T, H, hd).transpose(0, 2, 1, 3) for i in range(3))
        s = (q @ k.transpose(0, 1, 3, 2)) * scale
        s = np.where(mask, -np.inf, s)
        s = s - s.max(-1, keepdims=True)
        e = np.exp(s)
        att = e / e.sum(-1, keepdims=True)
        yh = att @ v
        y = yh.transpose(0, 2, 1, 3).reshape(B, T, d)
        x = x + y @ P[p + "attn.c_proj.weight"].T + P[p + "attn.c_proj.bias"]
        h2, c2 = _ln(x, P[p + "ln_2.weight"], P[p + "ln_2.bias"])
        a = h2 @ P[p + "mlp.c_fc.weight"].T + P[p + "mlp.c_fc.bias"]
        u, tg = _gelu(a)
        x = x + u @ P[p + "mlp.c_proj.weight"].T + P[p + "mlp.c_proj.bias"]
        caches.append((h, c1, q, k, v, att, y, h2, c2, a, tg, u))
    hf, cf = _ln(x, P["ln_f.weight"], P["ln_f.bias"])
    logits = hf @ P["wte"].T
    mx = logits.max(-1, keepdims=True)
    z = logits - mx
    lse = np.log(np.exp(z).sum(-1, keepdims=True))
    logp = z - lse
    nll = -np.take_along_axis(logp, yt[..., None], -1)[..., 0]
    loss = float(nll.mean(1).mean(0))
    if not need_grad:
        return loss, None
    G = {n: np.zeros(s) for n, s, _, _ in param_layout(cfg)}
    dlog = np.exp(logp)
    np.put_along_axis(dlog, yt[..., None], np.take_along_axis(dlog, yt[..., None], -1) - 1.0, -1)
    dlog /= float(T * B)
    G["wte"] += dlog.reshape(-1, cfg.vocab).T @ hf.reshape(-1, d)
    dhf = dlog @ P["wte"]
    dx, G["ln_f.weight"], G["ln_f.bias"] = _ln_bwd(dhf, P["ln_f.weight"], cf)
    for l in reversed(range(cfg.n_layer)):
        p = f"h.{l}."
        h, c1, q, k, v, att, y, h2, c2, a, tg, u = caches[l]
        # mlp
        G[p + "mlp.c_proj.weight"] += dx.reshape(-1, d).T @ u.reshape(-1, 4 * d)
        G[p + "mlp.c_proj.bias"] += dx.reshape(-1, d).sum(0)
        du = dx @ P[p + "mlp.c_proj.weight"]
        da = du * _dgelu(a, tg)
        G[p + "mlp.c_fc.weight"] += da.reshape(-1, 4 * d).T @ h2.reshape(-1, d)
        G[p + "mlp.c_fc.bias"] += da.reshape(-1, 4 * d).sum(0)
        dh2 = da @ P[p + "mlp.c_fc.weight"]
        ddx, dg, db = _ln_bwd(dh2, P[p + "ln_2.weight"], c2)
        G[p + "ln_2.weight"] += dg
        G[p + "ln_2.bias"] += db
        dx = dx + ddx
        # attention
        G[p + "attn.c_proj.weight"] += dx.reshape(-1, d).T @ y.reshape(-1, d)
        G[p + "attn.c_proj.bias"] += dx.reshape(-1, d).sum(0)
        dy = (dx @ P[p + "attn.c_proj.weight"]).reshape(B, T, H, hd).transpose(0, 2, 1, 3)
        dv = att.transpose(0, 1, 3, 2) @ dy
        datt = dy @ v.transpose(0, 1, 3, 2)
        ds = att * (datt - (datt * att).sum(-1, keepdims=True))
        dq = (ds @ k) * scale
        dk = (ds.transpose(0, 1, 3, 2) @ q) * scale
        dqkv = np.concatenate([t.transpose(0, 2, 1, 3).reshape(B, T, d) for t in (dq, dk, dv)], -1)
        G[p + "attn.c_attn.weight"] += dqkv.reshape(-1, 3 * d).T @ h.reshape(-1, d)
        G[p + "attn.c_attn.bias"] += dqkv.reshape(-1, 3 * d).sum(0)
        dh = dqkv @ P[p + "attn.c_attn.weight"]
        ddx, dg, db = _ln_bwd(dh, P[p + "ln_1.weight"], c1)
        G[p + "ln_1.weight"] += dg
        G[p + "ln_1.bias"] += db
        dx = dx + ddx
    np.add.at(G["wte"], xi.reshape(-1), dx.reshape(-1, d))
    G["wpe"][:T] += dx.sum(0)
    grad = np.concatenate([G[n].reshape(-1) for n, _, _, _ in param_layout(cfg)])
    return loss, grad


class LMProblem:
    """The LM as an accosim Problem (problems.hpp:86-92 contract)."""

    def __init__(self, cfg: GPTConfig):
        self.cfg = cfg
        self.tokens = dataset(cfg)
        self.dim = param_count(cfg)
        self.smoothness = None
        self.optimum = None

    def stochastic_grad(self, theta, stream: int, size: int, full_batch: bool = False):
        from .accosim_oracle import sample_indices

        idx = list(range(self.cfg.n_samples)) if full_batch else sample_indices(stream, size, self.cfg.n_samples)
        loss, g = loss_and_grad(self.cfg, theta, self.tokens[idx])
        return g, len(idx), loss

    def value_and_grad(self, theta, chunk: int = 64):
        n = self.cfg.n_samples
        tot_l, tot_g = 0.0, np.zeros(self.dim)
        for c in range(0, n, chunk):
            hi = min(n, c + chunk)
            l, g = loss_and_grad(self.cfg, theta, self.tokens[c:hi])
            tot_l += l * (hi - c)
            tot_g += g * (hi - c)
        return tot_l / n, tot_g / n
