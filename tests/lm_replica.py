"""Torch restatement of the GPT-2 LM plugin's forward/backward — TEST
INFRASTRUCTURE ONLY (never imported by the package, the bench's timed path or
the C-ABI).

Two uses:

* ``bf16=False, dtype=torch.float64``: the exact math of oracle/gpt_oracle.py
  (``loss_and_grad``), on any torch device. tests/test_lm_replica.py pins it to
  the numpy oracle (<= 1e-10), so at the benchmark shapes (V = 50257, T = 1024,
  B = 8), where the numpy oracle needs minutes, this runs on the GPU as the
  fp64 reference.
* ``bf16=True, dtype=torch.float32``: a *bf16-matched* replica of the
  throughput path. Every tensor the CUDA kernels store in bf16 is rounded to
  bf16 at the same point (parameters, embeddings, LayerNorm outputs, every GEMM
  output after its fused epilogue, the GELU slope aux, logits, dlogits, the
  attention P / dS operands of the P.V / dS.K / dS^T.Q / P^T.dO MMAs,
  activation gradients DT / DX / DA / DQKV); every contraction and reduction
  is fp32 (the tensor cores' fp32 accumulators, the fp32 gradient
  accumulator). What remains different is summation order and the kernels'
  approximate transcendentals (tanh.approx, ex2.approx), so the per-tensor
  agreement with the GPU is far tighter than either's distance to fp64.

Kernel rounding points this follows (paper_2406_02613_b200/csrc):
  model.cu:353-439 (GPT::run), gemm_tcgen05.cu epilogues (bias / residual /
  GELU slope / dGELU), attn_tc.cu (P bf16 for P.V; recomputed P and dS = P (dP
  - D) rounded for the dQ / dK / dV MMAs; D = sum dO.O over the bf16 output),
  lm_kernels.cu ce_vec_kernel (dlogits = (softmax - onehot) / T in bf16),
  ln_fwd_vec / ln_bwd_vec (fp32 statistics, bf16 outputs, dX accumulated into
  the bf16 residual gradient before rounding).

Convention: returns (loss_sum, grad_sum) with loss_sum = sum over the B
sequences of the per-sequence mean token CE and grad_sum = the gradient of
loss_sum — exactly what acco_model_stochastic_grad accumulates (B x the
per-sample mean gradient of problems.cpp:419-451).
"""
from __future__ import annotations

import math

import torch

LN_EPS = 1e-5


def param_layout(cfg):
    """oracle/gpt_oracle.py param_layout (GPT-2 family): (name, shape, offset)."""
    d, V, T = cfg["d_model"], cfg["vocab"], cfg["seq_len"]
    specs = [("wte", (V, d)), ("wpe", (T, d))]
    for l in range(cfg["n_layer"]):
        p = f"h.{l}."
        specs += [(p + "ln_1.weight", (d,)), (p + "ln_1.bias", (d,)),
                  (p + "attn.c_attn.weight", (3 * d, d)), (p + "attn.c_attn.bias", (3 * d,)),
                  (p + "attn.c_proj.weight", (d, d)), (p + "attn.c_proj.bias", (d,)),
                  (p + "ln_2.weight", (d,)), (p + "ln_2.bias", (d,)),
                  (p + "mlp.c_fc.weight", (4 * d, d)), (p + "mlp.c_fc.bias", (4 * d,)),
                  (p + "mlp.c_proj.weight", (d, 4 * d)), (p + "mlp.c_proj.bias", (d,))]
    specs += [("ln_f.weight", (d,)), ("ln_f.bias", (d,))]
    out, off = [], 0
    for n, s in specs:
        out.append((n, s, off))
        off += math.prod(s)
    return out


def _gelu_and_slope(x):
    k0, k1 = 0.7978845608028654, 0.044715
    t = torch.tanh(k0 * (x + k1 * x * x * x))
    return 0.5 * x * (1.0 + t), 0.5 * (1.0 + t) + 0.5 * x * (1.0 - t * t) * k0 * (1.0 + 3.0 * k1 * x * x)


def loss_and_grad(cfg, theta, tokens, bf16=False, dtype=torch.float64):
    """theta: flat parameters (any float dtype, on the target device);
    tokens: [B, T+1] int64 on the same device."""
    if bf16:
        assert dtype == torch.float32

        def R(x):
            return x.to(torch.bfloat16).to(torch.float32)
    else:
        def R(x):
            return x

    dev = theta.device
    V, d, L, H, T = cfg["vocab"], cfg["d_model"], cfg["n_layer"], cfg["n_head"], cfg["seq_len"]
    hd = d // H
    B = tokens.shape[0]
    M = B * T
    th = R(theta.to(dtype))
    P = {n: th[o:o + math.prod(s)].view(s) for n, s, o in param_layout(cfg)}
    xi = tokens[:, :T].reshape(-1)
    yt = tokens[:, 1:T + 1].reshape(-1)
    scale = 1.0 / math.sqrt(hd)
    mask = torch.triu(torch.ones(T, T, dtype=torch.bool, device=dev), 1)

    def ln(x, g, b):
        mu = x.mean(-1, keepdim=True)
        xc = x - mu
        rs = torch.rsqrt((xc * xc).mean(-1, keepdim=True) + LN_EPS)
        xh = xc * rs
        return R(xh * g + b), (xh, rs)

    def ln_bwd(dy, g, cache, prev=None):
        xh, rs = cache
        dxh = dy * g
        dx = rs * (dxh - dxh.mean(-1, keepdim=True) - xh * (dxh * xh).mean(-1, keepdim=True))
        if prev is not None:
            dx = dx + prev
        return R(dx), (dy * xh).sum(0), dy.sum(0)

    def heads(t):  # [M, d] -> [B, H, T, hd]
        return t.view(B, T, H, hd).permute(0, 2, 1, 3)

    def unheads(t):  # [B, H, T, hd] -> [M, d]
        return t.permute(0, 2, 1, 3).reshape(M, d)

    x = R(P["wte"][xi] + P["wpe"].repeat(B, 1))
    caches = []
    for l in range(L):
        p = f"h.{l}."
        h1, c1 = ln(x, P[p + "ln_1.weight"], P[p + "ln_1.bias"])
        qkv = R(h1 @ P[p + "attn.c_attn.weight"].t() + P[p + "attn.c_attn.bias"])
        q, k, v = (heads(qkv[:, i * d:(i + 1) * d]) for i in range(3))
        s = (q @ k.transpose(-1, -2)) * scale
        s = s.masked_fill(mask, float("-inf"))
        mx = s.amax(-1, keepdim=True)
        e = torch.exp(s - mx)
        lsum = e.sum(-1, keepdim=True)
        y = R(unheads((R(e) @ v) / lsum))
        lse = mx + torch.log(lsum)
        xm = R(y @ P[p + "attn.c_proj.weight"].t() + P[p + "attn.c_proj.bias"] + x)
        h2, c2 = ln(xm, P[p + "ln_2.weight"], P[p + "ln_2.bias"])
        a = h2 @ P[p + "mlp.c_fc.weight"].t() + P[p + "mlp.c_fc.bias"]
        u, slope = _gelu_and_slope(a)
        u, slope = R(u), R(slope)
        x_next = R(u @ P[p + "mlp.c_proj.weight"].t() + P[p + "mlp.c_proj.bias"] + xm)
        caches.append((x, h1, c1, q, k, v, s, lse, y, xm, h2, c2, u, slope))
        x = x_next
    hf, cf = ln(x, P["ln_f.weight"], P["ln_f.bias"])
    logits = R(hf @ P["wte"].t())
    lse_v = torch.logsumexp(logits, -1)
    row_loss = lse_v - logits.gather(1, yt[:, None])[:, 0]
    loss_sum = row_loss.sum() / T
    dlog = torch.exp(logits - lse_v[:, None])
    dlog[torch.arange(M, device=dev), yt] -= 1.0
    dlog = R(dlog / T)

    G = {n: None for n, _, _ in param_layout(cfg)}
    G["wte"] = dlog.t() @ hf
    dt = R(dlog @ P["wte"])
    dx, G["ln_f.weight"], G["ln_f.bias"] = ln_bwd(dt, P["ln_f.weight"], cf)
    for l in reversed(range(L)):
        p = f"h.{l}."
        x_in, h1, c1, q, k, v, s, lse, y, xm, h2, c2, u, slope = caches[l]
        G[p + "mlp.c_proj.bias"] = dx.sum(0)
        G[p + "mlp.c_proj.weight"] = dx.t() @ u
        da = R((dx @ P[p + "mlp.c_proj.weight"]) * slope)
        G[p + "mlp.c_fc.bias"] = da.sum(0)
        G[p + "mlp.c_fc.weight"] = da.t() @ h2
        dt = R(da @ P[p + "mlp.c_fc.weight"])
        dx, G[p + "ln_2.weight"], G[p + "ln_2.bias"] = ln_bwd(dt, P[p + "ln_2.weight"], c2, prev=dx)
        G[p + "attn.c_proj.bias"] = dx.sum(0)
        G[p + "attn.c_proj.weight"] = dx.t() @ y
        dy = R(dx @ P[p + "attn.c_proj.weight"])
        dyh = heads(dy)
        Dsum = (dyh * heads(y)).sum(-1, keepdim=True)
        pr = torch.exp(s - lse)  # recomputed P (masked entries: exp(-inf) = 0)
        dp = dyh @ v.transpose(-1, -2)
        ds = pr * (dp - Dsum)
        dv = R(R(pr).transpose(-1, -2) @ dyh)
        dq = R(scale * (R(ds) @ k))
        dk = R(scale * (R(ds).transpose(-1, -2) @ q))
        dqkv = torch.cat([unheads(dq), unheads(dk), unheads(dv)], -1)
        G[p + "attn.c_attn.bias"] = dqkv.sum(0)
        G[p + "attn.c_attn.weight"] = dqkv.t() @ h1
        dt = R(dqkv @ P[p + "attn.c_attn.weight"])
        dx, G[p + "ln_1.weight"], G[p + "ln_1.bias"] = ln_bwd(dt, P[p + "ln_1.weight"], c1, prev=dx)
    G["wte"] = G["wte"].index_add(0, xi, dx)
    G["wpe"] = dx.view(B, T, d).sum(0)
    grad = torch.cat([G[n].reshape(-1) for n, _, _ in param_layout(cfg)])
    return loss_sum, grad


# ----------------------------------------------------------------- Llama family
def llama_param_layout(cfg):
    """oracle/gpt_oracle.py param_layout, arch="llama": (name, shape, offset)."""
    d, V, H = cfg["d_model"], cfg["vocab"], cfg["n_head"]
    Hk = cfg.get("n_kv_head") or H
    hd = d // H
    F = cfg.get("d_ff") or 4 * d
    specs = [("wte", (V, d))]
    for l in range(cfg["n_layer"]):
        p = f"layers.{l}."
        specs += [(p + "attention_norm.weight", (d,)), (p + "attention.wqkv", ((H + 2 * Hk) * hd, d)),
                  (p + "attention.wo", (d, H * hd)), (p + "ffn_norm.weight", (d,)),
                  (p + "feed_forward.w_gate_up", (2 * F, d)), (p + "feed_forward.w_down", (d, F))]
    specs += [("norm.weight", (d,)), ("output.weight", (V, d))]
    out, off = [], 0
    for n, s in specs:
        out.append((n, s, off))
        off += math.prod(s)
    return out


def llama_loss_and_grad(cfg, theta, tokens, bf16=False, dtype=torch.float64):
    """The Llama block of oracle/gpt_oracle.py (_llama_loss_and_grad) — RMSNorm,
    fused q|k|v with grouped-query attention, rotary embeddings (rotate-half),
    SwiGLU with a fused gate|up projection, untied head — with the bf16
    rounding points of model.cu run_llama in bf16 mode (the fused SwiGLU
    epilogues: gate / up pre-activations and silu(gate) * up stored in bf16;
    the down projection's dgrad rounded to bf16 before the dSwiGLU math;
    RoPE applied to the bf16 q / k with the fp32 (cos, sin) table)."""
    if bf16:
        assert dtype == torch.float32

        def R(x):
            return x.to(torch.bfloat16).to(torch.float32)
    else:
        def R(x):
            return x

    dev = theta.device
    V, d, L, H, T = cfg["vocab"], cfg["d_model"], cfg["n_layer"], cfg["n_head"], cfg["seq_len"]
    Hk = cfg.get("n_kv_head") or H
    F = cfg.get("d_ff") or 4 * d
    base = cfg.get("rope_base") or 10000.0
    hd = d // H
    G_ = H // Hk
    B = tokens.shape[0]
    M = B * T
    th = R(theta.to(dtype))
    P = {n: th[o:o + math.prod(s)].view(s) for n, s, o in llama_param_layout(cfg)}
    xi = tokens[:, :T].reshape(-1)
    yt = tokens[:, 1:T + 1].reshape(-1)
    scale = 1.0 / math.sqrt(hd)
    mask = torch.triu(torch.ones(T, T, dtype=torch.bool, device=dev), 1)
    i = torch.arange(hd // 2, dtype=torch.float64, device=dev)
    ang = torch.arange(T, dtype=torch.float64, device=dev)[:, None] * (base ** (-2.0 * i / hd))[None, :]
    cos, sin = torch.cos(ang), torch.sin(ang)
    if bf16:  # the kernels read the fp64 angles' cos / sin rounded to fp32
        cos, sin = cos.float(), sin.float()
    cos, sin = cos.to(dtype), sin.to(dtype)

    def rms(x, g):
        rs = torch.rsqrt((x * x).mean(-1, keepdim=True) + LN_EPS)
        xh = x * rs
        return R(xh * g), (xh, rs)

    def rms_bwd(dy, g, cache, prev=None):
        xh, rs = cache
        dxh = dy * g
        dx = rs * (dxh - xh * (dxh * xh).mean(-1, keepdim=True))
        if prev is not None:
            dx = dx + prev
        return R(dx), (dy * xh).sum(0)

    def rope(t, inverse=False):  # t [B, nh, T, hd]
        h2 = hd // 2
        a, b = t[..., :h2], t[..., h2:]
        if inverse:
            return R(torch.cat([a * cos + b * sin, b * cos - a * sin], -1))
        return R(torch.cat([a * cos - b * sin, b * cos + a * sin], -1))

    def heads(t, n):  # [M, n*hd] -> [B, n, T, hd]
        return t.view(B, T, n, hd).permute(0, 2, 1, 3)

    def unheads(t):
        return t.permute(0, 2, 1, 3).reshape(M, -1)

    x = P["wte"][xi].clone()
    caches = []
    for l in range(L):
        p = f"layers.{l}."
        h1, c1 = rms(x, P[p + "attention_norm.weight"])
        qkv = R(h1 @ P[p + "attention.wqkv"].t())
        q = rope(heads(qkv[:, :H * hd], H))
        k = rope(heads(qkv[:, H * hd:(H + Hk) * hd], Hk))
        v = heads(qkv[:, (H + Hk) * hd:], Hk)
        kr, vr = k.repeat_interleave(G_, dim=1), v.repeat_interleave(G_, dim=1)
        s = (q @ kr.transpose(-1, -2)) * scale
        s = s.masked_fill(mask, float("-inf"))
        mx = s.amax(-1, keepdim=True)
        e = torch.exp(s - mx)
        lsum = e.sum(-1, keepdim=True)
        y = R(unheads((R(e) @ vr) / lsum))
        lse = mx + torch.log(lsum)
        xm = R(y @ P[p + "attention.wo"].t() + x)
        h2, c2 = rms(xm, P[p + "ffn_norm.weight"])
        gu = R(h2 @ P[p + "feed_forward.w_gate_up"].t())
        g, u = gu[:, :F], gu[:, F:]
        sg = torch.sigmoid(g)
        a = R(g * sg * u)
        x_next = R(a @ P[p + "feed_forward.w_down"].t() + xm)
        caches.append((h1, c1, q, kr, vr, s, lse, y, xm, h2, c2, g, u, sg, a))
        x = x_next
    hf, cf = rms(x, P["norm.weight"])
    logits = R(hf @ P["output.weight"].t())
    lse_v = torch.logsumexp(logits, -1)
    loss_sum = (lse_v - logits.gather(1, yt[:, None])[:, 0]).sum() / T
    dlog = torch.exp(logits - lse_v[:, None])
    dlog[torch.arange(M, device=dev), yt] -= 1.0
    dlog = R(dlog / T)

    Gd = {}
    Gd["output.weight"] = dlog.t() @ hf
    dt = R(dlog @ P["output.weight"])
    dx, Gd["norm.weight"] = rms_bwd(dt, P["norm.weight"], cf)
    for l in reversed(range(L)):
        p = f"layers.{l}."
        h1, c1, q, kr, vr, s, lse, y, xm, h2, c2, g, u, sg, a = caches[l]
        Gd[p + "feed_forward.w_down"] = dx.t() @ a
        dd = R(dx @ P[p + "feed_forward.w_down"])
        dgu = torch.cat([R(dd * u * sg * (1.0 + g * (1.0 - sg))), R(dd * g * sg)], -1)
        Gd[p + "feed_forward.w_gate_up"] = dgu.t() @ h2
        dt = R(dgu @ P[p + "feed_forward.w_gate_up"])
        dx, Gd[p + "ffn_norm.weight"] = rms_bwd(dt, P[p + "ffn_norm.weight"], c2, prev=dx)
        Gd[p + "attention.wo"] = dx.t() @ y
        dy = R(dx @ P[p + "attention.wo"])
        dyh = heads(dy, H)
        Dsum = (dyh * heads(y, H)).sum(-1, keepdim=True)
        pr = torch.exp(s - lse)
        dp = dyh @ vr.transpose(-1, -2)
        ds = pr * (dp - Dsum)
        dvr = R(pr).transpose(-1, -2) @ dyh
        dkr = scale * (R(ds).transpose(-1, -2) @ q)
        dq = R(scale * (R(ds) @ kr))
        dk = R(dkr.view(B, Hk, G_, T, hd).sum(2))  # the group's query heads fold into their KV head
        dv = R(dvr.view(B, Hk, G_, T, hd).sum(2))
        dq, dk = rope(dq, inverse=True), rope(dk, inverse=True)
        dqkv = torch.cat([unheads(dq), unheads(dk), unheads(dv)], -1)
        Gd[p + "attention.wqkv"] = dqkv.t() @ h1
        dt = R(dqkv @ P[p + "attention.wqkv"])
        dx, Gd[p + "attention_norm.weight"] = rms_bwd(dt, P[p + "attention_norm.weight"], c1, prev=dx)
    Gd["wte"] = torch.zeros_like(P["wte"]).index_add(0, xi, dx)
    grad = torch.cat([Gd[n].reshape(-1) for n, _, _ in llama_param_layout(cfg)])
    return loss_sum, grad
