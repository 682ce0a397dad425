"""Parity at the benchmarked configuration (VERDICT r01 "next" item 1).

bench.py times GPT-2 small in bf16: V = 50257, d = 768, H = 12, T = 1024,
B = 8 sequences per micro-batch. These tests run exactly those shapes (with
L = 2 layers, so the fp64 references fit a test) through the C-ABI
(acco_model_stochastic_grad) and compare every parameter tensor's gradient:

* bf16 path (tcgen05 GEMMs, tcgen05 flash attention, the vectorised LN / CE
  kernels): against the bf16-matched torch replica (tests/lm_replica.py, fp32
  math rounded to bf16 where the kernels store bf16) at <= 1e-2 per tensor and
  <= 2e-3 on the loss, and against fp64 (the bf16 distance, reported and
  bounded at 5e-2 per tensor);
* fp32 parity path (3xTF32 tcgen05 GEMMs): against fp64 at <= 1e-5 overall
  and per tensor, <= 1e-6 on the loss.

The fp64 reference at these shapes is the replica in fp64 on the GPU; it is
pinned to the numpy oracle (oracle/gpt_oracle.py) at these exact shapes with
one sequence (test_replica_is_oracle_at_bench_shape) and at small shapes on
CPU (tests/test_lm_replica.py).

test_llama_bench_shapes_bf16_and_fp32 does the same at config 4's shapes
(Llama-1B: d = 2048, GQA 32 / 4 heads, SwiGLU 5632, V = 32000, T = 2048,
B = 4; L = 2) against the Llama replica (lm_replica.llama_loss_and_grad).

test_reduced_width_loss_curve is BASELINE.json config 2's "loss-curve parity
vs CPU oracle at reduced width": d = 64, L = 12, V = 50257, T = 1024, 20 ACCO
updates on the GPU engine vs oracle.run_acco (the protocol restatement pinned
bitwise to the reference), fp32 <= 1e-5 per update, bf16 loss <= 1e-2.
"""
import ctypes as C

import numpy as np
import pytest
import torch

from oracle import accosim_oracle as O
from oracle import gpt_oracle as G
from paper_2406_02613_b200 import _lib, api
from tests import lm_replica

pytestmark = pytest.mark.gpu

C2L2 = dict(vocab=50257, d_model=768, n_layer=2, n_head=12, seq_len=1024, n_samples=64, data_seed=1)
B = 8


def _rel(a, b):
    a, b = torch.as_tensor(a).double(), torch.as_tensor(b).double()
    return ((a - b).norm() / b.norm().clamp_min(1e-300)).item()


def _kernel_grad(model, params, seed, batch, dev):
    g = torch.zeros(model.dim, device=dev)
    loss = torch.zeros(1, dtype=torch.float64, device=dev)
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        _lib.call("acco_model_stochastic_grad", model.handle, C.c_void_p(params.data_ptr()), C.c_uint64(seed),
                  batch, C.c_void_p(g.data_ptr()), C.c_void_p(loss.data_ptr()),
                  C.c_void_p(torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
    names = {e.name for e in prof.events()}
    return g, loss.item(), names


@pytest.fixture(scope="module")
def bench_case(cuda):
    torch.backends.cuda.matmul.allow_tf32 = False
    gc = G.GPTConfig(**C2L2)
    rng = np.random.default_rng(7)
    # theta0 plus noise: LN weights != 1 and biases != 0, so every tensor's
    # gradient is generic
    th = (G.default_theta0(gc, 1) + 0.02 * rng.standard_normal(G.param_count(gc))).astype(np.float32)
    seed = O.derive(1, 0, 0, 2, 0)
    idx = api.sample_indices(seed, B, gc.n_samples)
    assert idx == O.sample_indices(seed, B, gc.n_samples)  # token indexing bit-exact
    data = G.dataset(gc)
    tok = torch.tensor(data[idx], device=cuda)
    return gc, th, seed, tok, data


def _per_tensor(g, ref, cfg):
    out = {}
    for name, shape, off in lm_replica.param_layout(cfg):
        n = int(np.prod(shape))
        out[name] = _rel(g[off:off + n], ref[off:off + n])
    return out


def test_bf16_bench_shapes_match_bf16_replica(cuda, bench_case):
    gc, th, seed, tok, data = bench_case
    m = api.Model(api.LMConfig(**C2L2, precision="bf16", max_batch=B))
    assert np.array_equal(m.dataset(), data)  # dataset bit-exact at V = 50257
    th_bf = torch.tensor(th).to(torch.bfloat16).to(cuda)
    g, loss_sum, names = _kernel_grad(m, th_bf, seed, B, cuda)
    # the kernels the bench times at these shapes ran
    # (the LM head forward and weight gradient run on 256-wide CTA-pair tiles)
    for k in ("gemm_tc_kernel", "fa_fwd_tc2", "fa_bwd_dkv_tc", "fa_bwd_dq_tc", "ln_fwd_vec<3", "ln_bwd_vec_p<3", "ln_param_fold",
              "ce_vec_kernel", "f32_to_bf16_rows", "gemm_tc_kernel<256, 5, 0, 0, 0, 2>",
              "gemm_tc_kernel<256, 5, 1, 1, 0, 2>"):
        assert any(k in n for n in names), (k, sorted(names))
    assert not any("simt" in n for n in names)
    l16, g16 = lm_replica.loss_and_grad(C2L2, th_bf.float(), tok, bf16=True, dtype=torch.float32)
    l64, g64 = lm_replica.loss_and_grad(C2L2, th_bf.double(), tok)
    per16 = _per_tensor(g, g16, C2L2)
    per64 = _per_tensor(g, g64, C2L2)
    rep64 = _per_tensor(g16, g64, C2L2)  # the bf16 replica's own distance to fp64
    for name in per16:
        print(f"{name:28s} kernel vs bf16 replica {per16[name]:.2e}   kernel vs fp64 {per64[name]:.2e}   "
              f"bf16 replica vs fp64 {rep64[name]:.2e}")
    print("loss", loss_sum, l16.item(), l64.item())
    assert abs(loss_sum - l16.item()) <= 2e-3 * abs(l16.item())
    assert abs(loss_sum - l64.item()) <= 1e-2 * abs(l64.item())
    bad = {k: v for k, v in per16.items() if not v <= 1e-2}
    assert not bad, bad
    assert all(v <= 5e-2 for v in per64.values()), per64
    # The kernels' approximate transcendentals (tanh.approx in the GELU
    # epilogue, ex2.approx with a lazily updated max in attention) flip some
    # bf16 roundings relative to the replica, so kernel-vs-replica is itself
    # bf16-noise sized. The kernel's error against fp64 must then be no larger
    # than what bf16 storage alone costs (the replica's error): a wrong tile,
    # head or edge column would stand far above it.
    worse = {k: (per64[k], rep64[k]) for k in per64 if not per64[k] <= 1.5 * rep64[k] + 1e-3}
    assert not worse, worse


def test_fp32_bench_shapes_match_fp64(cuda, bench_case):
    gc, th, seed, tok, _ = bench_case
    m = api.Model(api.LMConfig(**C2L2, precision="fp32", max_batch=B))
    pt = torch.tensor(th, device=cuda)
    g, loss_sum, names = _kernel_grad(m, pt, seed, B, cuda)
    # fp32 parity mode contracts on the tensor cores (3xTF32), not the SIMT twin
    assert any("gemm_tc_kernel<128, 3, 0, 0, 1, 1>" in n for n in names), sorted(names)
    assert not any("gemm_simt_kernel" in n for n in names)
    l64, g64 = lm_replica.loss_and_grad(C2L2, pt.double(), tok)
    per = _per_tensor(g, g64, C2L2)
    for name, v in per.items():
        print(f"{name:28s} vs fp64 {v:.2e}")
    overall = _rel(g, g64)
    print("overall", overall, "loss", loss_sum, l64.item())
    assert abs(loss_sum - l64.item()) <= 1e-6 * abs(l64.item())
    assert overall <= 1e-5
    bad = {k: v for k, v in per.items() if not v <= 1e-5}
    assert not bad, bad


def test_replica_is_oracle_at_bench_shape(cuda, bench_case):
    """The GPU fp64 reference above is the numpy oracle at these shapes."""
    gc, th, _, tok, _ = bench_case
    t1 = tok[:1]
    ol, og = G.loss_and_grad(gc, th.astype(np.float64), t1.cpu().numpy())
    rl, rg = lm_replica.loss_and_grad(C2L2, torch.tensor(th, dtype=torch.float64, device=cuda), t1)
    assert abs(rl.item() - ol) <= 1e-12 * abs(ol)
    assert _rel(rg.cpu(), torch.tensor(og)) <= 1e-10


RW = dict(vocab=50257, d_model=64, n_layer=12, n_head=1, seq_len=1024, n_samples=8, data_seed=1)


def _oracle_acco(cuda, sim, opt, T):
    """oracle.run_acco (protocol restatement) with the fp64 LM gradient of the
    replica on the GPU (the numpy LM at V = 50257, T = 1024 needs seconds per
    sequence)."""
    gc = G.GPTConfig(**RW)
    tok_all = torch.tensor(G.dataset(gc), device=cuda)
    th0 = G.default_theta0(gc, sim.master_seed).astype(np.float32).astype(np.float64)

    def grad_fn(theta, stream):
        idx = O.sample_indices(stream, sim.batch_size, gc.n_samples)
        l, g = lm_replica.loss_and_grad(RW, torch.from_numpy(theta).to(cuda), tok_all[idx])
        return (g / sim.batch_size).cpu().numpy(), sim.batch_size, l.item() / sim.batch_size

    def eval_fn(theta):
        tl, tg = 0.0, None
        t = torch.from_numpy(theta).to(cuda)
        for c in range(0, gc.n_samples, 4):
            l, g = lm_replica.loss_and_grad(RW, t, tok_all[c:c + 4])
            tl += l.item()
            tg = g if tg is None else tg + g
        return tl / gc.n_samples, (tg / gc.n_samples).cpu().numpy()

    ocfg = O.OptimizerConfig(**{k: getattr(opt, k) for k in O.OptimizerConfig.__dataclass_fields__})
    osim = O.SimConfig(sim.n_workers, sim.batch_size, sim.n_grad_accumulation, False, sim.master_seed)
    return O.run_acco(grad_fn, th0, ocfg, osim, T, eval_fn=eval_fn)


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_reduced_width_loss_curve(cuda, precision):
    T = 20
    opt = api.OptimizerConfig(kind="adamw", learning_rate=6e-4, weight_decay=0.1, adam_beta2=0.95,
                              scheduler="cosine")
    sim = api.SimConfig(n_workers=1, batch_size=2, master_seed=1, eval_every=1, eval_batch=4)
    tr = api.run_protocol("acco", api.LMConfig(**RW, precision=precision, max_batch=4), opt, sim, T)
    ref = _oracle_acco(cuda, sim, opt, T)
    assert len(tr.records) == len(ref.records) == T
    for t, (r, o) in enumerate(zip(tr.records, ref.records)):
        assert r.samples_cum == o.samples_cum and r.mb_main == o.mb_main and r.mb_estimate == o.mb_estimate
        if precision == "fp32":
            assert abs(r.loss - o.loss) <= 1e-5 * abs(o.loss), (t, r.loss, o.loss)
            assert _rel(tr.theta_history[t + 1], ref.theta_history[t + 1]) <= 1e-5, t
            assert _rel(tr.estimate_history[t + 1], ref.estimate_history[t + 1]) <= 1e-5, t
            assert abs(r.train_loss - o.train_loss) <= 1e-5 * abs(o.train_loss)
        else:
            assert abs(r.loss - o.loss) <= 1e-2 * abs(o.loss), (t, r.loss, o.loss)
    print(precision, "loss curve", [round(r.loss, 5) for r in tr.records])
    assert tr.records[-1].loss < tr.records[0].loss


# BASELINE.json config 4 (bench.py --model llama-1b): d = 2048, 32 query / 4 KV
# heads of 64, SwiGLU 5632, V = 32000, T = 2048, B = 4 — at L = 2
LLAMA1B = dict(vocab=32000, d_model=2048, n_layer=2, n_head=32, seq_len=2048, n_samples=16, data_seed=1,
               arch="llama", n_kv_head=4, d_ff=5632)
LB = 4


def _llama_case(cuda):
    gc = G.GPTConfig(**LLAMA1B)
    rng = np.random.default_rng(11)
    th = (G.default_theta0(gc, 1) + 0.02 * rng.standard_normal(G.param_count(gc))).astype(np.float32)
    seed = O.derive(1, 0, 0, 2, 0)
    idx = O.sample_indices(seed, LB, gc.n_samples)
    tok = torch.tensor(G.dataset(gc)[idx], device=cuda)
    return th, seed, tok


def _per_tensor_llama(g, ref):
    return {name: _rel(g[off:off + int(np.prod(shape))], ref[off:off + int(np.prod(shape))])
            for name, shape, off in lm_replica.llama_param_layout(LLAMA1B)}


def test_llama_bench_shapes_bf16_and_fp32(cuda):
    """Config 4's compute path at its shapes: the bf16 tcgen05 path (fused
    SwiGLU / dSwiGLU epilogues, GQA attention, RoPE, wide-row RMSNorm backward)
    against the bf16-matched replica and fp64; the fp32 path against fp64."""
    torch.backends.cuda.matmul.allow_tf32 = False
    th, seed, tok = _llama_case(cuda)
    m = api.Model(api.LMConfig(**LLAMA1B, precision="bf16", max_batch=LB))
    th_bf = torch.tensor(th).to(torch.bfloat16).to(cuda)
    g, loss_sum, names = _kernel_grad(m, th_bf, seed, LB, cuda)
    for k in ("fa_fwd_tc2", "fa_bwd_dkv_tc", "fa_bwd_dq_tc", "rope_vec_kernel", "ln_bwd_wide",
              "gemm_tc_kernel<256, 5, 0, 0, 0, 2>"):  # (the SwiGLU GEMM on CTA-pair tiles)
        assert any(k in n for n in names), (k, sorted(names))
    del m
    l16, g16 = lm_replica.llama_loss_and_grad(LLAMA1B, th_bf.float(), tok, bf16=True, dtype=torch.float32)
    l64, g64 = lm_replica.llama_loss_and_grad(LLAMA1B, th_bf.double(), tok)
    per16, per64, rep64 = _per_tensor_llama(g, g16), _per_tensor_llama(g, g64), _per_tensor_llama(g16, g64)
    for name in per16:
        print(f"{name:34s} kernel vs bf16 replica {per16[name]:.2e}   kernel vs fp64 {per64[name]:.2e}   "
              f"replica vs fp64 {rep64[name]:.2e}")
    print("loss", loss_sum, l16.item(), l64.item())
    assert abs(loss_sum - l16.item()) <= 2e-3 * abs(l16.item())
    # d = 2048 and T = 2048 chains carry more bf16 rounding than GPT-2 small:
    # the replica itself sits 1.6-2.9e-2 from fp64 per tensor (measured), so
    # the kernel-vs-replica bound is 3e-2 here; the decisive check is the
    # next one — the kernel's fp64 error is the bf16-storage error (measured
    # ratio 1.00-1.02), nothing on top
    assert not {k: v for k, v in per16.items() if not v <= 3e-2}
    assert not {k: (per64[k], rep64[k]) for k in per64 if not per64[k] <= 1.5 * rep64[k] + 1e-3}
    del g16, g64
    torch.cuda.empty_cache()
    # fp32 parity path (3xTF32 GEMMs) at the same shapes
    m = api.Model(api.LMConfig(**LLAMA1B, precision="fp32", max_batch=LB))
    pt = torch.tensor(th, device=cuda)
    g, loss_sum, _ = _kernel_grad(m, pt, seed, LB, cuda)
    del m
    l64, g64 = lm_replica.llama_loss_and_grad(LLAMA1B, pt.double(), tok)
    per = _per_tensor_llama(g, g64)
    print("fp32 overall", _rel(g, g64), "worst", max(per.values()), "loss", loss_sum, l64.item())
    assert abs(loss_sum - l64.item()) <= 1e-6 * abs(l64.item())
    assert _rel(g, g64) <= 1e-5
    assert not {k: v for k, v in per.items() if not v <= 1e-5}
