"""The torch LM replica (tests/lm_replica.py) against the fp64 numpy oracle
(oracle/gpt_oracle.py) on CPU: in fp64 without rounding it is the same math
(<= 1e-10); in bf16-matched mode it stays within bf16 distance. This pins the
replica before the GPU tests use it as the fp64 / bf16-matched reference at
the benchmark shapes (tests/test_gpu_bench_shapes.py)."""
import numpy as np
import pytest
import torch

from oracle import accosim_oracle as O
from oracle import gpt_oracle as G
from tests import lm_replica

CFGS = {
    "tiny": dict(vocab=64, d_model=32, n_layer=2, n_head=2, seq_len=16, n_samples=32, data_seed=3),
    "ragged": dict(vocab=100, d_model=64, n_layer=1, n_head=1, seq_len=24, n_samples=16, data_seed=9),
    "c1": dict(vocab=256, d_model=128, n_layer=2, n_head=4, seq_len=64, n_samples=64, data_seed=1),
}


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)


@pytest.mark.parametrize("name", list(CFGS))
def test_replica_fp64_is_the_oracle(name):
    c = CFGS[name]
    gc = G.GPTConfig(**c)
    rng = np.random.default_rng(4)
    th = G.default_theta0(gc, 3) + 0.03 * rng.standard_normal(G.param_count(gc))
    idx = O.sample_indices(O.derive(3, 0, 1, 2, 0), 3, gc.n_samples)
    tok = G.dataset(gc)[idx]
    ol, og = G.loss_and_grad(gc, th, tok)
    rl, rg = lm_replica.loss_and_grad(c, torch.tensor(th), torch.tensor(tok))
    assert abs(rl.item() / 3 - ol) <= 1e-12 * abs(ol)
    assert _rel(rg.numpy() / 3, og) <= 1e-10
    # same flat layout as the oracle
    assert [(n, s, o) for n, s, _, o in G.param_layout(gc)] == lm_replica.param_layout(c)


def test_replica_bf16_mode_near_fp64():
    c = CFGS["c1"]
    gc = G.GPTConfig(**c)
    th = G.default_theta0(gc, 1)
    tok = torch.tensor(G.dataset(gc)[:4])
    th_bf = torch.tensor(th).to(torch.bfloat16).double()
    l64, g64 = lm_replica.loss_and_grad(c, th_bf, tok)
    l16, g16 = lm_replica.loss_and_grad(c, th_bf.float(), tok, bf16=True, dtype=torch.float32)
    assert abs(l16.item() - l64.item()) <= 1e-2 * abs(l64.item())
    assert _rel(g16.double().numpy(), g64.numpy()) <= 5e-2


LLAMA = dict(vocab=96, d_model=64, n_layer=2, n_head=4, seq_len=24, n_samples=16, data_seed=2, arch="llama",
             n_kv_head=2, d_ff=96)


def test_llama_replica_fp64_is_the_oracle():
    gc = G.GPTConfig(**LLAMA)
    rng = np.random.default_rng(5)
    th = G.default_theta0(gc, 4) + 0.03 * rng.standard_normal(G.param_count(gc))
    tok = G.dataset(gc)[:3]
    ol, og = G.loss_and_grad(gc, th, tok)
    rl, rg = lm_replica.llama_loss_and_grad(LLAMA, torch.tensor(th), torch.tensor(tok))
    assert abs(rl.item() / 3 - ol) <= 1e-12 * abs(ol)
    assert _rel(rg.numpy() / 3, og) <= 1e-10
    assert [(n, s, o) for n, s, _, o in G.param_layout(gc)] == lm_replica.llama_param_layout(LLAMA)


def test_llama_replica_bf16_mode_near_fp64():
    gc = G.GPTConfig(**LLAMA)
    th_bf = torch.tensor(G.default_theta0(gc, 1)).to(torch.bfloat16).double()
    tok = torch.tensor(G.dataset(gc)[:4])
    l64, g64 = lm_replica.llama_loss_and_grad(LLAMA, th_bf, tok)
    l16, g16 = lm_replica.llama_loss_and_grad(LLAMA, th_bf.float(), tok, bf16=True, dtype=torch.float32)
    assert abs(l16.item() - l64.item()) <= 1e-2 * abs(l64.item())
    assert _rel(g16.double().numpy(), g64.numpy()) <= 5e-2
