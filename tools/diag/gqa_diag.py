"""Per-tensor gradient error of the tcgen05 vs SIMT attention paths against the fp64 oracle (diagnostic)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from oracle import accosim_oracle as O  # noqa: E402
from oracle import gpt_oracle as G  # noqa: E402
from paper_2406_02613_b200 import _lib, api  # noqa: E402


def grad(m, th, seed, B):
    g = torch.zeros(m.dim, device="cuda")
    loss = torch.zeros(1, dtype=torch.float64, device="cuda")
    _lib.call("acco_model_stochastic_grad", m.handle, C.c_void_p(th.data_ptr()), C.c_uint64(seed), B,
              C.c_void_p(g.data_ptr()), C.c_void_p(loss.data_ptr()), C.c_void_p(torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    return g.double().cpu().numpy(), loss.item()


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30)


for seq, hkv, arch, amp in [(128, 2, "llama", 10), (320, 2, "llama", 10), (320, 2, "llama", 1), (320, 4, "gpt2", 10)]:
    c = dict(vocab=128, d_model=256, n_layer=1, n_head=4, seq_len=seq, n_samples=8, data_seed=6)
    if arch == "llama":
        c.update(arch="llama", n_kv_head=hkv, d_ff=256)
    m = api.Model(api.LMConfig(**c, precision="bf16", max_batch=2))
    gc = G.GPTConfig(**c)
    thf = torch.tensor(G.default_theta0(gc, 3) * amp).to(torch.bfloat16)
    th = thf.cuda()
    seed = O.derive(6, 0, 0, 2, 0)
    os.environ.pop("ACCO_ATTN_LEGACY", None)
    g_tc, l_tc = grad(m, th, seed, 2)
    os.environ["ACCO_ATTN_LEGACY"] = "1"
    g_s, l_s = grad(m, th, seed, 2)
    os.environ.pop("ACCO_ATTN_LEGACY", None)
    og, _, ol = G.LMProblem(gc).stochastic_grad(thf.float().double().numpy(), seed, 2)
    og *= 2
    print(f"seq {seq} hkv {hkv} {arch}: loss tc {l_tc/2:.6f} simt {l_s/2:.6f} oracle {ol:.6f}; "
          f"all: tc-vs-simt {rel(g_tc, g_s):.3e} tc-vs-oracle {rel(g_tc, og):.3e} simt-vs-oracle {rel(g_s, og):.3e}")
    for name, shape, _, off in G.param_layout(gc):
        n = int(np.prod(shape))
        if n < 1024:
            continue
        print(f"   {name:32s} tc {rel(g_tc[off:off+n], og[off:off+n]):.3e} simt {rel(g_s[off:off+n], og[off:off+n]):.3e}")
