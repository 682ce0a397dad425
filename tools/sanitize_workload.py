"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
every tcgen05 GEMM tile configuration (BN 128/192/256 on one SM or a CTA
pair, ordered split-K, the fp32-workspace split, the 3xTF32 fp32 path) with
all epilogues and the fused bias gradient, and one bf16
micro-batch (forward + backward) of a GPT-2-shaped LM at head size 64, so the
four tcgen05 attention kernels (fa_fwd_tc2, fa_bwd_dkv_tc, fa_bwd_dq_tc,
dsum_tc_kernel; and at head size 128), the LN / CE / embedding kernels and the
fused AdamW run.

  compute-sanitizer --tool memcheck python tools/sanitize_workload.py
"""
import ctypes as C
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2406_02613_b200 import _lib, api  # noqa: E402
from paper_2406_02613_b200.ops import gemm, gemm_bias_grad  # noqa: E402

dev = torch.device("cuda")
g = torch.Generator().manual_seed(0)
m, n, k = 384, 520, 320
for force in ("128,1", "192,1", "256,1", "192,3", "128,4", "256,1,2", "128,1,2", "256,3,2", "192,1,2", None):
    if force:
        os.environ["ACCO_GEMM_FORCE"] = force
    else:
        os.environ.pop("ACCO_GEMM_FORCE", None)
    for a_mn in (False, True):
        for b_mn in (False, True):
            if force == "192,1,2" and b_mn:
                continue  # (pair tiles of width 192 need a K-major B)
            a = torch.randn(m, k, generator=g).to(torch.bfloat16).to(dev)
            b = torch.randn(n, k, generator=g).to(torch.bfloat16).to(dev)
            a_st = a.t().contiguous() if a_mn else a
            b_st = b.t().contiguous() if b_mn else b
            c = torch.empty(m, n, dtype=torch.bfloat16, device=dev)
            gemm(a_st, a_mn, b_st, b_mn, m, n, k, c)
            c32 = torch.zeros(m, n, device=dev)
            gemm(a_st, a_mn, b_st, b_mn, m, n, k, c32, mode=3, beta=1)
            aux = torch.empty(m, n, dtype=torch.bfloat16, device=dev)
            gemm(a_st, a_mn, b_st, b_mn, m, n, k, c, mode=1, aux=aux, bias=torch.zeros(n, dtype=torch.bfloat16,
                                                                                      device=dev))
            gemm(a_st, a_mn, b_st, b_mn, m, n, k, c, mode=2, aux=aux)
            if force is None or not force.startswith("256"):  # weight gradient + fused bias gradient
                bg = torch.zeros(m, device=dev)
                gemm_bias_grad(a_st, a_mn, b_st, b_mn, m, n, k, c32, bg, beta=1)
os.environ.pop("ACCO_GEMM_FORCE", None)
# pure-store split into the fp32 workspace (long K, few tiles)
a = torch.randn(256, 8192, generator=g).to(torch.bfloat16).to(dev)
b = torch.randn(8192, 128, generator=g).to(torch.bfloat16).to(dev)
c = torch.empty(256, 128, dtype=torch.bfloat16, device=dev)
gemm(a, False, b, True, 256, 128, 8192, c)
# fp32 (3xTF32) path: direct accumulate, scratch + epilogue, split-K
for (mm, nn, kk) in ((200, 136, 72), (128, 256, 1000)):
    a = torch.randn(mm, kk, generator=g).to(dev)
    b = torch.randn(nn, kk, generator=g).to(dev)
    c = torch.empty(mm, nn, device=dev)
    gemm(a, False, b, False, mm, nn, kk, c)
    gemm(a, False, b.t().contiguous(), True, mm, nn, kk, c, mode=3, beta=1)
torch.cuda.synchronize()
# one bf16 ACCO update of a small GPT (tcgen05 attention at hd = 64, T = 256;
# d = 256: the fused norm backward with its parameter partials and the fold)
lm = api.LMConfig(vocab=128, d_model=256, n_layer=1, n_head=4, seq_len=256, n_samples=8, precision="bf16",
                  max_batch=2)
opt = api.OptimizerConfig(kind="adamw", learning_rate=1e-3, adam_beta2=0.95)
tr = api.run_protocol("acco", lm, opt, api.SimConfig(n_workers=1, batch_size=2, master_seed=1), 1)
torch.cuda.synchronize()
# head size 128 on the tcgen05 attention kernels (fa_fwd_tc2<128>, fa_bwd_dq_tc<128>, fa_bwd_dkv_tc<128>)
lm128 = api.LMConfig(vocab=128, d_model=256, n_layer=1, n_head=2, seq_len=256, n_samples=8, precision="bf16",
                     max_batch=2)
tr128 = api.run_protocol("acco", lm128, opt, api.SimConfig(n_workers=1, batch_size=2, master_seed=1), 1)
torch.cuda.synchronize()
# ragged T (T % 4 != 0): dK/dV lse / D through per-lane cp.async on the stage barrier
lm_r = api.LMConfig(vocab=128, d_model=256, n_layer=1, n_head=4, seq_len=141, n_samples=8, precision="bf16",
                    max_batch=2)
tr_r = api.run_protocol("acco", lm_r, opt, api.SimConfig(n_workers=1, batch_size=2, master_seed=1), 1)
torch.cuda.synchronize()
print("sanitize workload done", tr.records[0].loss, tr128.records[0].loss, tr_r.records[0].loss, flush=True)
