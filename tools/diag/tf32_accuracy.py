"""Accuracy of the fp32 GEMM paths vs fp64 as K grows: 3xTF32 tcgen05 (with
and without a capped TMEM accumulation chain), the SIMT kernel, and one bf16
pass. Prints one JSON line per (K, variant)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2406_02613_b200.ops import gemm  # noqa: E402


def rel(a, b):
    return ((a.double() - b).norm() / b.norm()).item()


dev = torch.device("cuda")
for K in (64, 256, 1024, 4096, 8192, 16384, 65536):
    m = n = 256
    g = torch.Generator().manual_seed(K)
    for dist in ("randn", "pos"):
        a = torch.randn(m, K, generator=g)
        b = torch.randn(n, K, generator=g)
        if dist == "pos":
            a, b = a.abs(), b.abs()
        a, b = a.to(dev), b.to(dev)
        ref = a.double() @ b.double().t()
        out = {"K": K, "dist": dist}
        for name, env in (("x3", {}), ("x3_unsplit", {"ACCO_TF32_CHAIN": "100000"}),
                          ("x3_chain16", {"ACCO_TF32_CHAIN": "16"}), ("simt", {"ACCO_GEMM_SIMT": "1"})):
            for k_, v in env.items():
                os.environ[k_] = v
            c = torch.empty(m, n, device=dev)
            gemm(a, False, b, False, m, n, K, c)
            torch.cuda.synchronize()
            out[name] = rel(c, ref)
            for k_ in env:
                del os.environ[k_]
        cb = torch.empty(m, n, device=dev)
        gemm(a.bfloat16(), False, b.bfloat16(), False, m, n, K, cb, mode=3)
        torch.cuda.synchronize()
        out["bf16"] = rel(cb, ref)
        print(json.dumps(out), flush=True)
