"""GEMM kernel duration (CUPTI, inside a CUDA graph, PDL off) by what ran
before it: the same GEMM (warm), a copy kernel rewriting A (producer), a
512 MB write (cold L2). Diagnostic only: run with ACCO_NO_PDL=1."""
import json
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2406_02613_b200.ops import gemm  # noqa: E402

dev = torch.device("cuda")
M = 8192
SH = {"proj_fwd": (M, 768, 768), "fc2_fwd": (M, 768, 3072), "qkv_fwd": (M, 2304, 768), "fc_fwd": (M, 3072, 768)}
flush = torch.empty(512 * 1024 * 1024 // 4, device=dev)
cs = torch.cuda.Stream()


def gemm_durs(body):
    with torch.cuda.stream(cs):
        body()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=cs):
        for _ in range(10):
            body()
    g.replay()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        g.replay()
        torch.cuda.synchronize()
    d = sorted(e.time_range.end - e.time_range.start for e in prof.events()
               if e.device_type.name == "CUDA" and "gemm_tc" in e.name)
    return round(d[len(d) // 2], 2)


for name, (m, n, k) in SH.items():
    a = torch.randn(m, k, device=dev).to(torch.bfloat16)
    a_src = a.clone()
    b = torch.randn(n, k, device=dev).to(torch.bfloat16)
    c = torch.empty(m, n, dtype=torch.bfloat16, device=dev)
    run = lambda: gemm(a, False, b, False, m, n, k, c)  # noqa: E731
    out = {"name": name}
    out["warm"] = gemm_durs(run)
    out["producer_writes_A"] = gemm_durs(lambda: (a.copy_(a_src), run()))
    out["cold_l2"] = gemm_durs(lambda: (flush.fill_(1.0), run()))
    out["cold_then_A"] = gemm_durs(lambda: (flush.fill_(1.0), a.copy_(a_src), run()))
    print(json.dumps(out), flush=True)
