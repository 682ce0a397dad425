"""Why a GEMM timed as one of 10 back-to-back launches in a CUDA graph is
faster than the same GEMM alone: per-kernel CUPTI durations inside the graph,
graph time / 10, and the single-launch event time. Run with and without
ACCO_NO_PDL=1. Diagnostic only."""
import json
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2406_02613_b200.ops import gemm  # noqa: E402

dev = torch.device("cuda")
M = 8192
SH = {"proj_fwd": (M, 768, 768), "fc2_fwd": (M, 768, 3072), "qkv_fwd": (M, 2304, 768)}
cs = torch.cuda.Stream()
for name, (m, n, k) in SH.items():
    a = torch.randn(m, k, device=dev).to(torch.bfloat16)
    b = torch.randn(n, k, device=dev).to(torch.bfloat16)
    c = torch.empty(m, n, dtype=torch.bfloat16, device=dev)
    run = lambda: gemm(a, False, b, False, m, n, k, c)  # noqa: E731
    with torch.cuda.stream(cs):
        run()
        run()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=cs):
        for _ in range(10):
            run()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 100)
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        g.replay()
        torch.cuda.synchronize()
    ks = []
    for e in prof.events():
        if e.device_type.name == "CUDA" and "gemm" in e.name:
            ks.append((e.time_range.start, e.time_range.end))
    ks.sort()
    durs = [round(b_ - a_, 1) for a_, b_ in ks]
    starts = [round(ks[i + 1][0] - ks[i][1], 1) for i in range(len(ks) - 1)]
    single = 1e9
    for _ in range(5):
        torch.cuda._sleep(200000)
        e0.record()
        run()
        e1.record()
        torch.cuda.synchronize()
        single = min(single, e0.elapsed_time(e1) * 1e3)
    print(json.dumps({"name": name, "pdl": os.environ.get("ACCO_NO_PDL") is None, "graph_per_launch_us": round(best, 2),
                      "cupti_durations_us": durs, "gaps_us": starts, "single_event_us": round(single, 2)}), flush=True)
