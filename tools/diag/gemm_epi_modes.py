"""Epilogue-mode cost on the GPT-2-small MLP shapes: the same GEMM as a plain
store, with the forward GELU epilogue (writes gelu(x) and the slope) and with
the dGELU epilogue (reads the slope). CUDA graph of 10 launches, min over 5
rounds. Diagnostic only."""
import json
import os
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2406_02613_b200.ops import gemm  # noqa: E402

dev = torch.device("cuda")
cs = torch.cuda.Stream()


def graph_us(run):
    with torch.cuda.stream(cs):
        run()
        run()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=cs):
        for _ in range(10):
            run()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 100)
    return round(best, 2)


M, F, d = 8192, 3072, 768
x = torch.randn(M, d, device=dev).to(torch.bfloat16)
w_fc = torch.randn(F, d, device=dev).to(torch.bfloat16)  # [out, in]
h = torch.empty(M, F, dtype=torch.bfloat16, device=dev)
aux = torch.empty(M, F, dtype=torch.bfloat16, device=dev)
dy = torch.randn(M, d, device=dev).to(torch.bfloat16)
w_fc2 = torch.randn(d, F, device=dev).to(torch.bfloat16)  # [out = d, in = F]
dh = torch.empty(M, F, dtype=torch.bfloat16, device=dev)
out = {}
for force in (None, "192,1,2", "256,1,2", "192,1,1", "256,1,1", "128,1,2"):
    if force:
        os.environ["ACCO_GEMM_FORCE"] = force
    else:
        os.environ.pop("ACCO_GEMM_FORCE", None)
    k = force or "auto"
    try:
        out[k] = {
            "fc_fwd_store": graph_us(lambda: gemm(x, False, w_fc, False, M, F, d, h)),
            "fc_fwd_gelu": graph_us(lambda: gemm(x, False, w_fc, False, M, F, d, h, mode="gelu", aux=aux)),
            # dH = dY W_fc2 : B = W_fc2 [d, F] read MN-major (n = F along its rows' contiguous dim)
            "fc2_dgrad_store": graph_us(lambda: gemm(dy, False, w_fc2, True, M, F, d, dh)),
            "fc2_dgrad_dgelu": graph_us(lambda: gemm(dy, False, w_fc2, True, M, F, d, dh, mode="dgelu", aux=aux)),
        }
    except Exception as e:  # noqa: BLE001
        out[k] = str(e)[:100]
    print(json.dumps({k: out[k]}), flush=True)
