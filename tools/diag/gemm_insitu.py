"""In-situ GEMM kernel times of one GPT-2-small micro-batch (CUPTI via
torch.profiler), in launch order, grouped by position in the layer pattern,
next to the isolated CUDA-graph times of profiles/r02_gemm_model.jsonl.
Diagnostic only."""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from oracle import accosim_oracle as O  # noqa: E402
from paper_2406_02613_b200 import _lib, api  # noqa: E402

cuda = torch.device("cuda")
cfg = dict(vocab=50257, d_model=768, n_layer=12, n_head=12, seq_len=1024)
m = api.Model(api.LMConfig(**cfg, n_samples=256, data_seed=1, precision="bf16", max_batch=8))
th = torch.tensor(m.default_theta0(1)).to(torch.bfloat16).to(cuda)
g = torch.zeros(m.dim, device=cuda)
loss = torch.zeros(1, dtype=torch.float64, device=cuda)
s = torch.cuda.current_stream()


def mb():
    _lib.call("acco_model_stochastic_grad", m.handle, C.c_void_p(th.data_ptr()), C.c_uint64(O.derive(1, 0, 0, 8, 0)), 8,
              C.c_void_p(g.data_ptr()), C.c_void_p(loss.data_ptr()), C.c_void_p(s.cuda_stream))


for _ in range(3):
    mb()
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

runs = []
for _ in range(3):
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        mb()
        torch.cuda.synchronize()
    ks = []
    for e in prof.events():
        if e.device_type.name != "CUDA":
            continue
        try:
            ks.append((e.time_range.start, e.time_range.end, e.name))
        except Exception:
            pass
    ks.sort()
    runs.append(ks)
# all kernels of the first run with durations, then per-position medians over runs
seqs = [[(n, b - a) for a, b, n in ks] for ks in runs]
tag = os.environ.get("TAG", "")
out = []
for i, (n, d) in enumerate(seqs[0]):
    ds = sorted(sq[i][1] for sq in seqs if i < len(sq) and sq[i][0] == n)
    out.append({"i": i, "k": n.replace("void ", "").replace("acco::(anonymous namespace)::", "")[:40],
                "us": round(ds[len(ds) // 2], 2)})
print(json.dumps({"tag": tag, "kernels": out}))
