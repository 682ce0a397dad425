"""Kernel timeline of one GPT-2-small micro-batch in situ (torch.profiler /
CUPTI): per-class device time, gaps between consecutive compute-stream
kernels, and the in-situ vs isolated kernel times."""
import collections
import ctypes as C
import json
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

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    mb()
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type.name == "CUDA" and e.name not in ("Activity Buffer Request",)]
ks = []
for e in evs:
    try:
        ks.append((e.time_range.start, e.time_range.end, e.name))
    except Exception:
        pass
ks.sort()
t0, t1 = ks[0][0], max(k[1] for k in ks)
cls = collections.defaultdict(float)
def klass(n):
    for key in ("gemm_tc_kernel", "fa_fwd", "fa_bwd_dkv", "fa_bwd_dq", "dsum", "ln_fwd", "ln_bwd", "ln_param_fold", "ce_vec",
                "embed", "radix", "gather", "loss_reduce", "colsum", "f32_to_bf16"):
        if key in n:
            return key
    return n[:30]
for a, b, n in ks:
    cls[klass(n)] += b - a
# union of busy time and gaps
busy = 0.0
cur_a, cur_b = ks[0][0], ks[0][1]
gaps = []
for a, b, n in ks[1:]:
    if a > cur_b:
        busy += cur_b - cur_a
        gaps.append((a - cur_b, n))
        cur_a, cur_b = a, b
    else:
        cur_b = max(cur_b, b)
busy += cur_b - cur_a
gaps.sort(reverse=True)
out = {"span_us": t1 - t0, "busy_us": busy, "sum_kernel_us": sum(b - a for a, b, _ in ks), "kernels": len(ks),
       "gaps_total_us": sum(g for g, _ in gaps), "n_gaps": len(gaps),
       "largest_gaps": [(round(g, 1), n[:40]) for g, n in gaps[:8]],
       "per_class_us": {k: round(v, 1) for k, v in sorted(cls.items(), key=lambda x: -x[1])}}
print(json.dumps(out, indent=1))
