"""GEMM time by L2 state: warm (back-to-back launches), cold (a 512 MB
write evicts L2 before each launch) and producer-warm (A rewritten by a copy
kernel right before each launch, as in the training step), for every tile
config of the GPT-2-small shapes. Device time of the GEMM alone (CUDA events
around it), interleaved rounds, min. Diagnostic only."""
import json
import os
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2406_02613_b200.ops import gemm  # noqa: E402

dev = torch.device("cuda")
M = 8192
SHAPES = [("qkv_fwd", M, 2304, 768, 0, 0, "store"), ("proj_fwd", M, 768, 768, 0, 0, "store"),
          ("fc_fwd", M, 3072, 768, 0, 0, "store"), ("fc2_fwd", M, 768, 3072, 0, 0, "store"),
          ("fc_dgrad", M, 768, 3072, 0, 1, "store"), ("qkv_dgrad", M, 768, 2304, 0, 1, "store"),
          ("fc2_wgrad", 768, 3072, M, 1, 1, "acc_f32"), ("fc_wgrad", 3072, 768, M, 1, 1, "acc_f32"),
          ("proj_wgrad", 768, 768, M, 1, 1, "acc_f32")]
only = sys.argv[1].split(",") if len(sys.argv) > 1 else None
flush = torch.empty(512 * 1024 * 1024 // 4, device=dev)
ROUNDS = 5


def t_one(run, pre):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(200000)  # the GPU is busy while the host queues the rest
    if pre:
        pre()
    e0.record()
    run()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3


for name, m, n, k, amn, bmn, mode in SHAPES:
    if only and name not in only:
        continue

    def mat(r, c):
        return torch.randn(r, (c + 63) // 64 * 64, device=dev).to(torch.bfloat16)[:, :c]
    a = mat(k, m) if amn else mat(m, k)
    a_src = a.clone()
    b = mat(k, n) if bmn else mat(n, k)
    ldc = (n + 63) // 64 * 64
    c = torch.zeros(m, ldc, device=dev) if mode == "acc_f32" else torch.empty(m, ldc, dtype=torch.bfloat16, device=dev)
    kw = dict(mode=mode, beta=1 if mode == "acc_f32" else 0)
    cfgs = ["auto"]
    for cg in (1, 2):
        for bn in (256, 192, 128):
            if cg == 2 and bn == 192 and bmn:
                continue
            for sp in ((1, 2, 3) if mode == "acc_f32" else (1,)):
                cfgs.append(f"{bn},{sp},{cg}")
    res = {cfg: {"warm": 1e9, "cold": 1e9, "prod": 1e9} for cfg in cfgs}
    pres = {"warm": None, "cold": lambda: flush.fill_(1.0), "prod": lambda: a.copy_(a_src)}
    for _ in range(ROUNDS):
        for cfg in cfgs:
            if cfg == "auto":
                os.environ.pop("ACCO_GEMM_FORCE", None)
            else:
                os.environ["ACCO_GEMM_FORCE"] = cfg
            try:
                run = lambda: gemm(a, bool(amn), b, bool(bmn), m, n, k, c, **kw)  # noqa: E731
                for st, pre in pres.items():
                    run()
                    res[cfg][st] = min(res[cfg][st], t_one(run, pre))
            except Exception as e:  # noqa: BLE001
                res[cfg] = str(e)[:60]
    os.environ.pop("ACCO_GEMM_FORCE", None)
    out = {"name": name, "shape": [m, n, k, amn, bmn, mode]}
    for cfg, v in res.items():
        out[cfg] = v if isinstance(v, str) else {s: round(x, 2) for s, x in v.items()}
    print(json.dumps(out), flush=True)
