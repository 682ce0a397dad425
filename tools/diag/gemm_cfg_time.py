"""Interleaved timing of forced GEMM configs on one shape:
python gemm_cfg_time.py M N K a_mn b_mn mode cfg1 cfg2 ... (cfg '' = auto)."""
import json
import os
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2406_02613_b200.ops import gemm  # noqa: E402

dev = torch.device("cuda")


def main():
    m, n, k, amn, bmn = (int(x) for x in sys.argv[1:6])
    mode = sys.argv[6]
    cfgs = sys.argv[7:]

    def mat(r, c):
        return torch.randn(r, (c + 63) // 64 * 64, device=dev).to(torch.bfloat16)[:, :c]
    a = mat(k, m) if amn else mat(m, k)
    b = mat(k, n) if bmn else mat(n, k)
    ldc = (n + 63) // 64 * 64
    c = torch.zeros(m, ldc, device=dev) if mode == "acc_f32" else torch.empty(m, ldc, dtype=torch.bfloat16, device=dev)
    aux = torch.randn(m, ldc, device=dev).to(torch.bfloat16) if mode in ("gelu", "dgelu") else None
    kw = dict(mode=mode, aux=aux, beta=1 if mode == "acc_f32" else 0)
    fl = 2.0 * m * n * k
    res = {c_: [] for c_ in cfgs}
    cs = torch.cuda.Stream()  # the capture stream (per-stream GEMM scratch is set up in the warm-up)
    for rnd in range(5):
        for cfg in cfgs:
            if cfg in ("auto", ""):
                os.environ.pop("ACCO_GEMM_FORCE", None)
            else:
                os.environ["ACCO_GEMM_FORCE"] = cfg
            with torch.cuda.stream(cs):
                for _ in range(3):
                    gemm(a, bool(amn), b, bool(bmn), m, n, k, c, **kw)
            torch.cuda.synchronize()
            # a CUDA graph of `reps` launches: device time, not the host's launch rate
            reps = 20
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=cs):
                for _ in range(reps):
                    gemm(a, bool(amn), b, bool(bmn), m, n, k, c, **kw)
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            res[cfg].append(e0.elapsed_time(e1) / reps * 1e3)
    print(json.dumps({"shape": [m, n, k, amn, bmn, mode],
                      **{c_: {"us_min": round(min(v), 2), "us_med": round(sorted(v)[2], 2),
                              "tflops": round(fl / min(v) / 1e6, 1)} for c_, v in res.items()}}), flush=True)


if __name__ == "__main__":
    main()
