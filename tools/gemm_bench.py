"""Per-shape timing of the tcgen05 GEMM on the GPT-2 small training shapes
(M = 8 x 1024 tokens). Prints TFLOP/s per (shape, layout). CUDA events,
warm-up, inputs > L2 are not needed here (kernel-level microbench)."""
import json
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2406_02613_b200.ops import gemm  # noqa: E402

M = 8192
d = int(sys.argv[1]) if len(sys.argv) > 1 else 768
V = 50257
SHAPES = [
    # name, m, n, k, a_mn, b_mn, mode
    ("qkv_fwd", M, 3 * d, d, False, False, "store"),
    ("proj_fwd", M, d, d, False, False, "store"),
    ("fc_fwd", M, 4 * d, d, False, False, "gelu"),
    ("fc2_fwd", M, d, 4 * d, False, False, "store"),
    ("head_fwd", M, V, d, False, False, "store"),
    ("head_dgrad", M, d, V, False, True, "store"),
    ("head_wgrad", V, d, M, True, True, "acc_f32"),
    ("fc2_dgrad", M, 4 * d, d, False, True, "dgelu"),
    ("fc2_wgrad", d, 4 * d, M, True, True, "acc_f32"),
    ("fc_wgrad", 4 * d, d, M, True, True, "acc_f32"),
    ("fc_dgrad", M, d, 4 * d, False, True, "store"),
    ("qkv_wgrad", 3 * d, d, M, True, True, "acc_f32"),
    ("qkv_dgrad", M, d, 3 * d, False, True, "store"),
    ("proj_wgrad", d, d, M, True, True, "acc_f32"),
    # epilogue-cost probes: the same shapes with the plain store epilogue
    ("fc_fwd_store", M, 4 * d, d, False, False, "store"),
    ("fc2_dgrad_store", M, 4 * d, d, False, True, "store"),
]


def main():
    dev = torch.device("cuda")
    out = []
    tot_ms = tot_fl = 0.0
    only = sys.argv[2].split(",") if len(sys.argv) > 2 else None
    for name, m, n, k, amn, bmn, mode in SHAPES:
        if only and name not in only:
            continue
        def mat(r, c):  # row stride padded to 64 elements (TMA needs 16B-multiple strides)
            return torch.randn(r, (c + 63) // 64 * 64, device=dev).to(torch.bfloat16)[:, :c]

        a = mat(k, m) if amn else mat(m, k)
        b = mat(k, n) if bmn else mat(n, k)
        ldc = (n + 63) // 64 * 64
        if mode == "acc_f32":
            c = torch.zeros(m, ldc, device=dev)
        else:
            c = torch.empty(m, ldc, dtype=torch.bfloat16, device=dev)
        aux = torch.randn(m, ldc, device=dev).to(torch.bfloat16) if mode in ("gelu", "dgelu") else None
        kw = dict(mode=mode, aux=aux, beta=1 if mode == "acc_f32" else 0)
        for _ in range(3):
            gemm(a, amn, b, bmn, m, n, k, c, **kw)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record()
        for _ in range(reps):
            gemm(a, amn, b, bmn, m, n, k, c, **kw)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        fl = 2.0 * m * n * k
        tot_ms += ms
        tot_fl += fl
        out.append({"name": name, "m": m, "n": n, "k": k, "ms": round(ms, 4), "tflops": round(fl / ms / 1e9, 1)})
        print(json.dumps(out[-1]), flush=True)
    print(json.dumps({"total_ms": tot_ms, "avg_tflops": tot_fl / tot_ms / 1e9}))


if __name__ == "__main__":
    main()
