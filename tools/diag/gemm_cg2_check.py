"""CTA-pair (cta_group::2) GEMM bring-up: correctness of every layout / epilogue
vs torch fp32 for forced tile configs, then TFLOP/s per GPT-2-small shape for
each config (ACCO_GEMM_FORCE='<bn>,<splits>,<cg>')."""
import itertools
import json
import os
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2406_02613_b200.ops import gemm  # noqa: E402

dev = torch.device("cuda")


def rel(a, b):
    return ((a.float() - b.float()).norm() / b.float().norm().clamp_min(1e-30)).item()


def operand(rows, k, mn, g):
    x = torch.randn(rows, k, generator=g).to(torch.bfloat16).to(dev)
    return (x, x.t().contiguous()) if mn else (x, x)


def check(force, m, n, k, a_mn, b_mn):
    os.environ["ACCO_GEMM_FORCE"] = force
    g = torch.Generator().manual_seed(m + n + k)
    a, ast = operand(m, k, a_mn, g)
    b, bst = operand(n, k, b_mn, g)
    ref = a.float() @ b.float().t()
    out = {}
    c = torch.empty(m, n, dtype=torch.bfloat16, device=dev)
    gemm(ast, a_mn, bst, b_mn, m, n, k, c)
    torch.cuda.synchronize()
    out["store"] = rel(c, ref)
    c32 = torch.randn(m, n, generator=g).to(dev)
    c0 = c32.clone()
    gemm(ast, a_mn, bst, b_mn, m, n, k, c32, mode=3, beta=1)
    torch.cuda.synchronize()
    out["acc"] = rel(c32, c0 + ref)
    aux = torch.empty(m, n, dtype=torch.bfloat16, device=dev)
    cg = torch.empty(m, n, dtype=torch.bfloat16, device=dev)
    gemm(ast, a_mn, bst, b_mn, m, n, k, cg, mode=1, aux=aux)
    torch.cuda.synchronize()
    out["gelu"] = rel(cg, torch.nn.functional.gelu(ref, approximate="tanh"))
    bias = torch.randn(n, generator=g).to(torch.bfloat16).to(dev)
    res = torch.randn(m, n, generator=g).to(torch.bfloat16).to(dev)
    gemm(ast, a_mn, bst, b_mn, m, n, k, c, bias=bias, residual=res)
    torch.cuda.synchronize()
    out["bias_res"] = rel(c, ref + bias.float() + res.float())
    ok = out["store"] < 6e-3 and out["acc"] < 2e-6 and out["gelu"] < 8e-3 and out["bias_res"] < 6e-3
    return ok, out


def main():
    bad = 0
    for force in ["256,1,2", "128,1,2", "192,1,2", "256,3,2", "128,4,2"]:
        for (m, n, k) in [(1000, 776, 520), (256, 256, 64), (2048, 1024, 1024), (800, 384, 96)]:
            for a_mn, b_mn in itertools.product([False, True], repeat=2):
                if force.startswith("192") and b_mn:
                    continue
                ok, out = check(force, m, n, k, a_mn, b_mn)
                bad += not ok
                print(json.dumps({"force": force, "shape": [m, n, k], "a_mn": a_mn, "b_mn": b_mn, "ok": ok,
                                  **{k2: round(v, 8) for k2, v in out.items()}}), flush=True)
    print(json.dumps({"correctness_failures": bad}), flush=True)
    # timing
    M, d, V = 8192, 768, 50257
    shapes = [("qkv_fwd", M, 3 * d, d, 0, 0, "store"), ("proj_fwd", M, d, d, 0, 0, "store"),
              ("fc_fwd", M, 4 * d, d, 0, 0, "gelu"), ("fc2_fwd", M, d, 4 * d, 0, 0, "store"),
              ("head_fwd", M, V, d, 0, 0, "store"),
              ("fc2_dgrad", M, 4 * d, d, 0, 1, "dgelu"), ("fc_dgrad", M, d, 4 * d, 0, 1, "store"),
              ("qkv_dgrad", M, d, 3 * d, 0, 1, "store"), ("proj_dgrad", M, d, d, 0, 1, "store"),
              ("fc2_wgrad", d, 4 * d, M, 1, 1, "acc_f32"), ("fc_wgrad", 4 * d, d, M, 1, 1, "acc_f32"),
              ("qkv_wgrad", 3 * d, d, M, 1, 1, "acc_f32"), ("proj_wgrad", d, d, M, 1, 1, "acc_f32"),
              ("head_wgrad", V, d, M, 1, 1, "acc_f32")]
    forces = ["", "256,1,2", "192,1,2", "128,1,2"]
    for name, m, n, k, amn, bmn, mode in shapes:
        def mat(r, c):
            return torch.randn(r, (c + 63) // 64 * 64, device=dev).to(torch.bfloat16)[:, :c]
        a = mat(k, m) if amn else mat(m, k)
        b = mat(k, n) if bmn else mat(n, k)
        ldc = (n + 63) // 64 * 64
        c = torch.zeros(m, ldc, device=dev) if mode == "acc_f32" else torch.empty(m, ldc, dtype=torch.bfloat16, device=dev)
        aux = torch.randn(m, ldc, device=dev).to(torch.bfloat16) if mode in ("gelu", "dgelu") else None
        row = {"name": name}
        fl = 2.0 * m * n * k
        for f in forces + (["256,2,2", "256,4,2", "128,2,2", "128,4,2"] if mode == "acc_f32" else []):
            if f.startswith("192") and bmn:
                continue
            if f:
                os.environ["ACCO_GEMM_FORCE"] = f
            else:
                os.environ.pop("ACCO_GEMM_FORCE", None)
            kw = dict(mode=mode, aux=aux, beta=1 if mode == "acc_f32" else 0)
            for _ in range(3):
                gemm(a, bool(amn), b, bool(bmn), m, n, k, c, **kw)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 10
            e0.record()
            for _ in range(reps):
                gemm(a, bool(amn), b, bool(bmn), m, n, k, c, **kw)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            row[f or "auto"] = round(fl / ms / 1e9, 1)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
