"""Repeatability of forced GEMM configs on short-K weight-gradient shapes."""
import itertools
import os
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2406_02613_b200.ops import gemm  # noqa: E402

dev = torch.device("cuda")


def run(m, n, k, amn, bmn, force, env=None, beta=1):
    os.environ.pop("ACCO_GEMM_NO_CLC", None)
    if env:
        os.environ.update(env)
    os.environ["ACCO_GEMM_FORCE"] = force
    g = torch.Generator().manual_seed(1)
    a = torch.randn(m, k, generator=g).to(torch.bfloat16).to(dev)
    b = torch.randn(n, k, generator=g).to(torch.bfloat16).to(dev)
    ast = a.t().contiguous() if amn else a
    bst = b.t().contiguous() if bmn else b
    ref = a.float() @ b.float().t()
    outs = []
    for _ in range(4):
        c = torch.zeros(m, n, device=dev)
        gemm(ast, amn, bst, bmn, m, n, k, c, mode=3, beta=beta)
        torch.cuda.synchronize()
        outs.append(c)
    rel = max(((o - ref).norm() / ref.norm()).item() for o in outs)
    same = all(torch.equal(outs[0], o) for o in outs)
    bad_rows = (outs[0] - ref).abs().amax(dim=1).gt(1e-2 * ref.abs().max()).nonzero().flatten()
    bad_cols = (outs[0] - ref).abs().amax(dim=0).gt(1e-2 * ref.abs().max()).nonzero().flatten()
    print(f"beta={beta} m={m} n={n} k={k} amn={amn} bmn={bmn} force={force} env={env} rel={rel:.2e} repeat_equal={same} "
          f"bad_rows={bad_rows[:4].tolist()}..{len(bad_rows)} bad_cols={bad_cols[:4].tolist()}..{len(bad_cols)}",
          flush=True)


for beta in (0, 1):
    for force in ("192,1", "256,1", "128,1"):
        run(4096, 2048, 128, 1, 1, force, beta=beta)
        run(8192, 2048, 128, 1, 1, force, beta=beta)
        run(8192, 2048, 1024, 1, 1, force, beta=beta)
