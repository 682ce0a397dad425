"""Debug: per-tensor differences between repeated llama d=2048 gradients."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from oracle import accosim_oracle as O  # noqa: E402
from oracle import gpt_oracle as G  # noqa: E402
from paper_2406_02613_b200 import api  # noqa: E402
from tests.test_gpu_model import _grad  # noqa: E402

cuda = torch.device("cuda")
d = 2048
c = dict(vocab=96, d_model=d, n_layer=1, n_head=d // 64, seq_len=64, n_samples=8, data_seed=2,
         arch="llama", n_kv_head=d // 128, d_ff=2 * d)
m = api.Model(api.LMConfig(**c, precision="bf16", max_batch=2))
gc = G.GPTConfig(**c)
rng = np.random.default_rng(3)
th = torch.tensor(G.default_theta0(gc, 1) + 0.02 * rng.standard_normal(m.dim)).to(torch.bfloat16)
seed = O.derive(2, 0, 0, 2, 0)
runs = {}
for tag, env in [("wide1", {}), ("wide2", {}), ("narrow", {"ACCO_LN_NARROW": "1"}),
                 ("serial", {"ACCO_SERIAL_REDUCE": "1"}), ("nocg2", {"ACCO_GEMM_NO_CG2": "1"}),
                 ("nopdl", {"ACCO_NO_PDL": "1"})]:
    for k in ("ACCO_LN_NARROW", "ACCO_SERIAL_REDUCE", "ACCO_GEMM_NO_CG2", "ACCO_NO_PDL"):
        os.environ.pop(k, None)
    os.environ.update(env)
    runs[tag] = _grad(m, th.to(cuda), seed, 2, cuda)
og, _, ol = G.LMProblem(gc).stochastic_grad(th.float().double().numpy(), seed, 2)
og = og * 2
segs = G.param_layout(gc) if hasattr(G, "param_layout") else None
print("layout", type(segs))
for tag, (g, l) in runs.items():
    rel = np.linalg.norm(g - og) / np.linalg.norm(og)
    print(tag, "loss", l, "rel vs oracle", rel)
    for tag2, (g2, _) in runs.items():
        if tag2 < tag:
            print("   vs", tag2, np.linalg.norm(g - g2) / np.linalg.norm(g2))
    if segs:
        worst = []
        for s in segs:
            name, off, n = s[0], s[3], int(np.prod(s[1]))
            a, b = g[off:off + n], og[off:off + n]
            worst.append((np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30), name))
        worst.sort(reverse=True)
        print("   worst tensors:", [(round(w, 4), nm) for w, nm in worst[:5]])
