"""Debug: which gradient tensors differ between repeated / fused / separate runs (d = 256 GPT-2)."""
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
d = int(sys.argv[1]) if len(sys.argv) > 1 else 256
c = dict(vocab=96, d_model=d, n_layer=2, n_head=max(1, d // 64), seq_len=128, n_samples=8, data_seed=4)
m = api.Model(api.LMConfig(**c, precision="bf16", max_batch=3))
gc = G.GPTConfig(**c)
rng = np.random.default_rng(5)
th = torch.tensor(G.default_theta0(gc, 2) + 0.02 * rng.standard_normal(m.dim)).to(torch.bfloat16).to(cuda)
seed = O.derive(4, 0, 0, 3, 0)
runs = {"f1": _grad(m, th, seed, 3, cuda)[0], "f2": _grad(m, th, seed, 3, cuda)[0]}
os.environ["ACCO_LN_PARAMS_SEPARATE"] = "1"
m2 = api.Model(api.LMConfig(**c, precision="bf16", max_batch=3))
runs["lnsep"] = _grad(m2, th, seed, 3, cuda)[0]
for a, b in [("f1", "f2"), ("f1", "lnsep")]:
    diff = []
    for name, shape, _k, off in G.param_layout(gc):
        n = int(np.prod(shape))
        x, y = runs[a][off:off + n], runs[b][off:off + n]
        if not np.array_equal(x, y):
            diff.append((name, float(np.abs(x - y).max()), int((x != y).sum())))
    print(a, "vs", b, diff)
