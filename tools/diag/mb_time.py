"""Device time of one GPT-2-small micro-batch (fwd + bwd + accumulate, B = 8 x 1024)
in isolation (acco_model_time_micro_batch), with and without PDL."""
import json
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2406_02613_b200 import api  # noqa: E402

cfg = dict(vocab=50257, d_model=768, n_layer=12, n_head=12, seq_len=1024)
m = api.Model(api.LMConfig(**cfg, n_samples=256, data_seed=1, precision="bf16", max_batch=8))
m.time_micro_batch(8, 3)
ns = m.time_micro_batch(8, 20)
print(json.dumps({"micro_batch_ms": ns / 1e6, "tokens_per_s_compute_only": 8192 / (ns / 1e9)}))
