"""CPU-only checks of the C-ABI boundary: the library loads, exports every
symbol include/acco.h declares, and its host-side integer/scalar functions
(shards, rng, token indexing, LR schedule) are bit-exact against the
reference golden vectors. No CUDA device is touched."""
import json
import os
import re

import pytest

from paper_2406_02613_b200 import _lib, api

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def declared_symbols():
    with open(os.path.join(ROOT, "include", "acco.h")) as f:
        src = f.read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(acco_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    syms = declared_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert lib.acco_version() == 2  # ABI 2: acco_run_stats.n_records (partial traces)


def test_shard_partition_bitexact():
    for c in _load("shard.json"):
        if c["n"] >= 1:
            assert [list(r) for r in api.shard_partition(c["dim"], c["n"])] == c["ranges"]
    with pytest.raises(api.InvalidArgument):
        api.shard_partition(4, 0)


def test_rng_and_token_indexing_bitexact():
    g = _load("rng.json")
    for m, a, b, c, d, out in g["derive"]:
        assert api.derive(m, a, b, c, d) == out
    for e in g["streams"]:
        # below(n) after 24 draws is pinned by the golden stream; the index
        # draw itself is Stream(seed).below(n) x B
        from oracle.accosim_oracle import sample_indices

        assert api.sample_indices(e["seed"], 16, 4096) == sample_indices(e["seed"], 16, 4096)


def test_scheduled_lr_matches_reference():
    for c in _load("lr.json"):
        cfg = api.OptimizerConfig(**{k: c["cfg"][k] for k in c["cfg"]})
        got = [api.scheduled_lr(cfg, t) for t in range(110)]
        assert got == c["lr"]


def test_parse_config_schema_and_validation():
    j = {"problem": {"kind": "gpt", "vocab": 256, "d_model": 128, "n_layer": 2, "n_head": 4, "seq_len": 64,
                     "seed": 3},
         "method_name": "acco", "optimizer": {"kind": "adamw", "learning_rate": 6e-4, "weight_decay": 0.1,
                                              "adam_beta2": 0.95, "scheduler": "cosine"},
         "n_workers": 2, "batch_size": 8, "t_updates": 200, "master_seed": 1}
    cfg = api.parse_config(j)
    assert cfg.optimizer.total_steps == 200 and cfg.optimizer.adam_beta2 == 0.95
    assert cfg.sim.n_workers == 2 and cfg.problem.data_seed == 3
    for bad in ({"t_updates": 0}, {"n_workers": 0}, {"batch_size": 0}, {"method_name": "xyz"},
                {"optimizer": {"kind": "adamw", "learning_rate": 0.0}},
                {"optimizer": {"kind": "adamw", "learning_rate": 1.0, "adam_beta1": 1.0}},
                {"optimizer": {"kind": "adamw", "learning_rate": 1.0, "scheduler": "linear"}},
                {"heterogeneity": {"worker_multipliers": [1, 1, 4]}}):
        with pytest.raises(api.InvalidArgument):
            api.parse_config({**j, **bad})
    with pytest.raises(api.InvalidArgument):
        api.parse_config({k: v for k, v in j.items() if k != "t_updates"})
    assert len(api.config_hash(j)) == 16


def test_parse_config_llama_problem():
    """problem.kind "llama" (BASELINE.json config C4) maps onto the Llama block."""
    j = {"problem": {"kind": "llama", "vocab": 32000, "d_model": 2048, "n_layer": 22, "n_head": 32, "n_kv_head": 4,
                     "d_ff": 5632, "seq_len": 2048, "rope_base": 10000.0, "precision": "bf16"},
         "method_name": "acco", "optimizer": {"kind": "adamw", "learning_rate": 3e-4},
         "n_workers": 8, "batch_size": 4, "t_updates": 10,
         "heterogeneity": {"worker_multipliers": [4, 1, 1, 1, 1, 1, 1, 1]}}
    cfg = api.parse_config(j)
    p = cfg.problem
    assert (p.arch, p.n_kv_head, p.d_ff, p.rope_base) == ("llama", 4, 5632, 10000.0)
    c = p.to_c()
    assert (c.arch, c.n_kv_head, c.d_ff) == (1, 4, 5632)
    assert cfg.sim.worker_multipliers == [4, 1, 1, 1, 1, 1, 1, 1]
    with pytest.raises(api.InvalidArgument):
        api.LMConfig(arch="mamba").to_c()
