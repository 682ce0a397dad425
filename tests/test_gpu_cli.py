"""CLI run / sweep / verify on the GPU path (proj/tools/accosim_main.cpp):
output files with the reference's schema, reproducible manifests (the echoed
config reruns to the same trajectory, proj/tests/test_io.cpp:117-145), seed
sweeps, and the GPU verification suites."""
import json

import pytest

from paper_2406_02613_b200 import api, csvio
from paper_2406_02613_b200.__main__ import main

pytestmark = pytest.mark.gpu

CFG = {
    "problem": {"kind": "gpt", "vocab": 64, "d_model": 32, "n_layer": 2, "n_head": 2, "seq_len": 16,
                "n_samples": 32, "seed": 3, "precision": "fp32"},
    "method_name": "acco",
    "optimizer": {"kind": "adamw", "learning_rate": 0.01, "weight_decay": 0.1, "adam_beta2": 0.95,
                  "scheduler": "cosine", "n_warmup_steps": 2},
    "n_workers": 2, "batch_size": 3, "n_grad_accumulation": 1, "warmup_rounds": 0, "t_updates": 5,
    "master_seed": 11,
}


def _metrics(path):
    with open(path) as f:
        lines = f.read().splitlines()
    return lines[0], [row.split(",") for row in lines[1:]]


@pytest.mark.parametrize("method", ["acco", "ddp", "zero1", "dpu", "wp"])
def test_run_writes_reference_schema(cuda, tmp_path, method):
    cfg = dict(CFG, method_name=method)
    path = tmp_path / "cfg.json"
    path.write_text(json.dumps(cfg))
    out = tmp_path / "out"
    assert main(["run", "--config", str(path), "--out", str(out)]) == 0
    header, rows = _metrics(out / "metrics.csv")
    assert header + "\n" == csvio.metrics_header(2)
    assert len(rows) == 5 and [int(r[0]) for r in rows] == list(range(5))
    assert all(0.0 <= float(x) <= 1.0 for r in rows for x in r[6:8])
    tl = (out / "timeline.csv").read_text().splitlines()
    assert tl[0] == "worker_id,stream,event_kind,t_start,t_end,micro_batches,bytes"
    kinds = {row.split(",")[2] for row in tl[1:]}
    assert {"microbatch", "all_reduce", "optimizer"} <= kinds
    for row in tl[1:]:
        f = row.split(",")
        assert float(f[3]) <= float(f[4])
    m = json.loads((out / "manifest.json").read_text())
    assert m["config"] == cfg and m["config_hash"] == api.config_hash(cfg) and m["updates"] == 5
    # the echoed config reruns to the same trajectory
    path2 = tmp_path / "cfg2.json"
    path2.write_text(json.dumps(m["config"]))
    out2 = tmp_path / "out2"
    assert main(["run", "--config", str(path2), "--out", str(out2)]) == 0
    _, rows2 = _metrics(out2 / "metrics.csv")
    assert [r[3] for r in rows2] == [r[3] for r in rows]  # loss column, bitwise (%.17g)


def test_sweep_aggregates_in_seed_order(cuda, tmp_path):
    path = tmp_path / "cfg.json"
    path.write_text(json.dumps(CFG))
    assert main(["sweep", "--config", str(path), "--seeds", "1,2,3", "--out", str(tmp_path / "sw")]) == 0
    lines = (tmp_path / "sw" / "sweep.csv").read_text().splitlines()
    assert lines[0] == "update,mean_loss,std_loss,n_seeds" and len(lines) == 6
    assert all(l.endswith(",3") for l in lines[1:])
    m = json.loads((tmp_path / "sw" / "manifest.json").read_text())
    assert m["seeds"] == [1, 2, 3] and m["outputs"] == ["sweep.csv"]


@pytest.mark.parametrize("suite", ["shard-equivalence", "collectives", "acco-gd-equivalence", "heterogeneous"])
def test_gpu_verify_suites_pass(cuda, tmp_path, suite):
    out = tmp_path / "rep.json"
    assert main(["verify", "--suite", suite, "--out", str(out)]) == 0
    rep = json.loads(out.read_text())
    print(json.dumps(rep))
    assert rep["pass"] and rep["suite"] == suite


def test_run_peer_fabric_config(cuda, tmp_path):
    cfg = dict(CFG, n_workers=1, fabric="peer")
    path = tmp_path / "cfg.json"
    path.write_text(json.dumps(cfg))
    assert main(["run", "--config", str(path), "--out", str(tmp_path / "o")]) == 0
    _, rows = _metrics(tmp_path / "o" / "metrics.csv")
    assert len(rows) == 5
