"""Config-level C entry acco_run (include/acco.h; SURVEY.md §8(b) "Trainer":
load_config -> run_protocol -> write_run_outputs, proj/src/config.cpp:80-145,
csvio.cpp:79-102) against the Python CLI on the same config: the same
manifest.json bytes (nlohmann dump of the echoed config and its FNV-1a hash),
the same deterministic metrics columns (update, samples, loss, grad_norm_sq),
the reference's exit codes."""
import json

import pytest

from paper_2406_02613_b200 import _lib, api
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


def _cols(path):
    rows = [r.split(",") for r in path.read_text().splitlines()]
    return rows[0], [[r[0], r[2], r[3], r[4]] for r in rows[1:]]  # update, samples, loss, grad_norm_sq


@pytest.mark.parametrize("method", ["acco", "ddp", "wp"])
def test_acco_run_matches_cli(cuda, tmp_path, method):
    cfg = dict(CFG, method_name=method)
    path = tmp_path / "cfg.json"
    path.write_text(json.dumps(cfg))
    rc, summ = api.run_config(str(path), str(tmp_path / "c"))
    assert rc == 0 and summ["updates"] == 5 and not summ["diverged"] and summ["out_dir"] == str(tmp_path / "c")
    assert main(["run", "--config", str(path), "--out", str(tmp_path / "py")]) == 0
    assert (tmp_path / "c" / "manifest.json").read_bytes() == (tmp_path / "py" / "manifest.json").read_bytes()
    hc, rc_rows = _cols(tmp_path / "c" / "metrics.csv")
    hp, py_rows = _cols(tmp_path / "py" / "metrics.csv")
    assert hc == hp and rc_rows == py_rows
    tl = (tmp_path / "c" / "timeline.csv").read_text().splitlines()
    assert tl[0] == "worker_id,stream,event_kind,t_start,t_end,micro_batches,bytes" and len(tl) > 10
    assert summ["samples"] == int(rc_rows[-1][1])


def test_acco_run_inline_json_and_default_out(cuda, tmp_path, monkeypatch):
    monkeypatch.setenv("ACCOSIM_OUT", str(tmp_path))
    rc, summ = api.run_config(json.dumps(CFG))
    assert rc == 0
    m = json.loads((tmp_path / f"run_{api.config_hash(CFG)}" / "manifest.json").read_text())
    assert m["config"] == CFG and m["config_hash"] == api.config_hash(CFG) and m["updates"] == 5


def test_acco_run_exit_codes(cuda, tmp_path):
    bad = {k: v for k, v in CFG.items() if k != "t_updates"}
    with pytest.raises(_lib.InvalidArgument, match="missing key 't_updates'"):
        api.run_config(json.dumps(bad), str(tmp_path / "x"))
    with pytest.raises(_lib.InvalidArgument, match="invalid JSON"):
        api.run_config("{not json", str(tmp_path / "x"))
    with pytest.raises(_lib.InvalidArgument):
        api.run_config(json.dumps(dict(CFG, batch_size="three")), str(tmp_path / "x"))  # type error: exit 2
    div = dict(CFG, optimizer={"kind": "adamw", "learning_rate": 1e300}, n_workers=1)
    rc, summ = api.run_config(json.dumps(div), str(tmp_path / "d"))
    assert rc == 3 and summ["diverged"] and summ["updates"] == 1  # outputs written, exit 3
    assert json.loads((tmp_path / "d" / "manifest.json").read_text())["diverged"] is True
