"""Output-format parity against files the reference's own
writer produced (oracle/golden_dump.cpp -> tests/golden/io/): metrics.csv,
timeline.csv and manifest.json byte for byte from the same trace, %.17g
formatting, the FNV-1a config hash, and the memory model table."""
import json
import math
import os
from types import SimpleNamespace

import pytest

from paper_2406_02613_b200 import api, csvio

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _trace():
    with open(os.path.join(GOLD, "io_trace.json")) as f:
        return json.load(f)


def _read(name):
    with open(os.path.join(GOLD, "io", name), newline="") as f:
        return f.read()


def test_format_g17_matches_reference():
    j = _trace()
    for v, s in j["g17"]:
        assert csvio.format_g17(v) == s
    assert csvio.format_g17(float("nan")) == j["g17_nan"]
    assert csvio.format_g17(float("inf")) == j["g17_inf"]
    assert csvio.metrics_header(1) == j["metrics_header_1"]
    assert csvio.metrics_header(3) == j["metrics_header_3"]


def test_metrics_timeline_manifest_bytes_match_reference_writer():
    j = _trace()
    recs = [SimpleNamespace(update=r["update"], time_s=r["time_s"], samples_cum=r["samples_cum"], loss=r["loss"],
                            grad_sq=r["grad_sq"], lyapunov=r["lyapunov"], idle_frac=r["idle_frac"])
            for r in j["records"]]
    ivs = [csvio.Interval(*row) for row in j["intervals"]]
    assert csvio.metrics_csv(recs, j["n_workers"]) == _read("metrics.csv")
    assert csvio.timeline_csv(ivs) == _read("timeline.csv")
    assert api.config_hash(j["config"]) == j["config_hash"]
    m = csvio.manifest(j["config"], j["diverged"], len(recs), api.config_hash(j["config"]))
    assert csvio.dump_json(m) + "\n" == _read("manifest.json")
    assert "\r" not in _read("metrics.csv")


def test_write_run_outputs_roundtrip(tmp_path):
    j = _trace()
    recs = [SimpleNamespace(update=r["update"], time_s=r["time_s"], samples_cum=r["samples_cum"], loss=r["loss"],
                            grad_sq=r["grad_sq"], lyapunov=r["lyapunov"], idle_frac=r["idle_frac"])
            for r in j["records"]]
    tr = SimpleNamespace(records=recs, timeline=[csvio.Interval(*row) for row in j["intervals"]],
                         diverged=j["diverged"])
    p = csvio.write_run_outputs(str(tmp_path / "out"), j["config"], tr, j["n_workers"])
    for path, name in ((p.metrics, "metrics.csv"), (p.timeline, "timeline.csv"), (p.manifest, "manifest.json")):
        with open(path, newline="") as f:
            assert f.read() == _read(name)


def test_config_hash_stable_and_sensitive():
    # proj/tests/test_io.cpp:108-115
    a = _trace()["config"]
    b = json.loads(json.dumps(a))
    assert api.config_hash(a) == api.config_hash(b)
    b["master_seed"] = 12
    assert api.config_hash(a) != api.config_hash(b) and len(api.config_hash(a)) == 16


def test_memory_model_matches_reference():
    with open(os.path.join(GOLD, "memory.json")) as f:
        rows = json.load(f)
    for r in rows:
        b = api.memory_model_bytes(r["method"], r["k"], r["n"], r["psi"])
        assert b == r["bytes"], r
        assert api.memory_reported_gb(b) == r["gb"]
    with pytest.raises(api.InvalidArgument):
        api.memory_model_bytes("acco", 0.0, 1, 1)


def test_sweep_csv_order_fixed():
    losses = [[1.0, 0.5], [3.0, 0.25]]
    s = csvio.sweep_csv(losses, [0, 1])
    lines = s.splitlines()
    assert lines[0] == "update,mean_loss,std_loss,n_seeds"
    assert lines[1] == f"0,2,{csvio.format_g17(math.sqrt(2.0))},2"
    assert csvio.sweep_csv([[1.0]], [0]).splitlines()[1] == "0,1,0,1"


def test_idle_fractions_from_intervals():
    recs = [SimpleNamespace(time_s=2.0), SimpleNamespace(time_s=4.0)]
    ivs = [csvio.Interval(0, "compute", "microbatch", 0.0, 1.0, 1, 0),
           csvio.Interval(0, "compute", "microbatch", 2.5, 4.0, 1, 0),
           csvio.Interval(0, "comm", "all_gather", 0.0, 4.0, 0, 8)]
    assert csvio.idle_fractions(recs, ivs, [0]) == [[0.5], [0.25]]
