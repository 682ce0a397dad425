"""The committed profile evidence that bench.py reads at run time
(profiles/prof_step_r02_raw.csv -> the roofline `traffic` fields) parses and
covers the kernel classes bench.py reports."""
import csv
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_ncu_summary_has_traffic_for_reported_kernels():
    path = os.path.join(ROOT, "profiles", "prof_step_r02_raw.csv")
    with open(path) as f:
        rows = list(csv.DictReader(f))
    assert {"kernel", "time_us", "dram_read_bytes", "dram_write_bytes"} <= set(rows[0])
    for prefix in ("gemm_tc_kernel", "opt_kernel", "fa_bwd_dkv_tc", "ce_vec_kernel"):
        sel = [r for r in rows if prefix in r["kernel"]]
        assert sel, prefix
        for r in sel:
            assert float(r["time_us"]) > 0
            assert float(r["dram_read_bytes"]) + float(r["dram_write_bytes"]) > 0


def test_launch_list_present():
    path = os.path.join(ROOT, "profiles", "r02_launches_bench_step.csv")
    with open(path) as f:
        text = f.read()
    assert "gemm_tc_kernel" in text and "gpu__time_duration.sum" in text


def test_capture_commit_recorded():
    import json

    with open(os.path.join(ROOT, "profiles", "prof_step_r02_meta.json")) as f:
        meta = json.load(f)
    assert len(meta["capture_commit"]) >= 7 and "ncu --set full" in meta["command"]
