"""Run outputs with the reference's formats: ``metrics.csv``, ``timeline.csv``
and ``manifest.json`` (proj/src/csvio.cpp:12-102), plus the sweep aggregate
``sweep.csv`` (proj/tools/accosim_main.cpp:96-121).

Same header strings, ``%.17g`` number formatting, LF line endings and the
nlohmann ``dump(2)`` manifest layout (keys sorted, two-space indent), so a
consumer of the reference's output directories reads these unchanged. The
difference is the data: times in ``timeline.csv`` / ``time_s`` are measured
with CUDA events on the compute and comm streams (seconds since the start of
the run), not simulated.
"""
from __future__ import annotations

import json
import math
import os
from dataclasses import dataclass
from typing import List, Sequence

TOOL, VERSION = "accosim", "0.1.0"  # manifest identity of the reference's writer (csvio.cpp:87-88)


def format_g17(v: float) -> str:
    """csvio.cpp:12-16 (``%.17g``; glibc spells NaN/inf as nan/-nan/inf/-inf)."""
    v = float(v)
    if math.isnan(v):
        return "-nan" if math.copysign(1.0, v) < 0 else "nan"
    return "%.17g" % v


def metrics_header(n_workers: int) -> str:
    """csvio.cpp:18-23."""
    return "update,time_s,samples,loss,grad_norm_sq,lyapunov" + "".join(
        f",idle_frac_w{w}" for w in range(n_workers)) + "\n"


@dataclass
class Interval:
    """Timeline interval (simclock.hpp): one timeline.csv row."""
    worker: int
    stream: str  # "compute" | "comm"
    kind: str
    t_start: float
    t_end: float
    micro_batches: int
    bytes: int


def metrics_csv(records: Sequence, n_workers: int) -> str:
    """csvio.cpp:25-46. ``records``: objects with update, time_s, samples_cum,
    loss, grad_sq, lyapunov, idle_frac (length n_workers)."""
    out = [metrics_header(n_workers)]
    for r in records:
        lyap = r.lyapunov if r.lyapunov is not None else float("nan")
        row = [str(int(r.update)), format_g17(r.time_s), str(int(r.samples_cum)), format_g17(r.loss),
               format_g17(r.grad_sq), format_g17(lyap)]
        row += [format_g17(r.idle_frac[w]) for w in range(n_workers)]
        out.append(",".join(row) + "\n")
    return "".join(out)


def timeline_csv(intervals: Sequence[Interval]) -> str:
    """csvio.cpp:48-66."""
    out = ["worker_id,stream,event_kind,t_start,t_end,micro_batches,bytes\n"]
    for iv in intervals:
        out.append(f"{int(iv.worker)},{iv.stream},{iv.kind},{format_g17(iv.t_start)},{format_g17(iv.t_end)},"
                   f"{int(iv.micro_batches)},{int(iv.bytes)}\n")
    return "".join(out)


def dump_json(obj) -> str:
    """nlohmann ``json::dump(2)``: std::map key order, two-space indent, ": " / ","."""
    return json.dumps(obj, indent=2, sort_keys=True, ensure_ascii=False)


def _write(path: str, text: str) -> None:
    with open(path, "w", newline="\n", encoding="utf-8") as f:
        f.write(text)


@dataclass
class RunPaths:
    metrics: str
    timeline: str
    manifest: str


def manifest(config: dict, diverged: bool, updates: int, config_hash: str) -> dict:
    """csvio.cpp:84-96."""
    return {"tool": TOOL, "version": VERSION, "config": config, "config_hash": config_hash,
            "master_seed": config.get("master_seed", 1), "diverged": bool(diverged), "updates": int(updates),
            "outputs": ["metrics.csv", "timeline.csv"]}


def write_run_outputs(out_dir: str, config: dict, trace, n_workers: int) -> RunPaths:
    """csvio.cpp:76-100: metrics.csv, timeline.csv, manifest.json in out_dir."""
    from .api import config_hash

    os.makedirs(out_dir, exist_ok=True)
    paths = RunPaths(os.path.join(out_dir, "metrics.csv"), os.path.join(out_dir, "timeline.csv"),
                     os.path.join(out_dir, "manifest.json"))
    _write(paths.metrics, metrics_csv(trace.records, n_workers))
    _write(paths.timeline, timeline_csv(trace.timeline))
    _write(paths.manifest, dump_json(manifest(config, trace.diverged, len(trace.records), config_hash(config))) + "\n")
    return paths


def sweep_csv(losses: List[List[float]], updates: List[int]) -> str:
    """accosim_main.cpp:96-110: per update, mean and sample std of the loss
    over seeds, aggregated sequentially in seed order (deterministic)."""
    n = len(losses)
    out = ["update,mean_loss,std_loss,n_seeds\n"]
    for r, upd in enumerate(updates):
        mean = 0.0
        for tr in losses:
            mean += tr[r]
        mean /= float(n)
        var = 0.0
        for tr in losses:
            d = tr[r] - mean
            var += d * d
        var = var / float(n - 1) if n > 1 else 0.0
        out.append(f"{upd},{format_g17(mean)},{format_g17(math.sqrt(var))},{n}\n")
    return "".join(out)


def write_sweep_outputs(out_dir: str, config: dict, seeds: List[int], losses: List[List[float]],
                        updates: List[int]) -> str:
    """accosim_main.cpp:111-124."""
    from .api import config_hash

    os.makedirs(out_dir, exist_ok=True)
    path = os.path.join(out_dir, "sweep.csv")
    _write(path, sweep_csv(losses, updates))
    m = {"tool": TOOL, "version": VERSION, "config": config, "config_hash": config_hash(config),
         "seeds": [int(s) for s in seeds], "outputs": ["sweep.csv"]}
    _write(os.path.join(out_dir, "manifest.json"), dump_json(m) + "\n")
    return path


def idle_fractions(records, intervals: Sequence[Interval], workers: Sequence[int]) -> List[List[float]]:
    """Per committed update and worker: the compute stream's idle share of the
    window since the previous commit, (window - busy) / window clipped at 0 —
    the reference's idle_frac (protocols.cpp:143-154), with busy time taken
    from the measured compute intervals instead of simulated ones."""
    out = []
    prev = 0.0
    comp = {w: [(iv.t_start, iv.t_end) for iv in intervals if iv.stream == "compute" and iv.worker == w]
            for w in workers}
    for r in records:
        t = r.time_s
        window = t - prev
        row = []
        for w in workers:
            busy = sum(max(0.0, min(b, t) - max(a, prev)) for a, b in comp[w])
            row.append(max(0.0, (window - busy) / window) if window > 0 else 0.0)
        out.append(row)
        prev = t
    return out
