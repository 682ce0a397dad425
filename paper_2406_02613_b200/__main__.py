"""Experiment runner on the B200 path — the reference's ``accosim`` CLI
(proj/tools/accosim_main.cpp:1-208) with the same subcommands, output files
and exit codes:

  python -m paper_2406_02613_b200 run    --config cfg.json [--out DIR]
  python -m paper_2406_02613_b200 sweep  --config cfg.json --seeds 1,2,3 [--out DIR]
  python -m paper_2406_02613_b200 verify --suite NAME [--out report.json]
  python -m paper_2406_02613_b200 memory --method acco --k 12 --n 64 --psi 7.5e9

Exit codes: 0 success, 1 verification failure, 2 invalid config/arguments,
3 diverged run, 4 CUDA/NCCL error (B200 addition). Launched under torchrun,
``run`` puts one worker per rank on NCCL (n_workers must equal the world
size) and ``sweep`` deals the seeds round-robin to the ranks, aggregating in
seed order on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

EXIT_OK, EXIT_VERIFY_FAILED, EXIT_CONFIG, EXIT_DIVERGED, EXIT_CUDA = 0, 1, 2, 3, 4


def _default_out_root() -> str:
    return os.environ.get("ACCOSIM_OUT", "out")  # accosim_main.cpp:37-40


def _dist():
    """(rank, world, local_rank) when launched by torchrun, else (0, 1, 0)."""
    if "WORLD_SIZE" not in os.environ or int(os.environ["WORLD_SIZE"]) <= 1:
        return 0, 1, 0
    import torch
    import torch.distributed as dist

    if not dist.is_initialized():
        dist.init_process_group("gloo")
    lr = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(lr)
    return dist.get_rank(), dist.get_world_size(), lr


def _load(path: str):
    from . import api

    try:
        with open(path) as f:
            j = json.load(f)
    except (OSError, json.JSONDecodeError) as e:
        raise api.InvalidArgument(2, f"cannot read config {path}: {e}")
    return api.parse_config(j)


def cmd_run(config_path: str, out_dir: str) -> int:
    from . import api, csvio

    cfg = _load(config_path)
    rank, world, local = _dist()
    comm = None
    fabric = cfg.raw.get("fabric", "nccl")  # B200 key: "nccl" or "peer" (fused NVLink fold kernel)
    if fabric not in ("nccl", "peer"):
        raise api.InvalidArgument(2, f"config: unknown fabric {fabric}")
    if world > 1 and cfg.sim.n_workers != world:
        raise api.InvalidArgument(2, f"run: n_workers ({cfg.sim.n_workers}) must equal the world size ({world})")
    if fabric == "peer" and (world > 1 or cfg.sim.n_workers == 1):
        comm = api.PeerComm(rank, world, local)
    elif world > 1:
        comm = api.Comm(rank, world, local)
    if not out_dir:
        out_dir = cfg.output_dir or os.path.join(_default_out_root(), "run_" + api.config_hash(cfg.raw))
    tr = api.run_protocol(cfg.method, cfg.problem, cfg.optimizer, cfg.sim, cfg.t_updates, comm=comm,
                          record_history=False)
    if world > 1:  # merge the ranks' timelines (each rank owns its worker's rows)
        import torch.distributed as dist

        parts = [None] * world
        dist.all_gather_object(parts, tr.timeline)
        tr.timeline = [iv for p in parts for iv in p]
    if rank == 0:
        p = csvio.write_run_outputs(out_dir, cfg.raw, tr, cfg.sim.n_workers)
        print(f"wrote {p.metrics}, {p.timeline}, {p.manifest}")
        if tr.diverged:
            print(f"run diverged after {len(tr.records)} updates", file=sys.stderr)
    return EXIT_DIVERGED if tr.diverged else EXIT_OK


def cmd_sweep(config_path: str, seeds_csv: str, out_dir: str) -> int:
    from . import api, csvio

    cfg = _load(config_path)
    try:
        seeds = [int(s) for s in seeds_csv.split(",") if s != ""]
    except ValueError:
        raise api.InvalidArgument(2, "sweep: seeds must be integers")
    if not seeds:
        raise api.InvalidArgument(2, "sweep: at least one seed required")
    if not out_dir:
        out_dir = os.path.join(_default_out_root(), "sweep_" + api.config_hash(cfg.raw))
    rank, world, _ = _dist()
    mine = {}
    for i in range(rank, len(seeds), world):  # seed runs are independent
        sim = api.SimConfig(**{**cfg.sim.__dict__, "master_seed": seeds[i]})
        tr = api.run_protocol(cfg.method, cfg.problem, cfg.optimizer, sim, cfg.t_updates, record_history=False)
        mine[i] = ([r.loss for r in tr.records], [r.update for r in tr.records], tr.diverged)
    if world > 1:
        import torch.distributed as dist

        parts = [None] * world
        dist.all_gather_object(parts, mine)
        for p in parts:
            mine.update(p)
    rows = len(mine[0][0])
    if any(len(mine[i][0]) != rows for i in range(len(seeds))):
        raise RuntimeError("sweep: inconsistent per-seed row counts")
    diverged = any(mine[i][2] for i in range(len(seeds)))
    if rank == 0:  # aggregation is sequential in seed order: deterministic for any rank count
        path = csvio.write_sweep_outputs(out_dir, cfg.raw, seeds, [mine[i][0] for i in range(len(seeds))], mine[0][1])
        print(f"wrote {path}")
    return EXIT_DIVERGED if diverged else EXIT_OK


def cmd_verify(suite: str, out_path: str) -> int:
    from . import csvio, verify

    rep = verify.run_suite(suite)
    text = csvio.dump_json(rep.to_json()) + "\n"
    print(text, end="")
    if out_path:
        with open(out_path, "w", newline="\n") as f:
            f.write(text)
    return EXIT_OK if rep.passed() else EXIT_VERIFY_FAILED


def cmd_memory(method: str, k: float, n: float, psi: float) -> int:
    from . import api, csvio

    b = api.memory_model_bytes(method, k, n, psi)
    print(csvio.dump_json({"method": method, "k": k, "n": n, "psi": psi, "bytes": b,
                           "gb": api.memory_reported_gb(b)}))
    return EXIT_OK


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2406_02613_b200",
                                 description="ACCO on B200: overlapped data-parallel training protocols")
    sub = ap.add_subparsers(dest="cmd")
    r = sub.add_parser("run", help="execute one protocol run")
    r.add_argument("--config", required=True)
    r.add_argument("--out", default="")
    s = sub.add_parser("sweep", help="aggregate runs across seeds")
    s.add_argument("--config", required=True)
    s.add_argument("--seeds", required=True)
    s.add_argument("--out", default="")
    v = sub.add_parser("verify", help="run a verification suite")
    v.add_argument("--suite", required=True)
    v.add_argument("--out", default="")
    m = sub.add_parser("memory", help="per-replica memory model")
    m.add_argument("--method", required=True)
    m.add_argument("--k", type=float, default=12.0)
    m.add_argument("--n", type=float, default=64.0)
    m.add_argument("--psi", type=float, default=7.5e9)
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:
        return EXIT_OK if e.code == 0 else EXIT_CONFIG
    if a.cmd is None:
        ap.print_usage(sys.stderr)
        return EXIT_CONFIG
    from ._lib import AccoError, InvalidArgument

    try:
        if a.cmd == "run":
            return cmd_run(a.config, a.out)
        if a.cmd == "sweep":
            return cmd_sweep(a.config, a.seeds, a.out)
        if a.cmd == "verify":
            return cmd_verify(a.suite, a.out)
        return cmd_memory(a.method, a.k, a.n, a.psi)
    except InvalidArgument as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_CONFIG
    except AccoError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_CUDA if e.code == 4 else EXIT_CONFIG
    except (ValueError, RuntimeError, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_CONFIG


if __name__ == "__main__":
    sys.exit(main())
