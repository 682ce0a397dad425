"""BASELINE.json config 5: optimizer-round microbench — one ACCO round's comm
stream: counts all-reduce + reduce-scatter + K6 estimate (transient) +
all-gather + counts AR + RS + K7 commit (with the retained shard) + AG, at
Psi in {10M, 100M, 1B, 2B} fp32 gradients ~ N(0,1) per rank (seeded per
rank), theta ~ 0.02 N(0,1), m = v = 0, N = 1/2/4/8 ranks (one per GPU).

  python tools/optim_microbench.py [--sizes 1e7,1e8,1e9,2e9] [--reps 10]
  torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/optim_microbench.py [--fabric nccl|peer]

--fabric nccl (default): the C-ABI ops in the reference's order
(proj/src/protocols.cpp:644-670): RS (NCCL, fp32) -> K6 on the shard -> AG
(NCCL, bf16) -> RS -> K7 -> AG, with CUDA events around every step. Reports
the fused optimizer's HBM throughput (52 B per shard element per round)
against the measured copy peak, and each collective's NCCL bus bandwidth
(bytes x (N-1)/N / time) next to the reference's own alpha+beta ring cost
model (proj/src/collectives.cpp:16-25) evaluated at the NVLink 5 link rate.

--fabric peer: the engine's fused peer-memory phase (one kernel: fold every
rank's shard over NVLink in rank order + AdamW + store into every rank's
replica) measured from the trainer's CUDA-event timeline, on a shell LM
whose parameter count is Psi (the phase does not depend on the model).

Timing: CUDA events on the launching stream, max over ranks; rank 0 prints
one JSON line per size. The reference CPU round (oracle/_ref/ref_round_bench,
fp64, single thread) is timed at Psi = 10M for context.
"""
import argparse
import ctypes as C
import json
import os
import subprocess
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2406_02613_b200 import _lib, api  # noqa: E402

NVLINK_GBS = 900.0  # NVLink 5 per direction per GPU (B200_PROFILING.md)


def ring_time_s(kind, nbytes, n, beta_s_per_byte=1.0 / (NVLINK_GBS * 1e9), alpha_s=0.0):
    """collective_time (proj/src/collectives.cpp:16-25): alpha + passes * beta * bytes * (N-1)/N."""
    if n == 1:
        return 0.0
    return alpha_s + (2.0 if kind == "all_reduce" else 1.0) * beta_s_per_byte * nbytes * (n - 1) / n


def max_over_ranks(x, world):
    if world == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item()


def nccl_round(psi, world, rank, comm, reps, hbm):
    dev = torch.device("cuda")
    stream = torch.cuda.current_stream()
    sp = C.c_void_p(stream.cuda_stream)
    h = comm.handle
    chunk = (psi + world - 1) // world  # owner-padded chunk
    cfg = api.OptimizerConfig(kind="adamw", learning_rate=6e-4, weight_decay=0.1, adam_beta2=0.95,
                              scheduler="cosine", total_steps=1000).to_c()
    gen = torch.Generator(device=dev).manual_seed(1000 + rank)
    g_main = torch.randn(world * chunk, device=dev, generator=gen)
    g_est = torch.randn(world * chunk, device=dev, generator=gen)
    red_main = torch.empty(chunk, device=dev)
    red_est = torch.empty(chunk, device=dev)
    theta = 0.02 * torch.randn(chunk, device=dev, generator=gen)
    m = torch.zeros(chunk, device=dev)
    v = torch.zeros(chunk, device=dev)
    est_rep = torch.empty(world * chunk, dtype=torch.bfloat16, device=dev)
    th_rep = torch.empty(world * chunk, dtype=torch.bfloat16, device=dev)
    cnt = torch.tensor([8], dtype=torch.int64, device=dev)
    tot = torch.zeros(2, dtype=torch.int64, device=dev)
    st = _lib.ShardState(0, theta.data_ptr(), m.data_ptr(), v.data_ptr(), 0, chunk)
    P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(9)]

    def round_():
        ev[0].record(stream)
        _lib.call("acco_all_reduce_i64", h, P(cnt), P(tot[0:1]), 1, sp)
        _lib.call("acco_reduce_scatter_f32", h, P(g_est), P(red_est), chunk, sp)
        ev[1].record(stream)
        _lib.call("acco_opt_estimate", C.byref(cfg), C.byref(st), P(red_est), P(tot[0:1]),
                  P(est_rep[rank * chunk:]), _lib.DTYPE_BF16, None, sp)
        ev[2].record(stream)
        _lib.call("acco_all_gather", h, P(est_rep[rank * chunk:]), P(est_rep), chunk, _lib.DTYPE_BF16, sp)
        ev[3].record(stream)
        _lib.call("acco_all_reduce_i64", h, P(cnt), P(tot[1:2]), 1, sp)
        ev[4].record(stream)
        _lib.call("acco_reduce_scatter_f32", h, P(g_main), P(red_main), chunk, sp)
        ev[5].record(stream)
        _lib.call("acco_opt_commit", C.byref(cfg), C.byref(st), P(red_main), P(red_est), P(tot[1:2]),
                  P(tot[0:1]), P(th_rep[rank * chunk:]), _lib.DTYPE_BF16, None, sp)
        ev[6].record(stream)
        _lib.call("acco_all_gather", h, P(th_rep[rank * chunk:]), P(th_rep), chunk, _lib.DTYPE_BF16, sp)
        ev[7].record(stream)

    for _ in range(3):
        round_()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    acc = dict(round=0.0, rs=0.0, est=0.0, ag=0.0, com=0.0)
    for _ in range(reps):
        round_()
        ev[7].synchronize()
        acc["round"] += ev[0].elapsed_time(ev[7])
        acc["rs"] += ev[4].elapsed_time(ev[5])          # the commit phase's reduce-scatter
        acc["est"] += ev[1].elapsed_time(ev[2])
        acc["ag"] += ev[6].elapsed_time(ev[7])          # the commit phase's all-gather
        acc["com"] += ev[5].elapsed_time(ev[6])
    t = {k: max_over_ranks(v / reps, world) for k, v in acc.items()}
    opt_gbs = 52.0 * chunk / ((t["est"] + t["com"]) / 1e3) / 1e9
    rs_bytes, ag_bytes = world * chunk * 4, world * chunk * 2  # per rank: the full fp32 / bf16 vectors
    out = {"round_ms": t["round"], "estimate_ms": t["est"], "commit_ms": t["com"], "rs_ms": t["rs"], "ag_ms": t["ag"],
           "roofline": {"bound": "hbm", "achieved": opt_gbs, "peak": hbm, "unit": "GB/s", "frac": opt_gbs / hbm,
                        "bytes_per_elem": 52, "kernel": "fused AdamW estimate (K6) + commit (K7) on the shard"}}
    if world > 1:
        rs_bus = rs_bytes * (world - 1) / world / (t["rs"] / 1e3) / 1e9
        ag_bus = ag_bytes * (world - 1) / world / (t["ag"] / 1e3) / 1e9
        out["nvlink"] = {
            "reduce_scatter_busbw_GBps": rs_bus, "all_gather_busbw_GBps": ag_bus, "link_GBps": NVLINK_GBS,
            "rs_frac_of_link": rs_bus / NVLINK_GBS, "ag_frac_of_link": ag_bus / NVLINK_GBS,
            "cost_model_ms": {"reduce_scatter": ring_time_s("reduce_scatter", rs_bytes, world) * 1e3,
                              "all_gather": ring_time_s("all_gather", ag_bytes, world) * 1e3,
                              "note": "reference collective_time (collectives.cpp:16-25) with alpha = 0 and "
                                      "beta = 1 / (900 GB/s), the NVLink 5 per-direction rate"}}
    del g_main, g_est, red_main, red_est, theta, m, v, est_rep, th_rep
    torch.cuda.empty_cache()
    return out


def peer_round(psi, world, rank, reps, hbm):
    d = 256
    V = max(64, (psi - 12 * d * d - 8 * d - 2 * d) // d)
    lm = api.LMConfig(vocab=V, d_model=d, n_layer=1, n_head=4, seq_len=8, n_samples=8, precision="bf16",
                      max_batch=1)
    model = api.Model(lm)
    peer = api.PeerComm(rank, world, torch.cuda.current_device())
    opt = api.OptimizerConfig(kind="adamw", learning_rate=6e-4, weight_decay=0.1, adam_beta2=0.95,
                              scheduler="cosine", total_steps=1000)
    sim = api.SimConfig(n_workers=world, batch_size=1, master_seed=1, eval_every=0)
    tr = api.Trainer("acco", model, opt, sim, peer)
    tr.set_theta(model.default_theta0(1))
    tr.run(2)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    tr.run(reps)
    tl = tr.timeline()
    phases = [iv for iv in tl if iv.stream == "comm" and iv.kind == "optimizer" and iv.worker == rank]
    ph_ms = sum((iv.t_end - iv.t_start) * 1e3 for iv in phases) / max(len(phases), 1)
    ph_ms = max_over_ranks(ph_ms, world)
    chunk = (model.dim + world - 1) // world
    # fused phase traffic per rank: read world shards' sums (4 B each) + retained (commit) + theta/m/v,
    # write theta/m/v + the bf16 shard into world replicas; average of the estimate and commit phases
    local = 0.5 * ((4 * world + 16 + 4 + 2 * world) + (4 * world + 4 + 24 + 2 * world)) * chunk
    del tr
    return {"psi_model": model.dim, "phase_ms": ph_ms, "round_ms": 2 * ph_ms,
            "phase_bytes_per_rank": local, "phase_GBps": local / (ph_ms / 1e3) / 1e9,
            "note": "peer fabric: counts barrier + fold of every rank's shard over NVLink + AdamW + replica "
                    "stores in one kernel; timed from the trainer's CUDA-event timeline (optimizer interval)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="1e7,1e8,1e9,2e9")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--fabric", default="nccl", choices=["nccl", "peer"])
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            hbm = json.load(f)["hbm_gbs"]
    except OSError:
        hbm = 6650.0
    if world > 1:
        dist.init_process_group("gloo")
    else:
        import socket

        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    comm = api.Comm(rank, world, local) if args.fabric == "nccl" else None
    for psi in [int(float(x)) for x in args.sizes.split(",")]:
        if args.fabric == "nccl":
            r = nccl_round(psi, world, rank, comm, args.reps, hbm)
        else:
            r = peer_round(psi, world, rank, args.reps, hbm)
        line = {"metric": f"optimizer-round params/s (ACCO estimate+commit, fused AdamW, {args.fabric}, N={world})",
                "psi": psi, "n_gpus": world, "fabric": args.fabric, "value": psi / (r["round_ms"] / 1e3),
                "unit": "params/s", **r}
        if psi == int(1e7) and rank == 0 and world == 1:
            exe = os.path.join(ROOT, "oracle", "_ref", "ref_round_bench")
            if os.path.exists(exe):
                p = subprocess.run([exe, str(psi), "8", "3"], capture_output=True, text=True, timeout=600)
                try:
                    ref = json.loads(p.stdout.strip().splitlines()[-1])
                    line["cpu_baseline"] = {"value": ref["params_per_s"], "unit": "params/s", "cores": 1,
                                            "kind": "reference", "sample": "reference Fabric RS + sharded_opt_step "
                                            "(estimate, commit) + all_gather, fp64, N=8 simulated workers, Psi=1e7"}
                except Exception as e:  # noqa: BLE001
                    line["cpu_baseline"] = {"error": str(e)[:200]}
        if rank == 0:
            print(json.dumps(line), flush=True)
    del comm
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
