#!/usr/bin/env python
"""ACCO round benchmark (BASELINE.json metric: tokens/s at 1/2/4/8 B200;
exposed comm %; ACCO vs ZeRO-1 step-time speedup).

Workload (N=1 default): GPT-2 small (124,439,808 params), synthetic seeded
Markov-chain tokens, random-init weights, bf16 compute / fp32 master shards,
B=8 sequences x 1024 tokens per micro-batch per GPU. One "step" = one
committed ACCO update (k=1: an estimate-stage and a main-stage micro-batch per
GPU, 2 comm phases of counts-AR + RS + fused AdamW + AG). ZeRO-1 and DDP
baselines run on the same kernels with k=2 (equal samples per update).

  python bench.py [--gpus N --steps K --warmup W]           # our arm
  python bench.py --impl reference [...]                     # CPU reference arm
  torchrun --nproc-per-node N bench.py --gpus N ...          # N > 1: one rank per GPU
"""
from __future__ import annotations

import argparse
import csv
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MODELS = {
    "gpt2-small": dict(vocab=50257, d_model=768, n_layer=12, n_head=12, seq_len=1024),
    "gpt2-medium": dict(vocab=50257, d_model=1024, n_layer=24, n_head=16, seq_len=1024),
    "c1": dict(vocab=256, d_model=128, n_layer=2, n_head=4, seq_len=64),
    # C4: Llama-style 1.1B (TinyLlama-1.1B shape: GQA 32/4 heads of 64, SwiGLU 5632, untied head)
    "llama-1b": dict(vocab=32000, d_model=2048, n_layer=22, n_head=32, seq_len=2048, arch="llama", n_kv_head=4,
                     d_ff=5632),
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops_sustained"], p["bf16_tflops"], "measured"
    except Exception:
        return 6650.0, 1400.0, 1590.0, "fallback"


class Clocks:
    """SM clock sampler during the timed region (B200_PROFILING.md clocks
    line): NVML every ~2 ms from a thread, so a timed region of a few hundred
    ms gets hundreds of samples under load (nvidia-smi -lms 200 caught mostly
    the idle clock around a short region). nvidia-smi is the fallback."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # NVML clocks-event reason bits
    BITS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
            0x80: "hw_power_brake_slowdown"}

    def __init__(self, index: int):
        self.index = index
        self.p = None
        self.nv = None
        self.samples = []

    def __enter__(self):
        try:
            import threading

            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.nv = (pynvml, h)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self.stop = False

            def run():
                while not self.stop:
                    try:
                        self.samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                                             pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                                             pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
                    except Exception:
                        pass
                    time.sleep(0.002)
            self.th = threading.Thread(target=run, daemon=True)
            self.th.start()
            return self
        except Exception:
            self.nv = None
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.nv:
            self.stop = True
            self.th.join()
            return
        if self.p:
            time.sleep(0.25)
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        if self.nv:
            if not self.samples:
                return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0, "source": "nvml"}
            clk = sorted(x[0] for x in self.samples)
            pw = sorted(x[1] for x in self.samples)
            reasons, capped = set(), 0
            for _, _, r in self.samples:
                for b, n in self.BITS.items():
                    if r & b:
                        reasons.add(n)
                capped += bool(r & 0x4)
            return {"sm_mhz": float(statistics.median(clk)), "sm_max_mhz": float(self.max_mhz),
                    "reasons": sorted(reasons), "samples": len(clk), "source": "nvml, every ~2 ms",
                    "sm_mhz_p10_p90": [clk[len(clk) // 10], clk[9 * len(clk) // 10]],
                    "power_w_median": round(statistics.median(pw), 1),
                    "sw_power_cap_fraction": round(capped / len(clk), 3)}
        sms, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (self.out or "").splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sms.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sms) if sms else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sms), "source": "nvidia-smi -lms 200"}


def dist_setup(n_gpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != n_gpus:
        raise SystemExit(f"--gpus {n_gpus} but WORLD_SIZE={world}: launch N>1 with torchrun")
    return world, rank, local


def reference_arm(args, cfgd):
    """CPU reference arm: the fp64 oracle port (the reference has no LM; its
    own optimizer round is timed separately by oracle/_ref/ref_round_bench)."""
    world, rank, _ = dist_setup(args.gpus)
    if rank != 0:
        return
    import numpy as np

    from oracle import accosim_oracle as O
    from oracle import gpt_oracle as G

    cfg = G.GPTConfig(**cfgd, n_samples=64, data_seed=1)
    th = G.default_theta0(cfg, 1)
    tok = G.dataset(cfg)
    ocfg = O.OptimizerConfig(kind="adamw", learning_rate=6e-4, weight_decay=0.1, adam_beta2=0.95,
                             scheduler="cosine", total_steps=args.warmup + args.steps)
    st = O.OptimizerState.for_range(ocfg, 0, th.shape[0])
    gret = None

    def step(i):
        # half an ACCO update: one micro-batch (B=1 sequence) + one comm phase
        nonlocal st, th, gret
        idx = O.sample_indices(O.derive(1, 0, i // 2, 2 + (i % 2), 0), 1, cfg.n_samples)
        _, g = G.loss_and_grad(cfg, th, tok[idx])
        if i % 2 == 0:
            gret = g
            O.opt_step(st.copy(), th, g, ocfg)
        else:
            st, th = O.opt_step(st, th, (g + gret) * 0.5, ocfg)

    for i in range(args.warmup):
        step(i)
    t0 = time.perf_counter()
    for i in range(args.steps):
        step(args.warmup + i)
    dt = time.perf_counter() - t0
    tokens = args.steps * cfg.seq_len
    v = tokens / dt
    from oracle.cpu_bench import blas_threads

    cores = blas_threads()
    line = {"impl": "reference", "metric": "tokens/s", "value": v, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded Markov-chain tokens, random-init weights)",
            "config": {"workload": f"{args.model} ACCO on CPU (oracle port, fp64 numpy)", "model": args.model,
                       "seq_len": cfg.seq_len},
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": cores, "kind": "port",
                             "sample": "per step: half an ACCO update = 1 micro-batch fwd/bwd of 1 sequence x "
                                       f"{cfg.seq_len} tokens + 1 AdamW phase over {th.shape[0]} params"},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--model", default="gpt2-small", choices=list(MODELS))
    ap.add_argument("--batch", type=int, default=8, help="sequences per micro-batch per GPU")
    ap.add_argument("--schedule", default="adaptive", choices=["adaptive", "floor"])
    ap.add_argument("--fabric", default="nccl", choices=["nccl", "peer"],
                    help="comm phase: NCCL RS/AG around the fused optimizer, or the fused peer-memory fold kernel")
    ap.add_argument("--straggler", type=float, default=1.0,
                    help="C4 heterogeneous scenario: rank 0's micro-batches take this many times longer "
                         "(HeterogeneityProfile multiplier, emulated by a measured spin after each micro-batch)")
    ap.add_argument("--straggler-mode", default="device", choices=["device", "host"],
                    help="device: a spin kernel on the slow rank's compute stream after each micro-batch; host: the "
                         "paper's time.sleep (PAPER.md:394) after each completed micro-batch, GPU idle")
    ap.add_argument("--emulate-comm-gpus", type=int, default=0,
                    help="single-GPU study of the overlap: every comm phase holds the comm stream for the NVLink "
                         "time (770 GB/s per direction) of an N-GPU reduce-scatter + all-gather (all-reduce for "
                         "DDP); 0 = off")
    ap.add_argument("--emulate-ctas", type=int, default=16,
                    help="with --emulate-comm-gpus: the stand-in collective is a paced HBM copy of the phase's bytes "
                         "on this many CTAs (NCCL's channel count), holding SMs like NCCL; 0 = a one-thread spin")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-baselines", action="store_true")
    ap.add_argument("--profile", action="store_true", help="ncu-friendly: short run, no baselines")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if not args.profile else args.warmup
    cfgd = MODELS[args.model]
    if args.impl == "reference":
        return reference_arm(args, cfgd)

    world, rank, local = dist_setup(args.gpus)
    if world > 1:
        # NCCL's INIT lines (nranks, transports, NVLS) on stderr, keeping stdout to the JSON line
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    import torch

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2406_02613_b200 import api

    nccl = api.Comm(rank, world, local) if world > 1 else None

    def make_comm(method):
        # the peer fabric registers one trainer's buffers, so each trainer gets its own
        if args.fabric == "peer" and method != "ddp":
            return api.PeerComm(rank, world, local)
        return nccl

    comm = nccl
    B, T = args.batch, cfgd["seq_len"]
    n_samples = 4096
    lm = api.LMConfig(**cfgd, n_samples=n_samples, data_seed=1, precision="bf16", max_batch=B)
    model = api.Model(lm)
    opt = api.OptimizerConfig(kind="adamw", learning_rate=6e-4, weight_decay=0.1, adam_beta2=0.95,
                              scheduler="cosine", total_steps=1000)
    hbm, tf_sus, tf_burst, peak_kind = peaks()
    mult = [args.straggler] + [1.0] * (world - 1) if args.straggler != 1.0 else None

    def comm_bytes(method):
        n = args.emulate_comm_gpus
        if n <= 1:
            return 0.0
        frac = (n - 1) / n
        # bytes each GPU sends per comm phase: RS fp32 + AG bf16 (ACCO, ZeRO-1), ring AR fp32 (DDP)
        return frac * model.dim * 8.0 if method == "ddp" else frac * model.dim * (4.0 + 2.0)

    def comm_delay_ns(method):
        return comm_bytes(method) / 770e9 * 1e9

    def standin(method):
        if args.emulate_comm_gpus <= 1 or args.emulate_ctas <= 0:
            return {}
        return {"comm_standin_ctas": args.emulate_ctas, "comm_standin_bytes": comm_bytes(method)}

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    def timed(method, k, schedule, profile=False, clocks=False):
        sim = api.SimConfig(n_workers=world, batch_size=B, n_grad_accumulation=k, master_seed=1,
                            schedule=schedule, eval_every=0, worker_multipliers=mult,
                            throttle_host=args.straggler_mode == "host",
                            comm_delay_ns=comm_delay_ns(method), **standin(method))
        tr = api.Trainer(method, model, opt, sim, make_comm(method))
        tr.set_theta(model.default_theta0(1))
        tr.run(args.warmup)
        barrier()
        ck = Clocks(local) if clocks else None
        if ck:
            ck.__enter__()
        l0 = api.launch_count()
        recs, _, stats, _ = tr.run(args.steps)
        torch.cuda.synchronize()
        launches = api.launch_count() - l0
        if ck:
            ck.__exit__()
        barrier()
        ms = max_over_ranks(stats["wall_ms"])
        # consumed micro-batches are counted from the counts all-reduce: all ranks
        tokens = stats["consumed_micro_batches"] * B * T
        prof = None
        if profile:
            # a second pass of the same K steps with per-launch CUDA events on the
            # launching streams (kept out of the timed pass: ~300 event records
            # per micro-batch are not free)
            api.prof_enable(True)
            _, _, pstats, _ = tr.run(args.steps)
            torch.cuda.synchronize()
            prof = api.prof_read()
            prof["wall_ms"] = pstats["wall_ms"]
            api.prof_enable(False)
        # collectives of the timed pass from its CUDA-event timeline (this rank)
        tl = [iv for iv in tr.timeline() if iv.stream == "comm"]
        del tr
        coll = {}
        for kind in ("reduce_scatter", "all_gather", "optimizer", "all_reduce"):
            ivs = [iv for iv in tl if iv.kind == kind]
            if ivs:
                coll[kind] = {"ms_per_phase": max_over_ranks(sum(iv.t_end - iv.t_start for iv in ivs) / len(ivs) * 1e3),
                              "phases": len(ivs), "bytes_per_phase": ivs[0].bytes}
        return {"tokens_per_s": tokens / (ms / 1e3), "ms": ms, "ms_per_step": ms / args.steps, "tokens": tokens,
                "stats": stats, "prof": prof, "launches": launches, "clocks": ck.summary() if ck else None,
                "mb": [(r.mb_estimate, r.mb_main) for r in recs[:4]], "coll": coll}

    acco = timed("acco", 1, args.schedule, profile=True, clocks=True)
    base = {}
    if not args.no_baselines and not args.profile:
        base["zero1"] = timed("zero1", 2, "floor")
        base["ddp"] = timed("ddp", 2, "floor")

    # ---- end to end through the public API with host buffers (data-loader path)
    e2e = None
    if not args.profile:
        lm_h = api.LMConfig(**cfgd, n_samples=n_samples, data_seed=1, precision="bf16", max_batch=B, host_data=True)
        model_h = api.Model(lm_h)
        sim = api.SimConfig(n_workers=world, batch_size=B, n_grad_accumulation=1, master_seed=1,
                            schedule=args.schedule, eval_every=0, worker_multipliers=mult,
                            throttle_host=args.straggler_mode == "host",
                            comm_delay_ns=comm_delay_ns("acco"), **standin("acco"))
        tr = api.Trainer("acco", model_h, opt, sim, make_comm("acco"))
        tr.set_theta(model_h.default_theta0(1))
        tr.run(args.warmup)
        barrier()
        t0 = time.perf_counter()
        recs, _, st, _ = tr.run(args.steps)
        barrier()
        dt = max_over_ranks(time.perf_counter() - t0)
        tokens = st["consumed_micro_batches"] * B * T
        e2e = {"value": tokens / dt, "unit": "tokens/s",
               "h2d_bytes_per_step": st["h2d_bytes"] / args.steps,
               "d2h_bytes_per_step": st["d2h_bytes"] / args.steps,
               "path": "api.Trainer.run with LMConfig(host_data=True): per micro-batch the host draws the sample "
                       "indices, copies the token rows into pinned memory and ships them H2D; every micro-batch "
                       "loss is read back D2H as it completes; host wall clock around run()"}
        del tr, model_h

    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel class (GEMMs, tensor bound)
    p = acco["prof"]
    # DRAM traffic per launch from the committed `ncu --set full` capture of a
    # bench step (tools/gpu_r2_profile.sh -> profiles/prof_step_r02_raw.csv; the
    # capture's commit is in profiles/prof_step_r02_meta.json): static evidence
    # taken once per round, not measured in this run
    prof_dir = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles")

    def ncu_traffic(prefix):
        path = os.path.join(prof_dir, "prof_step_r02_raw.csv")
        try:
            with open(path) as f:
                rows = [r for r in csv.DictReader(f) if prefix in r["kernel"]]
        except (OSError, KeyError):
            return None
        if not rows:
            return None
        return sum(float(r["dram_read_bytes"]) + float(r["dram_write_bytes"]) for r in rows) / len(rows)

    try:
        with open(os.path.join(prof_dir, "prof_step_r02_meta.json")) as f:
            traffic_source = {"file": "profiles/prof_step_r02_raw.csv", **json.load(f)}
    except (OSError, ValueError):
        traffic_source = None
    g = p["gemm"]
    gemm_tf = g["work"] / (g["ms"] / 1e3) / 1e12 if g["ms"] > 0 else 0.0
    roof = {"kernel": "tcgen05 bf16 GEMM (fwd/dgrad/wgrad, all launches of the timed steps)", "bound": "tensor",
            "achieved": gemm_tf, "peak": tf_sus, "unit": "TFLOP/s", "frac": gemm_tf / tf_sus,
            "traffic": ncu_traffic("gemm_tc_kernel"),
            "traffic_note": "mean DRAM read+write bytes per GEMM launch, ncu --set full capture of 12 step GEMMs "
                            "(static evidence, see traffic_source); operands are re-read from L2, not DRAM",
            "traffic_source": traffic_source,
            "peak_kind": f"{peak_kind} sustained bf16 (kernel timed inside a long step)",
            "launches": g["launches"], "avg_launch_ms": g["ms"] / max(g["launches"], 1),
            "share_of_step": g["ms"] / p["wall_ms"]}
    o = p["optimizer"]
    opt_gbs = o["work"] / (o["ms"] / 1e3) / 1e9 if o["ms"] > 0 else 0.0
    roof_opt = {"kernel": "fused sharded AdamW estimate (K6) / commit (K7)", "bound": "hbm", "achieved": opt_gbs,
                "peak": hbm, "unit": "GB/s", "frac": opt_gbs / hbm, "traffic": ncu_traffic("opt_kernel"),
                "launches": o["launches"], "avg_launch_ms": o["ms"] / max(o["launches"], 1),
                "bytes_per_elem": "18 (estimate) + 34 (commit) = 52 B per shard element per update"}
    a = p["attention"]
    attn = {"ms": a["ms"], "tflops": a["work"] / (a["ms"] / 1e3) / 1e12 if a["ms"] > 0 else 0.0,
            "share_of_step": a["ms"] / p["wall_ms"]}

    # per-class device time of the profiled pass (CUDA events on the launching
    # streams; the optimizer class runs on the comm stream, concurrently)
    breakdown = {c: {"ms_per_step": v["ms"] / args.steps, "share_of_step": v["ms"] / p["wall_ms"],
                     "launches_per_step": v["launches"] / args.steps}
                 for c, v in p.items() if isinstance(v, dict) and v.get("launches")}

    cpu = None
    if not args.no_cpu_baseline and world == 1 and not args.profile and cfgd.get("arch", "gpt2") == "gpt2":
        # (the fp64 port of the 1.1B Llama would need ~40 GB host RAM and minutes
        # per sample: its CPU baseline is not taken)
        from oracle import cpu_bench
        from oracle import gpt_oracle as G

        r = cpu_bench.acco_round_sample(G.GPTConfig(**cfgd, n_samples=64, data_seed=1), batch=1)
        cpu = {"value": r["tokens_per_s"], "unit": "tokens/s", "cores": r["cores"], "kind": "port",
               "sample": r["sample"]}

    st = acco["stats"]

    def bus(c, n):  # NCCL bus bandwidth of a collective moving `bytes` per rank: bytes x (N-1)/N / t
        if n <= 1 or not c or c["ms_per_phase"] <= 0:
            return None
        return c["bytes_per_phase"] * (n - 1) / n / (c["ms_per_phase"] / 1e3) / 1e9
    collectives = {
        "n_ranks": world, "fabric": args.fabric,
        "nccl_version": ".".join(map(str, torch.cuda.nccl.version())) if world > 1 and args.fabric == "nccl" else None,
        "per_phase_ms": {k: v["ms_per_phase"] for k, v in acco["coll"].items()},
        "reduce_scatter_busbw_GBps": bus(acco["coll"].get("reduce_scatter"), world),
        "all_gather_busbw_GBps": bus(acco["coll"].get("all_gather"), world),
        "link_GBps": 900.0,
        "cost_model_ms_per_phase": {  # reference collective_time (collectives.cpp:16-25) at NVLink 5, alpha = 0
            k: (acco["coll"][k]["bytes_per_phase"] * (world - 1) / world / 900e9 * 1e3 if world > 1 else 0.0)
            for k in ("reduce_scatter", "all_gather") if k in acco["coll"]},
        "note": "from the timed ACCO pass's CUDA-event timeline on the comm stream (in-situ, overlapping compute); "
                "max over ranks"}
    line = {
        "metric": "tokens/s", "value": acco["tokens_per_s"], "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": acco["ms_per_step"], "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (seeded Markov-chain tokens, random-init weights)",
        "config": {"workload": f"{args.model} ACCO ({args.schedule} schedule, k=1), B={B}x{T} tokens per "
                               f"micro-batch per GPU, 2 micro-batches + 2 comm phases per update",
                   "model": args.model, "global_batch": int(acco["tokens"] / args.steps), "seq_len": T,
                   "parallelism": f"dp{world} ACCO (ZeRO-1-sharded fp32 AdamW states, " +
                                  ("NCCL RS/AG)" if args.fabric == "nccl" else
                                   "fused peer-memory fold+AdamW+replica-store kernel over NVLink)"),
                   "l2": "inputs larger than L2 (bf16 params 249 MB + activations per step)",
                   "eval": "no full-dataset evaluation inside the timed region: the reference's TraceBuilder::commit "
                           "evaluates f(theta), f(theta~) every update (protocols.cpp:113-134); here the cadence "
                           "eval_every = 0 (SURVEY.md a19); parity runs use eval_every = 1",
                   **({"straggler": f"rank 0 x{args.straggler} (HeterogeneityProfile multiplier, "
                                    f"{args.straggler_mode} throttle)"}
                      if args.straggler != 1.0 else {}),
                   **({"emulated_interconnect": {
                       "gpus": args.emulate_comm_gpus, "link_GBps": 770,
                       "phase_ms": {m: comm_delay_ns(m) / 1e6 for m in ("acco", "zero1", "ddp")},
                       "standin_ctas": args.emulate_ctas,
                       "note": "single GPU; each comm phase holds the comm stream for the NVLink time of the N-GPU "
                               "collectives, as a paced HBM copy of their bytes on standin_ctas CTAs (0: a spin)"}}
                      if args.emulate_comm_gpus > 1 else {})},
        "exposed_comm_pct": 100.0 * st["comm_exposed_ms"] / st["comm_busy_ms"] if st["comm_busy_ms"] else 0.0,
        "comm_busy_ms_per_step": st["comm_busy_ms"] / args.steps,
        "compute_busy_ms_per_step": st["compute_busy_ms"] / args.steps,
        "baselines": {k: {"tokens_per_s": v["tokens_per_s"], "ms_per_step": v["ms_per_step"],
                          "exposed_comm_pct": 100.0 * v["stats"]["comm_exposed_ms"] / v["stats"]["comm_busy_ms"]
                          if v["stats"]["comm_busy_ms"] else 0.0} for k, v in base.items()},
        "acco_vs_zero1_speedup": acco["tokens_per_s"] / base["zero1"]["tokens_per_s"] if "zero1" in base else None,
        "acco_vs_ddp_speedup": acco["tokens_per_s"] / base["ddp"]["tokens_per_s"] if "ddp" in base else None,
        "collectives": collectives,
        "roofline": roof, "roofline_optimizer": roof_opt, "attention": attn, "breakdown": breakdown,
        "cpu_baseline": cpu, "e2e": e2e, "clocks": acco["clocks"], "gpu_launches": acco["launches"],
        "stage_counts_first_updates": acco["mb"],
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
