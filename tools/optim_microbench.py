"""BASELINE.json config 5: optimizer-round microbench — one ACCO round's comm
stream on one B200: counts all-reduce + reduce-scatter + K6 estimate (transient)
+ all-gather + counts AR + RS + K7 commit (with the retained shard) + AG, at
Psi in {10M, 100M, 1B, 2B} fp32 gradients ~ N(0,1), theta ~ 0.02 N(0,1), m=v=0.
Reports the fused-optimizer HBM throughput against the measured copy peak and
the whole round time; the reference CPU round (oracle/_ref/ref_round_bench,
fp64, single thread) is timed at 10M for context. One JSON line per size.

  python tools/optim_microbench.py [--sizes 1e7,1e8,1e9,2e9] [--reps 10]
"""
import argparse
import ctypes as C
import json
import os
import socket
import subprocess
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2406_02613_b200 import _lib, api  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="1e7,1e8,1e9,2e9")
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
        hbm = json.load(f)["hbm_gbs"]
    import torch.distributed as dist

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    comm = api.Comm(0, 1, 0)
    h = comm.handle
    dev = torch.device("cuda")
    stream = torch.cuda.current_stream()
    sp = C.c_void_p(stream.cuda_stream)
    cfg = api.OptimizerConfig(kind="adamw", learning_rate=6e-4, weight_decay=0.1, adam_beta2=0.95,
                              scheduler="cosine", total_steps=1000).to_c()
    for psi in [int(float(x)) for x in args.sizes.split(",")]:
        g_main = torch.randn(psi, device=dev)
        g_est = torch.randn(psi, device=dev)
        red_main = torch.empty(psi, device=dev)
        red_est = torch.empty(psi, device=dev)
        theta = 0.02 * torch.randn(psi, device=dev)
        m = torch.zeros(psi, device=dev)
        v = torch.zeros(psi, device=dev)
        est_out = torch.empty(psi, dtype=torch.bfloat16, device=dev)
        th_out = torch.empty(psi, dtype=torch.bfloat16, device=dev)
        cnt = torch.tensor([8], dtype=torch.int64, device=dev)
        tot = torch.zeros(2, dtype=torch.int64, device=dev)
        st = _lib.ShardState(0, theta.data_ptr(), m.data_ptr(), v.data_ptr(), 0, psi)
        P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731

        def round_():
            _lib.call("acco_all_reduce_i64", h, P(cnt), P(tot[0:1]), 1, sp)
            _lib.call("acco_reduce_scatter_f32", h, P(g_est), P(red_est), psi, sp)
            e0.record(stream)
            _lib.call("acco_opt_estimate", C.byref(cfg), C.byref(st), P(red_est), P(tot[0:1]), P(est_out),
                      _lib.DTYPE_BF16, None, sp)
            e1.record(stream)
            _lib.call("acco_all_gather", h, P(est_out), P(est_out), psi, _lib.DTYPE_BF16, sp)
            _lib.call("acco_all_reduce_i64", h, P(cnt), P(tot[1:2]), 1, sp)
            _lib.call("acco_reduce_scatter_f32", h, P(g_main), P(red_main), psi, sp)
            e2.record(stream)
            _lib.call("acco_opt_commit", C.byref(cfg), C.byref(st), P(red_main), P(red_est), P(tot[1:2]),
                      P(tot[0:1]), P(th_out), _lib.DTYPE_BF16, None, sp)
            e3.record(stream)
            _lib.call("acco_all_gather", h, P(th_out), P(th_out), psi, _lib.DTYPE_BF16, sp)

        e0, e1, e2, e3 = (torch.cuda.Event(enable_timing=True) for _ in range(4))
        for _ in range(3):
            round_()
        torch.cuda.synchronize()
        ta, tb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t_est = t_com = 0.0
        ta.record(stream)
        for _ in range(args.reps):
            round_()
            e3.synchronize()
            t_est += e0.elapsed_time(e1)
            t_com += e2.elapsed_time(e3)
        tb.record(stream)
        torch.cuda.synchronize()
        round_ms = ta.elapsed_time(tb) / args.reps
        t_est /= args.reps
        t_com /= args.reps
        gbs_est = 18.0 * psi / (t_est / 1e3) / 1e9
        gbs_com = 34.0 * psi / (t_com / 1e3) / 1e9
        gbs_opt = 52.0 * psi / ((t_est + t_com) / 1e3) / 1e9
        line = {"metric": "optimizer-round params/s (ACCO estimate+commit, fused AdamW, N=1)",
                "psi": psi, "value": psi / (round_ms / 1e3), "unit": "params/s", "round_ms": round_ms,
                "estimate_ms": t_est, "commit_ms": t_com,
                "roofline": {"bound": "hbm", "achieved": gbs_opt, "peak": hbm, "unit": "GB/s",
                             "frac": gbs_opt / hbm, "estimate_gbs": gbs_est, "commit_gbs": gbs_com,
                             "bytes_per_elem": 52}}
        if psi == int(1e7):
            exe = os.path.join(ROOT, "oracle", "_ref", "ref_round_bench")
            if os.path.exists(exe):
                r = subprocess.run([exe, str(psi), "8", "3"], capture_output=True, text=True, timeout=600)
                try:
                    ref = json.loads(r.stdout.strip().splitlines()[-1])
                    line["cpu_baseline"] = {"value": ref["params_per_s"], "unit": "params/s", "cores": 1,
                                            "kind": "reference", "sample": "reference Fabric RS + sharded_opt_step "
                                            "(estimate, commit) + all_gather, fp64, N=8 simulated workers, Psi=1e7"}
                except Exception as e:  # noqa: BLE001
                    line["cpu_baseline"] = {"error": str(e)[:200]}
        print(json.dumps(line), flush=True)
        del g_main, g_est, red_main, red_est, theta, m, v, est_out, th_out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
