"""the reference's acceptance criterion #7 at LM scale
(proj/tests/acceptance.cpp:166-205: 5 seeds x {DDP, DPU, ACCO}, final loss,
"DPU worse than DDP; ACCO within 2 % of DDP"; on the reference's MLP it
measured ddp 0.032016, dpu 0.0357662, acco 0.0319341), run on
the GPU engine for the LM configs:

  c1          BASELINE.json config 1: tiny GPT (V=256, d=128, L=2, T=64), 4 workers,
              B=8, 500 updates (acceptance #7's shape)
  c2-reduced  config 2 at reduced width: V=50257, d=64, L=12, T=1024, 2 workers,
              B=2, 500 updates, 1024 sequences, lr 6e-4 (the paper's pre-training lr)

Same protocol as the reference: free fabric (floor schedule; virtual workers on
one device), AdamW (beta2 0.95, cosine), n_grad_accumulation 1 for ACCO and 2
for DDP / DPU (equal samples per update, acceptance.cpp:180-182), theta0 =
default_theta0(seed), final loss = the full-dataset loss after the last update.
Prints one JSON object (per config: per-seed losses, means, the criteria).

  python tools/lm_acceptance.py [--configs c1,c2-reduced] [--seeds 101,...] [--precision bf16]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2406_02613_b200 import api  # noqa: E402

CONFIGS = {
    "c1": dict(lm=dict(vocab=256, d_model=128, n_layer=2, n_head=4, seq_len=64, n_samples=256, data_seed=1),
               workers=4, batch=8, updates=500, lr=3e-3),
    "c2-reduced": dict(lm=dict(vocab=50257, d_model=64, n_layer=12, n_head=1, seq_len=1024, n_samples=1024,
                               data_seed=1),
                       workers=2, batch=2, updates=500, lr=6e-4),
}


def final_losses(name, seeds, precision, methods=("ddp", "dpu", "acco")):
    c = CONFIGS[name]
    lm = api.LMConfig(**c["lm"], precision=precision, max_batch=max(c["batch"], 8))
    model = api.Model(lm)
    opt = api.OptimizerConfig(kind="adamw", learning_rate=c["lr"], adam_beta2=0.95, scheduler="cosine")
    out = {m: [] for m in methods}
    for seed in seeds:
        for m in methods:
            sim = api.SimConfig(n_workers=c["workers"], batch_size=c["batch"],
                                n_grad_accumulation=1 if m == "acco" else 2, master_seed=seed,
                                eval_every=c["updates"], eval_batch=8)
            tr = api.run_protocol(m, model, opt, sim, c["updates"], theta0=model.default_theta0(seed),
                                  record_history=False)
            out[m].append(tr.records[-1].loss)
    return out


def summarize(losses, seeds):
    mean = {m: sum(v) / len(v) for m, v in losses.items()}
    rel = abs(mean["acco"] - mean["ddp"]) / mean["ddp"]
    return {"seeds": seeds, "final_loss": losses, "mean": mean, "acco_vs_ddp_rel": rel,
            "acco_within_2pct_of_ddp": rel <= 0.02,
            "dpu_worse_than_ddp": mean["dpu"] > mean["ddp"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2-reduced")
    ap.add_argument("--seeds", default="101,102,103,104,105")
    ap.add_argument("--precision", default="bf16")
    ap.add_argument("--lr", type=float, default=0.0, help="override every config's learning rate")
    ap.add_argument("--updates", type=int, default=0, help="override every config's update count")
    ap.add_argument("--n-samples", type=int, default=0, help="override every config's dataset size")
    a = ap.parse_args()
    for c in CONFIGS.values():
        if a.lr > 0:
            c["lr"] = a.lr
        if a.updates > 0:
            c["updates"] = a.updates
        if a.n_samples > 0:
            c["lm"]["n_samples"] = a.n_samples
    seeds = [int(s) for s in a.seeds.split(",")]
    res = {"criterion": "reference acceptance #7 (proj/tests/acceptance.cpp:166-205) on the LM", "precision": a.precision}
    for name in a.configs.split(","):
        t0 = time.time()
        r = summarize(final_losses(name, seeds, a.precision), seeds)
        c = CONFIGS[name]
        r["config"] = {**c["lm"], "workers": c["workers"], "batch": c["batch"], "updates": c["updates"], "lr": c["lr"]}
        r["seconds"] = time.time() - t0
        res[name] = r
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
