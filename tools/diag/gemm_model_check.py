"""GEMM plan-model validation (configs captured as CUDA graphs, timed
interleaved over rounds, min per config): for every GEMM shape of GPT-2 small / medium and
Llama-1B (M = 8192 tokens), CUDA-graph device time of every tile config
(BN x CTA group x split-K) and of the model's own pick ("auto"). One JSON line
per shape: {cfg: us}; used to fit / check plan_time (gemm_tcgen05.cu)."""
import json
import os
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2406_02613_b200.ops import gemm  # noqa: E402

dev = torch.device("cuda")
M = 8192


def shapes(d, F, V, nqkv):
    return [("qkv_fwd", M, nqkv, d, 0, 0, "store"), ("proj_fwd", M, d, d, 0, 0, "store"),
            ("fc_fwd", M, F, d, 0, 0, "store"), ("fc2_fwd", M, d, F, 0, 0, "store"),
            ("head_fwd", M, V, d, 0, 0, "store"),
            ("fc2_dgrad", M, F, d, 0, 1, "store"), ("fc_dgrad", M, d, F, 0, 1, "store"),
            ("qkv_dgrad", M, d, nqkv, 0, 1, "store"), ("proj_dgrad", M, d, d, 0, 1, "store"),
            ("fc2_wgrad", d, F, M, 1, 1, "acc_f32"), ("fc_wgrad", F, d, M, 1, 1, "acc_f32"),
            ("qkv_wgrad", nqkv, d, M, 1, 1, "acc_f32"), ("proj_wgrad", d, d, M, 1, 1, "acc_f32"),
            ("head_wgrad", V, d, M, 1, 1, "acc_f32")]


MODELS = {"gpt2-small": shapes(768, 3072, 50257, 2304), "gpt2-medium": shapes(1024, 4096, 50257, 3072),
          "llama-1b": shapes(2048, 5632, 32000, 2560)}


REPS, ROUNDS = 10, 5


def capture(run, cs):
    with torch.cuda.stream(cs):
        for _ in range(2):
            run()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=cs):
        for _ in range(REPS):
            run()
    g.replay()
    torch.cuda.synchronize()
    return g


def replay_us(g):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / REPS * 1e3


def main():
    only = sys.argv[1].split(",") if len(sys.argv) > 1 else list(MODELS)
    cs = torch.cuda.Stream()
    for model in only:
        for name, m, n, k, amn, bmn, mode in MODELS[model]:
            def mat(r, c):
                return torch.randn(r, (c + 63) // 64 * 64, device=dev).to(torch.bfloat16)[:, :c]
            a = mat(k, m) if amn else mat(m, k)
            b = mat(k, n) if bmn else mat(n, k)
            ldc = (n + 63) // 64 * 64
            c = torch.zeros(m, ldc, device=dev) if mode == "acc_f32" else torch.empty(m, ldc, dtype=torch.bfloat16,
                                                                                       device=dev)
            kw = dict(mode=mode, beta=1 if mode == "acc_f32" else 0)
            cfgs = ["auto"]
            for cg in (1, 2):
                for bn in (256, 192, 128):
                    if cg == 2 and bn == 192 and bmn:
                        continue
                    for sp in ((1, 2, 3, 4) if mode == "acc_f32" else (1,)):
                        cfgs.append(f"{bn},{sp},{cg}")
            row = {"model": model, "name": name, "shape": [m, n, k, amn, bmn, mode]}
            graphs = {}
            for cfg in cfgs:  # capture every config once ...
                if cfg == "auto":
                    os.environ.pop("ACCO_GEMM_FORCE", None)
                else:
                    os.environ["ACCO_GEMM_FORCE"] = cfg
                try:
                    graphs[cfg] = capture(lambda: gemm(a, bool(amn), b, bool(bmn), m, n, k, c, **kw), cs)
                except Exception as e:  # noqa: BLE001
                    row[cfg] = str(e)[:80]
            best = {cfg: 1e9 for cfg in graphs}
            for _ in range(ROUNDS):  # ... then time them interleaved, min over rounds (clock drift under the power cap)
                for cfg, g in graphs.items():
                    best[cfg] = min(best[cfg], replay_us(g))
            row.update({cfg: round(v, 2) for cfg, v in best.items()})
            del graphs
            os.environ.pop("ACCO_GEMM_FORCE", None)
            print(json.dumps(row), flush=True)
            del a, b, c
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
