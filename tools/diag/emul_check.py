import sys, json
sys.path.insert(0, "/root/repo")
from paper_2406_02613_b200 import api
lm = api.LMConfig(vocab=50257, d_model=768, n_layer=12, n_head=12, seq_len=1024, n_samples=64, precision="bf16", max_batch=8)
model = api.Model(lm)
opt = api.OptimizerConfig(kind="adamw", learning_rate=6e-4, adam_beta2=0.95, total_steps=1000)
for method, k in (("zero1", 2), ("acco", 1)):
    for delay, ctas in ((0, 0), (5e6, 0), (5e6, 16)):
        sim = api.SimConfig(n_workers=1, batch_size=8, n_grad_accumulation=k, master_seed=1, eval_every=0,
                            comm_delay_ns=delay, comm_standin_ctas=ctas, comm_standin_bytes=650e6 if ctas else 0)
        tr = api.Trainer(method, model, opt, sim)
        tr.set_theta(model.default_theta0(1))
        tr.run(3)
        recs, _, st, _ = tr.run(8)
        tl = tr.timeline()
        comm = [iv for iv in tl if iv.stream == "comm"]
        print(json.dumps({"method": method, "delay_ms": delay/1e6, "ctas": ctas, "ms_per_update": st["wall_ms"]/8,
                          "comm_busy_ms": st["comm_busy_ms"]/8, "exposed_ms": st["comm_exposed_ms"]/8}), flush=True)
        del tr
