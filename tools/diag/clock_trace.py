"""SM clock / power / clock-event reasons sampled every ~2 ms (NVML) while
GPT-2-small micro-batches run back to back. Diagnostic only."""
import ctypes as C
import json
import sys
import threading
import time

import pynvml
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from oracle import accosim_oracle as O  # noqa: E402
from paper_2406_02613_b200 import _lib, api  # noqa: E402

cuda = torch.device("cuda")
cfg = dict(vocab=50257, d_model=768, n_layer=12, n_head=12, seq_len=1024)
m = api.Model(api.LMConfig(**cfg, n_samples=256, data_seed=1, precision="bf16", max_batch=8))
th = torch.tensor(m.default_theta0(1)).to(torch.bfloat16).to(cuda)
g = torch.zeros(m.dim, device=cuda)
loss = torch.zeros(1, dtype=torch.float64, device=cuda)
s = torch.cuda.current_stream()


def mb():
    _lib.call("acco_model_stochastic_grad", m.handle, C.c_void_p(th.data_ptr()), C.c_uint64(O.derive(1, 0, 0, 8, 0)), 8,
              C.c_void_p(g.data_ptr()), C.c_void_p(loss.data_ptr()), C.c_void_p(s.cuda_stream))


pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
samples = []
stop = False


def sampler():
    while not stop:
        samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                        pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
        time.sleep(0.002)


for _ in range(3):
    mb()
torch.cuda.synchronize()
t = threading.Thread(target=sampler)
t.start()
t0 = time.time()
n = 0
while time.time() - t0 < 4.0:
    for _ in range(10):
        mb()
    torch.cuda.synchronize()
    n += 10
stop = True
t.join()
clk = sorted(x[0] for x in samples)
pw = sorted(x[1] for x in samples)
reasons = {}
for x in samples:
    reasons[x[2]] = reasons.get(x[2], 0) + 1
print(json.dumps({"mb_per_s": n / (time.time() - t0), "samples": len(samples), "sm_mhz_p10_p50_p90": [clk[len(clk) // 10], clk[len(clk) // 2], clk[9 * len(clk) // 10]],
                  "min": clk[0], "power_w_p10_p50_p90": [pw[len(pw) // 10], pw[len(pw) // 2], pw[9 * len(pw) // 10]],
                  "reasons_hist": {hex(k): v for k, v in reasons.items()}}))
