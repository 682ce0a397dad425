"""cuBLAS (torch.matmul) bf16 throughput on the GPT-2 small GEMM shapes, as a
reference point for the tcgen05 GEMM (tools/gemm_bench.py)."""
import torch

M, d, V = 8192, 768, 50257
shapes = [("qkv_fwd", M, 3 * d, d), ("proj_fwd", M, d, d), ("fc_fwd", M, 4 * d, d), ("fc2_fwd", M, d, 4 * d),
          ("head_fwd", M, V, d), ("head_dgrad", M, d, V), ("head_wgrad", V, d, M)]
for name, m, n, k in shapes:
    a = torch.randn(m, k, device="cuda").bfloat16()
    b = torch.randn(k, n, device="cuda").bfloat16()
    for _ in range(3):
        c = a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        c = a @ b
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"{name:12s} cublas {ms * 1000:7.1f} us {2 * m * n * k / ms / 1e9:7.1f} TFLOP/s")
