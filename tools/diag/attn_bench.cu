// Standalone driver of the tcgen05 flash-attention kernels (attn_tc.cu) at the
// GPT-2-small shape (B = 8, T = 1024, H = 12, hd = 64): event-timed forward
// and backward, for A/B runs and ncu captures (args: B T H Hkv reps hd).
// Diagnostic only.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo \
//        -Ipaper_2406_02613_b200/csrc -Iinclude tools/diag/attn_bench.cu -lcuda -o tools/diag/attn_bench.bin
#include "../../paper_2406_02613_b200/csrc/attn_tc.cu"

#include <cstdio>
#include <vector>

namespace acco {
bool pdl_enabled() { return true; }
void count_launch() {}
int num_sms() { return 148; }
}  // namespace acco

int main(int argc, char** argv) {
    const int B = argc > 1 ? atoi(argv[1]) : 8, T = argc > 2 ? atoi(argv[2]) : 1024, H = argc > 3 ? atoi(argv[3]) : 12;
    const int Hkv = argc > 4 ? atoi(argv[4]) : H, reps = argc > 5 ? atoi(argv[5]) : 20,
              hd = argc > 6 ? atoi(argv[6]) : 64;
    const size_t n_qkv = size_t(B) * T * (H + 2 * Hkv) * hd, n_y = size_t(B) * T * H * hd;
    std::vector<__nv_bfloat16> h(n_qkv), hy(n_y);
    uint32_t st = 12345;
    for (auto& v : h) {
        st = st * 1664525u + 1013904223u;
        v = __float2bfloat16(((st >> 8) * (1.0f / 16777216.0f) - 0.5f) * 2.0f);
    }
    for (auto& v : hy) {
        st = st * 1664525u + 1013904223u;
        v = __float2bfloat16(((st >> 8) * (1.0f / 16777216.0f) - 0.5f));
    }
    __nv_bfloat16 *qkv, *y, *dy, *dqkv;
    float *lse, *dsum;
    cudaMalloc(&qkv, n_qkv * 2);
    cudaMalloc(&dqkv, n_qkv * 2);
    cudaMalloc(&y, n_y * 2);
    cudaMalloc(&dy, n_y * 2);
    cudaMalloc(&lse, size_t(B) * H * T * 4);
    cudaMalloc(&dsum, size_t(B) * H * T * 4);
    cudaMemcpy(qkv, h.data(), n_qkv * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dy, hy.data(), n_y * 2, cudaMemcpyHostToDevice);
    cudaStream_t s;
    cudaStreamCreate(&s);
    for (int i = 0; i < 3; ++i) {
        acco::attention_fwd_tc(qkv, y, lse, B, T, H, Hkv, hd, s);
        acco::attention_bwd_tc(qkv, y, lse, dy, dqkv, dsum, B, T, H, Hkv, hd, s);
    }
    cudaEvent_t e0, e1, e2;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventCreate(&e2);
    float tf = 0, tb = 0;
    for (int i = 0; i < reps; ++i) {
        cudaEventRecord(e0, s);
        acco::attention_fwd_tc(qkv, y, lse, B, T, H, Hkv, hd, s);
        cudaEventRecord(e1, s);
        acco::attention_bwd_tc(qkv, y, lse, dy, dqkv, dsum, B, T, H, Hkv, hd, s);
        cudaEventRecord(e2, s);
        cudaEventSynchronize(e2);
        float a, b;
        cudaEventElapsedTime(&a, e0, e1);
        cudaEventElapsedTime(&b, e1, e2);
        tf += a;
        tb += b;
    }
    tf /= reps;
    tb /= reps;
    // causal FLOPs: fwd 2 matmuls, bwd 5, each 2 * T^2/2 * hd per (b, h)
    const double f1 = 2.0 * B * H * (double(T) * T / 2) * hd * 2;
    printf("{\"hd\": %d, \"B\": %d, \"T\": %d, \"H\": %d, \"Hkv\": %d, \"fwd_us\": %.1f, \"bwd_us\": %.1f, \"fwd_tflops\": %.0f, "
           "\"bwd_tflops\": %.0f, \"err\": \"%s\"}\n",
           hd, B, T, H, Hkv, tf * 1e3, tb * 1e3, f1 / (tf * 1e-3) / 1e12, 2.5 * f1 / (tb * 1e-3) / 1e12,
           cudaGetErrorString(cudaGetLastError()));
    return 0;
}
