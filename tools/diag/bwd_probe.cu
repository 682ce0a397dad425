// Timeline probe of the persistent flash-attention dK/dV kernel (fa_bwd_dkv_tc):
// per CTA and tile g, the MMA warp's S^T/dP^T issue (0) and dV/dK issue (1), and
// softmax warp 4's tile barrier (2), S ready (3), math done (4), previous dV/dK
// done (5), P^T/dS^T stored (6). Diagnostic only.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DACCO_BWD_PROBE \
//        -Ipaper_2406_02613_b200/csrc -Iinclude tools/diag/bwd_probe.cu -lcuda -o tools/diag/bwd_probe.bin
#include "../../paper_2406_02613_b200/csrc/attn_tc.cu"

#include <cstdio>

namespace acco {
bool pdl_enabled() { return true; }
void count_launch() {}
int num_sms() { return 148; }
}  // namespace acco

int main(int argc, char** argv) {
    const int B = argc > 1 ? atoi(argv[1]) : 8, T = argc > 2 ? atoi(argv[2]) : 1024, H = argc > 3 ? atoi(argv[3]) : 12;
    const int Hkv = H, hd = 64;
    const size_t n_qkv = size_t(B) * T * (H + 2 * Hkv) * hd, n_y = size_t(B) * T * H * hd;
    std::vector<__nv_bfloat16> h(n_qkv), hy(n_y);
    uint32_t st = 12345;
    for (auto& v : h) {
        st = st * 1664525u + 1013904223u;
        v = __float2bfloat16(((st >> 8) * (1.0f / 16777216.0f) - 0.5f));
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
    acco::attention_fwd_tc(qkv, y, lse, B, T, H, Hkv, hd, s);
    for (int i = 0; i < 3; ++i) acco::attention_bwd_tc(qkv, y, lse, dy, dqkv, dsum, B, T, H, Hkv, hd, s);
    static unsigned long long pr[148][8][64];
    std::vector<unsigned long long> z(148 * 8 * 64, 0);
    cudaMemcpyToSymbol(acco::g_bprobe, z.data(), sizeof(pr));
    acco::attention_bwd_tc(qkv, y, lse, dy, dqkv, dsum, B, T, H, Hkv, hd, s);
    cudaStreamSynchronize(s);
    cudaMemcpyFromSymbol(pr, acco::g_bprobe, sizeof(pr));
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    unsigned long long t0 = ~0ull, t1 = 0;
    for (int c = 0; c < 148; ++c)
        for (int k = 0; k < 8; ++k)
            for (int i = 0; i < 64; ++i)
                if (pr[c][k][i]) {
                    t0 = std::min(t0, pr[c][k][i]);
                    t1 = std::max(t1, pr[c][k][i]);
                }
    printf("dkv span %.2f us\n", (t1 - t0) / 1000.0);
    // mean phase durations over steady-state tiles (g >= 2)
    const char* nm[] = {"bar->S ready", "S ready->math done", "math done->prev dVdK done", "prev done->P stored",
                        "P stored->next bar", "Sissue(g)->S ready(g)", "P stored(g)->dVdK issue(g)"};
    double acc[7] = {0};
    int n = 0;
    for (int c = 0; c < 148; ++c)
        for (int g = 2; g < 63; ++g) {
            if (!pr[c][6][g] || !pr[c][2][g + 1]) continue;
            acc[0] += pr[c][3][g] - pr[c][2][g];
            acc[1] += pr[c][4][g] - pr[c][3][g];
            acc[2] += pr[c][5][g] - pr[c][4][g];
            acc[3] += pr[c][6][g] - pr[c][5][g];
            acc[4] += pr[c][2][g + 1] - pr[c][6][g];
            acc[5] += double(pr[c][3][g]) - double(pr[c][0][g]);
            acc[6] += double(pr[c][1][g]) - double(pr[c][6][g]);
            ++n;
        }
    for (int k = 0; k < 7; ++k) printf("  %-28s %7.0f ns\n", nm[k], acc[k] / std::max(n, 1));
    {  // observer (warp 3): S^T/dP^T completion vs issue and vs the softmax seeing it
        double a = 0, b = 0;
        int m = 0;
        for (int c = 0; c < 148; ++c)
            for (int g = 1; g < 63; ++g)
                if (pr[c][7][g] && pr[c][0][g] && pr[c][3][g]) {
                    a += double(pr[c][7][g]) - double(pr[c][0][g]);
                    b += double(pr[c][3][g]) - double(pr[c][7][g]);
                    ++m;
                }
        printf("  S issue -> S complete (observer) %7.0f ns; complete -> softmax sees it %7.0f ns (n=%d)\n",
               a / std::max(m, 1), b / std::max(m, 1), m);
    }
    printf("cta 0 (us): \n");
    for (int k = 0; k < 8; ++k) {
        printf(" k%d:", k);
        for (int i = 0; i < 12; ++i)
            if (pr[0][k][i]) printf(" %.2f", (pr[0][k][i] - t0) / 1000.0);
        printf("\n");
    }
    return 0;
}
