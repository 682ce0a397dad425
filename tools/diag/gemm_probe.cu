// Timeline probe of the persistent tcgen05 GEMM: per CTA and tile, when the MMA
// warp starts / finishes issuing the tile and when epilogue warps 0 and last
// start / finish it. Diagnostic only.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DACCO_GEMM_PROBE \
//        --expt-relaxed-constexpr -Ipaper_2406_02613_b200/csrc -Iinclude tools/diag/gemm_probe.cu -lcuda -o tools/diag/gemm_probe.bin
#include "../../paper_2406_02613_b200/csrc/gemm_tcgen05.cu"

#include <vector>

namespace acco {
bool pdl_enabled() { return true; }
void count_launch() {}
int num_sms() { return 148; }
bool prof_on() { return false; }
cudaEvent_t prof_event() { return nullptr; }
void prof_record(int, double, cudaEvent_t, cudaEvent_t) {}
}  // namespace acco

int main(int argc, char** argv) {
    const int M = 8192, N = argc > 1 ? atoi(argv[1]) : 3072, K = argc > 2 ? atoi(argv[2]) : 768;
    const int mode = argc > 3 ? atoi(argv[3]) : 1;  // 0 store, 1 gelu, 2 dgelu
    __nv_bfloat16 *a, *b, *c, *aux;
    cudaMalloc(&a, size_t(M) * K * 2);
    cudaMalloc(&b, size_t(N) * K * 2);
    cudaMalloc(&c, size_t(M) * N * 2);
    cudaMalloc(&aux, size_t(M) * N * 2);
    cudaMemset(a, 0, size_t(M) * K * 2);
    cudaMemset(b, 0, size_t(N) * K * 2);
    cudaMemset(aux, 0, size_t(M) * N * 2);
    acco::GemmOperand A{a, K, false}, B{b, K, false};
    acco::Epilogue ep{};
    ep.mode = static_cast<acco::EpiMode>(mode);
    ep.C = c;
    ep.ldc = N;
    ep.aux = mode ? aux : nullptr;
    ep.ld_aux = N;
    cudaStream_t s;
    cudaStreamCreate(&s);
    for (int i = 0; i < 5; ++i) acco::gemm_bf16(A, B, M, N, K, ep, s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    for (int i = 0; i < 20; ++i) acco::gemm_bf16(A, B, M, N, K, ep, s);
    cudaEventRecord(e1, s);
    cudaStreamSynchronize(s);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("gemm %dx%dx%d mode %d: %.2f us\n", M, N, K, mode, ms * 50);
    static unsigned long long pr[148][6][16];
    std::vector<unsigned long long> z(148 * 6 * 16, 0);
    cudaMemcpyToSymbol(acco::g_gprobe, z.data(), sizeof(pr));
    acco::gemm_bf16(A, B, M, N, K, ep, s);
    cudaStreamSynchronize(s);
    cudaMemcpyFromSymbol(pr, acco::g_gprobe, sizeof(pr));
    printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
    unsigned long long t0 = ~0ull;
    for (int cta = 0; cta < 148; ++cta)
        for (int k = 0; k < 6; ++k)
            for (int i = 0; i < 16; ++i)
                if (pr[cta][k][i]) t0 = std::min(t0, pr[cta][k][i]);
    double mma = 0, epi0 = 0, epi7 = 0, stall = 0;
    int n = 0, ns = 0;
    for (int cta = 0; cta < 148; ++cta)
        for (int i = 0; i < 16; ++i)
            if (pr[cta][1][i] && pr[cta][3][i]) {
                mma += pr[cta][1][i] - pr[cta][0][i];
                epi0 += pr[cta][3][i] - pr[cta][2][i];
                epi7 += pr[cta][5][i] - pr[cta][4][i];
                ++n;
                if (i >= 2 && pr[cta][0][i]) {  // MMA start of tile i waited for the epilogue of tile i-2
                    stall += double(pr[cta][0][i]) - double(pr[cta][1][i - 1]);
                    ++ns;
                }
            }
    printf("per tile: MMA issue span %.0f ns, epilogue warp0 %.0f ns, warp last %.0f ns; gap MMA(i-1) end -> MMA(i) start %.0f ns (n=%d)\n",
           mma / n, epi0 / n, epi7 / n, stall / std::max(ns, 1), n);
    {
        unsigned long long t1 = 0;
        for (int cta = 0; cta < 148; ++cta)
            for (int k = 0; k < 6; ++k)
                for (int i = 0; i < 16; ++i) t1 = std::max(t1, pr[cta][k][i]);
        printf("kernel span (first MMA -> last epilogue): %.2f us\n", (t1 - t0) / 1000.0);
    }
    for (int cta : {0, 1, 100}) {
        printf("cta %d:\n", cta);
        for (int k = 0; k < 6; ++k) {
            printf("  kind %d:", k);
            for (int i = 0; i < 16; ++i)
                if (pr[cta][k][i]) printf(" %.2f", (pr[cta][k][i] - t0) / 1000.0);
            printf("\n");
        }
    }
    return 0;
}
