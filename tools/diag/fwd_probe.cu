// Timeline probe of the persistent flash-attention forward (fa_fwd_tc2):
// %globaltimer stamps of the MMA warp's S / PV issues and of one softmax warp
// per tile slot (S ready, P stored), per CTA. Diagnostic only.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DACCO_FWD_PROBE \
//        -Ipaper_2406_02613_b200/csrc -Iinclude tools/diag/fwd_probe.cu -lcuda -o /tmp/fwd_probe
#include "../../paper_2406_02613_b200/csrc/attn_tc.cu"

#include <cstdio>

namespace acco {
bool pdl_enabled() { return true; }
void count_launch() {}
int num_sms() { int d, n; cudaGetDevice(&d); cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d); return n; }
}  // namespace acco

int main(int argc, char** argv) {
    const int B = argc > 1 ? atoi(argv[1]) : 8, T = argc > 2 ? atoi(argv[2]) : 1024, H = argc > 3 ? atoi(argv[3]) : 12;
    const int Hkv = H, hd = 64;
    const size_t n_qkv = size_t(B) * T * (H + 2 * Hkv) * hd;
    std::vector<__nv_bfloat16> h(n_qkv);
    uint32_t st = 12345;
    for (auto& v : h) {
        st = st * 1664525u + 1013904223u;
        v = __float2bfloat16(((st >> 8) * (1.0f / 16777216.0f) - 0.5f));
    }
    __nv_bfloat16 *qkv, *y;
    float* lse;
    cudaMalloc(&qkv, n_qkv * 2);
    cudaMalloc(&y, size_t(B) * T * H * hd * 2);
    cudaMalloc(&lse, size_t(B) * H * T * 4);
    cudaMemcpy(qkv, h.data(), n_qkv * 2, cudaMemcpyHostToDevice);
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int i = 0; i < 5; ++i) acco::attention_fwd_tc(qkv, y, lse, B, T, H, Hkv, hd, s);
    cudaEventRecord(e0, s);
    const int reps = 20;
    for (int i = 0; i < reps; ++i) acco::attention_fwd_tc(qkv, y, lse, B, T, H, Hkv, hd, s);
    cudaEventRecord(e1, s);
    cudaStreamSynchronize(s);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("fa_fwd_tc2 B=%d T=%d H=%d: %.2f us per launch (back to back)\n", B, T, H, ms * 1000 / reps);
    {  // spot check against fp64 for a few rows of (b = B-1, h = H-1)
        std::vector<__nv_bfloat16> yh(size_t(B) * T * H * hd);
        cudaMemcpy(yh.data(), y, yh.size() * 2, cudaMemcpyDeviceToHost);
        const int ld = (H + 2 * Hkv) * hd, b = B - 1, hh = H - 1;
        double worst = 0;
        for (int q : {0, 1, 127, 128, 129, T / 2 + 5, T - 1}) {
            auto at = [&](int row, int col) { return double(__bfloat162float(h[(size_t(b) * T + row) * ld + col])); };
            std::vector<double> sc(q + 1);
            double mx = -1e300;
            for (int k = 0; k <= q; ++k) {
                double a = 0;
                for (int c = 0; c < hd; ++c) a += at(q, hh * hd + c) * at(k, (H + hh) * hd + c);
                sc[k] = a / std::sqrt(double(hd));
                mx = std::max(mx, sc[k]);
            }
            double l = 0;
            for (auto& v : sc) l += (v = std::exp(v - mx));
            for (int c = 0; c < hd; ++c) {
                double o = 0;
                for (int k = 0; k <= q; ++k) o += sc[k] * at(k, (H + Hkv + hh) * hd + c);
                o /= l;
                const double g = __bfloat162float(yh[(size_t(b) * T + q) * H * hd + hh * hd + c]);
                worst = std::max(worst, std::abs(g - o));
            }
        }
        printf("max abs err vs fp64 (7 rows): %.3e\n", worst);
    }
    static unsigned long long pr[148][10][128];
    cudaMemcpyFromSymbol(pr, acco::g_probe, sizeof(pr));
    // zero the probe then one more launch so every stamp belongs to it
    std::vector<unsigned long long> z(148 * 10 * 128, 0);
    cudaMemcpyToSymbol(acco::g_probe, z.data(), sizeof(pr));
    acco::attention_fwd_tc(qkv, y, lse, B, T, H, Hkv, hd, s);
    cudaStreamSynchronize(s);
    cudaMemcpyFromSymbol(pr, acco::g_probe, sizeof(pr));
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    unsigned long long t0 = ~0ull, t1 = 0;
    for (int c = 0; c < 148; ++c)
        for (int k = 0; k < 10; ++k)
            for (int i = 0; i < 128; ++i)
                if (pr[c][k][i]) {
                    t0 = std::min(t0, pr[c][k][i]);
                    t1 = std::max(t1, pr[c][k][i]);
                }
    printf("probe span %.2f us\n", (t1 - t0) / 1000.0);
    // per-CTA summary: first / last stamp, #S issues, mean softmax latency
    // (S ready -> P stored) per slot, mean S-ready wait after the previous P
    double sm_lat[2] = {0, 0}, gap[2] = {0, 0};
    int nlat[2] = {0, 0}, ngap[2] = {0, 0};
    for (int c = 0; c < 148; ++c) {
        unsigned long long a = ~0ull, b = 0;
        int ns = 0;
        for (int i = 0; i < 128; ++i)
            if (pr[c][0][i]) {
                ++ns;
                a = std::min(a, pr[c][0][i]);
            }
        for (int k = 0; k < 10; ++k)
            for (int i = 0; i < 128; ++i) b = std::max(b, pr[c][k][i]);
        for (int x = 0; x < 2; ++x)
            for (int i = 0; i < 128; ++i) {
                if (pr[c][2 + 2 * x][i] && pr[c][3 + 2 * x][i]) {
                    sm_lat[x] += pr[c][3 + 2 * x][i] - pr[c][2 + 2 * x][i];
                    ++nlat[x];
                }
                if (i > 0 && pr[c][2 + 2 * x][i] && pr[c][3 + 2 * x][i - 1]) {
                    gap[x] += double(pr[c][2 + 2 * x][i]) - double(pr[c][3 + 2 * x][i - 1]);
                    ++ngap[x];
                }
            }
        if (c < 6 || c % 37 == 0)
            printf("cta %3d: start %+8.2f us end %8.2f us, S issues %d\n", c, (a - t0) / 1000.0, (b - t0) / 1000.0, ns);
    }
    {  // slot-0 softmax phases: S ready -> ld done -> partner barrier -> exp done -> st done
        double ph[4] = {0, 0, 0, 0};
        int np = 0;
        for (int c = 0; c < 148; ++c)
            for (int i = 0; i < 128; ++i)
                if (pr[c][2][i] && pr[c][9][i]) {
                    ph[0] += pr[c][6][i] - pr[c][2][i];
                    ph[1] += pr[c][7][i] - pr[c][6][i];
                    ph[2] += pr[c][8][i] - pr[c][7][i];
                    ph[3] += pr[c][9][i] - pr[c][8][i];
                    ++np;
                }
        printf("slot 0 phases (ns): ld %.0f, max+barrier %.0f, exp+pack %.0f, st(+rescale) %.0f\n", ph[0] / np,
               ph[1] / np, ph[2] / np, ph[3] / np);
    }
    for (int x = 0; x < 2; ++x)
        printf("slot %d: softmax S-ready->P-stored %.0f ns (n=%d); P-stored -> next S-ready %.0f ns (n=%d)\n", x,
               sm_lat[x] / std::max(1, nlat[x]), nlat[x], gap[x] / std::max(1, ngap[x]), ngap[x]);
    // detailed trace of CTA 0
    printf("cta 0 trace (us from start): kind idx t\n");
    for (int k = 0; k < 10; ++k) {
        printf("kind %d:", k);
        for (int i = 0; i < 40; ++i)
            if (pr[0][k][i]) printf(" %.2f", (pr[0][k][i] - t0) / 1000.0);
        printf("\n");
    }
    return 0;
}
