// fp32 SIMT GEMM: the A/B twin of the fp32-accurate parity contraction
// (precision "fp32" runs the 3xTF32 tcgen05 kernel, gemm_f32_tc; this kernel
// is selected only by ACCO_GEMM_SIMT=1). Sequential-k accumulation, no
// atomics, so the result is bitwise deterministic.
#include "common.cuh"
#include "epilogue.cuh"
#include "gemm.h"

#include <cstdlib>

namespace acco {
namespace {

constexpr int kT = 64;   // output tile
constexpr int kTK = 16;  // k-slice

template <int A_MN, int B_MN>
__global__ void __launch_bounds__(256) gemm_simt_kernel(const float* __restrict__ A, int64_t lda,
                                                        const float* __restrict__ B, int64_t ldb,
                                                        int M, int N, int K, Epilogue ep) {
    ACCO_PDL_PROLOGUE();
    __shared__ float As[kTK][kT + 4];
    __shared__ float Bs[kTK][kT + 4];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int m0 = blockIdx.y * kT, n0 = blockIdx.x * kT;
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

    for (int k0 = 0; k0 < K; k0 += kTK) {
        for (int i = threadIdx.x; i < kT * kTK; i += 256) {
            int mm, kk;
            if (A_MN) { mm = i % kT; kk = i / kT; } else { kk = i % kTK; mm = i / kTK; }
            const int gm = m0 + mm, gk = k0 + kk;
            As[kk][mm] = (gm < M && gk < K) ? (A_MN ? A[(int64_t)gk * lda + gm] : A[(int64_t)gm * lda + gk]) : 0.f;
            int nn;
            if (B_MN) { nn = i % kT; kk = i / kT; } else { kk = i % kTK; nn = i / kTK; }
            const int gn = n0 + nn, gk2 = k0 + kk;
            Bs[kk][nn] = (gn < N && gk2 < K) ? (B_MN ? B[(int64_t)gk2 * ldb + gn] : B[(int64_t)gn * ldb + gk2]) : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < kTK; ++kk) {
            float a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int row = m0 + ty * 4 + i;
        const int col = n0 + tx * 4;
        if (row < M && col < N) epilogue_row<float, 4>(ep, row, col, min(4, N - col), acc[i]);
    }
}

}  // namespace

void gemm_f32(const GemmOperand& A, const GemmOperand& B, int M, int N, int K, const Epilogue& ep,
              cudaStream_t stream) {
    const bool simt = std::getenv("ACCO_GEMM_SIMT") != nullptr;  // A/B knob (read per call): the SIMT kernel
    if (simt)
        gemm_f32_simt(A, B, M, N, K, ep, stream);
    else
        gemm_f32_tc(A, B, M, N, K, ep, stream);
}

void gemm_f32_simt(const GemmOperand& A, const GemmOperand& B, int M, int N, int K, const Epilogue& ep,
                   cudaStream_t stream) {
    ACCO_REQUIRE(ep.mode <= kEpiAccF32, "gemm_f32: epilogue mode not supported by the SIMT path");
    ACCO_REQUIRE(M > 0 && N > 0 && K > 0, "gemm_f32: empty problem");
    ProfScope prof(kProfGemm, 2.0 * M * N * K, stream);
    dim3 grid(ceil_div(N, kT), ceil_div(M, kT));
    const float* a = static_cast<const float*>(A.ptr);
    const float* b = static_cast<const float*>(B.ptr);
    if (!A.mn_major && !B.mn_major)
        launch_pdl(gemm_simt_kernel<0, 0>, grid, 256, 0, stream, a, A.ld, b, B.ld, M, N, K, ep);
    else if (!A.mn_major && B.mn_major)
        launch_pdl(gemm_simt_kernel<0, 1>, grid, 256, 0, stream, a, A.ld, b, B.ld, M, N, K, ep);
    else if (A.mn_major && !B.mn_major)
        launch_pdl(gemm_simt_kernel<1, 0>, grid, 256, 0, stream, a, A.ld, b, B.ld, M, N, K, ep);
    else
        launch_pdl(gemm_simt_kernel<1, 1>, grid, 256, 0, stream, a, A.ld, b, B.ld, M, N, K, ep);
    ACCO_CHECK_LAUNCH();
}

}  // namespace acco
