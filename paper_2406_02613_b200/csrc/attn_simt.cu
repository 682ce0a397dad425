// Causal multi-head attention, SIMT fp32 arithmetic (both activation dtypes).
// Flash-style: online softmax forward saving the row log-sum-exp; backward
// recomputes probabilities from lse (dQ pass over keys, dK/dV pass over
// queries). Sequential per-thread loops => bitwise deterministic.
// This is the fp32-accurate parity path; the bf16 throughput path uses the
// tensor-core kernel in attn_mma.cu when available for the head size.
#include "epilogue.cuh"
#include "lm_kernels.h"

namespace acco {
namespace {

constexpr int kTile = 64;

template <class T, int HD>
__global__ void __launch_bounds__(kTile) attn_fwd_kernel(const T* __restrict__ qkv, T* __restrict__ y,
                                                         float* __restrict__ lse, int seq, int H, int Hkv,
                                                         float scale) {
    ACCO_PDL_PROLOGUE();
    extern __shared__ float sm[];
    float(*Ks)[HD + 1] = reinterpret_cast<float(*)[HD + 1]>(sm);
    float(*Vs)[HD + 1] = reinterpret_cast<float(*)[HD + 1]>(sm + kTile * (HD + 1));
    const int bh = blockIdx.x, b = bh / H, h = bh % H;
    const int d = H * HD;
    const int64_t ld = static_cast<int64_t>(H + 2 * Hkv) * HD;
    const int kc = d + (h / (H / Hkv)) * HD, vc = kc + Hkv * HD;  // this head's K / V columns
    const int t = blockIdx.y * kTile + threadIdx.x;
    const int64_t base = static_cast<int64_t>(b) * seq * ld;
    float q[HD], o[HD];
    if (t < seq) {
#pragma unroll
        for (int c = 0; c < HD; ++c) q[c] = to_f(qkv[base + t * ld + h * HD + c]) * scale;
    }
#pragma unroll
    for (int c = 0; c < HD; ++c) o[c] = 0.f;
    float m = -INFINITY, l = 0.f;
    const int jmax = min(seq - 1, blockIdx.y * kTile + kTile - 1);
    for (int j0 = 0; j0 <= jmax; j0 += kTile) {
        __syncthreads();
        for (int i = threadIdx.x; i < kTile * HD; i += kTile) {
            const int r = i / HD, c = i % HD;
            const int j = j0 + r;
            Ks[r][c] = j < seq ? to_f(qkv[base + j * ld + kc + c]) : 0.f;
            Vs[r][c] = j < seq ? to_f(qkv[base + j * ld + vc + c]) : 0.f;
        }
        __syncthreads();
        if (t < seq) {
            const int jend = min(kTile, t - j0 + 1);
            for (int jj = 0; jj < jend; ++jj) {
                float s = 0.f;
#pragma unroll
                for (int c = 0; c < HD; ++c) s = fmaf(q[c], Ks[jj][c], s);
                if (s > m) {
                    const float corr = expf(m - s);
                    l *= corr;
#pragma unroll
                    for (int c = 0; c < HD; ++c) o[c] *= corr;
                    m = s;
                }
                const float p = expf(s - m);
                l += p;
#pragma unroll
                for (int c = 0; c < HD; ++c) o[c] = fmaf(p, Vs[jj][c], o[c]);
            }
        }
    }
    if (t < seq) {
        const float inv = 1.f / l;
        T* yr = y + (static_cast<int64_t>(b) * seq + t) * d + h * HD;
#pragma unroll
        for (int c = 0; c < HD; ++c) yr[c] = from_f<T>(o[c] * inv);
        lse[(static_cast<int64_t>(bh)) * seq + t] = m + logf(l);
    }
}

// D[bh, t] = sum_c dO[t,c] * O[t,c]
template <class T, int HD>
__global__ void attn_dsum_kernel(const T* __restrict__ y, const T* __restrict__ dy, float* __restrict__ dsum,
                                 int B, int seq, int H) {
    ACCO_PDL_PROLOGUE();
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= static_cast<int64_t>(B) * H * seq) return;
    const int t = static_cast<int>(idx % seq);
    const int bh = static_cast<int>(idx / seq);
    const int b = bh / H, h = bh % H;
    const int d = H * HD;
    const int64_t o = (static_cast<int64_t>(b) * seq + t) * d + h * HD;
    float s = 0.f;
    for (int c = 0; c < HD; ++c) s += to_f(dy[o + c]) * to_f(y[o + c]);
    dsum[idx] = s;
}

template <class T, int HD>
__global__ void __launch_bounds__(kTile) attn_dq_kernel(const T* __restrict__ qkv, const float* __restrict__ lse,
                                                        const float* __restrict__ dsum, const T* __restrict__ dy,
                                                        T* __restrict__ dqkv, int seq, int H, int Hkv,
                                                        float scale) {
    ACCO_PDL_PROLOGUE();
    extern __shared__ float sm[];
    float(*Ks)[HD + 1] = reinterpret_cast<float(*)[HD + 1]>(sm);
    float(*Vs)[HD + 1] = reinterpret_cast<float(*)[HD + 1]>(sm + kTile * (HD + 1));
    const int bh = blockIdx.x, b = bh / H, h = bh % H;
    const int d = H * HD;
    const int64_t ld = static_cast<int64_t>(H + 2 * Hkv) * HD;
    const int kc = d + (h / (H / Hkv)) * HD, vc = kc + Hkv * HD;
    const int t = blockIdx.y * kTile + threadIdx.x;
    const int64_t base = static_cast<int64_t>(b) * seq * ld;
    float q[HD], dO[HD], dq[HD];
    float L = 0.f, Dt = 0.f;
    if (t < seq) {
#pragma unroll
        for (int c = 0; c < HD; ++c) {
            q[c] = to_f(qkv[base + t * ld + h * HD + c]);
            dO[c] = to_f(dy[(static_cast<int64_t>(b) * seq + t) * d + h * HD + c]);
        }
        L = lse[static_cast<int64_t>(bh) * seq + t];
        Dt = dsum[static_cast<int64_t>(bh) * seq + t];
    }
#pragma unroll
    for (int c = 0; c < HD; ++c) dq[c] = 0.f;
    const int jmax = min(seq - 1, blockIdx.y * kTile + kTile - 1);
    for (int j0 = 0; j0 <= jmax; j0 += kTile) {
        __syncthreads();
        for (int i = threadIdx.x; i < kTile * HD; i += kTile) {
            const int r = i / HD, c = i % HD;
            const int j = j0 + r;
            Ks[r][c] = j < seq ? to_f(qkv[base + j * ld + kc + c]) : 0.f;
            Vs[r][c] = j < seq ? to_f(qkv[base + j * ld + vc + c]) : 0.f;
        }
        __syncthreads();
        if (t < seq) {
            const int jend = min(kTile, t - j0 + 1);
            for (int jj = 0; jj < jend; ++jj) {
                float s = 0.f, dp = 0.f;
#pragma unroll
                for (int c = 0; c < HD; ++c) {
                    s = fmaf(q[c], Ks[jj][c], s);
                    dp = fmaf(dO[c], Vs[jj][c], dp);
                }
                const float p = expf(s * scale - L);
                const float ds = p * (dp - Dt);
#pragma unroll
                for (int c = 0; c < HD; ++c) dq[c] = fmaf(ds, Ks[jj][c], dq[c]);
            }
        }
    }
    if (t < seq) {
        T* o = dqkv + (static_cast<int64_t>(b) * seq + t) * ld + h * HD;
#pragma unroll
        for (int c = 0; c < HD; ++c) o[c] = from_f<T>(dq[c] * scale);
    }
}

// dK/dV: one block per (batch * KV head, key tile); the query heads of the
// group (H / Hkv of them) are folded in ascending order (GQA), each over the
// query rows at and after the key.
template <class T, int HD>
__global__ void __launch_bounds__(kTile) attn_dkv_kernel(const T* __restrict__ qkv, const float* __restrict__ lse,
                                                         const float* __restrict__ dsum, const T* __restrict__ dy,
                                                         T* __restrict__ dqkv, int seq, int H, int Hkv, float scale) {
    ACCO_PDL_PROLOGUE();
    extern __shared__ float sm[];
    float(*Ko)[HD + 1] = reinterpret_cast<float(*)[HD + 1]>(sm);
    float(*Vo)[HD + 1] = reinterpret_cast<float(*)[HD + 1]>(sm + 1 * kTile * (HD + 1));
    float(*Qs)[HD + 1] = reinterpret_cast<float(*)[HD + 1]>(sm + 2 * kTile * (HD + 1));
    float(*dOs)[HD + 1] = reinterpret_cast<float(*)[HD + 1]>(sm + 3 * kTile * (HD + 1));
    float* Ls = sm + 4 * kTile * (HD + 1);
    float* Ds = Ls + kTile;
    const int bk = blockIdx.x, b = bk / Hkv, hk = bk % Hkv;
    const int G = H / Hkv;
    const int d = H * HD;
    const int64_t ld = static_cast<int64_t>(H + 2 * Hkv) * HD;
    const int kc = d + hk * HD, vc = kc + Hkv * HD;
    const int j0b = blockIdx.y * kTile;
    const int j = j0b + threadIdx.x;
    const int64_t base = static_cast<int64_t>(b) * seq * ld;
    for (int i = threadIdx.x; i < kTile * HD; i += kTile) {
        const int r = i / HD, c = i % HD;
        const int jj = j0b + r;
        Ko[r][c] = jj < seq ? to_f(qkv[base + jj * ld + kc + c]) : 0.f;
        Vo[r][c] = jj < seq ? to_f(qkv[base + jj * ld + vc + c]) : 0.f;
    }
    float dk[HD], dv[HD];
#pragma unroll
    for (int c = 0; c < HD; ++c) dk[c] = dv[c] = 0.f;
    for (int g = 0; g < G; ++g) {
        const int h = hk * G + g;
        const int64_t bh = static_cast<int64_t>(b) * H + h;
        for (int i0 = j0b; i0 < seq; i0 += kTile) {
            __syncthreads();
            for (int i = threadIdx.x; i < kTile * HD; i += kTile) {
                const int r = i / HD, c = i % HD;
                const int ii = i0 + r;
                Qs[r][c] = ii < seq ? to_f(qkv[base + ii * ld + h * HD + c]) : 0.f;
                dOs[r][c] = ii < seq ? to_f(dy[(static_cast<int64_t>(b) * seq + ii) * d + h * HD + c]) : 0.f;
            }
            if (threadIdx.x < kTile) {
                const int ii = i0 + threadIdx.x;
                Ls[threadIdx.x] = ii < seq ? lse[bh * seq + ii] : 0.f;
                Ds[threadIdx.x] = ii < seq ? dsum[bh * seq + ii] : 0.f;
            }
            __syncthreads();
            if (j < seq) {
                const int istart = max(0, j - i0);
                const int iend = min(kTile, seq - i0);
                for (int r = istart; r < iend; ++r) {
                    float s = 0.f, dp = 0.f;
#pragma unroll
                    for (int c = 0; c < HD; ++c) {
                        s = fmaf(Qs[r][c], Ko[threadIdx.x][c], s);
                        dp = fmaf(dOs[r][c], Vo[threadIdx.x][c], dp);
                    }
                    const float p = expf(s * scale - Ls[r]);
                    const float ds = p * (dp - Ds[r]);
#pragma unroll
                    for (int c = 0; c < HD; ++c) {
                        dv[c] = fmaf(p, dOs[r][c], dv[c]);
                        dk[c] = fmaf(ds, Qs[r][c], dk[c]);
                    }
                }
            }
        }
    }
    if (j < seq) {
        T* o = dqkv + (static_cast<int64_t>(b) * seq + j) * ld;
#pragma unroll
        for (int c = 0; c < HD; ++c) {
            o[kc + c] = from_f<T>(dk[c] * scale);
            o[vc + c] = from_f<T>(dv[c]);
        }
    }
}

template <class T, int HD>
void fwd_impl(const T* qkv, T* y, float* lse, int B, int seq, int H, int Hkv, cudaStream_t s) {
    const int smem = 2 * kTile * (HD + 1) * 4;
    static bool cfg = false;
    if (!cfg) {
        ACCO_CUDA(cudaFuncSetAttribute(attn_fwd_kernel<T, HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        cfg = true;
    }
    launch_pdl(attn_fwd_kernel<T, HD>, dim3(B * H, ceil_div(seq, kTile)), kTile, smem, s,
        qkv, y, lse, seq, H, Hkv, 1.0f / sqrtf(static_cast<float>(HD)));
    ACCO_CHECK_LAUNCH();
}

template <class T, int HD>
void bwd_impl(const T* qkv, const T* y, const float* lse, const T* dy, T* dqkv, float* dsum, int B, int seq, int H,
              int Hkv, cudaStream_t s) {
    const float scale = 1.0f / sqrtf(static_cast<float>(HD));
    const int64_t rows = static_cast<int64_t>(B) * H * seq;
    launch_pdl(attn_dsum_kernel<T, HD>, static_cast<int>((rows + 255) / 256), 256, 0, s, y, dy, dsum, B, seq, H);
    ACCO_CHECK_LAUNCH();
    const int smem_q = 2 * kTile * (HD + 1) * 4;
    const int smem_kv = (4 * kTile * (HD + 1) + 2 * kTile) * 4;
    static bool cfg = false;
    if (!cfg) {
        ACCO_CUDA(cudaFuncSetAttribute(attn_dq_kernel<T, HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_q));
        ACCO_CUDA(cudaFuncSetAttribute(attn_dkv_kernel<T, HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kv));
        cfg = true;
    }
    launch_pdl(attn_dq_kernel<T, HD>, dim3(B * H, ceil_div(seq, kTile)), kTile, smem_q, s, qkv, lse, dsum, dy, dqkv, seq, H,
                                                                                  Hkv, scale);
    ACCO_CHECK_LAUNCH();
    launch_pdl(attn_dkv_kernel<T, HD>, dim3(B * Hkv, ceil_div(seq, kTile)), kTile, smem_kv, s, qkv, lse, dsum, dy, dqkv, seq,
                                                                                     H, Hkv, scale);
    ACCO_CHECK_LAUNCH();
}

}  // namespace

// Tensor-core paths for bf16: tcgen05 (attn_tc.cu), then mma.sync
// (attn_mma.cu); each returns false if not applicable.
bool attention_fwd_tc(const __nv_bfloat16* qkv, __nv_bfloat16* y, float* lse, int B, int seq, int H, int Hkv,
                      int hd, cudaStream_t s);
bool attention_fwd_mma(const __nv_bfloat16* qkv, __nv_bfloat16* y, float* lse, int B, int seq, int H, int hd,
                       cudaStream_t s);
bool attention_bwd_tc(const __nv_bfloat16* qkv, const __nv_bfloat16* y, const float* lse, const __nv_bfloat16* dy,
                      __nv_bfloat16* dqkv, float* dsum, int B, int seq, int H, int Hkv, int hd, cudaStream_t s);
bool attention_bwd_mma(const __nv_bfloat16* qkv, const __nv_bfloat16* y, const float* lse,
                       const __nv_bfloat16* dy, __nv_bfloat16* dqkv, float* dsum, int B, int seq, int H, int hd,
                       cudaStream_t s);

// algorithmic causal-attention flops: QK^T and PV over the lower triangle
static double attn_flops(int B, int seq, int H, int hd) {
    return 2.0 * 2.0 * B * H * (static_cast<double>(seq) * (seq + 1) / 2) * hd;
}

template <class T>
void attention_fwd(const T* qkv, T* y, float* lse, int B, int seq, int H, int Hkv, int hd, cudaStream_t s) {
    ProfScope prof(kProfAttn, attn_flops(B, seq, H, hd), s);
    ACCO_REQUIRE(Hkv >= 1 && H % Hkv == 0, "attention: n_head must be a multiple of n_kv_head");
    if constexpr (sizeof(T) == 2) {
        if (attention_fwd_tc(qkv, y, lse, B, seq, H, Hkv, hd, s)) return;
        if (Hkv == H && attention_fwd_mma(qkv, y, lse, B, seq, H, hd, s)) return;
    }
    if (hd == 32) fwd_impl<T, 32>(qkv, y, lse, B, seq, H, Hkv, s);
    else if (hd == 64) fwd_impl<T, 64>(qkv, y, lse, B, seq, H, Hkv, s);
    else if (hd == 128) fwd_impl<T, 128>(qkv, y, lse, B, seq, H, Hkv, s);
    else if (hd == 16) fwd_impl<T, 16>(qkv, y, lse, B, seq, H, Hkv, s);
    else if (hd == 8) fwd_impl<T, 8>(qkv, y, lse, B, seq, H, Hkv, s);
    else throw Error(kInvalidArg, "attention: head size must be 8, 16, 32, 64 or 128");
}

template <class T>
void attention_bwd(const T* qkv, const T* y, const float* lse, const T* dy, T* dqkv, float* dsum, int B, int seq,
                   int H, int Hkv, int hd, cudaStream_t s) {
    ProfScope prof(kProfAttn, 2.5 * attn_flops(B, seq, H, hd), s);
    ACCO_REQUIRE(Hkv >= 1 && H % Hkv == 0, "attention: n_head must be a multiple of n_kv_head");
    if constexpr (sizeof(T) == 2) {
        if (attention_bwd_tc(qkv, y, lse, dy, dqkv, dsum, B, seq, H, Hkv, hd, s)) return;
        if (Hkv == H && attention_bwd_mma(qkv, y, lse, dy, dqkv, dsum, B, seq, H, hd, s)) return;
    }
    if (hd == 32) bwd_impl<T, 32>(qkv, y, lse, dy, dqkv, dsum, B, seq, H, Hkv, s);
    else if (hd == 64) bwd_impl<T, 64>(qkv, y, lse, dy, dqkv, dsum, B, seq, H, Hkv, s);
    else if (hd == 128) bwd_impl<T, 128>(qkv, y, lse, dy, dqkv, dsum, B, seq, H, Hkv, s);
    else if (hd == 16) bwd_impl<T, 16>(qkv, y, lse, dy, dqkv, dsum, B, seq, H, Hkv, s);
    else if (hd == 8) bwd_impl<T, 8>(qkv, y, lse, dy, dqkv, dsum, B, seq, H, Hkv, s);
    else throw Error(kInvalidArg, "attention: head size must be 8, 16, 32, 64 or 128");
}

template void attention_fwd<float>(const float*, float*, float*, int, int, int, int, int, cudaStream_t);
template void attention_fwd<__nv_bfloat16>(const __nv_bfloat16*, __nv_bfloat16*, float*, int, int, int, int, int,
                                           cudaStream_t);
template void attention_bwd<float>(const float*, const float*, const float*, const float*, float*, float*, int,
                                   int, int, int, int, cudaStream_t);
template void attention_bwd<__nv_bfloat16>(const __nv_bfloat16*, const __nv_bfloat16*, const float*,
                                           const __nv_bfloat16*, __nv_bfloat16*, float*, int, int, int, int, int,
                                           cudaStream_t);

}  // namespace acco
