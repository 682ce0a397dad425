// LM element-wise / normalisation / loss kernels and engine utilities.
// See lm_kernels.h. The LM definition is oracle/gpt_oracle.py's.
#include "epilogue.cuh"
#include "host_util.h"
#include "lm_kernels.h"

#include <algorithm>
#include <cstdlib>
#include <vector>

namespace acco {
namespace {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// ----------------------------------------------------------------- tokens
__global__ void gather_tokens_kernel(const int32_t* __restrict__ data, int seq, int n_samples,
                                     uint64_t seed, int mode, int start, int32_t* tok_in,
                                     int32_t* tok_out, int32_t* idx_out) {
    ACCO_PDL_PROLOGUE();
    const int b = blockIdx.x;
    int idx;
    if (mode == 0)
        idx = static_cast<int>(stream_draw(seed, static_cast<uint64_t>(b)) % static_cast<uint64_t>(n_samples));
    else
        idx = start + b;
    if (threadIdx.x == 0 && idx_out) idx_out[b] = idx;
    const int32_t* row = data + static_cast<int64_t>(idx) * (seq + 1);
    for (int t = threadIdx.x; t < seq; t += blockDim.x) {
        tok_in[b * seq + t] = row[t];
        tok_out[b * seq + t] = row[t + 1];
    }
}

// bf16 x 8 <-> fp32 (16 B vectors)
__device__ __forceinline__ void unpack8b(const uint4& u, float* v) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        v[2 * k] = __uint_as_float(w[k] << 16);
        v[2 * k + 1] = __uint_as_float(w[k] & 0xffff0000u);
    }
}
__device__ __forceinline__ uint4 pack8b(const float* v) {
    uint32_t w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * k], v[2 * k + 1]);
        w[k] = *reinterpret_cast<uint32_t*>(&h);
    }
    return make_uint4(w[0], w[1], w[2], w[3]);
}

// ----------------------------------------------------------------- embedding
template <class T>
__global__ void embed_fwd_kernel(const int32_t* __restrict__ tok, const T* __restrict__ wte,
                                 const T* __restrict__ wpe, T* __restrict__ x, int seq, int d) {
    ACCO_PDL_PROLOGUE();
    const int m = blockIdx.x;
    const int t = m % seq;
    const T* e = wte + static_cast<int64_t>(tok[m]) * d;
    T* o = x + static_cast<int64_t>(m) * d;
    if (wpe == nullptr) {  // Llama: no learned positions (RoPE in attention)
        for (int c = threadIdx.x; c < d; c += blockDim.x) o[c] = e[c];
        return;
    }
    const T* p = wpe + static_cast<int64_t>(t) * d;
    if constexpr (sizeof(T) == 2) {
        if ((d & 7) == 0) {  // 16 B per thread (the same per-element rounding)
            for (int c = threadIdx.x; c < d / 8; c += blockDim.x) {
                float ev[8], pv[8], r[8];
                unpack8b(reinterpret_cast<const uint4*>(e)[c], ev);
                unpack8b(reinterpret_cast<const uint4*>(p)[c], pv);
#pragma unroll
                for (int k = 0; k < 8; ++k) r[k] = ev[k] + pv[k];
                reinterpret_cast<uint4*>(o)[c] = pack8b(r);
            }
            return;
        }
    }
    for (int c = threadIdx.x; c < d; c += blockDim.x) o[c] = from_f<T>(to_f(e[c]) + to_f(p[c]));
}

// ----------------------------------------------------------------- layernorm
constexpr float kLnEps = 1e-5f;

// RMS = true: RMSNorm (Llama): mean fixed at 0 (stored as 0, so the LN
// parameter-gradient kernels compute xhat = x * rstd unchanged), no bias.
template <class T, bool RMS>
__global__ void ln_fwd_kernel(const T* __restrict__ x, const T* __restrict__ g, const T* __restrict__ b,
                              T* __restrict__ y, float* __restrict__ mean, float* __restrict__ rstd,
                              int M, int d) {
    ACCO_PDL_PROLOGUE();
    const int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (row >= M) return;
    const T* xr = x + static_cast<int64_t>(row) * d;
    float s = 0.f;
    if (!RMS)
        for (int c = lane; c < d; c += 32) s += to_f(xr[c]);
    const float mu = RMS ? 0.f : warp_sum(s) / d;
    float v = 0.f;
    for (int c = lane; c < d; c += 32) {
        float t = to_f(xr[c]) - mu;
        v += t * t;
    }
    const float rs = rsqrtf(warp_sum(v) / d + kLnEps);
    T* yr = y + static_cast<int64_t>(row) * d;
    for (int c = lane; c < d; c += 32)
        yr[c] = from_f<T>((to_f(xr[c]) - mu) * rs * to_f(g[c]) + (RMS ? 0.f : to_f(b[c])));
    if (lane == 0) {
        mean[row] = mu;
        rstd[row] = rs;
    }
}

template <class T, bool RMS>
__global__ void ln_bwd_kernel(const T* __restrict__ dy, const T* __restrict__ x, const T* __restrict__ g,
                              const float* __restrict__ mean, const float* __restrict__ rstd,
                              T* __restrict__ dx, int accumulate, int M, int d) {
    ACCO_PDL_PROLOGUE();
    const int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (row >= M) return;
    const int64_t o = static_cast<int64_t>(row) * d;
    const float mu = mean[row], rs = rstd[row];
    float s1 = 0.f, s2 = 0.f;
    for (int c = lane; c < d; c += 32) {
        float xh = (to_f(x[o + c]) - mu) * rs;
        float dxh = to_f(dy[o + c]) * to_f(g[c]);
        s1 += dxh;
        s2 += dxh * xh;
    }
    s1 = RMS ? 0.f : warp_sum(s1) / d;
    s2 = warp_sum(s2) / d;
    for (int c = lane; c < d; c += 32) {
        float xh = (to_f(x[o + c]) - mu) * rs;
        float dxh = to_f(dy[o + c]) * to_f(g[c]);
        float v = rs * (dxh - s1 - xh * s2);
        if (accumulate) v += to_f(dx[o + c]);
        dx[o + c] = from_f<T>(v);
    }
}

// bf16 LayerNorm with 16B vector loads, row held in registers: lane owns
// chunks c = lane + 32*i (8 elements each), d = 256 * CH (unpack8b / pack8b above).
template <int CH, bool RMS>
__global__ void ln_fwd_vec(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ g,
                           const __nv_bfloat16* __restrict__ b, __nv_bfloat16* __restrict__ y, float* __restrict__ mean,
                           float* __restrict__ rstd, int M) {
    ACCO_PDL_PROLOGUE();
    constexpr int d = 256 * CH;
    const int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (row >= M) return;
    const uint4* xr = reinterpret_cast<const uint4*>(x + static_cast<int64_t>(row) * d);
    // every load of the row (x, gamma, beta) is issued before the reductions,
    // so their latencies overlap instead of adding up
    uint4 xv[CH], gw[CH], bw[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) {
        xv[i] = xr[lane + 32 * i];
        gw[i] = reinterpret_cast<const uint4*>(g)[lane + 32 * i];
        if (!RMS) bw[i] = reinterpret_cast<const uint4*>(b)[lane + 32 * i];
    }
    float v[CH * 8];
#pragma unroll
    for (int i = 0; i < CH; ++i) unpack8b(xv[i], v + 8 * i);
    float s = 0.f;
    if (!RMS) {
#pragma unroll
        for (int i = 0; i < CH * 8; ++i) s += v[i];
    }
    const float mu = RMS ? 0.f : warp_sum(s) / d;
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < CH * 8; ++i) q += (v[i] - mu) * (v[i] - mu);
    const float rs = rsqrtf(warp_sum(q) / d + kLnEps);
    uint4* yr = reinterpret_cast<uint4*>(y + static_cast<int64_t>(row) * d);
#pragma unroll
    for (int i = 0; i < CH; ++i) {
        float gv[8], bv[8] = {0, 0, 0, 0, 0, 0, 0, 0}, o[8];
        unpack8b(gw[i], gv);
        if (!RMS) unpack8b(bw[i], bv);
#pragma unroll
        for (int k = 0; k < 8; ++k) o[k] = (v[8 * i + k] - mu) * rs * gv[k] + bv[k];
        yr[lane + 32 * i] = pack8b(o);
    }
    if (lane == 0) {
        mean[row] = mu;
        rstd[row] = rs;
    }
}

// Per-element norm-backward math with explicit roundings (no FMA contraction
// left to the compiler), shared by ln_bwd_vec and ln_bwd_vec_p so their dx are
// bitwise equal: xhat = (x - mu) rs, dxh = dy g; s1 += dxh, s2 += dxh xhat;
// dx = rs (dxh - s1 - xhat s2).
__device__ __forceinline__ float ln_xhat(float x, float mu, float rs) { return __fmul_rn(__fsub_rn(x, mu), rs); }
__device__ __forceinline__ float ln_dx(float dxh, float xh, float s1, float s2, float rs) {
    return __fmul_rn(rs, __fsub_rn(__fsub_rn(dxh, s1), __fmul_rn(xh, s2)));
}

template <int CH, bool RMS>
__global__ void ln_bwd_vec(const __nv_bfloat16* __restrict__ dy, const __nv_bfloat16* __restrict__ x,
                           const __nv_bfloat16* __restrict__ g, const float* __restrict__ mean,
                           const float* __restrict__ rstd, __nv_bfloat16* __restrict__ dx, int accumulate, int M) {
    ACCO_PDL_PROLOGUE();
    constexpr int d = 256 * CH;
    const int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (row >= M) return;
    const int64_t o = static_cast<int64_t>(row) * d;
    const uint4* dyr = reinterpret_cast<const uint4*>(dy + o);
    const uint4* xr = reinterpret_cast<const uint4*>(x + o);
    const float mu = mean[row], rs = rstd[row];
    uint4* dxr = reinterpret_cast<uint4*>(dx + o);
    // the accumulated dx is loaded with the inputs (not after the reductions)
    uint4 pv[CH];
    if (accumulate) {
#pragma unroll
        for (int i = 0; i < CH; ++i) pv[i] = dxr[lane + 32 * i];
    }
    float xh[CH * 8], dxh[CH * 8];
#pragma unroll
    for (int i = 0; i < CH; ++i) {
        float dv[8], gv[8];
        unpack8b(xr[lane + 32 * i], xh + 8 * i);
        unpack8b(dyr[lane + 32 * i], dv);
        unpack8b(reinterpret_cast<const uint4*>(g)[lane + 32 * i], gv);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            xh[8 * i + k] = ln_xhat(xh[8 * i + k], mu, rs);
            dxh[8 * i + k] = __fmul_rn(dv[k], gv[k]);
        }
    }
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < CH * 8; ++i) {
        s1 = __fadd_rn(s1, dxh[i]);
        s2 = __fadd_rn(s2, __fmul_rn(dxh[i], xh[i]));
    }
    s1 = RMS ? 0.f : warp_sum(s1) / d;
    s2 = warp_sum(s2) / d;
#pragma unroll
    for (int i = 0; i < CH; ++i) {
        float r[8], prev[8];
        if (accumulate) unpack8b(pv[i], prev);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            r[k] = ln_dx(dxh[8 * i + k], xh[8 * i + k], s1, s2, rs);
            if (accumulate) r[k] = __fadd_rn(r[k], prev[k]);
        }
        dxr[lane + 32 * i] = pack8b(r);
    }
}

// Wide rows (d >= 1024): one block of d/8 threads per row, 8 elements (16 B)
// per thread, block reductions through smem — instead of one warp holding 64
// elements per lane (register-bound, latency-exposed at d = 2048).
template <int NT, bool RMS>
__global__ void __launch_bounds__(NT) ln_bwd_wide(const __nv_bfloat16* __restrict__ dy,
                                                  const __nv_bfloat16* __restrict__ x,
                                                  const __nv_bfloat16* __restrict__ g, const float* __restrict__ mean,
                                                  const float* __restrict__ rstd, __nv_bfloat16* __restrict__ dx,
                                                  int accumulate) {
    ACCO_PDL_PROLOGUE();
    constexpr int d = NT * 8, NW = NT / 32;
    __shared__ float red[2][NW];
    const int row = blockIdx.x, t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int64_t o = static_cast<int64_t>(row) * d;
    const float mu = mean[row], rs = rstd[row];
    float xh[8], dxh[8], gv[8], dv[8];
    unpack8b(reinterpret_cast<const uint4*>(x + o)[t], xh);
    unpack8b(reinterpret_cast<const uint4*>(dy + o)[t], dv);
    unpack8b(reinterpret_cast<const uint4*>(g)[t], gv);
    float prev[8];
    if (accumulate) unpack8b(reinterpret_cast<const uint4*>(dx + o)[t], prev);
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        xh[k] = (xh[k] - mu) * rs;
        dxh[k] = dv[k] * gv[k];
        s1 += dxh[k];
        s2 += dxh[k] * xh[k];
    }
    s1 = warp_sum(s1);
    s2 = warp_sum(s2);
    if (lane == 0) {
        red[0][w] = s1;
        red[1][w] = s2;
    }
    __syncthreads();
    float t1 = 0.f, t2 = 0.f;
#pragma unroll
    for (int i = 0; i < NW; ++i) {  // fixed order: deterministic
        t1 += red[0][i];
        t2 += red[1][i];
    }
    t1 = RMS ? 0.f : t1 / d;
    t2 /= d;
    float r[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        r[k] = rs * (dxh[k] - t1 - xh[k] * t2);
        if (accumulate) r[k] += prev[k];
    }
    reinterpret_cast<uint4*>(dx + o)[t] = pack8b(r);
}

// ------------------------- norm backward with fused parameter-gradient partials
// Persistent forms of ln_bwd_vec / ln_bwd_wide (the same per-row arithmetic,
// so dx is bitwise unchanged): block b takes rows b, b + G, ... (fixed) and
// also accumulates, per column, dgamma = sum dy * xhat and dbeta = sum dy over
// its rows in registers; at the end the block's partial sums go to
// part[b][q][d] (q = 0 dgamma, 1 dbeta). One ln_param_fold per micro-batch
// then sums every norm's G partials in block order into the gradient
// accumulator: the parameter reductions no longer re-read dy and x on a side
// stream (two launches and 2 x M x d x 2 bytes per norm before).
// Bulk async copies (TMA, non-tensor) of whole rows into shared memory,
// completing on a per-warp mbarrier
__device__ __forceinline__ void lnb_mbar_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar))));
}
__device__ __forceinline__ void lnb_expect(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(bar))),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void lnb_copy(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
        "l"(src), "r"(bytes), "r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar)))
        : "memory");
}
__device__ __forceinline__ void lnb_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(bar));
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                     : "=r"(ok)
                     : "r"(a), "r"(parity)
                     : "memory");
}

// Rows are staged through shared memory by bulk async copies, two rows ahead
// per warp (x, dy and the accumulated dx: 3 x 2 d bytes per row and stage), so
// the HBM latency of the next rows overlaps this row's math: each warp used
// to wait a full memory round trip per row. The values and their order of
// use are unchanged (dx and the partials are bitwise the same).
constexpr int kLnStages = 2;
template <int CH, bool RMS>
__global__ void __launch_bounds__(256, 2) ln_bwd_vec_p(const __nv_bfloat16* __restrict__ dy,
                                                       const __nv_bfloat16* __restrict__ x,
                                                       const __nv_bfloat16* __restrict__ g,
                                                       const float* __restrict__ mean, const float* __restrict__ rstd,
                                                       __nv_bfloat16* __restrict__ dx, int accumulate, int M,
                                                       float* __restrict__ part) {
    constexpr int d = 256 * CH;
    constexpr uint32_t kRow = d * 2;  // bytes per bf16 row
    // [8 warps][kLnStages][x | dy | dx rows]; reused as [8 warps][d] fp32 for the block reduction
    extern __shared__ __align__(128) uint8_t lnsm[];
    __shared__ uint64_t bars[8][kLnStages];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t* stage0 = lnsm + w * kLnStages * 3 * kRow;
    if (lane == 0) {
        for (int q = 0; q < kLnStages; ++q) lnb_mbar_init(&bars[w][q]);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    ACCO_PDL_PROLOGUE();
    const int step = gridDim.x * 8;
    const int row0 = blockIdx.x * 8 + w;
    auto issue = [&](int row, int q) {  // lane 0: the row's x, dy (and dx) into stage q
        const int64_t o = static_cast<int64_t>(row) * d;
        uint8_t* st = stage0 + q * 3 * kRow;
        lnb_expect(&bars[w][q], (accumulate ? 3 : 2) * kRow);
        lnb_copy(st, x + o, kRow, &bars[w][q]);
        lnb_copy(st + kRow, dy + o, kRow, &bars[w][q]);
        if (accumulate) lnb_copy(st + 2 * kRow, dx + o, kRow, &bars[w][q]);
    };
    if (lane == 0)
        for (int q = 0; q < kLnStages; ++q)
            if (row0 + q * step < M) issue(row0 + q * step, q);
    // (registers: the per-lane parameter sums stay resident, the row's values
    // are unpacked per 8-column chunk in each of the two passes, so two blocks
    // of 8 warps fit an SM)
    float ag[CH * 8], ab[CH * 8];
#pragma unroll
    for (int i = 0; i < CH * 8; ++i) ag[i] = ab[i] = 0.f;
    const uint4* gq = reinterpret_cast<const uint4*>(g);
    float mu = 0.f, rs = 0.f;
    if (row0 < M) {
        mu = mean[row0];
        rs = rstd[row0];
    }
    int k = 0;
    for (int row = row0; row < M; row += step, ++k) {
        const int64_t o = static_cast<int64_t>(row) * d;
        uint4* dxr = reinterpret_cast<uint4*>(dx + o);
        const int q = k % kLnStages;
        lnb_wait(&bars[w][q], (k / kLnStages) & 1);
        const uint4* st = reinterpret_cast<const uint4*>(stage0 + q * 3 * kRow);
        uint4 xv[CH], dvv[CH], pv[CH];
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            xv[i] = st[lane + 32 * i];
            dvv[i] = st[d / 8 + lane + 32 * i];
            if (accumulate) pv[i] = st[d / 4 + lane + 32 * i];
        }
        __syncwarp();  // every lane has the stage in registers: refill it
        if (lane == 0 && row + kLnStages * step < M) issue(row + kLnStages * step, q);
        const float cmu = mu, crs = rs;
        if (row + step < M) {  // the next row's statistics, under this row's math
            mu = mean[row + step];
            rs = rstd[row + step];
        }
        float s1 = 0.f, s2 = 0.f;
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            float xh[8], dv[8], gv[8];
            unpack8b(xv[i], xh);
            unpack8b(dvv[i], dv);
            unpack8b(gq[lane + 32 * i], gv);
#pragma unroll
            for (int k2 = 0; k2 < 8; ++k2) {
                xh[k2] = ln_xhat(xh[k2], cmu, crs);
                const float dxh = __fmul_rn(dv[k2], gv[k2]);
                s1 = __fadd_rn(s1, dxh);
                s2 = __fadd_rn(s2, __fmul_rn(dxh, xh[k2]));
                ag[8 * i + k2] += dv[k2] * xh[k2];
                if (!RMS) ab[8 * i + k2] += dv[k2];
            }
        }
        s1 = RMS ? 0.f : warp_sum(s1) / d;
        s2 = warp_sum(s2) / d;
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            float xh[8], dv[8], gv[8], r[8], prev[8];
            unpack8b(xv[i], xh);
            unpack8b(dvv[i], dv);
            unpack8b(gq[lane + 32 * i], gv);
            if (accumulate) unpack8b(pv[i], prev);
#pragma unroll
            for (int k2 = 0; k2 < 8; ++k2) {
                r[k2] = ln_dx(__fmul_rn(dv[k2], gv[k2]), ln_xhat(xh[k2], cmu, crs), s1, s2, crs);
                if (accumulate) r[k2] = __fadd_rn(r[k2], prev[k2]);
            }
            dxr[lane + 32 * i] = pack8b(r);
        }
    }
    // block partials: the 8 warps' column sums in warp order (the staging
    // buffers are free: every copy issued was waited for)
    __syncthreads();
    float* red = reinterpret_cast<float*>(lnsm);
#pragma unroll
    for (int q = 0; q < (RMS ? 1 : 2); ++q) {
#pragma unroll
        for (int i = 0; i < CH; ++i)
#pragma unroll
            for (int k2 = 0; k2 < 8; ++k2) red[w * d + 8 * (lane + 32 * i) + k2] = q ? ab[8 * i + k2] : ag[8 * i + k2];
        __syncthreads();
        for (int c = threadIdx.x; c < d; c += 256) {
            float t = 0.f;
#pragma unroll
            for (int j = 0; j < 8; ++j) t += red[j * d + c];
            part[(static_cast<int64_t>(blockIdx.x) * 2 + q) * d + c] = t;
        }
        __syncthreads();
    }
}

// Every norm of the micro-batch: grad[g_off + c] (+)= sum_b part[b][0][c] and
// grad[b_off + c] (+)= sum_b part[b][1][c] (b_off < 0: RMSNorm), blocks summed
// in kFoldSub fixed interleaved sub-sums (b = sub mod kFoldSub) then a fixed
// pairwise tree — deterministic. 32 columns x 8 sub-sums per block: each
// thread has ~G / 8 dependent-free loads in flight (it was 64 x 4, G / 4
// loads per thread and a latency-bound 23 us per micro-batch).
constexpr int kFoldCols = 32, kFoldSub = 8;
__global__ void __launch_bounds__(256) ln_param_fold_kernel(const LnFold* __restrict__ table, const float* __restrict__ parts,
                                                            float* __restrict__ grad, int G, int acc) {
    ACCO_PDL_PROLOGUE();
    __shared__ float sub_sum[kFoldSub][kFoldCols];
    const LnFold e = table[blockIdx.y];
    const int nq = e.b_off >= 0 ? 2 : 1;
    const int cc = threadIdx.x % kFoldCols, sub = threadIdx.x / kFoldCols;
    const int col = blockIdx.x * kFoldCols + cc;
    const bool live = col < nq * e.d;
    const int q = live ? col / e.d : 0, c = live ? col % e.d : 0;
    float t = 0.f;
    if (live) {
        const float* p = parts + e.part_off + static_cast<int64_t>(q) * e.d + c;
#pragma unroll 8
        for (int b = sub; b < G; b += kFoldSub) t += __ldcs(p + static_cast<int64_t>(b) * 2 * e.d);
    }
    sub_sum[sub][cc] = t;
    __syncthreads();
    if (sub == 0 && live) {
        const float r = ((sub_sum[0][cc] + sub_sum[1][cc]) + (sub_sum[2][cc] + sub_sum[3][cc])) +
                        ((sub_sum[4][cc] + sub_sum[5][cc]) + (sub_sum[6][cc] + sub_sum[7][cc]));
        float* o = grad + (q ? e.b_off : e.g_off) + c;
        *o = (acc ? *o : 0.f) + r;
    }
}

// ------------------------------------------------ deterministic column reduce
// partial[chunk][col] = sum over rows of the chunk (fixed order), then
// out[col] += sum_chunk partial[chunk][col] (fixed order).
constexpr int kColRows = 8;  // row lanes per block
constexpr int kColChunk = 256;

// F(row, col) -> float (two outputs for LN: dy*xhat and dy)
template <class T, int KIND>
__global__ void colreduce_partial(const T* __restrict__ y, int64_t ld, const T* __restrict__ x,
                                  const float* __restrict__ mean, const float* __restrict__ rstd,
                                  int M, int N, float* __restrict__ part0, float* __restrict__ part1) {
    ACCO_PDL_PROLOGUE();
    __shared__ float s0[kColRows][33], s1[kColRows][33];
    const int col = blockIdx.x * 32 + threadIdx.x;
    const int chunk = blockIdx.y;
    const int r0 = chunk * kColChunk;
    const int r1 = min(M, r0 + kColChunk);
    float a0 = 0.f, a1 = 0.f;
    if (col < N) {
        for (int r = r0 + threadIdx.y; r < r1; r += kColRows) {
            float dy = to_f(y[static_cast<int64_t>(r) * ld + col]);
            if (KIND == 0) {
                a0 += dy;
            } else {
                float xh = (to_f(x[static_cast<int64_t>(r) * N + col]) - mean[r]) * rstd[r];
                a0 += dy * xh;
                if (KIND == 1) a1 += dy;
            }
        }
    }
    s0[threadIdx.y][threadIdx.x] = a0;
    s1[threadIdx.y][threadIdx.x] = a1;
    __syncthreads();
    if (threadIdx.y == 0 && col < N) {
        float t0 = 0.f, t1 = 0.f;
#pragma unroll
        for (int i = 0; i < kColRows; ++i) {
            t0 += s0[i][threadIdx.x];
            t1 += s1[i][threadIdx.x];
        }
        part0[static_cast<int64_t>(chunk) * N + col] = t0;
        if (KIND == 1) part1[static_cast<int64_t>(chunk) * N + col] = t1;
    }
}

// Vectorised column reduction: a block owns a 64-column slab x one row chunk;
// threads = 8 column groups (8 contiguous columns, 16B bf16 loads) x 32 row
// lanes. Partial sums per chunk go to `part`; the last block of a slab (atomic
// ticket) folds the chunks in ascending order and adds into out (+ out1) —
// deterministic, one launch. KIND 0: sum y; KIND 1 (LayerNorm params):
// out += sum dy*xhat, out1 += sum dy; KIND 2 (RMSNorm weight): out += sum dy*xhat.
constexpr int kVecRows = 32;

template <class T>
__device__ __forceinline__ void load8(const T* p, float* v);
template <>
__device__ __forceinline__ void load8<__nv_bfloat16>(const __nv_bfloat16* p, float* v) {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        v[2 * k] = __uint_as_float(w[k] << 16);
        v[2 * k + 1] = __uint_as_float(w[k] & 0xffff0000u);
    }
}
template <>
__device__ __forceinline__ void load8<float>(const float* p, float* v) {
    const float4 a = *reinterpret_cast<const float4*>(p);
    const float4 b = *reinterpret_cast<const float4*>(p + 4);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}

template <class T, int KIND>
__global__ void __launch_bounds__(256) colsum_vec_kernel(const T* __restrict__ y, int64_t ld, const T* __restrict__ x,
                                                         const float* __restrict__ mean, const float* __restrict__ rstd,
                                                         int M, int N, int rows_per_chunk, float* __restrict__ part,
                                                         unsigned* __restrict__ tickets, float* __restrict__ out,
                                                         float* __restrict__ out1, int acc) {
    ACCO_PDL_PROLOGUE();
    __shared__ float s0[kVecRows][65], s1[kVecRows][65];
    __shared__ bool last;
    const int cg = threadIdx.x & 7, rl = threadIdx.x >> 3;
    const int c0 = blockIdx.x * 64 + cg * 8;
    const int chunk = blockIdx.y, nchunk = gridDim.y;
    const int r0 = chunk * rows_per_chunk, r1 = min(M, r0 + rows_per_chunk);
    float a0[8] = {0, 0, 0, 0, 0, 0, 0, 0}, a1[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (c0 < N) {
#pragma unroll 4
        for (int r = r0 + rl; r < r1; r += kVecRows) {
            float dy[8];
            load8<T>(y + static_cast<int64_t>(r) * ld + c0, dy);
            if (KIND == 0) {
#pragma unroll
                for (int k = 0; k < 8; ++k) a0[k] += dy[k];
            } else {
                float xv[8];
                load8<T>(x + static_cast<int64_t>(r) * N + c0, xv);
                const float mu = mean[r], rs = rstd[r];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    a0[k] += dy[k] * ((xv[k] - mu) * rs);
                    if (KIND == 1) a1[k] += dy[k];
                }
            }
        }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        s0[rl][cg * 8 + k] = a0[k];
        s1[rl][cg * 8 + k] = a1[k];
    }
    __syncthreads();
    const int ci = threadIdx.x;  // column within slab (first 64 threads)
    const int col = blockIdx.x * 64 + ci;
    if (ci < 64 && col < N) {
        float t0 = 0.f, t1 = 0.f;
        for (int i = 0; i < kVecRows; ++i) {
            t0 += s0[i][ci];
            t1 += s1[i][ci];
        }
        part[(static_cast<int64_t>(chunk) * 2 + 0) * N + col] = t0;
        if (KIND == 1) part[(static_cast<int64_t>(chunk) * 2 + 1) * N + col] = t1;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(&tickets[blockIdx.x], 1u) == static_cast<unsigned>(nchunk - 1);
    __syncthreads();
    if (!last) return;
    __threadfence();
    // the slab's last block folds the nchunk partials: 4 threads per column,
    // each a fixed strided subset (independent loads in flight), then the four
    // sub-sums in a fixed order — deterministic
    {
        const int cc = threadIdx.x & 63, sub = threadIdx.x >> 6;
        const int colc = blockIdx.x * 64 + cc;
        float t0 = 0.f, t1 = 0.f;
        if (colc < N) {
#pragma unroll 4
            for (int c = sub; c < nchunk; c += 4) {
                t0 += __ldcg(&part[(static_cast<int64_t>(c) * 2 + 0) * N + colc]);
                if (KIND == 1) t1 += __ldcg(&part[(static_cast<int64_t>(c) * 2 + 1) * N + colc]);
            }
        }
        s0[sub][cc] = t0;
        s1[sub][cc] = t1;
        __syncthreads();
        if (sub == 0 && colc < N) {
            const float r0 = ((s0[0][cc] + s0[1][cc]) + s0[2][cc]) + s0[3][cc];
            out[colc] = (acc ? out[colc] : 0.f) + r0;
            if (KIND == 1) {
                const float r1 = ((s1[0][cc] + s1[1][cc]) + s1[2][cc]) + s1[3][cc];
                out1[colc] = (acc ? out1[colc] : 0.f) + r1;
            }
        }
    }
    if (threadIdx.x == 0) tickets[blockIdx.x] = 0;  // ready for the next launch (stream-ordered)
}

__global__ void colreduce_final(const float* __restrict__ part, int nchunk, int N, float* __restrict__ out,
                                int acc) {
    ACCO_PDL_PROLOGUE();
    const int col = blockIdx.x * blockDim.x + threadIdx.x;
    if (col >= N) return;
    float t = 0.f;
    for (int c = 0; c < nchunk; ++c) t += part[static_cast<int64_t>(c) * N + col];
    out[col] = (acc ? out[col] : 0.f) + t;
}

// ------------------------------------------------------------- cross entropy
template <class T>
__global__ void __launch_bounds__(512) ce_kernel(T* __restrict__ logits, int64_t ld,
                                                 const int32_t* __restrict__ target, int V, float inv_seq,
                                                 float* __restrict__ row_loss) {
    ACCO_PDL_PROLOGUE();
    __shared__ float red[32];
    const int row = blockIdx.x;
    T* L = logits + static_cast<int64_t>(row) * ld;
    // pass 1: online max / sum-exp per thread
    float m = -INFINITY, s = 0.f;
    for (int c = threadIdx.x; c < V; c += blockDim.x) {
        float v = to_f(L[c]);
        if (v > m) {
            s = s * expf(m - v) + 1.f;
            m = v;
        } else {
            s += expf(v - m);
        }
    }
    // block reduce (max, then rescaled sums)
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    float wm = warp_max(m);
    if (lane == 0) red[wid] = wm;
    __syncthreads();
    float gm = -INFINITY;
    for (int i = 0; i < nw; ++i) gm = fmaxf(gm, red[i]);
    __syncthreads();
    float ls = (m == -INFINITY) ? 0.f : s * expf(m - gm);
    ls = warp_sum(ls);
    if (lane == 0) red[wid] = ls;
    __syncthreads();
    float tot = 0.f;
    for (int i = 0; i < nw; ++i) tot += red[i];
    const float lse = gm + logf(tot);
    const int tgt = target[row];
    if (threadIdx.x == 0) row_loss[row] = lse - to_f(L[tgt]);
    __syncthreads();
    // pass 2: dlogits
    for (int c = threadIdx.x; c < V; c += blockDim.x) {
        float p = expf(to_f(L[c]) - lse);
        if (c == tgt) p -= 1.f;
        L[c] = from_f<T>(p * inv_seq);
    }
}

// bf16 two-pass variant with 16B vector loads: pass 1 streams the row from HBM
// (online max / sum-exp per 8-element vector), pass 2 re-reads it while it is
// still in L2 (148 SMs x a few 100 KB rows << 126 MB) and writes dlogits, so
// HBM sees one read + one write per logit. Small blocks -> several rows per SM.
__device__ __forceinline__ void unpack8(const uint4& u, float* v) {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        v[2 * k] = __uint_as_float(w[k] << 16);
        v[2 * k + 1] = __uint_as_float(w[k] & 0xffff0000u);
    }
}

__global__ void __launch_bounds__(256) ce_vec_kernel(__nv_bfloat16* __restrict__ logits, int64_t ld,
                                                     const int32_t* __restrict__ target, int V, float inv_seq,
                                                     float* __restrict__ row_loss) {
    ACCO_PDL_PROLOGUE();
    __shared__ float red_m[8], red_s[8];
    const int row = blockIdx.x;
    uint4* L = reinterpret_cast<uint4*>(logits + static_cast<int64_t>(row) * ld);
    const int nvec = (V + 7) / 8;
    const int nfull = V / 8;  // vectors with 8 valid elements
    float m = -INFINITY, s = 0.f;
    // 4 independent 16 B loads in flight per thread (the loop was load-latency bound)
    constexpr int U = 4;
    int i0 = threadIdx.x;
    for (; i0 + (U - 1) * 256 < nfull; i0 += U * 256) {
        uint4 raw[U];
#pragma unroll
        for (int u = 0; u < U; ++u) raw[u] = L[i0 + u * 256];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            float v[8];
            unpack8(raw[u], v);
            float lm = v[0];
#pragma unroll
            for (int k = 1; k < 8; ++k) lm = fmaxf(lm, v[k]);
            if (lm > m) {
                s *= __expf(m - lm);
                m = lm;
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) s += __expf(v[k] - m);
        }
    }
    for (int i = i0; i < nvec; i += 256) {
        float v[8];
        unpack8(L[i], v);
        if (i >= nfull)
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (i * 8 + k >= V) v[k] = -INFINITY;
        float lm = v[0];
#pragma unroll
        for (int k = 1; k < 8; ++k) lm = fmaxf(lm, v[k]);
        if (lm > m) {
            s *= __expf(m - lm);
            m = lm;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) s += __expf(v[k] - m);
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    float wm = warp_max(m);
    float ws = (m == -INFINITY) ? 0.f : s * __expf(m - wm);
    ws = warp_sum(ws);
    if (lane == 0) {
        red_m[wid] = wm;
        red_s[wid] = ws;
    }
    __syncthreads();
    float gm = red_m[0];
    for (int i = 1; i < 8; ++i) gm = fmaxf(gm, red_m[i]);
    float tot = 0.f;
    for (int i = 0; i < 8; ++i) tot += red_m[i] == -INFINITY ? 0.f : red_s[i] * __expf(red_m[i] - gm);
    const float lse = gm + __logf(tot);
    const int tgt = target[row];
    // pass 2 (L2 re-read), same 4-deep batching of the loads
    int j0 = threadIdx.x;
    for (; j0 + (U - 1) * 256 < nvec; j0 += U * 256) {
        uint4 raw[U];
#pragma unroll
        for (int u = 0; u < U; ++u) raw[u] = L[j0 + u * 256];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int i = j0 + u * 256;
            float v[8];
            unpack8(raw[u], v);
            uint32_t w[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                float p0 = __expf(v[2 * k] - lse), p1 = __expf(v[2 * k + 1] - lse);
                const int e0 = i * 8 + 2 * k;
                if (e0 >= V) p0 = 0.f;
                if (e0 + 1 >= V) p1 = 0.f;
                if (e0 == tgt) {
                    row_loss[row] = lse - v[2 * k];
                    p0 -= 1.f;
                }
                if (e0 + 1 == tgt) {
                    row_loss[row] = lse - v[2 * k + 1];
                    p1 -= 1.f;
                }
                __nv_bfloat162 h = __floats2bfloat162_rn(p0 * inv_seq, p1 * inv_seq);
                w[k] = *reinterpret_cast<uint32_t*>(&h);
            }
            L[i] = make_uint4(w[0], w[1], w[2], w[3]);
        }
    }
    for (int i = j0; i < nvec; i += 256) {
        float v[8];
        unpack8(L[i], v);
        uint32_t w[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            float p0 = __expf(v[2 * k] - lse), p1 = __expf(v[2 * k + 1] - lse);
            const int e0 = i * 8 + 2 * k;
            if (e0 >= V) p0 = 0.f;
            if (e0 + 1 >= V) p1 = 0.f;
            if (e0 == tgt) {
                row_loss[row] = lse - v[2 * k];
                p0 -= 1.f;
            }
            if (e0 + 1 == tgt) {
                row_loss[row] = lse - v[2 * k + 1];
                p1 -= 1.f;
            }
            __nv_bfloat162 h = __floats2bfloat162_rn(p0 * inv_seq, p1 * inv_seq);
            w[k] = *reinterpret_cast<uint32_t*>(&h);
        }
        L[i] = make_uint4(w[0], w[1], w[2], w[3]);
    }
}

__global__ void loss_reduce_kernel(const float* __restrict__ row_loss, int M, int seq, double* out) {
    ACCO_PDL_PROLOGUE();
    __shared__ double red[1024];
    double s = 0.0;
#pragma unroll 8
    for (int i = threadIdx.x; i < M; i += blockDim.x) s += row_loss[i];  // (loads independent of the adds)
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = red[0] / seq;
}

// --------------------------------------------------------- embedding backward
// Keys (token << 32 | position) sorted by a stable LSD radix sort on the token
// bits (8-bit digits): positions come in ascending order, so every token's
// positions stay ascending, and the keys are unique, so the order is unique —
// deterministic, any micro-batch size, any vocabulary (< 2^31). Per pass:
// per-tile digit histograms [digit][tile], one exclusive scan, then each tile
// scatters its keys in index order (one warp per tile, match_any ranking).
constexpr int kSortTile = 1024;

__device__ __forceinline__ uint64_t sort_key_in(const uint64_t* keys, const int32_t* tok, int i) {
    return keys ? keys[i] : (static_cast<uint64_t>(static_cast<uint32_t>(tok[i])) << 32) | static_cast<uint32_t>(i);
}

__global__ void radix_hist_kernel(const uint64_t* __restrict__ keys, const int32_t* __restrict__ tok, int M, int shift,
                                  unsigned* __restrict__ hist) {
    ACCO_PDL_PROLOGUE();
    __shared__ unsigned cnt[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) cnt[i] = 0;
    __syncthreads();
    const int t0 = blockIdx.x * kSortTile, t1 = min(M, t0 + kSortTile);
    for (int i = t0 + threadIdx.x; i < t1; i += blockDim.x)
        atomicAdd(&cnt[(sort_key_in(keys, tok, i) >> (32 + shift)) & 255u], 1u);  // integer: order-free
    __syncthreads();
    for (int dgt = threadIdx.x; dgt < 256; dgt += blockDim.x) hist[dgt * gridDim.x + blockIdx.x] = cnt[dgt];
}

// in-place exclusive scan of n counters, one block of 1024 threads
__global__ void radix_scan_kernel(unsigned* __restrict__ h, int n) {
    ACCO_PDL_PROLOGUE();
    __shared__ unsigned part[32];
    const int per = (n + blockDim.x - 1) / blockDim.x;
    const int a = threadIdx.x * per, b = min(n, a + per);
    unsigned s = 0;
    for (int i = a; i < b; ++i) s += h[i];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned x = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) part[w] = x;
    __syncthreads();
    if (w == 0) {
        unsigned p = lane < static_cast<int>(blockDim.x >> 5) ? part[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, p, o);
            if (lane >= o) p += y;
        }
        part[lane] = p;
    }
    __syncthreads();
    unsigned run = x - s + (w > 0 ? part[w - 1] : 0u);  // exclusive prefix of this thread's segment
    for (int i = a; i < b; ++i) {
        const unsigned v = h[i];
        h[i] = run;
        run += v;
    }
}

// one warp per tile: stable scatter in index order
__global__ void radix_scatter_kernel(const uint64_t* __restrict__ keys, const int32_t* __restrict__ tok, int M,
                                     int shift, const unsigned* __restrict__ offs, uint64_t* __restrict__ out) {
    ACCO_PDL_PROLOGUE();
    __shared__ unsigned run[256];
    const int lane = threadIdx.x;
    for (int dgt = lane; dgt < 256; dgt += 32) run[dgt] = offs[dgt * gridDim.x + blockIdx.x];
    __syncwarp();
    const int t0 = blockIdx.x * kSortTile, t1 = min(M, t0 + kSortTile);
    const unsigned lt = (1u << lane) - 1u;
    for (int base = t0; base < t1; base += 32) {
        const int i = base + lane;
        const bool valid = i < t1;
        const uint64_t key = valid ? sort_key_in(keys, tok, i) : 0;
        const unsigned dgt = valid ? static_cast<unsigned>(key >> (32 + shift)) & 255u : 256u + lane;
        const unsigned peers = __match_any_sync(0xffffffffu, dgt);
        const unsigned rank = __popc(peers & lt);
        if (valid) out[run[dgt] + rank] = key;
        __syncwarp();
        if (valid && rank == 0) run[dgt] += __popc(peers);
        __syncwarp();
    }
}

// Parallel deterministic segment sums for the token-embedding gradient (the
// Markov data makes a few tokens very hot, so a per-segment serial loop is
// latency-bound). The sorted (token, position) list is cut into fixed chunks
// of kEmbChunk entries; pass 1 sums each run (maximal same-token stretch) of
// a chunk into run_sum[chunk * kEmbChunk + run]; pass 2, per token segment,
// folds its runs in ascending chunk order into grad_wte. Fixed order
// throughout: bitwise reproducible.
constexpr int kEmbChunk = 32;

template <class T>
__global__ void embed_runs_kernel(const uint64_t* __restrict__ sorted, int M, const T* __restrict__ dx, int d,
                                  float* __restrict__ run_sum) {
    ACCO_PDL_PROLOGUE();
    const int p0 = blockIdx.x * kEmbChunk, p1 = min(M, p0 + kEmbChunk);
    for (int cg = threadIdx.x; cg < d / 8; cg += blockDim.x) {
        float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        uint32_t prev = static_cast<uint32_t>(sorted[p0] >> 32);
        int r = 0;
        for (int p = p0; p < p1; ++p) {
            const uint64_t key = sorted[p];
            const uint32_t tok = static_cast<uint32_t>(key >> 32);
            if (tok != prev) {
                float4* o = reinterpret_cast<float4*>(run_sum + static_cast<int64_t>(p0 + r) * d + cg * 8);
                o[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
                o[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
#pragma unroll
                for (int k = 0; k < 8; ++k) acc[k] = 0.f;
                ++r;
                prev = tok;
            }
            float v[8];
            load8<T>(dx + static_cast<int64_t>(static_cast<uint32_t>(key)) * d + cg * 8, v);
#pragma unroll
            for (int k = 0; k < 8; ++k) acc[k] += v[k];
        }
        float4* o = reinterpret_cast<float4*>(run_sum + static_cast<int64_t>(p0 + r) * d + cg * 8);
        o[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
        o[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
    }
}

__global__ void embed_fold_kernel(const uint64_t* __restrict__ sorted, int M, const float* __restrict__ run_sum,
                                  int d, float* __restrict__ grad_wte) {
    ACCO_PDL_PROLOGUE();
    const int i = blockIdx.x;
    auto tok_at = [&](int p) { return static_cast<uint32_t>(sorted[p] >> 32); };
    const uint32_t tok = tok_at(i);
    if (i > 0 && tok_at(i - 1) == tok) return;  // not a segment start
    const int c = i / kEmbChunk;
    int r0 = 0;  // run index of this segment inside its first chunk
    for (int p = c * kEmbChunk + 1; p <= i; ++p) r0 += tok_at(p) != tok_at(p - 1) ? 1 : 0;
    for (int cg = threadIdx.x; cg < d / 8; cg += blockDim.x) {
        const float4* a = reinterpret_cast<const float4*>(run_sum + static_cast<int64_t>(c * kEmbChunk + r0) * d +
                                                          cg * 8);
        float4 s0 = a[0], s1 = a[1];
        for (int cc = c + 1; cc * kEmbChunk < M && tok_at(cc * kEmbChunk) == tok; ++cc) {
            const float4* b = reinterpret_cast<const float4*>(run_sum + static_cast<int64_t>(cc) * kEmbChunk * d +
                                                              cg * 8);
            const float4 t0 = b[0], t1 = b[1];
            s0.x += t0.x; s0.y += t0.y; s0.z += t0.z; s0.w += t0.w;
            s1.x += t1.x; s1.y += t1.y; s1.z += t1.z; s1.w += t1.w;
        }
        float4* g = reinterpret_cast<float4*>(grad_wte + static_cast<int64_t>(tok) * d + cg * 8);
        float4 g0 = g[0], g1 = g[1];
        g0.x += s0.x; g0.y += s0.y; g0.z += s0.z; g0.w += s0.w;
        g1.x += s1.x; g1.y += s1.y; g1.z += s1.z; g1.w += s1.w;
        g[0] = g0;
        g[1] = g1;
    }
}

template <class T>
__global__ void embed_bwd_wpe_kernel(const T* __restrict__ dx, int B, int seq, int d, float* __restrict__ grad_wpe,
                                     int accumulate) {
    ACCO_PDL_PROLOGUE();
    const int t = blockIdx.x;
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
        float acc = 0.f;
        for (int b = 0; b < B; ++b) acc += to_f(dx[(static_cast<int64_t>(b) * seq + t) * d + c]);
        float* g = grad_wpe + static_cast<int64_t>(t) * d + c;
        *g = (accumulate ? *g : 0.f) + acc;
    }
}

// ------------------------------------------------------------------ utilities
__global__ void fill_i64_kernel(int64_t* p, int64_t v) {
    ACCO_PDL_PROLOGUE(); *p = v; }
__global__ void add_i64_kernel(int64_t* dst, const int64_t* a, const int64_t* b) {
    ACCO_PDL_PROLOGUE(); *dst = *a + *b; }

struct PtrList {
    const float* p[16];
};

__global__ void sum_ordered_kernel(PtrList in, int nin, float* __restrict__ out, int64_t n) {
    ACCO_PDL_PROLOGUE();
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        float s = in.p[0][i];
        for (int w = 1; w < nin; ++w) s += in.p[w][i];
        out[i] = s;
    }
}

template <class T>
__global__ void f32_to_kernel(const float* __restrict__ src, T* __restrict__ dst, int64_t n) {
    ACCO_PDL_PROLOGUE();
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
        dst[i] = from_f<T>(src[i]);
}

__global__ void scale_kernel(float* x, float a, int64_t n) {
    ACCO_PDL_PROLOGUE();
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) x[i] *= a;
}

__global__ void norm_sq_partial(const float* __restrict__ x, int64_t n, double* __restrict__ part) {
    ACCO_PDL_PROLOGUE();
    __shared__ double red[256];
    double s = 0.0;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
        double v = x[i];
        s += v * v;
    }
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

__global__ void norm_sq_final(const double* __restrict__ part, int nb, double* out) {
    ACCO_PDL_PROLOGUE();
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < nb; ++i) s += part[i];
        *out = s;
    }
}

struct Ranges {
    uint64_t lo[64];
    uint64_t sz[64];
};

__global__ void pack_kernel(const float* __restrict__ flat, float* __restrict__ padded, Ranges r, int n,
                            uint64_t chunk) {
    ACCO_PDL_PROLOGUE();
    const uint64_t total = chunk * n;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += stride) {
        const int w = static_cast<int>(i / chunk);
        const uint64_t j = i % chunk;
        padded[i] = j < r.sz[w] ? flat[r.lo[w] + j] : 0.f;
    }
}

template <class E>
__global__ void unpack_kernel(const E* __restrict__ padded, E* __restrict__ flat, Ranges r, int n,
                              uint64_t chunk) {
    ACCO_PDL_PROLOGUE();
    const uint64_t total = chunk * n;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += stride) {
        const int w = static_cast<int>(i / chunk);
        const uint64_t j = i % chunk;
        if (j < r.sz[w]) flat[r.lo[w] + j] = padded[i];
    }
}

__global__ void replica_hash_kernel(const uint32_t* __restrict__ w, int64_t n, unsigned long long* out) {
    ACCO_PDL_PROLOGUE();
    unsigned long long h = 0;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        h += splitmix_finalize(static_cast<uint64_t>(i) * kGolden ^ (static_cast<uint64_t>(__ldg(w + i)) << 17));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, h);  // wrapping u64 sum: order-independent
}

__global__ void hash_compare_kernel(const unsigned long long* all, int n, int k, int* flag, int bit) {
    ACCO_PDL_PROLOGUE();
    bool bad = false;
    for (int r = 1; r < n; ++r)
        for (int j = 0; j < k; ++j) bad |= all[r * k + j] != all[j];
    if (bad) atomicOr(flag, bit);
}

__global__ void spin_kernel(uint64_t ns) {
    uint64_t t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    uint64_t t = t0;
    while (t - t0 < ns) {
        __nanosleep(1000);
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    }
}

// paced multi-CTA copy (see lm_kernels.h comm_standin)
__global__ void __launch_bounds__(512) comm_standin_kernel(const uint4* __restrict__ src, uint4* __restrict__ dst,
                                                           int64_t n16, uint64_t ns) {
    ACCO_PDL_PROLOGUE();
    __shared__ uint64_t t0s;
    if (threadIdx.x == 0) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        t0s = t;
    }
    __syncthreads();
    const uint64_t t0 = t0s;
    const int64_t per = (n16 + gridDim.x - 1) / gridDim.x;
    const int64_t lo = static_cast<int64_t>(blockIdx.x) * per, hi = min(n16, lo + per);
    constexpr int kChunk = 512 * 8;  // 64 KB per CTA step
    const int64_t steps = (hi - lo + kChunk - 1) / kChunk;
    for (int64_t s = 0; s < steps; ++s) {
        const int64_t b = lo + s * kChunk;
#pragma unroll 8
        for (int k = 0; k < 8; ++k) {
            const int64_t i = b + k * 512 + threadIdx.x;
            if (i < hi) dst[i] = __ldcs(src + i);
        }
        // pace: the link delivers (s + 1) / steps of this CTA's share by t0 + that fraction of ns
        const uint64_t due = t0 + static_cast<uint64_t>(static_cast<double>(ns) * (s + 1) / steps);
        uint64_t t;
        do {
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t < due) __nanosleep(500);
        } while (t < due);
    }
}

// ------------------------------------------------------ rotary / SwiGLU (Llama)
// In place on the q|k columns of qkv [M, ld]: nh = n_head + n_kv_head heads
// of hd columns from column 0. Pair (i, i + hd/2), angle table cs[t][i] =
// (cos, sin) (host fp64, rounded to fp32). dir = +1 rotates (forward);
// dir = -1 applies the transpose (backward of the rotation on dq, dk).
template <class T>
__global__ void rope_kernel(T* __restrict__ qkv, int64_t ld, const float2* __restrict__ cs, int M, int seq, int nh,
                            int hd, float dir) {
    ACCO_PDL_PROLOGUE();
    const int h2 = hd / 2;
    const int64_t n = static_cast<int64_t>(M) * nh * h2;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int j = static_cast<int>(i % h2);
        const int64_t mh = i / h2;
        const int head = static_cast<int>(mh % nh);
        const int m = static_cast<int>(mh / nh);
        const float2 c = cs[static_cast<int64_t>(m % seq) * h2 + j];
        const float sn = dir * c.y;
        T* p = qkv + static_cast<int64_t>(m) * ld + head * hd + j;
        const float x1 = to_f(p[0]), x2 = to_f(p[h2]);
        p[0] = from_f<T>(x1 * c.x - x2 * sn);
        p[h2] = from_f<T>(x2 * c.x + x1 * sn);
    }
}

// bf16, 8 pairs per thread (16 B loads of each half)
__global__ void rope_vec_kernel(__nv_bfloat16* __restrict__ qkv, int64_t ld, const float2* __restrict__ cs, int M,
                                int seq, int nh, int hd, float dir) {
    ACCO_PDL_PROLOGUE();
    const int h2 = hd / 2, nv = h2 / 8;
    const int64_t n = static_cast<int64_t>(M) * nh * nv;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int j0 = static_cast<int>(i % nv) * 8;
        const int64_t mh = i / nv;
        const int head = static_cast<int>(mh % nh);
        const int m = static_cast<int>(mh / nh);
        const float2* c = cs + static_cast<int64_t>(m % seq) * h2 + j0;
        __nv_bfloat16* p = qkv + static_cast<int64_t>(m) * ld + head * hd + j0;
        float a[8], b[8], ya[8], yb[8];
        unpack8b(*reinterpret_cast<const uint4*>(p), a);
        unpack8b(*reinterpret_cast<const uint4*>(p + h2), b);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const float2 t = c[k];
            const float sn = dir * t.y;
            ya[k] = a[k] * t.x - b[k] * sn;
            yb[k] = b[k] * t.x + a[k] * sn;
        }
        *reinterpret_cast<uint4*>(p) = pack8b(ya);
        *reinterpret_cast<uint4*>(p + h2) = pack8b(yb);
    }
}

__device__ __forceinline__ float sigmoid_f(float x) { return 1.0f / (1.0f + expf(-x)); }

// a[m, j] = silu(gu[m, j]) * gu[m, F + j]
template <class T>
__global__ void swiglu_fwd_kernel(const T* __restrict__ gu, T* __restrict__ a, int M, int F) {
    ACCO_PDL_PROLOGUE();
    const int64_t n = static_cast<int64_t>(M) * F;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t m = i / F;
        const int j = static_cast<int>(i % F);
        const float g = to_f(gu[m * 2 * F + j]), u = to_f(gu[m * 2 * F + F + j]);
        a[i] = from_f<T>(g * sigmoid_f(g) * u);
    }
}

// dgu[m, j] = da * u * s * (1 + g (1 - s)),  dgu[m, F + j] = da * g * s
template <class T>
__global__ void swiglu_bwd_kernel(const T* __restrict__ da, const T* __restrict__ gu, T* __restrict__ dgu, int M,
                                  int F) {
    ACCO_PDL_PROLOGUE();
    const int64_t n = static_cast<int64_t>(M) * F;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t m = i / F;
        const int j = static_cast<int>(i % F);
        const float g = to_f(gu[m * 2 * F + j]), u = to_f(gu[m * 2 * F + F + j]), d = to_f(da[i]);
        const float sg = sigmoid_f(g);
        dgu[m * 2 * F + j] = from_f<T>(d * u * sg * (1.0f + g * (1.0f - sg)));
        dgu[m * 2 * F + F + j] = from_f<T>(d * g * sg);
    }
}

// bf16, 8 columns per thread (F % 8 == 0)
__global__ void swiglu_fwd_vec(const __nv_bfloat16* __restrict__ gu, __nv_bfloat16* __restrict__ a, int M, int F) {
    ACCO_PDL_PROLOGUE();
    const int fv = F / 8;
    const int64_t n = static_cast<int64_t>(M) * fv;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t m = i / fv;
        const int j = static_cast<int>(i % fv) * 8;
        float g[8], u[8], o[8];
        unpack8b(*reinterpret_cast<const uint4*>(gu + m * 2 * F + j), g);
        unpack8b(*reinterpret_cast<const uint4*>(gu + m * 2 * F + F + j), u);
#pragma unroll
        for (int k = 0; k < 8; ++k) o[k] = g[k] * sigmoid_f(g[k]) * u[k];
        *reinterpret_cast<uint4*>(a + m * F + j) = pack8b(o);
    }
}

__global__ void swiglu_bwd_vec(const __nv_bfloat16* __restrict__ da, const __nv_bfloat16* __restrict__ gu,
                               __nv_bfloat16* __restrict__ dgu, int M, int F) {
    ACCO_PDL_PROLOGUE();
    const int fv = F / 8;
    const int64_t n = static_cast<int64_t>(M) * fv;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t m = i / fv;
        const int j = static_cast<int>(i % fv) * 8;
        float g[8], u[8], d[8], dg[8], du[8];
        unpack8b(*reinterpret_cast<const uint4*>(gu + m * 2 * F + j), g);
        unpack8b(*reinterpret_cast<const uint4*>(gu + m * 2 * F + F + j), u);
        unpack8b(*reinterpret_cast<const uint4*>(da + m * F + j), d);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const float sg = sigmoid_f(g[k]);
            dg[k] = d[k] * u[k] * sg * (1.0f + g[k] * (1.0f - sg));
            du[k] = d[k] * g[k] * sg;
        }
        *reinterpret_cast<uint4*>(dgu + m * 2 * F + j) = pack8b(dg);
        *reinterpret_cast<uint4*>(dgu + m * 2 * F + F + j) = pack8b(du);
    }
}

int grid_for(int64_t n, int threads = 256) {
    int64_t b = (n + threads - 1) / threads;
    int64_t cap = static_cast<int64_t>(num_sms()) * 8;
    return static_cast<int>(b < 1 ? 1 : (b > cap ? cap : b));
}

}  // namespace

// =================================================================== launchers
void gather_tokens(const int32_t* data, int seq, int n_samples, uint64_t seed, int mode, int start, int B,
                   int32_t* tok_in, int32_t* tok_out, int32_t* idx_out, cudaStream_t s) {
    ProfScope prof(kProfEmbed, 8.0 * B * seq, s);
    launch_pdl(gather_tokens_kernel, B, 128, 0, s, data, seq, n_samples, seed, mode, start, tok_in, tok_out, idx_out);
    ACCO_CHECK_LAUNCH();
}

template <class T>
void embed_fwd(const int32_t* tok, const T* wte, const T* wpe, T* x, int M, int seq, int d, cudaStream_t s) {
    ProfScope prof(kProfEmbed, 3.0 * M * d * sizeof(T), s);
    launch_pdl(embed_fwd_kernel<T>, M, 128, 0, s, tok, wte, wpe, x, seq, d);
    ACCO_CHECK_LAUNCH();
}

static bool a16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

template <bool RMS, class T>
static void layernorm_fwd_impl(const T* x, const T* g, const T* b, T* y, float* mean, float* rstd, int M, int d,
                               cudaStream_t s) {
    if constexpr (sizeof(T) == 2) {
        if (a16(x) && a16(g) && a16(b) && a16(y) && d % 256 == 0) {
            const int grid = ceil_div(M, 8);
            switch (d / 256) {
                case 1: launch_pdl(ln_fwd_vec<1, RMS>, grid, 256, 0, s, x, g, b, y, mean, rstd, M); ACCO_CHECK_LAUNCH(); return;
                case 2: launch_pdl(ln_fwd_vec<2, RMS>, grid, 256, 0, s, x, g, b, y, mean, rstd, M); ACCO_CHECK_LAUNCH(); return;
                case 3: launch_pdl(ln_fwd_vec<3, RMS>, grid, 256, 0, s, x, g, b, y, mean, rstd, M); ACCO_CHECK_LAUNCH(); return;
                case 4: launch_pdl(ln_fwd_vec<4, RMS>, grid, 256, 0, s, x, g, b, y, mean, rstd, M); ACCO_CHECK_LAUNCH(); return;
                case 8: launch_pdl(ln_fwd_vec<8, RMS>, grid, 256, 0, s, x, g, b, y, mean, rstd, M); ACCO_CHECK_LAUNCH(); return;
                default: break;
            }
        }
    }
    launch_pdl(ln_fwd_kernel<T, RMS>, ceil_div(M, 8), 256, 0, s, x, g, b, y, mean, rstd, M, d);
    ACCO_CHECK_LAUNCH();
}

template <class T>
void layernorm_fwd(const T* x, const T* g, const T* b, T* y, float* mean, float* rstd, int M, int d,
                   cudaStream_t s, bool rms) {
    ProfScope prof(kProfNorm, 2.0 * M * d * sizeof(T) + 8.0 * M, s);
    if (rms)
        layernorm_fwd_impl<true>(x, g, static_cast<const T*>(nullptr), y, mean, rstd, M, d, s);
    else
        layernorm_fwd_impl<false>(x, g, b, y, mean, rstd, M, d, s);
}

template <bool RMS, class T>
static bool ln_bwd_dx_vec(const T* dy, const T* x, const T* g, const float* mean, const float* rstd, T* dx,
                          bool accumulate_dx, int M, int d, cudaStream_t s) {
    if constexpr (sizeof(T) == 2) {
        if (a16(dy) && a16(x) && a16(g) && a16(dx) && d % 256 == 0) {
            const int grid = ceil_div(M, 8), acc = accumulate_dx ? 1 : 0;
            if (d >= 1024 && !std::getenv("ACCO_LN_NARROW")) {
                switch (d) {
                    case 1024: launch_pdl(ln_bwd_wide<128, RMS>, M, 128, 0, s, dy, x, g, mean, rstd, dx, acc); ACCO_CHECK_LAUNCH(); return true;
                    case 2048: launch_pdl(ln_bwd_wide<256, RMS>, M, 256, 0, s, dy, x, g, mean, rstd, dx, acc); ACCO_CHECK_LAUNCH(); return true;
                    case 4096: launch_pdl(ln_bwd_wide<512, RMS>, M, 512, 0, s, dy, x, g, mean, rstd, dx, acc); ACCO_CHECK_LAUNCH(); return true;
                    default: break;
                }
            }
            switch (d / 256) {
                case 1: launch_pdl(ln_bwd_vec<1, RMS>, grid, 256, 0, s, dy, x, g, mean, rstd, dx, acc, M); break;
                case 2: launch_pdl(ln_bwd_vec<2, RMS>, grid, 256, 0, s, dy, x, g, mean, rstd, dx, acc, M); break;
                case 3: launch_pdl(ln_bwd_vec<3, RMS>, grid, 256, 0, s, dy, x, g, mean, rstd, dx, acc, M); break;
                case 4: launch_pdl(ln_bwd_vec<4, RMS>, grid, 256, 0, s, dy, x, g, mean, rstd, dx, acc, M); break;
                case 8: launch_pdl(ln_bwd_vec<8, RMS>, grid, 256, 0, s, dy, x, g, mean, rstd, dx, acc, M); break;
                default: return false;
            }
            ACCO_CHECK_LAUNCH();
            return true;
        }
    }
    return false;
}

static unsigned* tickets() {
    static unsigned* t = nullptr;
    if (!t) {
        ACCO_CUDA(cudaMalloc(&t, 8192 * sizeof(unsigned)));
        ACCO_CUDA(cudaMemset(t, 0, 8192 * sizeof(unsigned)));
    }
    return t;
}

template <class T>
static bool vec_ok(const void* p, int64_t ld, int N) {
    return N % 8 == 0 && ld % 8 == 0 && (reinterpret_cast<uintptr_t>(p) & 15) == 0 && ceil_div(N, 64) <= 8192;
}

// grid: slabs x chunks with ~2 waves of 148 SMs
template <class T, int KIND>
static void colsum_vec(const T* y, int64_t ld, const T* x, const float* mean, const float* rstd, int M, int N,
                       float* out, float* out1, float* scratch, bool acc, cudaStream_t s) {
    const int slabs = ceil_div(N, 64);
    // ~8 blocks per SM: enough 16B loads in flight to stream the (L2-resident)
    // operand at bandwidth; partials are reduced by each slab's last block
    static const int per_sm = std::getenv("ACCO_COLSUM_PER_SM") ? std::atoi(std::getenv("ACCO_COLSUM_PER_SM")) : 4;
    int nchunk = std::max(1, std::min(ceil_div(per_sm * num_sms(), slabs), ceil_div(M, kVecRows)));
    const int rpc = ceil_div(ceil_div(M, nchunk), kVecRows) * kVecRows;
    nchunk = ceil_div(M, rpc);
    launch_pdl(colsum_vec_kernel<T, KIND>, dim3(slabs, nchunk), 256, 0, s, y, ld, x, mean, rstd, M, N, rpc, scratch,
                                                                    tickets(), out, out1, acc ? 1 : 0);
    ACCO_CHECK_LAUNCH();
}

template <class T>
void layernorm_bwd_params(const T* dy, const T* x, const float* mean, const float* rstd, float* gdst, float* bdst,
                          float* scratch, int M, int d, bool acc, cudaStream_t s) {
    ProfScope prof(kProfReduce, 2.0 * M * d * sizeof(T) + 8.0 * M, s);
    // bdst == nullptr: RMSNorm (weight only)
    if (vec_ok<T>(dy, d, d) && vec_ok<T>(x, d, d)) {
        if (bdst)
            colsum_vec<T, 1>(dy, d, x, mean, rstd, M, d, gdst, bdst, scratch, acc, s);
        else
            colsum_vec<T, 2>(dy, d, x, mean, rstd, M, d, gdst, nullptr, scratch, acc, s);
        return;
    }
    const int nchunk = ceil_div(M, kColChunk);
    float* p0 = scratch;
    float* p1 = scratch + static_cast<int64_t>(nchunk) * d;
    if (bdst)
        launch_pdl(colreduce_partial<T, 1>, dim3(ceil_div(d, 32), nchunk), dim3(32, kColRows), 0, s, dy, d, x, mean, rstd,
                                                                                             M, d, p0, p1);
    else
        launch_pdl(colreduce_partial<T, 2>, dim3(ceil_div(d, 32), nchunk), dim3(32, kColRows), 0, s, dy, d, x, mean, rstd,
                                                                                             M, d, p0, p1);
    ACCO_CHECK_LAUNCH();
    launch_pdl(colreduce_final, ceil_div(d, 256), 256, 0, s, p0, nchunk, d, gdst, acc ? 1 : 0);
    if (bdst) launch_pdl(colreduce_final, ceil_div(d, 256), 256, 0, s, p1, nchunk, d, bdst, acc ? 1 : 0);
    ACCO_CHECK_LAUNCH();
}

template <class T>
void layernorm_bwd_dx(const T* dy, const T* x, const T* g, const float* mean, const float* rstd, T* dx,
                      bool accumulate_dx, int M, int d, cudaStream_t s, bool rms) {
    ProfScope prof(kProfNorm, 3.0 * M * d * sizeof(T) + 8.0 * M, s);
    const bool v = vec_ok<T>(dy, d, d) && vec_ok<T>(x, d, d);
    if (rms) {
        if (v && ln_bwd_dx_vec<true>(dy, x, g, mean, rstd, dx, accumulate_dx, M, d, s)) return;
        launch_pdl(ln_bwd_kernel<T, true>, ceil_div(M, 8), 256, 0, s, dy, x, g, mean, rstd, dx, accumulate_dx ? 1 : 0, M, d);
    } else {
        if (v && ln_bwd_dx_vec<false>(dy, x, g, mean, rstd, dx, accumulate_dx, M, d, s)) return;
        launch_pdl(ln_bwd_kernel<T, false>, ceil_div(M, 8), 256, 0, s, dy, x, g, mean, rstd, dx, accumulate_dx ? 1 : 0, M, d);
    }
    ACCO_CHECK_LAUNCH();
}

int ln_part_blocks() {
    static const int per_sm = std::getenv("ACCO_LN_PART_PER_SM") ? std::atoi(std::getenv("ACCO_LN_PART_PER_SM")) : 2;
    return std::max(1, per_sm) * num_sms();
}

// The warp-per-row form keeps 2 x 8 CH parameter sums per lane: CH <= 3
// without spills. Wider rows keep the block-per-row dx kernel and the separate
// side-stream parameter reduction: a persistent block-per-row form with the
// sums in registers (d = 1024: 4 warps per block) measured slower end to end
// (GPT-2 medium 319.8k vs 335.2k tok/s, profiles/r02_summary.md).
bool ln_fused_supported(int d) {
    if (d % 256 != 0 || d > 768 || std::getenv("ACCO_LN_PARAMS_SEPARATE")) return false;
    const int ch = d / 256;
    return ch == 1 || ch == 2 || ch == 3;
}

template <class T>
void layernorm_bwd_fused(const T* dy, const T* x, const T* g, const float* mean, const float* rstd, T* dx,
                         bool accumulate_dx, int M, int d, float* part, cudaStream_t s, bool rms) {
    if constexpr (sizeof(T) != 2) {
        throw Error(kInvalidArg, "layernorm_bwd_fused: bf16 only");
    } else {
        ACCO_REQUIRE(ln_fused_supported(d) && a16(dy) && a16(x) && a16(g) && a16(dx),
                     "layernorm_bwd_fused: unsupported width or alignment");
        ProfScope prof(kProfNorm, 3.0 * M * d * sizeof(T) + 8.0 * M, s);
        const int G = ln_part_blocks(), acc = accumulate_dx ? 1 : 0;
#define ACCO_LNP(KERN, BLOCK, SMEM)                                                                    \
    do {                                                                                               \
        static bool cfg = false;                                                                       \
        if (!cfg && (SMEM) > 40 * 1024) { /* (+ the static barriers) */                               \
            ACCO_CUDA(cudaFuncSetAttribute(KERN, cudaFuncAttributeMaxDynamicSharedMemorySize, (SMEM))); \
        }                                                                                              \
        cfg = true;                                                                                    \
        launch_pdl(KERN, G, BLOCK, SMEM, s, dy, x, g, mean, rstd, dx, acc, M, part);                   \
    } while (0)
        {
            // per warp kLnStages x (x | dy | dx) staged rows; the block reduction reuses it
            const int smem = std::max(8 * kLnStages * 3 * d * 2, 8 * d * 4);
            switch ((d / 256) * 2 + (rms ? 1 : 0)) {
                case 2: ACCO_LNP((ln_bwd_vec_p<1, false>), 256, smem); break;
                case 3: ACCO_LNP((ln_bwd_vec_p<1, true>), 256, smem); break;
                case 4: ACCO_LNP((ln_bwd_vec_p<2, false>), 256, smem); break;
                case 5: ACCO_LNP((ln_bwd_vec_p<2, true>), 256, smem); break;
                case 6: ACCO_LNP((ln_bwd_vec_p<3, false>), 256, smem); break;
                case 7: ACCO_LNP((ln_bwd_vec_p<3, true>), 256, smem); break;
                default: throw Error(kInvalidArg, "layernorm_bwd_fused: unsupported width");
            }
        }
#undef ACCO_LNP
        ACCO_CHECK_LAUNCH();
    }
}

void ln_param_fold(const LnFold* table, int n, int d_max, const float* parts, float* grad, bool acc, cudaStream_t s) {
    if (n == 0) return;
    ProfScope prof(kProfReduce, 1.0 * n * ln_part_blocks() * 2 * d_max * 4, s);
    launch_pdl(ln_param_fold_kernel, dim3(ceil_div(2 * d_max, kFoldCols), n), kFoldCols * kFoldSub, 0, s, table, parts, grad, ln_part_blocks(),
               acc ? 1 : 0);
    ACCO_CHECK_LAUNCH();
}

template <class T>
void colsum_add(const T* y, int64_t ld, int M, int N, float* out, float* scratch, bool acc, cudaStream_t s) {
    ProfScope prof(kProfReduce, 1.0 * M * N * sizeof(T), s);
    if (vec_ok<T>(y, ld, N)) {
        colsum_vec<T, 0>(y, ld, nullptr, nullptr, nullptr, M, N, out, nullptr, scratch, acc, s);
        return;
    }
    const int nchunk = ceil_div(M, kColChunk);
    launch_pdl(colreduce_partial<T, 0>, dim3(ceil_div(N, 32), nchunk), dim3(32, kColRows), 0, s, 
        y, ld, nullptr, nullptr, nullptr, M, N, scratch, nullptr);
    ACCO_CHECK_LAUNCH();
    launch_pdl(colreduce_final, ceil_div(N, 256), 256, 0, s, scratch, nchunk, N, out, acc ? 1 : 0);
    ACCO_CHECK_LAUNCH();
}

template <class T>
void cross_entropy(T* logits, int64_t ld, const int32_t* target, int V, int M, int seq, float* row_loss,
                   cudaStream_t s) {
    ProfScope prof(kProfCE, 2.0 * M * V * sizeof(T), s);
    if constexpr (sizeof(T) == 2) {
        const bool aligned = (reinterpret_cast<uintptr_t>(logits) & 15) == 0 && ld % 8 == 0;
        if (aligned) {
            launch_pdl(ce_vec_kernel, M, 256, 0, s, reinterpret_cast<__nv_bfloat16*>(logits), ld, target, V, 1.0f / seq,
                                            row_loss);
            ACCO_CHECK_LAUNCH();
            return;
        }
    }
    launch_pdl(ce_kernel<T>, M, 512, 0, s, logits, ld, target, V, 1.0f / seq, row_loss);
    ACCO_CHECK_LAUNCH();
}

void loss_reduce(const float* row_loss, int M, int seq, double* out, cudaStream_t s) {
    launch_pdl(loss_reduce_kernel, 1, 1024, 0, s, row_loss, M, seq, out);
    ACCO_CHECK_LAUNCH();
}

void embed_sort(const int32_t* tok, int M, int V, uint64_t* sorted, uint64_t* tmp, unsigned* hist, cudaStream_t s) {
    ProfScope prof(kProfEmbed, 8.0 * M, s);
    ACCO_REQUIRE(V >= 1 && M >= 1, "embed_sort: empty input");
    int bits = 0;
    while ((1ll << bits) < V) ++bits;
    const int passes = std::max(1, (bits + 7) / 8);
    const int tiles = ceil_div(M, kSortTile);
    // ping-pong so the last pass lands in `sorted`
    uint64_t* bufs[2] = {passes % 2 ? sorted : tmp, passes % 2 ? tmp : sorted};
    const uint64_t* in = nullptr;  // pass 0 reads the tokens (keys built on the fly)
    for (int p = 0; p < passes; ++p) {
        uint64_t* out = bufs[p & 1];
        launch_pdl(radix_hist_kernel, tiles, 256, 0, s, in, tok, M, 8 * p, hist);
        ACCO_CHECK_LAUNCH();
        launch_pdl(radix_scan_kernel, 1, 1024, 0, s, hist, 256 * tiles);
        ACCO_CHECK_LAUNCH();
        launch_pdl(radix_scatter_kernel, tiles, 32, 0, s, in, tok, M, 8 * p, static_cast<const unsigned*>(hist), out);
        ACCO_CHECK_LAUNCH();
        in = out;
    }
}

template <class T>
void embed_bwd(const uint64_t* sorted, const T* dx, int M, int seq, int d, int V, float* grad_wte, float* grad_wpe,
               float* run_sum, bool acc_wpe, cudaStream_t s, bool zero_wte) {
    ProfScope prof(kProfEmbed, 1.0 * M * d * sizeof(T), s);
    ACCO_REQUIRE(d % 8 == 0, "embed_bwd: d_model must be a multiple of 8");
    // untied embedding (Llama) on the stage's first micro-batch: no earlier
    // kernel wrote grad_wte, so the rows no token touches must be zeroed
    if (zero_wte) ACCO_CUDA(cudaMemsetAsync(grad_wte, 0, static_cast<size_t>(V) * d * sizeof(float), s));
    const int threads = std::min(256, std::max(32, d / 8));
    launch_pdl(embed_runs_kernel<T>, ceil_div(M, kEmbChunk), threads, 0, s, sorted, M, dx, d, run_sum);
    ACCO_CHECK_LAUNCH();
    launch_pdl(embed_fold_kernel, M, threads, 0, s, sorted, M, run_sum, d, grad_wte);
    ACCO_CHECK_LAUNCH();
    if (grad_wpe) {
        launch_pdl(embed_bwd_wpe_kernel<T>, seq, 128, 0, s, dx, M / seq, seq, d, grad_wpe, acc_wpe ? 1 : 0);
        ACCO_CHECK_LAUNCH();
    }
}

template <class T>
void rope_apply(T* qkv, int64_t ld, const float2* cs, int M, int seq, int nh, int hd, bool inverse, cudaStream_t s) {
    ProfScope prof(kProfOther, 4.0 * M * nh * hd * sizeof(T), s);
    ACCO_REQUIRE(hd % 2 == 0, "rope: head size must be even");
    const float dir = inverse ? -1.0f : 1.0f;
    if constexpr (sizeof(T) == 2) {
        if ((hd / 2) % 8 == 0 && ld % 8 == 0 && a16(qkv)) {
            const int64_t n = static_cast<int64_t>(M) * nh * (hd / 16);
            launch_pdl(rope_vec_kernel, grid_for(n), 256, 0, s, qkv, ld, cs, M, seq, nh, hd, dir);
            ACCO_CHECK_LAUNCH();
            return;
        }
    }
    launch_pdl(rope_kernel<T>, grid_for(static_cast<int64_t>(M) * nh * (hd / 2)), 256, 0, s, qkv, ld, cs, M, seq, nh, hd, dir);
    ACCO_CHECK_LAUNCH();
}

template <class T>
void swiglu_fwd(const T* gu, T* a, int M, int F, cudaStream_t s) {
    ProfScope prof(kProfOther, 3.0 * M * F * sizeof(T), s);
    if constexpr (sizeof(T) == 2) {
        if (F % 8 == 0 && a16(gu) && a16(a)) {
            launch_pdl(swiglu_fwd_vec, grid_for(static_cast<int64_t>(M) * F / 8), 256, 0, s, gu, a, M, F);
            ACCO_CHECK_LAUNCH();
            return;
        }
    }
    launch_pdl(swiglu_fwd_kernel<T>, grid_for(static_cast<int64_t>(M) * F), 256, 0, s, gu, a, M, F);
    ACCO_CHECK_LAUNCH();
}

template <class T>
void swiglu_bwd(const T* da, const T* gu, T* dgu, int M, int F, cudaStream_t s) {
    ProfScope prof(kProfOther, 5.0 * M * F * sizeof(T), s);
    if constexpr (sizeof(T) == 2) {
        if (F % 8 == 0 && a16(gu) && a16(da) && a16(dgu)) {
            launch_pdl(swiglu_bwd_vec, grid_for(static_cast<int64_t>(M) * F / 8), 256, 0, s, da, gu, dgu, M, F);
            ACCO_CHECK_LAUNCH();
            return;
        }
    }
    launch_pdl(swiglu_bwd_kernel<T>, grid_for(static_cast<int64_t>(M) * F), 256, 0, s, da, gu, dgu, M, F);
    ACCO_CHECK_LAUNCH();
}

void replica_hash(const void* p, int64_t bytes, uint64_t* out, cudaStream_t s) {
    ACCO_REQUIRE(bytes % 4 == 0, "replica_hash: whole 32-bit words");
    ACCO_CUDA(cudaMemsetAsync(out, 0, sizeof(uint64_t), s));
    const int64_t n = bytes / 4;
    const int blocks = static_cast<int>(std::min<int64_t>((n + 255) / 256, 4 * num_sms()));
    launch_pdl(replica_hash_kernel, std::max(blocks, 1), 256, 0, s, static_cast<const uint32_t*>(p), n,
               reinterpret_cast<unsigned long long*>(out));
    ACCO_CHECK_LAUNCH();
}

void hash_compare(const uint64_t* all, int n, int k, int* flag, int bit, cudaStream_t s) {
    launch_pdl(hash_compare_kernel, 1, 1, 0, s, reinterpret_cast<const unsigned long long*>(all), n, k, flag, bit);
    ACCO_CHECK_LAUNCH();
}

void fill_i64(int64_t* p, int64_t v, cudaStream_t s) {
    launch_pdl(fill_i64_kernel, 1, 1, 0, s, p, v);
    ACCO_CHECK_LAUNCH();
}

void add_i64(int64_t* dst, const int64_t* a, const int64_t* b, cudaStream_t s) {
    launch_pdl(add_i64_kernel, 1, 1, 0, s, dst, a, b);
    ACCO_CHECK_LAUNCH();
}

void sum_ordered(const float* const* in, int nin, float* out, int64_t n, cudaStream_t s) {
    ACCO_REQUIRE(nin >= 1 && nin <= 16, "sum_ordered: 1..16 inputs");
    PtrList l{};
    for (int i = 0; i < nin; ++i) l.p[i] = in[i];
    launch_pdl(sum_ordered_kernel, grid_for(n), 256, 0, s, l, nin, out, n);
    ACCO_CHECK_LAUNCH();
}

void f32_to(const float* src, void* dst, int dtype, int64_t n, cudaStream_t s) {
    if (dtype == 1)
        launch_pdl(f32_to_kernel<__nv_bfloat16>, grid_for(n), 256, 0, s, src, static_cast<__nv_bfloat16*>(dst), n);
    else
        launch_pdl(f32_to_kernel<float>, grid_for(n), 256, 0, s, src, static_cast<float*>(dst), n);
    ACCO_CHECK_LAUNCH();
}

void scale_f32(float* x, double alpha, int64_t n, cudaStream_t s) {
    launch_pdl(scale_kernel, grid_for(n), 256, 0, s, x, static_cast<float>(alpha), n);
    ACCO_CHECK_LAUNCH();
}

void norm_sq(const float* x, int64_t n, double* out, double* scratch, cudaStream_t s) {
    const int nb = 256;
    launch_pdl(norm_sq_partial, nb, 256, 0, s, x, n, scratch);
    launch_pdl(norm_sq_final, 1, 32, 0, s, scratch, nb, out);
    ACCO_CHECK_LAUNCH();
}

static Ranges make_ranges(const uint64_t* lo, const uint64_t* sz, int n) {
    ACCO_REQUIRE(n >= 1 && n <= 64, "padded layout: 1..64 workers");
    Ranges r{};
    for (int i = 0; i < n; ++i) {
        r.lo[i] = lo[i];
        r.sz[i] = sz[i];
    }
    return r;
}

void pack_padded(const float* flat, float* padded, const uint64_t* lo, const uint64_t* sz, int n, uint64_t chunk,
                 cudaStream_t s) {
    launch_pdl(pack_kernel, grid_for(static_cast<int64_t>(chunk * n)), 256, 0, s, flat, padded, make_ranges(lo, sz, n), n,
                                                                          chunk);
    ACCO_CHECK_LAUNCH();
}

void unpack_padded(const void* padded, void* flat, int elem_bytes, const uint64_t* lo, const uint64_t* sz, int n,
                   uint64_t chunk, cudaStream_t s) {
    Ranges r = make_ranges(lo, sz, n);
    const int g = grid_for(static_cast<int64_t>(chunk * n));
    if (elem_bytes == 4)
        launch_pdl(unpack_kernel<float>, g, 256, 0, s, static_cast<const float*>(padded), static_cast<float*>(flat), r, n, chunk);
    else
        launch_pdl(unpack_kernel<__nv_bfloat16>, g, 256, 0, s, static_cast<const __nv_bfloat16*>(padded),
                                                        static_cast<__nv_bfloat16*>(flat), r, n, chunk);
    ACCO_CHECK_LAUNCH();
}

void spin_ns(uint64_t ns, cudaStream_t s) {
    if (ns == 0) return;
    spin_kernel<<<1, 1, 0, s>>>(ns);
    ACCO_CHECK_LAUNCH();
}

void comm_standin(const void* src, void* dst, int64_t bytes, int ctas, uint64_t ns, cudaStream_t s) {
    if (bytes <= 0 || ctas <= 0) return;
    launch_pdl(comm_standin_kernel, ctas, 512, 0, s, static_cast<const uint4*>(src), static_cast<uint4*>(dst),
               bytes / 16, ns);
    ACCO_CHECK_LAUNCH();
}

#define ACCO_INST(T)                                                                                          \
    template void embed_fwd<T>(const int32_t*, const T*, const T*, T*, int, int, int, cudaStream_t);          \
    template void layernorm_fwd<T>(const T*, const T*, const T*, T*, float*, float*, int, int, cudaStream_t,  \
                                   bool);                                                                     \
    template void layernorm_bwd_params<T>(const T*, const T*, const float*, const float*, float*, float*,      \
                                          float*, int, int, bool, cudaStream_t);                              \
    template void layernorm_bwd_dx<T>(const T*, const T*, const T*, const float*, const float*, T*, bool, int, \
                                      int, cudaStream_t, bool);                                               \
    template void colsum_add<T>(const T*, int64_t, int, int, float*, float*, bool, cudaStream_t);\
    template void layernorm_bwd_fused<T>(const T*, const T*, const T*, const float*, const float*, T*, bool, int, \
                                         int, float*, cudaStream_t, bool);             \
    template void cross_entropy<T>(T*, int64_t, const int32_t*, int, int, int, float*, cudaStream_t);         \
    template void embed_bwd<T>(const uint64_t*, const T*, int, int, int, int, float*, float*, float*,        \
                               bool, cudaStream_t, bool);                                                     \
    template void rope_apply<T>(T*, int64_t, const float2*, int, int, int, int, bool, cudaStream_t);          \
    template void swiglu_fwd<T>(const T*, T*, int, int, cudaStream_t);                                        \
    template void swiglu_bwd<T>(const T*, const T*, T*, int, int, cudaStream_t);
ACCO_INST(float)
ACCO_INST(__nv_bfloat16)
#undef ACCO_INST

}  // namespace acco
