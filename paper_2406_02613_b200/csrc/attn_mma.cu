// Causal flash attention on tensor cores (bf16 in, fp32 accumulate), head
// size 64: mma.sync m16n8k16 + ldmatrix, 128B-XOR-swizzled smem tiles loaded
// with cp.async (double buffered).
//   forward : one CTA per (batch*head, 64-query tile); online softmax, writes
//             O and the natural-log row log-sum-exp.
//   backward: dK/dV kernel per (batch*head, 64-key tile) looping over query
//             tiles, and a separate dQ kernel per query tile looping over key
//             tiles — no float atomics, so results are bitwise deterministic
//             (the reference's order-fixed folds, problems.cpp:92-131).
#include "common.cuh"

namespace acco {
namespace {

constexpr int HD = 64;
constexpr int BR = 64;  // tile rows (queries or keys)
constexpr int kThreads = 128;
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// byte offset of 16B chunk `c` of row `r` in a [64][64] bf16 swizzled tile
__device__ __forceinline__ uint32_t swz(int r, int c) { return r * 128 + ((c ^ (r & 7)) << 4); }

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

__device__ __forceinline__ void ldsm4(uint32_t* r, uint32_t addr) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm4t(uint32_t* r, uint32_t addr) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}
__device__ __forceinline__ void mma(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ float ex2(float x) {  // MUFU.EX2; ex2(-inf) = 0
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ uint32_t pack(float lo, float hi) {
    __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&h);
}

// Load a [64 rows][64] bf16 tile (row stride `ld` elements) into swizzled smem.
__device__ __forceinline__ void load_tile(uint8_t* s, const __nv_bfloat16* g, int64_t ld, int rows_valid) {
    for (int i = threadIdx.x; i < BR * 8; i += kThreads) {
        const int r = i >> 3, c = i & 7;
        const uint32_t dst = smem_u32(s) + swz(r, c);
        if (r < rows_valid)
            cp_async16(dst, g + r * ld + c * 8);
        else
            *reinterpret_cast<uint4*>(s + swz(r, c)) = make_uint4(0, 0, 0, 0);
    }
}

// A fragments (16 rows x 64) of the warp's slab of a [64][64] tile: a[kk][4]
__device__ __forceinline__ void load_a(uint32_t (*a)[4], const uint8_t* s, int r0) {
    const int t = threadIdx.x & 31;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
        ldsm4(a[kk], smem_u32(s) + swz(r0 + (t & 7) + ((t >> 3) & 1) * 8, kk * 2 + (t >> 4)));
}

// acc[8][4] (+)= A(16x64, regs) * B^T where B is a [64 n][64 k] tile (n-major rows)
__device__ __forceinline__ void mma_abt(float (*acc)[4], uint32_t (*a)[4], const uint8_t* sB) {
    const int t = threadIdx.x & 31;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
#pragma unroll
        for (int np = 0; np < 4; ++np) {
            uint32_t b[4];
            ldsm4(b, smem_u32(sB) + swz(np * 16 + (t & 7) + (t >> 4) * 8, kk * 2 + ((t >> 3) & 1)));
            mma(acc[2 * np], a[kk], b[0], b[1]);
            mma(acc[2 * np + 1], a[kk], b[2], b[3]);
        }
}

// acc[8][4] (+)= P(16 x 64, C-fragment registers) * B where B is a [64 k][64 n] tile (k-major rows)
__device__ __forceinline__ void mma_pb(float (*acc)[4], const float (*p)[4], const uint8_t* sB) {
    const int t = threadIdx.x & 31;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
        uint32_t a[4] = {pack(p[2 * kk][0], p[2 * kk][1]), pack(p[2 * kk][2], p[2 * kk][3]),
                         pack(p[2 * kk + 1][0], p[2 * kk + 1][1]), pack(p[2 * kk + 1][2], p[2 * kk + 1][3])};
#pragma unroll
        for (int np = 0; np < 4; ++np) {
            uint32_t b[4];
            ldsm4t(b, smem_u32(sB) + swz(kk * 16 + (t & 7) + ((t >> 3) & 1) * 8, np * 2 + (t >> 4)));
            mma(acc[2 * np], a, b[0], b[1]);
            mma(acc[2 * np + 1], a, b[2], b[3]);
        }
    }
}

// ------------------------------------------------------------------ forward
__global__ void __launch_bounds__(kThreads) fa_fwd(const __nv_bfloat16* __restrict__ qkv,
                                                   __nv_bfloat16* __restrict__ y, float* __restrict__ lse,
                                                   int T, int H, float scale) {
    ACCO_PDL_PROLOGUE();
    __shared__ __align__(128) uint8_t sQ[BR * 128];
    __shared__ __align__(128) uint8_t sK[2][BR * 128];
    __shared__ __align__(128) uint8_t sV[2][BR * 128];
    const int nqt = (T + BR - 1) / BR;
    const int qt = nqt - 1 - blockIdx.x;  // heavy (late) tiles first
    const int bh = blockIdx.y, b = bh / H, h = bh % H;
    const int d = H * HD;
    const int64_t ld = 3 * d;
    const __nv_bfloat16* base = qkv + static_cast<int64_t>(b) * T * ld;
    const int q0 = qt * BR;
    const int warp = threadIdx.x >> 5, t = threadIdx.x & 31;
    const float sl = scale * kLog2e;

    load_tile(sQ, base + static_cast<int64_t>(q0) * ld + h * HD, ld, min(BR, T - q0));
    load_tile(sK[0], base + d + h * HD, ld, min(BR, T));
    load_tile(sV[0], base + 2 * d + h * HD, ld, min(BR, T));
    cp_commit();

    float o[8][4] = {};
    float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};
    uint32_t qa[4][4];
    const int nkt = qt + 1;
    for (int j = 0; j < nkt; ++j) {
        if (j + 1 < nkt) {
            const int k0 = (j + 1) * BR;
            load_tile(sK[(j + 1) & 1], base + static_cast<int64_t>(k0) * ld + d + h * HD, ld, min(BR, T - k0));
            load_tile(sV[(j + 1) & 1], base + static_cast<int64_t>(k0) * ld + 2 * d + h * HD, ld, min(BR, T - k0));
        }
        cp_commit();
        cp_wait<1>();
        __syncthreads();
        if (j == 0) load_a(qa, sQ, warp * 16);
        float s[8][4] = {};
        mma_abt(s, qa, sK[j & 1]);
        // scale (log2 domain); causal / length mask only on the diagonal tile
        if (j == qt) {
            const int qr = q0 + warp * 16 + (t >> 2);
#pragma unroll
            for (int nt = 0; nt < 8; ++nt)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int key = j * BR + nt * 8 + (t & 3) * 2 + (e & 1);
                    const int q = qr + (e >> 1) * 8;
                    s[nt][e] = (key > q || key >= T) ? -INFINITY : s[nt][e] * sl;
                }
        } else {
#pragma unroll
            for (int nt = 0; nt < 8; ++nt)
#pragma unroll
                for (int e = 0; e < 4; ++e) s[nt][e] *= sl;
        }
#pragma unroll
        for (int hr = 0; hr < 2; ++hr) {
            float mx = m[hr];
#pragma unroll
            for (int nt = 0; nt < 8; ++nt) mx = fmaxf(mx, fmaxf(s[nt][2 * hr], s[nt][2 * hr + 1]));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
            // key 0 is always visible, so mx is finite after the first tile
            const float alpha = ex2(m[hr] - mx);
            m[hr] = mx;
            float rs = 0.f;
#pragma unroll
            for (int nt = 0; nt < 8; ++nt) {
                const float p0 = ex2(s[nt][2 * hr] - mx);
                const float p1 = ex2(s[nt][2 * hr + 1] - mx);
                s[nt][2 * hr] = p0;
                s[nt][2 * hr + 1] = p1;
                rs += p0 + p1;
                o[nt][2 * hr] *= alpha;
                o[nt][2 * hr + 1] *= alpha;
            }
            l[hr] = l[hr] * alpha + rs;
        }
        mma_pb(o, s, sV[j & 1]);
        __syncthreads();
    }
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
        float ls = l[hr];
        ls += __shfl_xor_sync(0xffffffffu, ls, 1);
        ls += __shfl_xor_sync(0xffffffffu, ls, 2);
        const int q = q0 + warp * 16 + (t >> 2) + hr * 8;
        if (q < T) {
            const float inv = 1.f / ls;
            __nv_bfloat16* yr = y + (static_cast<int64_t>(b) * T + q) * d + h * HD;
#pragma unroll
            for (int nt = 0; nt < 8; ++nt)
                *reinterpret_cast<uint32_t*>(yr + nt * 8 + (t & 3) * 2) =
                    pack(o[nt][2 * hr] * inv, o[nt][2 * hr + 1] * inv);
            if ((t & 3) == 0) lse[static_cast<int64_t>(bh) * T + q] = (m[hr] + log2f(ls)) / kLog2e;
        }
    }
}

// ------------------------------------------------------------- backward dK/dV
__global__ void __launch_bounds__(kThreads) fa_bwd_dkv(const __nv_bfloat16* __restrict__ qkv,
                                                       const __nv_bfloat16* __restrict__ dy,
                                                       const float* __restrict__ lse, const float* __restrict__ dsum,
                                                       __nv_bfloat16* __restrict__ dqkv, int T, int H, float scale) {
    ACCO_PDL_PROLOGUE();
    extern __shared__ __align__(128) uint8_t dsm[];  // 49 KB: dynamic
    uint8_t* sK = dsm;
    uint8_t* sV = dsm + BR * 128;
    uint8_t(*sQ)[BR * 128] = reinterpret_cast<uint8_t(*)[BR * 128]>(dsm + 2 * BR * 128);
    uint8_t(*sO)[BR * 128] = reinterpret_cast<uint8_t(*)[BR * 128]>(dsm + 4 * BR * 128);  // dO tiles
    float(*sL)[BR] = reinterpret_cast<float(*)[BR]>(dsm + 6 * BR * 128);
    float(*sD)[BR] = reinterpret_cast<float(*)[BR]>(dsm + 6 * BR * 128 + 2 * BR * 4);
    const int nkt = (T + BR - 1) / BR;
    const int kt = blockIdx.x;
    const int bh = blockIdx.y, b = bh / H, h = bh % H;
    const int d = H * HD;
    const int64_t ld = 3 * d;
    const __nv_bfloat16* base = qkv + static_cast<int64_t>(b) * T * ld;
    const __nv_bfloat16* dyb = dy + static_cast<int64_t>(b) * T * d;
    const int k0 = kt * BR;
    const int warp = threadIdx.x >> 5, t = threadIdx.x & 31;
    const float sl = scale * kLog2e;

    auto load_q = [&](int it, int buf) {
        const int q0 = it * BR;
        load_tile(sQ[buf], base + static_cast<int64_t>(q0) * ld + h * HD, ld, min(BR, T - q0));
        load_tile(sO[buf], dyb + static_cast<int64_t>(q0) * d + h * HD, d, min(BR, T - q0));
        for (int i = threadIdx.x; i < BR; i += kThreads) {
            const int q = q0 + i;
            sL[buf][i] = q < T ? lse[static_cast<int64_t>(bh) * T + q] * kLog2e : 0.f;
            sD[buf][i] = q < T ? dsum[static_cast<int64_t>(bh) * T + q] : 0.f;
        }
    };
    load_tile(sK, base + static_cast<int64_t>(k0) * ld + d + h * HD, ld, min(BR, T - k0));
    load_tile(sV, base + static_cast<int64_t>(k0) * ld + 2 * d + h * HD, ld, min(BR, T - k0));
    load_q(kt, 0);
    cp_commit();

    uint32_t ka[4][4], va[4][4];
    float dk[8][4] = {}, dv[8][4] = {};
    for (int it = kt; it < nkt; ++it) {
        const int buf = (it - kt) & 1;
        if (it + 1 < nkt) load_q(it + 1, buf ^ 1);
        cp_commit();
        cp_wait<1>();
        __syncthreads();
        if (it == kt) {
            load_a(ka, sK, warp * 16);
            load_a(va, sV, warp * 16);
        }
        // S^T = K Q^T (rows: this warp's 16 keys, cols: 64 queries)
        float s[8][4] = {};
        mma_abt(s, ka, sQ[buf]);
        float dp[8][4] = {};
        mma_abt(dp, va, sO[buf]);  // dP^T = V dO^T
        const int kr = k0 + warp * 16 + (t >> 2);
        const bool edge = it == kt || it == nkt - 1;  // diagonal or ragged tail
#pragma unroll
        for (int nt = 0; nt < 8; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int qi = nt * 8 + (t & 3) * 2 + (e & 1);
                float p = ex2(s[nt][e] * sl - sL[buf][qi]);
                if (edge) {
                    const int q = it * BR + qi;
                    const int key = kr + (e >> 1) * 8;
                    if (q < key || q >= T || key >= T) p = 0.f;
                }
                s[nt][e] = p;                                   // P^T
                dp[nt][e] = p * (dp[nt][e] - sD[buf][qi]);      // dS^T
            }
        mma_pb(dv, s, sO[buf]);  // dV += P^T dO
        mma_pb(dk, dp, sQ[buf]); // dK += dS^T Q
        __syncthreads();
    }
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
        const int key = k0 + warp * 16 + (t >> 2) + hr * 8;
        if (key < T) {
            __nv_bfloat16* o = dqkv + (static_cast<int64_t>(b) * T + key) * ld + h * HD;
#pragma unroll
            for (int nt = 0; nt < 8; ++nt) {
                const int c = nt * 8 + (t & 3) * 2;
                *reinterpret_cast<uint32_t*>(o + d + c) = pack(dk[nt][2 * hr] * scale, dk[nt][2 * hr + 1] * scale);
                *reinterpret_cast<uint32_t*>(o + 2 * d + c) = pack(dv[nt][2 * hr], dv[nt][2 * hr + 1]);
            }
        }
    }
}

// ----------------------------------------------------------------- backward dQ
__global__ void __launch_bounds__(kThreads) fa_bwd_dq(const __nv_bfloat16* __restrict__ qkv,
                                                      const __nv_bfloat16* __restrict__ dy,
                                                      const float* __restrict__ lse, const float* __restrict__ dsum,
                                                      __nv_bfloat16* __restrict__ dqkv, int T, int H, float scale) {
    ACCO_PDL_PROLOGUE();
    __shared__ __align__(128) uint8_t sQ[BR * 128];
    __shared__ __align__(128) uint8_t sO[BR * 128];
    __shared__ __align__(128) uint8_t sK[2][BR * 128];
    __shared__ __align__(128) uint8_t sV[2][BR * 128];
    const int nqt = (T + BR - 1) / BR;
    const int qt = nqt - 1 - blockIdx.x;
    const int bh = blockIdx.y, b = bh / H, h = bh % H;
    const int d = H * HD;
    const int64_t ld = 3 * d;
    const __nv_bfloat16* base = qkv + static_cast<int64_t>(b) * T * ld;
    const __nv_bfloat16* dyb = dy + static_cast<int64_t>(b) * T * d;
    const int q0 = qt * BR;
    const int warp = threadIdx.x >> 5, t = threadIdx.x & 31;
    const float sl = scale * kLog2e;

    load_tile(sQ, base + static_cast<int64_t>(q0) * ld + h * HD, ld, min(BR, T - q0));
    load_tile(sO, dyb + static_cast<int64_t>(q0) * d + h * HD, d, min(BR, T - q0));
    load_tile(sK[0], base + d + h * HD, ld, min(BR, T));
    load_tile(sV[0], base + 2 * d + h * HD, ld, min(BR, T));
    cp_commit();
    float L[2], Dv[2];
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
        const int q = q0 + warp * 16 + (t >> 2) + hr * 8;
        L[hr] = q < T ? lse[static_cast<int64_t>(bh) * T + q] * kLog2e : 0.f;
        Dv[hr] = q < T ? dsum[static_cast<int64_t>(bh) * T + q] : 0.f;
    }
    uint32_t qa[4][4], oa[4][4];
    float dq[8][4] = {};
    const int nkt = qt + 1;
    for (int j = 0; j < nkt; ++j) {
        if (j + 1 < nkt) {
            const int k0 = (j + 1) * BR;
            load_tile(sK[(j + 1) & 1], base + static_cast<int64_t>(k0) * ld + d + h * HD, ld, min(BR, T - k0));
            load_tile(sV[(j + 1) & 1], base + static_cast<int64_t>(k0) * ld + 2 * d + h * HD, ld, min(BR, T - k0));
        }
        cp_commit();
        cp_wait<1>();
        __syncthreads();
        if (j == 0) {
            load_a(qa, sQ, warp * 16);
            load_a(oa, sO, warp * 16);
        }
        float s[8][4] = {}, dp[8][4] = {};
        mma_abt(s, qa, sK[j & 1]);
        mma_abt(dp, oa, sV[j & 1]);
        const int qr = q0 + warp * 16 + (t >> 2);
#pragma unroll
        for (int nt = 0; nt < 8; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                float p = ex2(s[nt][e] * sl - L[e >> 1]);
                if (j == qt) {
                    const int key = j * BR + nt * 8 + (t & 3) * 2 + (e & 1);
                    const int q = qr + (e >> 1) * 8;
                    if (key > q || key >= T) p = 0.f;
                }
                s[nt][e] = p * (dp[nt][e] - Dv[e >> 1]);  // dS
            }
        mma_pb(dq, s, sK[j & 1]);  // dQ += dS K
        __syncthreads();
    }
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
        const int q = q0 + warp * 16 + (t >> 2) + hr * 8;
        if (q < T) {
            __nv_bfloat16* o = dqkv + (static_cast<int64_t>(b) * T + q) * ld + h * HD;
#pragma unroll
            for (int nt = 0; nt < 8; ++nt)
                *reinterpret_cast<uint32_t*>(o + nt * 8 + (t & 3) * 2) =
                    pack(dq[nt][2 * hr] * scale, dq[nt][2 * hr + 1] * scale);
        }
    }
}

__global__ void dsum_kernel(const __nv_bfloat16* __restrict__ y, const __nv_bfloat16* __restrict__ dy,
                            float* __restrict__ dsum, int B, int T, int H) {
    ACCO_PDL_PROLOGUE();
    // one warp per (b, h, t) row of 64: D = sum dO * O
    const int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (row >= static_cast<int64_t>(B) * H * T) return;
    const int t = static_cast<int>(row % T);
    const int bh = static_cast<int>(row / T);
    const int b = bh / H, h = bh % H;
    const int64_t o = (static_cast<int64_t>(b) * T + t) * (H * HD) + h * HD + lane * 2;
    const __nv_bfloat162 a = *reinterpret_cast<const __nv_bfloat162*>(y + o);
    const __nv_bfloat162 g = *reinterpret_cast<const __nv_bfloat162*>(dy + o);
    float s = __bfloat162float(a.x) * __bfloat162float(g.x) + __bfloat162float(a.y) * __bfloat162float(g.y);
#pragma unroll
    for (int w = 16; w > 0; w >>= 1) s += __shfl_xor_sync(0xffffffffu, s, w);
    if (lane == 0) dsum[row] = s;
}

bool applicable(const void* p0, const void* p1, int hd) {
    return hd == HD && (reinterpret_cast<uintptr_t>(p0) & 15) == 0 && (reinterpret_cast<uintptr_t>(p1) & 15) == 0;
}

}  // namespace

bool attention_fwd_mma(const __nv_bfloat16* qkv, __nv_bfloat16* y, float* lse, int B, int seq, int H, int hd,
                       cudaStream_t s) {
    if (!applicable(qkv, y, hd)) return false;
    dim3 grid((seq + BR - 1) / BR, B * H);
    launch_pdl(fa_fwd, grid, kThreads, 0, s, qkv, y, lse, seq, H, 1.0f / sqrtf(static_cast<float>(hd)));
    ACCO_CHECK_LAUNCH();
    return true;
}

bool attention_bwd_mma(const __nv_bfloat16* qkv, const __nv_bfloat16* y, const float* lse, const __nv_bfloat16* dy,
                       __nv_bfloat16* dqkv, float* dsum, int B, int seq, int H, int hd, cudaStream_t s) {
    if (!applicable(qkv, dy, hd) || !applicable(y, dqkv, hd)) return false;
    const int64_t rows = static_cast<int64_t>(B) * H * seq;
    launch_pdl(dsum_kernel, static_cast<int>((rows + 7) / 8), 256, 0, s, y, dy, dsum, B, seq, H);
    ACCO_CHECK_LAUNCH();
    const float scale = 1.0f / sqrtf(static_cast<float>(hd));
    dim3 grid((seq + BR - 1) / BR, B * H);
    constexpr int kDkvSmem = 6 * BR * 128 + 4 * BR * 4;
    static bool cfg = false;
    if (!cfg) {
        ACCO_CUDA(cudaFuncSetAttribute(fa_bwd_dkv, cudaFuncAttributeMaxDynamicSharedMemorySize, kDkvSmem));
        cfg = true;
    }
    launch_pdl(fa_bwd_dkv, grid, kThreads, kDkvSmem, s, qkv, dy, lse, dsum, dqkv, seq, H, scale);
    ACCO_CHECK_LAUNCH();
    launch_pdl(fa_bwd_dq, grid, kThreads, 0, s, qkv, dy, lse, dsum, dqkv, seq, H, scale);
    ACCO_CHECK_LAUNCH();
    return true;
}

}  // namespace acco
