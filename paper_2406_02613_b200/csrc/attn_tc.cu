// Causal flash-attention forward on the 5th-generation tensor cores (sm_100a),
// head size 64, bf16 in / fp32 accumulate.
//
// One CTA per (batch*head, 128-query tile), heavy (late) tiles first:
//   warp 0   : TMA producer — Q once, then K_j / V_j 128-key tiles into a
//              2-stage ring (both as [keys][64] rows, 128B-swizzled)
//   warp 1   : MMA issuer — S = Q K_j^T (UMMA 128x128x64, K-major x K-major)
//              into TMEM, then O += P_j V_j (UMMA 128x64x128: P from smem
//              K-major, V as an MN-major B operand) into a TMEM accumulator
//   warp 2   : TMEM allocator (256 columns: S 128 + O 64)
//   warps 4-7: softmax — thread = query row = TMEM lane: tcgen05.ld of the S
//              row, online softmax entirely thread-local (no shuffles), P
//              (bf16) to swizzled smem for the PV MMA. The O rescale is lazy:
//              the running max is only raised when it grows by > 2^8, so O
//              (in TMEM) is rarely touched; final O / l and lse from TMEM.
// S of tile j+1 is issued while the softmax of tile j runs.
#include "common.cuh"

#include <atomic>
#include <cmath>
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>
#include <queue>
#include <numeric>
#include <map>
#include <array>

namespace acco {
namespace {

constexpr int HD = 64;
constexpr int BQ = 128;  // queries per CTA (UMMA M)
constexpr int BKV = 128; // keys per tile (UMMA N of QK^T, K of PV)
constexpr int kStages = 2;
constexpr int kThreads = 384;  // warps 0-3: TMA, MMA, TMEM alloc, idle; 4-11: softmax (2 per TMEM quadrant)
constexpr float kLog2e = 1.4426950408889634f;

// Persistent kernels read their work items from a host-built LPT schedule:
// sched[cta * k_max + k] = k-th item of this CTA (-1 past the end). Items are
// assigned largest-first to the least-loaded CTA (cost = tiles of the item), so
// the heavy diagonal-far items do not pile up on the CTAs that round-robin
// dealing would give them to (GQA dK/dV: 1.56x -> ~1.1x of the mean load).
__device__ __forceinline__ int item_at(const int* __restrict__ sched, int k_max, int k) {
    return k < k_max ? __ldg(sched + static_cast<int64_t>(blockIdx.x) * k_max + k) : -1;
}
// Dynamic alternative (when collectives run beside compute and hold SMs, a
// static table waits for its late CTAs): items in the same heaviest-first
// order, each CTA's producer warp claiming the next one from a per-stream
// counter (list scheduling) and publishing it into the CTA's smem list, one
// item ahead of its own loads (a CTA holds at most two unstarted claims).
// ctr == nullptr: the static table. The last CTA to retire resets ctr.
struct ItemQueue {
    const int* order;  // items, heaviest first
    int n;
    int* ctr;          // [claimed, retired] or nullptr
};
constexpr int kItemQ = 64;  // smem list entries per CTA (the last is always -1)
__device__ __forceinline__ int iq_claim(const ItemQueue& q) {
    const int c = atomicAdd(q.ctr, 1);
    return c < q.n ? __ldg(q.order + c) : -1;
}
#ifdef ACCO_FWD_PROBE  // timeline probe of fa_fwd_tc2 (tools/diag/fwd_probe.cu only)
__device__ unsigned long long g_probe[148][10][128];
#define FWD_PROBE(kind, idx)                                                                     \
    do {                                                                                         \
        unsigned long long _t;                                                                   \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));                                   \
        if ((idx) < 128 && blockIdx.x < 148) g_probe[blockIdx.x][kind][idx] = _t;                \
    } while (0)
#else
#define FWD_PROBE(kind, idx)
#endif
#ifdef ACCO_BWD_PROBE  // timeline probe of fa_bwd_dkv_tc (tools/diag/bwd_probe.cu only)
__device__ unsigned long long g_bprobe[148][8][64];
#define BWD_PROBE(kind, idx)                                                                     \
    do {                                                                                         \
        unsigned long long _t;                                                                   \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));                                   \
        if ((idx) < 64 && blockIdx.x < 148) g_bprobe[blockIdx.x][kind][idx] = _t;                \
    } while (0)
#else
#define BWD_PROBE(kind, idx)
#endif
constexpr float kRescaleThresh = 8.0f;  // log2 domain: rescale O only if the max grows by > 2^8

constexpr int Q_BYTES = BQ * HD * 2;          // 16 KB
constexpr int KV_BYTES = BKV * HD * 2;        // 16 KB per K or V tile
constexpr int P_BYTES = BQ * BKV * 2;         // 32 KB (two 64-key chunks)
constexpr int SMEM = 1024 + Q_BYTES + kStages * 2 * KV_BYTES + P_BYTES + 256 + 4096;  // + row-max/sum exchange

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// A waiting thread is suspended in try_wait (up to this many ns) instead of
// spinning, so waiting warps do not steal issue slots from the softmax warps.
constexpr uint32_t kSuspendNs = 20000;
// Watchdog for mbarrier spins: a pipeline bug becomes a launch error (trap)
// after ~4 s instead of a hung GPU.
__device__ __forceinline__ void watchdog(uint64_t& t0) {
    uint64_t now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    if (t0 == 0) t0 = now;
    else if (now - t0 > 4000000000ull) __trap();
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    uint32_t ok = 0;
    uint32_t spins = 0;
    uint64_t t0 = 0;
    while (!ok) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}\n"
            : "=r"(ok)
            : "r"(a), "r"(parity), "r"(kSuspendNs)
            : "memory");
        if (!ok && (++spins & 255u) == 0) watchdog(t0);
    }
}
// bytes (a multiple of 16, 16 B aligned) global -> shared, completing on bar
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void tc_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void umma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// one lane of a converged warp (the MMA issuers walk their schedule warp-wide so
// descriptors stay in uniform registers; only the elected lane issues)
__device__ __forceinline__ bool elect_one() {
    uint32_t pred;
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "elect.sync _|P, 0xffffffff;\n\t"
        "selp.b32 %0, 1, 0, P;\n\t}\n"
        : "=r"(pred));
    return pred != 0;
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* v) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),
          "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
          "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
        "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
        "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
        "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
        : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(2) << 61;  // SWIZZLE_128B
    return d;
}
__host__ __device__ constexpr uint32_t idesc_bf16(int m, int n, int a_mn, int b_mn) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(a_mn) << 15) |
           (static_cast<uint32_t>(b_mn) << 16) | (static_cast<uint32_t>(n >> 3) << 17) |
           (static_cast<uint32_t>(m >> 4) << 24);
}

__global__ void __launch_bounds__(kThreads, 1)
    fa_fwd_tc(const __grid_constant__ CUtensorMap tmQKV, __nv_bfloat16* __restrict__ y, float* __restrict__ lse,
              int T, int H, int Hkv, float scale) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // 1 KB aligned, still a shared pointer (LDS/STS, not generic LD/ST)
    uint8_t* sQ = smem;
    uint8_t* sK = sQ + Q_BYTES;                       // [stage] K tiles
    uint8_t* sV = sK + kStages * KV_BYTES;            // [stage] V tiles
    uint8_t* sP = sV + kStages * KV_BYTES;            // two 64-key chunks of [128][64] bf16
    uint64_t* bars = reinterpret_cast<uint64_t*>(sP + P_BYTES);
    uint64_t* q_full = bars;
    uint64_t* kv_full = bars + 1;            // [kStages]
    uint64_t* kv_empty = kv_full + kStages;  // [kStages]
    uint64_t* s_full = kv_empty + kStages;
    uint64_t* s_free = s_full + 1;
    uint64_t* p_full = s_free + 1;
    uint64_t* o_done = p_full + 1;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(o_done + 1);

    const int nqt = (T + BQ - 1) / BQ;
    const int qt = nqt - 1 - blockIdx.x;
    const int bh = blockIdx.y, b = bh / H, h = bh % H;
    const int d = H * HD;
    const int ldq = (H + 2 * Hkv) * HD;  // qkv row: H q heads | Hkv k heads | Hkv v heads
    const int kc = d + (h / (H / Hkv)) * HD, vc = kc + Hkv * HD;  // this head's K / V columns
    const int q0 = qt * BQ;
    const int nkt = (min(T, q0 + BQ) + BKV - 1) / BKV;  // causal: key tiles up to the diagonal
    const int row_base = b * T;                          // qkv row of (b, t=0)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        mbar_init(q_full, 1);
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&kv_full[s], 1);
            mbar_init(&kv_empty[s], 1);
        }
        mbar_init(s_full, 1);
        mbar_init(s_free, 256);
        mbar_init(p_full, 256);
        mbar_init(o_done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                     "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_before();
    __syncthreads();
    tc_after();
    const uint32_t tmem = *tslot;
    pdl_trigger();
    pdl_wait();
    const uint32_t tS = tmem, tO = tmem + 128;

    if (warp == 0) {
        if (lane == 0) {
            mbar_expect_tx(q_full, Q_BYTES);
            tma_load_2d(sQ, &tmQKV, q_full, h * HD, row_base + q0);
            for (int j = 0; j < nkt; ++j) {
                const int s = j % kStages;
                mbar_wait(&kv_empty[s], ((j / kStages) & 1) ^ 1);
                mbar_expect_tx(&kv_full[s], 2 * KV_BYTES);
                tma_load_2d(sK + s * KV_BYTES, &tmQKV, &kv_full[s], kc, row_base + j * BKV);
                tma_load_2d(sV + s * KV_BYTES, &tmQKV, &kv_full[s], vc, row_base + j * BKV);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t id_s = idesc_bf16(BQ, BKV, 0, 0);  // Q K^T: both K-major
            constexpr uint32_t id_o = idesc_bf16(BQ, HD, 0, 1);   // P V: P K-major, V MN-major
            const uint32_t q_base = smem_u32(sQ), p_base = smem_u32(sP);
            mbar_wait(q_full, 0);
            auto issue_s = [&](int j) {
                const int s = j % kStages;
                mbar_wait(&kv_full[s], (j / kStages) & 1);
                tc_after();
                const uint32_t k_base = smem_u32(sK + s * KV_BYTES);
#pragma unroll
                for (int kk = 0; kk < HD / 16; ++kk)
                    umma(tS, sdesc(q_base + kk * 32, 16, 1024), sdesc(k_base + kk * 32, 16, 1024), id_s, kk > 0);
                umma_commit(s_full);
            };
            issue_s(0);
            for (int j = 0; j < nkt; ++j) {
                const int s = j % kStages;
                if (j + 1 < nkt) {
                    mbar_wait(s_free, j & 1);  // softmax has S_j in registers
                    tc_after();
                    issue_s(j + 1);
                }
                mbar_wait(p_full, j & 1);  // P_j in smem (and O rescaled if needed)
                tc_after();
                const uint32_t v_base = smem_u32(sV + s * KV_BYTES);
#pragma unroll
                for (int kk = 0; kk < BKV / 16; ++kk) {
                    const uint64_t ad = sdesc(p_base + (kk >> 2) * (BQ * 128) + (kk & 3) * 32, 16, 1024);
                    const uint64_t bd = sdesc(v_base + kk * 2048, 64 * 128, 1024);
                    umma(tO, ad, bd, id_o, (j > 0 || kk > 0) ? 1u : 0u);
                }
                umma_commit(&kv_empty[s]);
                umma_commit(o_done);
            }
        }
    } else if (warp >= 4) {
        // 8 softmax warps: quadrant wq (TMEM lanes) x half (64 of the 128 keys,
        // 32 of the 64 O columns); the row max is combined with the partner warp
        const int wq = warp & 3, half = (warp - 4) >> 2;
        const int r = wq * 32 + lane;  // query row within the tile = TMEM lane
        const int q = q0 + r;
        const uint32_t lane_off = static_cast<uint32_t>(wq * 32) << 16;
        const float sl = scale * kLog2e;
        float* red = reinterpret_cast<float*>(tslot + 4);  // [2 parity][2 half][128] row maxima
        float m = -INFINITY, l = 0.f;
        for (int j = 0; j < nkt; ++j) {
            mbar_wait(s_full, j & 1);
            tc_after();
            uint32_t sr[64];  // this half of the S row, scaled in place (log2 domain)
            tmem_ld32(tS + lane_off + half * 64, sr);
            tmem_ld32(tS + lane_off + half * 64 + 32, sr + 32);
            tmem_wait_ld();
            tc_before();
            mbar_arrive(s_free);  // S TMEM may be overwritten by the next QK^T
            const bool diag = (j + 1) * BKV > q0;  // tile touching the causal edge (or T tail)
            float mx = m;
#pragma unroll
            for (int i = 0; i < 64; ++i) {
                float x = __uint_as_float(sr[i]) * sl;
                if (diag) {
                    const int key = j * BKV + half * 64 + i;
                    if (key > q || key >= T) x = -INFINITY;
                }
                sr[i] = __float_as_uint(x);
                mx = fmaxf(mx, x);
            }
            float* rb = red + (j & 1) * 256;
            rb[half * 128 + r] = mx;
            asm volatile("bar.sync %0, 64;" ::"r"(2 + wq) : "memory");  // the quadrant's two warps
            mx = fmaxf(mx, rb[(1 - half) * 128 + r]);
            // lazy rescale: raise the running max only when it grows by > 2^8
            const bool need = mx > m + kRescaleThresh;
            const float alpha = need ? ex2(m - mx) : 1.f;
            if (need) m = mx;
            l *= alpha;
            if (j > 0) {
                mbar_wait(o_done, (j - 1) & 1);  // PV_{j-1} finished: O stable, P buffer free
                tc_after();
            }
            // P = 2^(s - m) -> bf16, swizzled K-major into this half's 64-key chunk
            float rs = 0.f;
#pragma unroll
            for (int unit = 0; unit < 8; ++unit) {
                float p[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    p[k] = ex2(__uint_as_float(sr[unit * 8 + k]) - m);
                    rs += p[k];
                }
                uint4 u;
                __nv_bfloat162 h0 = __floats2bfloat162_rn(p[0], p[1]), h1 = __floats2bfloat162_rn(p[2], p[3]);
                __nv_bfloat162 h2 = __floats2bfloat162_rn(p[4], p[5]), h3 = __floats2bfloat162_rn(p[6], p[7]);
                u.x = *reinterpret_cast<uint32_t*>(&h0);
                u.y = *reinterpret_cast<uint32_t*>(&h1);
                u.z = *reinterpret_cast<uint32_t*>(&h2);
                u.w = *reinterpret_cast<uint32_t*>(&h3);
                *reinterpret_cast<uint4*>(sP + half * (BQ * 128) + r * 128 + ((unit ^ (r & 7)) << 4)) = u;
            }
            l += rs;
            // O *= alpha for rows whose max moved (warp-collective TMEM access, 32 of 64 columns)
            if (j > 0 && __any_sync(0xffffffffu, need)) {
                uint32_t o[32];
                tmem_ld32(tO + lane_off + half * 32, o);
                tmem_wait_ld();
#pragma unroll
                for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
                tmem_st32(tO + lane_off + half * 32, o);
                tmem_wait_st();
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            tc_before();
            mbar_arrive(p_full);
        }
        // epilogue: O / l (l = both halves' partial sums), lse
        float* lb = red + 512;
        lb[half * 128 + r] = l;
        asm volatile("bar.sync %0, 64;" ::"r"(2 + wq) : "memory");
        l += lb[(1 - half) * 128 + r];
        mbar_wait(o_done, (nkt - 1) & 1);
        tc_after();
        uint32_t o[32];
        tmem_ld32(tO + lane_off + half * 32, o);
        tmem_wait_ld();
        if (q < T) {
            const float inv = 1.f / l;
            __nv_bfloat16* yr = y + (static_cast<int64_t>(b) * T + q) * d + h * HD + half * 32;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                uint4 u;
                __nv_bfloat162 h0 = __floats2bfloat162_rn(__uint_as_float(o[8 * c + 0]) * inv, __uint_as_float(o[8 * c + 1]) * inv);
                __nv_bfloat162 h1 = __floats2bfloat162_rn(__uint_as_float(o[8 * c + 2]) * inv, __uint_as_float(o[8 * c + 3]) * inv);
                __nv_bfloat162 h2 = __floats2bfloat162_rn(__uint_as_float(o[8 * c + 4]) * inv, __uint_as_float(o[8 * c + 5]) * inv);
                __nv_bfloat162 h3 = __floats2bfloat162_rn(__uint_as_float(o[8 * c + 6]) * inv, __uint_as_float(o[8 * c + 7]) * inv);
                u.x = *reinterpret_cast<uint32_t*>(&h0);
                u.y = *reinterpret_cast<uint32_t*>(&h1);
                u.z = *reinterpret_cast<uint32_t*>(&h2);
                u.w = *reinterpret_cast<uint32_t*>(&h3);
                reinterpret_cast<uint4*>(yr)[c] = u;
            }
            if (half == 0) lse[static_cast<int64_t>(bh) * T + q] = (m + log2f(l)) / kLog2e;
        }
    }
    tc_before();
    __syncthreads();
    if (warp == 2) {
        tc_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
    }
}

// ------------------------------------------------- forward, two-tile ping-pong
// One CTA per (batch*head, pair of adjacent 128-query tiles 2p, 2p+1), heavy
// pairs first. Both tiles share every K/V tile they both need (keys up to
// tile 2p), loaded once. Two softmax groups (warps 4-7: tile 2p, warps 8-11:
// tile 2p+1), thread = query row = TMEM lane, own the S/P and O of their tile
// in TMEM. P never leaves TMEM: it is written (bf16 pairs) over the consumed
// S columns and fed to O += P V as the A operand from tensor memory. The MMA
// warp interleaves the tiles, so the tensor core runs one tile's PV / next QK^T
// while the other tile's softmax runs:
//     S0(0) S1(0) | [P0] PV0(0) S0(1) | [P1] PV1(0) S1(1) | [P0] PV0(1) S0(2) ...
// Row sums accumulate in fp32 with packed f32x2 adds (sm_100), so lse stays
// consistent with the fp32 P the backward recomputes.
__device__ __forceinline__ void st_row32_global_fwd(__nv_bfloat16* dst, const uint32_t* o, float scale) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        uint4 u;
        __nv_bfloat162 h0 = __floats2bfloat162_rn(__uint_as_float(o[8 * c + 0]) * scale, __uint_as_float(o[8 * c + 1]) * scale);
        __nv_bfloat162 h1 = __floats2bfloat162_rn(__uint_as_float(o[8 * c + 2]) * scale, __uint_as_float(o[8 * c + 3]) * scale);
        __nv_bfloat162 h2 = __floats2bfloat162_rn(__uint_as_float(o[8 * c + 4]) * scale, __uint_as_float(o[8 * c + 5]) * scale);
        __nv_bfloat162 h3 = __floats2bfloat162_rn(__uint_as_float(o[8 * c + 6]) * scale, __uint_as_float(o[8 * c + 7]) * scale);
        u.x = *reinterpret_cast<uint32_t*>(&h0);
        u.y = *reinterpret_cast<uint32_t*>(&h1);
        u.z = *reinterpret_cast<uint32_t*>(&h2);
        u.w = *reinterpret_cast<uint32_t*>(&h3);
        reinterpret_cast<uint4*>(dst)[c] = u;
    }
}

// Head size D = 64 or 128. Tiles of D > 64 columns are D / 64 TMA boxes of
// 64 columns (SW128 sub-tiles 16 KB apart); D = 128 keeps one item slot of Q
// and a 2-stage K/V ring to fit shared memory.
template <int D>
struct Fwd2 {
    static constexpr int QB = BQ * D * 2, KVB = BKV * D * 2;
    static constexpr int STAGES = D == 64 ? 3 : 2, QSLOTS = D == 64 ? 2 : 1;
    // + per tile slot: row-max exchange [2 parity][2 half][128] and row sums [2 half][128]
    static constexpr int SMEM = 1024 + QSLOTS * 2 * QB + STAGES * 2 * KVB + 256 + 2 * 6 * 128 * 4;
};
// two softmax groups of 8 warps (one per tile slot): quadrant x half of the 128 keys
constexpr int F2_THREADS = 640;
// a [128 rows][D] bf16 tile as D / 64 boxes of 64 columns, 16 KB apart
template <int D>
__device__ __forceinline__ void tma_tile(void* dst, const CUtensorMap* map, uint64_t* bar, int col, int row) {
#pragma unroll
    for (int sub = 0; sub < D / 64; ++sub) tma_load_2d(static_cast<uint8_t*>(dst) + sub * 16384, map, bar, col + 64 * sub, row);
}
// K-major descriptor of 16-deep k-slice kk of such a tile
__device__ __forceinline__ uint64_t kslice(uint64_t desc, int kk) { return desc + (kk >> 2) * (16384 >> 4) + (kk & 3) * 2; }

__device__ __forceinline__ void umma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
        "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
        "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}

__device__ __forceinline__ float max3(float a, float b, float c) {
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));  // FMNMX3
    return r;
}
// Max of 64 S values (columns base..base+63 of the tile); MASK: columns >= lim
// are outside the causal window / sequence.
template <bool MASK>
__device__ __forceinline__ float row_max64(const uint32_t* sv, int base, int lim, float mx) {
#pragma unroll
    for (int i = 0; i < 64; i += 2) {
        float x0 = __uint_as_float(sv[i]), x1 = __uint_as_float(sv[i + 1]);
        if (MASK) {
            x0 = base + i < lim ? x0 : -INFINITY;
            x1 = base + i + 1 < lim ? x1 : -INFINITY;
        }
        mx = max3(mx, x0, x1);
    }
    return mx;
}
// P = 2^(s * sl - m) for 64 S values -> 32 packed bf16 pairs; row sum in l2.
template <bool MASK>
__device__ __forceinline__ void exp_pack64(const uint32_t* sv, float sl, float m, int base, int lim, float2& l2,
                                           uint32_t* pk) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
        const float2 xs = fma_f32x2(make_float2(__uint_as_float(sv[2 * i]), __uint_as_float(sv[2 * i + 1])),
                                    make_float2(sl, sl), make_float2(-m, -m));
        float p0 = ex2(xs.x), p1 = ex2(xs.y);
        if (MASK) {
            p0 = base + 2 * i < lim ? p0 : 0.f;
            p1 = base + 2 * i + 1 < lim ? p1 : 0.f;
        }
        l2 = add_f32x2(l2, make_float2(p0, p1));
        __nv_bfloat162 hb = __floats2bfloat162_rn(p0, p1);
        pk[i] = *reinterpret_cast<uint32_t*>(&hb);
    }
}

// Persistent two-tile forward: grid = #SMs; work item = (pair of 128-query
// tiles, batch*head), heaviest pairs first, dealt round-robin. Within an item
// the two tiles share every K/V load and ping-pong on the tensor core (the
// MMAs of one tile run under the other's softmax). Q is double-buffered
// across items and the K/V ring, S/P, O barriers run over the CTA's whole
// tile sequence, so CTA launch / TMEM alloc / pipeline fill are paid once per
// SM. TMEM: S/P tile 0 [0,128), S/P tile 1 [128,256), O tile 0 [256,320),
// O tile 1 [320,384).
template <int D>
__global__ void __launch_bounds__(F2_THREADS, 1)
    fa_fwd_tc2(const __grid_constant__ CUtensorMap tmQKV, __nv_bfloat16* __restrict__ y, float* __restrict__ lse,
               int B, int T, int H, int Hkv, float scale, const int* __restrict__ sched, int sk, ItemQueue iq) {
    __shared__ uint64_t q_ready[kItemQ];
    __shared__ int q_list[kItemQ];
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // 1 KB aligned, still a shared pointer (LDS/STS, not generic LD/ST)
    constexpr int Q_BYTES = Fwd2<D>::QB, KV_BYTES = Fwd2<D>::KVB, F2_STAGES = Fwd2<D>::STAGES,
                  QSLOTS = Fwd2<D>::QSLOTS;
    uint8_t* sQ = smem;                         // [QSLOTS items][2 tiles]
    uint8_t* sK = sQ + QSLOTS * 2 * Q_BYTES;    // [stage]
    uint8_t* sV = sK + F2_STAGES * KV_BYTES;    // [stage]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sV + F2_STAGES * KV_BYTES);
    uint64_t* q_full = bars;                     // [item slots] (2 reserved)
    uint64_t* q_empty = bars + 2;                // [item slots] (2 reserved)
    uint64_t* kv_full = bars + 4;                // [F2_STAGES]
    uint64_t* kv_empty = kv_full + F2_STAGES;    // [F2_STAGES]
    uint64_t* s_full = kv_empty + F2_STAGES;     // [2 tiles]
    uint64_t* p_full = s_full + 2;               // [2 tiles]
    uint64_t* o_done = p_full + 2;               // [2 tiles]
    uint64_t* s_free = o_done + 2;               // [2 tiles] (SEPP) S in the softmax warps' registers
    uint64_t* pv_done = s_free + 2;              // [2 tiles] (SEPP) PV done: P and O free
    uint32_t* tslot = reinterpret_cast<uint32_t*>(pv_done + 2);
    // SEPP (D = 64): P in its own TMEM columns [384 + 64 x, +64) instead of over
    // S, so S(j + 1) is issued as soon as the softmax warps hold S(j) in
    // registers instead of after PV(j) (D = 128: O takes those columns)
    constexpr bool SEPP = D == 64;

    const int nqt = (T + BQ - 1) / BQ;
    const int npair = (nqt + 1) / 2;
    const int nbh = B * H;
    const int n_items = npair * nbh;
    const int d = H * D;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    struct Item {
        int pr, b, h, kc, vc, nt0, nt1, nkv;
    };
    auto item_of = [&](int u) {
        Item w;
        w.pr = npair - 1 - u / nbh;  // heavy pairs first
        const int bh = u % nbh;
        w.b = bh / H;
        w.h = bh % H;
        w.kc = d + (w.h / (H / Hkv)) * D;  // this head's K / V columns
        w.vc = w.kc + Hkv * D;
        w.nt0 = 2 * w.pr + 1;                               // kv tiles of query tile 0
        w.nt1 = 2 * w.pr + 2 <= nqt ? 2 * w.pr + 2 : 0;     // of query tile 1 (0: absent)
        w.nkv = w.nt1 ? w.nt1 : w.nt0;
        return w;
    };

    if (threadIdx.x == 0) {
        for (int q = 0; q < kItemQ; ++q) mbar_init(&q_ready[q], 1);
        for (int s = 0; s < 2; ++s) {
            mbar_init(&q_full[s], 1);
            mbar_init(&q_empty[s], 1);
        }
        for (int s = 0; s < F2_STAGES; ++s) {
            mbar_init(&kv_full[s], 1);
            mbar_init(&kv_empty[s], 1);
        }
        for (int x = 0; x < 2; ++x) {
            mbar_init(&s_full[x], 1);
            mbar_init(&p_full[x], 256);
            mbar_init(&o_done[x], 1);
            mbar_init(&s_free[x], 256);
            mbar_init(&pv_done[x], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_before();
    __syncthreads();
    tc_after();
    const uint32_t tmem = *tslot;
    pdl_trigger();
    pdl_wait();
    // the item sequence of this CTA: the static LPT table, or the dynamic queue
    // (q_list filled by the producer warp, q_ready[k] completes when entry k is in)
    // static tables are copied to q_list once (a global load per item start
    // stalled every warp on a memory round trip before its first tile)
    const bool st_smem = !iq.ctr && sk <= kItemQ;
    if (st_smem) {
        for (int k = threadIdx.x; k < sk; k += blockDim.x) q_list[k] = item_at(sched, sk, k);
        __syncthreads();
    }
    auto citem = [&](int k) -> int {
        if (st_smem) return k < sk ? q_list[k] : -1;
        if (!iq.ctr) return item_at(sched, sk, k);
        if (k >= kItemQ) return -1;
        mbar_wait(&q_ready[k], 0);
        return *reinterpret_cast<volatile int*>(&q_list[k]);
    };
    // producer warp: publish entry k + 1 as item k starts (claimed during item
    // k - 1), claim for entry k + 2; entry kItemQ - 1 is always the end marker
    int q_pend = -1;
    auto q_publish = [&](int k, int u) {
        q_list[k] = u;
        mbar_arrive(&q_ready[k]);
    };
    auto q_retire = [&]() {  // after the end marker: no claim of this CTA is left; the last CTA resets
        if (atomicAdd(iq.ctr + 1, 1) == static_cast<int>(gridDim.x) - 1) {
            atomicExch(iq.ctr, 0);
            atomicExch(iq.ctr + 1, 0);
        }
    };
    auto q_start = [&]() {  // producer lane 0, before the first item
        const int c0 = iq_claim(iq);
        q_publish(0, c0);
        q_pend = c0 >= 0 ? iq_claim(iq) : -1;
        if (c0 < 0) q_retire();
    };
    auto q_next = [&](int k) {  // producer lane 0, as item k starts
        const int nx = k + 1 <= kItemQ - 2 ? q_pend : -1;
        q_publish(k + 1, nx);
        q_pend = nx >= 0 && k + 2 <= kItemQ - 2 ? iq_claim(iq) : -1;
        if (nx < 0) q_retire();
    };

    if (warp == 0) {
        {  // warp-wide walk and waits, one elected lane issues
            int kvit = 0, ni = 0;
            if (iq.ctr) {  // dynamic queue: entry 0 (and the claim for entry 1)
                if (lane == 0) q_start();
                __syncwarp();
            }
            for (int k = 0, u = citem(0); u >= 0; ++ni, u = citem(++k)) {
                if (iq.ctr) {  // publish entry k + 1 as item k starts
                    if (lane == 0) q_next(k);
                    __syncwarp();
                }
                const Item w = item_of(u);
                const int row_base = w.b * T;
                const int qs = ni % QSLOTS;
                mbar_wait(&q_empty[qs], ((ni / QSLOTS) & 1) ^ 1);  // item ni-QSLOTS's S MMAs are done with this slot
                if (elect_one()) {
                    mbar_expect_tx(&q_full[qs], (w.nt1 ? 2 : 1) * Q_BYTES);
                    uint8_t* q_dst = sQ + qs * 2 * Q_BYTES;
                    tma_tile<D>(q_dst, &tmQKV, &q_full[qs], w.h * D, row_base + 2 * w.pr * BQ);
                    if (w.nt1) tma_tile<D>(q_dst + Q_BYTES, &tmQKV, &q_full[qs], w.h * D, row_base + (2 * w.pr + 1) * BQ);
                }
                __syncwarp();
                for (int j = 0; j < w.nkv; ++j, ++kvit) {
                    const int s = kvit % F2_STAGES;
                    mbar_wait(&kv_empty[s], ((kvit / F2_STAGES) & 1) ^ 1);
                    if (elect_one()) {
                        mbar_expect_tx(&kv_full[s], 2 * KV_BYTES);
                        tma_tile<D>(sK + s * KV_BYTES, &tmQKV, &kv_full[s], w.kc, row_base + j * BKV);
                        tma_tile<D>(sV + s * KV_BYTES, &tmQKV, &kv_full[s], w.vc, row_base + j * BKV);
                    }
                    __syncwarp();
                }
            }
        }
    } else if (warp == 1) {
        // warp-wide walk and waits, one elected lane issues (it shares its SM
        // sub-partition with four softmax warps: keep its instruction count low)
        constexpr uint32_t id_s = idesc_bf16(BQ, BKV, 0, 0);  // Q K^T: both K-major
        constexpr uint32_t id_o = idesc_bf16(BQ, D, 0, 1);    // P V: P from TMEM (K-major), V MN-major
        int kvit = 0, ni = 0;
        int cnt[2] = {0, 0};  // tiles issued so far per slot (s_full / p_full phases)
        int pc_s = 0, pc_pv = 0;
        (void)pc_s;
        (void)pc_pv;
        for (int k = 0, u = citem(0); u >= 0; ++ni, u = citem(++k)) {
            const Item w = item_of(u);
            const int nt[2] = {w.nt0, w.nt1};
            const int qs = ni % QSLOTS;
            mbar_wait(&q_full[qs], (ni / QSLOTS) & 1);
            const uint32_t q_item = smem_u32(sQ + qs * 2 * Q_BYTES);
            auto issue_s = [&](int x, int j) {
                const int s = (kvit + j) % F2_STAGES;
                if (SEPP && cnt[x] + j > 0) {  // the softmax warps hold the slot's previous S
                    mbar_wait(&s_free[x], (cnt[x] + j - 1) & 1);
                    tc_after();
                }
                if (x == 0 || !nt[0] || j >= nt[0]) {  // first user of K_j waits for it
                    mbar_wait(&kv_full[s], ((kvit + j) / F2_STAGES) & 1);
                    tc_after();
                }
                if (lane == 0) FWD_PROBE(0, pc_s);
                ++pc_s;
                // K-major: the 16-deep k slices are 32 B apart inside the 128B swizzle row
                const uint64_t qd = sdesc(q_item + x * Q_BYTES, 16, 1024), kd = sdesc(smem_u32(sK + s * KV_BYTES), 16, 1024);
                if (elect_one()) {
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk)
                        umma(tmem + x * 128, kslice(qd, kk), kslice(kd, kk), id_s, kk > 0);
                    umma_commit(&s_full[x]);
                }
                __syncwarp();
            };
            auto issue_pv = [&](int x, int j) {
                const int s = (kvit + j) % F2_STAGES;
                mbar_wait(&p_full[x], (cnt[x] + j) & 1);
                tc_after();
                if (lane == 0) FWD_PROBE(1, pc_pv);
                ++pc_pv;
                // V MN-major: 16-key slices are two 8-row atoms (2048 B) apart
                // (N = D: 64-wide MN atoms, one 16 KB sub-tile apart)
                const uint64_t vd = sdesc(smem_u32(sV + s * KV_BYTES), D == 64 ? 64 * 128 : 16384, 1024);
                const uint32_t tp = SEPP ? tmem + 384 + x * 64 : tmem + x * 128;
                if (elect_one()) {
#pragma unroll
                    for (int kk = 0; kk < BKV / 16; ++kk)
                        umma_ts(tmem + 256 + x * D, tp + kk * 8, vd + 128 * kk, id_o, (j > 0 || kk > 0) ? 1u : 0u);
                    if (SEPP) umma_commit(&pv_done[x]);
                }
                __syncwarp();
            };
            issue_s(0, 0);
            if (nt[1]) issue_s(1, 0);
            for (int j = 0; j < w.nkv; ++j) {
                for (int x = 0; x < 2; ++x) {
                    if (j >= nt[x]) continue;
                    if (SEPP && j + 1 < nt[x]) issue_s(x, j + 1);  // under this tile's softmax
                    issue_pv(x, j);
                    if (!SEPP && j + 1 < nt[x]) {
                        issue_s(x, j + 1);
                    } else if (j + 1 >= nt[x]) {
                        if (elect_one()) umma_commit(&o_done[x]);
                        __syncwarp();
                    }
                }
                if (elect_one()) {
                    if (j + 1 == w.nkv) umma_commit(&q_empty[qs]);  // every S of the item issued
                    umma_commit(&kv_empty[(kvit + j) % F2_STAGES]);  // both tiles' PV_j issued
                }
                __syncwarp();
            }
            kvit += w.nkv;
            cnt[0] += nt[0];
            cnt[1] += nt[1];
        }
    } else if (warp >= 4) {
        // two groups of 8 softmax warps, one per tile slot x; in a group, warp
        // (quadrant wq, half) owns TMEM lanes wq*32.. and keys half*64..+63 of
        // each S tile (and O columns half*32..+31): the row max is exchanged with
        // the partner warp through smem, and P (bf16 pairs) lands on packed
        // columns half*32.. after both halves have read their S
        const int x = (warp - 4) >> 3;
        const int wq = warp & 3, half = ((warp - 4) >> 2) & 1;
        const int r = wq * 32 + lane;
        const uint32_t lane_off = static_cast<uint32_t>(wq * 32) << 16;
        const uint32_t tS = tmem + x * 128 + lane_off, tO = tmem + 256 + x * D + lane_off;
        constexpr int OH = D / 2;  // O columns per half warp pair
        const float sl = scale * kLog2e;
        float* red = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(tslot) + 16) + x * 6 * 128;  // [2][2][128] max
        float* lsum = red + 4 * 128;                                                                  // [2][128] sums
        const int bar_id = 2 + x * 4 + wq;  // the quadrant's two warps
        int cnt = 0, nitem = 0;  // tiles / items this slot has processed (barrier phases)
        for (int k = 0, u = citem(0); u >= 0; u = citem(++k)) {
            const Item w = item_of(u);
            const int n = x == 0 ? w.nt0 : w.nt1;
            if (n == 0) continue;  // absent tile (odd tile count): no phases consumed
            const int q = (2 * w.pr + x) * BQ + r;
            float m = -INFINITY;
            float2 l2 = make_float2(0.f, 0.f);  // fp32 partial row sum over this half's keys
            for (int j = 0; j < n; ++j) {
                mbar_wait(&s_full[x], (cnt + j) & 1);
                tc_after();
                if (lane == 0 && wq == 0 && half == 0) FWD_PROBE(2 + 2 * x, cnt + j);
                const bool diag = j == n - 1;  // the causal edge (and any ragged tail) sits in the last tile
                const int kbase = j * BKV;
                const int lim = min(q + 1, T) - kbase;  // valid keys of this row: [kbase, kbase + lim)
                uint32_t sv[64];
                tmem_ld32(tS + half * 64, sv);
                tmem_ld32(tS + half * 64 + 32, sv + 32);
                tmem_wait_ld();
                if (SEPP) {  // S(j + 1) may land now
                    tc_before();
                    mbar_arrive(&s_free[x]);
                }
                if (lane == 0 && wq == 0 && half == 0 && x == 0) FWD_PROBE(6, cnt + j);
                float mx = diag ? row_max64<true>(sv, half * 64, lim, -INFINITY)
                                : row_max64<false>(sv, half * 64, lim, -INFINITY);
                float* rb = red + (j & 1) * 256;
                rb[half * 128 + r] = mx;
                asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");  // both halves have read S
                if (lane == 0 && wq == 0 && half == 0 && x == 0) FWD_PROBE(7, cnt + j);
                mx = fmaxf(mx, rb[(1 - half) * 128 + r]) * sl;
                // lazy rescale: move the reference max only when it grows by > 2^8;
                // O is stable once PV(j-1) is done (!SEPP: s_full(j) is committed
                // after it; SEPP: pv_done, waited below before O or P is touched)
                bool need = false;
                float alpha = 1.f;
                if (j == 0) {
                    m = mx;
                } else {
                    need = mx > m + kRescaleThresh;
                    alpha = need ? ex2(m - mx) : 1.f;
                    if (need) m = mx;
                    l2.x *= alpha;
                    l2.y *= alpha;
                }
                // P = 2^(s - m) -> bf16 pairs on packed columns half*32.. (over S columns
                // both halves have already read: the barrier above)
                {
                    uint32_t pk[32];
                    if (diag)
                        exp_pack64<true>(sv, sl, m, half * 64, lim, l2, pk);
                    else
                        exp_pack64<false>(sv, sl, m, half * 64, lim, l2, pk);
                    if (lane == 0 && wq == 0 && half == 0 && x == 0) FWD_PROBE(8, cnt + j);
                    if (SEPP && cnt + j > 0) {  // PV(j-1) has read P and updated O
                        mbar_wait(&pv_done[x], (cnt + j - 1) & 1);
                        tc_after();
                    }
                    const uint32_t tPk = SEPP ? tmem + 384 + x * 64 + lane_off : tS;
                    tmem_st16(tPk + half * 32, pk);
                    tmem_st16(tPk + half * 32 + 16, pk + 16);
                }
                // O *= alpha where the max moved (before this tile's PV, which waits p_full)
                if (__any_sync(0xffffffffu, need)) {  // tcgen05.ld/st are warp-collective
#pragma unroll
                    for (int c = 0; c < OH / 32; ++c) {
                        uint32_t o[32];
                        tmem_ld32(tO + half * OH + c * 32, o);
                        tmem_wait_ld();
#pragma unroll
                        for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
                        tmem_st32(tO + half * OH + c * 32, o);
                    }
                }
                tmem_wait_st();
                if (lane == 0 && wq == 0 && half == 0 && x == 0) FWD_PROBE(9, cnt + j);
                tc_before();
                mbar_arrive(&p_full[x]);
                if (lane == 0 && wq == 0 && half == 0) FWD_PROBE(3 + 2 * x, cnt + j);
            }
            cnt += n;
            // epilogue: O / l, l = both halves' partial sums (fp32: lse stays consistent
            // with the fp32 P of the backward)
            lsum[half * 128 + r] = l2.x + l2.y;
            asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");
            const float l = lsum[0 * 128 + r] + lsum[1 * 128 + r];
            mbar_wait(&o_done[x], nitem & 1);
            ++nitem;
            tc_after();
            const float inv = 1.f / l;
            __nv_bfloat16* yr = y + (static_cast<int64_t>(w.b) * T + q) * d + w.h * D + half * OH;
#pragma unroll
            for (int c = 0; c < OH / 32; ++c) {
                uint32_t o[32];
                tmem_ld32(tO + half * OH + c * 32, o);  // warp-collective: every lane loads
                tmem_wait_ld();
                if (q < T) st_row32_global_fwd(yr + c * 32, o, inv);
            }
            tc_before();
            if (q < T && half == 0) lse[(static_cast<int64_t>(w.b) * H + w.h) * T + q] = (m + log2f(l)) / kLog2e;
            asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory");  // lsum reusable
        }
    }
    tc_before();
    __syncthreads();
    if (warp == 2) {
        tc_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

// ---- backward softmax helpers (masking hoisted out of the unrolled loops)
// p[c] = 2^(s_c * sl - lse[c] * log2 e) for 32 columns; MASK: columns outside
// [lo, hi) -> 0 (dK/dV: thread = key, columns = queries)
template <bool MASK>
__device__ __forceinline__ void exp_cols32(const uint32_t* st, const float4* L4, float sl, int base, int lo, int hi,
                                           float* p) {
#pragma unroll
    for (int c4 = 0; c4 < 8; ++c4) {
        const float4 l4 = L4[c4];
        const float2 a = fma_f32x2(make_float2(__uint_as_float(st[4 * c4]), __uint_as_float(st[4 * c4 + 1])),
                                   make_float2(sl, sl), make_float2(-(l4.x * kLog2e), -(l4.y * kLog2e)));
        const float2 b = fma_f32x2(make_float2(__uint_as_float(st[4 * c4 + 2]), __uint_as_float(st[4 * c4 + 3])),
                                   make_float2(sl, sl), make_float2(-(l4.z * kLog2e), -(l4.w * kLog2e)));
        float v[4] = {ex2(a.x), ex2(a.y), ex2(b.x), ex2(b.y)};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int c = base + 4 * c4 + e;
            if (MASK) v[e] = (c >= lo && c < hi) ? v[e] : 0.f;
            p[4 * c4 + e] = v[e];
        }
    }
}
// p[c] = 2^(s_c * sl - L) for 64 columns (dQ: thread = query, columns = keys);
// MASK: columns >= lim -> 0
template <bool MASK, int N = 64>
__device__ __forceinline__ void exp_row64(const uint32_t* st, float sl, float L, int lim, float* p) {
#pragma unroll
    for (int c = 0; c < N; c += 2) {
        const float2 a = fma_f32x2(make_float2(__uint_as_float(st[c]), __uint_as_float(st[c + 1])),
                                   make_float2(sl, sl), make_float2(-L, -L));
        float p0 = ex2(a.x), p1 = ex2(a.y);
        if (MASK) {
            p0 = c < lim ? p0 : 0.f;
            p1 = c + 1 < lim ? p1 : 0.f;
        }
        p[c] = p0;
        p[c + 1] = p1;
    }
}
// ds[c] = p[c] * (dp[c] - D[c]) with packed f32x2 math
__device__ __forceinline__ void ds_pairs(const float* p, const uint32_t* dp, const float* D, int n, float* ds) {
#pragma unroll
    for (int c = 0; c < n; c += 2) {
        const float2 t = fma_f32x2(make_float2(__uint_as_float(dp[c]), __uint_as_float(dp[c + 1])), make_float2(1.f, 1.f),
                                   make_float2(-D[c], -D[c + 1]));
        const float2 r = fma_f32x2(make_float2(p[c], p[c + 1]), t, make_float2(0.f, 0.f));
        ds[c] = r.x;
        ds[c + 1] = r.y;
    }
}

// ----------------------------------------------------------------- backward
// A [128 rows][128] bf16 tile written by threads (thread = row) as a K-major
// UMMA A operand = two 64-column chunks of [128][128B], SW128.
// One 64-column chunk (8 x 16B units) of such a tile: row r of chunk `chunk`.
__device__ __forceinline__ void st_row64_chunk(uint8_t* buf, int chunk, int r, const float* v) {
#pragma unroll
    for (int unit = 0; unit < 8; ++unit) {
        __nv_bfloat162 h0 = __floats2bfloat162_rn(v[8 * unit + 0], v[8 * unit + 1]);
        __nv_bfloat162 h1 = __floats2bfloat162_rn(v[8 * unit + 2], v[8 * unit + 3]);
        __nv_bfloat162 h2 = __floats2bfloat162_rn(v[8 * unit + 4], v[8 * unit + 5]);
        __nv_bfloat162 h3 = __floats2bfloat162_rn(v[8 * unit + 6], v[8 * unit + 7]);
        uint4 u;
        u.x = *reinterpret_cast<uint32_t*>(&h0);
        u.y = *reinterpret_cast<uint32_t*>(&h1);
        u.z = *reinterpret_cast<uint32_t*>(&h2);
        u.w = *reinterpret_cast<uint32_t*>(&h3);
        *reinterpret_cast<uint4*>(buf + chunk * (128 * 128) + r * 128 + ((unit ^ (r & 7)) << 4)) = u;
    }
}
// Half of such a 64-column chunk: units 4*part .. 4*part+3 (32 columns)
__device__ __forceinline__ void st_row32_part(uint8_t* buf, int chunk, int r, int part, const float* v) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const int unit = 4 * part + k;
        __nv_bfloat162 h0 = __floats2bfloat162_rn(v[8 * k + 0], v[8 * k + 1]);
        __nv_bfloat162 h1 = __floats2bfloat162_rn(v[8 * k + 2], v[8 * k + 3]);
        __nv_bfloat162 h2 = __floats2bfloat162_rn(v[8 * k + 4], v[8 * k + 5]);
        __nv_bfloat162 h3 = __floats2bfloat162_rn(v[8 * k + 6], v[8 * k + 7]);
        uint4 u;
        u.x = *reinterpret_cast<uint32_t*>(&h0);
        u.y = *reinterpret_cast<uint32_t*>(&h1);
        u.z = *reinterpret_cast<uint32_t*>(&h2);
        u.w = *reinterpret_cast<uint32_t*>(&h3);
        *reinterpret_cast<uint4*>(buf + chunk * (128 * 128) + r * 128 + ((unit ^ (r & 7)) << 4)) = u;
    }
}
// K-major A descriptor for k-step kk (16 columns) of such a tile
__device__ __forceinline__ uint64_t a128_desc(uint32_t base, int kk) {
    return sdesc(base + (kk >> 2) * (128 * 128) + (kk & 3) * 32, 16, 1024);
}
// Store 32 floats of a thread's row (scaled) as bf16 to global (64 B contiguous)
__device__ __forceinline__ void st_row32_global(__nv_bfloat16* dst, const uint32_t* o, float scale) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        __nv_bfloat162 h0 = __floats2bfloat162_rn(__uint_as_float(o[8 * c + 0]) * scale, __uint_as_float(o[8 * c + 1]) * scale);
        __nv_bfloat162 h1 = __floats2bfloat162_rn(__uint_as_float(o[8 * c + 2]) * scale, __uint_as_float(o[8 * c + 3]) * scale);
        __nv_bfloat162 h2 = __floats2bfloat162_rn(__uint_as_float(o[8 * c + 4]) * scale, __uint_as_float(o[8 * c + 5]) * scale);
        __nv_bfloat162 h3 = __floats2bfloat162_rn(__uint_as_float(o[8 * c + 6]) * scale, __uint_as_float(o[8 * c + 7]) * scale);
        uint4 u;
        u.x = *reinterpret_cast<uint32_t*>(&h0);
        u.y = *reinterpret_cast<uint32_t*>(&h1);
        u.z = *reinterpret_cast<uint32_t*>(&h2);
        u.w = *reinterpret_cast<uint32_t*>(&h3);
        reinterpret_cast<uint4*>(dst)[c] = u;
    }
}

constexpr int BW_T = 128;                          // tile rows (keys or queries)
// backward kernels: warps 0-3 (TMA, MMA, TMEM alloc, idle) + 16 softmax warps
// (4 per TMEM lane quadrant, 32 columns each): the per-element chain
// (TMEM load -> ex2 -> dS -> bf16 smem) is latency-bound at 2 warps per
// scheduler, so 4 per scheduler keep the issue slots busy
constexpr int BW_THREADS = 640;
constexpr int BW_SOFTMAX = 512;
constexpr int BW_SQ = BW_T * BW_T * 2;             // 32 KB [128][128] bf16 (P / dS operand)
// dKV smem: K, V (KVS item slots) + DKV_ST stages x (Q, dO, lse | D of the
// stage's 128 queries). D = 64: K/V double-buffered (the next item's K/V under the current
// item), a 4-deep Q/dO ring. D = 128: one K/V slot, a 2-deep ring, and TMEM
// S^T | dP^T | dV | dK (128 columns each) with P^T / dS^T (bf16) written over
// the consumed S^T / dP^T columns, so the next tile's S^T / dP^T are issued
// after this tile's dV / dK MMAs (in-order tensor pipe).
template <int D>
struct Dkv {
    static constexpr int TILE = BW_T * D * 2, ST = D == 64 ? 4 : 2, KVS = D == 64 ? 2 : 1;
    static constexpr bool P_IN_S = D > 64;
    static constexpr int SMEM = 1024 + KVS * 2 * TILE + ST * 2 * TILE + ST * 2 * BW_T * 4 + 256 + 64;
};

// dK/dV, persistent: grid = #SMs; work item = (128-key tile kt, batch * KV
// head), heaviest key tiles first (kt = 0 sees every query tile), dealt
// round-robin. Per item the CTA loops over the query tiles at and after the
// diagonal of each of the G = H / Hkv query heads of the group (GQA; G = 1 for
// MHA). Per query tile:
//   S^T = K Q^T, dP^T = V dO^T          (TMEM, 128 x 128 each)
//   softmax-bwd warps (thread = key row): P^T = 2^(S^T sl - lse2[q]),
//   dS^T = P^T (dP^T - D[q])  -> bf16 smem operands
//   dV += P^T dO, dK += dS^T Q          (TMEM, 128 x 64 each; Q/dO MN-major B)
// Barrier phases run over the CTA's global tile sequence, so the next item's
// K/V load and first S^T/dP^T overlap the current item's last tile and the
// dK/dV epilogue; a CTA launch + TMEM alloc + pipeline fill is paid once per SM
// instead of once per item (it was ~7 us of a ~100 us kernel per wave).
template <int D>
__global__ void __launch_bounds__(BW_THREADS, 1)
    fa_bwd_dkv_tc(const __grid_constant__ CUtensorMap tmQKV, const __grid_constant__ CUtensorMap tmDO,
                  const float* __restrict__ lse, const float* __restrict__ dsum, __nv_bfloat16* __restrict__ dqkv,
                  int B, int T, int H, int Hkv, float scale, const int* __restrict__ sched, int sk, ItemQueue iq) {
    __shared__ uint64_t q_ready[kItemQ];
    __shared__ int q_list[kItemQ];
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // 1 KB aligned, still a shared pointer (LDS/STS, not generic LD/ST)
    constexpr int BW_TILE = Dkv<D>::TILE, DKV_ST = Dkv<D>::ST, KVS = Dkv<D>::KVS;
    constexpr bool P_IN_S = Dkv<D>::P_IN_S;
    uint8_t* sK = smem;                    // [KVS items]
    uint8_t* sV = sK + KVS * BW_TILE;      // [KVS items]
    uint8_t* sQ = sV + KVS * BW_TILE;      // [DKV_ST stages]
    uint8_t* sO = sQ + DKV_ST * BW_TILE;   // dO [DKV_ST stages]
    // per stage: lse | D of the stage's 128 queries (float4 broadcasts to the softmax warps)
    float* sLD = reinterpret_cast<float*>(sO + DKV_ST * BW_TILE);  // [DKV_ST][lse 128 | D 128]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sLD + DKV_ST * 2 * BW_T);
    uint64_t* kv_full = bars;                 // [KVS] (2 reserved)
    uint64_t* kv_empty = bars + 2;            // [KVS]: every S^T/dP^T MMA of the item issued and done
    uint64_t* q_full = bars + 4;              // [DKV_ST]
    uint64_t* q_empty = q_full + DKV_ST;      // [DKV_ST]
    uint64_t* s_full = q_empty + DKV_ST;      // S^T and dP^T ready
    uint64_t* s_free = s_full + 1;            // softmax has them in registers
    uint64_t* p_full = s_free + 1;            // P^T, dS^T (bf16) in TMEM
    uint64_t* g_done = p_full + 1;            // dV/dK MMAs of this tile done (operands free)
    uint32_t* tslot = reinterpret_cast<uint32_t*>(g_done + 1);

    const int nt = (T + BW_T - 1) / BW_T;
    const int nbk = B * Hkv;
    const int n_items = nt * nbk;
    const int G = H / Hkv;
    const int d = H * D;
    const int ldq = (H + 2 * Hkv) * D;  // qkv row: H q heads | Hkv k heads | Hkv v heads
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    struct Item {
        int kt, b, hk, nq;
    };
    auto item_of = [&](int u) {  // u < n_items: kt ascending = heaviest first
        Item w;
        w.kt = u / nbk;
        const int bk = u % nbk;
        w.b = bk / Hkv;
        w.hk = bk % Hkv;
        w.nq = nt - w.kt;  // query tiles kt .. nt-1 per query head
        return w;
    };

    // lse / D rows move as two bulk copies per stage when every row start is
    // 16 B aligned; the columns past T then keep older (finite) values, which
    // the mask zeroes (the ring starts zeroed)
    const bool lse_bulk = (T & 3) == 0;
    for (int k = threadIdx.x; k < DKV_ST * 2 * BW_T; k += blockDim.x) sLD[k] = 0.f;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x == 0) {
        for (int q = 0; q < kItemQ; ++q) mbar_init(&q_ready[q], 1);
        for (int s = 0; s < 2; ++s) {
            mbar_init(&kv_full[s], 1);
            mbar_init(&kv_empty[s], 1);
        }
        for (int s = 0; s < DKV_ST; ++s) {
            // the TMA expect_tx (+ each producer lane's lse / D copies when T % 4 != 0)
            mbar_init(&q_full[s], lse_bulk ? 1 : 1 + 32);
            mbar_init(&q_empty[s], 1);
        }
        mbar_init(s_full, 1);
        mbar_init(s_free, BW_SOFTMAX);
        mbar_init(p_full, BW_SOFTMAX);
        mbar_init(g_done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_before();
    __syncthreads();
    tc_after();
    const uint32_t tmem = *tslot;
    pdl_trigger();
    pdl_wait();
    // the item sequence of this CTA: the static LPT table, or the dynamic queue
    // (q_list filled by the producer warp, q_ready[k] completes when entry k is in)
    // static tables are copied to q_list once (a global load per item start
    // stalled every warp on a memory round trip before its first tile)
    const bool st_smem = !iq.ctr && sk <= kItemQ;
    if (st_smem) {
        for (int k = threadIdx.x; k < sk; k += blockDim.x) q_list[k] = item_at(sched, sk, k);
        __syncthreads();
    }
    auto citem = [&](int k) -> int {
        if (st_smem) return k < sk ? q_list[k] : -1;
        if (!iq.ctr) return item_at(sched, sk, k);
        if (k >= kItemQ) return -1;
        mbar_wait(&q_ready[k], 0);
        return *reinterpret_cast<volatile int*>(&q_list[k]);
    };
    // producer warp: publish entry k + 1 as item k starts (claimed during item
    // k - 1), claim for entry k + 2; entry kItemQ - 1 is always the end marker
    int q_pend = -1;
    auto q_publish = [&](int k, int u) {
        q_list[k] = u;
        mbar_arrive(&q_ready[k]);
    };
    auto q_retire = [&]() {  // after the end marker: no claim of this CTA is left; the last CTA resets
        if (atomicAdd(iq.ctr + 1, 1) == static_cast<int>(gridDim.x) - 1) {
            atomicExch(iq.ctr, 0);
            atomicExch(iq.ctr + 1, 0);
        }
    };
    auto q_start = [&]() {  // producer lane 0, before the first item
        const int c0 = iq_claim(iq);
        q_publish(0, c0);
        q_pend = c0 >= 0 ? iq_claim(iq) : -1;
        if (c0 < 0) q_retire();
    };
    auto q_next = [&](int k) {  // producer lane 0, as item k starts
        const int nx = k + 1 <= kItemQ - 2 ? q_pend : -1;
        q_publish(k + 1, nx);
        q_pend = nx >= 0 && k + 2 <= kItemQ - 2 ? iq_claim(iq) : -1;
        if (nx < 0) q_retire();
    };
    // TMEM: S^T | dP^T (fp32, 128 cols each) | dV | dK (64 each) | P^T | dS^T
    // (bf16 pairs, 64 cols each): the dV/dK MMAs take A straight from TMEM, so
    // P^T/dS^T never touch shared memory, and S^T/dP^T of the next tile can
    // land while dV/dK of this one still read P^T/dS^T
    // (D = 128: dV | dK 128 columns each, P^T / dS^T over S^T / dP^T)
    const uint32_t tS = tmem, tP = tmem + 128, tDV = tmem + 256, tDK = tmem + 256 + D,
                   tPT = P_IN_S ? tS : tmem + 384, tDST = P_IN_S ? tP : tmem + 448;

    if (warp == 0) {
        {  // warp-wide walk and waits, one elected lane issues
            int it = 0, ni = 0;
            if (iq.ctr) {  // dynamic queue: entry 0 (and the claim for entry 1)
                if (lane == 0) q_start();
                __syncwarp();
            }
            for (int k = 0, u = citem(0); u >= 0; ++ni, u = citem(++k)) {
                if (iq.ctr) {  // publish entry k + 1 as item k starts
                    if (lane == 0) q_next(k);
                    __syncwarp();
                }
                const Item w = item_of(u);
                const int kc = d + w.hk * D, vc = kc + Hkv * D;
                const int row_base = w.b * T;
                const int kb = ni % KVS;
                mbar_wait(&kv_empty[kb], ((ni / KVS) & 1) ^ 1);  // item ni-KVS's S^T/dP^T MMAs are done with it
                if (elect_one()) {
                    mbar_expect_tx(&kv_full[kb], 2 * BW_TILE);
                    tma_tile<D>(sK + kb * BW_TILE, &tmQKV, &kv_full[kb], kc, row_base + w.kt * BW_T);
                    tma_tile<D>(sV + kb * BW_TILE, &tmQKV, &kv_full[kb], vc, row_base + w.kt * BW_T);
                }
                __syncwarp();
                const int niter = G * w.nq;
                for (int i = 0; i < niter; ++i, ++it) {
                    const int s = it % DKV_ST;
                    const int h = w.hk * G + i / w.nq;
                    const int q0 = (w.kt + i % w.nq) * BW_T;
                    mbar_wait(&q_empty[s], ((it / DKV_ST) & 1) ^ 1);
                    // lse | D of the 128 queries next to Q / dO, completing on the same
                    // barrier: the softmax warps issue no loads and wait on nothing else
                    const int64_t bh = static_cast<int64_t>(w.b) * H + h;
                    float* dl = sLD + s * 2 * BW_T;
                    if (elect_one()) {
                        const uint32_t nb = static_cast<uint32_t>(min(BW_T, T - q0)) * 4u;
                        mbar_expect_tx(&q_full[s], 2 * BW_TILE + (lse_bulk ? 2 * nb : 0u));
                        tma_tile<D>(sQ + s * BW_TILE, &tmQKV, &q_full[s], h * D, row_base + q0);
                        tma_tile<D>(sO + s * BW_TILE, &tmDO, &q_full[s], h * D, row_base + q0);
                        if (lse_bulk) {
                            bulk_g2s(dl, lse + bh * T + q0, nb, &q_full[s]);
                            bulk_g2s(dl + BW_T, dsum + bh * T + q0, nb, &q_full[s]);
                        }
                    }
                    if (!lse_bulk) {  // 4 B copies, zero-filling the columns past T
#pragma unroll
                        for (int t = 0; t < BW_T / 32; ++t) {
                            const int j = t * 32 + lane, q = q0 + j;
                            const uint32_t n = q < T ? 4u : 0u;
                            const int64_t off = q < T ? bh * T + q : 0;
                            asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(dl + j)),
                                         "l"(lse + off), "r"(n) : "memory");
                            asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(dl + BW_T + j)),
                                         "l"(dsum + off), "r"(n) : "memory");
                        }
                        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&q_full[s]))
                                     : "memory");
                    }
                    __syncwarp();
                }
            }
        }
    } else if (warp == 1) {
        // warp-wide walk and waits, one elected lane issues (see fa_fwd_tc2);
        // descriptors are built once per operand tile and stepped per 16-deep slice
        constexpr uint32_t id_s = idesc_bf16(BW_T, BW_T, 0, 0);  // K Q^T / V dO^T
        constexpr uint32_t id_g = idesc_bf16(BW_T, D, 0, 1);     // P^T dO / dS^T Q (B MN-major)
        auto issue_s = [&](int g, int kb) {  // S^T = K Q_g^T, dP^T = V dO_g^T (global tile g, K/V slot kb)
            const int s = g % DKV_ST;
            mbar_wait(&q_full[s], (g / DKV_ST) & 1);
            tc_after();
            const uint64_t kd = sdesc(smem_u32(sK + kb * BW_TILE), 16, 1024), vd = sdesc(smem_u32(sV + kb * BW_TILE), 16, 1024);
            const uint64_t qd = sdesc(smem_u32(sQ + s * BW_TILE), 16, 1024), od = sdesc(smem_u32(sO + s * BW_TILE), 16, 1024);
            if (lane == 0) BWD_PROBE(0, g);
            if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) {  // K-major: 32 B per slice (sub-tiles of 64 columns)
                    umma(tS, kslice(kd, kk), kslice(qd, kk), id_s, kk > 0);
                    umma(tP, kslice(vd, kk), kslice(od, kk), id_s, kk > 0);
                }
                umma_commit(s_full);
            }
            __syncwarp();
        };
        int it = 0, ni = 0;
        if (citem(0) >= 0) {
            mbar_wait(&kv_full[0], 0);
            issue_s(0, 0);
        }
        for (int k = 0, u = citem(0); u >= 0; ++ni, u = citem(++k)) {
            const Item w = item_of(u);
            const int niter = G * w.nq;
            const int kb = ni % KVS;
            const bool more = citem(k + 1) >= 0;
            for (int i = 0; i < niter; ++i) {
                const int g = it + i;
                const int s = g % DKV_ST;
                // MN-major B: 16-query slices are two 8-row atoms (2048 B) apart;
                // N = D: 64-wide atoms one 16 KB sub-tile apart
                const uint64_t qd = sdesc(smem_u32(sQ + s * BW_TILE), D == 64 ? 64 * 128 : 16384, 1024);
                const uint64_t od = sdesc(smem_u32(sO + s * BW_TILE), D == 64 ? 64 * 128 : 16384, 1024);
                // the next tile's S^T/dP^T (possibly the next item's first, whose
                // K/V is already in the other slot): D = 64 under this tile's
                // softmax (its S^T/dP^T columns are free once read), D = 128 after
                // this tile's dV/dK MMAs (which read P^T/dS^T from those columns)
                auto next_s = [&](bool wait_free) {
                    if (i + 1 < niter) {
                        if (wait_free) mbar_wait(s_free, g & 1);
                        tc_after();
                        issue_s(g + 1, kb);
                    } else {
                        if (elect_one()) umma_commit(&kv_empty[kb]);  // every S^T/dP^T of this item issued
                        __syncwarp();
                        if (more) {
                            mbar_wait(&kv_full[(ni + 1) % KVS], ((ni + 1) / KVS) & 1);
                            if (wait_free) mbar_wait(s_free, g & 1);
                            tc_after();
                            issue_s(g + 1, (ni + 1) % KVS);
                        }
                    }
                };
                if (!P_IN_S) next_s(true);
                mbar_wait(p_full, g & 1);  // P^T / dS^T written
                tc_after();
                if (lane == 0) BWD_PROBE(1, g);
                if (elect_one()) {
#pragma unroll
                    for (int kk = 0; kk < BW_T / 16; ++kk) {  // 16 queries = 8 packed TMEM columns per step
                        umma_ts(tDV, tPT + kk * 8, od + 128 * kk, id_g, (i > 0 || kk > 0) ? 1u : 0u);
                        umma_ts(tDK, tDST + kk * 8, qd + 128 * kk, id_g, (i > 0 || kk > 0) ? 1u : 0u);
                    }
                    umma_commit(&q_empty[s]);
                    umma_commit(g_done);
                }
                __syncwarp();
                if (P_IN_S) next_s(false);
            }
            it += niter;
        }
#ifdef ACCO_BWD_PROBE
    } else if (warp == 3) {  // observer (diagnostic builds only): when each tile's S^T/dP^T completes
        int it = 0;
        for (int k = 0, u = citem(0); u >= 0; u = citem(++k)) {
            const Item w = item_of(u);
            const int niter = G * w.nq;
            for (int i = 0; i < niter; ++i) {
                mbar_wait(s_full, (it + i) & 1);
                if (lane == 0) BWD_PROBE(7, it + i);
            }
            it += niter;
        }
#endif
    } else if (warp >= 4) {
        // 16 warps: quadrant wq (key rows = TMEM lanes) x quarter qq (32 of 128 queries)
        const int wq = warp & 3, qq = (warp - 4) >> 2;
        const int r = wq * 32 + lane;  // key row = TMEM lane
        const uint32_t lane_off = static_cast<uint32_t>(wq * 32) << 16;
        const float sl = scale * kLog2e;
        // dK/dV of item `prev` leave TMEM -> global: deferred into the next
        // item's first tile (after its exp/dS math, which overlaps the item's
        // last dV/dK MMAs), or after the loop for the CTA's last item
        int prev = -1;
        auto epilogue = [&](int pu) {
            const Item w = item_of(pu);
            const int key = w.kt * BW_T + r;
            const int kc = d + w.hk * D, vc = kc + Hkv * D;
            __nv_bfloat16* dst = dqkv + (static_cast<int64_t>(w.b) * T + key) * ldq;
            if (D == 64) {  // quarters 0/1: dV columns, 2/3: dK columns (32 each)
                uint32_t o[32];
                tmem_ld32((qq < 2 ? tDV : tDK) + lane_off + (qq & 1) * 32, o);
                tmem_wait_ld();
                if (key < T) st_row32_global(dst + (qq < 2 ? vc : kc) + (qq & 1) * 32, o, qq < 2 ? 1.f : scale);
            } else {  // quarter qq: dV and dK columns qq*32 ..
#pragma unroll
                for (int t = 0; t < 2; ++t) {
                    uint32_t o[32];
                    tmem_ld32((t ? tDK : tDV) + lane_off + qq * 32, o);
                    tmem_wait_ld();
                    if (key < T) st_row32_global(dst + (t ? kc : vc) + qq * 32, o, t ? scale : 1.f);
                }
            }
        };
        int it = 0;
        for (int k = 0, u = citem(0); u >= 0; u = citem(++k)) {
            const Item w = item_of(u);
            const int niter = G * w.nq;
            const int k0 = w.kt * BW_T;
            const int key = k0 + r;
            for (int i = 0; i < niter; ++i) {
                const int g = it + i;
                const int qi = i % w.nq;
                const int q0 = (w.kt + qi) * BW_T;
                if (warp == 4 && lane == 0) BWD_PROBE(2, g);
                mbar_wait(s_full, g & 1);
                tc_after();
                // this tile's lse / D arrived with its Q / dO (stage g % DKV_ST; the
                // phase completed before the S^T MMAs were issued)
                const int st_ = g % DKV_ST;
                mbar_wait(&q_full[st_], (g / DKV_ST) & 1);
                const float* cur = sLD + st_ * 2 * BW_T + qq * 32;
                if (warp == 4 && lane == 0) BWD_PROBE(3, g);
                // masked tiles: the diagonal (q >= key) and a ragged tail (q < T; the
                // rows past T belong to the next sequence)
                const bool edge = qi == 0 || q0 + BW_T > T;
                const float4* L4 = reinterpret_cast<const float4*>(cur);  // lse (natural log: x kLog2e at use)
                const float4* D4 = reinterpret_cast<const float4*>(cur + BW_T);
                {
                    // S^T and dP^T (this warp's 32 columns each) go to registers first
                    // and their TMEM is released at once, so the MMA warp computes the
                    // next tile's S^T / dP^T under this tile's exp / dS math
                    uint32_t st[32], dp[32];
#ifndef ACCO_DIAG_DKV_NO_TMEM
                    tmem_ld32(tS + lane_off + qq * 32, st);
                    tmem_ld32(tP + lane_off + qq * 32, dp);
                    tmem_wait_ld();
#else  // diagnostic builds only (tools/diag/attn_bench.cu): what bounds the tile
#pragma unroll
                    for (int c = 0; c < 32; ++c) st[c] = dp[c] = 0u;
#endif
                    tc_before();
                    mbar_arrive(s_free);
                    float* p = reinterpret_cast<float*>(st);  // in place
                    // valid query columns c of this quarter: q0 + qq*32 + c in [key, T)
                    const int lo = key - (q0 + qq * 32), hi = T - (q0 + qq * 32);
                    float* ds = reinterpret_cast<float*>(dp);  // dS^T = P^T (dP^T - D), in place
#ifndef ACCO_DIAG_DKV_NO_MATH
                    if (edge)
                        exp_cols32<true>(st, L4, sl, 0, lo, hi, p);
                    else
                        exp_cols32<false>(st, L4, sl, 0, lo, hi, p);
                    ds_pairs(p, dp, reinterpret_cast<const float*>(D4), 32, ds);
#endif
                    uint32_t pk[16], dk[16];  // bf16 pairs: query 2c (low) and 2c+1 (high)
#pragma unroll
                    for (int c = 0; c < 16; ++c) {
                        __nv_bfloat162 a = __floats2bfloat162_rn(p[2 * c], p[2 * c + 1]);
                        __nv_bfloat162 e = __floats2bfloat162_rn(ds[2 * c], ds[2 * c + 1]);
                        pk[c] = *reinterpret_cast<uint32_t*>(&a);
                        dk[c] = *reinterpret_cast<uint32_t*>(&e);
                    }
                    if (warp == 4 && lane == 0) BWD_PROBE(4, g);
                    if (g > 0) {  // the previous dV/dK MMAs have read P^T / dS^T
                        mbar_wait(g_done, (g - 1) & 1);
                        tc_after();
                    }
                    if (warp == 4 && lane == 0) BWD_PROBE(5, g);
                    if (i == 0 && prev >= 0) {  // previous item's accumulators are final
                        epilogue(prev);
                        prev = -1;
                    }
                    // (D = 128: P^T / dS^T go over S^T / dP^T columns other warps read:
                    // every softmax thread has them in registers once s_free completes)
                    if (P_IN_S) mbar_wait(s_free, g & 1);
#ifndef ACCO_DIAG_DKV_NO_TMEM
                    tmem_st16(tPT + lane_off + qq * 16, pk);
                    tmem_st16(tDST + lane_off + qq * 16, dk);
                    tmem_wait_st();
#endif
                }
                tc_before();
                mbar_arrive(p_full);
                if (warp == 4 && lane == 0) BWD_PROBE(6, g);
            }
            it += niter;
            prev = u;
        }
        if (prev >= 0) {
            mbar_wait(g_done, (it - 1) & 1);
            tc_after();
            epilogue(prev);
        }
    }
    tc_before();
    __syncthreads();
    if (warp == 2) {
        tc_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

// dQ, persistent: grid = #SMs; work item = (128-query tile qt, batch*head),
// heaviest (last) query tiles first, dealt round-robin. Per item: loop over
// the key tiles up to the diagonal: S = Q K^T, dP = dO V^T (TMEM); thread =
// query row: P, dS -> smem; dQ += dS K (K as MN-major B). Q/dO are
// double-buffered across items and the next item's first S/dP is issued
// under the current item's last tile (barrier phases follow the CTA's global
// tile sequence), so CTA launch / TMEM alloc / pipeline fill are paid once.
// head size D = 64 or 128: D = 128 keeps one item slot of Q / dO and a 2-deep
// K/V ring (shared memory)
// With fuse_d the kernel also loads the item's O tile and computes D =
// rowsum(dO o O) for its 128 queries itself (written to dsum for the dK/dV
// kernel, which then runs after it): the separate D pass over O and dO
// (25 MB at GPT-2 small, ~6 us per layer) is gone.
template <int D>
struct Dq {
    static constexpr int TILE = BW_T * D * 2, ST = D == 64 ? 4 : 2, QS = D == 64 ? 2 : 1;
    static constexpr int SMEM = 1024 + QS * 3 * TILE + ST * 2 * TILE + 256 + 64;
};
// D of query row r from K-major SW128 tiles of dO and O ([128 rows][128 B]
// sub-tiles of 64 columns, 16 B unit u of row r at (u ^ (r & 7)) << 4):
// columns in order, one fp32 FMA chain
template <int D>
__device__ __forceinline__ float row_dot_sw128(const uint8_t* a, const uint8_t* b, int r) {
    float acc = 0.f;
#pragma unroll
    for (int sub = 0; sub < D / 64; ++sub)
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int off = sub * (BW_T * 128) + r * 128 + ((u ^ (r & 7)) << 4);
            const uint4 x = *reinterpret_cast<const uint4*>(a + off), y = *reinterpret_cast<const uint4*>(b + off);
            const uint32_t xw[4] = {x.x, x.y, x.z, x.w}, yw[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                acc = fmaf(__uint_as_float(xw[k] << 16), __uint_as_float(yw[k] << 16), acc);
                acc = fmaf(__uint_as_float(xw[k] & 0xffff0000u), __uint_as_float(yw[k] & 0xffff0000u), acc);
            }
        }
    return acc;
}

template <int D>
__global__ void __launch_bounds__(BW_THREADS, 1)
    fa_bwd_dq_tc(const __grid_constant__ CUtensorMap tmQKV, const __grid_constant__ CUtensorMap tmDO,
                 const __grid_constant__ CUtensorMap tmY, const float* __restrict__ lse, float* __restrict__ dsum,
                 __nv_bfloat16* __restrict__ dqkv, int B, int T, int H, int Hkv, float scale,
                 const int* __restrict__ sched, int sk, ItemQueue iq, int fuse_d) {
    __shared__ uint64_t q_ready[kItemQ];
    __shared__ int q_list[kItemQ];
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // 1 KB aligned, still a shared pointer (LDS/STS, not generic LD/ST)
    constexpr int BW_TILE = Dq<D>::TILE, DQ_ST = Dq<D>::ST, QS = Dq<D>::QS;
    uint8_t* sQ = smem;                   // [QS items]
    uint8_t* sO = sQ + QS * BW_TILE;      // dO [QS items]
    uint8_t* sY = sO + QS * BW_TILE;      // O [QS items] (fuse_d)
    uint8_t* sK = sY + QS * BW_TILE;      // [DQ_ST stages]
    uint8_t* sV = sK + DQ_ST * BW_TILE;   // [DQ_ST stages]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sV + DQ_ST * BW_TILE);
    uint64_t* q_full = bars;               // [QS] (2 reserved)
    uint64_t* q_empty = bars + 2;          // [QS] (2 reserved)
    uint64_t* kv_full = bars + 4;          // [DQ_ST]
    uint64_t* kv_empty = kv_full + DQ_ST;  // [DQ_ST]
    uint64_t* s_full = kv_empty + DQ_ST;
    uint64_t* s_free = s_full + 1;
    uint64_t* p_full = s_free + 1;
    uint64_t* g_done = p_full + 1;
    uint64_t* d_free = g_done + 1;  // [2] (fuse_d) the softmax warps have read dO / O of the slot
    uint32_t* tslot = reinterpret_cast<uint32_t*>(d_free + 2);

    const int nt = (T + BW_T - 1) / BW_T;
    const int nbh = B * H;
    const int n_items = nt * nbh;
    const int d = H * D;
    const int ldq = (H + 2 * Hkv) * D;  // qkv row: H q heads | Hkv k heads | Hkv v heads
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    struct Item {
        int qt, b, h, nk, kc, vc;
    };
    auto item_of = [&](int u) {  // heaviest (last) query tiles first
        Item w;
        w.qt = nt - 1 - u / nbh;
        const int bh = u % nbh;
        w.b = bh / H;
        w.h = bh % H;
        w.nk = w.qt + 1;  // key tiles 0 .. qt
        w.kc = d + (w.h / (H / Hkv)) * D;  // this head's K / V columns
        w.vc = w.kc + Hkv * D;
        return w;
    };

    if (threadIdx.x == 0) {
        for (int q = 0; q < kItemQ; ++q) mbar_init(&q_ready[q], 1);
        for (int s = 0; s < 2; ++s) {
            mbar_init(&q_full[s], 1);
            mbar_init(&q_empty[s], 1);
        }
        for (int s = 0; s < DQ_ST; ++s) {
            mbar_init(&kv_full[s], 1);
            mbar_init(&kv_empty[s], 1);
        }
        mbar_init(s_full, 1);
        mbar_init(s_free, BW_SOFTMAX);
        mbar_init(p_full, BW_SOFTMAX);
        mbar_init(g_done, 1);
        mbar_init(&d_free[0], BW_SOFTMAX);
        mbar_init(&d_free[1], BW_SOFTMAX);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_before();
    __syncthreads();
    tc_after();
    const uint32_t tmem = *tslot;
    pdl_trigger();
    pdl_wait();
    // the item sequence of this CTA: the static LPT table, or the dynamic queue
    // (q_list filled by the producer warp, q_ready[k] completes when entry k is in)
    // static tables are copied to q_list once (a global load per item start
    // stalled every warp on a memory round trip before its first tile)
    const bool st_smem = !iq.ctr && sk <= kItemQ;
    if (st_smem) {
        for (int k = threadIdx.x; k < sk; k += blockDim.x) q_list[k] = item_at(sched, sk, k);
        __syncthreads();
    }
    auto citem = [&](int k) -> int {
        if (st_smem) return k < sk ? q_list[k] : -1;
        if (!iq.ctr) return item_at(sched, sk, k);
        if (k >= kItemQ) return -1;
        mbar_wait(&q_ready[k], 0);
        return *reinterpret_cast<volatile int*>(&q_list[k]);
    };
    // producer warp: publish entry k + 1 as item k starts (claimed during item
    // k - 1), claim for entry k + 2; entry kItemQ - 1 is always the end marker
    int q_pend = -1;
    auto q_publish = [&](int k, int u) {
        q_list[k] = u;
        mbar_arrive(&q_ready[k]);
    };
    auto q_retire = [&]() {  // after the end marker: no claim of this CTA is left; the last CTA resets
        if (atomicAdd(iq.ctr + 1, 1) == static_cast<int>(gridDim.x) - 1) {
            atomicExch(iq.ctr, 0);
            atomicExch(iq.ctr + 1, 0);
        }
    };
    auto q_start = [&]() {  // producer lane 0, before the first item
        const int c0 = iq_claim(iq);
        q_publish(0, c0);
        q_pend = c0 >= 0 ? iq_claim(iq) : -1;
        if (c0 < 0) q_retire();
    };
    auto q_next = [&](int k) {  // producer lane 0, as item k starts
        const int nx = k + 1 <= kItemQ - 2 ? q_pend : -1;
        q_publish(k + 1, nx);
        q_pend = nx >= 0 && k + 2 <= kItemQ - 2 ? iq_claim(iq) : -1;
        if (nx < 0) q_retire();
    };
    // TMEM: S | dP (fp32, 128 cols each) | dQ (D) | dS (bf16 pairs, 64): the dQ
    // MMA takes A = dS straight from TMEM
    const uint32_t tS = tmem, tP = tmem + 128, tDQ = tmem + 256, tDS = tmem + 256 + D;

    if (warp == 0) {
        {  // warp-wide walk and waits, one elected lane issues
            int it = 0, ni = 0;
            if (iq.ctr) {  // dynamic queue: entry 0 (and the claim for entry 1)
                if (lane == 0) q_start();
                __syncwarp();
            }
            for (int k = 0, u = citem(0); u >= 0; ++ni, u = citem(++k)) {
                if (iq.ctr) {  // publish entry k + 1 as item k starts
                    if (lane == 0) q_next(k);
                    __syncwarp();
                }
                const Item w = item_of(u);
                const int row_base = w.b * T;
                const int qb = ni % QS;
                mbar_wait(&q_empty[qb], ((ni / QS) & 1) ^ 1);  // item ni-QS is done with this Q/dO slot
                if (fuse_d) mbar_wait(&d_free[qb], ((ni / QS) & 1) ^ 1);  // ... and its D is computed
                if (elect_one()) {
                    mbar_expect_tx(&q_full[qb], (fuse_d ? 3 : 2) * BW_TILE);
                    tma_tile<D>(sQ + qb * BW_TILE, &tmQKV, &q_full[qb], w.h * D, row_base + w.qt * BW_T);
                    tma_tile<D>(sO + qb * BW_TILE, &tmDO, &q_full[qb], w.h * D, row_base + w.qt * BW_T);
                    if (fuse_d) tma_tile<D>(sY + qb * BW_TILE, &tmY, &q_full[qb], w.h * D, row_base + w.qt * BW_T);
                }
                __syncwarp();
                for (int j = 0; j < w.nk; ++j, ++it) {
                    const int s = it % DQ_ST;
                    mbar_wait(&kv_empty[s], ((it / DQ_ST) & 1) ^ 1);
                    if (elect_one()) {
                        mbar_expect_tx(&kv_full[s], 2 * BW_TILE);
                        tma_tile<D>(sK + s * BW_TILE, &tmQKV, &kv_full[s], w.kc, row_base + j * BW_T);
                        tma_tile<D>(sV + s * BW_TILE, &tmQKV, &kv_full[s], w.vc, row_base + j * BW_T);
                    }
                    __syncwarp();
                }
            }
        }
    } else if (warp == 1) {
        // warp-wide walk and waits, one elected lane issues (see fa_fwd_tc2)
        constexpr uint32_t id_s = idesc_bf16(BW_T, BW_T, 0, 0);
        constexpr uint32_t id_g = idesc_bf16(BW_T, D, 0, 1);
        auto issue_s = [&](int g, int qb) {  // S = Q K_g^T, dP = dO V_g^T (global tile g, Q/dO slot qb)
            const int s = g % DQ_ST;
            mbar_wait(&kv_full[s], (g / DQ_ST) & 1);
            tc_after();
            const uint64_t qd = sdesc(smem_u32(sQ + qb * BW_TILE), 16, 1024), od = sdesc(smem_u32(sO + qb * BW_TILE), 16, 1024);
            const uint64_t kd = sdesc(smem_u32(sK + s * BW_TILE), 16, 1024), vd = sdesc(smem_u32(sV + s * BW_TILE), 16, 1024);
            if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) {  // K-major: 32 B per slice (sub-tiles of 64 columns)
                    umma(tS, kslice(qd, kk), kslice(kd, kk), id_s, kk > 0);
                    umma(tP, kslice(od, kk), kslice(vd, kk), id_s, kk > 0);
                }
                umma_commit(s_full);
            }
            __syncwarp();
        };
        int it = 0, ni = 0;
        if (citem(0) >= 0) {
            mbar_wait(&q_full[0], 0);
            issue_s(0, 0);
        }
        for (int k = 0, u = citem(0); u >= 0; ++ni, u = citem(++k)) {
            const Item w = item_of(u);
            const int qb = ni % QS;
            const bool more = citem(k + 1) >= 0;
            for (int j = 0; j < w.nk; ++j) {
                const int g = it + j;
                const int s = g % DQ_ST;
                // MN-major B (N = D: 64-wide atoms one 16 KB sub-tile apart)
                const uint64_t kd = sdesc(smem_u32(sK + s * BW_TILE), D == 64 ? 64 * 128 : 16384, 1024);
                if (j + 1 < w.nk) {
                    mbar_wait(s_free, g & 1);
                    tc_after();
                    issue_s(g + 1, qb);
                } else {
                    if (elect_one()) umma_commit(&q_empty[qb]);  // every S/dP of this item issued
                    __syncwarp();
                    if (more) {  // the next item's first S/dP under this tile's softmax
                        mbar_wait(&q_full[(ni + 1) % QS], ((ni + 1) / QS) & 1);
                        mbar_wait(s_free, g & 1);
                        tc_after();
                        issue_s(g + 1, (ni + 1) % QS);
                    }
                }
                mbar_wait(p_full, g & 1);
                tc_after();
                if (elect_one()) {
#pragma unroll
                    for (int kk = 0; kk < BW_T / 16; ++kk)  // 16 keys = 8 packed TMEM columns per step
                        umma_ts(tDQ, tDS + kk * 8, kd + 128 * kk, id_g, (j > 0 || kk > 0) ? 1u : 0u);
                    umma_commit(&kv_empty[s]);
                    umma_commit(g_done);
                }
                __syncwarp();
            }
            it += w.nk;
        }
    } else if (warp >= 4) {
        // 16 warps: quadrant wq (query rows = TMEM lanes) x quarter qq (32 of 128 keys)
        const int wq = warp & 3, qq = (warp - 4) >> 2;
        const int r = wq * 32 + lane;
        const uint32_t lane_off = static_cast<uint32_t>(wq * 32) << 16;
        const float sl = scale * kLog2e;
        // dQ of item `prev` leaves TMEM -> global inside the next item's first
        // tile (after its math, overlapping the last dQ MMA), or after the loop
        int prev = -1;
        auto epilogue = [&](int pu) {
            if (qq >= D / 32) return;
            const Item w = item_of(pu);
            const int q = w.qt * BW_T + r;
            uint32_t o[32];
            tmem_ld32(tDQ + lane_off + qq * 32, o);
            tmem_wait_ld();
            if (q < T) st_row32_global(dqkv + (static_cast<int64_t>(w.b) * T + q) * ldq + w.h * D + qq * 32, o, scale);
        };
        // this row's lse (log2) and D, loaded one item ahead
        auto fetch = [&](int u, float& L, float& Dq) {
            L = Dq = 0.f;
            if (u < 0) return;
            const Item w = item_of(u);
            const int q = w.qt * BW_T + r;
            const int64_t bh = static_cast<int64_t>(w.b) * H + w.h;
            if (q < T) {
                L = __ldg(lse + bh * T + q);  // (scaled to log2 at the item start: no stall here)
                if (!fuse_d) Dq = __ldg(dsum + bh * T + q);
            }
        };
        float nL, nD;
        fetch(citem(0), nL, nD);
        int it = 0;
        for (int k = 0, u = citem(0); u >= 0; u = citem(++k)) {
            const Item w = item_of(u);
            const int q = w.qt * BW_T + r;
            float Dq = nD;
            if (fuse_d) {  // D of this row from the item's dO and O tiles (every warp of the row alike)
                const int qb = k % QS;
                mbar_wait(&q_full[qb], (k / QS) & 1);
                Dq = row_dot_sw128<D>(sO + qb * BW_TILE, sY + qb * BW_TILE, r);
                mbar_arrive(&d_free[qb]);
                if (qq == 0 && q < T) dsum[(static_cast<int64_t>(w.b) * H + w.h) * T + q] = Dq;
                if (q >= T) Dq = 0.f;
            }
            const float L = nL * kLog2e;
            fetch(citem(k + 1), nL, nD);
            for (int j = 0; j < w.nk; ++j) {
                const int g = it + j;
                mbar_wait(s_full, g & 1);
                tc_after();
                const bool diag = j == w.nk - 1;
                {
                    // S and dP to registers first, TMEM released at once: the next
                    // tile's S / dP MMAs run under this tile's exp / dS math
                    uint32_t st[32], dp[32];
                    tmem_ld32(tS + lane_off + qq * 32, st);
                    tmem_ld32(tP + lane_off + qq * 32, dp);
                    tmem_wait_ld();
                    tc_before();
                    mbar_arrive(s_free);
                    float* p = reinterpret_cast<float*>(st);  // in place
                    // valid key columns c: j*128 + qq*32 + c <= q and < T
                    const int lim = min(q + 1, T) - (j * BW_T + qq * 32);
                    if (diag)
                        exp_row64<true, 32>(st, sl, L, lim, p);
                    else
                        exp_row64<false, 32>(st, sl, L, lim, p);
                    {
                        float dv[32];
#pragma unroll
                        for (int c = 0; c < 32; ++c) dv[c] = Dq;
                        ds_pairs(p, dp, dv, 32, p);
                    }
                    uint32_t pk[16];  // bf16 pairs: key 2c (low), 2c+1 (high)
#pragma unroll
                    for (int c = 0; c < 16; ++c) {
                        __nv_bfloat162 e = __floats2bfloat162_rn(p[2 * c], p[2 * c + 1]);
                        pk[c] = *reinterpret_cast<uint32_t*>(&e);
                    }
                    if (g > 0) {  // the previous dQ MMA has read dS
                        mbar_wait(g_done, (g - 1) & 1);
                        tc_after();
                    }
                    if (j == 0 && prev >= 0) {  // previous item's dQ is final
                        epilogue(prev);
                        prev = -1;
                    }
                    tmem_st16(tDS + lane_off + qq * 16, pk);
                    tmem_wait_st();
                }
                tc_before();
                mbar_arrive(p_full);
            }
            it += w.nk;
            prev = u;
        }
        if (prev >= 0) {
            mbar_wait(g_done, (it - 1) & 1);
            tc_after();
            epilogue(prev);
        }
    }
    tc_before();
    __syncthreads();
    if (warp == 2) {
        tc_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        ACCO_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p) throw Error(kCudaError, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<EncodeFn>(p);
    });
    return fn;
}

// [rows][cols] bf16 matrix (row stride ld), box 64 x 128, SW128
CUtensorMap rows_map(const void* p, int64_t cols, int64_t rows, int64_t ld) {
    CUtensorMap m;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
    cuuint32_t box[2] = {64, 128};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(p), dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(kCudaError, "attention tensor map: " + std::to_string(r));
    return m;
}

// D[bh, t] = sum_c dO[t, c] O[t, c]. y / dy are read as one flat stream of
// D-element head rows in memory order (token-major, head-minor): D / 8
// threads per row, 16 B each, a shuffle reduction.
template <int D>
__global__ void dsum_tc_kernel(const __nv_bfloat16* __restrict__ y, const __nv_bfloat16* __restrict__ dy,
                               float* __restrict__ dsum, int B, int T, int H) {
    ACCO_PDL_PROLOGUE();
    constexpr int TPR = D / 8;  // threads per head row
    const int64_t nrow = static_cast<int64_t>(B) * T * H;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t row = i / TPR;  // (b*T + t)*H + h
    float s = 0.f;
    if (row < nrow) {
        const uint4 a = __ldg(reinterpret_cast<const uint4*>(y) + i);
        const uint4 g = __ldg(reinterpret_cast<const uint4*>(dy) + i);
        const uint32_t wa[4] = {a.x, a.y, a.z, a.w}, wg[4] = {g.x, g.y, g.z, g.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            s = fmaf(__uint_as_float(wa[k] << 16), __uint_as_float(wg[k] << 16), s);
            s = fmaf(__uint_as_float(wa[k] & 0xffff0000u), __uint_as_float(wg[k] & 0xffff0000u), s);
        }
    }
#pragma unroll
    for (int o = 1; o < TPR; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (row < nrow && (threadIdx.x & (TPR - 1)) == 0) {
        const int h = static_cast<int>(row % H);
        const int64_t bt = row / H;
        const int t = static_cast<int>(bt % T), b = static_cast<int>(bt / T);
        dsum[(static_cast<int64_t>(b) * H + h) * T + t] = s;
    }
}

// LPT schedule of `costs.size()` items over min(items, SMs) CTAs, cached per
// (kernel kind, shape): device table [grid][k_max] (-1 padded).
struct Schedule {
    const int* table = nullptr;
    int grid = 0, k_max = 0;
    const int* order = nullptr;  // every item, heaviest first (the dynamic queue's order)
    int n = 0;
};

// Dynamic attention schedules (see ItemQueue): set by the trainer together
// with the CTA-pair GEMM queue when collectives run beside compute;
// ACCO_ATTN_STATIC / ACCO_ATTN_DYNAMIC override.
std::atomic<int> g_attn_dynamic{0};
struct StreamKeyA {
    int dev;
    cudaStream_t s;
    bool operator<(const StreamKeyA& o) const { return dev != o.dev ? dev < o.dev : s < o.s; }
};
ItemQueue item_queue(const Schedule& sc, cudaStream_t stream) {
    ItemQueue q{sc.order, sc.n, nullptr};
    const bool st = std::getenv("ACCO_ATTN_STATIC") != nullptr, dy = std::getenv("ACCO_ATTN_DYNAMIC") != nullptr;
    if (!(dy || (!st && g_attn_dynamic.load(std::memory_order_relaxed)))) return q;
    static std::mutex mu;
    static std::map<StreamKeyA, int*> ctrs;  // [claimed, retired] per (device, stream): launches are stream-ordered
    int dev = 0;
    ACCO_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    int*& c = ctrs[StreamKeyA{dev, stream}];
    if (!c) {
        ACCO_CUDA(cudaMalloc(&c, 32 * sizeof(int)));
        ACCO_CUDA(cudaMemset(c, 0, 32 * sizeof(int)));
    }
    q.ctr = c;
    return q;
}

Schedule lpt_schedule(int kind, int nt, int nbh, int G) {
    static std::mutex mu;
    static std::map<std::array<int, 4>, Schedule> cache;
    std::lock_guard<std::mutex> lock(mu);
    const std::array<int, 4> key{kind, nt, nbh, G};
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    // item u -> cost (tiles processed + a fixed per-item overhead)
    static const int ovh = std::getenv("ACCO_ATTN_OVH") ? std::atoi(std::getenv("ACCO_ATTN_OVH")) : 2;
    std::vector<int> cost;
    if (kind == 0) {  // forward: pair pr = npair - 1 - u / nbh; both tiles share K/V
        const int npair = (nt + 1) / 2;
        for (int u = 0; u < npair * nbh; ++u) {
            const int pr = npair - 1 - u / nbh;
            const int n0 = 2 * pr + 1, n1 = 2 * pr + 2 <= nt ? 2 * pr + 2 : 0;
            cost.push_back(n0 + n1 + ovh);
        }
    } else if (kind == 1) {  // dK/dV: kt = u / nbh, G query heads x (nt - kt) tiles
        for (int u = 0; u < nt * nbh; ++u) cost.push_back(G * (nt - u / nbh) + ovh);
    } else {  // dQ: qt = nt - 1 - u / nbh, qt + 1 key tiles
        for (int u = 0; u < nt * nbh; ++u) cost.push_back(nt - u / nbh + ovh);
    }
    const int n = static_cast<int>(cost.size());
    const int grid = std::min(n, num_sms());
    if (const char* e = std::getenv("ACCO_ATTN_SCHED")) {  // A/B knob: "rr" = round-robin heavy-first
        if (std::string(e) == "rr") {
            const int k_max = (n + grid - 1) / grid;
            std::vector<int> host(static_cast<size_t>(grid) * k_max, -1);
            for (int u = 0; u < n; ++u) host[static_cast<size_t>(u % grid) * k_max + u / grid] = u;
            int* dev = nullptr;
            ACCO_CUDA(cudaMalloc(&dev, host.size() * sizeof(int)));
            ACCO_CUDA(cudaMemcpy(dev, host.data(), host.size() * sizeof(int), cudaMemcpyHostToDevice));
            std::vector<int> ord(static_cast<size_t>(n));
            std::iota(ord.begin(), ord.end(), 0);
            int* dord = nullptr;
            ACCO_CUDA(cudaMalloc(&dord, ord.size() * sizeof(int)));
            ACCO_CUDA(cudaMemcpy(dord, ord.data(), ord.size() * sizeof(int), cudaMemcpyHostToDevice));
            Schedule sc{dev, grid, k_max, dord, n};
            cache[key] = sc;
            return sc;
        }
    }
    std::vector<int> order(static_cast<size_t>(n));
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cost[a] > cost[b]; });
    std::vector<std::vector<int>> lists(static_cast<size_t>(grid));
    using Load = std::pair<long long, int>;  // (load, cta): least-loaded first, ties by CTA index
    std::priority_queue<Load, std::vector<Load>, std::greater<Load>> pq;
    for (int c = 0; c < grid; ++c) pq.push({0, c});
    for (int u : order) {
        Load l = pq.top();
        pq.pop();
        lists[static_cast<size_t>(l.second)].push_back(u);
        pq.push({l.first + cost[u], l.second});
    }
    int k_max = 0;
    for (auto& v : lists) k_max = std::max(k_max, static_cast<int>(v.size()));
    std::vector<int> host(static_cast<size_t>(grid) * k_max, -1);
    for (int c = 0; c < grid; ++c)
        for (size_t k = 0; k < lists[static_cast<size_t>(c)].size(); ++k)
            host[static_cast<size_t>(c) * k_max + k] = lists[static_cast<size_t>(c)][k];
    int* dev = nullptr;
    ACCO_CUDA(cudaMalloc(&dev, host.size() * sizeof(int)));
    ACCO_CUDA(cudaMemcpy(dev, host.data(), host.size() * sizeof(int), cudaMemcpyHostToDevice));
    int* dord = nullptr;
    ACCO_CUDA(cudaMalloc(&dord, order.size() * sizeof(int)));
    ACCO_CUDA(cudaMemcpy(dord, order.data(), order.size() * sizeof(int), cudaMemcpyHostToDevice));
    Schedule sc{dev, grid, k_max, dord, n};
    cache[key] = sc;
    return sc;
}

// head size 64 (forward and backward) or 128 (allow128: the kernels templated on it)
bool tc_applicable(const void* a, const void* b, int hd, bool allow128 = false) {
    return (hd == HD || (allow128 && hd == 128)) && !(reinterpret_cast<uintptr_t>(a) & 15) &&
           !(reinterpret_cast<uintptr_t>(b) & 15) && !std::getenv("ACCO_ATTN_LEGACY");
}

}  // namespace

void attention_set_dynamic(bool on) { g_attn_dynamic.store(on ? 1 : 0, std::memory_order_relaxed); }

bool attention_bwd_tc(const __nv_bfloat16* qkv, const __nv_bfloat16* y, const float* lse, const __nv_bfloat16* dy,
                      __nv_bfloat16* dqkv, float* dsum, int B, int T, int H, int Hkv, int hd, cudaStream_t s) {
    if (!tc_applicable(qkv, dy, hd, true) || !tc_applicable(y, dqkv, hd, true)) return false;
    const int d = H * hd;
    const int ldq = (H + 2 * Hkv) * hd;  // qkv row: H q heads | Hkv k heads | Hkv v heads
    const int64_t rows = static_cast<int64_t>(B) * T;
    const int64_t nrow = rows * H;
    // D = rowsum(dO o O): inside the dQ kernel (which then runs first), or
    // as its own pass (ACCO_ATTN_DSUM_PASS, A/B)
    const bool fuse_d = std::getenv("ACCO_ATTN_DSUM_PASS") == nullptr;
    if (!fuse_d) {
        if (hd == 128)
            launch_pdl(dsum_tc_kernel<128>, static_cast<int>((nrow * 16 + 255) / 256), 256, 0, s, y, dy, dsum, B, T,
                       H);
        else
            launch_pdl(dsum_tc_kernel<64>, static_cast<int>((nrow * 8 + 255) / 256), 256, 0, s, y, dy, dsum, B, T, H);
        ACCO_CHECK_LAUNCH();
    }
    CUtensorMap mq = rows_map(qkv, ldq, rows, ldq);
    CUtensorMap mo = rows_map(dy, d, rows, d);
    CUtensorMap my = rows_map(y, d, rows, d);
    static bool cfg = false;
    if (!cfg) {
        ACCO_CUDA(cudaFuncSetAttribute(fa_bwd_dkv_tc<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, Dkv<64>::SMEM));
        ACCO_CUDA(cudaFuncSetAttribute(fa_bwd_dkv_tc<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, Dkv<128>::SMEM));
        ACCO_CUDA(cudaFuncSetAttribute(fa_bwd_dq_tc<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, Dq<64>::SMEM));
        ACCO_CUDA(cudaFuncSetAttribute(fa_bwd_dq_tc<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, Dq<128>::SMEM));
        cfg = true;
    }
    const float scale = 1.0f / sqrtf(static_cast<float>(hd));
    const int nt = (T + BW_T - 1) / BW_T;
    const Schedule skv = lpt_schedule(1, nt, B * Hkv, H / Hkv);
    auto dkv = [&] {
        if (hd == 128)
            launch_pdl(fa_bwd_dkv_tc<128>, skv.grid, BW_THREADS, Dkv<128>::SMEM, s, mq, mo, lse,
                       static_cast<const float*>(dsum), dqkv, B, T, H, Hkv, scale, skv.table, skv.k_max,
                       item_queue(skv, s));
        else
            launch_pdl(fa_bwd_dkv_tc<64>, skv.grid, BW_THREADS, Dkv<64>::SMEM, s, mq, mo, lse,
                       static_cast<const float*>(dsum), dqkv, B, T, H, Hkv, scale, skv.table, skv.k_max,
                       item_queue(skv, s));
        ACCO_CHECK_LAUNCH();
    };
    const Schedule sq = lpt_schedule(2, nt, B * H, 1);
    auto dq = [&] {
        if (hd == 128)
            launch_pdl(fa_bwd_dq_tc<128>, sq.grid, BW_THREADS, Dq<128>::SMEM, s, mq, mo, my, lse, dsum, dqkv, B, T, H,
                       Hkv, scale, sq.table, sq.k_max, item_queue(sq, s), fuse_d ? 1 : 0);
        else
            launch_pdl(fa_bwd_dq_tc<64>, sq.grid, BW_THREADS, Dq<64>::SMEM, s, mq, mo, my, lse, dsum, dqkv, B, T, H,
                       Hkv, scale, sq.table, sq.k_max, item_queue(sq, s), fuse_d ? 1 : 0);
        ACCO_CHECK_LAUNCH();
    };
    if (fuse_d) {  // dQ computes D, the dK/dV kernel reads it
        dq();
        dkv();
    } else {
        dkv();
        dq();
    }
    return true;
}

// qkv: [B*T, (H + 2*Hkv)*64] bf16 (H q heads | Hkv k heads | Hkv v heads);
// returns false if the tensor-core path does not apply (head size, alignment).
bool attention_fwd_tc(const __nv_bfloat16* qkv, __nv_bfloat16* y, float* lse, int B, int T, int H, int Hkv, int hd,
                      cudaStream_t s) {
    if (!tc_applicable(qkv, y, hd, true)) return false;
    const int ldq = (H + 2 * Hkv) * hd;  // qkv row: H q heads | Hkv k heads | Hkv v heads
    CUtensorMap m = rows_map(qkv, ldq, static_cast<int64_t>(B) * T, ldq);
    static bool cfg = false;
    if (!cfg) {
        ACCO_CUDA(cudaFuncSetAttribute(fa_fwd_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
        ACCO_CUDA(cudaFuncSetAttribute(fa_fwd_tc2<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, Fwd2<64>::SMEM));
        ACCO_CUDA(cudaFuncSetAttribute(fa_fwd_tc2<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, Fwd2<128>::SMEM));
        cfg = true;
    }
    const float scale = 1.0f / sqrtf(static_cast<float>(hd));
    const int nqt = (T + BQ - 1) / BQ;
    if (hd == 64 && std::getenv("ACCO_ATTN_FWD_V1")) {  // single-tile kernel (A/B reference)
        launch_pdl(fa_fwd_tc, dim3(nqt, B * H), kThreads, SMEM, s, m, y, lse, T, H, Hkv, scale);
    } else {
        const Schedule sf = lpt_schedule(0, nqt, B * H, 1);
        if (hd == 128)
            launch_pdl(fa_fwd_tc2<128>, sf.grid, F2_THREADS, Fwd2<128>::SMEM, s, m, y, lse, B, T, H, Hkv, scale, sf.table,
                       sf.k_max, item_queue(sf, s));
        else
            launch_pdl(fa_fwd_tc2<64>, sf.grid, F2_THREADS, Fwd2<64>::SMEM, s, m, y, lse, B, T, H, Hkv, scale, sf.table,
                       sf.k_max, item_queue(sf, s));
    }
    ACCO_CHECK_LAUNCH();
    return true;
}

}  // namespace acco
