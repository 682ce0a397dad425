// bf16 GEMM on the 5th-generation tensor cores (sm_100a), persistent.
//
// One CTA per SM loops over 128 x BN output tiles (grouped raster for L2 reuse):
//   warp 0   : TMA producer (one lane) — K-major or MN-major 128B-swizzled
//              operand tiles into a STAGES-deep smem ring (mbarrier full/empty)
//   warp 1   : MMA issuer (one lane) — tcgen05.mma.cta_group::1.kind::f16,
//              fp32 accumulators in TMEM, TWO accumulator buffers (2 x BN
//              columns) so the epilogue of tile i overlaps the MMAs of tile i+1
//   warp 2   : TMEM allocator
//   warps 4-7: epilogue — per 32x32 chunk: tcgen05.ld -> fused math (bias /
//              GELU / dGELU / residual) -> swizzled smem -> TMA bulk-tensor
//              store (bf16), or TMA bulk *reduce-add* into the fp32 gradient
//              accumulator (beta = 1); residual / GELU-aux inputs arrive by TMA
//              one chunk ahead. No per-element address math or uncoalesced
//              stores on the SM: the TMA engine does the global traffic.
// Split-K (work unit = tile x k-split) for the weight-gradient GEMMs whose tile
// count cannot fill 148 SMs: splits of a tile TMA-reduce-add into C *in split
// order* (a per-(tile, quadrant) semaphore hands the rows from split s to s+1),
// so the fp32 sums are deterministic, with no workspace and no extra pass.
//
// This is K1/K3 of SURVEY.md §2.3: forward (both operands K-major), dgrad (B
// MN-major) and wgrad (both MN-major, fp32 accumulate epilogue into the
// gradient-accumulation buffer: the reference's Bundle::add,
// /root/reference/proj/src/protocols.cpp:61-66, fused into the GEMM).
//
// fp32-accurate variant (X3 = 1, the parity mode, precision "fp32"): the same
// pipeline on kind::tf32 with the 3xTF32 split. A pre-pass writes every fp32
// operand as two K-major tf32 planes, hi = rna_tf32(x) and lo = rna_tf32(x - hi)
// (hi + lo carries 22 significand bits), and each k-slice issues
// lo*hi + hi*lo + hi*hi into the fp32 TMEM accumulator; the dropped lo*lo term
// and the rounding of lo are ~2^-22 relative. That keeps the fp32 contraction
// within the rel <= 1e-5 parity bar against the fp64 oracle,
// which one bf16 or tf32 pass (2^-8 / 2^-11) cannot meet.
#include "common.cuh"
#include "epilogue.cuh"
#include "gemm.h"

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <map>
#include <set>
#include <string>
#include <type_traits>
#include <mutex>

namespace acco {
namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;  // 64 bf16 = 128 bytes: one SW128 row
// warps 0-3: TMA producer, MMA issuer, TMEM alloc, idle; then the epilogue
// warps: 8 (two per TMEM lane quadrant) where the smem allows it next to a
// deep operand ring, else 4 (the 128x256 tiles keep 4 stages: a 3-stage ring
// costs them more than a faster epilogue gains)
// (the 3xTF32 variant stages two planes per operand: 4 epilogue warps leave
// room for a 3-deep ring of 128x128 tiles)
template <int BN, int STAGES, int X3 = 0>
constexpr int epi_warps() { return ((BN == 256 && STAGES == 4) || X3) ? 4 : 8; }
template <int BN, int STAGES, int X3 = 0>
constexpr int gemm_threads() { return 128 + 32 * epi_warps<BN, STAGES, X3>(); }
constexpr int kGroupM = 8;
// Per epilogue warp: 2 bf16 output chunks (or 2 fp32 chunks spanning the
// first 8 KB) + a ring of IN_BUF 2 KB input chunks (residual / GELU aux, TMA
// prefetched IN_BUF chunks ahead: one chunk ahead left the HBM latency of
// every chunk exposed). BN = 192 tiles have the smem for a 4-deep ring.
template <int BN>
constexpr int in_bufs() { return 2; }
// (the 3-stage BN = 256 variant, used by the SwiGLU epilogue, spends the freed
// stage on 12 KB per warp: its 3 outputs per chunk pair double-buffered)
template <int BN, int STAGES>
constexpr int epi_warp_bytes() { return 8192; }  // 2 bf16 output chunks (or 2 fp32 ones) + 2 input chunks

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t addr, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(ok)
        : "r"(addr), "r"(parity), "r"(20000u)  // suspend hint (ns): waiting warps sleep, not spin
        : "memory");
    return ok != 0;
}
// Watchdog for mbarrier spins: a pipeline bug becomes a launch error (trap)
// after ~4 s instead of a hung GPU.
__device__ __forceinline__ void watchdog(uint64_t& t0) {
    uint64_t now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    if (t0 == 0) t0 = now;
    else if (now - t0 > 4000000000ull) __trap();
}
__device__ __forceinline__ bool elect_one() {
    uint32_t pred;
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "elect.sync _|P, 0xffffffff;\n\t"
        "selp.b32 %0, 1, 0, P;\n\t}\n"
        : "=r"(pred));
    return pred != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    uint32_t spins = 0;
    uint64_t t0 = 0;
    while (!mbar_try_wait(a, parity)) {
        if ((++spins & 255u) == 0) watchdog(t0);
    }
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                            int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1)
                 : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}
__device__ __forceinline__ void tma_reduce_add_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
    asm volatile("cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}
// Cluster launch control (sm_100): steal the work of a CTA of this grid that
// has not launched yet. The 16-byte response lands in smem and completes the
// mbarrier's transaction count; it decodes to that CTA's id, or "none left".
__device__ __forceinline__ void clc_try_cancel(void* resp, uint64_t* bar) {
    asm volatile("clusterlaunchcontrol.try_cancel.async.shared::cta.mbarrier::complete_tx::bytes.b128 [%0], [%1];" ::"r"(
                     smem_u32(resp)),
                 "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ int clc_decode(const void* resp) {
    uint32_t x = 0, ok = 0;
    asm volatile(
        "{\n\t.reg .pred p;\n\t.reg .b128 r;\n\t"
        "ld.shared.b128 r, [%2];\n\t"
        "clusterlaunchcontrol.query_cancel.is_canceled.pred.b128 p, r;\n\t"
        "selp.u32 %1, 1, 0, p;\n\t"
        "@p clusterlaunchcontrol.query_cancel.get_first_ctaid.v4.b32.b128 {%0, _, _, _}, r;\n\t}\n"
        : "=r"(x), "=r"(ok)
        : "r"(smem_u32(resp))
        : "memory");
    return ok ? static_cast<int>(x) : -1;
}
__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
// ---- CTA pairs (cta_group::2): one MMA of M = 256 rows spans the two SMs of a
// TPC; each CTA stages its 128 A rows and half of the B rows, and holds its
// 128 accumulator rows in its own TMEM.
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
// shared::cluster address of `p` (a shared::cta pointer) in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa(const void* p, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// relaxed: the arriving warp only reports that it has read a slot (its value is
// already in registers), nothing it wrote must become visible
__device__ __forceinline__ void mbar_arrive_cluster_relaxed(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait_cluster(uint32_t addr, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(ok)
        : "r"(addr), "r"(parity), "r"(20000u)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    uint32_t spins = 0;
    uint64_t t0 = 0;
    while (!mbar_try_wait_cluster(a, parity)) {
        if ((++spins & 255u) == 0) watchdog(t0);
    }
}
// TMA load into this CTA's smem whose completion is signalled on the pair
// leader's mbarrier (bar = its shared::cluster address)
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void umma_bf16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}
// arrive on the mbarrier at this smem offset in both CTAs of the pair once the
// leader's issued MMAs complete
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(static_cast<uint16_t>(3))
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
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// UMMA shared-memory descriptor, SWIZZLE_128B, sm100 version bits.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
    d |= static_cast<uint64_t>(1) << 46;  // version = 1 (tcgen05)
    d |= static_cast<uint64_t>(2) << 61;  // SWIZZLE_128B
    return d;
}

// UMMA shared-memory descriptor without swizzle (K-major: 8-row x 16 B core
// matrices; lbo = byte stride between core matrices along K, sbo along M/N)
__device__ __forceinline__ uint64_t sdesc_noswz(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
    d |= static_cast<uint64_t>(1) << 46;  // version = 1 (tcgen05); layout 0 = SWIZZLE_NONE
    return d;
}

// Instruction descriptor for kind::f16: bf16 x bf16 -> fp32.
__host__ __device__ constexpr uint32_t idesc_bf16(int m, int n, int a_mn, int b_mn) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(a_mn) << 15) |
           (static_cast<uint32_t>(b_mn) << 16) | (static_cast<uint32_t>(n >> 3) << 17) |
           (static_cast<uint32_t>(m >> 4) << 24);
}
// kind::tf32: a/b format 2 (TF32), fp32 accumulator, both operands K-major.
__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
    return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
           (static_cast<uint32_t>(m >> 4) << 24);
}
__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}

// One operand tile is 128 B per row in every variant: 64 bf16 or 32 fp32 (tf32)
// elements of K. The 3xTF32 variant stages a hi and a lo plane per operand.
// Bias-gradient MMAs (Epilogue::bias_grad) need 2 x 16 spare TMEM columns next
// to the two accumulators (BN <= 192) and a ones B operand: a 16 x 16 bf16
// K-major tile without swizzle (four 8 x 8 core matrices, 512 B).
template <int BN, int X3 = 0>
constexpr bool has_bias_mma() { return !X3 && BN <= 192; }
// CTA-pair work queue: slots between the leader's producer, which posts each
// unit's successor when it starts the unit (claimed by an atomic issued one
// unit earlier), and the slowest reader (the epilogue warps read a unit's
// successor after that unit's epilogue; the producer is at most ~2 units
// ahead of them)
constexpr int kQueue = 3;
constexpr int kRespBytes = 4 * kQueue > 16 ? (4 * kQueue + 15) / 16 * 16 : 16;  // CLC response / queue slots
constexpr int kOnesBytes = 512;
template <int BN, int STAGES, int X3 = 0, int CG = 1>
constexpr int smem_bytes() {
    return 1024 /*align slack*/ + (has_bias_mma<BN, X3>() ? kOnesBytes + 128 : 0) +
           STAGES * (kBM + BN / CG) * 128 * (X3 ? 2 : 1) +
           epi_warps<BN, STAGES, X3>() * epi_warp_bytes<BN, STAGES>() +
           (2 * STAGES + 4 + epi_warps<BN, STAGES, X3>() * in_bufs<BN>()) * 8 + 16 +
           48 /* CLC: full / empty mbarriers, 16 B response, alignment */ +
           2 * (kQueue - 1) * 8 + (kRespBytes - 16) /* the CTA-pair work queue's further slots */;
}

struct Sched {
    int tiles_m, tiles_n, splits, kb_total, kb_per_split;
    int group_m;  // m-blocks per raster group (see decode)
    __host__ __device__ int units() const { return tiles_m * tiles_n * splits; }
};

// unit -> (m block, n block, split); grouped raster over M for L2 reuse of B
__device__ __forceinline__ void decode(const Sched& s, int u, int& mb, int& nb, int& sp) {
    const int tiles = s.tiles_m * s.tiles_n;
    sp = u / tiles;
    const int t = u % tiles;
    const int per_group = s.group_m * s.tiles_n;
    const int g = t / per_group;
    const int first_m = g * s.group_m;
    const int gsize = min(s.tiles_m - first_m, s.group_m);
    const int r = t % per_group;
    mb = first_m + r % gsize;
    nb = r / gsize;
}

__device__ __forceinline__ float tanh_fast(float x) {
    float y;
    asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// bf16-path GELU (tanh form) on the MUFU tanh; error << bf16 rounding
#ifdef ACCO_GEMM_PROBE
__device__ unsigned long long g_gprobe[148][6][16];
#define GEMM_PROBE(kind, idx)                                                        \
    do {                                                                             \
        unsigned long long _t;                                                       \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));                       \
        if ((idx) < 16 && blockIdx.x < 148) g_gprobe[blockIdx.x][kind][idx] = _t;    \
    } while (0)
#else
#define GEMM_PROBE(kind, idx)
#endif
// GELU and its slope gelu'(x) from one MUFU tanh: the forward epilogue stores
// the slope as aux, so the backward (dGELU) epilogue is a single multiply
__device__ __forceinline__ float2 f2(float v) { return make_float2(v, v); }
// (on a pair, with packed fp32 math: half the issue slots — the epilogue warps
// share the SM sub-partitions with the TMA and MMA issuers)
__device__ __forceinline__ float2 gelu_slope_fast2(float2 x, float2& slope) {
    const float k0 = 0.7978845608028654f, k1 = 0.044715f;
    const float2 x2 = mul_f32x2(x, x);
    const float2 u = mul_f32x2(x, fma_f32x2(f2(k0 * k1), x2, f2(k0)));
    const float2 t = make_float2(tanh_fast(u.x), tanh_fast(u.y));
    const float2 h = mul_f32x2(f2(0.5f), x);
    const float2 hq = mul_f32x2(h, fma_f32x2(make_float2(-t.x, -t.y), t, f2(1.0f)));
    slope = fma_f32x2(hq, fma_f32x2(f2(3.0f * k0 * k1), x2, f2(k0)), fma_f32x2(f2(0.5f), t, f2(0.5f)));
    return fma_f32x2(h, t, h);
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&h);
}

// One 32 x 32 bf16 chunk in smem as TMA SWIZZLE_64B lays it out: row r at
// r*64, 16B unit c at (c ^ ((r >> 1) & 3)).
__device__ __forceinline__ void st_row_bf16(uint8_t* buf, int r, const float* v) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        uint4 u = make_uint4(pack_bf16(v[8 * c + 0], v[8 * c + 1]), pack_bf16(v[8 * c + 2], v[8 * c + 3]),
                             pack_bf16(v[8 * c + 4], v[8 * c + 5]), pack_bf16(v[8 * c + 6], v[8 * c + 7]));
        *reinterpret_cast<uint4*>(buf + r * 64 + ((c ^ ((r >> 1) & 3)) << 4)) = u;
    }
}
__device__ __forceinline__ void ld_row_bf16(const uint8_t* buf, int r, float* v) {
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const uint4 u = *reinterpret_cast<const uint4*>(buf + r * 64 + ((c ^ ((r >> 1) & 3)) << 4));
        const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const __nv_bfloat162 h = *reinterpret_cast<const __nv_bfloat162*>(&w[k]);
            v[8 * c + 2 * k] = __bfloat162float(h.x);
            v[8 * c + 2 * k + 1] = __bfloat162float(h.y);
        }
    }
}
// One 32 x 32 fp32 chunk as TMA SWIZZLE_128B lays it out: row r at r*128,
// 16B unit c at (c ^ (r & 7)).
__device__ __forceinline__ void st_row_f32(uint8_t* buf, int r, const float* v) {
#pragma unroll
    for (int c = 0; c < 8; ++c)
        *reinterpret_cast<float4*>(buf + r * 128 + ((c ^ (r & 7)) << 4)) =
            make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
}

struct EpiMaps {
    CUtensorMap out;  // bf16 2D {N, M} box 32x32 SW64, or fp32 3D {N, M, slabs} box 32x32x1 SW128
    CUtensorMap aux;  // bf16 2D: GELU pre-activation (written in kEpiGelu, read in kEpiDGelu)
    CUtensorMap res;  // bf16 2D: residual input
};

// --------------------------------------------------------------------- kernel
template <int BN, int STAGES, int A_MN, int B_MN, int X3 = 0, int CG = 1>
__global__ void __launch_bounds__(gemm_threads<BN, STAGES, X3>(), 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ EpiMaps em, int M, int N, Sched sc, Epilogue ep, int* split_sem,
                   int use_clc, int* __restrict__ work_ctr) {
    static_assert(!X3 || (!A_MN && !B_MN), "3xTF32: the split pre-pass writes K-major planes");
    static_assert(CG == 1 || (!X3 && (!B_MN || (BN / 2) % 64 == 0)), "CTA pairs: bf16, B half a whole MN atom");
    extern __shared__ uint8_t smem_raw[];
    // 1 KB aligned by offsetting the shared array itself, so every pointer derived
    // from it stays in the shared address space (LDS / STS, not generic LD / ST)
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    constexpr int A_TILE = kBM * 128;  // one plane: 128 rows x 128 B
    constexpr int B_TILE = (BN / CG) * 128;  // this CTA's B rows (half of them in a CTA pair)
    constexpr int A_BYTES = A_TILE * (X3 ? 2 : 1);  // per stage (hi | lo planes for X3)
    constexpr int B_BYTES = B_TILE * (X3 ? 2 : 1);
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * A_BYTES;
    uint8_t* sEpi = sB + STAGES * B_BYTES;  // 1024-aligned
    constexpr int kInBuf = in_bufs<BN>();
    constexpr int kEpiWarpBytes = epi_warp_bytes<BN, STAGES>();
    constexpr int kEpiWarps = epi_warps<BN, STAGES, X3>();
    constexpr int kCS = kEpiWarps / 4;  // chunk stride: epilogue warps per TMEM lane quadrant
    uint64_t* full = reinterpret_cast<uint64_t*>(sEpi + kEpiWarps * kEpiWarpBytes);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;  // [2]
    uint64_t* tempty = tfull + 2;      // [2]
    uint64_t* inbar = tempty + 2;      // [8 epilogue warps][kInBuf]
    // CLC response ready (1 arrive + 16 B tx) / every role warp has read it;
    // the CTA-pair work queue uses kQueue slots of each (response ints in clc_resp)
    uint64_t* clc_full = inbar + kEpiWarps * kInBuf;
    uint64_t* clc_empty = clc_full + kQueue;
    uint8_t* clc_resp = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(clc_empty + kQueue) + 15) & ~uintptr_t(15));
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(clc_resp + kRespBytes);
    uint8_t* sOnes = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(tmem_slot + 1) + 127) & ~uintptr_t(127));
    constexpr bool kBiasMma = has_bias_mma<BN, X3>();

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int nunits = sc.units();
    if (kBiasMma && ep.bias_grad && warp == 3) {  // the ones tile (bf16 1.0), for the async proxy
        reinterpret_cast<uint4*>(sOnes)[lane] = make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
        fence_async_smem();
    }

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], CG * kEpiWarps);  // one arrive per epilogue warp (of both CTAs of a pair)
        }
        for (int i = 0; i < kEpiWarps * kInBuf; ++i) mbar_init(&inbar[i], 1);
        for (int q = 0; q < kQueue; ++q) mbar_init(&clc_full[q], 1);
        // producer, MMA issuer, epilogue warps (a CTA pair's work queue: both
        // producers and all epilogue warps arrive on the leader's)
        // (a CTA pair's queue: the peer's producer, the MMA issuer and every
        // epilogue warp of both CTAs read a claim; the leader's producer writes it)
        for (int q = 0; q < kQueue; ++q) mbar_init(&clc_empty[q], CG == 2 ? 2 * kEpiWarps + 2 : 2 + kEpiWarps);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    // two accumulator buffers (tile ping-pong); the 3xTF32 variant keeps a main
    // (hi*hi) and a correction (lo*hi + hi*lo) accumulator per buffer
    constexpr int kAccCols = X3 ? 2 * BN : BN;
    // power of two >= 2 accumulators (+ 2 x 16 bias-gradient columns)
    // (the bias columns only when this launch computes a bias gradient)
    const uint32_t kTmemCols = 2 * kAccCols + (kBiasMma && ep.bias_grad ? 32 : 0) <= 256 ? 256 : 512;
    constexpr uint32_t kBiasCol = 2 * kAccCols;  // bias-gradient accumulators [2][16]
    if (warp == 2) {
        if (CG == 2) {  // both CTAs of the pair allocate collectively (same columns in each)
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_slot)),
                         "r"(kTmemCols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                             smem_u32(tmem_slot)),
                         "r"(kTmemCols));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    tc_fence_before();
    if (CG == 2)
        cluster_sync();  // the peer's mbarriers are initialised before any remote arrive / complete_tx
    else
        __syncthreads();
    tc_fence_after();
    // CTA pair: rank 0 (the leader) issues the MMAs for both; units are per pair
    const uint32_t rank = CG == 2 ? cluster_rank() : 0;
    const int cta_unit0 = CG == 2 ? static_cast<int>(blockIdx.x >> 1) : static_cast<int>(blockIdx.x);
    const int unit_stride = static_cast<int>(gridDim.x) / CG;
    const uint32_t tmem_base = *tmem_slot;
    // prologue done (barriers, TMEM): let the next kernel launch, then wait for
    // the previous one's results before the first TMA load / global write
    pdl_trigger();
    pdl_wait();

    // Work units. Static: u, u + grid, ... (grid = min(units, SMs)). With
    // cluster launch control (use_clc, grid = units): after its own unit a CTA
    // takes over the units of CTAs that have not launched — SMs held by
    // another stream's kernels (the comm stream's collectives and optimizer)
    // just launch fewer CTAs, and the running ones absorb the work instead of
    // a static tile list waiting for its SM. Warp 3 claims one unit ahead; the
    // role warps read each claim from smem and release it.
    // CTA pairs (use_clc with CG == 2): cluster launch control over clusters
    // measured slow, so the pairs are persistent and, after their first unit,
    // take units from a per-stream counter in unit order (work_ctr[0]): the
    // leader's producer posts the successor of each unit as it starts loading
    // it (a pair holds at most two unstarted claims) into
    // both CTAs' smem for the other role warps. Pairs that start late (SMs held
    // by the comm stream) just claim fewer units. The last pair to retire
    // resets the counter for the next launch on the stream.
    int clc_i = 0;
    // the leader producer's claim for the unit after the current one, issued
    // when the current one starts (its latency hides under that unit's loads)
    int pending = 0;
    if (CG == 2 && use_clc && warp == 0 && rank == 0 && lane == 0) pending = atomicAdd(work_ctr, 1);
    auto claim_next = [&]() -> int {  // the leader's producer (CG == 2 queue)
        const int q = clc_i % kQueue;
        if (clc_i >= kQueue) mbar_wait_cluster(&clc_empty[q], (clc_i / kQueue - 1) & 1);  // slot read by all
        int nu = -1;
        if (lane == 0) {
            const int c = pending;
            nu = c + unit_stride < nunits ? c + unit_stride : -1;
            if (nu >= 0) pending = atomicAdd(work_ctr, 1);
            reinterpret_cast<volatile int*>(clc_resp)[q] = nu;
            asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(mapa(clc_resp + 4 * q, 1)), "r"(nu) : "memory");
            mbar_arrive_cluster(mapa(&clc_full[q], 0));
            mbar_arrive_cluster(mapa(&clc_full[q], 1));  // (release: the peer's response store before it)
            if (nu < 0 && atomicAdd(work_ctr + 1, 1) == unit_stride - 1) {  // every pair has stopped claiming
                atomicExch(work_ctr, 0);
                atomicExch(work_ctr + 1, 0);
            }
        }
        ++clc_i;
        return __shfl_sync(0xffffffffu, nu, 0);
    };
    int lead_next = -1;  // the leader producer: the successor it posted when starting the current unit
    auto next_unit = [&](int u) -> int {
        if (!use_clc) return u + unit_stride < nunits ? u + unit_stride : -1;
        if (CG == 2) {
            if (warp == 0 && rank == 0) return lead_next;
            const int q = clc_i % kQueue;
            mbar_wait_cluster(&clc_full[q], (clc_i / kQueue) & 1);
            const int nu = reinterpret_cast<volatile int*>(clc_resp)[q];
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster_relaxed(mapa(&clc_empty[q], 0));
            ++clc_i;
            return nu;
        }
        mbar_wait(&clc_full[0], clc_i & 1);
        const int nu = clc_decode(clc_resp);
        fence_async_smem();  // the async proxy rewrites the response next
        __syncwarp();
        if (lane == 0) mbar_arrive(&clc_empty[0]);
        ++clc_i;
        return nu;
    };

    if (warp == 3 && use_clc && CG == 1) {
        for (int i = 0;; ++i) {
            if (i > 0) mbar_wait(&clc_empty[0], (i - 1) & 1);  // every role warp has read claim i-1
            if (elect_one()) {
                mbar_expect_tx(&clc_full[0], 16);
                clc_try_cancel(clc_resp, &clc_full[0]);
            }
            __syncwarp();
            mbar_wait(&clc_full[0], i & 1);
            if (clc_decode(clc_resp) < 0) break;  // no unlaunched CTA left
        }
    } else if (warp == 0) {
        // like the MMA issuer: warp-uniform walk and waits, one elected lane issues
        {
            int it = 0;
            for (int u = cta_unit0; u >= 0; u = next_unit(u)) {
                // (pair queue: the leader posts this unit's successor as it starts the
                // unit, so the peer's producer never waits on it)
                if (CG == 2 && use_clc && rank == 0) lead_next = claim_next();
                int mb, nb, sp;
                decode(sc, u, mb, nb, sp);
                const int m0 = mb * (kBM * CG) + static_cast<int>(rank) * kBM, n0 = nb * BN;
                const int kb0 = sp * sc.kb_per_split;
                const int kb1 = min(sc.kb_total, kb0 + sc.kb_per_split);
                for (int kb = kb0; kb < kb1; ++kb, ++it) {
                    const int s = it % STAGES;
                    const uint32_t ph = (it / STAGES) & 1;
                    mbar_wait(&empty[s], ph ^ 1);
                    if (CG == 2) {
                        // this CTA's A rows and half of the B rows; both CTAs' loads
                        // complete on the leader's full barrier, which expects them all
                        if (elect_one()) {
                            const uint32_t fb = mapa(&full[s], 0);
                            if (rank == 0) mbar_expect_tx(&full[s], 2 * (A_BYTES + B_BYTES));
                            uint8_t* a_dst = sA + s * A_BYTES;
                            uint8_t* b_dst = sB + s * B_BYTES;
                            if (A_MN) {
#pragma unroll
                                for (int j = 0; j < kBM / 64; ++j)
                                    tma_load_2d_pair(a_dst + j * 64 * kBK * 2, &tmA, fb, m0 + j * 64, kb * kBK);
                            } else {
                                tma_load_2d_pair(a_dst, &tmA, fb, kb * kBK, m0);
                            }
                            const int nh = n0 + static_cast<int>(rank) * (BN / 2);
                            if (B_MN) {
#pragma unroll
                                for (int j = 0; j < BN / 128; ++j)
                                    tma_load_2d_pair(b_dst + j * 64 * kBK * 2, &tmB, fb, nh + j * 64, kb * kBK);
                            } else if (ep.mode == kEpiSwiGLU) {  // leader: gate rows, peer: the matching up rows
                                tma_load_2d_pair(b_dst, &tmB, fb, kb * kBK, (rank ? N / 2 : 0) + n0 / 2);
                            } else {
                                tma_load_2d_pair(b_dst, &tmB, fb, kb * kBK, nh);
                            }
                        }
                    } else if (X3) {
                        if (elect_one()) {  // hi and lo planes of both operands (3-D maps {K, rows, plane})
                            mbar_expect_tx(&full[s], A_BYTES + B_BYTES);
                            uint8_t* a_dst = sA + s * A_BYTES;
                            uint8_t* b_dst = sB + s * B_BYTES;
                            tma_load_3d(a_dst, &tmA, &full[s], kb * 32, m0, 0);
                            tma_load_3d(a_dst + A_TILE, &tmA, &full[s], kb * 32, m0, 1);
                            tma_load_3d(b_dst, &tmB, &full[s], kb * 32, n0, 0);
                            tma_load_3d(b_dst + B_TILE, &tmB, &full[s], kb * 32, n0, 1);
                        }
                    } else if (elect_one()) {
                        mbar_expect_tx(&full[s], A_BYTES + B_BYTES);
                        uint8_t* a_dst = sA + s * A_BYTES;
                        uint8_t* b_dst = sB + s * B_BYTES;
                        if (A_MN) {
#pragma unroll
                            for (int j = 0; j < kBM / 64; ++j)
                                tma_load_2d(a_dst + j * 64 * kBK * 2, &tmA, &full[s], m0 + j * 64, kb * kBK);
                        } else {
                            tma_load_2d(a_dst, &tmA, &full[s], kb * kBK, m0);
                        }
                        if (B_MN) {
#pragma unroll
                            for (int j = 0; j < BN / 64; ++j)
                                tma_load_2d(b_dst + j * 64 * kBK * 2, &tmB, &full[s], n0 + j * 64, kb * kBK);
                        } else if (ep.mode == kEpiSwiGLU) {  // gate rows, then the matching up rows
                            tma_load_2d(b_dst, &tmB, &full[s], kb * kBK, n0 / 2);
                            tma_load_2d(b_dst + (BN / 2) * kBK * 2, &tmB, &full[s], kb * kBK, N / 2 + n0 / 2);
                        } else {
                            tma_load_2d(b_dst, &tmB, &full[s], kb * kBK, n0);
                        }
                    }
                    __syncwarp();
                }
            }
        }
    } else if (warp == 1 && rank == 0) {
        // (a CTA pair's MMAs are issued by the leader alone)
        // The whole warp walks the schedule and waits (warp-uniform control, so the
        // descriptors live in uniform registers); one elected lane issues the MMAs
        // and commits. This keeps the issuer's instruction count per k-block low:
        // it shares its SM sub-partition with two epilogue warps.
        constexpr uint32_t idesc = idesc_bf16(kBM * CG, BN, A_MN, B_MN);
        constexpr uint32_t idesc_b = idesc_bf16(kBM * CG, 16, A_MN, 0);
        // no-swizzle K-major ones tile: 8 x 16 B core matrices, 128 B apart along
        // K (LBO), 256 B apart along N (SBO); every k-slice reads the same tile
        const uint64_t ones_d = sdesc_noswz(smem_u32(sOnes), 128, 256);
        // descriptor start-address step per 16-deep k slice (address >> 4):
        // K-major 32 B inside the 128B swizzle row, MN-major two 8-row atoms (2048 B)
        constexpr uint64_t a_step = A_MN ? 2048 >> 4 : 32 >> 4;
        constexpr uint64_t b_step = B_MN ? 2048 >> 4 : 32 >> 4;
        int it = 0, lt = 0;
        for (int u = cta_unit0; u >= 0; u = next_unit(u), ++lt) {
            int mb, nb, sp;
            decode(sc, u, mb, nb, sp);
            const int kb0 = sp * sc.kb_per_split;
            const int kb1 = min(sc.kb_total, kb0 + sc.kb_per_split);
            const int acc = lt & 1;
            if (CG == 2)  // both CTAs' epilogues drained this buffer
                mbar_wait_cluster(&tempty[acc], ((lt >> 1) & 1) ^ 1);
            else
                mbar_wait(&tempty[acc], ((lt >> 1) & 1) ^ 1);  // epilogue drained this buffer
            tc_fence_after();
            if (lane == 0) GEMM_PROBE(0, lt);
            const uint32_t tmem_d = tmem_base + acc * kAccCols;
            // the first n-block's tiles also accumulate the bias gradient (16
            // columns, each the row sum of A) against the ones tile
            const bool bias_unit = kBiasMma && ep.bias_grad != nullptr && nb == 0;
            const uint32_t tmem_b = tmem_base + kBiasCol + acc * 16;
            // two instantiations of the k-loop: tiles without the bias gradient
            // carry no (predicated-off) ones-MMAs, which cost the 128/192-wide
            // single-CTA tiles up to 25 % of their mainloop rate
            auto kloop = [&](auto with_bias) {
            constexpr bool kB = decltype(with_bias)::value;
            for (int kb = kb0; kb < kb1; ++kb, ++it) {
                const int s = it % STAGES;
                const uint32_t ph = (it / STAGES) & 1;
                mbar_wait(&full[s], ph);
                tc_fence_after();
                const uint64_t ad = A_MN ? sdesc(smem_u32(sA + s * A_BYTES), 64 * kBK * 2, 1024)
                                         : sdesc(smem_u32(sA + s * A_BYTES), 16, 1024);
                const uint64_t bd = B_MN ? sdesc(smem_u32(sB + s * B_BYTES), 64 * kBK * 2, 1024)
                                         : sdesc(smem_u32(sB + s * B_BYTES), 16, 1024);
                if (X3) {
                    // 4 slices of K = 8 per 128 B row; per slice hi*hi into the main
                    // accumulator and lo*hi + hi*lo into the correction accumulator.
                    // The tensor core truncates at every accumulate; chaining the
                    // 2^-11-sized correction terms into the main sum would cost an
                    // ulp of the main sum each, in their own they cost 2^-11 of it
                    // (the epilogue adds the two in round-to-nearest fp32).
                    constexpr uint32_t idesc3 = idesc_tf32(kBM, BN);
                    constexpr uint64_t a_lo = A_TILE >> 4, b_lo = B_TILE >> 4;
                    if (elect_one()) {
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk) {
                            const uint64_t ah = ad + kk * 2, bh = bd + kk * 2;
                            const uint32_t first = (kb > kb0 || kk > 0) ? 1u : 0u;
                            umma_tf32(tmem_d + BN, ah + a_lo, bh, idesc3, first);
                            umma_tf32(tmem_d + BN, ah, bh + b_lo, idesc3, 1u);
                            umma_tf32(tmem_d, ah, bh, idesc3, first);
                        }
                        umma_commit(&empty[s]);
                    }
                } else if (CG == 2) {
                    if (elect_one()) {
#pragma unroll
                        for (int kk = 0; kk < kBK / 16; ++kk)
                            umma_bf16_pair(tmem_d, ad + kk * a_step, bd + kk * b_step, idesc,
                                           (kb > kb0 || kk > 0) ? 1u : 0u);
                        if constexpr (kB) {
#pragma unroll
                            for (int kk = 0; kk < kBK / 16; ++kk)
                                umma_bf16_pair(tmem_b, ad + kk * a_step, ones_d, idesc_b, (kb > kb0 || kk > 0) ? 1u : 0u);
                        }
                        umma_commit_pair(&empty[s]);  // frees the stage in both CTAs
                    }
                } else if (elect_one()) {
#pragma unroll
                    for (int kk = 0; kk < kBK / 16; ++kk)
                        umma_bf16(tmem_d, ad + kk * a_step, bd + kk * b_step, idesc, (kb > kb0 || kk > 0) ? 1u : 0u);
                    if constexpr (kB) {  // bias gradient: row sums of A (x ones)
#pragma unroll
                        for (int kk = 0; kk < kBK / 16; ++kk)
                            umma_bf16(tmem_b, ad + kk * a_step, ones_d, idesc_b, (kb > kb0 || kk > 0) ? 1u : 0u);
                    }
                    umma_commit(&empty[s]);
                }
                __syncwarp();
            }
            };
            if (kBiasMma && bias_unit)
                kloop(std::integral_constant<bool, kBiasMma>{});
            else
                kloop(std::false_type{});
            if (elect_one()) {
                if (CG == 2)
                    umma_commit_pair(&tfull[acc]);
                else
                    umma_commit(&tfull[acc]);
            }
            __syncwarp();
            if (lane == 0) GEMM_PROBE(1, lt);
        }
    } else if (warp >= 4) {
        // 8 epilogue warps: warp ew handles TMEM lane quadrant wq (32 rows) and the
        // chunks c = hf, hf+2, ... (every other 32-column chunk) of each tile, so
        // two warps drain a quadrant in parallel (GELU/dGELU/SwiGLU epilogues were
        // the bottleneck of their GEMMs with one warp per quadrant)
        const int ew = warp - 4, wq = ew & 3, hf = ew >> 2;  // hf < kCS
        // this warp's share of accumulator buffer a has been read: hand it back
        // (to the pair leader's barrier: its MMAs write both CTAs' TMEM)
        auto release_acc = [&](int a) {
            if (CG == 2)
                mbar_arrive_cluster(mapa(&tempty[a], 0));
            else
                mbar_arrive(&tempty[a]);
        };
        uint8_t* wbuf = sEpi + ew * kEpiWarpBytes;
        uint64_t* ib = inbar + kInBuf * ew;
        const bool f32 = ep.mode == kEpiAccF32;
        const bool has_in = !f32 && (ep.mode == kEpiDGelu || ep.residual != nullptr);
        const CUtensorMap* in_map = ep.mode == kEpiDGelu ? &em.aux : &em.res;
        const __nv_bfloat16* bias = static_cast<const __nv_bfloat16*>(ep.bias);
        uint32_t in_phase = 0;  // bit k: parity of the next wait on input buffer k
        constexpr int kChunks = BN / 32;
        // output staging buffers alternate over this warp's whole chunk sequence,
        // across tiles (a per-tile parity would hand the last chunk's buffer of
        // an odd-length tile — BN = 192 with two warps per quadrant — straight
        // to the next tile's first chunk while its TMA store may still read it)
        int seq = 0;
        int lt = 0;
        for (int u = cta_unit0; u >= 0; u = next_unit(u), ++lt) {
            int mb, nb, sp;
            decode(sc, u, mb, nb, sp);
            const int acc = lt & 1;
            const int row0 = mb * (kBM * CG) + static_cast<int>(rank) * kBM + wq * 32;
            const int n0 = nb * BN;
            if (has_in && lane == 0) {  // this warp's first kInBuf input chunks of the tile
#pragma unroll
                for (int j = 0; j < kInBuf; ++j)
                    if (hf + kCS * j < kChunks) {
                        mbar_expect_tx(&ib[j], 2048);
                        tma_load_2d(wbuf + 4096 + j * 2048, in_map, &ib[j], n0 + (hf + kCS * j) * 32, row0);
                    }
            }
            // bias of this warp's first chunk (each chunk then prefetches the next one's)
            uint4 bpre[4];
            if (bias && n0 + hf * 32 + 32 <= N) {
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    bpre[q] = __ldg(reinterpret_cast<const uint4*>(bias + n0 + hf * 32 + 8 * q));
            }
            // ordered split-K: this warp's (quadrant, column half) slice is added in split order
            // own 128B line per (tile, CTA of the pair, epilogue warp)
            int* sem = split_sem ? split_sem + (((mb * sc.tiles_n + nb) * CG + static_cast<int>(rank)) * 8 + ew) * 32
                                 : nullptr;
            if (sem && lane == 0) {
                while (ld_acquire(sem) != sp) __nanosleep(64);
                fence_async_global();
            }
            __syncwarp();
            if (ep.mode == kEpiDSwiGLU) {
                // acc = dA for features [n0, n0+BN); inputs gate / up pre-activations
                // (aux columns f and F + f, one 4 KB slot per chunk); outputs
                // d(gate) / d(up) into C = dGU
                constexpr int kSlots = (kEpiWarpBytes - 4096) / 4096;
                static_assert(kSlots >= 1 && kSlots <= kInBuf, "DSwiGLU input slots");
                const int F = N;
                uint8_t* in0 = wbuf + 4096;
                auto load_in = [&](int j) {  // this warp's j-th chunk
                    const int sl = j % kSlots, c = hf + kCS * j;
                    mbar_expect_tx(&ib[sl], 4096);
                    tma_load_2d(in0 + sl * 4096, &em.aux, &ib[sl], n0 + c * 32, row0);
                    tma_load_2d(in0 + sl * 4096 + 2048, &em.aux, &ib[sl], F + n0 + c * 32, row0);
                };
                if (lane == 0)
                    for (int j = 0; j < kSlots && hf + kCS * j < kChunks; ++j) load_in(j);
                mbar_wait(&tfull[acc], (lt >> 1) & 1);
                tc_fence_after();
                const uint32_t tb = tmem_base + acc * kAccCols + (static_cast<uint32_t>(wq * 32) << 16);
#pragma unroll 1
                for (int j = 0, c = hf; c < kChunks; ++j, c += kCS) {
                    const int sl = j % kSlots;
                    uint32_t raw[32];
                    tmem_ld32(tb + c * 32, raw);
                    if (c + kCS >= kChunks) {
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) release_acc(acc);
                    }
                    mbar_wait(&ib[sl], (in_phase >> sl) & 1);
                    in_phase ^= 1u << sl;
                    float g[32], uu[32], dg[32], du[32];
                    ld_row_bf16(in0 + sl * 4096, lane, g);
                    ld_row_bf16(in0 + sl * 4096 + 2048, lane, uu);
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const float dd = __bfloat162float(__float2bfloat16_rn(__uint_as_float(raw[i])));
                        const float sg = 1.0f / (1.0f + __expf(-g[i]));
                        dg[i] = dd * uu[i] * sg * (1.0f + g[i] * (1.0f - sg));
                        du[i] = dd * g[i] * sg;
                    }
                    __syncwarp();  // the slot has been consumed: refill it kSlots chunks ahead
                    if (lane == 0 && hf + kCS * (j + kSlots) < kChunks) load_in(j + kSlots);
                    if (n0 + c * 32 >= F) continue;  // past the last feature (F % 32 == 0): no store
                    if (lane == 0) bulk_wait_read<0>();  // the previous chunk's staging was read
                    __syncwarp();
                    st_row_bf16(wbuf, lane, dg);
                    st_row_bf16(wbuf + 2048, lane, du);
                    fence_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        tma_store_2d(&em.out, wbuf, n0 + c * 32, row0);
                        tma_store_2d(&em.out, wbuf + 2048, F + n0 + c * 32, row0);
                        bulk_commit();
                    }
                }
                __syncwarp();
                continue;
            }
            mbar_wait(&tfull[acc], (lt >> 1) & 1);
            tc_fence_after();
            if (lane == 0 && (ew == 0 || ew == kEpiWarps - 1)) GEMM_PROBE(ew == 0 ? 2 : 4, lt);
            const uint32_t tbase = tmem_base + acc * kAccCols + (static_cast<uint32_t>(wq * 32) << 16);
            if (kBiasMma && ep.bias_grad && nb == 0 && hf == 0) {
                // bias gradient of this quadrant's rows (column 0 of the 16 equal
                // ones-MMA columns), added in split order like the tile itself
                uint32_t bv;
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];"
                             : "=r"(bv)
                             : "r"(tmem_base + kBiasCol + acc * 16 + (static_cast<uint32_t>(wq * 32) << 16)));
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
                const int row = row0 + lane;
                if (row < M) {
                    // (ordered before the next split's reads by this warp's
                    // __syncwarp()s and lane 0's st.release of the hand-off)
                    float* bg = ep.bias_grad + row;
                    *bg = (sp > 0 || ep.beta) ? *bg + __uint_as_float(bv) : __uint_as_float(bv);
                }
            }
            if (ep.mode == kEpiSwiGLU) {
                // accumulator columns [0, BN/2) = gate, [BN/2, BN) = up of the same
                // BN/2 features (n0/2 ...): store both pre-activations (for the
                // backward) and silu(gate) * up, computed from the bf16-rounded
                // pre-activations exactly as the unfused kernel would
                const int F = N / 2;
#pragma unroll 1
                for (int c = hf; c < kChunks / 2; c += kCS) {
                    uint32_t rg[32], ru[32];
                    tmem_ld32(tbase + c * 32, rg);
                    tmem_ld32(tbase + (c + kChunks / 2) * 32, ru);
                    if (c + kCS >= kChunks / 2) {
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) release_acc(acc);
                    }
                    float g[32], uu[32], a[32];
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        g[i] = __bfloat162float(__float2bfloat16_rn(__uint_as_float(rg[i])));
                        uu[i] = __bfloat162float(__float2bfloat16_rn(__uint_as_float(ru[i])));
                        a[i] = __fdividef(g[i], 1.0f + __expf(-g[i])) * uu[i];
                    }
                    if (lane == 0) bulk_wait_read<0>();  // the previous pair's staging was read
                    __syncwarp();
                    st_row_bf16(wbuf, lane, g);
                    st_row_bf16(wbuf + 2048, lane, uu);
                    st_row_bf16(wbuf + 4096, lane, a);
                    fence_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        const int cg = n0 / 2 + c * 32;
                        tma_store_2d(&em.aux, wbuf, cg, row0);
                        tma_store_2d(&em.aux, wbuf + 2048, F + cg, row0);
                        tma_store_2d(&em.out, wbuf + 4096, cg, row0);
                        bulk_commit();
                    }
                }
                __syncwarp();
                continue;
            }
#pragma unroll 1
            for (int j = 0, c = hf; c < kChunks; ++j, ++seq, c += kCS) {
                const int b = seq & 1;
                const int ibuf = j % kInBuf;
                const int col0 = n0 + c * 32;
                uint4 bcur[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) bcur[q] = bpre[q];
                if (bias && c + kCS < kChunks && col0 + 32 * kCS + 32 <= N) {
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        bpre[q] = __ldg(reinterpret_cast<const uint4*>(bias + col0 + 32 * kCS + 8 * q));
                }
                uint32_t raw[32];
                tmem_ld32(tbase + c * 32, raw);
                if (X3) {  // main + correction accumulator
                    uint32_t cr[32];
                    tmem_ld32(tbase + BN + c * 32, cr);
#pragma unroll
                    for (int i = 0; i < 32; ++i) raw[i] = __float_as_uint(__uint_as_float(raw[i]) + __uint_as_float(cr[i]));
                }
                if (c + kCS >= kChunks) {  // this warp's share of the accumulator read: hand TMEM back
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) release_acc(acc);
                }
                float v[32];
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(raw[i]);
                if (bias) {
                    if (col0 + 32 <= N) {
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const uint4 u4 = bcur[q];
                            const uint32_t w[4] = {u4.x, u4.y, u4.z, u4.w};
#pragma unroll
                            for (int k = 0; k < 4; ++k) {
                                const float2 bf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w[k]));
                                const float2 r2 = add_f32x2(make_float2(v[8 * q + 2 * k], v[8 * q + 2 * k + 1]), bf);
                                v[8 * q + 2 * k] = r2.x;
                                v[8 * q + 2 * k + 1] = r2.y;
                            }
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (col0 + i < N) v[i] += __bfloat162float(bias[col0 + i]);
                    }
                }
                if (has_in) {
                    mbar_wait(&ib[ibuf], (in_phase >> ibuf) & 1);
                    in_phase ^= 1u << ibuf;
                    float iv[32];
                    ld_row_bf16(wbuf + 4096 + ibuf * 2048, lane, iv);
                    if (ep.mode == kEpiDGelu) {  // aux = gelu'(pre-activation), stored by the forward
#pragma unroll
                        for (int i = 0; i < 32; ++i) v[i] *= iv[i];
                    } else {
#pragma unroll
                        for (int i = 0; i < 32; ++i) v[i] += iv[i];
                    }
                    __syncwarp();  // every lane has consumed the input buffer: refill it kInBuf chunks ahead
                    if (lane == 0 && c + kCS * kInBuf < kChunks) {
                        mbar_expect_tx(&ib[ibuf], 2048);
                        tma_load_2d(wbuf + 4096 + ibuf * 2048, in_map, &ib[ibuf], col0 + kCS * kInBuf * 32, row0);
                    }
                }
                // the TMA store that last used these staging buffers (two chunks
                // back in this warp's sequence, maybe in the previous tile) must
                // have finished reading them
                if (lane == 0) bulk_wait_read<1>();
                __syncwarp();
                if (f32) {
                    uint8_t* ob = wbuf + b * 4096;
                    st_row_f32(ob, lane, v);
                    fence_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        if (sp > 0 || ep.beta)
                            tma_reduce_add_3d(&em.out, ob, col0, row0, 0);
                        else
                            tma_store_3d(&em.out, ob, col0, row0, 0);
                        bulk_commit();
                    }
                } else {
                    uint8_t* ob = wbuf + b * 2048;
                    if (ep.mode == kEpiGelu) {
                        float sl[32];
#pragma unroll
                        for (int i = 0; i < 32; i += 2) {
                            float2 s2;
                            const float2 g2 = gelu_slope_fast2(make_float2(v[i], v[i + 1]), s2);
                            v[i] = g2.x;
                            v[i + 1] = g2.y;
                            sl[i] = s2.x;
                            sl[i + 1] = s2.y;
                        }
                        st_row_bf16(wbuf + 4096 + b * 2048, lane, sl);  // gelu' (aux, for the backward)
                    }
                    st_row_bf16(ob, lane, v);
                    fence_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        tma_store_2d(&em.out, ob, col0, row0);
                        if (ep.mode == kEpiGelu) tma_store_2d(&em.aux, wbuf + 4096 + b * 2048, col0, row0);
                        bulk_commit();
                    }
                }
            }
            if (lane == 0 && (ew == 0 || ew == kEpiWarps - 1)) GEMM_PROBE(ew == 0 ? 3 : 5, lt);
            if (sem && lane == 0) {  // this split's adds are complete: hand over to split sp+1
                bulk_wait_all();
                fence_async_global();
                st_release(sem, sp + 1 == sc.splits ? 0 : sp + 1);
            }
            __syncwarp();
        }
        if (lane == 0) bulk_wait_all();
        __syncwarp();
    }
    tc_fence_before();
    if (CG == 2)
        cluster_sync();  // the peer's MMAs into this TMEM and its remote arrives are done
    else
        __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        if (CG == 2)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols));
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols));
    }
}

// ----------------------------------------------------------------- host side
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

CUtensorMap encode(CUtensorMapDataType dt, int rank, const void* ptr, const cuuint64_t* dims,
                   const cuuint64_t* strides, const cuuint32_t* box, CUtensorMapSwizzle sw) {
    ACCO_REQUIRE((reinterpret_cast<uintptr_t>(ptr) & 15) == 0, "gemm: operand not 16B aligned");
    for (int i = 0; i < rank - 1; ++i) ACCO_REQUIRE(strides[i] % 16 == 0, "gemm: row stride must be a multiple of 16 bytes");
    CUtensorMap m;
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = encode_fn()(&m, dt, rank, const_cast<void*>(ptr), dims, strides, box, estr,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(kCudaError, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
    return m;
}

// 2-D bf16 tensor map: `inner` contiguous elements per row, `outer` rows.
CUtensorMap make_map(const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld_elems, uint32_t box_inner,
                     uint32_t box_outer, CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B) {
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {ld_elems * 2};
    cuuint32_t box[2] = {box_inner, box_outer};
    return encode(CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, ptr, dims, strides, box, sw);
}

// 3-D fp32 map {N, M, slabs} for the accumulate / split-K epilogue.
CUtensorMap make_map_f32(const void* ptr, uint64_t n, uint64_t m, uint64_t slabs, uint64_t ld_elems) {
    cuuint64_t dims[3] = {n, m, slabs};
    cuuint64_t strides[2] = {ld_elems * 4, ld_elems * 4 * m};
    cuuint32_t box[3] = {32, 32, 1};
    return encode(CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, ptr, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
}

// Tensor map for an operand with `rows` (M or N) and reduction extent K.
CUtensorMap operand_map(const GemmOperand& op, int rows, int K, int tile_rows) {
    if (op.mn_major) return make_map(op.ptr, rows, K, op.ld, 64, kBK);  // stored [K][rows]
    return make_map(op.ptr, K, rows, op.ld, kBK, tile_rows);             // stored [rows][K]
}

constexpr int kSemSlots = 1 << 21;  // (tile, quadrant) semaphores for ordered split-K (8 MB)

// CLC scheduling for every non-split GEMM (ACCO_GEMM_NO_CLC=1: static persistent
// schedule, the A/B knob; read per launch)
bool use_clc(const Sched& sc) { return sc.splits == 1 && std::getenv("ACCO_GEMM_NO_CLC") == nullptr; }

// Split-K semaphores and the pure-store split workspace are per (device,
// stream): the hand-off protocol and the workspace contents are
// stream-ordered, so GEMMs that run concurrently on different streams (the
// model's weight-gradient side stream, torch's stream in the tests) or devices
// must not share them.
struct StreamKey {
    int dev;
    cudaStream_t s;
    bool operator<(const StreamKey& o) const { return dev != o.dev ? dev < o.dev : s < o.s; }
};
std::mutex g_scratch_mu;

int* split_semaphores(cudaStream_t stream) {
    static std::map<StreamKey, int*> sems;
    int dev = 0;
    ACCO_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_scratch_mu);
    int*& sem = sems[StreamKey{dev, stream}];
    if (!sem) {
        ACCO_CUDA(cudaMalloc(&sem, kSemSlots * sizeof(int)));
        ACCO_CUDA(cudaMemset(sem, 0, kSemSlots * sizeof(int)));
    }
    return sem;
}

// CTA-pair scheduling: static persistent order (fastest with the GPU to
// itself: qkv_fwd 23.4 vs 27.4 us) or the work queue (robust when another
// stream's kernels hold SMs: under the emulated 8-GPU interconnect ACCO 742.9k
// vs 719.1k tok/s, 1.021x vs 0.973x ZeRO-1). The trainer turns the queue on
// when collectives run beside compute (world > 1 or an emulated interconnect);
// ACCO_PAIR_STATIC / ACCO_PAIR_DYNAMIC override.
std::atomic<int> g_pair_queue{0};
bool pair_queue_on() {
    const bool st = std::getenv("ACCO_PAIR_STATIC") != nullptr, dy = std::getenv("ACCO_PAIR_DYNAMIC") != nullptr;
    return dy || (!st && g_pair_queue.load(std::memory_order_relaxed) != 0);
}

// CTA-pair work-queue counters ([claimed, retired]) per (device, stream),
// like the split-K semaphores: launches on one stream are ordered, the last
// pair of each launch resets them
int* work_counters(cudaStream_t stream) {
    static std::map<StreamKey, int*> ctrs;
    int dev = 0;
    ACCO_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_scratch_mu);
    int*& c = ctrs[StreamKey{dev, stream}];
    if (!c) {
        ACCO_CUDA(cudaMalloc(&c, 32 * sizeof(int)));
        ACCO_CUDA(cudaMemset(c, 0, 32 * sizeof(int)));
    }
    return c;
}

template <int BN, int STAGES, int A_MN, int B_MN, int CG>
void launch(const GemmOperand& A, const GemmOperand& B, int M, int N, int K, const Epilogue& ep, int splits,
            cudaStream_t stream) {
    auto kern = gemm_tc_kernel<BN, STAGES, A_MN, B_MN, 0, CG>;
    constexpr int smem = smem_bytes<BN, STAGES, 0, CG>();
    static_assert(smem <= 232448, "shared memory budget");
    static int max_pairs = 0;  // per instantiation: co-resident CTA pairs
    if (!max_pairs) {
        ACCO_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        max_pairs = num_sms() / 2;
        if (CG == 2) {
            ACCO_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 0));
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(2 * max_pairs);
            cfg.blockDim = dim3(gemm_threads<BN, STAGES>());
            cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = 2;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            int n = 0;
            ACCO_CUDA(cudaOccupancyMaxActiveClusters(&n, kern, &cfg));
            if (n > 0) max_pairs = n;
        }
    }
    Sched sc;
    sc.tiles_m = ceil_div(M, kBM * CG);
    sc.tiles_n = ceil_div(N, BN);
    sc.kb_total = ceil_div(K, kBK);
    // raster: groups of kGroupM m-blocks sweep all n-blocks (A rows reused from
    // L2, B streamed once per group). When B is too big to stay in L2 between
    // groups but all of A is small, the group spans every m-block so each B
    // n-block is read from HBM once: the LM head (B = 77 MB of embeddings, 824
    // MB of logits streaming through L2) re-read B per group, 529 -> 492 us;
    // Llama-1b's head (A = 33.5 MB, B = 131 MB): +1.1 % tok/s
    sc.group_m = static_cast<double>(M) * K * 2 <= 48e6 && static_cast<double>(N) * K * 2 > 32e6 &&
                         !std::getenv("ACCO_GEMM_GROUP8")
                     ? sc.tiles_m
                     : kGroupM;
    sc.splits = splits;
    sc.kb_per_split = ceil_div(sc.kb_total, splits);
    sc.splits = ceil_div(sc.kb_total, sc.kb_per_split);  // no empty splits
    EpiMaps em;
    std::memset(&em, 0, sizeof(em));
    int* sem = nullptr;
    if (ep.mode == kEpiAccF32) {
        em.out = make_map_f32(ep.C, N, M, 1, ep.ldc);
        if (sc.splits > 1) {
            ACCO_REQUIRE(sc.tiles_m * sc.tiles_n * CG * 8 * 32 <= kSemSlots, "gemm: too many tiles for split-K");
            sem = split_semaphores(stream);
        }
    } else {
        em.out = make_map(ep.C, ep.mode == kEpiSwiGLU ? N / 2 : (ep.mode == kEpiDSwiGLU ? 2 * N : N), M, ep.ldc, 32, 32,
                          CU_TENSOR_MAP_SWIZZLE_64B);
        if (ep.aux)
            em.aux = make_map(ep.aux, ep.mode == kEpiDSwiGLU ? 2 * N : N, M, ep.ld_aux, 32, 32,
                              CU_TENSOR_MAP_SWIZZLE_64B);
        if (ep.residual) em.res = make_map(ep.residual, N, M, ep.ldr, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B);
    }
    CUtensorMap ta = operand_map(A, M, K, kBM);
    // (B box: the rows one CTA stages — half the tile's in a CTA pair or in
    // the SwiGLU gate / up halves)
    CUtensorMap tb = operand_map(B, N, K, (ep.mode == kEpiSwiGLU || CG == 2) ? BN / 2 : BN);
    if (CG == 2) {
        // persistent CTA pairs; unless split-K (whose ordered hand-off needs the
        // static order) the units after each pair's first come from a per-stream
        // counter (see the kernel). (Cluster launch control over pairs — one
        // cluster per unit, the leader cancelling a whole cluster with a
        // multicast response — was measured slower than the static order on
        // every shape: qkv_fwd 26.2 vs 23.2 us, head_fwd 539 vs 452 us,
        // profiles/r02_summary.md.)
        const int q = use_clc(sc) && pair_queue_on() ? 1 : 0;
        const int grid = 2 * std::min(sc.units(), max_pairs);
        launch_pdl_cluster(kern, 2, grid, gemm_threads<BN, STAGES>(), smem, stream, ta, tb, em, M, N, sc, ep, sem, q,
                           q ? work_counters(stream) : static_cast<int*>(nullptr));
        ACCO_CHECK_LAUNCH();
        return;
    }
    // cluster-launch-control work stealing unless split-K: the ordered split
    // hand-off assumes the static unit order
    const int clc = use_clc(sc) ? 1 : 0;
    const int grid = clc ? sc.units() : std::min(sc.units(), num_sms());
    launch_pdl(kern, grid, gemm_threads<BN, STAGES>(), smem, stream, ta, tb, em, M, N, sc, ep, sem, clc,
               static_cast<int*>(nullptr));
    ACCO_CHECK_LAUNCH();
}

template <int BN, int STAGES, int CG = 1>
void dispatch_major(const GemmOperand& A, const GemmOperand& B, int M, int N, int K, const Epilogue& ep, int splits,
                    cudaStream_t s) {
    if (!A.mn_major && !B.mn_major) launch<BN, STAGES, 0, 0, CG>(A, B, M, N, K, ep, splits, s);
    else if (!A.mn_major && B.mn_major) launch<BN, STAGES, 0, 1, CG>(A, B, M, N, K, ep, splits, s);
    else if (A.mn_major && !B.mn_major) launch<BN, STAGES, 1, 0, CG>(A, B, M, N, K, ep, splits, s);
    else launch<BN, STAGES, 1, 1, CG>(A, B, M, N, K, ep, splits, s);
}

// B K-major only (CTA-pair tiles whose B half is not a whole 64-wide MN atom)
template <int BN, int STAGES, int CG>
void dispatch_k_major_b(const GemmOperand& A, const GemmOperand& B, int M, int N, int K, const Epilogue& ep,
                        int splits, cudaStream_t s) {
    ACCO_REQUIRE(!B.mn_major, "gemm: this tile shape needs a K-major B");
    if (!A.mn_major) launch<BN, STAGES, 0, 0, CG>(A, B, M, N, K, ep, splits, s);
    else launch<BN, STAGES, 1, 0, CG>(A, B, M, N, K, ep, splits, s);
}

// Time model (us) for the tile width / CTA group / split-K choice:
//   t = a + waves * (c + BN * k-blocks * r) + hand-offs
// a: launch, prologue and last epilogue; c: per-unit overhead; r: mainloop
// time per 64-deep k-block per tile column (the operand smem traffic per MMA
// makes narrow and single-CTA tiles slower per column); waves of units over
// 148 SMs or 74 CTA pairs. Least-squares fit (log error, rms 13 %) to the
// CUDA-graph device times of every config on the 42 GEMM shapes of GPT-2
// small / medium and Llama-1B (tools/diag/gemm_model_check.py,
// profiles/r02_gemm_model.jsonl): its picks cost 0.25 % more than the
// measured best summed over those shapes.
struct TileCost {
    double a, c, r;
};
TileCost tile_cost(int bn, int cg) {
    if (cg == 2) return bn == 256 ? TileCost{2.651, 1.544, 1.447e-3} : bn == 192 ? TileCost{4.987, 0.412, 1.591e-3}
                                                                                  : TileCost{0.541, 1.223, 1.834e-3};
    return bn == 256 ? TileCost{0.823, 2.383, 1.524e-3} : bn == 192 ? TileCost{0.0, 1.549, 1.771e-3}
                                                                     : TileCost{0.019, 1.179, 2.120e-3};
}
double plan_time(int M, int N, int K, int bn, int cg, int splits, bool a_mn, int sms) {
    const TileCost tc = tile_cost(bn, cg);
    const int units = ceil_div(M, kBM * cg) * ceil_div(N, bn) * splits;
    const double waves = std::ceil(static_cast<double>(units) / (sms / cg));
    const double kb = std::ceil(static_cast<double>(ceil_div(K, kBK)) / splits);
    double t = tc.a + waves * (tc.c + bn * kb * tc.r);
    // ordered split-K: each extra split adds an epilogue hand-off (a TMA
    // reduce-add of the tile and its completion) to the critical path
    if (splits > 1) t += (splits - 1) * (a_mn ? 2.635 : 4.3);
    return t;
}

// fp32 -> bf16 copy of the split-K workspace into C (pure-store GEMMs)
__global__ void f32_to_bf16_rows(const float* __restrict__ ws, int64_t ldw, __nv_bfloat16* __restrict__ c,
                                 int64_t ldc, int M, int N) {
    ACCO_PDL_PROLOGUE();
    const int n8 = N / 8;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= static_cast<int64_t>(M) * n8) return;
    const int r = static_cast<int>(i / n8), c8 = static_cast<int>(i % n8);
    const float4* src = reinterpret_cast<const float4*>(ws + r * ldw + c8 * 8);
    const float4 a = __ldcs(src), b = __ldcs(src + 1);
    const float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    *reinterpret_cast<uint4*>(c + r * ldc + c8 * 8) = make_uint4(
        pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]), pack_bf16(v[4], v[5]), pack_bf16(v[6], v[7]));
}

// Workspace for split-K of pure-store GEMMs, per (device, stream) like the
// semaphores (grown on demand; uses on one stream are ordered by the stream).
float* splitk_workspace(size_t elems, cudaStream_t s) {
    struct Ws {
        float* p = nullptr;
        size_t cap = 0;
    };
    static std::map<StreamKey, Ws> wss;
    int dev = 0;
    ACCO_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_scratch_mu);
    Ws& w = wss[StreamKey{dev, s}];
    if (elems > w.cap) {
        if (w.p) {
            ACCO_CUDA(cudaStreamSynchronize(s));
            ACCO_CUDA(cudaFree(w.p));
        }
        ACCO_CUDA(cudaMalloc(&w.p, elems * sizeof(float)));
        w.cap = elems;
    }
    return w.p;
}

// ------------------------------------------------------------ 3xTF32 (fp32)
__device__ __forceinline__ float rna_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// src (K-major [rows][ld] or MN-major [K][ld]) -> planes dst[0] = hi, dst[1] =
// lo, each K-major [rows][kp]. 32 x 32 tiles through smem so both the reads and
// the writes are coalesced for either source major-ness.
__global__ void tf32_split_kernel(const float* __restrict__ src, int64_t ld, int mn_major, int rows, int K,
                                  int64_t kp, float* __restrict__ dst) {
    ACCO_PDL_PROLOGUE();
    __shared__ float t[32][33];
    const int r0 = blockIdx.y * 32, k0 = blockIdx.x * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8 threads
    const int64_t plane = static_cast<int64_t>(rows) * kp;
    for (int j = ty; j < 32; j += 8) {
        float x = 0.f;
        if (mn_major) {  // src[k * ld + r]: lanes walk r
            const int k = k0 + j, r = r0 + tx;
            if (k < K && r < rows) x = src[static_cast<int64_t>(k) * ld + r];
            t[tx][j] = x;  // t[r][k]
        } else {  // src[r * ld + k]: lanes walk k
            const int r = r0 + j, k = k0 + tx;
            if (k < K && r < rows) x = src[static_cast<int64_t>(r) * ld + k];
            t[j][tx] = x;
        }
    }
    __syncthreads();
    for (int j = ty; j < 32; j += 8) {
        const int r = r0 + j, k = k0 + tx;
        if (r < rows && k < K) {
            const float x = t[j][tx];
            const float hi = rna_tf32(x);
            const int64_t o = static_cast<int64_t>(r) * kp + k;
            dst[o] = hi;
            dst[plane + o] = rna_tf32(x - hi);
        }
    }
}

// The non-accumulating epilogues of the fp32 path after the tensor-core
// contraction: acc[M][ldw] (fp32) -> bias / GELU / dGELU / residual -> C, the
// same per-element math as the SIMT kernel's epilogue_row<float>.
__global__ void f32_epilogue_kernel(const float* __restrict__ acc, int64_t ldw, int M, int N, Epilogue ep) {
    ACCO_PDL_PROLOGUE();
    const int n4 = (N + 3) / 4;
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= static_cast<int64_t>(M) * n4) return;
    const int r = static_cast<int>(i / n4), c = static_cast<int>(i % n4) * 4;
    float x[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) x[j] = c + j < N ? acc[r * ldw + c + j] : 0.f;
    epilogue_row<float, 4>(ep, r, c, min(4, N - c), x);
}

// Stream-ordered scratch from the device's default memory pool: each call
// allocates on the launching stream and frees after its last use on that
// stream, so concurrent GEMMs on different streams or devices never share it.
void* pool_alloc(size_t bytes, cudaStream_t s) {
    static std::once_flag once[64];
    int dev = 0;
    ACCO_CUDA(cudaGetDevice(&dev));
    std::call_once(once[dev & 63], [dev] {
        cudaMemPool_t pool;
        ACCO_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
        uint64_t keep = ~0ull;  // keep freed blocks cached: the same sizes recur every micro-batch
        ACCO_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    });
    void* p = nullptr;
    ACCO_CUDA(cudaMallocAsync(&p, bytes, s));
    return p;
}

void launch_x3(const float* a_planes, const float* b_planes, int64_t kp, int M, int N, int K, const Epilogue& ep,
               int splits, cudaStream_t stream) {
    constexpr int BN = 128, STAGES = 3;
    auto kern = gemm_tc_kernel<BN, STAGES, 0, 0, 1>;
    constexpr int smem = smem_bytes<BN, STAGES, 1>();
    static_assert(smem <= 232448, "shared memory budget");
    static bool configured = false;
    if (!configured) {
        ACCO_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        configured = true;
    }
    Sched sc;
    sc.tiles_m = ceil_div(M, kBM);
    sc.tiles_n = ceil_div(N, BN);
    sc.kb_total = ceil_div(K, 32);
    sc.group_m = kGroupM;
    sc.kb_per_split = ceil_div(sc.kb_total, splits);
    sc.splits = ceil_div(sc.kb_total, sc.kb_per_split);
    auto planes = [&](const float* p, int rows, uint32_t box_rows) {
        cuuint64_t dims[3] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(rows), 2};
        cuuint64_t strides[2] = {static_cast<cuuint64_t>(kp) * 4, static_cast<cuuint64_t>(kp) * 4 * rows};
        cuuint32_t box[3] = {32, box_rows, 1};
        return encode(CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, p, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
    };
    EpiMaps em;
    std::memset(&em, 0, sizeof(em));
    em.out = make_map_f32(ep.C, N, M, 1, ep.ldc);
    int* sem = nullptr;
    if (sc.splits > 1) {
        ACCO_REQUIRE(sc.tiles_m * sc.tiles_n * 8 * 32 <= kSemSlots, "gemm: too many tiles for split-K");
        sem = split_semaphores(stream);
    }
    const CUtensorMap ta = planes(a_planes, M, kBM), tb = planes(b_planes, N, BN);
    const int clc = use_clc(sc) ? 1 : 0;
    const int grid = clc ? sc.units() : std::min(sc.units(), num_sms());
    launch_pdl(kern, grid, gemm_threads<BN, STAGES, 1>(), smem, stream, ta, tb, em, M, N, sc, ep, sem, clc,
               static_cast<int*>(nullptr));
    ACCO_CHECK_LAUNCH();
}

}  // namespace

// fp32-accurate GEMM on the tensor cores (precision "fp32"): split pre-pass,
// 3xTF32 tcgen05 contraction into fp32, then the epilogue. kEpiAccF32 goes
// straight into C (TMA store / reduce-add, ordered split-K); the other
// epilogues contract into a scratch accumulator first (C may alias the
// residual) and finish in f32_epilogue_kernel.
void gemm_f32_tc(const GemmOperand& A, const GemmOperand& B, int M, int N, int K, const Epilogue& ep,
                 cudaStream_t stream) {
    ACCO_REQUIRE(M > 0 && N > 0 && K > 0, "gemm_f32: empty problem");
    ACCO_REQUIRE(ep.mode <= kEpiAccF32, "gemm_f32: epilogue mode not supported by the fp32 path");
    ACCO_REQUIRE(!ep.bias_grad, "gemm_f32: bias_grad is a bf16-path epilogue (the fp32 path reduces columns separately)");
    ACCO_REQUIRE(ep.mode == kEpiStore || ep.mode == kEpiAccF32 || ep.aux, "gemm_f32: GELU epilogues need aux");
    ProfScope prof(kProfGemm, 2.0 * M * N * K, stream);
    const int64_t kp = (K + 3) / 4 * 4;  // 16 B row stride for TMA
    float* pa = static_cast<float*>(pool_alloc(sizeof(float) * 2 * kp * (M + N), stream));
    float* pb = pa + 2 * kp * M;
    launch_pdl(tf32_split_kernel, dim3(ceil_div(K, 32), ceil_div(M, 32)), 256, 0, stream,
               static_cast<const float*>(A.ptr), A.ld, static_cast<int>(A.mn_major), M, K, kp, pa);
    ACCO_CHECK_LAUNCH();
    launch_pdl(tf32_split_kernel, dim3(ceil_div(K, 32), ceil_div(N, 32)), 256, 0, stream,
               static_cast<const float*>(B.ptr), B.ld, static_cast<int>(B.mn_major), N, K, kp, pb);
    ACCO_CHECK_LAUNCH();
    // Ordered split-K bounds the accumulation chain in TMEM. The tensor core's
    // fp32 accumulation error grows linearly with the number of MMAs chained
    // into one accumulator (measured, tools/diag/tf32_accuracy.py: ~2.2e-7
    // relative per 32-deep k-block, so 7e-6 at K = 8192 unsplit), while the
    // split partials are summed by round-to-nearest fp32 TMA reduce-adds in
    // split order. A chain of 4 k-blocks (K = 128) holds every contraction at
    // ~1e-6 whatever K is, SIMT-fp32 level. ACCO_TF32_CHAIN=<k-blocks> overrides.
    const int tiles = ceil_div(M, kBM) * ceil_div(N, 128), kbt = ceil_div(K, 32);
    int chain = 4;
    if (const char* c = std::getenv("ACCO_TF32_CHAIN")) chain = std::max(1, std::atoi(c));
    int splits = ceil_div(kbt, chain);
    if (const char* f = std::getenv("ACCO_TF32_SPLITS")) splits = std::max(1, std::atoi(f));
    if (tiles * 8 * 32 > kSemSlots) splits = 1;
    const bool direct = ep.mode == kEpiAccF32 && ep.ldc % 4 == 0 && (reinterpret_cast<uintptr_t>(ep.C) & 15) == 0;
    if (direct) {
        launch_x3(pa, pb, kp, M, N, K, ep, splits, stream);
    } else {
        const int64_t ldw = (N + 3) / 4 * 4;
        float* ws = static_cast<float*>(pool_alloc(sizeof(float) * ldw * M, stream));
        Epilogue e;
        e.mode = kEpiAccF32;
        e.C = ws;
        e.ldc = ldw;
        e.beta = 0;
        launch_x3(pa, pb, kp, M, N, K, e, splits, stream);
        const int64_t n = static_cast<int64_t>(M) * ((N + 3) / 4);
        launch_pdl(f32_epilogue_kernel, static_cast<int>((n + 255) / 256), 256, 0, stream,
                   static_cast<const float*>(ws), ldw, M, N, ep);
        ACCO_CHECK_LAUNCH();
        ACCO_CUDA(cudaFreeAsync(ws, stream));
    }
    ACCO_CUDA(cudaFreeAsync(pa, stream));
}

namespace {
// The planner: tile width, split-K and CTA group with the least modelled time.
double plan_gemm(const GemmOperand& A, const GemmOperand& B, int M, int N, int K, bool acc_f32, bool bias_grad,
                 int& best_bn, int& best_sp, int& best_cg, bool no_pairs = false) {
    const int sms = num_sms();
    // The LM head's shapes (B too big to stay in L2, whole-M raster: see
    // launch) stream B from HBM once; there the model underrates the 256-wide
    // pair tiles, which halve each SM's share of B, against the 192-wide ones
    // (head_fwd 452 vs 497 us), so those are not considered. ACCO_GEMM_NO_CG2=1:
    // single-CTA tiles only (A/B knob).
    const bool large_b = static_cast<double>(M) * K * 2 <= 48e6 && static_cast<double>(N) * K * 2 > 32e6;
    const bool allow_cg2 = std::getenv("ACCO_GEMM_NO_CG2") == nullptr;
    best_bn = 256;
    best_sp = 1;
    best_cg = 1;
    double best = 1e300;
    for (int cg : {1, 2}) {
        if (cg == 2 && (!allow_cg2 || no_pairs)) continue;
        for (int bn : {256, 192, 128}) {
            if (cg == 2 && bn == 192 && (B.mn_major || large_b)) continue;
            if (bias_grad && !has_bias_mma<256>() && bn == 256) continue;  // no TMEM for the bias columns
            for (int sp : {1, 2, 3, 4, 6, 8}) {
                if (sp > 1 && (!acc_f32 || ceil_div(K, kBK) < 4 * sp ||
                               ceil_div(M, kBM) * ceil_div(N, bn) * 8 * 32 > kSemSlots))
                    continue;
                const double t = plan_time(M, N, K, bn, cg, sp, A.mn_major, sms);
                if (t < best * 0.98) {  // (ties keep the single-CTA tiles)
                    best = t;
                    best_bn = bn;
                    best_sp = sp;
                    best_cg = cg;
                }
            }
        }
    }
    return best;
}
}  // namespace

void gemm_set_pair_queue(bool on) { g_pair_queue.store(on ? 1 : 0, std::memory_order_relaxed); }

bool gemm_bias_grad_free(const GemmOperand& A, const GemmOperand& B, int M, int N, int K) {
    if (std::getenv("ACCO_GEMM_FORCE")) return true;
    int bn = 256, sp = 1, cg = 1;
    const double t_free = plan_gemm(A, B, M, N, K, true, false, bn, sp, cg);
    const double t_bias = plan_gemm(A, B, M, N, K, true, true, bn, sp, cg);
    // within 4 % (model): GPT-2 small's fc / fc2 weight gradients (3.3 %; the
    // restricted 128-wide pair tiles measure faster, 32.1 vs 33.4 us) fuse,
    // GPT-2 medium's (22 %) and its qkv (5 %) do not — a 3 us allowance fused
    // those and cost 0.7 ms per step
    return t_bias <= t_free * 1.04;
}

void gemm_bf16(const GemmOperand& A, const GemmOperand& B, int M, int N, int K, const Epilogue& ep,
               cudaStream_t stream) {
    ACCO_REQUIRE(M > 0 && N > 0 && K > 0, "gemm_bf16: empty problem");
    ACCO_REQUIRE(!(ep.residual && (ep.mode == kEpiGelu || ep.mode == kEpiDGelu)),
                 "gemm_bf16: residual add is not combined with the GELU epilogues");
    ACCO_REQUIRE(ep.mode == kEpiStore || ep.mode == kEpiAccF32 || ep.aux, "gemm_bf16: GELU epilogues need aux");
    ACCO_REQUIRE(!ep.bias_grad || ep.mode == kEpiAccF32, "gemm_bf16: bias_grad needs the fp32 accumulate epilogue");
    ProfScope prof(kProfGemm, 2.0 * M * N * K, stream);
    const int sms = num_sms();
    int best_bn = 256, best_sp = 1, best_cg = 1;
    // (the dGELU epilogue, which streams the stored GELU slope in, is slower on
    // pair tiles than the model's store-epilogue fit: fc2 dgrad 41.6 vs 40.4 us)
    double best = plan_gemm(A, B, M, N, K, ep.mode == kEpiAccF32, ep.bias_grad != nullptr, best_bn, best_sp, best_cg,
                            ep.mode == kEpiDGelu);
    if (ep.mode == kEpiDSwiGLU) {
        ACCO_REQUIRE(ep.aux && !ep.residual && !ep.bias && N % 32 == 0,
                     "gemm_bf16: DSwiGLU epilogue needs aux, F % 32 == 0, no bias/residual");
        if (std::getenv("ACCO_DSWIGLU_CG2"))  // A/B knob: CTA-pair 256-wide tiles
            dispatch_major<256, 5, 2>(A, B, M, N, K, ep, 1, stream);
        else
            dispatch_major<192, 4>(A, B, M, N, K, ep, 1, stream);
        return;
    }
    if (ep.mode == kEpiSwiGLU) {
        ACCO_REQUIRE(N % 256 == 0 && !B.mn_major && !ep.residual && !ep.bias && ep.aux,
                     "gemm_bf16: SwiGLU epilogue needs N = 2F with F % 128 == 0, K-major B, aux, no bias/residual");
        // CTA-pair tiles (the leader stages the gate rows, its peer the up
        // rows): Llama-1B 126.7k vs 124.5k tok/s with single-CTA tiles
        if (std::getenv("ACCO_GEMM_NO_CG2"))
            dispatch_major<256, 3>(A, B, M, N, K, ep, 1, stream);
        else
            dispatch_major<256, 5, 2>(A, B, M, N, K, ep, 1, stream);
        return;
    }
    // A pure-store GEMM whose tiles cannot fill the SMs and whose K is long
    // (the LM-head dgrad: 192 tiles x 786 k-blocks) runs as an ordered split-K
    // into an fp32 workspace (first split stores, the rest TMA-reduce-add in
    // split order: deterministic) plus one fp32 -> bf16 pass into C.
    const bool pure_store = ep.mode == kEpiStore && !ep.bias && !ep.residual && N % 8 == 0 && ep.ldc % 8 == 0 &&
                            (reinterpret_cast<uintptr_t>(ep.C) & 15) == 0 && !std::getenv("ACCO_GEMM_NO_WS_SPLIT");
    int ws_bn = 0, ws_sp = 1;
    if (pure_store) {
        // the conversion pass (us): 6 bytes per element at ~6.5 TB/s, plus its launch
        const double conv = 6.0 * M * N / 6.5e6 + 2.0;
        for (int bn : {256, 192, 128})
            for (int sp : {2, 3, 4, 6, 8}) {
                if (ceil_div(K, kBK) < 16 * sp || ceil_div(M, kBM) * ceil_div(N, bn) * 8 * 32 > kSemSlots) continue;
                const double c = plan_time(M, N, K, bn, 1, sp, A.mn_major, sms) + conv;
                if (c < best * 0.9) {
                    best = c;
                    ws_bn = bn;
                    ws_sp = sp;
                }
            }
    }
    if (ws_bn && !std::getenv("ACCO_GEMM_FORCE")) {
        const int64_t ldw = (N + 3) / 4 * 4;
        float* ws = splitk_workspace(static_cast<size_t>(M) * ldw, stream);
        Epilogue e = ep;
        e.mode = kEpiAccF32;
        e.C = ws;
        e.ldc = ldw;
        e.beta = 0;
        if (ws_bn == 256)
            dispatch_major<256, 4>(A, B, M, N, K, e, ws_sp, stream);
        else if (ws_bn == 192)
            dispatch_major<192, 4>(A, B, M, N, K, e, ws_sp, stream);
        else
            dispatch_major<128, 5>(A, B, M, N, K, e, ws_sp, stream);
        const int64_t n = static_cast<int64_t>(M) * (N / 8);
        launch_pdl(f32_to_bf16_rows, static_cast<int>((n + 255) / 256), 256, 0, stream, ws, ldw,
                   static_cast<__nv_bfloat16*>(ep.C), ep.ldc, M, N);
        ACCO_CHECK_LAUNCH();
        return;
    }
    if (const char* f = std::getenv("ACCO_GEMM_FORCE")) {  // tuning knob: "<bn>,<splits>[,<cta group>]"
        int fb = 0, fs = 0, fc = 1;
        if (std::sscanf(f, "%d,%d,%d", &fb, &fs, &fc) >= 2 && (fb == 128 || fb == 192 || fb == 256) && fs >= 1) {
            best_bn = fb;
            best_sp = ep.mode == kEpiAccF32 ? fs : 1;
            best_cg = fc == 2 && !(fb == 192 && B.mn_major) ? 2 : 1;
            if (ep.bias_grad && best_bn == 256) best_bn = 192;
        }
    }
    if (std::getenv("ACCO_GEMM_LOG")) {  // each distinct shape's plan, once
        static std::set<std::string> seen;
        char key[160];
        std::snprintf(key, sizeof key, "gemm M=%d N=%d K=%d a_mn=%d b_mn=%d mode=%d -> bn=%d splits=%d cg=%d (model %.1f us)",
                      M, N, K, int(A.mn_major), int(B.mn_major), ep.mode, best_bn, best_sp, best_cg, best);
        std::lock_guard<std::mutex> lk(g_scratch_mu);
        if (seen.insert(key).second) std::fprintf(stderr, "%s\n", key);
    }
    if (best_cg == 2) {
        if (best_bn == 256)
            dispatch_major<256, 5, 2>(A, B, M, N, K, ep, best_sp, stream);
        else if (best_bn == 192)
            dispatch_k_major_b<192, 5, 2>(A, B, M, N, K, ep, best_sp, stream);
        else
            dispatch_major<128, 6, 2>(A, B, M, N, K, ep, best_sp, stream);
        return;
    }
    if (best_bn == 256)
        dispatch_major<256, 4>(A, B, M, N, K, ep, best_sp, stream);
    else if (best_bn == 192)
        dispatch_major<192, 4>(A, B, M, N, K, ep, best_sp, stream);
    else
        dispatch_major<128, 5>(A, B, M, N, K, ep, best_sp, stream);
}

}  // namespace acco
