// bf16 GEMM on the 5th-generation tensor cores (sm_100a).
//
// One CTA computes a 128 x BN output tile:
//   warp 0  : TMA producer (one elected lane) — K-major or MN-major operand
//             tiles, 128B-swizzled, into a STAGES-deep smem ring
//   warp 1  : MMA issuer (one lane) — tcgen05.mma.cta_group::1.kind::f16,
//             fp32 accumulator in TMEM, tcgen05.commit frees smem slots
//   warp 2  : TMEM allocator
//   warps 4-7: epilogue — tcgen05.ld TMEM -> registers -> fused epilogue
//             (bias / GELU / dGELU / residual / fp32 gradient accumulate)
//
// This is the K1/K3 kernel of SURVEY.md §2.3: forward (both operands K-major),
// dgrad (B MN-major) and wgrad (both MN-major, fp32 beta=1 epilogue into the
// gradient-accumulation buffer, i.e. Bundle::add of
// /root/reference/proj/src/protocols.cpp:61-66 fused into the GEMM).
#include "common.cuh"
#include "epilogue.cuh"
#include "gemm.h"

#include <mutex>

namespace acco {
namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;  // 64 bf16 = 128 bytes: one SW128 row
constexpr int kThreads = 256;

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t addr, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t a = smem_u32(bar);
    while (!mbar_try_wait(a, parity)) {
    }
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t* v) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
          "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
          "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
          "=r"(v[31])
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

// Instruction descriptor for kind::f16: bf16 x bf16 -> fp32.
__host__ __device__ constexpr uint32_t idesc_bf16(int m, int n, int a_mn, int b_mn) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(a_mn) << 15) |
           (static_cast<uint32_t>(b_mn) << 16) | (static_cast<uint32_t>(n >> 3) << 17) |
           (static_cast<uint32_t>(m >> 4) << 24);
}

template <int BN, int STAGES>
constexpr int smem_bytes() {
    return 1024 /*align slack*/ + STAGES * (kBM + BN) * kBK * 2 + (2 * STAGES + 1) * 8 + 16;
}

// --------------------------------------------------------------------- kernel
template <int BN, int STAGES, int A_MN, int B_MN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   int M, int N, int K, Epilogue ep) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                               ~static_cast<uintptr_t>(1023));
    constexpr int A_BYTES = kBM * kBK * 2;
    constexpr int B_BYTES = BN * kBK * 2;
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tmem_full = empty + STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int m0 = blockIdx.y * kBM;
    const int n0 = blockIdx.x * BN;
    const int num_kb = (K + kBK - 1) / kBK;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tmem_full, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(BN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_d = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            for (int kb = 0; kb < num_kb; ++kb) {
                const int s = kb % STAGES;
                const uint32_t ph = (kb / STAGES) & 1;
                mbar_wait(&empty[s], ph ^ 1);
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
                } else {
                    tma_load_2d(b_dst, &tmB, &full[s], kb * kBK, n0);
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = idesc_bf16(kBM, BN, A_MN, B_MN);
            for (int kb = 0; kb < num_kb; ++kb) {
                const int s = kb % STAGES;
                const uint32_t ph = (kb / STAGES) & 1;
                mbar_wait(&full[s], ph);
                tc_fence_after();
                const uint32_t a_base = smem_u32(sA + s * A_BYTES);
                const uint32_t b_base = smem_u32(sB + s * B_BYTES);
#pragma unroll
                for (int kk = 0; kk < kBK / 16; ++kk) {
                    // K-major: advance 16 elements (32 B) inside the 128B swizzle row.
                    // MN-major: advance 16 K-rows = two 8-row atoms (2048 B).
                    uint64_t ad = A_MN ? sdesc(a_base + kk * 2048, 64 * kBK * 2, 1024)
                                       : sdesc(a_base + kk * 32, 16, 1024);
                    uint64_t bd = B_MN ? sdesc(b_base + kk * 2048, 64 * kBK * 2, 1024)
                                       : sdesc(b_base + kk * 32, 16, 1024);
                    umma_bf16(tmem_d, ad, bd, idesc, (kb | kk) != 0);
                }
                umma_commit(&empty[s]);
            }
            umma_commit(tmem_full);
        }
    } else if (warp >= 4) {
        const int wq = warp - 4;
        mbar_wait(tmem_full, 0);
        tc_fence_after();
        const int row = m0 + wq * 32 + lane;
        for (int c = 0; c < BN; c += 32) {
            uint32_t v[32];
            tmem_ld32(tmem_d + (static_cast<uint32_t>(wq * 32) << 16) + c, v);
            const int col = n0 + c;
            if (row < M && col < N) {
                float x[32];
#pragma unroll
                for (int i = 0; i < 32; ++i) x[i] = __uint_as_float(v[i]);
                epilogue_row<__nv_bfloat16, 32>(ep, row, col, min(32, N - col), x);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_d), "r"(BN));
    }
}

// ----------------------------------------------------------------- host side
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                              CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        ACCO_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !p)
            throw Error(kCudaError, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<EncodeFn>(p);
    });
    return fn;
}

// 2-D bf16 tensor map: `inner` contiguous elements per row, `outer` rows.
CUtensorMap make_map(const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld_elems,
                     uint32_t box_inner, uint32_t box_outer) {
    ACCO_REQUIRE((reinterpret_cast<uintptr_t>(ptr) & 15) == 0, "gemm: operand not 16B aligned");
    ACCO_REQUIRE((ld_elems * 2) % 16 == 0, "gemm: leading dimension must be a multiple of 8");
    CUtensorMap m;
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {ld_elems * 2};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims,
                             strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw Error(kCudaError, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
    return m;
}

// Tensor map for an operand with `rows` (M or N) and reduction extent K.
CUtensorMap operand_map(const GemmOperand& op, int rows, int K, int tile_rows) {
    if (op.mn_major)  // stored [K][rows]: inner = rows
        return make_map(op.ptr, rows, K, op.ld, 64, kBK);
    return make_map(op.ptr, K, rows, op.ld, kBK, tile_rows);  // stored [rows][K]
}

template <int BN, int STAGES, int A_MN, int B_MN>
void launch(const GemmOperand& A, const GemmOperand& B, int M, int N, int K, const Epilogue& ep,
            cudaStream_t stream) {
    auto kern = gemm_tc_kernel<BN, STAGES, A_MN, B_MN>;
    constexpr int smem = smem_bytes<BN, STAGES>();
    static bool configured = false;  // per instantiation
    if (!configured) {
        ACCO_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        configured = true;
    }
    CUtensorMap ta = operand_map(A, M, K, kBM);
    CUtensorMap tb = operand_map(B, N, K, BN);
    dim3 grid(ceil_div(N, BN), ceil_div(M, kBM));
    kern<<<grid, kThreads, smem, stream>>>(ta, tb, M, N, K, ep);
    ACCO_CHECK_LAUNCH();
}

template <int BN, int STAGES>
void dispatch_major(const GemmOperand& A, const GemmOperand& B, int M, int N, int K,
                    const Epilogue& ep, cudaStream_t s) {
    if (!A.mn_major && !B.mn_major) launch<BN, STAGES, 0, 0>(A, B, M, N, K, ep, s);
    else if (!A.mn_major && B.mn_major) launch<BN, STAGES, 0, 1>(A, B, M, N, K, ep, s);
    else if (A.mn_major && !B.mn_major) launch<BN, STAGES, 1, 0>(A, B, M, N, K, ep, s);
    else launch<BN, STAGES, 1, 1>(A, B, M, N, K, ep, s);
}

}  // namespace

void gemm_bf16(const GemmOperand& A, const GemmOperand& B, int M, int N, int K, const Epilogue& ep,
               cudaStream_t stream) {
    ACCO_REQUIRE(M > 0 && N > 0 && K > 0, "gemm_bf16: empty problem");
    ProfScope prof(kProfGemm, 2.0 * M * N * K, stream);
    // Wide tiles amortise the A re-reads; narrow N (e.g. attn-proj, N=768) keeps
    // enough CTAs in flight to fill 148 SMs.
    const long long tiles256 = static_cast<long long>(ceil_div(N, 256)) * ceil_div(M, kBM);
    if (N >= 256 && tiles256 >= 148)
        dispatch_major<256, 4>(A, B, M, N, K, ep, stream);
    else
        dispatch_major<128, 6>(A, B, M, N, K, ep, stream);
}

}  // namespace acco
