// Round-trip latencies of the synchronisation the attention kernels chain per
// tile (B200, sm_100a): (1) 8 back-to-back 128x128x16 MMAs + tcgen05.commit ->
// mbarrier wait, (2) an mbarrier ping-pong between two warps, each with
// mbarrier.try_wait suspend-time hints 0 and 20000 ns. Diagnostic only.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/diag/sync_latency.cu -o tools/diag/sync_latency.bin
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
    uint64_t d = static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>(1) << 16;
    d |= static_cast<uint64_t>(1024 >> 4) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(2) << 61;
    return d;
}
template <int HINT>
__device__ __forceinline__ void wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok) {
        if (HINT)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\tselp.u32 %0,1,0,p;\n\t}"
                         : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity), "r"(HINT) : "memory");
        else
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                         : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    }
}
__device__ __forceinline__ void arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

template <int HINT, int NMMA>
__global__ void lat(int rounds, unsigned long long* out) {
    __shared__ __align__(1024) uint8_t sm[2 * 16384];
    __shared__ uint64_t bar[3];
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 2 * 16384 / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x == 0) {
        for (int i = 0; i < 3; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tslot;
    unsigned long long t0, t1;
    if (warp == 0 && lane == 0) {  // MMA group + commit -> wait, serially
        constexpr uint32_t id = (1u << 4) | (1u << 7) | (1u << 10) | (128u >> 3 << 17) | (128u >> 4 << 24);
        const uint64_t ad = sdesc(smem_u32(sm)), bd = sdesc(smem_u32(sm + 16384));
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        for (int r = 0; r < rounds; ++r) {
            for (int k = 0; k < NMMA; ++k)
                asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                             ::"r"(tmem), "l"(ad + 2 * (k & 3)), "l"(bd + 2 * (k & 3)), "r"(id), "r"(1u));
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar[0])) : "memory");
            wait<HINT>(&bar[0], r & 1);
        }
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        out[0] = (t1 - t0) / rounds;
    }
    __syncthreads();
    // ping-pong between warp 0 and warp 1
    if (lane == 0 && warp < 2) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        for (int r = 0; r < rounds; ++r) {
            if (warp == 0) {
                arrive(&bar[1]);
                wait<HINT>(&bar[2], r & 1);
            } else {
                wait<HINT>(&bar[1], r & 1);
                arrive(&bar[2]);
            }
        }
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        if (warp == 0) out[1] = (t1 - t0) / rounds;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

template <int HINT, int NMMA>
void run() {
    unsigned long long* d;
    cudaMallocManaged(&d, 16);
    lat<HINT, NMMA><<<1, 128>>>(1000, d);
    cudaDeviceSynchronize();
    lat<HINT, NMMA><<<1, 128>>>(1000, d);
    cudaError_t e = cudaDeviceSynchronize();
    printf("{\"suspend_hint_ns\": %d, \"mmas_per_group\": %d, \"mma_group_commit_wait_ns\": %llu, "
           "\"mbarrier_pingpong_roundtrip_ns\": %llu, \"mma_only_ns_est\": %.0f, \"err\": \"%s\"}\n",
           HINT, NMMA, d[0], d[1], NMMA * 35.5, cudaGetErrorString(e));
    cudaFree(d);
}

int main() {
    run<0, 1>();
    run<0, 8>();
    run<20000, 1>();
    run<20000, 8>();
    run<2000, 8>();
    return 0;
}
