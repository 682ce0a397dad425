// Shared device/host helpers for the ACCO B200 library (sm_100a only).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <utility>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "paper_2406_02613_b200 targets sm_100a only"
#endif

namespace acco {

// Thrown inside the library; the C-ABI layer converts it to a status code
// (see include/acco.h) and stores the message for acco_last_error().
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

enum Status : int {
    kOk = 0,
    kVerifyFail = 1,     // accosim exit code 1
    kInvalidArg = 2,     // accosim exit code 2 (std::invalid_argument)
    kDiverged = 3,       // accosim exit code 3
    kCudaError = 4,      // B200-only: CUDA / NCCL failure
    kLogicError = 5,     // std::logic_error in the reference (invariants)
};

#define ACCO_CUDA(expr)                                                                 \
    do {                                                                                \
        cudaError_t _e = (expr);                                                        \
        if (_e != cudaSuccess)                                                          \
            throw ::acco::Error(::acco::kCudaError, std::string(#expr) + ": " +         \
                                                        cudaGetErrorString(_e) + " @" + \
                                                        __FILE__ + ":" + std::to_string(__LINE__)); \
    } while (0)

#define ACCO_CHECK_LAUNCH()              \
    do {                                 \
        ACCO_CUDA(cudaGetLastError());   \
        ::acco::count_launch();          \
    } while (0)

#define ACCO_REQUIRE(cond, msg)                                                  \
    do {                                                                         \
        if (!(cond)) throw ::acco::Error(::acco::kInvalidArg, std::string(msg)); \
    } while (0)

inline int ceil_div(long long a, long long b) { return static_cast<int>((a + b - 1) / b); }

// ------------------------------------------------ programmatic dependent launch
// Every kernel of the training step starts with ACCO_PDL_PROLOGUE (or calls
// pdl_trigger / pdl_wait itself after a prologue that touches no global
// data): it lets the next kernel in the stream launch as soon as all of this
// grid's CTAs are running, and blocks until the previous grid has completed
// and its memory is visible. Launched through launch_pdl, a kernel's launch
// latency and prologue (barrier init, TMEM alloc, descriptor prefetch) then
// overlap the previous kernel's tail. ACCO_NO_PDL=1 disables the attribute
// (the device instructions are no-ops without it).
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
#define ACCO_PDL_PROLOGUE() \
    do {                    \
        ::acco::pdl_trigger(); \
        ::acco::pdl_wait();    \
    } while (0)

bool pdl_enabled();

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
    if (e != cudaSuccess) throw Error(kCudaError, std::string("launch_pdl: ") + cudaGetErrorString(e));
}

// launch_pdl with a 1-D thread-block cluster of `cluster` CTAs (CTA pairs of
// the 2-SM tcgen05 kernels: consecutive blockIdx.x share a TPC)
template <typename... KArgs, typename... Args>
inline void launch_pdl_cluster(void (*kern)(KArgs...), int cluster, dim3 grid, dim3 block, size_t smem,
                               cudaStream_t s, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = cluster;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
    if (e != cudaSuccess) throw Error(kCudaError, std::string("launch_pdl_cluster: ") + cudaGetErrorString(e));
}

// Number of SMs on the current device (148 on B200); cached per process.
int num_sms();

// Every kernel launch of this library increments a process-wide counter
// (acco_launch_count), so benches can report how many of *our* kernels ran.
void count_launch();

// Optional per-class kernel timing with CUDA events on the launching stream
// (acco_prof_*): used by bench.py for the live roofline numbers.
enum ProfClass : int {
    kProfGemm = 0,    // work = algorithmic flops
    kProfAttn = 1,    // flops
    kProfOpt = 2,     // algorithmic bytes
    kProfReduce = 3,  // bias / LN-parameter column reductions: bytes
    kProfNorm = 4,    // LayerNorm fwd/bwd: bytes
    kProfCE = 5,      // cross-entropy fwd+bwd: bytes
    kProfEmbed = 6,   // token gather, embedding fwd/bwd: bytes
    kProfOther = 7,
    kProfClasses = 8
};
bool prof_on();
void prof_record(int cls, double work, cudaEvent_t a, cudaEvent_t b);
cudaEvent_t prof_event();
struct ProfScope {
    int cls;
    double work;
    cudaStream_t s;
    cudaEvent_t a = nullptr;
    ProfScope(int c, double w, cudaStream_t st) : cls(c), work(w), s(st) {
        if (prof_on()) {
            a = prof_event();
            cudaEventRecord(a, s);
        }
    }
    ~ProfScope() {
        if (a) {
            cudaEvent_t b = prof_event();
            cudaEventRecord(b, s);
            prof_record(cls, work, a, b);
        }
    }
};

// Packed fp32 pair arithmetic (sm_100a FFMA2 / FADD2 / FMUL2): one issue slot
// for two lanes' worth of math.
__device__ __forceinline__ float2 fma_f32x2(float2 a, float2 b, float2 c) {
    uint64_t r;
    asm("{\n\t.reg .b64 ra, rb, rc;\n\t"
        "mov.b64 ra, {%1, %2};\n\t"
        "mov.b64 rb, {%3, %4};\n\t"
        "mov.b64 rc, {%5, %6};\n\t"
        "fma.rn.f32x2 %0, ra, rb, rc;\n\t}\n"
        : "=l"(r)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    float2 o;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(o.x), "=f"(o.y) : "l"(r));
    return o;
}
__device__ __forceinline__ float2 add_f32x2(float2 a, float2 b) {
    uint64_t r;
    asm("{\n\t.reg .b64 ra, rb;\n\t"
        "mov.b64 ra, {%1, %2};\n\t"
        "mov.b64 rb, {%3, %4};\n\t"
        "add.rn.f32x2 %0, ra, rb;\n\t}\n"
        : "=l"(r)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    float2 o;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(o.x), "=f"(o.y) : "l"(r));
    return o;
}
__device__ __forceinline__ float2 mul_f32x2(float2 a, float2 b) {
    uint64_t r;
    asm("{\n\t.reg .b64 ra, rb;\n\t"
        "mov.b64 ra, {%1, %2};\n\t"
        "mov.b64 rb, {%3, %4};\n\t"
        "mul.rn.f32x2 %0, ra, rb;\n\t}\n"
        : "=l"(r)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
    float2 o;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(o.x), "=f"(o.y) : "l"(r));
    return o;
}

}  // namespace acco
