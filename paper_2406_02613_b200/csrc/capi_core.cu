// C-ABI plumbing: error state, device info, and the raw GEMM entry point.
#include "acco.h"
#include "common.cuh"
#include "capi_util.h"
#include "gemm.h"

#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

namespace acco {

static thread_local std::string g_last_error;

void set_last_error(const std::string& m) { g_last_error = m; }

int num_sms() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        ACCO_CUDA(cudaGetDevice(&dev));
        ACCO_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
    }
    return n;
}

bool pdl_enabled() {
    static const bool on = std::getenv("ACCO_NO_PDL") == nullptr;
    return on;
}

static std::atomic<long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

namespace {
struct ProfEntry {
    int cls;
    double work;
    cudaEvent_t a, b;
};
std::mutex g_prof_mu;
std::atomic<bool> g_prof_on{false};
std::vector<ProfEntry> g_prof;
std::vector<cudaEvent_t> g_prof_pool;
size_t g_prof_next = 0;
}  // namespace

bool prof_on() { return g_prof_on.load(std::memory_order_relaxed); }

cudaEvent_t prof_event() {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    if (g_prof_next == g_prof_pool.size()) {
        cudaEvent_t e;
        ACCO_CUDA(cudaEventCreate(&e));
        g_prof_pool.push_back(e);
    }
    return g_prof_pool[g_prof_next++];
}

void prof_record(int cls, double work, cudaEvent_t a, cudaEvent_t b) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof.push_back({cls, work, a, b});
}

}  // namespace acco

using namespace acco;

extern "C" {

long long acco_launch_count(void) { return g_launches.load(); }

void acco_prof_enable(int on) { g_prof_on.store(on != 0); }

int acco_prof_reset(void) {
    return guarded([&] {
        std::lock_guard<std::mutex> lk(g_prof_mu);
        g_prof.clear();
        g_prof_next = 0;
    });
}

int acco_prof_read(double* ms, double* work, long long* launches) {
    return guarded([&] {
        std::lock_guard<std::mutex> lk(g_prof_mu);
        for (int c = 0; c < kProfClasses; ++c) {
            ms[c] = 0;
            work[c] = 0;
            launches[c] = 0;
        }
        for (const ProfEntry& e : g_prof) {
            ACCO_CUDA(cudaEventSynchronize(e.b));
            float t = 0.f;
            ACCO_CUDA(cudaEventElapsedTime(&t, e.a, e.b));
            ms[e.cls] += t;
            work[e.cls] += e.work;
            launches[e.cls] += 1;
        }
    });
}

const char* acco_last_error(void) { return g_last_error.c_str(); }

int acco_version(void) { return ACCO_ABI_VERSION; }

int acco_gemm(const void* a, int64_t lda, int a_mn_major, const void* b, int64_t ldb,
              int b_mn_major, int m, int n, int k, int dtype, int epi_mode, void* c, int64_t ldc,
              const void* bias, const void* residual, int64_t ldr, void* aux, int64_t ld_aux,
              int beta, void* stream) {
    return guarded([&] {
        GemmOperand A{a, lda, a_mn_major != 0};
        GemmOperand B{b, ldb, b_mn_major != 0};
        Epilogue ep;
        ep.mode = epi_mode;
        ep.C = c;
        ep.ldc = ldc;
        ep.bias = bias;
        ep.residual = residual;
        ep.ldr = ldr;
        ep.aux = aux;
        ep.ld_aux = ld_aux;
        ep.beta = beta;
        ACCO_REQUIRE(epi_mode >= kEpiStore && epi_mode <= kEpiAccF32, "acco_gemm: bad epilogue");
        if (dtype == ACCO_DTYPE_BF16)
            gemm_bf16(A, B, m, n, k, ep, static_cast<cudaStream_t>(stream));
        else if (dtype == ACCO_DTYPE_F32)
            gemm_f32(A, B, m, n, k, ep, static_cast<cudaStream_t>(stream));
        else
            throw Error(kInvalidArg, "acco_gemm: dtype must be f32 or bf16");
    });
}

int acco_gemm_bias_grad(const void* a, int64_t lda, int a_mn_major, const void* b, int64_t ldb,
                        int b_mn_major, int m, int n, int k, float* c, int64_t ldc, float* bias_grad,
                        int beta, void* stream) {
    return guarded([&] {
        ACCO_REQUIRE(bias_grad != nullptr, "acco_gemm_bias_grad: bias_grad is null");
        GemmOperand A{a, lda, a_mn_major != 0};
        GemmOperand B{b, ldb, b_mn_major != 0};
        Epilogue ep;
        ep.mode = kEpiAccF32;
        ep.C = c;
        ep.ldc = ldc;
        ep.beta = beta;
        ep.bias_grad = bias_grad;
        gemm_bf16(A, B, m, n, k, ep, static_cast<cudaStream_t>(stream));
    });
}

}  // extern "C"
