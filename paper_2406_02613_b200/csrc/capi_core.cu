// C-ABI plumbing: error state, device info, and the raw GEMM entry point.
#include "acco.h"
#include "common.cuh"
#include "capi_util.h"
#include "gemm.h"

#include <cstring>
#include <string>

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

}  // namespace acco

using namespace acco;

extern "C" {

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

}  // extern "C"
