// GEMM entry points used by the LM plugin (K1/K3 in SURVEY.md §2.3).
//
//   C[M,N] (op)= sum_k A(m,k) * B(n,k)
//
// Operand addressing (row-major storage, `ld` in elements):
//   K-major : A(m,k) = A.ptr[m*ld + k]      (the usual X[M,K] / W[N,K] layout)
//   MN-major: A(m,k) = A.ptr[k*ld + m]      (a transposed view, e.g. dY^T in wgrad)
//
// The bf16 path is the tcgen05/TMA/TMEM kernel (gemm_tcgen05.cu); the fp32
// path (the fp32-accurate parity mode, SURVEY.md §7 "fp64 oracle vs
// fp32/bf16 GPU") is the same kernel on kind::tf32 with the 3xTF32 split.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace acco {

struct GemmOperand {
    const void* ptr = nullptr;
    int64_t ld = 0;
    bool mn_major = false;
};

enum EpiMode : int {
    kEpiStore = 0,   // C = acc + bias + residual            (activation dtype)
    kEpiGelu = 1,    // x = acc + bias; C = gelu(x); aux = gelu'(x)  (activation dtype)
    kEpiDGelu = 2,   // C = acc * aux (aux = the slope kEpiGelu stored)
    kEpiAccF32 = 3,  // C_f32 = beta*C_f32 + acc              (fp32 gradient accumulator)
    // SwiGLU (Llama MLP): N = 2F output features stored [gate (F) | up (F)];
    // the tile's B rows come half from each half, so the epilogue sees gate and
    // up of the same features: aux[M, 2F] = pre-activations, C[M, F] =
    // silu(gate) * up (bf16 tcgen05 path, K-major B, F % 128 == 0)
    kEpiSwiGLU = 4,
    // SwiGLU backward (dgrad of the down projection, N = F): acc = dA;
    // aux = GU [M, 2F] pre-activations; C = dGU [M, 2F] (gate | up halves)
    kEpiDSwiGLU = 5,
};

struct Epilogue {
    int mode = kEpiStore;
    void* C = nullptr;
    int64_t ldc = 0;
    const void* bias = nullptr;      // [N], activation dtype
    const void* residual = nullptr;  // [M, ldr], activation dtype (may alias C)
    int64_t ldr = 0;
    void* aux = nullptr;             // [M, ld_aux] pre-activation (gelu modes)
    int64_t ld_aux = 0;
    int beta = 0;                    // kEpiAccF32: accumulate into C when 1
    // kEpiAccF32 (weight gradients dW = dY^T X, A = dY^T): also the bias
    // gradient db[m] (+)= sum_k A(m, k) = the column sums of dY, fp32 [M],
    // accumulated like C (beta). Computed on the tensor core by the tiles of
    // the first n-block: one extra 16-wide MMA per k-slice against a ones tile.
    float* bias_grad = nullptr;
};

void gemm_bf16(const GemmOperand& A, const GemmOperand& B, int M, int N, int K,
               const Epilogue& ep, cudaStream_t stream);
// Whether a bf16 fp32-accumulate GEMM of this shape should take
// Epilogue::bias_grad: the bias MMA needs a tile width <= 192 (TMEM), so it is
// fused when the best such plan is modelled within 4 % of the best plan
// overall (else the caller reduces the columns separately).
bool gemm_bias_grad_free(const GemmOperand& A, const GemmOperand& B, int M, int N, int K);
// CTA-pair tiles: take units from a work queue instead of the static
// persistent order (set by the trainer when collectives run beside compute).
void gemm_set_pair_queue(bool on);
// fp32 operands: the 3xTF32 tcgen05 kernel (gemm_tcgen05.cu) ...
void gemm_f32_tc(const GemmOperand& A, const GemmOperand& B, int M, int N, int K,
                 const Epilogue& ep, cudaStream_t stream);
// ... or the SIMT kernel (gemm_simt.cu; ACCO_GEMM_SIMT=1 A/B knob). gemm_f32
// dispatches between them.
void gemm_f32_simt(const GemmOperand& A, const GemmOperand& B, int M, int N, int K,
                   const Epilogue& ep, cudaStream_t stream);
void gemm_f32(const GemmOperand& A, const GemmOperand& B, int M, int N, int K,
              const Epilogue& ep, cudaStream_t stream);

}  // namespace acco
