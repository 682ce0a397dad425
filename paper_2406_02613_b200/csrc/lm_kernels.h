// Non-GEMM kernels of the LM plugin (K2 of SURVEY.md §2.3) and the small
// device utilities of the engine. Activation dtype T is float (parity mode)
// or __nv_bfloat16 (throughput mode); all arithmetic is fp32; every reduction
// is order-fixed (no float atomics) so runs are bitwise deterministic, like
// the reference's fixed-order folds (proj/src/problems.cpp:92-131).
#pragma once

#include "common.cuh"

namespace acco {

// tokens of a micro-batch: mode 0 = B indices Stream(seed).below(n_samples)
// (problems.cpp:442-444); mode 1 = contiguous samples [start, start+B).
void gather_tokens(const int32_t* data, int seq, int n_samples, uint64_t seed, int mode, int start,
                   int B, int32_t* tok_in, int32_t* tok_out, int32_t* idx_out, cudaStream_t s);

template <class T>
void embed_fwd(const int32_t* tok, const T* wte, const T* wpe, T* x, int M, int seq, int d,
               cudaStream_t s);

// rms = true: RMSNorm (Llama; b unused, mean stored as 0 so the parameter
// reduction below computes xhat = x * rstd unchanged).
template <class T>
void layernorm_fwd(const T* x, const T* g, const T* b, T* y, float* mean, float* rstd, int M, int d,
                   cudaStream_t s, bool rms = false);

// LN backward, split so the parameter reductions can run on a side stream:
// dg/db (+)= sum_rows dy * xhat, dy into fp32 gdst/bdst (uses `scratch`;
// bdst == nullptr: RMSNorm, weight only) ...
template <class T>
void layernorm_bwd_params(const T* dy, const T* x, const float* mean, const float* rstd, float* gdst,
                          float* bdst, float* scratch, int M, int d, bool accumulate_params, cudaStream_t s);
// ... and dx (+)= the input gradient.
template <class T>
void layernorm_bwd_dx(const T* dy, const T* x, const T* g, const float* mean, const float* rstd, T* dx,
                      bool accumulate_dx, int M, int d, cudaStream_t s, bool rms = false);

// bf16 norm backward with the parameter gradients fused: dx as
// layernorm_bwd_dx, plus per-block column partials part[G][2][d] (dgamma =
// sum dy * xhat, dbeta = sum dy; G = ln_part_blocks()) for ln_param_fold.
// ln_fused_supported(d): d % 256 == 0 and a width the vec / wide kernels take.
int ln_part_blocks();
bool ln_fused_supported(int d);
template <class T>
void layernorm_bwd_fused(const T* dy, const T* x, const T* g, const float* mean, const float* rstd, T* dx,
                         bool accumulate_dx, int M, int d, float* part, cudaStream_t s, bool rms = false);
// One norm's partials -> its gradient entries (offsets into the gradient
// buffer; b_off < 0: RMSNorm, weight only). part_off indexes `parts`.
struct LnFold {
    int64_t part_off;
    int64_t g_off;
    int64_t b_off;
    int d;
    int pad;
};
// every norm of a micro-batch in one launch: grad[g_off..] (+)= sum_b part[b][0],
// grad[b_off..] (+)= sum_b part[b][1]; `table` in device memory
void ln_param_fold(const LnFold* table, int n, int d_max, const float* parts, float* grad, bool accumulate,
                   cudaStream_t s);

// out[c] += sum_r y[r*ld + c] (deterministic two-level), fp32 out.
template <class T>
void colsum_add(const T* y, int64_t ld, int M, int N, float* out, float* scratch, bool accumulate,
                cudaStream_t s);

// In place: logits[M, ld] -> dlogits = (softmax - onehot(target)) / seq;
// row_loss[m] = logsumexp - logit[target].
template <class T>
void cross_entropy(T* logits, int64_t ld, const int32_t* target, int V, int M, int seq,
                   float* row_loss, cudaStream_t s);

// out[slot] = sum over rows of row_loss / seq (fixed order) = sum of sample losses.
void loss_reduce(const float* row_loss, int M, int seq, double* out, cudaStream_t s);

// Embedding backward, step 1 (token-only, so it runs early on a side
// stream): sorted[i] = keys (tok[m] << 32 | m) in ascending order (stable LSD
// radix sort on the token bits; tmp: M keys, hist: 256 x ceil(M / 1024)).
void embed_sort(const int32_t* tok, int M, int V, uint64_t* sorted, uint64_t* tmp, unsigned* hist, cudaStream_t s);
// Step 2: grad_wte[tok] += sum of dx rows of the token's segment (fixed
// chunk/run order, run_sum = [M, d] fp32 scratch), grad_wpe[t] += sum_b
// dx[b*seq + t] (skipped when grad_wpe == nullptr); zero_wte: grad_wte is
// zeroed first (untied embedding, first micro-batch).
template <class T>
void embed_bwd(const uint64_t* sorted, const T* dx, int M, int seq, int d, int V, float* grad_wte,
               float* grad_wpe, float* run_sum, bool accumulate_wpe, cudaStream_t s, bool zero_wte = false);

// Rotary embedding in place on the first nh heads (q then k) of qkv [M, ld]:
// pairs (i, i + hd/2), cs[t][i] = (cos, sin); inverse = the transpose (bwd).
template <class T>
void rope_apply(T* qkv, int64_t ld, const float2* cs, int M, int seq, int nh, int hd, bool inverse,
                cudaStream_t s);
// SwiGLU: a[M, F] = silu(gu[:, :F]) * gu[:, F:]; backward dgu[M, 2F] from da.
template <class T>
void swiglu_fwd(const T* gu, T* a, int M, int F, cudaStream_t s);
template <class T>
void swiglu_bwd(const T* da, const T* gu, T* dgu, int M, int F, cudaStream_t s);

// Causal attention over qkv [B*seq, (H + 2*Hkv)*hd] (q heads, then Hkv k
// heads, then Hkv v heads; query head h reads KV head h / (H / Hkv)), y and
// dy [B*seq, H*hd]; dqkv has qkv's layout. Hkv == H: plain MHA (GPT-2).
template <class T>
void attention_fwd(const T* qkv, T* y, float* lse, int B, int seq, int H, int Hkv, int hd, cudaStream_t s);
// tcgen05 attention kernels: take their work items from a per-stream queue
// (list scheduling) instead of the static LPT tables (set by the trainer
// when collectives run beside compute)
void attention_set_dynamic(bool on);
template <class T>
void attention_bwd(const T* qkv, const T* y, const float* lse, const T* dy, T* dqkv, float* dsum,
                   int B, int seq, int H, int Hkv, int hd, cudaStream_t s);

// ---- engine utilities
void fill_i64(int64_t* p, int64_t v, cudaStream_t s);
void add_i64(int64_t* dst, const int64_t* a, const int64_t* b, cudaStream_t s);
// out = sum_w in[w] in ascending w (the Fabric's fixed order), n floats each.
void sum_ordered(const float* const* in, int nin, float* out, int64_t n, cudaStream_t s);
void f32_to(const float* src, void* dst, int dtype, int64_t n, cudaStream_t s);
void scale_f32(float* x, double alpha, int64_t n, cudaStream_t s);
// out = sum x^2 in a fixed order (double accumulation).
void norm_sq(const float* x, int64_t n, double* out, double* scratch, cudaStream_t s);
// owner-padded layout: padded[w*chunk + j] <-> flat[lo_w + j]
void pack_padded(const float* flat, float* padded, const uint64_t* lo, const uint64_t* sz, int n,
                 uint64_t chunk, cudaStream_t s);
void unpack_padded(const void* padded, void* flat, int elem_bytes, const uint64_t* lo,
                   const uint64_t* sz, int n, uint64_t chunk, cudaStream_t s);
// Replica consistency (the reference's check_replicas, protocols.cpp:208-212,
// as a debug cross-rank checksum): out = order-independent 64-bit hash of the
// buffer (wrapping sum of mixed (word index, word) pairs: deterministic for any
// launch shape); compare sets `bit` in *flag when all[r*k + j] != all[j].
void replica_hash(const void* p, int64_t bytes, uint64_t* out, cudaStream_t s);
void hash_compare(const uint64_t* all, int n, int k, int* flag, int bit, cudaStream_t s);
// straggler throttle (HeterogeneityProfile, protocols.hpp:19-27): spin ns on the stream
void spin_ns(uint64_t ns, cudaStream_t s);
// Single-GPU stand-in for an NVLink collective: `ctas` CTAs (NCCL's channel
// count) copy `bytes` through HBM from src to dst (both >= bytes), paced so the
// copy lasts `ns` — occupying SMs and HBM bandwidth the way the real
// reduce-scatter / all-gather kernels would, for as long as they would.
void comm_standin(const void* src, void* dst, int64_t bytes, int ctas, uint64_t ns, cudaStream_t s);

}  // namespace acco
