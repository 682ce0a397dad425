// GPT-style LM plugin: the B200 implementation of the reference's gradient
// oracle contract `stochastic_grad(Problem, theta, MicroBatch)`
// (/root/reference/proj/include/accosim/problems.hpp:86-92,
// proj/src/problems.cpp:419-451) for the LM defined in oracle/gpt_oracle.py.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "common.cuh"
#include "lm_kernels.h"

namespace acco {

struct LMConfig {
    int vocab = 256;
    int d_model = 128;
    int n_layer = 2;
    int n_head = 4;
    int seq_len = 64;
    int n_samples = 256;
    uint64_t data_seed = 1;
    int precision = 0;  // 0 = fp32 (parity), 1 = bf16 (tcgen05 throughput)
    int max_batch = 8;  // samples per micro-batch (workspace sizing)
    int host_data = 0;  // 1: per-micro-batch H2D of the token rows from pinned host memory
    int arch = 0;       // 0 GPT-2 block, 1 Llama block (RMSNorm, RoPE, GQA, SwiGLU, untied head)
    int n_kv_head = 0;  // llama: 0 -> n_head
    int d_ff = 0;       // llama: 0 -> 4 * d_model
    double rope_base = 0.0;  // llama: 0 -> 10000
    int kv_heads() const { return n_kv_head > 0 ? n_kv_head : n_head; }
    int ffn() const { return d_ff > 0 ? d_ff : 4 * d_model; }
    double rope() const { return rope_base > 0.0 ? rope_base : 10000.0; }
};

struct ParamSpec {
    std::string name;
    int64_t rows, cols;  // cols == 1 for vectors
    int kind;            // 0 w(.02) 1 wp(.02/sqrt(2L)) 2 one 3 zero
    int64_t off;
    int64_t numel() const { return rows * cols; }
};

std::vector<ParamSpec> lm_param_layout(const LMConfig& c);
// Markov dataset [n_samples, seq_len+1] (int32), host.
std::vector<int32_t> lm_dataset(const LMConfig& c);
// theta0 (fp64 on host -> float), the oracle's default_theta0.
void lm_default_theta0(const LMConfig& c, uint64_t master_seed, float* out);

class GPTModel {
public:
    explicit GPTModel(const LMConfig& c);
    ~GPTModel();
    GPTModel(const GPTModel&) = delete;
    GPTModel& operator=(const GPTModel&) = delete;

    const LMConfig& cfg() const { return c_; }
    int64_t num_params() const { return psi_; }
    int act_dtype() const { return c_.precision; }  // ACCO_DTYPE_*
    size_t act_bytes() const { return c_.precision ? 2 : 4; }
    const std::vector<ParamSpec>& layout() const { return layout_; }

    // One micro-batch fwd+bwd at `params` (activation dtype, flat layout):
    // grad_acc[psi] (fp32) += sum over the B samples of their gradients
    // (= Bundle::add of N * per-sample-mean, protocols.cpp:61-66), and
    // *loss_sum (device double) = sum over samples of the per-sample loss.
    // mode 0: indices Stream(stream_seed).below(n_samples); mode 1: [start, start+B).
    // accumulate=false: the gradient of this micro-batch *overwrites* grad_acc
    // (first micro-batch of a stage; no memset needed).
    void micro_batch(const void* params, uint64_t stream_seed, int mode, int start, int B, float* grad_acc,
                     double* loss_sum, cudaStream_t s, bool accumulate = true);
    // Token indices drawn by the last micro_batch (device int32 [B]).
    const int32_t* last_indices() const { return idx_; }
    // Forward only (loss), used by evaluation when no gradient is needed.
    void forward_loss(const void* params, uint64_t stream_seed, int mode, int start, int B, double* loss_sum,
                      cudaStream_t s);
    bool host_data() const { return c_.host_data != 0; }
    long long h2d_bytes() const { return h2d_bytes_; }

private:
    template <class T>
    void run(const T* P, uint64_t seed, int mode, int start, int B, float* G, double* loss, bool backward,
             cudaStream_t s);
    template <class T>
    void run_llama(const T* P, uint64_t seed, int mode, int start, int B, float* G, double* loss, bool backward,
                   cudaStream_t s);
    void stage_input(uint64_t seed, int mode, int start, int B, cudaStream_t s);
    void sort_tokens(int M, cudaStream_t s);

    LMConfig c_;
    std::vector<ParamSpec> layout_;
    int64_t psi_ = 0;
    int vpad_ = 0;
    // device buffers
    int32_t* data_ = nullptr;
    int32_t *tok_in_ = nullptr, *tok_out_ = nullptr, *idx_ = nullptr;
    uint64_t* sort_ = nullptr;      // sorted (token, position) keys of the embedding backward
    uint64_t* sort_tmp_ = nullptr;
    unsigned* sort_hist_ = nullptr;
    float* run_sum_ = nullptr;  // embedding-gradient run sums [M, d]
    void* arena_ = nullptr;
    size_t arena_bytes_ = 0;
    float* row_loss_ = nullptr;
    float* stats_ = nullptr;    // per-layer LN mean/rstd
    float* lse_ = nullptr;      // per-layer attention lse
    float* dsum_ = nullptr;
    float* scratch_ = nullptr;  // column-reduce partials
    // bf16: the norms' parameter gradients as per-block partials of the fused
    // norm backward (ln_part_ [n_ln][G][2][d]), folded once per micro-batch
    // through ln_fold_ (device table, entry = norm index, see ln_index)
    bool fuse_ln_ = false;
    float* ln_part_ = nullptr;
    LnFold* ln_fold_ = nullptr;
    int n_ln_ = 0;
    float* ln_part(int i) const { return ln_part_ + static_cast<int64_t>(i) * ln_part_blocks() * 2 * c_.d_model; }
    float2* rope_ = nullptr;    // llama: (cos, sin) [seq][hd/2]
    // side stream for the bias / LN-parameter column reductions: they only feed
    // the gradient accumulator, so they run beside the GEMMs (fork/join events)
    cudaStream_t aux_ = nullptr;
    cudaEvent_t ev_fork_ = nullptr, ev_join_ = nullptr, ev_sort_ = nullptr;
    // last side-stream reader of each backward scratch buffer (DX, DA, DT, DQKV):
    // the compute stream waits on it only right before overwriting that buffer
    cudaEvent_t ev_rd_[4] = {nullptr, nullptr, nullptr, nullptr};
    std::vector<char*> act_;    // activation slots (see model.cu)
    // host-data path
    int32_t* pinned_data_ = nullptr;
    int32_t* stage_host_ = nullptr;  // [kStages][max_batch*(seq+1)] pinned
    int32_t* stage_dev_ = nullptr;
    std::vector<cudaEvent_t> stage_ev_;
    int stage_next_ = 0;
    long long h2d_bytes_ = 0;
    bool accumulate_ = true;
    const int32_t* stage_tokens(uint64_t seed, int B, cudaStream_t s);
};

// Device time of one micro-batch of `batch` samples (fwd + bwd + accumulate),
// mean of `reps`, ns (the HeterogeneityProfile throttle base, protocols.hpp:19-27).
double time_micro_batch(GPTModel& g, int batch, int reps);

}  // namespace acco
