// GPT-style LM plugin (see model.h). Forward + backward of one micro-batch,
// accumulating the summed per-sample gradients straight into the fp32
// gradient-accumulation buffer through the wgrad GEMM epilogues (K3: the
// reference's Bundle::add, proj/src/protocols.cpp:61-66, has no separate pass).
#include "gemm.h"
#include "host_util.h"
#include "lm_kernels.h"
#include "model.h"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

namespace acco {

// ------------------------------------------------------------ host definitions
std::vector<ParamSpec> lm_param_layout(const LMConfig& c) {
    const int64_t d = c.d_model;
    std::vector<ParamSpec> v;
    auto add = [&](const std::string& n, int64_t r, int64_t cc, int kind) {
        int64_t off = v.empty() ? 0 : v.back().off + v.back().numel();
        v.push_back({n, r, cc, kind, off});
    };
    add("wte", c.vocab, d, 0);
    if (c.arch == 1) {  // oracle/gpt_oracle.py param_layout, arch="llama"
        const int64_t hd = d / c.n_head, nqkv = (c.n_head + 2 * c.kv_heads()) * hd, F = c.ffn();
        for (int l = 0; l < c.n_layer; ++l) {
            const std::string p = "layers." + std::to_string(l) + ".";
            add(p + "attention_norm.weight", d, 1, 2);
            add(p + "attention.wqkv", nqkv, d, 0);
            add(p + "attention.wo", d, c.n_head * hd, 1);
            add(p + "ffn_norm.weight", d, 1, 2);
            add(p + "feed_forward.w_gate_up", 2 * F, d, 0);
            add(p + "feed_forward.w_down", d, F, 1);
        }
        add("norm.weight", d, 1, 2);
        add("output.weight", c.vocab, d, 0);
        return v;
    }
    add("wpe", c.seq_len, d, 0);
    for (int l = 0; l < c.n_layer; ++l) {
        const std::string p = "h." + std::to_string(l) + ".";
        add(p + "ln_1.weight", d, 1, 2);
        add(p + "ln_1.bias", d, 1, 3);
        add(p + "attn.c_attn.weight", 3 * d, d, 0);
        add(p + "attn.c_attn.bias", 3 * d, 1, 3);
        add(p + "attn.c_proj.weight", d, d, 1);
        add(p + "attn.c_proj.bias", d, 1, 3);
        add(p + "ln_2.weight", d, 1, 2);
        add(p + "ln_2.bias", d, 1, 3);
        add(p + "mlp.c_fc.weight", 4 * d, d, 0);
        add(p + "mlp.c_fc.bias", 4 * d, 1, 3);
        add(p + "mlp.c_proj.weight", d, 4 * d, 1);
        add(p + "mlp.c_proj.bias", d, 1, 3);
    }
    add("ln_f.weight", d, 1, 2);
    add("ln_f.bias", d, 1, 3);
    return v;
}

std::vector<int32_t> lm_dataset(const LMConfig& c) {
    // oracle/gpt_oracle.py dataset(): integer-only Markov chain
    const uint64_t V = static_cast<uint64_t>(c.vocab);
    std::vector<int32_t> succ(static_cast<size_t>(V));
    Stream ss(rng_derive(c.data_seed, 0x5eed, V));
    for (uint64_t v = 0; v < V; ++v) succ[v] = static_cast<int32_t>(ss.below(V));
    const int T1 = c.seq_len + 1;
    std::vector<int32_t> tok(static_cast<size_t>(c.n_samples) * T1);
    for (int s = 0; s < c.n_samples; ++s) {
        Stream st(rng_derive(c.data_seed, 0xda7a, static_cast<uint64_t>(s)));
        uint64_t x = st.below(V);
        int32_t* row = tok.data() + static_cast<size_t>(s) * T1;
        row[0] = static_cast<int32_t>(x);
        for (int t = 1; t < T1; ++t) {
            uint64_t r = st.next_u64();
            x = (r & 3) ? static_cast<uint64_t>(succ[x]) : (r >> 2) % V;
            row[t] = static_cast<int32_t>(x);
        }
    }
    return tok;
}

void lm_default_theta0(const LMConfig& c, uint64_t master_seed, float* out) {
    // oracle/gpt_oracle.py default_theta0(): exact arithmetic in fp64
    const double kSqrt3 = 1.7320508075688772;
    Stream st(rng_derive(master_seed, 0x7e7a0));
    for (const ParamSpec& p : lm_param_layout(c)) {
        float* o = out + p.off;
        const int64_t n = p.numel();
        if (p.kind == 2) {
            for (int64_t i = 0; i < n; ++i) o[i] = 1.0f;
        } else if (p.kind == 3) {
            for (int64_t i = 0; i < n; ++i) o[i] = 0.0f;
        } else {
            const double stdv = p.kind == 0 ? 0.02 : 0.02 / std::sqrt(2.0 * c.n_layer);
            const double a = stdv * kSqrt3;
            for (int64_t i = 0; i < n; ++i) o[i] = static_cast<float>(a * (2.0 * st.uniform01() - 1.0));
        }
    }
}

// ------------------------------------------------------------------- model
namespace {
enum Slot { sX, sH1, sQKV, sY, sXM, sH2, sA, sU, kPerLayer };
constexpr int kStages = 4;  // host-data staging slots in flight
}

GPTModel::GPTModel(const LMConfig& c) : c_(c) {
    ACCO_REQUIRE(c.vocab >= 2 && c.d_model >= 8 && c.n_layer >= 1 && c.n_head >= 1 && c.seq_len >= 1,
                 "lm config: positive sizes required");
    ACCO_REQUIRE(c.d_model % c.n_head == 0, "lm config: d_model must be divisible by n_head");
    ACCO_REQUIRE(c.d_model % 8 == 0, "lm config: d_model must be a multiple of 8 (TMA alignment)");
    ACCO_REQUIRE(c.n_samples >= 1 && c.max_batch >= 1, "lm config: n_samples, max_batch >= 1");
    ACCO_REQUIRE(c.precision == 0 || c.precision == 1, "lm config: precision must be fp32 or bf16");
    ACCO_REQUIRE(c.arch == 0 || c.arch == 1, "lm config: arch must be 0 (gpt2) or 1 (llama)");
    if (c.arch == 1) {
        ACCO_REQUIRE(c.kv_heads() >= 1 && c.n_head % c.kv_heads() == 0,
                     "lm config: n_head must be a multiple of n_kv_head");
        ACCO_REQUIRE((c.d_model / c.n_head) % 2 == 0, "lm config: rotary embeddings need an even head size");
        ACCO_REQUIRE(c.ffn() % 8 == 0, "lm config: d_ff must be a multiple of 8 (TMA alignment)");
    } else {
        ACCO_REQUIRE(c.n_kv_head == 0 || c.n_kv_head == c.n_head, "lm config: gpt2 has no grouped-query attention");
    }
    layout_ = lm_param_layout(c);
    psi_ = layout_.back().off + layout_.back().numel();
    vpad_ = (c.vocab + 63) / 64 * 64;
    const int64_t M = static_cast<int64_t>(c.max_batch) * c.seq_len;
    const int64_t d = c.d_model, L = c.n_layer, H = c.n_head;
    const size_t e = act_bytes();
    const bool llama = c.arch == 1;
    const int64_t nqkv = llama ? (H + 2 * c.kv_heads()) * (d / H) : 3 * d;
    const int64_t F = c.ffn();
    auto sz = [&](int slot) -> int64_t {
        switch (slot) {
            case sQKV: return nqkv;
            case sA: return llama ? 2 * F : 4 * d;  // llama: gate|up pre-activation; gpt2: gelu slope
            case sU: return llama ? F : 4 * d;      // MLP activation (gelu / swiglu output)
            default: return d;
        }
    };
    // arena: L layers x kPerLayer slots, then x[L], hf, logits, dx, dt, dqkv, da
    std::vector<int64_t> cols;
    for (int l = 0; l < L; ++l)
        for (int s = 0; s < kPerLayer; ++s) cols.push_back(sz(s));
    cols.push_back(d);          // x[L]
    cols.push_back(d);          // hf
    cols.push_back(vpad_);      // logits
    cols.push_back(d);          // dx
    cols.push_back(d);          // dt
    cols.push_back(nqkv);       // dqkv
    cols.push_back(llama ? 2 * F : 4 * d);  // da (llama: d(gate|up))
    cols.push_back(llama ? F : 0);          // llama: d(swiglu output)
    size_t total = 0;
    std::vector<size_t> offs;
    for (int64_t cc : cols) {
        offs.push_back(total);
        total += (static_cast<size_t>(M * cc) * e + 255) / 256 * 256;
    }
    arena_bytes_ = total;
    ACCO_CUDA(cudaMalloc(&arena_, arena_bytes_));
    for (size_t o : offs) act_.push_back(static_cast<char*>(arena_) + o);

    std::vector<int32_t> data = lm_dataset(c);
    ACCO_CUDA(cudaMalloc(&data_, data.size() * sizeof(int32_t)));
    ACCO_CUDA(cudaMemcpy(data_, data.data(), data.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    if (c.host_data) {
        const size_t row = static_cast<size_t>(c.seq_len) + 1;
        ACCO_CUDA(cudaHostAlloc(&pinned_data_, data.size() * sizeof(int32_t), cudaHostAllocDefault));
        std::memcpy(pinned_data_, data.data(), data.size() * sizeof(int32_t));
        ACCO_CUDA(cudaHostAlloc(&stage_host_, kStages * c.max_batch * row * sizeof(int32_t), cudaHostAllocDefault));
        ACCO_CUDA(cudaMalloc(&stage_dev_, kStages * c.max_batch * row * sizeof(int32_t)));
        stage_ev_.resize(kStages);
        for (auto& e : stage_ev_) ACCO_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    ACCO_CUDA(cudaMalloc(&tok_in_, M * sizeof(int32_t)));
    ACCO_CUDA(cudaMalloc(&tok_out_, M * sizeof(int32_t)));
    ACCO_CUDA(cudaMalloc(&idx_, c.max_batch * sizeof(int32_t)));
    ACCO_CUDA(cudaMalloc(&sort_, M * sizeof(uint64_t)));
    ACCO_CUDA(cudaMalloc(&sort_tmp_, M * sizeof(uint64_t)));
    ACCO_CUDA(cudaMalloc(&sort_hist_, 256 * ((M + 1023) / 1024) * sizeof(unsigned)));
    ACCO_CUDA(cudaMalloc(&run_sum_, static_cast<size_t>(M) * d * sizeof(float)));
    ACCO_CUDA(cudaMalloc(&row_loss_, M * sizeof(float)));
    ACCO_CUDA(cudaMalloc(&stats_, (4 * L + 2) * M * sizeof(float)));
    ACCO_CUDA(cudaMalloc(&lse_, L * H * M * sizeof(float)));
    ACCO_CUDA(cudaMalloc(&dsum_, H * M * sizeof(float)));
    // column-reduction partials: [chunks][2][N] with N <= 4d; chunks <= max(M/256,
    // 8 x SMs) (see colsum_vec / colreduce in lm_kernels.cu)
    const int64_t nchunk = std::max<int64_t>((M + 255) / 256, 8 * num_sms());
    ACCO_CUDA(cudaMalloc(&scratch_, nchunk * 4 * d * 2 * sizeof(float)));
    // fused norm-parameter gradients (bf16): norm i = 0 the final norm, 1 + 2l
    // the first norm of layer l, 2 + 2l its second; LnFold entries in that order
    fuse_ln_ = c.precision == 1 && ln_fused_supported(d);  // (precision 1: bf16, see micro_batch)
    if (fuse_ln_) {
        n_ln_ = 2 * L + 1;
        ACCO_CUDA(cudaMalloc(&ln_part_, static_cast<size_t>(n_ln_) * ln_part_blocks() * 2 * d * sizeof(float)));
        std::vector<LnFold> tab(static_cast<size_t>(n_ln_));
        auto off = [&](int i) { return static_cast<int64_t>(layout_[static_cast<size_t>(i)].off); };
        for (int i = 0; i < n_ln_; ++i) {
            LnFold& e = tab[static_cast<size_t>(i)];
            e.part_off = static_cast<int64_t>(i) * ln_part_blocks() * 2 * d;
            e.d = d;
            e.pad = 0;
            // parameter indices (layout_ order, see run / run_llama)
            int gi, bi;
            if (llama) {
                const int l = (i - 1) / 2;
                gi = i == 0 ? 1 + 6 * L : 1 + 6 * l + (i % 2 == 1 ? 0 : 3);
                bi = -1;
            } else {
                const int l = (i - 1) / 2;
                gi = i == 0 ? 2 + 12 * L : 2 + 12 * l + (i % 2 == 1 ? 0 : 6);
                bi = gi + 1;
            }
            e.g_off = off(gi);
            e.b_off = bi >= 0 ? off(bi) : -1;
        }
        ACCO_CUDA(cudaMalloc(&ln_fold_, tab.size() * sizeof(LnFold)));
        ACCO_CUDA(cudaMemcpy(ln_fold_, tab.data(), tab.size() * sizeof(LnFold), cudaMemcpyHostToDevice));
    }
    if (llama) {  // rotary table, fp64 angles rounded to fp32 (oracle rope_table)
        const int hd = c.d_model / c.n_head, h2 = hd / 2;
        std::vector<float2> tab(static_cast<size_t>(c.seq_len) * h2);
        for (int t = 0; t < c.seq_len; ++t)
            for (int i = 0; i < h2; ++i) {
                const double inv = std::pow(c.rope(), -2.0 * i / hd);
                const double a = static_cast<double>(t) * inv;
                tab[static_cast<size_t>(t) * h2 + i] = make_float2(static_cast<float>(std::cos(a)),
                                                                   static_cast<float>(std::sin(a)));
            }
        ACCO_CUDA(cudaMalloc(&rope_, tab.size() * sizeof(float2)));
        ACCO_CUDA(cudaMemcpy(rope_, tab.data(), tab.size() * sizeof(float2), cudaMemcpyHostToDevice));
    }
    ACCO_CUDA(cudaStreamCreateWithFlags(&aux_, cudaStreamNonBlocking));
    ACCO_CUDA(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
    ACCO_CUDA(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming));
    ACCO_CUDA(cudaEventCreateWithFlags(&ev_sort_, cudaEventDisableTiming));
    for (auto& e : ev_rd_) ACCO_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
}

GPTModel::~GPTModel() {
    cudaFree(arena_);
    cudaFree(data_);
    cudaFree(tok_in_);
    cudaFree(tok_out_);
    cudaFree(idx_);
    cudaFree(sort_);
    cudaFree(sort_tmp_);
    cudaFree(sort_hist_);
    cudaFree(run_sum_);
    cudaFree(row_loss_);
    cudaFree(stats_);
    cudaFree(lse_);
    cudaFree(dsum_);
    if (aux_) {
        cudaStreamSynchronize(aux_);
        cudaStreamDestroy(aux_);
        cudaEventDestroy(ev_fork_);
        cudaEventDestroy(ev_join_);
        cudaEventDestroy(ev_sort_);
        for (auto& e : ev_rd_) cudaEventDestroy(e);
    }
    cudaFree(scratch_);
    if (ln_part_) cudaFree(ln_part_);
    if (ln_fold_) cudaFree(ln_fold_);
    if (rope_) cudaFree(rope_);
    if (pinned_data_) cudaFreeHost(pinned_data_);
    if (stage_host_) cudaFreeHost(stage_host_);
    if (stage_dev_) cudaFree(stage_dev_);
    for (auto& e : stage_ev_) cudaEventDestroy(e);
}

// Host data-loader path: draw the B sample indices on the host
// (Stream(seed).below(n), problems.cpp:442-444), copy those token rows into a
// pinned staging slot and ship them H2D on the compute stream.
const int32_t* GPTModel::stage_tokens(uint64_t seed, int B, cudaStream_t s) {
    const size_t row = static_cast<size_t>(c_.seq_len) + 1;
    const int slot = stage_next_;
    stage_next_ = (stage_next_ + 1) % kStages;
    ACCO_CUDA(cudaEventSynchronize(stage_ev_[static_cast<size_t>(slot)]));  // slot's previous H2D done
    int32_t* h = stage_host_ + static_cast<size_t>(slot) * c_.max_batch * row;
    int32_t* d = stage_dev_ + static_cast<size_t>(slot) * c_.max_batch * row;
    Stream st(seed);
    for (int b = 0; b < B; ++b) {
        const uint64_t idx = st.below(static_cast<uint64_t>(c_.n_samples));
        std::memcpy(h + b * row, pinned_data_ + idx * row, row * sizeof(int32_t));
    }
    ACCO_CUDA(cudaMemcpyAsync(d, h, B * row * sizeof(int32_t), cudaMemcpyHostToDevice, s));
    ACCO_CUDA(cudaEventRecord(stage_ev_[static_cast<size_t>(slot)], s));
    h2d_bytes_ += static_cast<long long>(B * row * sizeof(int32_t));
    return d;
}

namespace {

template <class T>
void mm(const T* a, int64_t lda, bool amn, const T* b, int64_t ldb, bool bmn, int m, int n, int k,
        const Epilogue& ep, cudaStream_t s) {
    GemmOperand A{a, lda, amn}, B{b, ldb, bmn};
    if constexpr (sizeof(T) == 2)
        gemm_bf16(A, B, m, n, k, ep, s);
    else
        gemm_f32(A, B, m, n, k, ep, s);
}

Epilogue ep_store(void* c, int64_t ldc, const void* bias = nullptr, const void* res = nullptr, int64_t ldr = 0) {
    Epilogue e;
    e.mode = kEpiStore;
    e.C = c;
    e.ldc = ldc;
    e.bias = bias;
    e.residual = res;
    e.ldr = ldr;
    return e;
}
Epilogue ep_gelu(void* c, int64_t ldc, const void* bias, void* aux) {
    Epilogue e = ep_store(c, ldc, bias);
    e.mode = kEpiGelu;
    e.aux = aux;
    e.ld_aux = ldc;
    return e;
}
Epilogue ep_dgelu(void* c, int64_t ldc, void* aux) {
    Epilogue e = ep_store(c, ldc);
    e.mode = kEpiDGelu;
    e.aux = aux;
    e.ld_aux = ldc;
    return e;
}
Epilogue ep_acc(float* c, int64_t ldc, int beta) {
    Epilogue e;
    e.mode = kEpiAccF32;
    e.C = c;
    e.ldc = ldc;
    e.beta = beta;
    return e;
}

}  // namespace

// The embedding-gradient sort needs only the tokens: it runs on the side
// stream under the forward pass; embed_bwd waits on ev_sort_.
void GPTModel::sort_tokens(int M, cudaStream_t s) {
    static const bool serial = std::getenv("ACCO_SERIAL_REDUCE") != nullptr;
    if (serial) {
        embed_sort(tok_in_, M, c_.vocab, sort_, sort_tmp_, sort_hist_, s);
        ACCO_CUDA(cudaEventRecord(ev_sort_, s));
        return;
    }
    ACCO_CUDA(cudaEventRecord(ev_fork_, s));
    ACCO_CUDA(cudaStreamWaitEvent(aux_, ev_fork_, 0));
    embed_sort(tok_in_, M, c_.vocab, sort_, sort_tmp_, sort_hist_, aux_);
    ACCO_CUDA(cudaEventRecord(ev_sort_, aux_));
}

void GPTModel::stage_input(uint64_t seed, int mode, int start, int B, cudaStream_t s) {
    const int Tq = c_.seq_len;
    if (host_data() && mode == 0)
        gather_tokens(stage_tokens(seed, B, s), Tq, B, 0, 1, 0, B, tok_in_, tok_out_, idx_, s);
    else
        gather_tokens(data_, Tq, c_.n_samples, seed, mode, start, B, tok_in_, tok_out_, idx_, s);
}

template <class T>
void GPTModel::run(const T* P, uint64_t seed, int mode, int start, int B, float* G, double* loss, bool backward,
                   cudaStream_t s) {
    if (c_.arch == 1) return run_llama<T>(P, seed, mode, start, B, G, loss, backward, s);
    const int Tq = c_.seq_len, d = c_.d_model, H = c_.n_head, hd = d / H, V = c_.vocab, L = c_.n_layer;
    ACCO_REQUIRE(B >= 1 && B <= c_.max_batch, "micro_batch: batch size exceeds the model workspace");
    if (mode == 1) ACCO_REQUIRE(start >= 0 && start + B <= c_.n_samples, "micro_batch: sample range out of bounds");
    const int M = B * Tq;
    const int64_t Mmax = static_cast<int64_t>(c_.max_batch) * Tq;
    auto slot = [&](int l, int sl) { return reinterpret_cast<T*>(act_[static_cast<size_t>(l * kPerLayer + sl)]); };
    const int tail = L * kPerLayer;
    T* XL = reinterpret_cast<T*>(act_[tail + 0]);
    T* HF = reinterpret_cast<T*>(act_[tail + 1]);
    T* LOG = reinterpret_cast<T*>(act_[tail + 2]);
    T* DX = reinterpret_cast<T*>(act_[tail + 3]);
    T* DT = reinterpret_cast<T*>(act_[tail + 4]);
    T* DQKV = reinterpret_cast<T*>(act_[tail + 5]);
    T* DA = reinterpret_cast<T*>(act_[tail + 6]);
    auto X = [&](int l) { return l == L ? XL : slot(l, sX); };
    auto stat = [&](int i) { return stats_ + static_cast<int64_t>(i) * Mmax; };
    // parameter pointers: index into layout_ (oracle order)
    auto W = [&](int i) { return P + layout_[static_cast<size_t>(i)].off; };
    auto Gp = [&](int i) { return G + layout_[static_cast<size_t>(i)].off; };
    const int kWte = 0, kWpe = 1, kLnf = 2 + 12 * L;
    auto li = [&](int l, int j) { return 2 + 12 * l + j; };  // j: 0 ln1w 1 ln1b 2 Wqkv 3 bqkv 4 Wproj 5 bproj
                                                            //    6 ln2w 7 ln2b 8 Wfc 9 bfc 10 Wfc2 11 bfc2

    stage_input(seed, mode, start, B, s);
    if (backward) sort_tokens(M, s);
    embed_fwd<T>(tok_in_, W(kWte), W(kWpe), X(0), M, Tq, d, s);
    for (int l = 0; l < L; ++l) {
        T *H1 = slot(l, sH1), *QKV = slot(l, sQKV), *Y = slot(l, sY), *XM = slot(l, sXM), *H2 = slot(l, sH2),
          *A = slot(l, sA), *U = slot(l, sU);
        layernorm_fwd<T>(X(l), W(li(l, 0)), W(li(l, 1)), H1, stat(4 * l), stat(4 * l + 1), M, d, s);
        mm<T>(H1, d, false, W(li(l, 2)), d, false, M, 3 * d, d, ep_store(QKV, 3 * d, W(li(l, 3))), s);
        attention_fwd<T>(QKV, Y, lse_ + static_cast<int64_t>(l) * H * Mmax, B, Tq, H, H, hd, s);
        mm<T>(Y, d, false, W(li(l, 4)), d, false, M, d, d, ep_store(XM, d, W(li(l, 5)), X(l), d), s);
        layernorm_fwd<T>(XM, W(li(l, 6)), W(li(l, 7)), H2, stat(4 * l + 2), stat(4 * l + 3), M, d, s);
        mm<T>(H2, d, false, W(li(l, 8)), d, false, M, 4 * d, d, ep_gelu(U, 4 * d, W(li(l, 9)), A), s);
        mm<T>(U, 4 * d, false, W(li(l, 10)), 4 * d, false, M, d, 4 * d, ep_store(X(l + 1), d, W(li(l, 11)), XM, d), s);
    }
    layernorm_fwd<T>(X(L), W(kLnf), W(kLnf + 1), HF, stat(4 * L), stat(4 * L + 1), M, d, s);
    mm<T>(HF, d, false, W(kWte), d, false, M, V, d, ep_store(LOG, vpad_), s);
    cross_entropy<T>(LOG, vpad_, tok_out_, V, M, Tq, row_loss_, s);
    loss_reduce(row_loss_, M, Tq, loss, s);
    if (!backward) return;

    // Every gradient element is written by exactly one kernel first in this
    // order, so with acc == false the first write *stores* and the caller's
    // per-stage memset of the accumulator is unnecessary.
    const bool acc = accumulate_;
    const int beta = acc ? 1 : 0;
    // The column reductions (bias and LN-parameter gradients) depend on
    // nothing the input-gradient chain produces next, so they run on the side
    // stream aux_, concurrently with the chain on s: each is forked right
    // after its input exists, and s waits for a buffer's last side-stream
    // reader (ev_rd_) only right before it overwrites that buffer. Same
    // kernels and summation orders as inline, so results are bitwise unchanged.
    // ACCO_WGRAD_SIDE=1 also moves the weight-gradient GEMMs there (measured:
    // neutral, 810-813k vs 815-828k tok/s inline, profiles/r02_summary.md);
    // ACCO_SERIAL_REDUCE=1: everything inline on s (A/B).
    static const bool serial = std::getenv("ACCO_SERIAL_REDUCE") != nullptr;
    const bool wg_side = !serial && std::getenv("ACCO_WGRAD_SIDE") != nullptr;
    cudaStream_t aux_ = serial ? s : this->aux_;
    cudaStream_t ws = wg_side ? aux_ : s;  // weight-gradient stream
    enum { kRdDX, kRdDA, kRdDT, kRdDQKV };
    // bf16: every bias gradient (the column sums of the dY that is the A
    // operand of its weight-gradient GEMM) comes off the tensor core in that
    // GEMM (Epilogue::bias_grad) instead of a separate column reduction that
    // re-reads dY; ACCO_BIAS_COLSUM=1: the separate reductions (A/B)
    // (per weight gradient: only where its best tile plan leaves TMEM for the
    // bias columns, gemm_bias_grad_free; GPT-2 small: all four)
    const bool colsum_env = std::getenv("ACCO_BIAS_COLSUM") != nullptr;
    auto bias_free = [&](int m, int n) {
        return sizeof(T) == 2 && !colsum_env && gemm_bias_grad_free({nullptr, 0, true}, {nullptr, 0, true}, m, n, M);
    };
    const bool fb_fc2 = bias_free(d, 4 * d), fb_fc = bias_free(4 * d, d), fb_proj = bias_free(d, d),
               fb_qkv = bias_free(3 * d, d);
    auto ep_wg = [&](float* c, int64_t ldc, float* bias_grad, bool fuse) {
        Epilogue e = ep_acc(c, ldc, beta);
        if (fuse) e.bias_grad = bias_grad;
        return e;
    };
    auto fork = [&] {
        if (serial) return;
        ACCO_CUDA(cudaEventRecord(ev_fork_, s));
        ACCO_CUDA(cudaStreamWaitEvent(aux_, ev_fork_, 0));
    };
    auto mark = [&](int b) {  // the side-stream work issued so far is buffer b's last reader
        if (!serial) ACCO_CUDA(cudaEventRecord(ev_rd_[b], aux_));
    };
    auto guard = [&](int b) {  // s is about to overwrite buffer b
        if (!serial) ACCO_CUDA(cudaStreamWaitEvent(s, ev_rd_[b], 0));
    };
    auto join = [&] {
        if (serial) return;
        ACCO_CUDA(cudaEventRecord(ev_join_, aux_));
        ACCO_CUDA(cudaStreamWaitEvent(s, ev_join_, 0));
    };
    // LM head (tied to wte): dwte (+)= dlogits^T hf ; dhf = dlogits wte
    if (wg_side) fork();
    mm<T>(LOG, vpad_, true, HF, d, true, V, d, M, ep_acc(Gp(kWte), d, beta), ws);
    mm<T>(LOG, vpad_, false, W(kWte), d, true, M, d, V, ep_store(DT, d), s);
    // norm backward: with fuse_ln_ the parameter gradients leave as per-block
    // partials of the dx kernel (one fold per micro-batch at the end), else a
    // separate reduction on the side stream reads dy and x again
    auto norm_bwd = [&](int ni, const T* dy, const T* x, const T* gam, const float* mu, const float* rs, int gi,
                        bool acc_dx) {
        if (fuse_ln_) {
            layernorm_bwd_fused<T>(dy, x, gam, mu, rs, DX, acc_dx, M, d, ln_part(ni), s);
            return;
        }
        fork();
        layernorm_bwd_params<T>(dy, x, mu, rs, Gp(gi), Gp(gi + 1), scratch_, M, d, acc, aux_);
        mark(kRdDT);
        guard(kRdDX);
        layernorm_bwd_dx<T>(dy, x, gam, mu, rs, DX, acc_dx, M, d, s);
    };
    norm_bwd(0, DT, X(L), W(kLnf), stat(4 * L), stat(4 * L + 1), kLnf, false);
    for (int l = L - 1; l >= 0; --l) {
        T *H1 = slot(l, sH1), *QKV = slot(l, sQKV), *Y = slot(l, sY), *XM = slot(l, sXM), *H2 = slot(l, sH2),
          *A = slot(l, sA), *U = slot(l, sU);
        // MLP
        fork();
        if (!fb_fc2) colsum_add<T>(DX, d, M, d, Gp(li(l, 11)), scratch_, acc, aux_);
        mm<T>(DX, d, true, U, 4 * d, true, d, 4 * d, M, ep_wg(Gp(li(l, 10)), 4 * d, Gp(li(l, 11)), fb_fc2), ws);
        mark(kRdDX);
        guard(kRdDA);
        mm<T>(DX, d, false, W(li(l, 10)), 4 * d, true, M, 4 * d, d, ep_dgelu(DA, 4 * d, A), s);
        fork();
        if (!fb_fc) colsum_add<T>(DA, 4 * d, M, 4 * d, Gp(li(l, 9)), scratch_, acc, aux_);
        mm<T>(DA, 4 * d, true, H2, d, true, 4 * d, d, M, ep_wg(Gp(li(l, 8)), d, Gp(li(l, 9)), fb_fc), ws);
        mark(kRdDA);
        guard(kRdDT);
        mm<T>(DA, 4 * d, false, W(li(l, 8)), d, true, M, d, 4 * d, ep_store(DT, d), s);
        guard(kRdDX);
        norm_bwd(2 + 2 * l, DT, XM, W(li(l, 6)), stat(4 * l + 2), stat(4 * l + 3), li(l, 6), true);
        // attention
        fork();
        if (!fb_proj) colsum_add<T>(DX, d, M, d, Gp(li(l, 5)), scratch_, acc, aux_);
        mm<T>(DX, d, true, Y, d, true, d, d, M, ep_wg(Gp(li(l, 4)), d, Gp(li(l, 5)), fb_proj), ws);
        mark(kRdDX);
        guard(kRdDT);
        mm<T>(DX, d, false, W(li(l, 4)), d, true, M, d, d, ep_store(DT, d), s);
        guard(kRdDQKV);
        attention_bwd<T>(QKV, Y, lse_ + static_cast<int64_t>(l) * H * Mmax, DT, DQKV, dsum_, B, Tq, H, H, hd, s);
        fork();
        if (!fb_qkv) colsum_add<T>(DQKV, 3 * d, M, 3 * d, Gp(li(l, 3)), scratch_, acc, aux_);
        mm<T>(DQKV, 3 * d, true, H1, d, true, 3 * d, d, M, ep_wg(Gp(li(l, 2)), d, Gp(li(l, 3)), fb_qkv), ws);
        mark(kRdDQKV);
        mm<T>(DQKV, 3 * d, false, W(li(l, 2)), d, true, M, d, 3 * d, ep_store(DT, d), s);
        guard(kRdDX);
        norm_bwd(1 + 2 * l, DT, X(l), W(li(l, 0)), stat(4 * l), stat(4 * l + 1), li(l, 0), true);
    }
    if (fuse_ln_) ln_param_fold(ln_fold_, n_ln_, d, ln_part_, G, acc, s);
    // wte rows: the head wgrad stored/added every row; the embedding adds (after it)
    join();
    ACCO_CUDA(cudaStreamWaitEvent(s, ev_sort_, 0));
    embed_bwd<T>(sort_, DX, M, Tq, d, V, Gp(kWte), Gp(kWpe), run_sum_, acc, s);
    join();  // the accumulator is complete when the compute stream passes this point
}

// Llama block (oracle/gpt_oracle.py _llama_loss_and_grad). Parameter indices
// in layout_: 0 wte; per layer 1 + 6l + {0 attention_norm, 1 wqkv, 2 wo,
// 3 ffn_norm, 4 w_gate_up, 5 w_down}; then norm, output.
template <class T>
void GPTModel::run_llama(const T* P, uint64_t seed, int mode, int start, int B, float* G, double* loss,
                         bool backward, cudaStream_t s) {
    const int Tq = c_.seq_len, d = c_.d_model, H = c_.n_head, Hk = c_.kv_heads(), hd = d / H, V = c_.vocab,
              L = c_.n_layer, F = c_.ffn();
    const int nqkv = (H + 2 * Hk) * hd;
    ACCO_REQUIRE(B >= 1 && B <= c_.max_batch, "micro_batch: batch size exceeds the model workspace");
    if (mode == 1) ACCO_REQUIRE(start >= 0 && start + B <= c_.n_samples, "micro_batch: sample range out of bounds");
    const int M = B * Tq;
    const int64_t Mmax = static_cast<int64_t>(c_.max_batch) * Tq;
    auto slot = [&](int l, int sl) { return reinterpret_cast<T*>(act_[static_cast<size_t>(l * kPerLayer + sl)]); };
    const int tail = L * kPerLayer;
    T* XL = reinterpret_cast<T*>(act_[tail + 0]);
    T* HF = reinterpret_cast<T*>(act_[tail + 1]);
    T* LOG = reinterpret_cast<T*>(act_[tail + 2]);
    T* DX = reinterpret_cast<T*>(act_[tail + 3]);
    T* DT = reinterpret_cast<T*>(act_[tail + 4]);
    T* DQKV = reinterpret_cast<T*>(act_[tail + 5]);
    T* DGU = reinterpret_cast<T*>(act_[tail + 6]);
    T* DU = reinterpret_cast<T*>(act_[tail + 7]);
    auto X = [&](int l) { return l == L ? XL : slot(l, sX); };
    auto stat = [&](int i) { return stats_ + static_cast<int64_t>(i) * Mmax; };
    auto W = [&](int i) { return P + layout_[static_cast<size_t>(i)].off; };
    auto Gp = [&](int i) { return G + layout_[static_cast<size_t>(i)].off; };
    const int kWte = 0, kNorm = 1 + 6 * L, kOut = 2 + 6 * L;
    auto li = [&](int l, int j) { return 1 + 6 * l + j; };
    auto lse_l = [&](int l) { return lse_ + static_cast<int64_t>(l) * H * Mmax; };

    // SwiGLU fused into the gate|up GEMM epilogue on the bf16 tcgen05 path
    const bool no_fuse = std::getenv("ACCO_NO_SWIGLU_FUSION") != nullptr;  // A/B knob, read per call
    const bool swiglu_fused = sizeof(T) == 2 && F % 128 == 0 && !no_fuse;
    stage_input(seed, mode, start, B, s);
    if (backward) sort_tokens(M, s);
    embed_fwd<T>(tok_in_, W(kWte), nullptr, X(0), M, Tq, d, s);
    for (int l = 0; l < L; ++l) {
        T *H1 = slot(l, sH1), *QKV = slot(l, sQKV), *Y = slot(l, sY), *XM = slot(l, sXM), *H2 = slot(l, sH2),
          *GU = slot(l, sA), *A = slot(l, sU);
        layernorm_fwd<T>(X(l), W(li(l, 0)), nullptr, H1, stat(4 * l), stat(4 * l + 1), M, d, s, true);
        mm<T>(H1, d, false, W(li(l, 1)), d, false, M, nqkv, d, ep_store(QKV, nqkv), s);
        rope_apply<T>(QKV, nqkv, rope_, M, Tq, H + Hk, hd, false, s);
        attention_fwd<T>(QKV, Y, lse_l(l), B, Tq, H, Hk, hd, s);
        mm<T>(Y, d, false, W(li(l, 2)), d, false, M, d, d, ep_store(XM, d, nullptr, X(l), d), s);
        layernorm_fwd<T>(XM, W(li(l, 3)), nullptr, H2, stat(4 * l + 2), stat(4 * l + 3), M, d, s, true);
        if (swiglu_fused) {  // gate|up GEMM with silu(gate) * up in its epilogue
            Epilogue e = ep_store(A, F);
            e.mode = kEpiSwiGLU;
            e.aux = GU;
            e.ld_aux = 2 * F;
            mm<T>(H2, d, false, W(li(l, 4)), d, false, M, 2 * F, d, e, s);
        } else {
            mm<T>(H2, d, false, W(li(l, 4)), d, false, M, 2 * F, d, ep_store(GU, 2 * F), s);
            swiglu_fwd<T>(GU, A, M, F, s);
        }
        mm<T>(A, F, false, W(li(l, 5)), F, false, M, d, F, ep_store(X(l + 1), d, nullptr, XM, d), s);
    }
    layernorm_fwd<T>(X(L), W(kNorm), nullptr, HF, stat(4 * L), stat(4 * L + 1), M, d, s, true);
    mm<T>(HF, d, false, W(kOut), d, false, M, V, d, ep_store(LOG, vpad_), s);
    cross_entropy<T>(LOG, vpad_, tok_out_, V, M, Tq, row_loss_, s);
    loss_reduce(row_loss_, M, Tq, loss, s);
    if (!backward) return;

    const bool acc = accumulate_;
    const int beta = acc ? 1 : 0;
    // ACCO_SERIAL_REDUCE=1 (diagnostic A/B): the reductions run inline on s
    static const bool serial = std::getenv("ACCO_SERIAL_REDUCE") != nullptr;
    cudaStream_t aux_ = serial ? s : this->aux_;
    auto fork = [&] {
        if (serial) return;
        ACCO_CUDA(cudaEventRecord(ev_fork_, s));
        ACCO_CUDA(cudaStreamWaitEvent(aux_, ev_fork_, 0));
    };
    auto join = [&] {
        if (serial) return;
        ACCO_CUDA(cudaEventRecord(ev_join_, aux_));
        ACCO_CUDA(cudaStreamWaitEvent(s, ev_join_, 0));
    };
    // LM head (untied): doutput (+)= dlogits^T hf ; dhf = dlogits output
    mm<T>(LOG, vpad_, true, HF, d, true, V, d, M, ep_acc(Gp(kOut), d, beta), s);
    mm<T>(LOG, vpad_, false, W(kOut), d, true, M, d, V, ep_store(DT, d), s);
    // RMSNorm backward (see run: fused parameter partials, or a side-stream reduction)
    auto norm_bwd = [&](int ni, const T* x, const T* gam, const float* mu, const float* rs, int gi, bool acc_dx) {
        if (fuse_ln_) {
            layernorm_bwd_fused<T>(DT, x, gam, mu, rs, DX, acc_dx, M, d, ln_part(ni), s, true);
            return;
        }
        fork();
        layernorm_bwd_params<T>(DT, x, mu, rs, Gp(gi), nullptr, scratch_, M, d, acc, aux_);
        layernorm_bwd_dx<T>(DT, x, gam, mu, rs, DX, acc_dx, M, d, s, true);
    };
    norm_bwd(0, X(L), W(kNorm), stat(4 * L), stat(4 * L + 1), kNorm, false);
    for (int l = L - 1; l >= 0; --l) {
        T *H1 = slot(l, sH1), *QKV = slot(l, sQKV), *Y = slot(l, sY), *XM = slot(l, sXM), *H2 = slot(l, sH2),
          *GU = slot(l, sA), *A = slot(l, sU);
        // MLP
        mm<T>(DX, d, true, A, F, true, d, F, M, ep_acc(Gp(li(l, 5)), F, beta), s);
        if (swiglu_fused) {  // SwiGLU backward in the down-projection dgrad epilogue
            Epilogue e = ep_store(DGU, 2 * F);
            e.mode = kEpiDSwiGLU;
            e.aux = GU;
            e.ld_aux = 2 * F;
            mm<T>(DX, d, false, W(li(l, 5)), F, true, M, F, d, e, s);
        } else {
            mm<T>(DX, d, false, W(li(l, 5)), F, true, M, F, d, ep_store(DU, F), s);
            swiglu_bwd<T>(DU, GU, DGU, M, F, s);
        }
        mm<T>(DGU, 2 * F, true, H2, d, true, 2 * F, d, M, ep_acc(Gp(li(l, 4)), d, beta), s);
        join();  // DT (read by the previous norm-weight reduction) is overwritten next
        mm<T>(DGU, 2 * F, false, W(li(l, 4)), d, true, M, d, 2 * F, ep_store(DT, d), s);
        norm_bwd(2 + 2 * l, XM, W(li(l, 3)), stat(4 * l + 2), stat(4 * l + 3), li(l, 3), true);
        // attention
        mm<T>(DX, d, true, Y, d, true, d, d, M, ep_acc(Gp(li(l, 2)), d, beta), s);
        join();
        mm<T>(DX, d, false, W(li(l, 2)), d, true, M, d, d, ep_store(DT, d), s);
        attention_bwd<T>(QKV, Y, lse_l(l), DT, DQKV, dsum_, B, Tq, H, Hk, hd, s);
        rope_apply<T>(DQKV, nqkv, rope_, M, Tq, H + Hk, hd, true, s);
        mm<T>(DQKV, nqkv, true, H1, d, true, nqkv, d, M, ep_acc(Gp(li(l, 1)), d, beta), s);
        mm<T>(DQKV, nqkv, false, W(li(l, 1)), d, true, M, d, nqkv, ep_store(DT, d), s);
        norm_bwd(1 + 2 * l, X(l), W(li(l, 0)), stat(4 * l), stat(4 * l + 1), li(l, 0), true);
    }
    if (fuse_ln_) ln_param_fold(ln_fold_, n_ln_, d, ln_part_, G, acc, s);
    ACCO_CUDA(cudaStreamWaitEvent(s, ev_sort_, 0));
    embed_bwd<T>(sort_, DX, M, Tq, d, V, Gp(kWte), nullptr, run_sum_, acc, s, !acc);
    join();
}

void GPTModel::micro_batch(const void* params, uint64_t seed, int mode, int start, int B, float* grad_acc,
                           double* loss_sum, cudaStream_t s, bool accumulate) {
    accumulate_ = accumulate;
    if (c_.precision == 1)
        run<__nv_bfloat16>(static_cast<const __nv_bfloat16*>(params), seed, mode, start, B, grad_acc, loss_sum, true, s);
    else
        run<float>(static_cast<const float*>(params), seed, mode, start, B, grad_acc, loss_sum, true, s);
}

void GPTModel::forward_loss(const void* params, uint64_t seed, int mode, int start, int B, double* loss_sum,
                            cudaStream_t s) {
    if (c_.precision == 1)
        run<__nv_bfloat16>(static_cast<const __nv_bfloat16*>(params), seed, mode, start, B, nullptr, loss_sum, false, s);
    else
        run<float>(static_cast<const float*>(params), seed, mode, start, B, nullptr, loss_sum, false, s);
}

}  // namespace acco
