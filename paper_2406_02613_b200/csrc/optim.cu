// Fused sharded optimizer kernels — K6 (ACCO estimate) and K7 (ACCO commit)
// of SURVEY.md §2.3, restating opt_step (/root/reference/proj/src/optim.cpp:50-92)
// as one HBM-streaming pass over the shard:
//
//   estimate: reads g_sum, theta, m, v; writes theta_est (bf16/fp32 all-gather
//             payload). Moments are read but never written: the reference runs
//             the estimate on a *transient copy* of the shard state
//             (protocols.cpp:654), so it is a pure function here.      18 B/elem (AdamW, bf16 out)
//   commit  : reads g_sum, g_retained, theta, m, v; writes theta, m, v and the
//             all-gather payload.                                       34 B/elem
//
// 1/total, 1/(total+retained), the learning-rate schedule and both bias
// corrections are folded in; totals are read from device memory (the output of
// the counts all-reduce), so the comm stream never synchronises with the host.
#include "acco.h"
#include "capi_util.h"
#include "common.cuh"
#include "optim.h"

#include <algorithm>
#include <cmath>
#include <cstdlib>

namespace acco {

double scheduled_lr(const OptConfig& cfg, long long t) {
    // proj/src/optim.cpp:37-48
    const double peak = cfg.learning_rate;
    const long long warmup = cfg.n_warmup_steps;
    if (t < warmup) return peak * static_cast<double>(t + 1) / static_cast<double>(warmup);
    if (cfg.scheduler == 0) return peak;
    const double floor = peak * cfg.cosine_min_factor;
    const long long span = cfg.total_steps - 1 - warmup;
    if (span <= 0) return peak;
    double x = static_cast<double>(t - warmup) / static_cast<double>(span);
    if (x > 1.0) x = 1.0;
    return floor + (peak - floor) * 0.5 * (1.0 + std::cos(3.14159265358979323846 * x));
}

void validate(const OptConfig& cfg) {
    ACCO_REQUIRE(cfg.kind >= 0 && cfg.kind <= 2, "optimizer: unknown kind");
    ACCO_REQUIRE(cfg.learning_rate > 0.0, "optimizer: learning_rate > 0");
    ACCO_REQUIRE(cfg.adam_beta1 >= 0.0 && cfg.adam_beta1 < 1.0 && cfg.adam_beta2 >= 0.0 &&
                     cfg.adam_beta2 < 1.0,
                 "optimizer: adam betas must lie in [0, 1)");
    ACCO_REQUIRE(cfg.weight_decay >= 0.0, "optimizer: weight_decay >= 0");
}

namespace {

struct KArgs {
    const float* src[kMaxFold];  // gradient sums folded in this order (reference: ascending worker)
    int nsrc;
    void* dst[kMaxFold];         // every destination receives the new parameters (activation dtype)
    int ndst;
    float* ret_out;              // estimate: keep the raw folded sum (the retained shard)
    const float* gret;
    const int64_t* total;
    const int64_t* rtotal;
    float* theta;  // read; written by commit
    float* m;
    float* v;
    int64_t n;
    float lr, b1, b2, omb1, omb2, c1, c2, eps, wd;
    int* flag;
};

template <class OutT>
__device__ __forceinline__ void store_out(void* out, int64_t i, float x) {
    static_cast<OutT*>(out)[i] = from_f_opt<OutT>(x);
}

// One element of opt_step; returns the new theta and updates m/v in registers.
// Every rounding is pinned with _rn intrinsics (no compiler-chosen FMA
// contraction), so the float4 path, the scalar path and any shard split give
// bitwise-identical results — sharded == unsharded (verify.cpp:274-324).
template <int KIND>
__device__ __forceinline__ float step_elem(const KArgs& a, float g, float th, float& m, float& v) {
    if (KIND == 0) {  // sgd: theta -= lr * (g + wd*theta)
        return __fmaf_rn(-a.lr, __fmaf_rn(a.wd, th, g), th);
    }
    if (KIND == 1) g = __fmaf_rn(a.wd, th, g);  // adam: coupled decay
    m = __fmaf_rn(a.b1, m, __fmul_rn(a.omb1, g));
    v = __fmaf_rn(a.b2, v, __fmul_rn(__fmul_rn(a.omb2, g), g));
    const float mh = __fdiv_rn(m, a.c1);
    const float vh = __fdiv_rn(v, a.c2);
    float u = __fdiv_rn(mh, __fadd_rn(__fsqrt_rn(vh), a.eps));
    if (KIND == 2) u = __fmaf_rn(a.wd, th, u);  // adamw: decoupled decay
    return __fmaf_rn(-a.lr, u, th);
}

__device__ __forceinline__ float scale_grad(float g, float r, float inv, bool has_ret) {
    return __fmul_rn(has_ret ? __fadd_rn(g, r) : g, inv);
}

template <int KIND, bool COMMIT, bool HAS_RET, class OutT, bool VEC>
__global__ void __launch_bounds__(256) opt_kernel(KArgs a) {
    ACCO_PDL_PROLOGUE();
    int64_t tot = *a.total;
    if (HAS_RET && a.rtotal) tot += *a.rtotal;
    const float inv = static_cast<float>(1.0 / static_cast<double>(tot));
    bool bad = false, bad_out = false;  // non-finite input (opt_step's invalid_argument) / new parameters
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t n4 = VEC ? a.n / 4 : 0;
    if (VEC) {
        for (int64_t q = tid; q < n4; q += stride) {
            // Fabric fold (collectives.cpp:55-75): copy of the first input, then
            // += the others in order
            float4 g = __ldcs(reinterpret_cast<const float4*>(a.src[0]) + q);
            for (int k = 1; k < a.nsrc; ++k) {
                const float4 h = __ldcs(reinterpret_cast<const float4*>(a.src[k]) + q);
                g.x = __fadd_rn(g.x, h.x);
                g.y = __fadd_rn(g.y, h.y);
                g.z = __fadd_rn(g.z, h.z);
                g.w = __fadd_rn(g.w, h.w);
            }
            if (!COMMIT && a.ret_out) reinterpret_cast<float4*>(a.ret_out)[q] = g;
            float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
            if (HAS_RET) r = __ldcs(reinterpret_cast<const float4*>(a.gret) + q);
            g.x = scale_grad(g.x, r.x, inv, HAS_RET);
            g.y = scale_grad(g.y, r.y, inv, HAS_RET);
            g.z = scale_grad(g.z, r.z, inv, HAS_RET);
            g.w = scale_grad(g.w, r.w, inv, HAS_RET);
            float4 th = reinterpret_cast<const float4*>(a.theta)[q];
            float4 m = make_float4(0.f, 0.f, 0.f, 0.f), v = m;
            if (KIND != 0) {
                m = reinterpret_cast<const float4*>(a.m)[q];
                v = reinterpret_cast<const float4*>(a.v)[q];
            }
            bad |= !(isfinite(g.x) && isfinite(g.y) && isfinite(g.z) && isfinite(g.w) &&
                     isfinite(th.x) && isfinite(th.y) && isfinite(th.z) && isfinite(th.w));
            float4 nt;
            nt.x = step_elem<KIND>(a, g.x, th.x, m.x, v.x);
            nt.y = step_elem<KIND>(a, g.y, th.y, m.y, v.y);
            nt.z = step_elem<KIND>(a, g.z, th.z, m.z, v.z);
            nt.w = step_elem<KIND>(a, g.w, th.w, m.w, v.w);
            if (COMMIT) {
                reinterpret_cast<float4*>(a.theta)[q] = nt;
                if (KIND != 0) {
                    reinterpret_cast<float4*>(a.m)[q] = m;
                    reinterpret_cast<float4*>(a.v)[q] = v;
                }
            }
            bad_out |= !(isfinite(nt.x) && isfinite(nt.y) && isfinite(nt.z) && isfinite(nt.w));
            for (int k = 0; k < a.ndst; ++k) store4<OutT>(a.dst[k], q, nt);
        }
    }
    // scalar path (unaligned shards) and the n % 4 tail of the vector path
    for (int64_t i = n4 * 4 + tid; i < a.n; i += stride) {
        float g = a.src[0][i];
        for (int k = 1; k < a.nsrc; ++k) g = __fadd_rn(g, a.src[k][i]);
        if (!COMMIT && a.ret_out) a.ret_out[i] = g;
        g = scale_grad(g, HAS_RET ? a.gret[i] : 0.f, inv, HAS_RET);
        float th = a.theta[i];
        float m = KIND != 0 ? a.m[i] : 0.f, v = KIND != 0 ? a.v[i] : 0.f;
        bad |= !(isfinite(g) && isfinite(th));
        float nt = step_elem<KIND>(a, g, th, m, v);
        bad_out |= !isfinite(nt);
        if (COMMIT) {
            a.theta[i] = nt;
            if (KIND != 0) { a.m[i] = m; a.v[i] = v; }
        }
        for (int k = 0; k < a.ndst; ++k) store_out<OutT>(a.dst[k], i, nt);
    }
    // bit 0: a non-finite gradient or parameter entered the step (the
    // reference's opt_step throws invalid_argument, optim.cpp:56-57); bit 1:
    // the step produced a non-finite parameter (the next commit's finite-state
    // check makes the loss +inf: diverged, protocols.cpp:113-119,164-167)
    if ((bad || bad_out) && a.flag) atomicOr(a.flag, (bad ? 1 : 0) | (bad_out ? 2 : 0));
}

template <int KIND, bool COMMIT, bool HAS_RET, class OutT>
const void* vec_kernel_ptr() {
    return reinterpret_cast<const void*>(opt_kernel<KIND, COMMIT, HAS_RET, OutT, true>);
}

template <int KIND, bool COMMIT, bool HAS_RET, class OutT>
void launch_vec(const KArgs& a, bool vec, cudaStream_t s) {
    const int threads = 256;
    // persistent grid: exactly the blocks that are resident at once (40-54
    // registers: 4-6 blocks of 256 per SM, not 8 — a fixed 8 x 148 grid left a
    // second, partly occupied wave behind the first one)
    const int64_t work = vec ? (a.n + 3) / 4 : a.n;
    static const int per_sm = [] {
        int nb = 0;
        auto k = vec_kernel_ptr<KIND, COMMIT, HAS_RET, OutT>();
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, 256, 0) != cudaSuccess || nb < 1) nb = 4;
        return nb;
    }();
    int64_t cap = static_cast<int64_t>(num_sms()) * per_sm;
    if (const char* e = std::getenv("ACCO_OPT_BLOCKS")) cap = std::max<int64_t>(1, std::atoll(e));  // tuning knob
    int blocks = static_cast<int>(std::min<int64_t>((work + threads - 1) / threads, cap));
    if (blocks < 1) blocks = 1;
    if (vec)
        launch_pdl(opt_kernel<KIND, COMMIT, HAS_RET, OutT, true>, blocks, threads, 0, s, a);
    else
        launch_pdl(opt_kernel<KIND, COMMIT, HAS_RET, OutT, false>, blocks, threads, 0, s, a);
    ACCO_CHECK_LAUNCH();
}

template <bool COMMIT, bool HAS_RET, class OutT>
void launch_kind(int kind, const KArgs& a, bool vec, cudaStream_t s) {
    if (kind == 0) launch_vec<0, COMMIT, HAS_RET, OutT>(a, vec, s);
    else if (kind == 1) launch_vec<1, COMMIT, HAS_RET, OutT>(a, vec, s);
    else launch_vec<2, COMMIT, HAS_RET, OutT>(a, vec, s);
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

void opt_fold(const OptConfig& cfg, long long step, bool commit, const FoldIO& io, const float* gret,
              const int64_t* total_dev, const int64_t* rtotal_dev, float* theta, float* m, float* v, int64_t n,
              int out_dtype, int* flag, cudaStream_t stream) {
    if (n == 0) return;  // empty trailing shard: no-op (test_optim.cpp:168-181)
    validate(cfg);
    ACCO_REQUIRE(io.nsrc >= 1 && io.nsrc <= kMaxFold && io.ndst >= 0 && io.ndst <= kMaxFold,
                 "optimizer: 1..16 sources, 0..16 destinations");
    ACCO_REQUIRE(theta && total_dev, "optimizer: null shard pointer");
    ACCO_REQUIRE(cfg.kind == 0 || (m && v), "optimizer: adam/adamw need m and v");
    ACCO_REQUIRE(out_dtype == ACCO_DTYPE_F32 || out_dtype == ACCO_DTYPE_BF16, "optimizer: bad out dtype");
    KArgs a{};
    bool vec = aligned16(theta) && (cfg.kind == 0 || (aligned16(m) && aligned16(v))) && (!gret || aligned16(gret)) &&
               (!io.ret_out || aligned16(io.ret_out));
    for (int k = 0; k < io.nsrc; ++k) {
        ACCO_REQUIRE(io.src[k], "optimizer: null gradient source");
        a.src[k] = io.src[k];
        vec = vec && aligned16(io.src[k]);
    }
    for (int k = 0; k < io.ndst; ++k) {
        a.dst[k] = io.dst[k];
        vec = vec && (reinterpret_cast<uintptr_t>(io.dst[k]) & (out_dtype == ACCO_DTYPE_BF16 ? 7 : 15)) == 0;
    }
    a.nsrc = io.nsrc;
    a.ndst = io.ndst;
    a.ret_out = io.ret_out;
    a.gret = gret;
    a.total = total_dev;
    a.rtotal = rtotal_dev;
    a.theta = theta;
    a.m = m;
    a.v = v;
    a.n = n;
    a.flag = flag;
    // lr(t) and bias correction with step t+1 (optim.cpp:59-74); the estimate
    // and the commit of round t both use the same `step`.
    const double lr = scheduled_lr(cfg, step);
    const double st = static_cast<double>(step + 1);
    a.lr = static_cast<float>(lr);
    a.b1 = static_cast<float>(cfg.adam_beta1);
    a.b2 = static_cast<float>(cfg.adam_beta2);
    a.omb1 = static_cast<float>(1.0 - cfg.adam_beta1);
    a.omb2 = static_cast<float>(1.0 - cfg.adam_beta2);
    a.c1 = static_cast<float>(1.0 - std::pow(cfg.adam_beta1, st));
    a.c2 = static_cast<float>(1.0 - std::pow(cfg.adam_beta2, st));
    a.eps = static_cast<float>(cfg.adam_eps);
    a.wd = static_cast<float>(cfg.weight_decay);
    const bool has_ret = gret != nullptr;
    // algorithmic bytes per element: reads the folded sums
    // (+ retained), theta (+ m, v); commit writes theta (+ m, v); estimate may
    // keep the retained sum; payload 2 (bf16) / 4 B per destination.
    const int mv = cfg.kind != 0 ? 8 : 0;
    const double per_elem = 4.0 * io.nsrc + (has_ret ? 4 : 0) + 4 + mv + (commit ? 4 + mv : 0) +
                            (io.ret_out ? 4 : 0) + io.ndst * (out_dtype == ACCO_DTYPE_BF16 ? 2 : 4);
    ProfScope prof(kProfOpt, per_elem * static_cast<double>(n), stream);
#define ACCO_OPT_DISPATCH(C)                                                                    \
    if (out_dtype == ACCO_DTYPE_BF16) {                                                         \
        if (has_ret) launch_kind<C, true, __nv_bfloat16>(cfg.kind, a, vec, stream);             \
        else launch_kind<C, false, __nv_bfloat16>(cfg.kind, a, vec, stream);                    \
    } else {                                                                                    \
        if (has_ret) launch_kind<C, true, float>(cfg.kind, a, vec, stream);                     \
        else launch_kind<C, false, float>(cfg.kind, a, vec, stream);                            \
    }
    if (commit) {
        ACCO_OPT_DISPATCH(true)
    } else {
        ACCO_OPT_DISPATCH(false)
    }
#undef ACCO_OPT_DISPATCH
}

void opt_apply(const OptConfig& cfg, long long step, bool commit, const float* gsum, const float* gret,
               const int64_t* total_dev, const int64_t* rtotal_dev, float* theta, float* m, float* v, int64_t n,
               void* out, int out_dtype, int* flag, cudaStream_t stream) {
    FoldIO io;
    io.src[0] = gsum;
    io.nsrc = 1;
    if (out) {
        io.dst[0] = out;
        io.ndst = 1;
    }
    opt_fold(cfg, step, commit, io, gret, total_dev, rtotal_dev, theta, m, v, n, out_dtype, flag, stream);
}

}  // namespace acco

using namespace acco;

extern "C" {

double acco_scheduled_lr(const acco_opt_cfg* cfg, long long t) {
    return scheduled_lr(from_c(*cfg), t);
}

int acco_opt_estimate(const acco_opt_cfg* cfg, const acco_shard_state* st, const float* gsum,
                      const int64_t* total_dev, void* theta_out, int out_dtype, int* nonfinite_flag,
                      void* stream) {
    return guarded([&] {
        ACCO_REQUIRE(cfg && st, "acco_opt_estimate: null argument");
        ACCO_REQUIRE(st->hi >= st->lo, "acco_opt_estimate: bad shard range");
        ACCO_REQUIRE(theta_out, "acco_opt_estimate: theta_out required");
        opt_apply(from_c(*cfg), st->step, false, gsum, nullptr, total_dev, nullptr, st->theta, st->m,
                  st->v, static_cast<int64_t>(st->hi - st->lo), theta_out, out_dtype, nonfinite_flag,
                  static_cast<cudaStream_t>(stream));
    });
}

int acco_opt_commit(const acco_opt_cfg* cfg, acco_shard_state* st, const float* gsum,
                    const float* g_retained, const int64_t* total_dev,
                    const int64_t* retained_total_dev, void* theta_out, int out_dtype,
                    int* nonfinite_flag, void* stream) {
    return guarded([&] {
        ACCO_REQUIRE(cfg && st, "acco_opt_commit: null argument");
        ACCO_REQUIRE(st->hi >= st->lo, "acco_opt_commit: bad shard range");
        opt_apply(from_c(*cfg), st->step, true, gsum, g_retained, total_dev,
                  g_retained ? retained_total_dev : nullptr, st->theta, st->m, st->v,
                  static_cast<int64_t>(st->hi - st->lo), theta_out, out_dtype, nonfinite_flag,
                  static_cast<cudaStream_t>(stream));
        st->step += 1;
    });
}

}  // extern "C"
