// Host-side optimizer types (mirror of proj/include/accosim/optim.hpp:21-64).
#pragma once

#include "acco.h"
#include "common.cuh"

namespace acco {

struct OptConfig {
    int kind = 0;  // 0 sgd, 1 adam, 2 adamw
    double learning_rate = 0.0;
    double adam_beta1 = 0.9;
    double adam_beta2 = 0.999;
    double adam_eps = 1e-8;
    double weight_decay = 0.0;
    int scheduler = 0;  // 0 constant, 1 cosine
    int n_warmup_steps = 0;
    long long total_steps = 0;
    double cosine_min_factor = 0.0;
};

inline OptConfig from_c(const acco_opt_cfg& c) {
    OptConfig o;
    o.kind = c.kind;
    o.learning_rate = c.learning_rate;
    o.adam_beta1 = c.adam_beta1;
    o.adam_beta2 = c.adam_beta2;
    o.adam_eps = c.adam_eps;
    o.weight_decay = c.weight_decay;
    o.scheduler = c.scheduler;
    o.n_warmup_steps = c.n_warmup_steps;
    o.total_steps = c.total_steps;
    o.cosine_min_factor = c.cosine_min_factor;
    return o;
}

double scheduled_lr(const OptConfig& cfg, long long t);
void validate(const OptConfig& cfg);

// One fused pass per comm phase over a shard of n elements: fold the gradient
// sums src[0..nsrc) in order (the reference Fabric's reduce order — local
// virtual workers, or peers' accumulators over NVLink), optionally keep the
// folded sum (estimate's retained shard), apply the optimizer step, and write
// the new parameters to every destination replica (local and/or peers').
constexpr int kMaxFold = 16;
struct FoldIO {
    const float* src[kMaxFold] = {};
    int nsrc = 0;
    void* dst[kMaxFold] = {};
    int ndst = 0;
    float* ret_out = nullptr;
};
void opt_fold(const OptConfig& cfg, long long step, bool commit, const FoldIO& io, const float* gret,
              const int64_t* total_dev, const int64_t* rtotal_dev, float* theta, float* m, float* v, int64_t n,
              int out_dtype, int* flag, cudaStream_t stream);

// Single-source form (see optim.cu).
// commit=false: estimate (pure); commit=true: persistent update of theta/m/v.
void opt_apply(const OptConfig& cfg, long long step, bool commit, const float* gsum,
               const float* gret, const int64_t* total_dev, const int64_t* rtotal_dev,
               float* theta, float* m, float* v, int64_t n, void* out, int out_dtype, int* flag,
               cudaStream_t stream);

template <class T>
__device__ __forceinline__ T from_f_opt(float x);
template <>
__device__ __forceinline__ float from_f_opt<float>(float x) { return x; }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f_opt<__nv_bfloat16>(float x) {
    return __float2bfloat16_rn(x);
}

template <class OutT>
__device__ __forceinline__ void store4(void* out, int64_t q, float4 v);
template <>
__device__ __forceinline__ void store4<float>(void* out, int64_t q, float4 v) {
    reinterpret_cast<float4*>(out)[q] = v;
}
template <>
__device__ __forceinline__ void store4<__nv_bfloat16>(void* out, int64_t q, float4 v) {
    __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y);
    __nv_bfloat162 hi = __floats2bfloat162_rn(v.z, v.w);
    uint2 pk;
    pk.x = *reinterpret_cast<uint32_t*>(&lo);
    pk.y = *reinterpret_cast<uint32_t*>(&hi);
    reinterpret_cast<uint2*>(out)[q] = pk;
}

}  // namespace acco
