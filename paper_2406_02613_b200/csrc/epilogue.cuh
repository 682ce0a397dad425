// GEMM epilogue shared by the tcgen05 (bf16) and SIMT (fp32) kernels.
#pragma once

#include "common.cuh"
#include "gemm.h"

namespace acco {

__device__ __forceinline__ float to_f(float x) { return x; }
__device__ __forceinline__ float to_f(__nv_bfloat16 x) { return __bfloat162float(x); }
template <class T> __device__ __forceinline__ T from_f(float x);
template <> __device__ __forceinline__ float from_f<float>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) {
    return __float2bfloat16_rn(x);
}

// GPT-2 "gelu_new" (tanh form); the fp64 oracle uses the same formula.
__device__ __forceinline__ float gelu_f(float x) {
    const float k0 = 0.7978845608028654f, k1 = 0.044715f;
    float t = tanhf(k0 * (x + k1 * x * x * x));
    return 0.5f * x * (1.0f + t);
}
__device__ __forceinline__ float dgelu_f(float x) {
    const float k0 = 0.7978845608028654f, k1 = 0.044715f;
    float t = tanhf(k0 * (x + k1 * x * x * x));
    return 0.5f * (1.0f + t) + 0.5f * x * (1.0f - t * t) * k0 * (1.0f + 3.0f * k1 * x * x);
}

// Apply the epilogue to `n` consecutive output columns [col, col+n) of one row.
// x[] holds the fp32 accumulators and is clobbered.
template <class T, int NV>
__device__ __forceinline__ void epilogue_row(const Epilogue& ep, int row, int col, int n, float* x) {
    if (ep.mode == kEpiAccF32) {
        float* c = static_cast<float*>(ep.C) + (int64_t)row * ep.ldc + col;
        if (n == NV && (ep.ldc % 4 == 0) && (col % 4 == 0)) {
#pragma unroll
            for (int i = 0; i < NV; i += 4) {
                float4 o = make_float4(x[i], x[i + 1], x[i + 2], x[i + 3]);
                if (ep.beta) {
                    float4 p = *reinterpret_cast<const float4*>(c + i);
                    o.x += p.x; o.y += p.y; o.z += p.z; o.w += p.w;
                }
                *reinterpret_cast<float4*>(c + i) = o;
            }
        } else {
#pragma unroll
            for (int i = 0; i < NV; ++i)
                if (i < n) c[i] = ep.beta ? c[i] + x[i] : x[i];
        }
        return;
    }
    const T* bias = static_cast<const T*>(ep.bias);
    if (bias) {
#pragma unroll
        for (int i = 0; i < NV; ++i)
            if (i < n) x[i] += to_f(bias[col + i]);
    }
    if (ep.mode == kEpiGelu) {
        T* aux = static_cast<T*>(ep.aux) + (int64_t)row * ep.ld_aux + col;
#pragma unroll
        for (int i = 0; i < NV; ++i)
            if (i < n) {
                aux[i] = from_f<T>(dgelu_f(x[i]));  // the slope, consumed by kEpiDGelu
                x[i] = gelu_f(x[i]);
            }
    } else if (ep.mode == kEpiDGelu) {
        const T* aux = static_cast<const T*>(ep.aux) + (int64_t)row * ep.ld_aux + col;
#pragma unroll
        for (int i = 0; i < NV; ++i)
            if (i < n) x[i] *= to_f(aux[i]);
    }
    if (ep.residual) {
        const T* r = static_cast<const T*>(ep.residual) + (int64_t)row * ep.ldr + col;
#pragma unroll
        for (int i = 0; i < NV; ++i)
            if (i < n) x[i] += to_f(r[i]);
    }
    T* c = static_cast<T*>(ep.C) + (int64_t)row * ep.ldc + col;
    if constexpr (sizeof(T) == 2 && NV % 8 == 0) {
        if (n == NV && (ep.ldc % 8 == 0) && (col % 8 == 0)) {
#pragma unroll
            for (int i = 0; i < NV; i += 8) {
                uint4 pk;
                __nv_bfloat162 h0 = __floats2bfloat162_rn(x[i], x[i + 1]);
                __nv_bfloat162 h1 = __floats2bfloat162_rn(x[i + 2], x[i + 3]);
                __nv_bfloat162 h2 = __floats2bfloat162_rn(x[i + 4], x[i + 5]);
                __nv_bfloat162 h3 = __floats2bfloat162_rn(x[i + 6], x[i + 7]);
                pk.x = *reinterpret_cast<uint32_t*>(&h0);
                pk.y = *reinterpret_cast<uint32_t*>(&h1);
                pk.z = *reinterpret_cast<uint32_t*>(&h2);
                pk.w = *reinterpret_cast<uint32_t*>(&h3);
                *reinterpret_cast<uint4*>(c + i) = pk;
            }
            return;
        }
    }
#pragma unroll
    for (int i = 0; i < NV; ++i)
        if (i < n) c[i] = from_f<T>(x[i]);
}

}  // namespace acco
