// common.cuh — shared device helpers and the GEMM epilogue contract.
//
// Internal HBM layout: every per-site tensor is [bin][slot][row] x C
// ("site row" m = (b*L + l)*K + k) and every per-edge tensor is [bin][edge][row] x C
// ("edge row" r = (b*E + e)*K + k): the K rows of one slot / edge are adjacent, which keeps the
// demixing softmax over rows and all Tanner gathers inside one small contiguous group.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace cider {

// Programmatic dependent launch (kernels launched with programmatic stream serialization, engine.cu
// launch_pdl): griddep_wait() blocks until the preceding grid has completed and its writes are
// visible — every such kernel calls it before reading anything an earlier kernel produced; a
// persistent kernel (all CTAs resident) then lets the next grid start launching (its prologue
// overlaps this grid's tail) with griddep_launch_dependents().
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }


typedef __nv_bfloat16 bf16;

__device__ __forceinline__ float to_f(float v) { return v; }
__device__ __forceinline__ float to_f(bf16 v) { return __bfloat162float(v); }
template <typename T> __device__ __forceinline__ T from_f(float v);
template <> __device__ __forceinline__ float from_f<float>(float v) { return v; }
template <> __device__ __forceinline__ bf16 from_f<bf16>(float v) { return __float2bfloat16_rn(v); }

// erf-form GELU and logistic sigmoid, as the reference (denoiser.cpp:13-15)
__device__ __forceinline__ float gelu_f(float x) { return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f)); }
// 2^x on the MUFU unit (BF16-mode softmaxes; FP32 mode keeps expf)
__device__ __forceinline__ float ex2_approx(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float sigmoid_f(float x) { return 1.0f / (1.0f + expf(-x)); }

enum EpKind : int {
    EP_STORE = 0,  // out = acc (+ bias)
    EP_GELU = 1,   // out = gelu(acc + bias)
    EP_GATE = 2,   // g = sigmoid(acc + bias); out = g*z + (1-g)*e        (Module A gate, denoiser.cpp:156)
    EP_RESID = 3,  // out = z + acc + bias                                (Module B fusion, denoiser.cpp:224)
    EP_LBAR = 4,   // out = acc + beta * S[bin, slot, n]                  (intermediate logits, denoiser.cpp:96)
    EP_LOGITS = 5, // row statistics of final logits: kappa(tau), argmax  (refine.cpp:61-78); optional f32 logits
    EP_SCORES = 6, // attention head scores: out[m][h] = acc[h] + acc[16 + h], h < K (hi + lo bf16 split of u_h)
    EP_DEMIX = 7,  // Module A demix fused on the intermediate logits x = acc + beta S: per (bin, slot) group of K
                   // rows, out = softmax_k(x / tau) * S, normaliser in 2^-26 fixed point (= demix_block_kernel)
};

// Everything an epilogue may need. Pointers the kind does not use are ignored.
struct Epi {
    int kind;
    int M, N;
    const float* bias;   // [N]
    float* out_f;        // fp32 output [M x ldo]
    void* out_t;         // activation-typed output [M x ldo] (bf16 in BF16 mode, float in FP32 mode)
    int ldo;
    const float* z;      // fp32 [M x ldz]: gate's z, residual's z
    const float* e;      // fp32 [M x ldz]: gate's e
    int ldz;
    const bf16* zb;      // BF16 mode: bf16 z / e [M x ldz] (fused-MLP final epilogue)
    const bf16* eb;
    const float* S;      // evidence [bins x L x Q]
    int L, K;
    float beta;
    float inv_tau;       // EP_LOGITS
    float* kappa;        // EP_LOGITS: [M]
    int* amax;           // EP_LOGITS: [M]
};

// Evidence index of site row m for column n (EP_LBAR): m = (b*L + l)*K + k -> S[(b*L + l)*N + n].
__device__ __forceinline__ size_t lbar_s_index(const Epi& ep, int m, int n) {
    return size_t(m / ep.K) * ep.N + n;
}

// Applies an element-wise epilogue to `cnt` consecutive columns [n0, n0+cnt) of row m.
template <typename T>
__device__ __forceinline__ void epi_apply(const Epi& ep, int m, int n0, float* v, int cnt) {
    if (ep.bias)
        for (int i = 0; i < cnt; ++i) v[i] += ep.bias[n0 + i];
    switch (ep.kind) {
        case EP_GELU:
            for (int i = 0; i < cnt; ++i) v[i] = gelu_f(v[i]);
            break;
        case EP_GATE:
            for (int i = 0; i < cnt; ++i) {
                float g = sigmoid_f(v[i]);
                float zz = ep.z[size_t(m) * ep.ldz + n0 + i];
                float ee = ep.e[size_t(m) * ep.ldz + n0 + i];
                v[i] = g * zz + (1.0f - g) * ee;
            }
            break;
        case EP_RESID:
            for (int i = 0; i < cnt; ++i) v[i] += ep.z[size_t(m) * ep.ldz + n0 + i];
            break;
        case EP_LBAR: {
            const float* s = ep.S + lbar_s_index(ep, m, n0);
            for (int i = 0; i < cnt; ++i) v[i] += ep.beta * s[i];
            break;
        }
        default:
            break;
    }
    if (ep.out_f) {
        float* o = ep.out_f + size_t(m) * ep.ldo + n0;
        for (int i = 0; i < cnt; ++i) o[i] = v[i];
    }
    if (ep.out_t) {
        T* o = reinterpret_cast<T*>(ep.out_t) + size_t(m) * ep.ldo + n0;
        for (int i = 0; i < cnt; ++i) o[i] = from_f<T>(v[i]);
    }
}

} // namespace cider
