// path.cuh — the non-GEMM kernels of the refinement path: embedding, demixing, Tanner-graph
// gathers (coefficient permutations, extrinsic pooling / attention, ordered per-slot
// accumulation), site statistics, reveal / remask selection and layout transforms.
//
// All of them are HBM-bound integer/byte or element-wise work: coalesced along the contiguous
// Q / D axis, no atomics (bitwise row symmetry), one thread per output element unless a
// per-bin selection needs a block.
#pragma once

#include "common.cuh"

namespace cider {

// ---- embed_grid (denoiser.cpp:71-84): Z[m] = E[X[m]], MASK -> row Q --------------------
template <typename T>
__global__ void embed_kernel(const int* __restrict__ X, const float* __restrict__ Etab, int Q, int D,
                             int64_t M, float* __restrict__ Zf, T* __restrict__ Zt) {
    int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= M * D) return;
    int64_t m = i / D;
    int t = int(i % D);
    int tok = X[m];
    int row = (tok < 0 || tok >= Q) ? Q : tok;
    float v = Etab[size_t(row) * D + t];
    if (Zf) Zf[i] = v;
    if (Zt) Zt[i] = from_f<T>(v);
}

// Vectorised BF16 variant (D % 8 == 0) on the bf16 copy of the table: 8 columns per thread, one 16-byte load and
// one 16-byte store.
__global__ void embed_bf16x8_kernel(const int* __restrict__ X, const bf16* __restrict__ Etab16, int Q, int D, int64_t M,
                                    bf16* __restrict__ Zt) {
    griddep_wait(); // (programmatic dependent launch) the grid X of the previous step
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int cpr = D / 8; // 16-byte chunks per row
    if (i >= M * cpr) return;
    const int64_t m = i / cpr;
    const int c = int(i - m * cpr);
    const int tok = __ldg(X + m);
    const int row = (tok < 0 || tok >= Q) ? Q : tok;
    *reinterpret_cast<uint4*>(Zt + m * D + c * 8) = __ldg(reinterpret_cast<const uint4*>(Etab16 + size_t(row) * D + c * 8));
}

// ---- demix_responsibilities x S (denoiser.cpp:103-122, 130) -------------------------------
// r_{k,l,a} = softmax over the K rows of lbar/tau; out = r * S_{l,a}. The normaliser is summed in
// 2^-52 fixed point (exact integer adds), which is order-independent: the same bitwise
// row-permutation invariance the reference gets by summing in descending order.
template <typename T>
__global__ void demix_kernel(const float* __restrict__ lbar, const float* __restrict__ S, int64_t n_slotrows,
                             int K, int Q, float tau, T* __restrict__ out) {
    int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n_slotrows * Q) return;
    int64_t s = i / Q;
    int a = int(i % Q);
    const float* x = lbar + size_t(s) * K * Q + a;
    float mx = x[0];
    for (int k = 1; k < K; ++k) mx = fmaxf(mx, x[size_t(k) * Q]);
    long long den = 0;
    for (int k = 0; k < K; ++k) {
        float e = expf((x[size_t(k) * Q] - mx) / tau);
        den += __double2ll_rn(double(e) * 4503599627370496.0);
    }
    float denf = float(double(den) * (1.0 / 4503599627370496.0));
    float sv = S[size_t(s) * Q + a];
    for (int k = 0; k < K; ++k) {
        float e = expf((x[size_t(k) * Q] - mx) / tau);
        out[(size_t(s) * K + k) * Q + a] = from_f<T>((e / denf) * sv);
    }
}

// ---- coefficient normalisation Pi_alpha W z per edge (denoiser.cpp:162-179, 192-195) -------
// Ae[(b,e,k)][c] = U[(b, slot_e, k)][perm_in[e][c]], perm_in[e][c] = alpha_e^-1 * c.
template <typename T>
__global__ void gather_perm_kernel(const T* __restrict__ U, const int* __restrict__ e_slot,
                                   const uint8_t* __restrict__ perm_in, int L, int E, int K, int Q,
                                   int64_t n_rows, T* __restrict__ Ae) {
    int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n_rows * Q) return;
    int64_t r = i / Q;
    int c = int(i % Q);
    int k = int(r % K);
    int64_t be = r / K;
    int e = int(be % E);
    int64_t b = be / E;
    int src = perm_in[size_t(e) * Q + c];
    Ae[i] = U[((b * L + e_slot[e]) * K + k) * Q + src];
}

// ---- extrinsic sum-pool Psi (denoiser.cpp:196-203) -----------------------------------------
// pooled[(b,e,k)] = sum over the other edges e2 of e's check, ascending, of N[(b,e2,k)].
template <typename Tin, typename T>
__global__ void pool_sum_kernel(const Tin* __restrict__ Nn, const int* __restrict__ e_check,
                                const int* __restrict__ check_ptr, int E, int K, int D, int64_t n_rows,
                                T* __restrict__ pooled) {
    int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n_rows * D) return;
    int64_t r = i / D;
    int t = int(i % D);
    int k = int(r % K);
    int64_t be = r / K;
    int e = int(be % E);
    int64_t b = be / E;
    int j = e_check[e];
    float s = 0.0f;
    for (int e2 = check_ptr[j]; e2 < check_ptr[j + 1]; ++e2) {
        if (e2 == e) continue;
        s += to_f(Nn[((b * E + e2) * K + k) * D + t]);
    }
    pooled[i] = from_f<T>(s);
}

// ---- extrinsic pooling attention Psi (config mode) ---------------------------
// One block per (bin, check, row). score_i,h = <q_h, key_i,h> / sqrt(dh); for target i the
// weights are the softmax of score_i2,h over the OTHER edges i2 of the check, and
// pooled_i = (d-1) * sum_i2 w_i2,h * N_i2 on head h's slice. q = 0 recovers the sum-pool.
constexpr int ATT_MAXD = 32, ATT_MAXH = 32;
template <typename Tin, typename T>
__global__ void pool_attn_kernel(const Tin* __restrict__ Nn, const float* __restrict__ keys,
                                 const float* __restrict__ query, const int* __restrict__ check_ptr,
                                 int P, int E, int K, int D, int heads, T* __restrict__ pooled) {
    __shared__ float part[1024];
    __shared__ float score[ATT_MAXD][ATT_MAXH];
    const int grp = blockIdx.x; // (b*P + j)*K + k
    const int k = grp % K;
    const int bj = grp / K;
    const int j = bj % P;
    const int64_t b = bj / P;
    const int e0 = check_ptr[j], d = check_ptr[j + 1] - e0;
    const int dh = D / heads;
    const float scale = rsqrtf(float(dh));
    for (int i = 0; i < d; ++i) {
        const float* kr = keys + ((b * E + e0 + i) * K + k) * D;
        for (int t = threadIdx.x; t < D; t += blockDim.x) part[t] = query[t] * kr[t];
        __syncthreads();
        for (int h = threadIdx.x; h < heads; h += blockDim.x) {
            float s = 0.0f;
            for (int t = h * dh; t < (h + 1) * dh; ++t) s += part[t];
            score[i][h] = s * scale;
        }
        __syncthreads();
    }
    for (int i = 0; i < d; ++i) {
        T* out = pooled + ((b * E + e0 + i) * K + k) * D;
        for (int t = threadIdx.x; t < D; t += blockDim.x) {
            const int h = t / dh;
            float mx = -INFINITY;
            for (int i2 = 0; i2 < d; ++i2)
                if (i2 != i) mx = fmaxf(mx, score[i2][h]);
            float den = 0.0f;
            for (int i2 = 0; i2 < d; ++i2)
                if (i2 != i) den += expf(score[i2][h] - mx);
            float s = 0.0f;
            for (int i2 = 0; i2 < d; ++i2) {
                if (i2 == i) continue;
                float w = float(d - 1) * expf(score[i2][h] - mx) / den;
                s += w * to_f(Nn[((b * E + e0 + i2) * K + k) * D + t]);
            }
            out[t] = from_f<T>(s);
        }
    }
}

// ---- warp-per-group Tanner kernels (the fast paths) -------------------------------------------
// A lane owns V consecutive channels of a row (V = C/32), so every row access is one 4..16-byte
// vector per lane: fully coalesced, no 64-bit index arithmetic per element.
template <typename T, int V> struct Vec;
template <> struct Vec<float, 2> { typedef float2 type; };
template <> struct Vec<float, 4> { typedef float4 type; };
template <> struct Vec<float, 8> { typedef struct { float4 a, b; } type; };
template <> struct Vec<bf16, 2> { typedef uint32_t type; };
template <> struct Vec<bf16, 4> { typedef uint2 type; };
template <> struct Vec<bf16, 8> { typedef uint4 type; };

template <typename T, int V>
__device__ __forceinline__ void load_v(const T* p, float* out) {
    if constexpr (sizeof(T) == 2) {
        if constexpr (V == 8) {
            uint4 u = *reinterpret_cast<const uint4*>(p);
            const bf16* h = reinterpret_cast<const bf16*>(&u);
#pragma unroll
            for (int i = 0; i < 8; ++i) out[i] = __bfloat162float(h[i]);
        } else if constexpr (V == 4) {
            uint2 u = *reinterpret_cast<const uint2*>(p);
            const bf16* h = reinterpret_cast<const bf16*>(&u);
#pragma unroll
            for (int i = 0; i < 4; ++i) out[i] = __bfloat162float(h[i]);
        } else {
            uint32_t u = *reinterpret_cast<const uint32_t*>(p);
            const bf16* h = reinterpret_cast<const bf16*>(&u);
#pragma unroll
            for (int i = 0; i < 2; ++i) out[i] = __bfloat162float(h[i]);
        }
    } else {
#pragma unroll
        for (int i = 0; i < V; i += 2) {
            float2 f = *reinterpret_cast<const float2*>(p + i);
            out[i] = f.x;
            out[i + 1] = f.y;
        }
    }
}
template <typename T, int V>
__device__ __forceinline__ void store_v(T* p, const float* v) {
    if constexpr (sizeof(T) == 2) {
        bf16 h[V];
#pragma unroll
        for (int i = 0; i < V; ++i) h[i] = __float2bfloat16_rn(v[i]);
        if constexpr (V == 8) *reinterpret_cast<uint4*>(p) = *reinterpret_cast<uint4*>(h);
        else if constexpr (V == 4) *reinterpret_cast<uint2*>(p) = *reinterpret_cast<uint2*>(h);
        else *reinterpret_cast<uint32_t*>(p) = *reinterpret_cast<uint32_t*>(h);
    } else {
#pragma unroll
        for (int i = 0; i < V; i += 2) *reinterpret_cast<float2*>(p + i) = make_float2(v[i], v[i + 1]);
    }
}

// Extrinsic pooling of one (bin, check, row) group per warp. heads == 0: sum-pool
// (denoiser.cpp:196-203); heads > 0: pooling attention with scores <u_h, n_i>, where
// u_h = Wk_h^T q_h (precomputed per layer) equals <q_h, (Wk n_i)_h> of DESIGN.md §2.
// Lane l owns channels [lV, lV+V) — all inside head l*heads/32 — so a reduce-scatter butterfly
// (log2(heads) halving exchanges, then a plain xor-reduce) leaves every lane holding exactly its
// own head's score: 9 shuffles per edge for 8 heads instead of 40. The max / normaliser run over
// the OTHER edges only, so pooled_i is bitwise independent of edge i (extrinsic).
constexpr int POOL_DMAX = 8;
template <int NH>
__device__ __forceinline__ float head_score(float* p, int lane) {
    // p[NH] per-lane partials; returns the full sum for head (lane * NH / 32)
    int width = NH;
    int xo = 16;
#pragma unroll
    for (int step = 0; (1 << step) < NH; ++step) {
        const int half = width / 2;
        const bool upper = (lane & xo) != 0;
#pragma unroll
        for (int j = 0; j < NH / 2; ++j) {
            if (j >= half) break;
            const float send = upper ? p[j] : p[j + half];
            const float keep = upper ? p[j + half] : p[j];
            p[j] = keep + __shfl_xor_sync(0xffffffffu, send, xo);
        }
        width = half;
        xo >>= 1;
    }
    float v = p[0];
    for (; xo; xo >>= 1) v += __shfl_xor_sync(0xffffffffu, v, xo);
    return v;
}

template <typename T, int V, int NH, int DMAX>
__global__ void __launch_bounds__(256, 2)
pool_warp_kernel(const T* __restrict__ Nn, const float* __restrict__ U, const int* __restrict__ check_ptr, int P, int E,
                 int K, int D, int64_t n_groups, T* __restrict__ pooled) {
    extern __shared__ float u_s[]; // NH x D score vectors
    if constexpr (NH > 0) {
        for (int i = threadIdx.x; i < NH * D; i += blockDim.x) u_s[i] = U[i];
        __syncthreads();
    }
    const int64_t g = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
    const int lane = threadIdx.x % 32;
    if (g >= n_groups) return;
    const int k = int(g % K);
    const int64_t bj = g / K;
    const int j = int(bj % P);
    const int64_t b = bj / P;
    const int e0 = check_ptr[j], d = check_ptr[j + 1] - e0;
    const int c0 = lane * V;
    // neighbour rows kept in their storage type (bf16 rows: V/2 registers each)
    typedef typename Vec<T, V>::type VT;
    VT raw[DMAX];
#pragma unroll
    for (int i = 0; i < DMAX; ++i)
        if (i < d) raw[i] = *reinterpret_cast<const VT*>(Nn + ((b * E + e0 + i) * K + k) * D + c0);
    auto unpack = [&](int i, float* f) { load_v<T, V>(reinterpret_cast<const T*>(&raw[i]), f); };
    float sc[DMAX];
    if constexpr (NH > 0) {
        const float scale = rsqrtf(float(D / NH));
#pragma unroll
        for (int i = 0; i < DMAX; ++i) {
            if (i >= d) break;
            float f[V];
            unpack(i, f);
            float p[NH];
#pragma unroll
            for (int h = 0; h < NH; ++h) {
                const float* uh = u_s + h * D + c0;
                float a = 0.0f;
#pragma unroll
                for (int v = 0; v < V; ++v) a = fmaf(uh[v], f[v], a);
                p[h] = a;
            }
            sc[i] = head_score<NH>(p, lane) * scale;
        }
    }
#pragma unroll 1
    for (int i = 0; i < d; ++i) {
        float out[V];
#pragma unroll
        for (int v = 0; v < V; ++v) out[v] = 0.0f;
        if constexpr (NH > 0) {
            float mx = -INFINITY, den = 0.0f;
#pragma unroll
            for (int i2 = 0; i2 < DMAX; ++i2)
                if (i2 < d && i2 != i) mx = fmaxf(mx, sc[i2]);
            float ex[DMAX];
#pragma unroll
            for (int i2 = 0; i2 < DMAX; ++i2) {
                ex[i2] = (i2 < d && i2 != i) ? __expf(sc[i2] - mx) : 0.0f;
                den += ex[i2];
            }
            const float fct = float(d - 1) / den;
#pragma unroll
            for (int i2 = 0; i2 < DMAX; ++i2) {
                if (i2 >= d || i2 == i) continue;
                const float w = ex[i2] * fct;
                float f[V];
                unpack(i2, f);
#pragma unroll
                for (int v = 0; v < V; ++v) out[v] = fmaf(w, f[v], out[v]);
            }
        } else {
#pragma unroll
            for (int i2 = 0; i2 < DMAX; ++i2) {
                if (i2 >= d || i2 == i) continue;
                float f[V];
                unpack(i2, f);
#pragma unroll
                for (int v = 0; v < V; ++v) out[v] += f[v];
            }
        }
        store_v<T, V>(pooled + ((b * E + e0 + i) * K + k) * D + c0, out);
    }
}


// Fixed-degree variant for check-regular codes (every check has exactly DEG edges — all BASELINE
// codes, degree 3L/P = 6): fully unrolled, neighbour rows unpacked once, no runtime degree tests
// (the generic kernel spent ~70% of its instructions on them — profiles/r1/pool_ncu_full.txt).
template <typename T, int V, int NH, int DEG>
__global__ void __launch_bounds__(256, 2)
pool_warp_fixed_kernel(const T* __restrict__ Nn, const float* __restrict__ U, const int* __restrict__ check_ptr, int P,
                       int E, int K, int D, int64_t n_groups, T* __restrict__ pooled) {
    extern __shared__ float u_s[]; // NH x D score vectors
    if constexpr (NH > 0) {
        for (int i = threadIdx.x; i < NH * D; i += blockDim.x) u_s[i] = U[i];
        __syncthreads();
    }
    const int64_t g = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
    const int lane = threadIdx.x % 32;
    if (g >= n_groups) return;
    const int k = int(g % K);
    const int64_t bj = g / K;
    const int j = int(bj % P);
    const int64_t b = bj / P;
    const int e0 = check_ptr[j];
    const int c0 = lane * V;
    float f[DEG][V];
#pragma unroll
    for (int i = 0; i < DEG; ++i) load_v<T, V>(Nn + ((b * E + e0 + i) * K + k) * D + c0, f[i]);
    float sc[DEG];
    if constexpr (NH > 0) {
        const float scale = rsqrtf(float(D / NH));
#pragma unroll
        for (int i = 0; i < DEG; ++i) {
            float p[NH];
#pragma unroll
            for (int h = 0; h < NH; ++h) {
                const float* uh = u_s + h * D + c0;
                float a = 0.0f;
#pragma unroll
                for (int v = 0; v < V; ++v) a = fmaf(uh[v], f[i][v], a);
                p[h] = a;
            }
            sc[i] = head_score<NH>(p, lane) * scale;
        }
    }
#pragma unroll
    for (int i = 0; i < DEG; ++i) {
        float out[V];
#pragma unroll
        for (int v = 0; v < V; ++v) out[v] = 0.0f;
        if constexpr (NH > 0) {
            float mx = -INFINITY;
#pragma unroll
            for (int i2 = 0; i2 < DEG; ++i2)
                if (i2 != i) mx = fmaxf(mx, sc[i2]);
            float ex[DEG], den = 0.0f;
#pragma unroll
            for (int i2 = 0; i2 < DEG; ++i2) {
                ex[i2] = i2 != i ? __expf(sc[i2] - mx) : 0.0f;
                den += ex[i2];
            }
            const float fct = float(DEG - 1) / den;
#pragma unroll
            for (int i2 = 0; i2 < DEG; ++i2) {
                if (i2 == i) continue;
                const float w = ex[i2] * fct;
#pragma unroll
                for (int v = 0; v < V; ++v) out[v] = fmaf(w, f[i2][v], out[v]);
            }
        } else {
#pragma unroll
            for (int i2 = 0; i2 < DEG; ++i2) {
                if (i2 == i) continue;
#pragma unroll
                for (int v = 0; v < V; ++v) out[v] += f[i2][v];
            }
        }
        store_v<T, V>(pooled + ((b * E + e0 + i) * K + k) * D + c0, out);
    }
}

// Streaming variant of pool_warp_fixed_kernel: the head scores come precomputed from a tensor-core
// GEMM (scores = N . [hi(u) | lo(u)]^T, EP_SCORES), so a warp only loads its check's DEG rows and
// its lane's head score per row, forms the DEG leave-one-out softmaxes and writes DEG rows.
template <typename T, int V, int NH, int DEG>
__global__ void __launch_bounds__(256)
pool_warp_scored_kernel(const T* __restrict__ Nn, const float* __restrict__ scores, const int* __restrict__ check_ptr,
                        int P, int E, int K, int D, int64_t n_groups, T* __restrict__ pooled) {
    const int64_t g = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
    const int lane = threadIdx.x % 32;
    if (g >= n_groups) return;
    const int k = int(g % K);
    const int64_t bj = g / K;
    const int j = int(bj % P);
    const int64_t b = bj / P;
    const int e0 = check_ptr[j];
    const int c0 = lane * V;
    const int h = lane * NH / 32; // the head this lane's columns belong to
    float f[DEG][V];
    float sc[DEG];
#pragma unroll
    for (int i = 0; i < DEG; ++i) {
        const int64_t r = (b * E + e0 + i) * K + k;
        load_v<T, V>(Nn + r * D + c0, f[i]);
        sc[i] = __ldg(scores + r * NH + h);
    }
#pragma unroll
    for (int i = 0; i < DEG; ++i) {
        float mx = -INFINITY;
#pragma unroll
        for (int i2 = 0; i2 < DEG; ++i2)
            if (i2 != i) mx = fmaxf(mx, sc[i2]);
        float ex[DEG], den = 0.0f;
#pragma unroll
        for (int i2 = 0; i2 < DEG; ++i2) {
            ex[i2] = i2 != i ? __expf(sc[i2] - mx) : 0.0f;
            den += ex[i2];
        }
        const float fct = float(DEG - 1) / den;
        float out[V];
#pragma unroll
        for (int v = 0; v < V; ++v) out[v] = 0.0f;
#pragma unroll
        for (int i2 = 0; i2 < DEG; ++i2) {
            if (i2 == i) continue;
            const float w = ex[i2] * fct;
#pragma unroll
            for (int v = 0; v < V; ++v) out[v] = fmaf(w, f[i2][v], out[v]);
        }
        store_v<T, V>(pooled + ((b * E + e0 + i) * K + k) * D + c0, out);
    }
}

// Pi_alpha gather, one edge row per warp, V = Q/32 symbols per lane.
template <typename T, int V>
__global__ void __launch_bounds__(256)
gather_perm_warp_kernel(const T* __restrict__ U, const int* __restrict__ e_slot, const uint8_t* __restrict__ perm_in,
                        int L, int E, int K, int Q, int64_t n_rows, T* __restrict__ Ae) {
    const int64_t r = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
    const int lane = threadIdx.x % 32;
    if (r >= n_rows) return;
    const int k = int(r % K);
    const int64_t be = r / K;
    const int e = int(be % E);
    const int64_t b = be / E;
    const T* src = U + ((b * L + e_slot[e]) * K + k) * Q;
    const uint8_t* pm = perm_in + size_t(e) * Q + lane * V;
    float v[V];
#pragma unroll
    for (int i = 0; i < V; ++i) v[i] = to_f(src[pm[i]]);
    store_v<T, V>(Ae + r * Q + lane * V, v);
}

// Ordered per-slot accumulation in symbol space, one site row per warp.
template <typename T, int V>
__global__ void __launch_bounds__(256)
scatter_perm_warp_kernel(const T* __restrict__ Mq, const int* __restrict__ slot_ptr, const int* __restrict__ slot_edge,
                         const uint8_t* __restrict__ perm_out, int L, int E, int K, int Q, int64_t n_rows,
                         T* __restrict__ accq) {
    const int64_t m = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
    const int lane = threadIdx.x % 32;
    if (m >= n_rows) return;
    const int k = int(m % K);
    const int64_t bl = m / K;
    const int l = int(bl % L);
    const int64_t b = bl / L;
    float s[V];
#pragma unroll
    for (int i = 0; i < V; ++i) s[i] = 0.0f;
    for (int p = slot_ptr[l]; p < slot_ptr[l + 1]; ++p) {
        const int e = slot_edge[p];
        const T* src = Mq + ((b * E + e) * K + k) * Q;
        const uint8_t* pm = perm_out + size_t(e) * Q + lane * V;
#pragma unroll
        for (int i = 0; i < V; ++i) s[i] += to_f(src[pm[i]]);
    }
    store_v<T, V>(accq + m * Q + lane * V, s);
}

// Demixing, one slot row (b, l) per block, one symbol per thread (see demix_kernel). The
// normaliser is summed in 2^-26 fixed point in 32-bit integers (K <= 32 terms <= 1 each, so no
// overflow): exact integer adds, hence order-independent — bitwise row-permutation invariant —
// without the fp64 conversions of the generic kernel (the demix ncu profile was issue-bound).
// BF16 mode uses the MUFU exp2; FP32 mode keeps expf.
template <typename T>
__global__ void __launch_bounds__(256)
demix_block_kernel(const float* __restrict__ lbar, const float* __restrict__ S, int K, int Q, float tau,
                   T* __restrict__ out) {
    const int64_t s = blockIdx.x;
    const float inv_tau = 1.0f / tau;
    for (int a = threadIdx.x; a < Q; a += blockDim.x) {
        const float* x = lbar + s * K * Q + a;
        float xv[32];
        float mx = -INFINITY;
#pragma unroll 8
        for (int k = 0; k < K; ++k) { xv[k] = __ldg(x + size_t(k) * Q); mx = fmaxf(mx, xv[k]); }
        uint32_t den = 0;
#pragma unroll 8
        for (int k = 0; k < K; ++k) {
            float e;
            if constexpr (sizeof(T) == 2) e = ex2_approx((xv[k] - mx) * (inv_tau * 1.4426950408889634f));
            else e = expf((xv[k] - mx) / tau);
            xv[k] = e;
            den += __float2uint_rn(e * 67108864.0f); // 2^26
        }
        const float rden = 1.0f / (float(den) * (1.0f / 67108864.0f));
        const float sv = __ldg(S + s * Q + a);
#pragma unroll 8
        for (int k = 0; k < K; ++k) out[(s * K + k) * Q + a] = from_f<T>((xv[k] * rden) * sv);
    }
}

// ---- de-normalisation + ordered scatter-add (denoiser.cpp:205-207), in symbol space --------
// accq[(b,l,k)][c] = sum over slot l's edges e, ascending check, of Mq[(b,e,k)][perm_out[e][c]],
// perm_out[e][c] = alpha_e * c. A gather in a fixed order: no atomics, bitwise deterministic.
template <typename Tin, typename T>
__global__ void scatter_perm_kernel(const Tin* __restrict__ Mq, const int* __restrict__ slot_ptr,
                                    const int* __restrict__ slot_edge, const uint8_t* __restrict__ perm_out,
                                    int L, int E, int K, int Q, int64_t n_rows, T* __restrict__ accq) {
    int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n_rows * Q) return;
    int64_t m = i / Q;
    int c = int(i % Q);
    int k = int(m % K);
    int64_t bl = m / K;
    int l = int(bl % L);
    int64_t b = bl / L;
    float s = 0.0f;
    for (int p = slot_ptr[l]; p < slot_ptr[l + 1]; ++p) {
        int e = slot_edge[p];
        s += to_f(Mq[((b * E + e) * K + k) * Q + perm_out[size_t(e) * Q + c]]);
    }
    accq[i] = from_f<T>(s);
}

// ---- site confidence + argmax (refine.cpp:61-78) over fp32 logits rows, one warp per row --
__global__ void row_stats_kernel(const float* __restrict__ logits, int64_t M, int Q, float tau,
                                 float* __restrict__ kappa, int* __restrict__ amax) {
    int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
    int lane = threadIdx.x % 32;
    if (w >= M) return;
    const float* x = logits + size_t(w) * Q;
    float bv = -INFINITY;
    int bi = 0x7fffffff;
    for (int a = lane; a < Q; a += 32) {
        float v = x[a];
        if (v > bv) { bv = v; bi = a; }
    }
    for (int o = 16; o; o >>= 1) {
        float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    float s = 0.0f;
    for (int a = lane; a < Q; a += 32) s += expf((x[a] - bv) / tau);
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
        kappa[w] = 1.0f / s;
        amax[w] = bi;
    }
}

// ---- reveal_step (refine.cpp:83-127), one block per bin ------------------------------------
// first: one site per slot, the masked row with the largest kappa (strict >, lowest row wins).
// else : reveal the (target - revealed) masked sites smallest in (kappa desc, row asc, slot asc)
//        via a bitonic sort of 64-bit keys (~bits(kappa), row, slot) — in dynamic shared memory
//        when the padded site count fits (REVEAL_SMEM_SITES), else in a per-bin global scratch
//        slice (gkeys + b * key_cap), so any K x L the reference accepts is handled.
// count (nullable): count[b * count_stride] = sites revealed by this step (RefineTrace::reveal_counts,
// refine.hpp:48-54); sites (nullable, zeroed by the caller): 1 for every site revealed by this step
// (RefineTrace::first_step_sites when called at t = 1).
constexpr int REVEAL_SMEM_SITES = 16384; // 128 KB of keys
__host__ __device__ inline int reveal_key_cap(int n) {
    int size = 1;
    while (size < n) size <<= 1;
    return size;
}
__global__ void __launch_bounds__(512)
reveal_kernel(int* __restrict__ X, const float* __restrict__ kappa, const int* __restrict__ amax, int L,
              int K, const int* __restrict__ init_masked, double rho, int first,
              int* __restrict__ count, int count_stride, uint8_t* __restrict__ sites,
              unsigned long long* __restrict__ gkeys) {
    griddep_wait(); // (programmatic dependent launch) kappa / argmax of the forward
    extern __shared__ unsigned long long skey[];
    __shared__ int red[32];
    const int b = blockIdx.x;
    const int n = L * K;
    int* x = X + size_t(b) * n;
    const float* kp = kappa + size_t(b) * n;
    const int* am = amax + size_t(b) * n;
    uint8_t* st = sites ? sites + size_t(b) * n : nullptr;
    int before = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) before += x[i] == -1;
    for (int o = 16; o; o >>= 1) before += __shfl_xor_sync(0xffffffffu, before, o);
    if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = before;
    __syncthreads();
    if (threadIdx.x == 0) {
        int s = 0;
        for (int w = 0; w < int(blockDim.x / 32); ++w) s += red[w];
        red[0] = s;
    }
    __syncthreads();
    const int masked = red[0];
    __syncthreads();
    if (first) {
        int cnt = 0;
        for (int l = threadIdx.x; l < L; l += blockDim.x) {
            int br = -1;
            float bk = 0.0f;
            for (int k = 0; k < K; ++k) {
                int i = l * K + k;
                if (x[i] != -1) continue;
                if (br < 0 || kp[i] > bk) { br = k; bk = kp[i]; }
            }
            if (br >= 0) {
                x[l * K + br] = am[l * K + br];
                if (st) st[l * K + br] = 1;
                ++cnt;
            }
        }
        if (count) {
            for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
            __syncthreads();
            if (threadIdx.x % 32 == 0) red[threadIdx.x / 32] = cnt;
            __syncthreads();
            if (threadIdx.x == 0) {
                int s = 0;
                for (int w = 0; w < int(blockDim.x / 32); ++w) s += red[w];
                count[size_t(b) * count_stride] = s;
            }
        }
        return;
    }
    const int base = n - init_masked[b];
    const int target = base + int(llround(rho * double(init_masked[b])));
    const int need = target - (n - masked); // <= masked: target <= n
    if (count && threadIdx.x == 0) count[size_t(b) * count_stride] = need > 0 ? need : 0;
    if (need <= 0) return;
    const int size = reveal_key_cap(n);
    unsigned long long* key = size <= REVEAL_SMEM_SITES ? skey : gkeys + size_t(b) * size;
    for (int i = threadIdx.x; i < size; i += blockDim.x) {
        unsigned long long kk = ~0ull;
        if (i < n && x[i] == -1) {
            int l = i / K, k = i % K;
            unsigned int bits = __float_as_uint(kp[i]);
            kk = (static_cast<unsigned long long>(~bits) << 32) | (static_cast<unsigned long long>(k) << 16) |
                 static_cast<unsigned long long>(l);
        }
        key[i] = kk;
    }
    __syncthreads();
    for (int len = 2; len <= size; len <<= 1)
        for (int j = len >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < size; i += blockDim.x) {
                int p = i ^ j;
                if (p > i) {
                    bool up = (i & len) == 0;
                    unsigned long long a = key[i], c = key[p];
                    if ((a > c) == up) { key[i] = c; key[p] = a; }
                }
            }
            __syncthreads();
        }
    for (int r = threadIdx.x; r < need; r += blockDim.x) {
        unsigned long long kk = key[r];
        if (kk == ~0ull) continue;
        int k = int((kk >> 16) & 0xffff), l = int(kk & 0xffff);
        x[l * K + k] = am[l * K + k];
        if (st) st[l * K + k] = 1;
    }
}

// ---- end of a pass (refine.cpp:175-192) ------------------------------------------------------
// residual masks -> the last step's argmax
__global__ void force_residual_kernel(int* __restrict__ X, const int* __restrict__ amax, int64_t n) {
    griddep_wait();
    int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n && X[i] == -1) X[i] = amax[i];
}
// updatable rows take the final (gamma = 0) pass's argmax; the rest stay bit-identical
__global__ void finalize_kernel(int* __restrict__ X, const int* __restrict__ amax,
                                const uint32_t* __restrict__ upd_mask, int K, int64_t n_bins_x_n, int n) {
    griddep_wait();
    int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n_bins_x_n) return;
    int64_t b = i / n;
    int k = int(i % K);
    if ((upd_mask[b] >> k) & 1u) X[i] = amax[i];
}

// ---- MaxProbScorer (refine.cpp:207-225) + remask selection, one block per bin --------------
// mode 2 (rank): the k_low rows of lowest confidence, ties -> lower row.
// mode 1 (threshold): rows with confidence < thr (refine.cpp:245-252).
// Selected rows are re-masked; upd_mask / init_masked / n_low describe the coming pass.
__global__ void remask_select_kernel(int* __restrict__ X, const float* __restrict__ kappa1, int L, int K,
                                     int mode, int k_low, double thr, uint32_t* __restrict__ upd_mask,
                                     int* __restrict__ init_masked, int* __restrict__ n_low_out,
                                     float* __restrict__ conf_out) {
    __shared__ double conf[32];
    __shared__ uint32_t sel;
    const int b = blockIdx.x;
    const int n = L * K;
    const float* kp = kappa1 + size_t(b) * n;
    if (threadIdx.x < K) {
        double s = 0.0;
        for (int l = 0; l < L; ++l) s += double(kp[l * K + threadIdx.x]);
        conf[threadIdx.x] = s / L;
        if (conf_out) conf_out[size_t(b) * K + threadIdx.x] = float(conf[threadIdx.x]);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t m = 0;
        if (mode == 1) {
            for (int k = 0; k < K; ++k)
                if (conf[k] < thr) m |= 1u << k;
        } else {
            for (int r = 0; r < k_low; ++r) { // selection by repeated minimum, stable in k
                int best = -1;
                for (int k = 0; k < K; ++k)
                    if (!((m >> k) & 1u) && (best < 0 || conf[k] < conf[best])) best = k;
                m |= 1u << best;
            }
        }
        sel = m;
        upd_mask[b] = m;
        int nl = __popc(m);
        init_masked[b] = nl * L;
        if (n_low_out) n_low_out[b] = nl;
    }
    __syncthreads();
    const uint32_t m = sel;
    int* x = X + size_t(b) * n;
    for (int i = threadIdx.x; i < n; i += blockDim.x)
        if ((m >> (i % K)) & 1u) x[i] = -1;
}

// ---- layout transforms between the reference's K x L views and the internal (l, k) order ---
__global__ void grid_to_internal_kernel(const int* __restrict__ ref, int* __restrict__ in, int L, int K,
                                        int64_t total) {
    int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= total) return;
    int64_t b = i / (int64_t(L) * K);
    int r = int(i % (int64_t(L) * K));
    int l = r / K, k = r % K;
    in[i] = ref[b * L * K + int64_t(k) * L + l];
}
__global__ void grid_to_ref_kernel(const int* __restrict__ in, int* __restrict__ ref, int L, int K,
                                   int64_t total) {
    int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= total) return;
    int64_t b = i / (int64_t(L) * K);
    int r = int(i % (int64_t(L) * K));
    int l = r / K, k = r % K;
    ref[b * L * K + int64_t(k) * L + l] = in[i];
}
// rows of C values: internal (b,l,k) -> reference (b,k,l), optional leading layer index
__global__ void rows_to_ref_kernel(const float* __restrict__ in, float* __restrict__ ref, int L, int K, int C,
                                   int64_t total, int64_t ref_bin_stride, int64_t ref_offset) {
    int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= total) return;
    int c = int(i % C);
    int64_t row = i / C;
    int64_t b = row / (int64_t(L) * K);
    int r = int(row % (int64_t(L) * K));
    int l = r / K, k = r % K;
    ref[b * ref_bin_stride + ref_offset + (int64_t(k) * L + l) * C + c] = in[i];
}

__global__ void fill_i32_kernel(int* __restrict__ p, int v, int64_t n) {
    int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}
__global__ void fill_u32_kernel(uint32_t* __restrict__ p, uint32_t v, int64_t n) {
    int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}
__global__ void f32_to_bf16_kernel(const float* __restrict__ in, bf16* __restrict__ out, int64_t n) {
    int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) out[i] = __float2bfloat16_rn(in[i]);
}
// decoded grids as one byte per symbol (Q <= 256) for the final gather
__global__ void pack_u8_kernel(const int* __restrict__ in, uint8_t* __restrict__ out, int64_t n) {
    int64_t i = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
    if (i + 3 < n) {
        const int4 v = *reinterpret_cast<const int4*>(in + i);
        *reinterpret_cast<uchar4*>(out + i) = make_uchar4(uint8_t(v.x), uint8_t(v.y), uint8_t(v.z), uint8_t(v.w));
    } else {
        for (; i < n; ++i) out[i] = uint8_t(in[i]);
    }
}
__global__ void flush_kernel(int4* __restrict__ p, int64_t n, int v) {
    int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) p[i] = make_int4(v, v, v, v);
}

} // namespace cider
