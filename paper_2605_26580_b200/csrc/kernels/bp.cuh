// bp.cuh — batched GF(Q) FFT-BP decoder (reference bp.cpp:11-79, 222-368):
// flooding-schedule joint BP with WHT-domain check updates and successive-cancellation (SIC) over
// the K users, for many bins at once. One bin's state lives in HBM ([bin][edge][Q] fp64 messages);
// bins that converged (early exit) are frozen by a per-bin flag, so every bin follows exactly the
// reference's per-decode control flow.
//
// Precision: the reference keeps the spectral pipeline of the check update in long double because
// the transform reconstructs small probabilities by cancellation (bp.cpp:189-193). The GPU has no
// 80-bit type, so the WHTs, prefix/suffix spectral products and the inverse transform run in
// double-double (~106-bit significand, more than long double's 64); everything else is fp64 in the
// reference's operation order (products over edges in slot/check order, normalisation sums in
// symbol order, ties to the lowest symbol).
#pragma once

#include "common.cuh"

namespace cider {
namespace bp {

struct dd {
    double hi, lo;
};
__device__ __forceinline__ dd quick_two_sum(double a, double b) {
    const double s = a + b;
    return {s, b - (s - a)};
}
__device__ __forceinline__ dd two_sum(double a, double b) {
    const double s = a + b;
    const double bb = s - a;
    return {s, (a - (s - bb)) + (b - bb)};
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {
    dd s = two_sum(a.hi, b.hi);
    const dd t = two_sum(a.lo, b.lo);
    s.lo += t.hi;
    s = quick_two_sum(s.hi, s.lo);
    s.lo += t.lo;
    return quick_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_neg(dd a) { return {-a.hi, -a.lo}; }
__device__ __forceinline__ dd dd_mul(dd a, dd b) {
    const double p = a.hi * b.hi;
    double e = fma(a.hi, b.hi, -p);
    e = fma(a.hi, b.lo, e);
    e = fma(a.lo, b.hi, e);
    return quick_two_sum(p, e);
}

// WHT of one row held by LW lanes of a warp (LW = min(32, Q / 4): 4-8 symbols per lane; 32 / LW rows
// per warp): lane-in-row r owns symbols r + LW j. Butterfly stages with len >= LW pair registers of
// the same lane, stages with len < LW pair lanes through warp shuffles — no shared memory, no block
// barrier. Each pair (u = y[a], v = y[a + len], bit len of a clear) becomes (u + v, u - v) with the same
// dd operations as an SMEM butterfly, so the result is bit-identical to one.
constexpr int WHT_MAXE = 8; // symbols per lane (Q <= 256)
__host__ __device__ inline int wht_lanes(int Q) { return Q >= 128 ? 32 : (Q >= 4 ? Q / 4 : 1); }
__device__ __forceinline__ dd shfl_dd(dd x, int m) {
    return {__shfl_xor_sync(0xffffffffu, x.hi, m), __shfl_xor_sync(0xffffffffu, x.lo, m)};
}
__device__ __forceinline__ void wht_warp_dd(dd (&r)[WHT_MAXE], int Q, int LW, int lr) {
    const int E = Q / LW;
    for (int len = 1; len < LW; len <<= 1) {
#pragma unroll
        for (int j = 0; j < WHT_MAXE; ++j) {
            if (j >= E) break;
            const dd p = shfl_dd(r[j], len);
            r[j] = (lr & len) ? dd_add(p, dd_neg(r[j])) : dd_add(r[j], p);
        }
    }
    for (int h = 1; h < E; h <<= 1) // len = LW h
#pragma unroll
        for (int j = 0; j < WHT_MAXE; ++j) {
            if (j >= E || (j & h)) continue;
            const dd u = r[j], v = r[j + h];
            r[j] = dd_add(u, v);
            r[j + h] = dd_add(u, dd_neg(v));
        }
}

// normalize_or_uniform (bp.cpp:11-19): sequential sum in symbol order, then x *= 1/s.
__device__ __forceinline__ void normalize_row_seq(double* v, int Q) {
    double s = 0.0;
    for (int a = 0; a < Q; ++a) s += v[a];
    if (s > 0.0) {
        const double inv = 1.0 / s;
        for (int a = 0; a < Q; ++a) v[a] *= inv;
    } else {
        for (int a = 0; a < Q; ++a) v[a] = 1.0 / Q;
    }
}

// slot_beliefs (bp.cpp:61-77): per (bin, slot) softmax of the (residual) evidence row.
__global__ void slot_beliefs_kernel(const double* __restrict__ S, int64_t rows, int Q, double* __restrict__ lambda) {
    const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const double* row = S + r * Q;
    double* out = lambda + r * Q;
    double hi = row[0];
    for (int a = 1; a < Q; ++a) hi = fmax(hi, row[a]);
    double sum = 0.0;
    for (int a = 0; a < Q; ++a) {
        out[a] = exp(row[a] - hi);
        sum += out[a];
    }
    const double inv = 1.0 / sum;
    for (int a = 0; a < Q; ++a) out[a] *= inv;
}

// v2c[e] = lambda[slot(e)], c2v[e] = 1/Q; state flags of every bin reset (bp.cpp:285-289)
__global__ void bp_init_kernel(const double* __restrict__ lambda, const int* __restrict__ e_slot, int L, int E, int Q,
                               int64_t n, double* __restrict__ v2c, double* __restrict__ c2v) {
    const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return; // n = bins * E * Q
    const int a = int(i % Q);
    const int64_t be = i / Q;
    const int e = int(be % E);
    const int64_t b = be / E;
    v2c[i] = lambda[(b * L + e_slot[e]) * Q + a];
    c2v[i] = 1.0 / Q;
}

// update_check_wht (bp.cpp:222-269) for every (bin, check) of the active bins: one CTA each, warp i
// on edge i's row for the transforms (registers + shuffles), all threads on the prefix / suffix
// spectral products (thread per symbol, over the rows in SMEM).
// SMEM: y [d][Q] and spec [d][Q] in double-double.
__global__ void bp_check_kernel(const double* __restrict__ v2c, const int* __restrict__ check_ptr,
                                const int* __restrict__ e_coef, const uint8_t* __restrict__ mul, int P, int E, int Q,
                                const int* __restrict__ active, double* __restrict__ c2v) {
    const int64_t bj = blockIdx.x;
    const int j = int(bj % P);
    const int64_t b = bj / P;
    if (!active[b]) return;
    extern __shared__ dd sm_dd[];
    const int e0 = check_ptr[j], d = check_ptr[j + 1] - e0;
    dd* y = sm_dd;                   // d x Q permuted spectra
    dd* sp = sm_dd + size_t(d) * Q;  // d x Q extrinsic spectra
    const double* in = v2c + (b * E + e0) * Q;
    const int LW = wht_lanes(Q), RPW = 32 / LW, EL = Q / LW;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
    const int lr = lane % LW;
    for (int i0 = warp * RPW; i0 < d; i0 += nw * RPW) { // scatter_by (y[alpha a] = msg[a]), then the forward transform
        const int i = i0 + lane / LW;
        const bool on = i < d;
        if (on) {
            const uint8_t* mrow = mul + e_coef[e0 + i] * Q;
            for (int a = lr; a < Q; a += LW) y[size_t(i) * Q + mrow[a]] = dd{in[size_t(i) * Q + a], 0.0};
        }
        __syncwarp();
        dd r[WHT_MAXE];
#pragma unroll
        for (int t = 0; t < WHT_MAXE; ++t) r[t] = (t < EL && on) ? y[size_t(i) * Q + lr + LW * t] : dd{0.0, 0.0};
        wht_warp_dd(r, Q, LW, lr);
#pragma unroll
        for (int t = 0; t < WHT_MAXE; ++t)
            if (t < EL && on) y[size_t(i) * Q + lr + LW * t] = r[t];
    }
    __syncthreads();
    for (int a = threadIdx.x; a < Q; a += blockDim.x) {
        // prefix left to right, suffix right to left, spec_i = pre_i * suf_{i+1} (bp.cpp:240-259)
        dd pre = {1.0, 0.0};
        for (int i = 0; i < d; ++i) {
            sp[size_t(i) * Q + a] = pre;
            pre = dd_mul(pre, y[size_t(i) * Q + a]);
        }
        dd suf = {1.0, 0.0};
        for (int i = d - 1; i >= 0; --i) {
            sp[size_t(i) * Q + a] = dd_mul(sp[size_t(i) * Q + a], suf);
            suf = dd_mul(suf, y[size_t(i) * Q + a]);
        }
    }
    __syncthreads();
    // inverse transform per row, then out[a] = max(double(spec[map[a]] / Q), 0) staged over the row's
    // dead y slot, normalize_or_uniform per edge (sequential sum by lane 0), a coalesced write
    double* out = c2v + (b * E + e0) * Q;
    const double scale = 1.0 / Q;
    for (int i0 = warp * RPW; i0 < d; i0 += nw * RPW) {
        const int i = i0 + lane / LW;
        const bool on = i < d;
        dd r[WHT_MAXE];
#pragma unroll
        for (int t = 0; t < WHT_MAXE; ++t) r[t] = (t < EL && on) ? sp[size_t(i) * Q + lr + LW * t] : dd{0.0, 0.0};
        wht_warp_dd(r, Q, LW, lr);
#pragma unroll
        for (int t = 0; t < WHT_MAXE; ++t)
            if (t < EL && on) sp[size_t(i) * Q + lr + LW * t] = r[t];
        __syncwarp();
        double* xo = reinterpret_cast<double*>(y + size_t(on ? i : 0) * Q);
        if (on) {
            const uint8_t* mrow = mul + e_coef[e0 + i] * Q;
            for (int a = lr; a < Q; a += LW) {
                const dd v = sp[size_t(i) * Q + mrow[a]];
                xo[a] = fmax((v.hi + v.lo) * scale, 0.0); // scale is a power of two: exact
            }
        }
        __syncwarp();
        double t = 0.0;
        if (on && lr == 0)
            for (int a = 0; a < Q; ++a) t += xo[a];
        t = __shfl_sync(0xffffffffu, t, lane - lr); // from the row's first lane
        const double iv = t > 0.0 ? 1.0 / t : -1.0;
        if (on)
            for (int a = lr; a < Q; a += LW) out[size_t(i) * Q + a] = iv < 0.0 ? 1.0 / Q : xo[a] * iv;
    }
}

// Sequential (symbol-order) normaliser of a row a warp holds in SMEM: lane 0 sums, all lanes scale
// their own symbols (normalize_or_uniform, bp.cpp:11-19, in the reference's summation order).
__device__ __forceinline__ double warp_row_inv(const double* row, int Q, int lane) {
    double s = 0.0;
    if (lane == 0)
        for (int a = 0; a < Q; ++a) s += row[a];
    s = __shfl_sync(0xffffffffu, s, 0);
    return s > 0.0 ? 1.0 / s : -1.0; // -1: uniform
}

// Beliefs and hard decision (bp.cpp:306-313): b = lambda * prod over slot edges (in slot order) of
// c2v, normalised, argmax with ties to the lowest symbol. One warp per (bin, slot), lanes over symbols.
constexpr int BP_QMAX = 256;
__global__ void __launch_bounds__(256) bp_belief_kernel(const double* __restrict__ lambda, const double* __restrict__ c2v,
                                 const int* __restrict__ slot_ptr, const int* __restrict__ slot_edge, int L, int E,
                                 int Q, const int* __restrict__ active, int64_t rows, double* __restrict__ beliefs,
                                 int* __restrict__ hard) {
    __shared__ double rowbuf[8][BP_QMAX];
    const int wib = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int64_t r = int64_t(blockIdx.x) * 8 + wib;
    if (r >= rows) return;
    const int l = int(r % L);
    const int64_t b = r / L;
    if (!active[b]) return;
    double* sb = rowbuf[wib];
    const double* lam = lambda + r * Q;
    const int p0 = slot_ptr[l], p1 = slot_ptr[l + 1];
    for (int a = lane; a < Q; a += 32) {
        double v = lam[a];
        for (int p = p0; p < p1; ++p) v *= c2v[(b * E + slot_edge[p]) * Q + a];
        sb[a] = v;
    }
    __syncwarp();
    const double inv = warp_row_inv(sb, Q, lane);
    double* bl = beliefs + r * Q;
    double best = -1.0;
    int bi = 0x7fffffff;
    for (int a = lane; a < Q; a += 32) {
        const double v = inv < 0.0 ? 1.0 / Q : sb[a] * inv;
        bl[a] = v;
        if (v > best) { best = v; bi = a; } // ascending a within the lane: first maximum kept
    }
    for (int o = 16; o; o >>= 1) { // lowest index among equal maxima
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    if (lane == 0) hard[r] = bi;
}

// Syndrome test and the per-bin control flow of one iteration (bp.cpp:315-318): one warp per bin.
__global__ void bp_syndrome_kernel(const int* __restrict__ hard, const int* __restrict__ check_ptr,
                                   const int* __restrict__ e_slot, const int* __restrict__ e_coef,
                                   const uint8_t* __restrict__ mul, int P, int L, int Q, int iter, int max_iters,
                                   int early_exit, int64_t bins, int* __restrict__ active, int* __restrict__ converged,
                                   int* __restrict__ iters, int* __restrict__ n_active) {
    const int64_t b = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
    const int lane = threadIdx.x % 32;
    if (b >= bins || !active[b]) return;
    bool ok = true;
    for (int j = lane; j < P; j += 32) {
        int s = 0;
        for (int p = check_ptr[j]; p < check_ptr[j + 1]; ++p) s ^= mul[e_coef[p] * Q + hard[b * L + e_slot[p]]];
        ok = ok && s == 0;
    }
    ok = __all_sync(0xffffffffu, ok);
    if (lane == 0) {
        converged[b] = ok ? 1 : 0;
        iters[b] = iter;
        if ((ok && early_exit) || iter == max_iters) active[b] = 0;
        else atomicAdd(n_active, 1);
    }
}

// Variable update (bp.cpp:320-344) for the bins still active: extrinsic prefix/suffix products over
// the slot's edges, floored at message_floor, normalised. One warp per (bin, slot), lanes over symbols.
__global__ void __launch_bounds__(256) bp_var_kernel(const double* __restrict__ lambda, const double* __restrict__ c2v,
                              const int* __restrict__ slot_ptr, const int* __restrict__ slot_edge, int L, int E, int Q,
                              double floor_v, const int* __restrict__ active, int64_t rows, double* __restrict__ v2c) {
    __shared__ double rowbuf[8][BP_QMAX];
    const int wib = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int64_t r = int64_t(blockIdx.x) * 8 + wib;
    if (r >= rows) return;
    const int l = int(r % L);
    const int64_t b = r / L;
    if (!active[b]) return;
    double* sb = rowbuf[wib];
    const int p0 = slot_ptr[l], d = slot_ptr[l + 1] - p0;
    const double* lam = lambda + r * Q;
    for (int i = 0; i < d; ++i) {
        double* out = v2c + (b * E + slot_edge[p0 + i]) * Q;
        for (int a = lane; a < Q; a += 32) {
            double pre = lam[a]; // pre[i] = lambda * c2v[e_0] ... c2v[e_{i-1}]
            for (int t = 0; t < i; ++t) pre *= c2v[(b * E + slot_edge[p0 + t]) * Q + a];
            double suf = 1.0;    // suf[i+1] = c2v[e_{d-1}] ... c2v[e_{i+1}], built right to left
            for (int t = d - 1; t > i; --t) suf *= c2v[(b * E + slot_edge[p0 + t]) * Q + a];
            const double x = pre * suf;
            sb[a] = x < floor_v ? floor_v : x;
        }
        __syncwarp();
        const double inv = warp_row_inv(sb, Q, lane);
        for (int a = lane; a < Q; a += 32) out[a] = inv < 0.0 ? 1.0 / Q : sb[a] * inv;
        __syncwarp();
    }
}

// SIC cancellation (bp.cpp:361-364): residual[l][hard[l]] = cancel_value for every slot.
__global__ void sic_cancel_kernel(const int* __restrict__ hard, int L, int Q, double cancel_value, int64_t rows,
                                  double* __restrict__ residual, int* __restrict__ grid, int K, int stage) {
    const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const int l = int(r % L);
    const int64_t b = r / L;
    const int h = hard[r];
    grid[(b * K + stage) * L + l] = h;
    residual[r * Q + h] = cancel_value;
}

} // namespace bp
} // namespace cider
