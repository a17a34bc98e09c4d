// wht.cuh — batched GF(Q) check-node update in the Walsh–Hadamard domain (
// reference: update_check_wht / check_update_wht, bp.cpp:128-149, 195-269).
//
// For every check (one CTA per check; bins x checks in one launch) and every edge i of it:
//   y_i   = WHT( scatter(v2c_i by coefficient) )          y_i[alpha_i * a] = v2c_i[a]
//   spec_i = prod_{j<i} y_j  *  prod_{j>i} y_j            (prefix / suffix products, extrinsic)
//   c2v_i[a] = max( WHT(spec_i)[alpha_i * a] / Q, 0 ),  normalised (uniform if all mass vanished)
// Thread a owns spectral index a of every edge for the prefix/suffix products (register loops over
// the rows in SMEM); the transforms run one row per warp in registers with warp-shuffle butterflies
// for the strides below 32. fp64 throughout (the reference keeps the
// spectra in long double; the GPU has no 80-bit type — parity tolerance in tests/test_gpu.py).
#pragma once

#include "common.cuh"

namespace cider {

constexpr int WHT_MAXD = 32;

// One row per LW lanes (LW = min(32, Q / 4), 4-8 symbols per lane, 32 / LW rows per warp) in
// registers: butterflies with len >= LW inside a lane, len < LW across lanes by warp shuffles:
// (u, v) -> (u + v, u - v) in fp64, the same operations as an SMEM butterfly, without block barriers.
constexpr int WHT_MAXE = 8; // symbols per lane (Q <= 256)
__host__ __device__ inline int wht_lanes(int Q) { return Q >= 128 ? 32 : (Q >= 4 ? Q / 4 : 1); }
__device__ __forceinline__ void wht_warp(double (&r)[WHT_MAXE], int Q, int LW, int lr) {
    const int E = Q / LW;
    for (int len = 1; len < LW; len <<= 1) {
#pragma unroll
        for (int j = 0; j < WHT_MAXE; ++j) {
            if (j >= E) break;
            const double p = __shfl_xor_sync(0xffffffffu, r[j], len);
            r[j] = (lr & len) ? p - r[j] : r[j] + p;
        }
    }
    for (int h = 1; h < E; h <<= 1)
#pragma unroll
        for (int j = 0; j < WHT_MAXE; ++j) {
            if (j >= E || (j & h)) continue;
            const double u = r[j], v = r[j + h];
            r[j] = u + v;
            r[j + h] = u - v;
        }
}

// v2c, c2v: [n_checks][d][Q]; coef: [n_checks][d] (nonzero); mul: GF(Q) multiplication table [Q][Q].
// Warp i transforms edge i's row (scatter by coefficient, forward WHT), all threads form the
// prefix / suffix spectral products (thread per symbol over the rows in SMEM), warp i inverse-
// transforms, gathers by the coefficient, clamps and normalises its edge.
__global__ void __launch_bounds__(1024)
wht_check_update_kernel(const double* __restrict__ v2c, const int* __restrict__ coef, const uint8_t* __restrict__ mul,
                        int d, int Q, double* __restrict__ c2v) {
    extern __shared__ double sm[];
    double* y = sm;                         // d x Q spectra of the inputs
    double* s = sm + size_t(d) * Q;         // d x Q extrinsic products / outputs
    const int64_t ch = blockIdx.x;
    const double* in = v2c + size_t(ch) * d * Q;
    const int* cf = coef + size_t(ch) * d;
    const int LW = wht_lanes(Q), RPW = 32 / LW, EL = Q / LW;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
    const int lr = lane % LW;
    for (int i0 = warp * RPW; i0 < d; i0 += nw * RPW) {
        const int i = i0 + lane / LW;
        const bool on = i < d;
        if (on)
            for (int a = lr; a < Q; a += LW) y[size_t(i) * Q + mul[cf[i] * Q + a]] = in[size_t(i) * Q + a]; // y[alpha a] = msg[a]
        __syncwarp();
        double r[WHT_MAXE];
#pragma unroll
        for (int t = 0; t < WHT_MAXE; ++t) r[t] = (t < EL && on) ? y[size_t(i) * Q + lr + LW * t] : 0.0;
        wht_warp(r, Q, LW, lr);
#pragma unroll
        for (int t = 0; t < WHT_MAXE; ++t)
            if (t < EL && on) y[size_t(i) * Q + lr + LW * t] = r[t];
    }
    __syncthreads();
    for (int a = threadIdx.x; a < Q; a += blockDim.x) {
        double pre = 1.0;
        for (int i = 0; i < d; ++i) { // prefix into s, then multiply the suffix in from the back
            s[size_t(i) * Q + a] = pre;
            pre *= y[size_t(i) * Q + a];
        }
        double suf = 1.0;
        for (int i = d - 1; i >= 0; --i) {
            s[size_t(i) * Q + a] *= suf;
            suf *= y[size_t(i) * Q + a];
        }
    }
    __syncthreads();
    const double scale = 1.0 / Q;
    double* out = c2v + size_t(ch) * d * Q;
    for (int i0 = warp * RPW; i0 < d; i0 += nw * RPW) {
        const int i = i0 + lane / LW;
        const bool on = i < d;
        double r[WHT_MAXE];
#pragma unroll
        for (int t = 0; t < WHT_MAXE; ++t) r[t] = (t < EL && on) ? s[size_t(i) * Q + lr + LW * t] : 0.0;
        wht_warp(r, Q, LW, lr);
#pragma unroll
        for (int t = 0; t < WHT_MAXE; ++t)
            if (t < EL && on) s[size_t(i) * Q + lr + LW * t] = r[t];
        __syncwarp();
        // gather by the target coefficient, clamp, then the edge's sum (lane-strided, xor tree over the row's lanes)
        double acc = 0.0;
        if (on)
            for (int a = lr; a < Q; a += LW) {
                const double v = fmax(s[size_t(i) * Q + mul[cf[i] * Q + a]] * scale, 0.0);
                y[size_t(i) * Q + a] = v;
                acc += v;
            }
        for (int o = LW / 2; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        __syncwarp();
        if (on)
            for (int a = lr; a < Q; a += LW) out[size_t(i) * Q + a] = acc > 0.0 ? y[size_t(i) * Q + a] / acc : 1.0 / Q;
    }
}

} // namespace cider
