// wht.cuh — batched GF(Q) check-node update in the Walsh–Hadamard domain (
// reference: update_check_wht / check_update_wht, bp.cpp:128-149, 195-269).
//
// For every check (one CTA per check; bins x checks in one launch) and every edge i of it:
//   y_i   = WHT( scatter(v2c_i by coefficient) )          y_i[alpha_i * a] = v2c_i[a]
//   spec_i = prod_{j<i} y_j  *  prod_{j>i} y_j            (prefix / suffix products, extrinsic)
//   c2v_i[a] = max( WHT(spec_i)[alpha_i * a] / Q, 0 ),  normalised (uniform if all mass vanished)
// Thread a owns spectral index a of every edge, so the prefix/suffix products are per-thread
// register loops; the transforms are SMEM butterflies. fp64 throughout (the reference keeps the
// spectra in long double; the GPU has no 80-bit type — parity tolerance in tests/test_gpu.py).
#pragma once

#include "common.cuh"

namespace cider {

constexpr int WHT_MAXD = 32;

__device__ __forceinline__ void wht_rows_smem(double* y, int rows, int Q) {
    for (int len = 1; len < Q; len <<= 1) {
        __syncthreads();
        for (int idx = threadIdx.x; idx < rows * (Q / 2); idx += blockDim.x) {
            const int r = idx / (Q / 2), p = idx % (Q / 2);
            const int a = (p / len) * (2 * len) + (p % len);
            double* row = y + size_t(r) * Q;
            const double u = row[a], v = row[a + len];
            row[a] = u + v;
            row[a + len] = u - v;
        }
    }
    __syncthreads();
}

// v2c, c2v: [n_checks][d][Q]; coef: [n_checks][d] (nonzero); mul: GF(Q) multiplication table [Q][Q]
__global__ void __launch_bounds__(256)
wht_check_update_kernel(const double* __restrict__ v2c, const int* __restrict__ coef, const uint8_t* __restrict__ mul,
                        int d, int Q, double* __restrict__ c2v) {
    extern __shared__ double sm[];
    double* y = sm;                         // d x Q spectra of the inputs
    double* s = sm + size_t(d) * Q;         // d x Q extrinsic products / outputs
    __shared__ double red[WHT_MAXD][8];
    const int64_t ch = blockIdx.x;
    const double* in = v2c + size_t(ch) * d * Q;
    const int* cf = coef + size_t(ch) * d;
    for (int idx = threadIdx.x; idx < d * Q; idx += blockDim.x) {
        const int i = idx / Q, a = idx % Q;
        y[size_t(i) * Q + mul[cf[i] * Q + a]] = in[idx]; // scatter_by: y[alpha a] = msg[a]
    }
    wht_rows_smem(y, d, Q);
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
    wht_rows_smem(s, d, Q);
    // gather by the target coefficient, clamp, normalise per edge
    const double scale = 1.0 / Q;
    for (int idx = threadIdx.x; idx < d * Q; idx += blockDim.x) {
        const int i = idx / Q, a = idx % Q;
        y[idx] = fmax(s[size_t(i) * Q + mul[cf[i] * Q + a]] * scale, 0.0);
    }
    __syncthreads();
    // per-edge sums (in ascending symbol order, one warp per edge), then normalise
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
    for (int i = warp; i < d; i += nw) {
        double acc = 0.0;
        for (int a = lane; a < Q; a += 32) acc += y[size_t(i) * Q + a];
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) red[i][0] = acc;
    }
    __syncthreads();
    double* out = c2v + size_t(ch) * d * Q;
    for (int idx = threadIdx.x; idx < d * Q; idx += blockDim.x) {
        const int i = idx / Q;
        const double sum = red[i][0];
        out[idx] = sum > 0.0 ? y[idx] / sum : 1.0 / Q;
    }
}

} // namespace cider
