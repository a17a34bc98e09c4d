// amp.cuh — batched AMP slot detector (the step before the path; the reference's
// amp_detect / evidence_row / detect_frame, amp.cpp:63-148) for many bins at once.
//
// One CTA per (bin, slot): the slot's partial-DFT dictionary A_l (fixed per dataset, resident in
// HBM / L2, stored transposed [n_s][q] so a thread per column reads coalesced rows) against that
// bin's observation y. Per iteration, in the reference's operation order (fp64, no FMA contraction:
// every complex product is (ac - bd, ad + bc) with separately rounded products, as g++ computes it
// on x86-64 without -ffast-math):
//   nu     = sum_r |resid_r|^2 / n_s (floored at 1e-12)            — one thread, r ascending
//   pseudo = u + A^H resid                                         — thread per column, r ascending
//   (u, div) = mmse_denoise(pseudo, nu)                            — thread per column (log domain)
//   onsager = sum_col div / n_s                                    — one thread, column ascending
//   resid' = y - sum_{col, u != 0} u_col A[:, col] + resid * onsager — thread per row, col ascending
// then S[col] = max(floor, log_bg_posterior(u + A^H resid, nu)). Non-finite residuals set a flag with
// the iteration (the reference throws std::runtime_error naming it).
#pragma once

#include <cuda_runtime.h>

namespace cider {

struct AmpParams {
    int iters;
    double rho_bg, sigma_u2, floor;
    double log_rho, log1m_rho; // log(rho_bg), log1p(-rho_bg)
};

__device__ __forceinline__ double2 cmul_rn(double2 a, double2 b) { // (a.x + i a.y)(b.x + i b.y)
    return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)), __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}
__device__ __forceinline__ double norm_rn(double2 a) { return __dadd_rn(__dmul_rn(a.x, a.x), __dmul_rn(a.y, a.y)); }

// log_bg_posterior (amp.cpp:40-47): log P(active | r) of the Bernoulli-Gaussian scalar channel
__device__ __forceinline__ double amp_log_post(double r2, double nu, const AmpParams& p) {
    const double v1 = __dadd_rn(nu, p.sigma_u2);
    const double la = __dsub_rn(__dsub_rn(p.log_rho, log(v1)), __ddiv_rn(r2, v1));
    const double li = __dsub_rn(__dsub_rn(p.log1m_rho, log(nu)), __ddiv_rn(r2, nu));
    const double hi = la > li ? la : li, lo = la > li ? li : la;
    return __dsub_rn(la, __dadd_rn(hi, log1p(exp(__dsub_rn(lo, hi)))));
}

template <int NT>
__global__ void __launch_bounds__(NT)
amp_detect_kernel(const double2* __restrict__ At /*[L][n_s][q]*/, const double2* __restrict__ y /*[B][L][n_s]*/, int B,
                  int L, int q, int n_s, AmpParams p, double* __restrict__ S /*[B][L][q]*/, int* __restrict__ bad_iter) {
    extern __shared__ double2 amp_sm[];
    double2* res = amp_sm;        // [n_s]
    double2* nxt = res + n_s;     // [n_s]
    double2* ys = nxt + n_s;      // [n_s]
    double2* u = ys + n_s;        // [q]
    double* div = reinterpret_cast<double*>(u + q); // [q]
    __shared__ double s_nu, s_ons;
    __shared__ int s_bad;
    const int bl = blockIdx.x, l = bl % L;
    const double2* A = At + size_t(l) * n_s * q;
    const double2* yb = y + size_t(bl) * n_s;
    for (int r = threadIdx.x; r < n_s; r += NT) { ys[r] = yb[r]; res[r] = yb[r]; }
    for (int c = threadIdx.x; c < q; c += NT) u[c] = make_double2(0.0, 0.0);
    if (threadIdx.x == 0) s_bad = 0;
    __syncthreads();
    auto residual_nu = [&] {
        if (threadIdx.x == 0) {
            double e = 0.0;
            for (int r = 0; r < n_s; ++r) e = __dadd_rn(e, norm_rn(res[r]));
            const double nu = __ddiv_rn(e, double(n_s));
            s_nu = nu < 1e-12 ? 1e-12 : nu;
        }
        __syncthreads();
    };
    auto ah_resid = [&](int c) { // sum_r conj(A[r][c]) resid[r], r ascending
        double2 acc = make_double2(0.0, 0.0);
        for (int r = 0; r < n_s; ++r) {
            const double2 a = A[size_t(r) * q + c];
            const double2 pr = cmul_rn(make_double2(a.x, -a.y), res[r]);
            acc = make_double2(__dadd_rn(acc.x, pr.x), __dadd_rn(acc.y, pr.y));
        }
        return acc;
    };
    for (int it = 0; it < p.iters; ++it) {
        residual_nu();
        const double nu = s_nu;
        // pseudo and the MMSE denoiser (amp.cpp:52-61), thread per column
        for (int c = threadIdx.x; c < q; c += NT) {
            const double2 acc = ah_resid(c);
            const double2 ps = make_double2(__dadd_rn(u[c].x, acc.x), __dadd_rn(u[c].y, acc.y));
            const double r2 = norm_rn(ps);
            const double v1 = __dadd_rn(nu, p.sigma_u2);
            const double gain = __ddiv_rn(p.sigma_u2, v1);
            const double delta = __ddiv_rn(p.sigma_u2, __dmul_rn(nu, v1));
            const double pa = exp(amp_log_post(r2, nu, p));
            const double pg = __dmul_rn(pa, gain);
            u[c] = make_double2(__dmul_rn(pg, ps.x), __dmul_rn(pg, ps.y)); // (p * gain) * r
            // gain * (p + |r|^2 p (1 - p) delta)
            div[c] = __dmul_rn(gain, __dadd_rn(pa, __dmul_rn(__dmul_rn(__dmul_rn(r2, pa), __dsub_rn(1.0, pa)), delta)));
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double ds = 0.0;
            for (int c = 0; c < q; ++c) ds = __dadd_rn(ds, div[c]);
            s_ons = __ddiv_rn(ds, double(n_s));
        }
        __syncthreads();
        const double ons = s_ons;
        // Onsager-corrected residual (amp.cpp:99-106), thread per row
        for (int r = threadIdx.x; r < n_s; r += NT) {
            double2 v = ys[r];
            const double2* ar = A + size_t(r) * q;
            for (int c = 0; c < q; ++c) {
                const double2 uc = u[c];
                if (uc.x == 0.0 && uc.y == 0.0) continue;
                const double2 pr = cmul_rn(uc, ar[c]);
                v = make_double2(__dsub_rn(v.x, pr.x), __dsub_rn(v.y, pr.y));
            }
            const double2 co = cmul_rn(res[r], make_double2(ons, 0.0));
            v = make_double2(__dadd_rn(v.x, co.x), __dadd_rn(v.y, co.y));
            nxt[r] = v;
            if (!isfinite(v.x) || !isfinite(v.y)) atomicCAS(&s_bad, 0, it + 1);
        }
        __syncthreads();
        for (int r = threadIdx.x; r < n_s; r += NT) res[r] = nxt[r];
        __syncthreads();
        if (s_bad) break;
    }
    if (s_bad) {
        if (threadIdx.x == 0) atomicMin(bad_iter, s_bad - 1);
        return;
    }
    residual_nu();
    const double nu = s_nu;
    double* Sb = S + size_t(bl) * q;
    for (int c = threadIdx.x; c < q; c += NT) { // evidence_row (amp.cpp:124-131)
        const double2 acc = ah_resid(c);
        const double2 ps = make_double2(__dadd_rn(u[c].x, acc.x), __dadd_rn(u[c].y, acc.y));
        const double s = amp_log_post(norm_rn(ps), nu, p);
        Sb[c] = s < p.floor ? p.floor : s;
    }
}

} // namespace cider
