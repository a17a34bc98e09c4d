// workload.cuh — the BASELINE evidence generator on the device (the step before
// the path). One thread per bin replays, on its own mt19937_64 stream seeded derive_seed(master,
// 16 + bin), exactly the host generator cider_workload_bins (host.cpp):
//   sample_codewords: K distinct info vectors of uniform symbols, systematic encode;
//   per slot: K erasure U(0,1), one false-candidate U(0,1) (+ its symbol), Q normals,
//   y = one-hots + sigma N(0,1), S = float(log_softmax(y)).
// The libstdc++ (GCC 13) distribution algorithms are restated bit for bit: uniform_int_distribution
// = Lemire's nearly divisionless downscaling of a 64-bit draw, uniform_real_distribution =
// generate_canonical (double(x) / 2^64, clamped below 1), normal_distribution = the Marsaglia
// polar method with one cached value. Floating point is written with explicit _rn intrinsics so
// nvcc cannot contract it into FMAs the host build does not use; only exp/log may differ from
// glibc in the last ulp of a double, which the final float cast hides (tests check it).
#pragma once

#include <cstdint>

namespace cider {
namespace wl {

struct Mt64 {
    uint64_t mt[312];
    int idx;
    __device__ void seed(uint64_t s) {
        mt[0] = s;
        for (int i = 1; i < 312; ++i) mt[i] = 6364136223846793005ULL * (mt[i - 1] ^ (mt[i - 1] >> 62)) + uint64_t(i);
        idx = 312;
    }
    __device__ void twist() {
        for (int i = 0; i < 312; ++i) {
            const uint64_t x = (mt[i] & 0xFFFFFFFF80000000ULL) | (mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            mt[i] = mt[(i + 156) % 312] ^ xa;
        }
        idx = 0;
    }
    __device__ uint64_t next() {
        if (idx >= 312) twist();
        uint64_t y = mt[idx++];
        y ^= (y >> 29) & 0x5555555555555555ULL;
        y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
        y ^= (y << 37) & 0xFFF7EEE000000000ULL;
        y ^= y >> 43;
        return y;
    }
};

__device__ __forceinline__ uint64_t mix64(uint64_t z) { // = host.hpp mix64 (seeding.hpp:10-22)
    z += 0x9e3779b97f4a7c15ULL;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t derive_seed(uint64_t master, uint64_t index) {
    return mix64(master ^ mix64(index + 0x517cc1b727220a95ULL));
}

// uniform_int_distribution<int>(0, range - 1) with a 64-bit engine (GCC 13: _S_nd<unsigned __int128>)
__device__ __forceinline__ int uniform_int(Mt64& g, uint64_t range) {
    uint64_t x = g.next();
    uint64_t low = x * range, high = __umul64hi(x, range);
    if (low < range) {
        const uint64_t threshold = (0ULL - range) % range;
        while (low < threshold) {
            x = g.next();
            low = x * range;
            high = __umul64hi(x, range);
        }
    }
    return int(high);
}
// generate_canonical<double, 53>: double(x) / 2^64, clamped below 1
__device__ __forceinline__ double canonical(Mt64& g) {
    const double r = __dmul_rn(__ull2double_rn(g.next()), 5.421010862427522170037264e-20); // 2^-64, exact
    return r >= 1.0 ? 0.99999999999999988898 : r;                                         // nextafter(1, 0)
}
struct Normal {
    double saved = 0.0;
    bool have = false;
    __device__ double operator()(Mt64& g) {
        if (have) {
            have = false;
            return saved;
        }
        double x, y, r2;
        do {
            x = __dadd_rn(__dmul_rn(2.0, canonical(g)), -1.0);
            y = __dadd_rn(__dmul_rn(2.0, canonical(g)), -1.0);
            r2 = __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y));
        } while (r2 > 1.0 || r2 == 0.0);
        const double mult = sqrt(__ddiv_rn(__dmul_rn(-2.0, log(r2)), r2));
        saved = __dmul_rn(x, mult);
        have = true;
        return __dmul_rn(y, mult); // * stddev 1 + mean 0: exact
    }
};

struct Sys { // systematic encoder tables (host systematic_form)
    int n_info, n_pivot;
    const int* info;     // [n_info] slot of info symbol j
    const int* pivot;    // [n_pivot] slot of parity row i
    const uint8_t* red;  // [n_pivot][n_info] coefficients
    const uint8_t* mul;  // [Q][Q]
};

constexpr int WL_MAXQ = 256, WL_MAXK = 16, WL_MAXL = 512;

__global__ void __launch_bounds__(64) workload_bins_kernel(Sys sys, int L, int K, int Q, double sigma, double p_erase,
                                                         double p_false, uint64_t master, int64_t first, int n,
                                                         int* __restrict__ truth, float* __restrict__ S) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    Mt64 g;
    g.seed(derive_seed(master, uint64_t(16 + first + i)));
    // ---- sample_codewords: K distinct info vectors, systematic encode
    int* cw = truth + size_t(i) * K * L;
    int info[WL_MAXL];
    int nk = 0;
    while (nk < K) {
        for (int j = 0; j < sys.n_info; ++j) info[j] = uniform_int(g, uint64_t(Q));
        bool dup = false; // distinct info vectors (compared at the info positions of the rows so far)
        for (int r = 0; r < nk && !dup; ++r) {
            bool same = true;
            for (int j = 0; j < sys.n_info; ++j) same = same && cw[size_t(r) * L + sys.info[j]] == info[j];
            dup = same;
        }
        if (dup) continue;
        int* c = cw + size_t(nk) * L;
        for (int j = 0; j < sys.n_info; ++j) c[sys.info[j]] = info[j];
        for (int p = 0; p < sys.n_pivot; ++p) {
            int acc = 0;
            for (int j = 0; j < sys.n_info; ++j) acc ^= sys.mul[sys.red[p * sys.n_info + j] * Q + info[j]];
            c[sys.pivot[p]] = acc;
        }
        ++nk;
    }
    // ---- evidence rows
    Normal nrm;
    double y[WL_MAXQ];
    for (int l = 0; l < L; ++l) {
        for (int a = 0; a < Q; ++a) y[a] = 0.0;
        for (int k = 0; k < K; ++k) {
            const bool erased = canonical(g) < p_erase;
            if (!erased) y[cw[size_t(k) * L + l]] += 1.0;
        }
        if (canonical(g) < p_false) y[uniform_int(g, uint64_t(Q))] += 1.0;
        for (int a = 0; a < Q; ++a) y[a] = __dadd_rn(y[a], __dmul_rn(sigma, nrm(g)));
        double mx = y[0];
        for (int a = 1; a < Q; ++a) mx = fmax(mx, y[a]);
        double se = 0.0;
        for (int a = 0; a < Q; ++a) se = __dadd_rn(se, exp(__dadd_rn(y[a], -mx)));
        const double lse = __dadd_rn(mx, log(se));
        float* out = S + (size_t(i) * L + l) * Q;
        for (int a = 0; a < Q; ++a) out[a] = __double2float_rn(__dadd_rn(y[a], -lse));
    }
}

} // namespace wl
} // namespace cider
