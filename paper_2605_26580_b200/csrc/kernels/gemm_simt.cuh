// gemm_simt.cuh — fp32 SIMT GEMM for the FP32 (parity) mode.
//
// C[M x N] = [A0 | A1][M x K] . B[N x K]^T, fp32 FFMA, then the shared epilogue. Each output is
// accumulated by one thread in ascending k order, so rows with identical inputs produce
// bitwise-identical outputs (the reference's exact row-permutation equivariance,
// test_denoiser.cpp:293-313, survives on the device). 64x64 tiles, 256 threads, 4x4 per thread.
#pragma once

#include "common.cuh"

namespace cider {

constexpr int SG_BM = 64, SG_BN = 64, SG_BK = 16;

__global__ void __launch_bounds__(256)
gemm_simt_f32(const float* __restrict__ A0, int lda0, int K0, const float* __restrict__ A1, int lda1,
              const float* __restrict__ Bw, int ldb, int M, int N, int K, Epi ep) {
    __shared__ float As[SG_BK][SG_BM + 4];
    __shared__ float Bs[SG_BK][SG_BN + 4];
    const int tid = threadIdx.x;
    const int tx = tid % 16, ty = tid / 16;
    const int m0 = blockIdx.y * SG_BM, n0 = blockIdx.x * SG_BN;
    float acc[4][4] = {};
    for (int kb = 0; kb < K; kb += SG_BK) {
        // 64 x 16 A tile and 64 x 16 B tile: 1024 elements each, 4 per thread
        for (int i = tid; i < SG_BM * SG_BK; i += 256) {
            int r = i / SG_BK, kk = i % SG_BK;
            int m = m0 + r, k = kb + kk;
            float va = 0.0f;
            if (m < M && k < K) va = k < K0 ? A0[size_t(m) * lda0 + k] : A1[size_t(m) * lda1 + (k - K0)];
            As[kk][r] = va;
            int n = n0 + r;
            float vb = 0.0f;
            if (n < N && k < K) vb = Bw[size_t(n) * ldb + k];
            Bs[kk][r] = vb;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < SG_BK; ++kk) {
            float a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
    for (int i = 0; i < 4; ++i) {
        int m = m0 + ty * 4 + i;
        if (m >= M) continue;
        int n = n0 + tx * 4;
        int cnt = min(4, N - n);
        if (cnt <= 0) continue;
        epi_apply<float>(ep, m, n, acc[i], cnt);
    }
}

} // namespace cider
