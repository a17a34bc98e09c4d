// pool_mma.cuh — Module B extrinsic attention pooling (denoiser.cpp:196-203
// with the attention Psi of DESIGN.md §4) in ONE pass over the edge rows, BF16 mode.
//
// For a check-regular code (every check has DEG = 6 edges, all BASELINE codes) the DEG x K edge rows
// (b, e0..e0+5, k) of one (bin, check) block are contiguous in HBM. A persistent CTA streams blocks:
//   1. TMA (SWIZZLE_128B boxes of 64 columns) brings the block into SMEM, double-buffered;
//   2. head scores s = n . [hi(u_h) | lo(u_h)] on the tensor cores with mma.sync m16n8k16 (bf16 in,
//      fp32 accumulate; the hi/lo split of u_h keeps the scores fp32-grade), fragments by ldmatrix;
//   3. per (k, 8-column chunk) thread: leave-one-out softmax over the other DEG-1 edges of its head and
//      the weighted sum (DEG-1) sum_{i2 != i} w n_{i2}, written as whole 512-byte rows.
// N is read once and pooled written once: the kernel is an HBM stream (the scores GEMM and its second
// read of N are gone).
#pragma once

#include "gemm_tc.cuh"

namespace cider {

constexpr int PM_THREADS = 256;
constexpr int PM_DEG = 6;
constexpr int PM_NBUF = 4;            // blocks in flight per CTA (two CTAs per SM)
constexpr int PM_BUF = 4 * 48 * 128;  // 4 k-blocks x 6K rows x 128 B, K <= 8 (k-block stride R x 128, 1 KB aligned)
struct PoolMmaLayout {
    static constexpr int U_OFF = PM_NBUF * PM_BUF;     // 16 x 256 bf16 score matrix, swizzled
    static constexpr int S_OFF = U_OFF + 16 * 512;     // per-warp score scratch [16 rows][8] fp32
    static constexpr int BAR_OFF = S_OFF + 8 * 128 * 4;
    static constexpr int TOTAL = BAR_OFF + 64 + 1024;
};

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& a0, uint32_t& a1, uint32_t& a2, uint32_t& a3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3)
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x2(uint32_t addr, uint32_t& b0, uint32_t& b1) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0, %1}, [%2];" : "=r"(b0), "=r"(b1) : "r"(addr));
}
__device__ __forceinline__ void mma_16816(float* d, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
                 "{%0, %1, %2, %3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// Nn: edge rows [(b*E + e)*K + k][256] bf16 through tmN (box {64, 6K}); Uhl: [16][256] bf16, rows
// h < NH = hi(u_h / sqrt(D/NH)), rows 8 + h = the bf16 remainder; n_blocks = bins * P.
// Two independent 4-warp groups per CTA alternate blocks (each with PM_NBUF / 2 buffers and its own
// named barrier); warp w of a group computes the head scores of block rows [12 w, 12 w + 12) (one m16
// tile) into the group's scratch, and after the group barrier pools rows k = w K/4 .. (w + 1) K/4 - 1
// (all four warps pool, for K = 4 as well as K = 8); no CTA-wide barrier sits between the phases.
// K (rows per edge, 4 or 8) is a template parameter: block geometry and the pooled-row loop are
// compile-time, so the per-row address arithmetic folds away (the kernel is issue-bound).
template <int K, int D>
__global__ void __launch_bounds__(PM_THREADS, 2)
pool_mma_kernel(const __grid_constant__ CUtensorMap tmN, const bf16* __restrict__ Uhl, const int* __restrict__ check_ptr,
                int P, int E, int NH, int64_t n_blocks, bf16* __restrict__ pooled) {
    using Lay = PoolMmaLayout;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* us = smem + Lay::U_OFF;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + Lay::BAR_OFF);
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    const int grp = warp / 4, wg = warp % 4;         // group, warp within the group
    // per-group score scratch [48 block rows][8 heads]: warp wg scores block rows [12 wg, 12 wg + 12)
    // (consecutive rows: distinct SW128 phases, conflict-free ldmatrix) and pools rows k = 2 wg, 2 wg + 1
    float* ss = reinterpret_cast<float*>(smem + Lay::S_OFF) + grp * 512;
    constexpr int CPB = 8 / K;       // checks per block (K = 4: two adjacent checks, so blocks stay 48 rows)
    constexpr int R = PM_DEG * K * CPB; // rows per block (48)
    constexpr int KBS = R * 128;     // k-block stride inside a block buffer
    constexpr int NKB = D / 64;      // 64-column k-blocks per row (4 or 2)
    // pooling: every lane takes 8 columns (one 16-byte chunk) of a row, so a row is D / 8 lanes and at
    // D = 128 a warp pools two (check, k) rows at once (the softmax work per lane is the same whatever the
    // width: with 4 columns per lane the D = 128 kernel spent twice the instructions per byte)
    constexpr int CPL = 8;           // pooled columns per lane
    constexpr int V = CPL / 2;       // float2 per lane per row
    constexpr int LPR = D / CPL;     // lanes per row (32 or 16)
    constexpr int UPW = 32 / LPR;    // (check, k) rows pooled per warp pass (1 or 2)
    constexpr int RB = D * 2;        // bytes per row of the score matrix
    static_assert(D == 256 || D == 128, "pool_mma: D = 128 or 256");
    constexpr int GB = PM_NBUF / 2;  // buffers per group

    // score matrix into SMEM: 16-byte chunk c of row n at (c & ~7) | ((c ^ n) & 7) (ldmatrix conflict-free)
    for (int i = tid; i < 16 * (D / 8); i += PM_THREADS) {
        const int n = i / (D / 8), c = i % (D / 8);
        *reinterpret_cast<uint4*>(us + n * RB + (((c & ~7) | ((c ^ n) & 7)) * 16)) =
            *reinterpret_cast<const uint4*>(Uhl + n * D + c * 8);
    }
    if (tid == 0) {
        for (int s = 0; s < PM_NBUF; ++s) tc::mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    griddep_wait(); // (programmatic dependent launch) inputs of the previous kernel visible
    griddep_launch_dependents();

    // this group's blocks: blockIdx.x + (2 i + grp) * gridDim.x, i = 0, 1, ...
    const int stride = 2 * int(gridDim.x);
    const int first = int(blockIdx.x) + grp * int(gridDim.x);
    const int nblk = int(n_blocks);
    const int PB = P / CPB; // blocks per bin
    auto issue = [&](int blk, int slot) { // one thread of the group: the block's column boxes
        const int b = blk / PB;
        const int j = (blk - b * PB) * CPB;
        const int row0 = (b * E + check_ptr[j]) * K;
        uint64_t* bar = &full[grp * GB + slot];
        tc::mbar_expect_tx(bar, NKB * R * 128);
        for (int kb = 0; kb < NKB; ++kb)
            tc::tma_load_2d(smem + (grp * GB + slot) * PM_BUF + kb * KBS, &tmN, bar, kb * 64, row0);
    };
    const bool leader = wg == 0 && tc::elect_one_sync(); // (all warps converged here) single-thread TMA issue
    if (leader)
        for (int s = 0; s < GB - 1; ++s)
            if (first + s * stride < nblk) issue(first + s * stride, s);
    // rows of this warp's m16 tile: block rows 12 wg + q for q < 12
    const int q = lane & 15;
    const int arow = 12 * wg + (q < 2 * PM_DEG ? q : q - 4); // pad lanes repeat rows 8-11 (same address: broadcast)
    const int lr = lane % LPR, sub = lane / LPR; // pooling: lane = columns [8 lr, 8 lr + 8) of row `sub` of the pass
    const int h = (lr * CPL) / (D / NH);         // ... a slice of head h
    int slot = 0;
    uint32_t ph = 0; // bit s: phase of this group's full[s]
    for (int blk = first; blk < nblk; blk += stride) {
        const int nxt = blk + (GB - 1) * stride;
        if (leader && nxt < nblk) issue(nxt, (slot + GB - 1) % GB); // released by the last group barrier
        tc::mbar_wait(&full[grp * GB + slot], (ph >> slot) & 1u);
        ph ^= 1u << slot;
        const uint8_t* nb = smem + (grp * GB + slot) * PM_BUF;
        const int b = blk / PB;
        const int e0 = check_ptr[(blk - b * PB) * CPB];
        if (12 * wg < R) {
            // (1) head scores of the warp's 12 rows: n-tile 0 = hi(u), 1 = lo(u)
            float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll 4
            for (int ks = 0; ks < D / 16; ++ks) {
                const int kc = ks * 2 + (lane >> 4);
                uint32_t a0, a1, a2, a3;
                ldsm_x4(tc::smem_u32(nb + (kc >> 3) * KBS + arow * 128 + (((kc & 7) ^ (arow & 7)) * 16)), a0, a1, a2, a3);
                const int kc2 = ks * 2 + ((lane >> 3) & 1);
#pragma unroll
                for (int nt = 0; nt < 2; ++nt) {
                    const int n = nt * 8 + (lane & 7);
                    uint32_t b0, b1;
                    ldsm_x2(tc::smem_u32(us + n * RB + (((kc2 & ~7) | ((kc2 ^ n) & 7)) * 16)), b0, b1);
                    mma_16816(acc[nt], a0, a1, a2, a3, b0, b1);
                }
            }
            // C rows lane/4 (+8), cols 2 (lane % 4) (+1): scores = hi + lo, into the group's scratch
            const int r0 = lane >> 2, c0 = (lane & 3) * 2;
            ss[(12 * wg + r0) * 8 + c0] = acc[0][0] + acc[1][0];
            ss[(12 * wg + r0) * 8 + c0 + 1] = acc[0][1] + acc[1][1];
            if (r0 + 8 < 2 * PM_DEG) {
                ss[(12 * wg + r0 + 8) * 8 + c0] = acc[0][2] + acc[1][2];
                ss[(12 * wg + r0 + 8) * 8 + c0 + 1] = acc[0][3] + acc[1][3];
            }
        }
        if (grp == 0) asm volatile("bar.sync 1, 128;" ::: "memory"); // the group's scores are in
        else asm volatile("bar.sync 2, 128;" ::: "memory");
        constexpr int kpw = 2; // pooled (check, k) rows per warp: 8 = CPB K per block over the 4 warps
        {
            // (2) pooling of rows k = wg kpw + kk (not unrolled: 128-register cap at 2 CTAs / SM)
#pragma unroll 1
            for (int kk = 0; kk < kpw / UPW; ++kk) {
                const int task = wg * kpw + kk * UPW + sub, cb = task / K, k = task % K; // check cb of the block, row k
                bf16* orow = pooled + (size_t(b * E + e0 + cb * PM_DEG) * K + k) * D + lr * CPL; // edge i at + i K D
                float2 f[PM_DEG][V];
                float sc[PM_DEG];
#pragma unroll
                for (int i = 0; i < PM_DEG; ++i) {
                    const int r = (cb * PM_DEG + i) * K + k;
                    sc[i] = ss[r * 8 + h];
                    { // 8 columns = one 16-byte chunk of k-block lr / 8
                        const uint4 u = *reinterpret_cast<const uint4*>(nb + (lr >> 3) * KBS + r * 128 + (((lr & 7) ^ (r & 7)) * 16));
                        const __nv_bfloat162* p2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
                        for (int v = 0; v < 4; ++v) f[i][v] = __bfloat1622float2(p2[v]);
                    }
                }
                // leave-one-out softmax: max over the edges other than i is the overall max M1 for every
                // i except the (first) argmax i1, whose max over the others is the runner-up M2 — the same
                // values as taking the max per i, with 12 exponentials instead of 36.
                int i1 = 0;
                float m1 = sc[0];
#pragma unroll
                for (int i2 = 1; i2 < PM_DEG; ++i2)
                    if (sc[i2] > m1) { m1 = sc[i2]; i1 = i2; }
                float m2 = -INFINITY;
#pragma unroll
                for (int i2 = 0; i2 < PM_DEG; ++i2)
                    if (i2 != i1) m2 = fmaxf(m2, sc[i2]);
                // exp(s - m) = 2^(s log2e - m log2e): one FFMA + one MUFU.EX2 each (flush-to-zero: a weight below
                // 2^-126 of the largest is dropped); __expf spends ~6 instructions on the denormal range
                float e1[PM_DEG], e2[PM_DEG];
                const float nm1 = -m1 * 1.4426950408889634f, nm2 = -m2 * 1.4426950408889634f;
#pragma unroll
                for (int i2 = 0; i2 < PM_DEG; ++i2) {
                    e1[i2] = ex2_approx(fmaf(sc[i2], 1.4426950408889634f, nm1));
                    e2[i2] = ex2_approx(fmaf(sc[i2], 1.4426950408889634f, nm2));
                }
                // Leave-one-out sums by prefix / suffix over the edges (no term of edge i enters output i,
                // so extrinsicity stays bitwise): for i != i1, out_i = (d-1) (P_i + S_i) / (pd_i + sd_i)
                // with P_i = sum_{i2 < i} e1 n, S_i = sum_{i2 > i} e1 n (pd, sd the same sums of e1); row
                // i1 uses e2 in the same association (below) and is stored over the e1 value.
                auto store_row = [&](int i, const float2* out, float fct) {
                    __nv_bfloat162 po[V];
#pragma unroll
                    for (int v = 0; v < V; ++v) {
                        const float2 sc2 = __fmul2_rn(out[v], make_float2(fct, fct)); // (packed: same products)
                        po[v] = __floats2bfloat162_rn(sc2.x, sc2.y);
                    }
                    *reinterpret_cast<uint4*>(orow + i * K * D) = *reinterpret_cast<const uint4*>(po);
                };
                float2 pre[PM_DEG][V]; // pre[i] = P_i (i >= 1)
                float pd[PM_DEG];
#pragma unroll
                for (int v = 0; v < V; ++v) pre[1][v] = __fmul2_rn(make_float2(e1[0], e1[0]), f[0][v]);
                pd[1] = e1[0];
#pragma unroll
                for (int i = 2; i < PM_DEG; ++i) {
#pragma unroll
                    for (int v = 0; v < V; ++v) pre[i][v] = __ffma2_rn(make_float2(e1[i - 1], e1[i - 1]), f[i - 1][v], pre[i - 1][v]);
                    pd[i] = pd[i - 1] + e1[i - 1];
                }
                float2 suf[V]; // running S_i, from the top
                float sd = 0.0f;
#pragma unroll
                for (int i = PM_DEG - 1; i >= 0; --i) {
                    float2 out[V];
                    float den;
                    if (i == PM_DEG - 1) {
#pragma unroll
                        for (int v = 0; v < V; ++v) out[v] = pre[i][v];
                        den = pd[i];
                    } else if (i == 0) {
#pragma unroll
                        for (int v = 0; v < V; ++v) out[v] = suf[v];
                        den = sd;
                    } else {
#pragma unroll
                        for (int v = 0; v < V; ++v) out[v] = __fadd2_rn(pre[i][v], suf[v]);
                        den = pd[i] + sd;
                    }
                    store_row(i, out, __fdividef(float(PM_DEG - 1), den));
                    if (i > 0) { // S_{i-1} = S_i + e1_i n_i
                        if (i == PM_DEG - 1) {
#pragma unroll
                            for (int v = 0; v < V; ++v) suf[v] = __fmul2_rn(make_float2(e1[i], e1[i]), f[i][v]);
                            sd = e1[i];
                        } else {
#pragma unroll
                            for (int v = 0; v < V; ++v) suf[v] = __ffma2_rn(make_float2(e1[i], e1[i]), f[i][v], suf[v]);
                            sd = sd + e1[i];
                        }
                    }
                }
                { // row i1 with the runner-up max (e2), in the SAME prefix / suffix association as the rows above:
                    // the edges on the other side of a partial sum enter it with weight zero (+ 0 leaves a sum
                    // unchanged), so an output row is one fixed function of the OTHER edges' rows and scores
                    // whether or not its own score is the largest — extrinsicity holds bit for bit by construction
                    // (an ascending sum over the others differs from prefix + suffix in the last bit, which a
                    // change of the row's own tokens can expose by moving the argmax: rare after the bf16
                    // rounding, but not excluded)
                    float2 pp[V], sp[V];
                    float pdn, sdn;
                    {
                        const float w = 0 < i1 ? e2[0] : 0.0f;
#pragma unroll
                        for (int v = 0; v < V; ++v) pp[v] = __fmul2_rn(make_float2(w, w), f[0][v]);
                        pdn = w;
                    }
#pragma unroll
                    for (int j = 1; j < PM_DEG - 1; ++j) {
                        const float w = j < i1 ? e2[j] : 0.0f;
#pragma unroll
                        for (int v = 0; v < V; ++v) pp[v] = __ffma2_rn(make_float2(w, w), f[j][v], pp[v]);
                        pdn = pdn + w;
                    }
                    {
                        const float w = PM_DEG - 1 > i1 ? e2[PM_DEG - 1] : 0.0f;
#pragma unroll
                        for (int v = 0; v < V; ++v) sp[v] = __fmul2_rn(make_float2(w, w), f[PM_DEG - 1][v]);
                        sdn = w;
                    }
#pragma unroll
                    for (int j = PM_DEG - 2; j >= 1; --j) {
                        const float w = j > i1 ? e2[j] : 0.0f;
#pragma unroll
                        for (int v = 0; v < V; ++v) sp[v] = __ffma2_rn(make_float2(w, w), f[j][v], sp[v]);
                        sdn = sdn + w;
                    }
                    float2 out[V];
#pragma unroll
                    for (int v = 0; v < V; ++v) out[v] = __fadd2_rn(pp[v], sp[v]);
                    store_row(i1, out, __fdividef(float(PM_DEG - 1), pdn + sdn));
                }
            }
        }
        if (grp == 0) asm volatile("bar.sync 1, 128;" ::: "memory"); // the group is done with this buffer
        else asm volatile("bar.sync 2, 128;" ::: "memory");
        slot = (slot + 1) % GB;
    }
}

} // namespace cider
