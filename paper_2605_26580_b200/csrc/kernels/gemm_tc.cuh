// gemm_tc.cuh — persistent warp-specialised tcgen05 GEMM for sm_100a (BF16 mode).
//
//   C[M x N] = [A0 | A1][M x K] . B[N x K]^T     bf16 operands, fp32 accumulation in TMEM
//
// warp 0     : TMA producer — 128x64 A tiles (from A0 for k < K0, else A1: the [z; e] / [z~; m]
//              concatenations of the gate and fusion maps never materialise) and BNx64 B tiles,
//              SWIZZLE_128B, STAGES-deep mbarrier ring.
// warp 1     : TMEM allocator + single-thread tcgen05.mma.cta_group::1.kind::f16 issuer
//              (M=128, N=BN, K=16 per instruction), tcgen05.commit to free smem stages and to
//              publish a finished accumulator.
// warps 2..5 : epilogue — tcgen05.ld 32x32b.x32 (one TMEM lane = one output row per thread),
//              fused element-wise epilogue (bias, GELU, sigmoid gate, residual, +beta*S,
//              kappa/argmax row statistics), vectorised global stores.
// Two TMEM accumulators (2*BN columns) let the epilogue of tile i overlap the MMAs of tile i+1.
// Tiles are visited m-major so the N tiles that share an A block run back to back (L2 reuse).
#pragma once

#include <cuda.h>

#include "common.cuh"

namespace cider {
namespace tc {

constexpr int BM = 128, BK = 64, STAGES = 4;
constexpr int NUM_THREADS = 192;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// try_wait with a suspend-time hint (ns): a waiting warp sleeps in the barrier unit instead of re-issuing
// the try_wait loop every few dozen cycles — in the fused MLPs ~28% of the executed instructions were such
// retries of the producer / issuer / final-epilogue warps, competing with the GELU warps for issue slots
// (c5 +0.35% in a same-box bench A/B, profiles/r2/experiments/README.md).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    uint32_t ok = 0;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(a), "r"(parity), "r"(1000000u)
            : "memory");
    } while (!ok);
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y)
        : "memory");
}
// One lane of the (converged) warp, by elect.sync: ptxas then knows that the region it guards runs in a
// single thread and keeps the TMA / MMA operands (descriptors, coordinates, barrier addresses) in uniform
// registers. A `lane == 0` guard compiles every tcgen05.mma into an ELECT + R2UR.BROADCAST x5 + retry-branch
// sequence (~14 instructions per MMA against ~3).
__device__ __forceinline__ bool elect_one_sync() {
    uint32_t pred = 0;
    asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(pred));
    return pred != 0;
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// SMEM matrix descriptor: K-major, SWIZZLE_128B, 8-row core groups 1024 B apart (SBO), version 1.
__device__ __forceinline__ uint64_t sw128_desc(const void* p) {
    const uint32_t a = smem_u32(p);
    uint64_t d = 0;
    d |= uint64_t((a & 0x3FFFF) >> 4);
    d |= uint64_t(16 >> 4) << 16;
    d |= uint64_t(1024 >> 4) << 32;
    d |= uint64_t(1) << 46;
    d |= uint64_t(2) << 61;
    return d;
}
// instruction descriptor kind::f16: D=f32, A=B=bf16, both K-major, N>>3 @17, M>>4 @24
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
    return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(M >> 4) << 24);
}
__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
          "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
          "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

struct Args {
    int M, N, K, K0;
    int tiles_n, tiles;
    Epi ep;
};

// EPW epilogue warps (0 = layout without the EP_DEMIX staging, for gemm_grp.cuh). BRES: the whole
// B operand (N = BN, K <= 256: at most 4 k-blocks) is loaded once per CTA and stays resident; the
// ring then streams only A tiles (the tall-skinny GEMMs against W, W^T, V^T re-read 128 KB of B per
// 128-row tile otherwise). Kernels with more than 4 epilogue warps and a streamed B use a 2-stage ring.
template <int BN, int EPW = 4, bool BRES = false>
struct SmemLayout {
    static constexpr int A_BYTES = BM * BK * 2;
    static constexpr int B_BYTES = BN * BK * 2;
    static constexpr int BRES_BYTES = BRES ? 4 * B_BYTES : 0;
    static constexpr int STAGE_BYTES = BRES ? A_BYTES : A_BYTES + B_BYTES;
    // EP_DEMIX transpose staging per epilogue warp: [32][33] fp32 (padded: conflict-free rows and
    // columns) + [32][32] bf16 results; EPW <= 4 kernels only stage bf16 stores ([32][32] bf16)
    static constexpr int STG_WARP = EPW > 4 ? 32 * 33 * 4 + 32 * 32 * 2 : 32 * 32 * 2;
    static constexpr int FREE = 232448 - 1024 - 256 - BRES_BYTES - EPW * STG_WARP;
    static constexpr int NST_FIT = (FREE / STAGE_BYTES) > 8 ? 8 : (FREE / STAGE_BYTES);
    static constexpr int NST_STREAM = (196608 / STAGE_BYTES) > 8 ? 8 : (196608 / STAGE_BYTES);
    static constexpr int NST = BRES ? NST_FIT : EPW > 4 ? 2 : EPW == 0 ? STAGES : NST_STREAM;
    static constexpr int RING_OFF = BRES_BYTES;
    static constexpr int STG_OFF = RING_OFF + NST * STAGE_BYTES;
    static constexpr int BAR_OFF = STG_OFF + EPW * STG_WARP;
    static constexpr int TOTAL = BAR_OFF + 256 + 1024; // barriers + 1 KB alignment slack
    static constexpr int TMEM_COLS = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128 : (2 * BN <= 256) ? 256 : 512;
    static_assert(NST >= 2, "gemm_tc ring");
    static_assert(TOTAL <= 232448, "gemm_tc shared memory");
};

// 32 consecutive output columns of one row through the shared epilogue, vectorised.
__device__ __forceinline__ void epi_row32(const Epi& ep, int m, int n0, float* v) {
    if (ep.kind == EP_SCORES) { // columns [0,16) hold hi(u_h).n, [16,32) lo(u_h).n; the rest is padding
        if (n0 == 0) {
#pragma unroll
            for (int h = 0; h < 16; ++h) // static indices: v stays in registers
                if (h < ep.K) ep.out_f[size_t(m) * ep.ldo + h] = v[h] + v[16 + h];
        }
        return;
    }
    if (ep.bias) {
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
            float4 b = *reinterpret_cast<const float4*>(ep.bias + n0 + i);
            v[i] += b.x; v[i + 1] += b.y; v[i + 2] += b.z; v[i + 3] += b.w;
        }
    }
    if (ep.kind == EP_GELU) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = 2.0f * gelu_f(v[i]); // BF16 mode: 2 GELU, second layer stored halved
    } else if (ep.kind == EP_GATE || ep.kind == EP_RESID) {
        // z / e from the fp32 stream when present, else from the bf16 stream (BF16 mode)
        float zz[32], ee[32];
        if (ep.z) {
            const float* zr = ep.z + size_t(m) * ep.ldz + n0;
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
                float4 z4 = *reinterpret_cast<const float4*>(zr + i);
                zz[i] = z4.x; zz[i + 1] = z4.y; zz[i + 2] = z4.z; zz[i + 3] = z4.w;
            }
        } else {
            const bf16* zr = ep.zb + size_t(m) * ep.ldz + n0;
#pragma unroll
            for (int i = 0; i < 32; ++i) zz[i] = __bfloat162float(zr[i]);
        }
        if (ep.kind == EP_GATE) {
            if (ep.e) {
                const float* er = ep.e + size_t(m) * ep.ldz + n0;
#pragma unroll
                for (int i = 0; i < 32; ++i) ee[i] = er[i];
            } else {
                const bf16* er = ep.eb + size_t(m) * ep.ldz + n0;
#pragma unroll
                for (int i = 0; i < 32; ++i) ee[i] = __bfloat162float(er[i]);
            }
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                float g = sigmoid_f(v[i]);
                v[i] = g * zz[i] + (1.0f - g) * ee[i];
            }
        } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] += zz[i];
        }
    } else if (ep.kind == EP_LBAR) {
        const float* s = ep.S + lbar_s_index(ep, m, n0);
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
            float4 s4 = *reinterpret_cast<const float4*>(s + i);
            v[i] += ep.beta * s4.x; v[i + 1] += ep.beta * s4.y; v[i + 2] += ep.beta * s4.z; v[i + 3] += ep.beta * s4.w;
        }
    }
    if (ep.out_f) {
        float* o = ep.out_f + size_t(m) * ep.ldo + n0;
#pragma unroll
        for (int i = 0; i < 32; i += 4) *reinterpret_cast<float4*>(o + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
    }
    if (ep.out_t) {
        bf16* o = reinterpret_cast<bf16*>(ep.out_t) + size_t(m) * ep.ldo + n0;
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
            __nv_bfloat162 p0 = __floats2bfloat162_rn(v[i], v[i + 1]);
            __nv_bfloat162 p1 = __floats2bfloat162_rn(v[i + 2], v[i + 3]);
            __nv_bfloat162 p2 = __floats2bfloat162_rn(v[i + 4], v[i + 5]);
            __nv_bfloat162 p3 = __floats2bfloat162_rn(v[i + 6], v[i + 7]);
            uint4 u;
            u.x = *reinterpret_cast<uint32_t*>(&p0);
            u.y = *reinterpret_cast<uint32_t*>(&p1);
            u.z = *reinterpret_cast<uint32_t*>(&p2);
            u.w = *reinterpret_cast<uint32_t*>(&p3);
            *reinterpret_cast<uint4*>(o + i) = u;
        }
    }
}

// EP_DEMIX column pass: lane = column n0 + lane, the warp's 32 rows in groups of KK (= one
// (bin, slot) row each); arithmetic identical to demix_block_kernel (path.cuh).
template <int KK>
__device__ __forceinline__ void demix_cols(const float* xs, bf16* os, const Epi& ep, int m0, const float* svs, int lane,
                                           float scale2) {
#pragma unroll
    for (int g0 = 0; g0 < 32; g0 += KK) {
        if (m0 + g0 >= ep.M) break;
        float xv[KK];
        float mx = -INFINITY;
#pragma unroll
        for (int k = 0; k < KK; ++k) { xv[k] = xs[(g0 + k) * 33 + lane]; mx = fmaxf(mx, xv[k]); }
        uint32_t den = 0;
#pragma unroll
        for (int k = 0; k < KK; ++k) {
            const float e = ex2_approx((xv[k] - mx) * scale2);
            xv[k] = e;
            den += __float2uint_rn(e * 67108864.0f); // 2^26
        }
        const float rden = 1.0f / (float(den) * (1.0f / 67108864.0f));
        const float sv = svs[g0 / KK]; // S[(bin, slot)][n0 + lane], requested at the chunk start
#pragma unroll
        for (int k = 0; k < KK; ++k) os[(g0 + k) * 32 + lane] = __float2bfloat16_rn((xv[k] * rden) * sv);
    }
}

// EPW epilogue warps: 4 = one per TMEM lane quarter (row statistics need whole rows); 16 = four
// per quarter splitting the columns (EP_DEMIX, whose per-element work would otherwise leave one warp
// per scheduler latency-bound).
template <int BN, int EPW, bool BRES>
__global__ void __launch_bounds__(64 + 32 * EPW, 1)
gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA0, const __grid_constant__ CUtensorMap tmA1,
               const __grid_constant__ CUtensorMap tmB, const Args args) {
    using Lay = SmemLayout<BN, EPW, BRES>;
    constexpr int NST = Lay::NST;
    constexpr int CSTEP = (EPW / 4) * 32; // column stride of one warp's 32-column chunks
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u); // 1 KB aligned, stays in the shared window
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + Lay::BAR_OFF);
    uint64_t* empty = full + NST;
    uint64_t* tfull = empty + NST;
    uint64_t* tempty = tfull + 2;
    uint64_t* bfull = tempty + 2; // BRES: resident B landed
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bfull + 1);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const bool elected = elect_one_sync(); // the lane of the single-thread TMA / MMA issue loops (uniform operands)
    const int kblocks = args.K / BK;

    if (threadIdx.x == 0) {
        for (int s = 0; s < NST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 32 * EPW); }
        mbar_init(bfull, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA0)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA1)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "n"(Lay::TMEM_COLS));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem_base = *tmem_slot;
    griddep_wait(); // (programmatic dependent launch) inputs of the previous kernel visible
    griddep_launch_dependents();

    if (warp == 0) {
        if (elected) {
            int stage = 0;
            uint32_t phase = 0;
            if (BRES) { // the whole B (one N tile) once
                mbar_expect_tx(bfull, kblocks * Lay::B_BYTES);
                for (int kb = 0; kb < kblocks; ++kb) tma_load_2d(smem + kb * Lay::B_BYTES, &tmB, bfull, kb * BK, 0);
            }
            for (int tile = blockIdx.x; tile < args.tiles; tile += gridDim.x) {
                const int mb = tile / args.tiles_n, nb = tile % args.tiles_n;
                for (int kb = 0; kb < kblocks; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* sa = smem + Lay::RING_OFF + stage * Lay::STAGE_BYTES;
                    uint8_t* sb = sa + Lay::A_BYTES;
                    mbar_expect_tx(&full[stage], Lay::STAGE_BYTES);
                    const int k = kb * BK;
                    if (k < args.K0)
                        tma_load_2d(sa, &tmA0, &full[stage], k, mb * BM);
                    else
                        tma_load_2d(sa, &tmA1, &full[stage], k - args.K0, mb * BM);
                    if (!BRES) tma_load_2d(sb, &tmB, &full[stage], k, nb * BN);
                    if (++stage == NST) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (elected) {
            constexpr uint32_t idesc = idesc_bf16(BM, BN);
            int stage = 0, acc = 0;
            uint32_t phase = 0, acc_phase = 0;
            if (BRES) mbar_wait(bfull, 0);
            for (int tile = blockIdx.x; tile < args.tiles; tile += gridDim.x) {
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                fence_after();
                const uint32_t d = tmem_base + uint32_t(acc * BN);
                for (int kb = 0; kb < kblocks; ++kb) {
                    mbar_wait(&full[stage], phase);
                    fence_after();
                    uint8_t* sa = smem + Lay::RING_OFF + stage * Lay::STAGE_BYTES;
                    uint8_t* sb = BRES ? smem + kb * Lay::B_BYTES : sa + Lay::A_BYTES;
                    const uint64_t da = sw128_desc(sa), db = sw128_desc(sb);
#pragma unroll
                    for (int kk = 0; kk < BK / 16; ++kk)
                        mma_bf16(d, da + uint64_t(kk * 2), db + uint64_t(kk * 2), idesc, (kb | kk) != 0);
                    mma_commit(&empty[stage]);
                    if (++stage == NST) { stage = 0; phase ^= 1; }
                }
                mma_commit(&tfull[acc]);
                if (++acc == 2) { acc = 0; acc_phase ^= 1; }
            }
        }
    } else {
        // epilogue: warp w may only touch TMEM lanes [32*(w%4), 32*(w%4)+32)
        const int quarter = warp % 4;
        const int sub = (warp - 2) / 4; // column share of this warp among the EPW / 4 of its quarter
        const int row = quarter * 32 + lane;
        int acc = 0;
        uint32_t acc_phase = 0;
        const Epi& ep = args.ep;
        for (int tile = blockIdx.x; tile < args.tiles; tile += gridDim.x) {
            const int mb = tile / args.tiles_n, nb = tile % args.tiles_n;
            mbar_wait(&tfull[acc], acc_phase);
            fence_after();
            const int m = mb * BM + row;
            const uint32_t tbase = tmem_base + (uint32_t(quarter * 32) << 16) + uint32_t(acc * BN);
            if (EPW <= 4 && ep.kind == EP_LOGITS) {
                // whole row in this tile (N == BN): argmax (lowest index on ties) then
                // kappa = 1 / sum exp((x - max) / tau)   (refine.cpp:61-78)
                float bv = -INFINITY;
                int bi = 0;
                float v[32];
                for (int c0 = 0; c0 < BN; c0 += 32) {
                    tmem_ld32(tbase + c0, v);
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        if (v[i] > bv) { bv = v[i]; bi = c0 + i; }
                    if (ep.out_f && m < ep.M) {
                        float* o = ep.out_f + size_t(m) * ep.ldo + c0;
#pragma unroll
                        for (int i = 0; i < 32; i += 4) *reinterpret_cast<float4*>(o + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
                    }
                }
                // exp((x - max) / tau) = 2^(x c - max c), c = log2(e) / tau: one FFMA + one MUFU.EX2 per logit (expf
                // spends ~10 instructions on range reduction; the 2^-22 relative difference is far below the bf16
                // logit error that the decision checks account for)
                float s = 0.0f;
                const float cexp = ep.inv_tau * 1.4426950408889634f, nb2 = -bv * cexp;
                for (int c0 = 0; c0 < BN; c0 += 32) {
                    tmem_ld32(tbase + c0, v);
#pragma unroll
                    for (int i = 0; i < 32; ++i) s += ex2_approx(fmaf(v[i], cexp, nb2));
                }
                if (m < ep.M) {
                    ep.kappa[m] = 1.0f / s;
                    ep.amax[m] = bi;
                }
            } else if (EPW > 4 && ep.kind == EP_DEMIX) {
                // rows of a (bin, slot) group are K consecutive lanes of this warp (K | 32): write
                // the logits row-wise, then each lane runs one column over the warp's groups
                // (demix_block_kernel's arithmetic), results transposed back for whole-row stores
                float* xs = reinterpret_cast<float*>(smem + Lay::STG_OFF + (warp - 2) * Lay::STG_WARP);
                bf16* os = reinterpret_cast<bf16*>(smem + Lay::STG_OFF + (warp - 2) * Lay::STG_WARP + 32 * 33 * 4);
                const int K = ep.K, m0 = mb * BM + quarter * 32;
                const float scale2 = ep.inv_tau * 1.4426950408889634f;
                float v[32];
                for (int c0 = sub * 32; c0 < BN; c0 += CSTEP) {
                    const int n0 = nb * BN + c0;
                    float svs[8]; // this lane's column of S for the warp's (<= 8) groups, in flight during the row pass
#pragma unroll
                    for (int gi = 0; gi < 8; ++gi)
                        svs[gi] = (gi * K < 32 && m0 + gi * K < ep.M) ? __ldg(ep.S + size_t((m0 + gi * K) / K) * ep.N + n0 + lane) : 0.0f;
                    tmem_ld32(tbase + c0, v);
                    // beta S[(bin, slot), n] is the same for the K rows of a group: a constant shift
                    // inside softmax_k that the max subtraction removes, so only acc is staged
                    if (m < ep.M) {
#pragma unroll
                        for (int i = 0; i < 32; ++i) xs[lane * 33 + i] = v[i];
                    }
                    __syncwarp();
                    switch (K) {
                        case 4: demix_cols<4>(xs, os, ep, m0, svs, lane, scale2); break;
                        case 8: demix_cols<8>(xs, os, ep, m0, svs, lane, scale2); break;
                        case 16: demix_cols<16>(xs, os, ep, m0, svs, lane, scale2); break;
                        default: demix_cols<32>(xs, os, ep, m0, svs, lane, scale2); break;
                    }
                    __syncwarp();
                    bf16* ot = reinterpret_cast<bf16*>(ep.out_t);
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int r = i * 8 + lane / 4;
                        if (m0 + r < ep.M)
                            *reinterpret_cast<uint4*>(ot + size_t(m0 + r) * ep.ldo + n0 + (lane % 4) * 8) =
                                *reinterpret_cast<const uint4*>(os + r * 32 + (lane % 4) * 8);
                    }
                    __syncwarp();
                }
            } else if (EPW <= 4 && ep.kind == EP_STORE && ep.out_t && !ep.out_f) {
                // bf16 store through the warp's staging block: whole 64-byte row segments per lane group
                bf16* os = reinterpret_cast<bf16*>(smem + Lay::STG_OFF + (warp - 2) * Lay::STG_WARP);
                const int m0 = mb * BM + quarter * 32;
                bf16* ot = reinterpret_cast<bf16*>(ep.out_t);
                float v[32];
                for (int c0 = sub * 32; c0 < BN; c0 += CSTEP) {
                    tmem_ld32(tbase + c0, v);
                    const int n0 = nb * BN + c0;
                    if (ep.bias) {
#pragma unroll
                        for (int i = 0; i < 32; i += 4) {
                            const float4 b = __ldg(reinterpret_cast<const float4*>(ep.bias + n0 + i));
                            v[i] += b.x; v[i + 1] += b.y; v[i + 2] += b.z; v[i + 3] += b.w;
                        }
                    }
                    // row `lane`, 16-byte chunk j at (j ^ (lane & 3)) of its 64-byte row: conflict-free
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        uint32_t pk[4];
#pragma unroll
                        for (int t = 0; t < 4; ++t) {
                            __nv_bfloat162 p = __floats2bfloat162_rn(v[j * 8 + 2 * t], v[j * 8 + 2 * t + 1]);
                            pk[t] = *reinterpret_cast<uint32_t*>(&p);
                        }
                        *reinterpret_cast<uint4*>(os + lane * 32 + ((j ^ (lane & 3)) * 8)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                    }
                    __syncwarp();
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int r = i * 8 + lane / 4, j = lane % 4;
                        if (m0 + r < ep.M)
                            *reinterpret_cast<uint4*>(ot + size_t(m0 + r) * ep.ldo + n0 + j * 8) =
                                *reinterpret_cast<const uint4*>(os + r * 32 + ((j ^ (r & 3)) * 8));
                    }
                    __syncwarp();
                }
            } else if (EPW <= 4) {
                float v[32];
                for (int c0 = sub * 32; c0 < BN; c0 += CSTEP) {
                    tmem_ld32(tbase + c0, v);
                    if (m < ep.M) epi_row32(ep, m, nb * BN + c0, v);
                }
            }
            fence_before();
            mbar_arrive(&tempty[acc]);
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
    }
    __syncthreads();
    if (warp == 1) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(Lay::TMEM_COLS));
    }
}

} // namespace tc
} // namespace cider
