// mlp_tc.cuh — fused two-layer map on tcgen05 (BF16 mode):
//
//   Y = epilogue( GELU([A0 | A1] . W1^T + b1) . W2^T + b2 )        (TwoLayerMap, denoiser.cpp:29-39)
//
// used for Module A's gate (epilogue: sigmoid gate mix, denoiser.cpp:156), Module B's check
// aggregator Psi (plain) and fusion map (residual, denoiser.cpp:224). The H-wide hidden layer
// never touches HBM: per 128-row tile the input rows stay resident in SMEM, hidden chunks of
// HC=128 columns are accumulated in TMEM (double-buffered), GELU'd by the epilogue warps and
// written back to SMEM in the SWIZZLE_128B K-major layout, where the second MMA consumes them
// as its A operand while the first MMA of the next chunk already runs.
//
//   warp 0     TMA producer: the row tile once per tile, then W1 / W2 k-blocks through a ring
//              in exactly the order the MMA warp consumes them (W1(0); W1(c+1), W2(c); ...)
//   warp 1     TMEM allocator + single-thread MMA issuer
//   warps 2..5 epilogue: TMEM -> GELU -> swizzled SMEM (hidden), then the final epilogue
//
// TMEM: acc2 = columns [0, D), acc1 buffers at [256, 384) and [384, 512).
#pragma once

#include "gemm_tc.cuh"

namespace cider {
namespace tc {

// tanh-form GELU on the MUFU tanh unit (BF16 mode only; |err| vs the erf form < 1e-3, below
// bf16 resolution — DESIGN.md §3). FP32 mode keeps the reference's erf form.
__device__ __forceinline__ float tanh_approx(float x) {
    float y;
    asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
// sigmoid(x) = 0.5 tanh(x/2) + 0.5: one MUFU op (abs error ~2.5e-4, below the bf16 output rounding)
__device__ __forceinline__ float sigmoid_fast(float x) { return fmaf(0.5f, tanh_approx(0.5f * x), 0.5f); }
// The device GELUs return 2 GELU(x) = x + x tanh(...): the 1/2 lives in the second-layer weights,
// which BF16 mode stores halved (engine.cu upload_model) — exact, one multiply less per element.
__device__ __forceinline__ float gelu_fast(float x) { // 2 GELU(x)
    const float inner = x * fmaf(0.0356774081f, x * x, 0.7978845608f);
    return fmaf(x, tanh_approx(inner), x);
}
// Two lanes at once with the sm_100 packed fp32 ops (FFMA2/FMUL2/FADD2): same arithmetic as
// gelu_fast(x + b) per element, half the FP32 instructions. Returns bf16(2 GELU(x + b)).
__device__ __forceinline__ uint32_t gelu2_bias_bf16(float x0, float x1, float b0, float b1) {
    const float2 x = __fadd2_rn(make_float2(x0, x1), make_float2(b0, b1));
    const float2 p = __ffma2_rn(__fmul2_rn(x, x), make_float2(0.0356774081f, 0.0356774081f), make_float2(0.7978845608f, 0.7978845608f));
    const float2 in = __fmul2_rn(x, p);
    const float2 y = __ffma2_rn(x, make_float2(tanh_approx(in.x), tanh_approx(in.y)), x);
    __nv_bfloat162 r = __floats2bfloat162_rn(y.x, y.y);
    return *reinterpret_cast<uint32_t*>(&r);
}

constexpr int MLP_HC = 128;
constexpr int MLP_THREADS = 320; // producer, MMA, 8 epilogue warps (two per TMEM lane quarter)
constexpr int MLP_EPI = 256;
constexpr int SMEM_LIMIT = 232448; // 227 KB opt-in per block

template <int KIN, int D>
struct MlpLayout {
    static constexpr int KB1 = KIN / 64;                     // k-blocks of the first MMA
    static constexpr int KB2 = MLP_HC / 64;                  // k-blocks of the second MMA
    static constexpr int NB2 = D > 128 ? D / 128 : 1;        // N halves of the second MMA (N <= 128 each)
    static constexpr int N2 = D > 128 ? 128 : D;
    static constexpr int X_BYTES = KB1 * 128 * 64 * 2;       // resident row tile
    static constexpr int H_BYTES = KB2 * 128 * 64 * 2;       // one hidden chunk (32 KB)
    static constexpr int SLOT = 16384;                       // ring slot: one 128x64 bf16 k-block
    static constexpr int FIXED = 1024 + 512;                 // alignment slack + barriers
    static constexpr int NHB = (X_BYTES + 2 * H_BYTES + 4 * SLOT + FIXED <= SMEM_LIMIT) ? 2 : 1;
    static constexpr int NS_RAW = (SMEM_LIMIT - FIXED - X_BYTES - NHB * H_BYTES) / SLOT;
    static constexpr int NS = NS_RAW > 12 ? 12 : NS_RAW;
    static constexpr int H_OFF = X_BYTES;
    static constexpr int R_OFF = H_OFF + NHB * H_BYTES;
    static constexpr int BAR_OFF = R_OFF + NS * SLOT;
    static constexpr int TOTAL = BAR_OFF + 512 + 1024;
    static_assert(NS >= 2, "fused MLP does not fit in shared memory");
    static_assert(D <= 256 && D % 16 == 0, "output width must be <= 256");
};

struct MlpArgs {
    int M, K0, H, tiles;
    const float* b1;
    long long* trace; // diagnostic build (-DCIDER_MLP_TRACE) with CIDER_TRACE_MLP=1: per-chunk clock64 stamps of CTA 0
    Epi ep; // final epilogue (bias = b2)
};

template <int KIN, int D>
__global__ void __launch_bounds__(MLP_THREADS, 1)
mlp_tc_kernel(const __grid_constant__ CUtensorMap tmX0, const __grid_constant__ CUtensorMap tmX1,
              const __grid_constant__ CUtensorMap tmW1, const __grid_constant__ CUtensorMap tmW2, const MlpArgs args_in) {
#ifdef CIDER_MLP_TRACE
    const MlpArgs& args = args_in;
#else
    MlpArgs args = args_in; // (timeline stamps compiled out)
    args.trace = nullptr;
#endif
    using Lay = MlpLayout<KIN, D>;
    constexpr int KB1 = Lay::KB1, KB2 = Lay::KB2, NS = Lay::NS, NHB = Lay::NHB;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u); // 1 KB aligned, stays in the shared window
    uint8_t* xs = smem;
    uint8_t* hs = smem + Lay::H_OFF;
    uint8_t* ring = smem + Lay::R_OFF;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Lay::BAR_OFF);
    uint64_t* x_full = bar;
    uint64_t* x_empty = bar + 1;
    uint64_t* r_full = bar + 2;
    uint64_t* r_empty = r_full + NS;
    uint64_t* a1_full = r_empty + NS;
    uint64_t* a1_empty = a1_full + 2;
    uint64_t* h_full = a1_empty + 2;
    uint64_t* h_empty = h_full + NHB;
    uint64_t* a2_full = h_empty + NHB;
    uint64_t* a2_empty = a2_full + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(a2_empty + 1);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const bool elected = elect_one_sync(); // the lane of the single-thread TMA / MMA issue loops (uniform operands)
    const int NC = args.H / MLP_HC;

    if (threadIdx.x == 0) {
        mbar_init(x_full, 1);
        mbar_init(x_empty, 1);
        for (int s = 0; s < NS; ++s) { mbar_init(&r_full[s], 1); mbar_init(&r_empty[s], 1); }
        for (int b = 0; b < 2; ++b) { mbar_init(&a1_full[b], 1); mbar_init(&a1_empty[b], MLP_EPI); }
        for (int b = 0; b < NHB; ++b) { mbar_init(&h_full[b], MLP_EPI); mbar_init(&h_empty[b], 1); }
        mbar_init(a2_full, 1);
        mbar_init(a2_empty, MLP_EPI);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmW1)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmW2)) : "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (elected) {
            int slot = 0;
            uint32_t rph = 0, xph = 0;
            auto load_w = [&](const CUtensorMap* map, int x, int y, int bytes) {
                mbar_wait(&r_empty[slot], rph ^ 1);
                mbar_expect_tx(&r_full[slot], bytes);
                tma_load_2d(ring + slot * Lay::SLOT, map, &r_full[slot], x, y);
                if (++slot == NS) { slot = 0; rph ^= 1; }
            };
            auto load_w1 = [&](int c) {
                for (int kb = 0; kb < KB1; ++kb) load_w(&tmW1, kb * 64, c * MLP_HC, MLP_HC * 64 * 2);
            };
            auto load_w2 = [&](int c) {
                for (int kb = 0; kb < KB2; ++kb)
                    for (int nh = 0; nh < Lay::NB2; ++nh) load_w(&tmW2, c * MLP_HC + kb * 64, nh * 128, Lay::N2 * 64 * 2);
            };
            for (int tile = blockIdx.x; tile < args.tiles; tile += gridDim.x) {
                mbar_wait(x_empty, xph ^ 1);
                xph ^= 1;
                mbar_expect_tx(x_full, Lay::X_BYTES);
                for (int kb = 0; kb < KB1; ++kb) {
                    const int k = kb * 64;
                    if (k < args.K0) tma_load_2d(xs + kb * 16384, &tmX0, x_full, k, tile * 128);
                    else tma_load_2d(xs + kb * 16384, &tmX1, x_full, k - args.K0, tile * 128);
                }
                load_w1(0);
                for (int c = 0; c < NC; ++c) {
                    if (c + 1 < NC) load_w1(c + 1);
                    load_w2(c);
                }
            }
        }
    } else if (warp == 1) {
        if (elected) {
            constexpr uint32_t id1 = idesc_bf16(128, MLP_HC);
            constexpr uint32_t id2 = idesc_bf16(128, Lay::N2);
            int slot = 0;
            uint32_t rph = 0, xph = 0, a2ph = 0;
            uint32_t a1ph[2] = {0, 0}, hph[NHB];
            for (int b = 0; b < NHB; ++b) hph[b] = 0;
            auto mma1 = [&](int c) {
                const int b = c & 1;
                mbar_wait(&a1_empty[b], a1ph[b] ^ 1);
                a1ph[b] ^= 1;
                fence_after();
                const uint32_t d = tmem + 256 + b * MLP_HC;
                for (int kb = 0; kb < KB1; ++kb) {
                    mbar_wait(&r_full[slot], rph);
                    fence_after();
                    const uint64_t da = sw128_desc(xs + kb * 16384), db = sw128_desc(ring + slot * Lay::SLOT);
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) mma_bf16(d, da + uint64_t(kk * 2), db + uint64_t(kk * 2), id1, (kb | kk) != 0);
                    mma_commit(&r_empty[slot]);
                    if (++slot == NS) { slot = 0; rph ^= 1; }
                }
                mma_commit(&a1_full[b]);
            };
            for (int tile = blockIdx.x; tile < args.tiles; tile += gridDim.x) {
                mbar_wait(x_full, xph);
                xph ^= 1;
                fence_after();
                mma1(0);
                if (NC == 1) mma_commit(x_empty);
                for (int c = 0; c < NC; ++c) {
                    if (c + 1 < NC) {
                        mma1(c + 1);
                        if (c + 1 == NC - 1) mma_commit(x_empty); // row tile no longer read
                    }
                    const int hb = c % NHB;
                    if (args.trace && blockIdx.x == 0 && tile == 0) args.trace[c * 8 + 0] = clock64();
                    mbar_wait(&h_full[hb], hph[hb]);
                    hph[hb] ^= 1;
                    fence_after();
                    if (args.trace && blockIdx.x == 0 && tile == 0) args.trace[c * 8 + 1] = clock64();
                    if (c == 0) {
                        mbar_wait(a2_empty, a2ph ^ 1);
                        a2ph ^= 1;
                        fence_after();
                    }
                    for (int kb = 0; kb < KB2; ++kb) {
                        const uint64_t da = sw128_desc(hs + hb * Lay::H_BYTES + kb * 16384);
                        for (int nh = 0; nh < Lay::NB2; ++nh) {
                            mbar_wait(&r_full[slot], rph);
                            fence_after();
                            const uint64_t db = sw128_desc(ring + slot * Lay::SLOT);
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk)
                                mma_bf16(tmem + nh * 128, da + uint64_t(kk * 2), db + uint64_t(kk * 2), id2, (c | kb | kk) != 0);
                            mma_commit(&r_empty[slot]);
                            if (++slot == NS) { slot = 0; rph ^= 1; }
                        }
                    }
                    mma_commit(&h_empty[hb]);
                }
                mma_commit(a2_full);
            }
        }
    } else {
        // 8 epilogue warps: warp w touches TMEM lane quarter (w % 4); the two warps of a quarter
        // split every chunk's columns in halves, so each SM sub-partition runs two epilogue warps.
        const int quarter = warp % 4;
        const int half = (warp - 2) / 4;
        const int row = quarter * 32 + lane;
        const uint32_t lane_off = uint32_t(quarter * 32) << 16;
        uint32_t e1ph[2] = {0, 0}, ehph[NHB], e2ph = 0;
        for (int b = 0; b < NHB; ++b) ehph[b] = 0;
        const Epi& ep = args.ep;
        for (int tile = blockIdx.x; tile < args.tiles; tile += gridDim.x) {
            for (int c = 0; c < NC; ++c) {
                const int b = c & 1, hb = c % NHB;
                const float* b1 = args.b1 + c * MLP_HC + half * 64;
                float4 bias4[16]; // this warp's 64 bias values, fetched before any wait
#pragma unroll
                for (int q = 0; q < 16; ++q) bias4[q] = __ldg(reinterpret_cast<const float4*>(b1) + q);
                const bool tr = args.trace && blockIdx.x == 0 && tile == 0 && warp == 2 && lane == 0;
                if (tr) args.trace[c * 8 + 2] = clock64();
                mbar_wait(&a1_full[b], e1ph[b]);
                e1ph[b] ^= 1;
                if (tr) args.trace[c * 8 + 3] = clock64();
                mbar_wait(&h_empty[hb], ehph[hb] ^ 1);
                ehph[hb] ^= 1;
                fence_after();
                uint8_t* hrow = hs + hb * Lay::H_BYTES + half * 16384 + row * 128; // k-block = half
#pragma unroll
                for (int g = 0; g < 2; ++g) {
                    float v[32];
                    tmem_ld32(tmem + lane_off + 256 + b * MLP_HC + half * 64 + g * 32, v);
                    uint32_t pk[16];
#pragma unroll
                    for (int i = 0; i < 32; i += 4) {
                        const float4 bb = bias4[g * 8 + i / 4];
                        __nv_bfloat162 p0 = __floats2bfloat162_rn(gelu_fast(v[i] + bb.x), gelu_fast(v[i + 1] + bb.y));
                        __nv_bfloat162 p1 = __floats2bfloat162_rn(gelu_fast(v[i + 2] + bb.z), gelu_fast(v[i + 3] + bb.w));
                        pk[i / 2] = *reinterpret_cast<uint32_t*>(&p0);
                        pk[i / 2 + 1] = *reinterpret_cast<uint32_t*>(&p1);
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int chunk = (g * 4 + q) ^ (row & 7);
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(smem_u32(hrow + chunk * 16)),
                                     "r"(pk[4 * q]), "r"(pk[4 * q + 1]), "r"(pk[4 * q + 2]), "r"(pk[4 * q + 3])
                                     : "memory");
                    }
                }
                fence_before();
                mbar_arrive(&a1_empty[b]);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                mbar_arrive(&h_full[hb]);
                if (tr) args.trace[c * 8 + 4] = clock64();
            }
            // Final epilogue, transposed through the (now idle) hidden buffer so that global
            // traffic is lane-contiguous: 64-column fp32 slabs, row-per-thread in (from TMEM),
            // row-per-warp out (z / e reads and the output writes coalesce).
            float* slab = reinterpret_cast<float*>(hs);
            const int m0 = tile * 128;
            const int wq = warp - 2; // rows [16 wq, 16 wq + 16) of every slab
            mbar_wait(a2_full, e2ph);
            e2ph ^= 1;
            fence_after();
#pragma unroll 1
            for (int n0 = 0; n0 < D; n0 += 64) {
                uint32_t zr[16], er[16];
                if (ep.kind == EP_GATE || ep.kind == EP_RESID) {
#pragma unroll
                    for (int rr = 0; rr < 16; ++rr) {
                        const int m = m0 + wq * 16 + rr;
                        const size_t off = size_t(m < ep.M ? m : 0) * ep.ldz + n0 + 2 * lane;
                        zr[rr] = __ldg(reinterpret_cast<const unsigned int*>(ep.zb + off));
                        er[rr] = ep.kind == EP_GATE ? __ldg(reinterpret_cast<const unsigned int*>(ep.eb + off)) : 0u;
                    }
                }
                float4 bias4[8];
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    bias4[q] = ep.bias ? __ldg(reinterpret_cast<const float4*>(ep.bias + n0 + half * 32) + q)
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
                {
                    float v[32];
                    tmem_ld32(tmem + lane_off + n0 + half * 32, v);
                    if (n0 + 64 >= D) {
                        fence_before();
                        mbar_arrive(a2_empty); // accumulator drained: next tile's MMA2 may start
                    }
#pragma unroll
                    for (int i = 0; i < 32; i += 4) {
                        const int cidx = (half * 32 + i) / 4; // 16-byte chunk 0..15 of the 256-byte row
                        const float4 bb = bias4[i / 4];
                        float4 q = make_float4(v[i] + bb.x, v[i + 1] + bb.y, v[i + 2] + bb.z, v[i + 3] + bb.w);
                        *reinterpret_cast<float4*>(slab + row * 64 + ((cidx ^ (row & 15)) * 4)) = q;
                    }
                }
                asm volatile("bar.sync 1, 256;" ::: "memory");
#pragma unroll
                for (int rr = 0; rr < 16; ++rr) {
                    const int r = wq * 16 + rr;
                    const int m = m0 + r;
                    if (m >= ep.M) break;
                    const int cidx = lane / 2;
                    const float2 a = *reinterpret_cast<const float2*>(slab + r * 64 + ((cidx ^ (r & 15)) * 4) + (lane & 1) * 2);
                    const int n = n0 + 2 * lane;
                    float o0 = a.x, o1 = a.y;
                    if (ep.kind == EP_GATE) {
                        const float2 z = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&zr[rr]));
                        const float2 e = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&er[rr]));
                        const float g0 = sigmoid_f(o0), g1 = sigmoid_f(o1);
                        o0 = g0 * z.x + (1.0f - g0) * e.x;
                        o1 = g1 * z.y + (1.0f - g1) * e.y;
                    } else if (ep.kind == EP_RESID) {
                        const float2 z = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&zr[rr]));
                        o0 += z.x;
                        o1 += z.y;
                    }
                    if (ep.out_f) *reinterpret_cast<float2*>(ep.out_f + size_t(m) * ep.ldo + n) = make_float2(o0, o1);
                    if (ep.out_t)
                        *reinterpret_cast<__nv_bfloat162*>(reinterpret_cast<bf16*>(ep.out_t) + size_t(m) * ep.ldo + n) =
                            __floats2bfloat162_rn(o0, o1);
                }
                asm volatile("bar.sync 1, 256;" ::: "memory");
            }
        }
    }
    __syncthreads();
    if (warp == 1) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

} // namespace tc
} // namespace cider
