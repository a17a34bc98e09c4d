// mlp_tc2.cuh — the fused two-layer map on a CTA PAIR (tcgen05.mma.cta_group::2, M = 256).
//
// Same math and epilogues as mlp_tc.cuh, but the two SMs of a cluster share one 256-row MMA:
// each CTA keeps its own 128 input rows, hidden chunks and accumulator lanes, and loads only HALF
// of every weight k-block (the N-half the pair's MMA reads from it). Per SM this halves the
// weight bytes that must stream from L2 per unit of tensor work — the resource the 1-SM kernel
// is starved of (tests/trace_mlp.py: the MMA thread waited on the weight ring 5-7k cycles per
// chunk).
//
// Protocol (leader = cluster rank 0):
//   * both CTAs allocate 512 TMEM columns with tcgen05.alloc.cta_group::2 (same warp, same slot);
//   * both producers TMA their own rows / weight halves with the .cta_group::2 form, signalling
//     the LEADER's full barriers; only the leader arms them (arrive.expect_tx, both halves' bytes);
//   * only the leader issues MMAs; its commits multicast to the barrier copies in both CTAs;
//   * epilogue warps of both CTAs release TMEM / hidden buffers by remote-arriving (one elected
//     lane per warp) on the leader's empty/full barriers.
// The hidden chunk never goes to SMEM at all: the epilogue GELUs the fp32 accumulator and packs the
// bf16 result IN PLACE into the same TMEM columns (each warp only overwrites columns it already
// read), and the second MMA takes its A operand straight from TMEM (tcgen05.mma [d], [a_tmem], b).
// SMEM then holds only the resident row tile and a deep weight ring.
// Ring slot = 16 KB: a W2 half k-block (D/2 x 64) or two W1 half k-blocks (HC/2 x 64 each).
#pragma once

#include "mlp_tc.cuh"

namespace cider {
namespace tc {

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t mapa_u32(uint32_t local_addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local_addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx_cl(uint32_t cl_addr, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(cl_addr), "r"(bytes)
                 : "memory");
}
// Remote (peer-CTA) arrive with the default semantics, as CUTLASS's ClusterBarrier::arrive does; an
// explicit .release.cluster costs a cluster-scope fence (~900 cycles) per arrive.
__device__ __forceinline__ void mbar_arrive_cl(uint32_t cl_addr) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cl_addr) : "memory");
}
__device__ __forceinline__ void tma_load_2d_2sm(void* dst, const CUtensorMap* map, uint32_t cl_bar, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(cl_bar), "r"(x), "r"(y)
        : "memory");
}
// 3-D box (64 cols x rows x kblocks): two adjacent 64-column k-blocks of the same weight rows in
// ONE TMA (the TMA unit completes roughly one box per ~330 cycles per SM whatever its size, so
// 16 KB boxes double the weight stream of 8 KB ones — tools/tma_bench.cu).
__device__ __forceinline__ void tma_load_3d_2sm(void* dst, const CUtensorMap* map, uint32_t cl_bar, int x, int y, int z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(cl_bar), "r"(x), "r"(y), "r"(z)
        : "memory");
}
__device__ __forceinline__ void mma_bf16_2sm(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_bf16_2sm_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
        "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}
__device__ __forceinline__ void mma_commit_2sm(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(uint16_t(3))
        : "memory");
}

template <int KIN, int D>
struct Mlp2Layout {
    static constexpr int KB1 = KIN / 64;
    static constexpr int KB2 = MLP_HC / 64;
    static constexpr int W1_HALF = (MLP_HC / 2) * 64 * 2;   // 8 KB: this CTA's 64 rows of a W1 k-block
    static constexpr int W2_HALF = (D / 2) * 64 * 2;        // this CTA's D/2 rows of a W2 k-block
    static constexpr int SLOT = 16384;
    static constexpr int W1_PER_SLOT = SLOT / W1_HALF;       // 2
    static constexpr int X_BYTES = KB1 * 128 * 64 * 2;
    static constexpr int FIXED = 1024 + 512;
    static constexpr int NS_RAW = (SMEM_LIMIT - FIXED - X_BYTES) / SLOT;
    static constexpr int NS = NS_RAW > 16 ? 16 : NS_RAW;
    static constexpr int R_OFF = X_BYTES;
    static constexpr int BAR_OFF = R_OFF + NS * SLOT;
    static constexpr int TOTAL = BAR_OFF + 512 + 1024;
    static_assert(NS >= 4, "fused MLP (2-SM) does not fit in shared memory");
    static_assert(D % 32 == 0 && D <= 256 && W2_HALF <= SLOT, "output width must be <= 256");
    static_assert(KB1 % W1_PER_SLOT == 0, "input width must be a multiple of 128");
};

template <int KIN, int D>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(MLP_THREADS, 1)
mlp_tc2_kernel(const __grid_constant__ CUtensorMap tmX0, const __grid_constant__ CUtensorMap tmX1,
               const __grid_constant__ CUtensorMap tmW1, const __grid_constant__ CUtensorMap tmW2, const MlpArgs args) {
    using Lay = Mlp2Layout<KIN, D>;
    constexpr int KB1 = Lay::KB1, KB2 = Lay::KB2, NS = Lay::NS;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* xs = smem;
    uint8_t* ring = smem + Lay::R_OFF;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Lay::BAR_OFF);
    uint64_t* x_full = bar;
    uint64_t* x_empty = bar + 1;
    uint64_t* r_full = bar + 2;
    uint64_t* r_empty = r_full + NS;
    uint64_t* a1_full = r_empty + NS;   // [2] first-layer accumulator ready
    uint64_t* h_full = a1_full + 2;     // [2] bf16 hidden packed in TMEM (leader copy counts both CTAs)
    uint64_t* a2_full = h_full + 2;
    uint64_t* a2_empty = a2_full + 1;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(a2_empty + 1);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    const int pair = blockIdx.x / 2, npairs = gridDim.x / 2;
    const int NC = args.H / MLP_HC;
    constexpr int EPI_ARRIVALS = 2 * 8; // one elected lane per epilogue warp, both CTAs

    // gate / fusion epilogues read z (and e) back from the resident row tile X, so X is released by
    // the last MMA1's commit AND by the 8 epilogue warps once their final epilogue is done
    const bool epi_reads_x = args.ep.kind == EP_GATE || args.ep.kind == EP_RESID;
    if (threadIdx.x == 0) {
        mbar_init(x_full, 1);
        mbar_init(x_empty, epi_reads_x ? 1 + 8 : 1);
        for (int s = 0; s < NS; ++s) { mbar_init(&r_full[s], 1); mbar_init(&r_empty[s], 1); }
        for (int b = 0; b < 2; ++b) { mbar_init(&a1_full[b], 1); mbar_init(&h_full[b], EPI_ARRIVALS); }
        mbar_init(a2_full, 1);
        mbar_init(a2_empty, EPI_ARRIVALS);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    fence_before();
    cluster_sync_all(); // barriers of both CTAs initialised before any remote signal
    fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t L_x_full = mapa_u32(smem_u32(x_full), 0);
    const uint32_t L_r_full0 = mapa_u32(smem_u32(&r_full[0]), 0);
    const uint32_t L_h_full0 = mapa_u32(smem_u32(&h_full[0]), 0);
    const uint32_t L_a2_empty = mapa_u32(smem_u32(a2_empty), 0);

    if (warp == 0) {
        if (lane == 0) {
            int slot = 0;
            uint32_t rph = 0, xph = 0;
            auto next = [&] { if (++slot == NS) { slot = 0; rph ^= 1; } };
            int nload = 0;
            const bool trp = args.trace && blockIdx.x == 0;
            auto acquire = [&](uint32_t bytes_both) {
                if (trp && nload < 40) args.trace[512 + nload * 4 + 0] = clock64();
                mbar_wait(&r_empty[slot], rph ^ 1);
                if (trp && nload < 40) args.trace[512 + nload * 4 + 1] = clock64();
                if (leader) mbar_expect_tx(&r_full[slot], bytes_both); // the leader arms its own barrier
                if (trp && nload < 40) args.trace[512 + nload * 4 + 2] = clock64();
            };
            auto issued = [&] {
                if (trp && nload < 40) args.trace[512 + nload * 4 + 3] = clock64();
                ++nload;
            };
            auto load_w1 = [&](int c) { // tmW1 is 3-D: {64 cols, H rows, KIN/64 k-blocks}
                for (int kb = 0; kb < KB1; kb += Lay::W1_PER_SLOT) {
                    acquire(2 * Lay::W1_PER_SLOT * Lay::W1_HALF);
                    tma_load_3d_2sm(ring + slot * Lay::SLOT, &tmW1, L_r_full0 + slot * 8, 0,
                                    c * MLP_HC + int(rank) * (MLP_HC / 2), kb);
                    issued();
                    next();
                }
            };
            auto load_w2 = [&](int c) {
                for (int kb = 0; kb < KB2; ++kb) {
                    acquire(2 * Lay::W2_HALF);
                    tma_load_2d_2sm(ring + slot * Lay::SLOT, &tmW2, L_r_full0 + slot * 8, c * MLP_HC + kb * 64,
                                    int(rank) * (D / 2));
                    issued();
                    next();
                }
            };
            for (int tile = pair; tile < args.tiles; tile += npairs) {
                mbar_wait(x_empty, xph ^ 1);
                xph ^= 1;
                if (leader) mbar_expect_tx(x_full, 2 * Lay::X_BYTES);
                const int row0 = tile * 256 + int(rank) * 128;
                for (int kb = 0; kb < KB1; ++kb) {
                    const int k = kb * 64;
                    if (k < args.K0) tma_load_2d_2sm(xs + kb * 16384, &tmX0, L_x_full, k, row0);
                    else tma_load_2d_2sm(xs + kb * 16384, &tmX1, L_x_full, k - args.K0, row0);
                }
                // consumption order of the MMA warp: W1(0), W1(1), then W2(c), W1(c+2) ...
                load_w1(0);
                if (NC > 1) load_w1(1);
                for (int c = 0; c < NC; ++c) {
                    load_w2(c);
                    if (c + 2 < NC) load_w1(c + 2);
                }
            }
        }
    } else if (warp == 1) {
        if (leader && lane == 0) {
            constexpr uint32_t id1 = idesc_bf16(256, MLP_HC);
            constexpr uint32_t id2 = idesc_bf16(256, D);
            int slot = 0;
            uint32_t rph = 0, xph = 0, a2ph = 0;
            uint32_t hph[2] = {0, 0};
            int ncons = 0;
            const bool trm = args.trace && blockIdx.x == 0;
            auto next = [&] {
                if (trm && ncons < 40) args.trace[768 + ncons * 4 + 2] = clock64(); // slot's MMAs issued
                ++ncons;
                if (++slot == NS) { slot = 0; rph ^= 1; }
            };
            auto wfull = [&] {
                if (trm && ncons < 40) args.trace[768 + ncons * 4 + 0] = clock64();
                mbar_wait(&r_full[slot], rph);
                if (trm && ncons < 40) args.trace[768 + ncons * 4 + 1] = clock64();
            };
            auto mma1 = [&](int c) { // acc1[c&1] = X . W1(c)^T   (both operands in SMEM)
                const uint32_t d = tmem + 256 + (c & 1) * MLP_HC;
                for (int kb = 0; kb < KB1; kb += Lay::W1_PER_SLOT) {
                    wfull();
                    fence_after();
                    for (int j = 0; j < Lay::W1_PER_SLOT; ++j) {
                        const uint64_t da = sw128_desc(xs + (kb + j) * 16384);
                        const uint64_t db = sw128_desc(ring + slot * Lay::SLOT + j * Lay::W1_HALF);
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)
                            mma_bf16_2sm(d, da + uint64_t(kk * 2), db + uint64_t(kk * 2), id1, ((kb + j) | kk) != 0);
                    }
                    mma_commit_2sm(&r_empty[slot]);
                    next();
                }
                mma_commit_2sm(&a1_full[c & 1]);
            };
            for (int tile = pair; tile < args.tiles; tile += npairs) {
                mbar_wait(x_full, xph);
                xph ^= 1;
                fence_after();
                mma1(0);
                if (NC > 1) mma1(1);
                if (NC <= 2) mma_commit_2sm(x_empty);
                for (int c = 0; c < NC; ++c) {
                    const int b = c & 1;
                    const bool tr = args.trace && blockIdx.x == 0 && tile == pair;
                    if (tr) args.trace[c * 8 + 0] = clock64();
                    mbar_wait(&h_full[b], hph[b]); // GELU(c) packed into acc1[b]
                    hph[b] ^= 1;
                    fence_after();
                    if (tr) args.trace[c * 8 + 1] = clock64();
                    if (c == 0) {
                        mbar_wait(a2_empty, a2ph ^ 1);
                        a2ph ^= 1;
                        fence_after();
                    }
                    // acc2 += H(c) . W2(c)^T with A = bf16 hidden in TMEM: k-steps 0-3 at cols
                    // [0,32), 4-7 at [64,96) of the chunk's buffer (see the epilogue packing)
                    const uint32_t a_base = tmem + 256 + b * MLP_HC;
                    for (int kb = 0; kb < KB2; ++kb) {
                            mbar_wait(&r_full[slot], rph);
                        fence_after();
                        const uint64_t db = sw128_desc(ring + slot * Lay::SLOT);
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)
                            mma_bf16_2sm_ts(tmem, a_base + kb * 64 + kk * 8, db + uint64_t(kk * 2), id2, (c | kb | kk) != 0);
                        mma_commit_2sm(&r_empty[slot]);
                        next();
                    }
                    if (c + 2 < NC) { // in-order tensor pipe: MMA2(c) has read acc1[b] before this overwrites it
                        mma1(c + 2);
                        if (c + 2 == NC - 1) mma_commit_2sm(x_empty);
                    }
                    if (tr) args.trace[c * 8 + 5] = clock64();
                }
                mma_commit_2sm(a2_full);
            }
        }
    } else {
        // 8 epilogue warps: TMEM lane quarter = warp % 4; the two warps of a quarter own the two
        // 64-column halves of every chunk (and of the output).
        const int quarter = warp % 4;
        const int half = (warp - 2) / 4;
        const int row = quarter * 32 + lane;
        const uint32_t lane_off = uint32_t(quarter * 32) << 16;
        uint32_t e1ph[2] = {0, 0}, e2ph = 0;
        const Epi& ep = args.ep;
        auto release = [&](uint32_t leader_bar) { // elected remote arrive once the whole warp is done
            __syncwarp();
            if (lane == 0) mbar_arrive_cl(leader_bar);
        };
        for (int tile = pair; tile < args.tiles; tile += npairs) {
            for (int c = 0; c < NC; ++c) {
                const int b = c & 1;
                const float* b1 = args.b1 + c * MLP_HC + half * 64;
                float4 bias4[16];
#pragma unroll
                for (int q = 0; q < 16; ++q) bias4[q] = __ldg(reinterpret_cast<const float4*>(b1) + q);
                const bool tr = args.trace && blockIdx.x == 0 && tile == pair && warp == 2 && lane == 0;
                if (tr) args.trace[c * 8 + 2] = clock64();
                mbar_wait(&a1_full[b], e1ph[b]);
                e1ph[b] ^= 1;
                fence_after();
                if (tr) args.trace[c * 8 + 3] = clock64();
                // fp32 columns [64 half, 64 half + 64) -> GELU -> bf16 pairs packed into the first 32
                // of those columns (32 g .. ): every column is read before it is overwritten.
                const uint32_t base = tmem + lane_off + 256 + b * MLP_HC + half * 64;
#pragma unroll
                for (int g = 0; g < ((args.dbg & 1) ? 0 : 2); ++g) {
                    float v[32];
                    tmem_ld32(base + g * 32, v);
                    uint32_t pk[16];
#pragma unroll
                    for (int i = 0; i < 32; i += 4) {
                        const float4 bb = bias4[g * 8 + i / 4];
                        __nv_bfloat162 p0 = __floats2bfloat162_rn(gelu_fast(v[i] + bb.x), gelu_fast(v[i + 1] + bb.y));
                        __nv_bfloat162 p1 = __floats2bfloat162_rn(gelu_fast(v[i + 2] + bb.z), gelu_fast(v[i + 3] + bb.w));
                        pk[i / 2] = *reinterpret_cast<uint32_t*>(&p0);
                        pk[i / 2 + 1] = *reinterpret_cast<uint32_t*>(&p1);
                    }
                    tmem_st16(base + g * 16, pk);
                }
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                fence_before();
                release(L_h_full0 + b * 8);
                if (tr) args.trace[c * 8 + 4] = clock64();
            }
            // final epilogue straight from TMEM: this thread's row, this warp's half of D in
            // 32-column groups; z (and e) come from the row tile X still resident in SMEM
            // (SWIZZLE_128B K-major: 16-byte chunk c of row r sits at chunk c ^ (r & 7)).
            const int m = tile * 256 + int(rank) * 128 + row;
            const bool live = m < ep.M;
            const int ncol = D / 2;
            const int c0 = half * ncol;
            auto xrow_chunk = [&](int col) -> uint4 { // 8 bf16 at columns [col, col+8) of this row of X
                const int kb = col / 64, ch = (col % 64) / 8;
                return *reinterpret_cast<const uint4*>(xs + kb * 16384 + row * 128 + ((ch ^ (row & 7)) * 16));
            };
            mbar_wait(a2_full, e2ph);
            e2ph ^= 1;
            fence_after();
#pragma unroll 1
            for (int g = 0; g < ncol / 32; ++g) {
                const int n0 = c0 + g * 32;
                float v[32];
                tmem_ld32(tmem + lane_off + n0, v);
                if (g + 1 == ncol / 32) {
                    fence_before();
                    release(L_a2_empty); // accumulator drained: next tile's MMA2 may start
                }
                uint4 zq[4], eq[4];
                if (epi_reads_x) {
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        zq[q] = xrow_chunk(n0 + q * 8);
                        if (ep.kind == EP_GATE) eq[q] = xrow_chunk(D + n0 + q * 8);
                    }
                }
                if (!live) continue;
#pragma unroll
                for (int i = 0; i < 32; i += 4) {
                    const float4 bb = ep.bias ? __ldg(reinterpret_cast<const float4*>(ep.bias + n0 + i)) : make_float4(0.f, 0.f, 0.f, 0.f);
                    v[i] += bb.x; v[i + 1] += bb.y; v[i + 2] += bb.z; v[i + 3] += bb.w;
                }
                if (epi_reads_x) {
                    const bf16* zz = reinterpret_cast<const bf16*>(zq);
                    const bf16* ee = reinterpret_cast<const bf16*>(eq);
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const float z = __bfloat162float(zz[i]);
                        if (ep.kind == EP_GATE) {
                            const float gt = sigmoid_f(v[i]);
                            v[i] = gt * z + (1.0f - gt) * __bfloat162float(ee[i]);
                        } else {
                            v[i] += z;
                        }
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
            if (epi_reads_x) { // this warp no longer reads X: the producer may load the next tile
                __syncwarp();
                if (lane == 0) mbar_arrive(x_empty);
            }
        }
    }
    fence_before();
    cluster_sync_all(); // no CTA leaves while its peer may still signal its barriers or read its smem
    if (warp == 1) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

} // namespace tc
} // namespace cider
