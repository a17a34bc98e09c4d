// gemm_grp.cuh — grouped tcgen05 GEMM for Module B's coefficient actions when Q >= D (BF16 mode).
//
// T_alpha(x) = W^T Pi_alpha W x (denoiser.cpp:162-179) is linear in x, so for each GF(Q)
// coefficient the D x D matrix T_alpha = W^T P_alpha W is precomputed once and Module B's
// projection / permutation / back-projection chains become two grouped GEMMs:
//
//   normalise  (group = edge e):  N[(b,e,k)] = z~[(b, slot_e, k)] . T_{alpha_e}
//   messages   (group = slot s):  acc[(b,s,k)] = sum_{e in s, ascending check} mapped[(b,e,k)] . T_{alpha_e^-1}
//
// The message GEMM concatenates the slot's edges along K, so the per-slot sum happens inside the
// tensor core in a fixed order (no atomics). A rows are gathered by 3-D TMA boxes
// {64 cols, K rows, 128/K bins} straight out of the [bin][slot|edge][row] layouts; B tiles come
// from a 3-D map over the T table [alpha][n][k]. Same warp roles / pipeline as gemm_tc.cuh.
// Tiles run m-tile-major (all groups of one 128-row block back to back, groups sorted so edges of
// one slot are adjacent): the A rows a slot shares among its edges are L2 hits, and the <= 24 MB
// of T matrices stay L2-resident.
#pragma once

#include "gemm_tc.cuh"
#include "mlp_tc2.cuh" // 2-SM TMA / MMA / commit helpers

namespace cider {
namespace tc {

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y, int z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z)
        : "memory");
}

struct GrpArgs {
    int groups, mtiles, bins, K, bb;  // bb = bins per 128-row tile (K * bb <= 128)
    int kb_per_seg;                   // D / 64
    int max_seg;                      // segments (edges) per group
    const int* seg_count;             // [groups]
    const int* seg_arow;              // [groups][max_seg]: A row block (slot or edge index)
    const int* seg_alpha;             // [groups][max_seg]: T-table index
    int out_rows_per_bin;             // L (site output) or E (edge output)
    const int* out_row;               // [groups]: output row block (edge or slot index)
    int D;
    bf16* out_t;                      // bf16 output [bins * out_rows_per_bin * K x D]
    float* out_f;                     // optional fp32 copy
};

constexpr int GRP_THREADS = 320; // producer, MMA, 8 epilogue warps (two per TMEM lane quarter)

__global__ void __launch_bounds__(GRP_THREADS, 1)
gemm_grp_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmT, const GrpArgs args) {
    constexpr int BN = 256;
    using Lay = SmemLayout<BN, 0>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u); // 1 KB aligned, stays in the shared window
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + Lay::BAR_OFF);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const bool elected = elect_one_sync(); // the lane of the single-thread TMA / MMA issue loops (uniform operands)
    const int tiles = args.groups * args.mtiles;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 256); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
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
    const int a_bytes = args.K * args.bb * 128; // the A box actually filled (<= 16 KB)

    if (warp == 0) {
        if (elected) {
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
                const int g = tile % args.groups, mt = tile / args.groups; // m-tile major: L2 reuse of A rows
                const int nseg = args.seg_count[g];
                for (int sg = 0; sg < nseg; ++sg) {
                    const int arow = args.seg_arow[g * args.max_seg + sg];
                    const int alpha = args.seg_alpha[g * args.max_seg + sg];
                    for (int kk = 0; kk < args.kb_per_seg; ++kk) {
                        mbar_wait(&empty[stage], phase ^ 1);
                        uint8_t* sa = smem + stage * Lay::STAGE_BYTES;
                        uint8_t* sb = sa + Lay::A_BYTES;
                        mbar_expect_tx(&full[stage], a_bytes + Lay::B_BYTES);
                        tma_load_3d(sa, &tmA, &full[stage], kk * 64, arow * args.K, mt * args.bb);
                        tma_load_3d(sb, &tmT, &full[stage], kk * 64, 0, alpha);
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (elected) {
            constexpr uint32_t idesc = idesc_bf16(BM, BN);
            int stage = 0, acc = 0;
            uint32_t phase = 0, acc_phase = 0;
            for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
                const int g = tile % args.groups;
                const int kblocks = args.seg_count[g] * args.kb_per_seg;
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                fence_after();
                const uint32_t d = tmem_base + uint32_t(acc * BN);
                for (int kb = 0; kb < kblocks; ++kb) {
                    mbar_wait(&full[stage], phase);
                    fence_after();
                    uint8_t* sa = smem + stage * Lay::STAGE_BYTES;
                    uint8_t* sb = sa + Lay::A_BYTES;
                    const uint64_t da = sw128_desc(sa), db = sw128_desc(sb);
#pragma unroll
                    for (int kk = 0; kk < BK / 16; ++kk)
                        mma_bf16(d, da + uint64_t(kk * 2), db + uint64_t(kk * 2), idesc, (kb | kk) != 0);
                    mma_commit(&empty[stage]);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                mma_commit(&tfull[acc]);
                if (++acc == 2) { acc = 0; acc_phase ^= 1; }
            }
        }
    } else {
        const int quarter = warp % 4;
        const int half = (warp - 2) / 4; // the two warps of a lane quarter split the columns
        const int row = quarter * 32 + lane;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
            const int g = tile % args.groups, mt = tile / args.groups;
            mbar_wait(&tfull[acc], acc_phase);
            fence_after();
            const int b = mt * args.bb + row / args.K, k = row % args.K;
            const bool live = row < args.K * args.bb && b < args.bins;
            const size_t orow = (size_t(b) * args.out_rows_per_bin + args.out_row[g]) * args.K + k;
            const uint32_t tbase = tmem_base + (uint32_t(quarter * 32) << 16) + uint32_t(acc * BN);
            const int cw = args.D / 2;
            for (int c0 = half * cw; c0 < (half + 1) * cw; c0 += 32) {
                float v[32];
                tmem_ld32(tbase + c0, v);
                if (!live) continue;
                if (args.out_f) {
                    float* o = args.out_f + orow * args.D + c0;
#pragma unroll
                    for (int i = 0; i < 32; i += 4) *reinterpret_cast<float4*>(o + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
                }
                bf16* o = args.out_t + orow * args.D + c0;
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

// ---- CTA-pair variant: one cta_group::2 MMA over two m-tiles ---------------------------------------
// Per SM the message GEMM is bound by the bytes it must pull into SMEM (per 128-row tile 3 x 64 KB of
// gathered A rows + 3 x 128 KB of T). With M = 256 tiles on a CTA pair each CTA loads its own A rows
// and only HALF of every T k-block (the N-half the pair's MMA reads from it): 3 x (64 + 64) KB per SM
// per tile. Protocol as the 2-SM MLP (mlp_tc2.cuh): both producers signal the leader's full barrier,
// the leader arms it and issues the MMAs, its commits multicast to both CTAs; the epilogue warps of
// both CTAs release the accumulator on the leader's barrier.
template <int D>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(GRP_THREADS, 1)
gemm_grp2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmT,
                 const __grid_constant__ CUtensorMap tmO, const GrpArgs args) {
    constexpr int BN = D;
    constexpr int A_BYTES = BM * BK * 2;            // 16 KB: this CTA's 128 rows of a k-block
    constexpr int B_HALF = (BN / 2) * BK * 2;       // 16 KB: this CTA's N-half of a T k-block
    constexpr int STAGE = A_BYTES + B_HALF;
    constexpr int NST = 6;
    constexpr int STG_OFF = NST * STAGE;       // 2 x 16 KB output k-block staging (SW128, TMA store)
    constexpr int BAR_OFF = STG_OFF + 2 * 16384;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u); // same offset in both CTAs
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + BAR_OFF);
    uint64_t* empty = full + NST;
    uint64_t* tfull = empty + NST;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const bool elected = elect_one_sync(); // the lane of the single-thread TMA / MMA issue loops (uniform operands)
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    const int pair = int(blockIdx.x) / 2, npairs = int(gridDim.x) / 2;
    const int mpairs = (args.mtiles + 1) / 2;
    const int supers = args.groups * mpairs;

    if (threadIdx.x == 0) {
        for (int s = 0; s < NST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 2 * 8); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    fence_before();
    cluster_sync_all();
    fence_after();
    const uint32_t tmem_base = *tmem_slot;
    griddep_wait(); // (programmatic dependent launch) inputs of the previous kernel visible
    griddep_launch_dependents();
    const int a_bytes = args.K * args.bb * 128; // the A box actually filled (<= 16 KB)
    const uint32_t L_full0 = mapa_u32(smem_u32(&full[0]), 0);
    const uint32_t L_tempty0 = mapa_u32(smem_u32(&tempty[0]), 0);

    if (warp == 0) {
        if (elected) {
            int stage = 0;
            uint32_t phase = 0;
            for (int st = pair; st < supers; st += npairs) {
                const int g = st % args.groups, mt = 2 * (st / args.groups) + int(rank);
                const int nseg = args.seg_count[g];
                for (int sg = 0; sg < nseg; ++sg) {
                    const int arow = args.seg_arow[g * args.max_seg + sg];
                    const int alpha = args.seg_alpha[g * args.max_seg + sg];
                    for (int kk = 0; kk < args.kb_per_seg; ++kk) {
                        mbar_wait(&empty[stage], phase ^ 1);
                        if (leader) mbar_expect_tx(&full[stage], 2 * (a_bytes + B_HALF)); // both CTAs' bytes
                        uint8_t* sa = smem + stage * STAGE;
                        // (rows past the bins: zero-filled box, bytes still counted)
                        asm volatile(
                            "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
                                smem_u32(sa)),
                            "l"(reinterpret_cast<uint64_t>(&tmA)), "r"(L_full0 + stage * 8), "r"(kk * 64), "r"(arow * args.K), "r"(mt * args.bb)
                            : "memory");
                        tma_load_3d_2sm(sa + A_BYTES, &tmT, L_full0 + stage * 8, kk * 64, int(rank) * (BN / 2), alpha);
                        if (++stage == NST) { stage = 0; phase ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (leader && elected) {
            constexpr uint32_t idesc = idesc_bf16(256, BN);
            int stage = 0, acc = 0;
            uint32_t phase = 0, acc_phase = 0;
            for (int st = pair; st < supers; st += npairs) {
                const int g = st % args.groups;
                const int kblocks = args.seg_count[g] * args.kb_per_seg;
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                fence_after();
                const uint32_t d = tmem_base + uint32_t(acc * BN);
                for (int kb = 0; kb < kblocks; ++kb) {
                    mbar_wait(&full[stage], phase);
                    fence_after();
                    uint8_t* sa = smem + stage * STAGE;
                    const uint64_t da = sw128_desc(sa), db = sw128_desc(sa + A_BYTES);
#pragma unroll
                    for (int kk = 0; kk < BK / 16; ++kk)
                        mma_bf16_2sm(d, da + uint64_t(kk * 2), db + uint64_t(kk * 2), idesc, (kb | kk) != 0);
                    mma_commit_2sm(&empty[stage]);
                    if (++stage == NST) { stage = 0; phase ^= 1; }
                }
                mma_commit_2sm(&tfull[acc]);
                if (++acc == 2) { acc = 0; acc_phase ^= 1; }
            }
        }
    } else {
        // epilogue: output k-block kb (128 rows x 64 columns) staged by all 8 warps (SW128, double
        // buffered) and sent by one 3-D TMA store, as in gemm_grp_res_kernel; the optional fp32 copy
        // (incoming messages) is written directly
        const int quarter = warp % 4;
        const int half = (warp - 2) / 4; // 32-column half of every 64-column output k-block
        const int row = quarter * 32 + lane;
        const bool issuer = warp == 2 && elected;
        int acc = 0, step = 0;
        uint32_t acc_phase = 0;
        for (int st = pair; st < supers; st += npairs) {
            const int g = st % args.groups, mt = 2 * (st / args.groups) + int(rank);
            mbar_wait(&tfull[acc], acc_phase);
            fence_after();
            const int b = mt * args.bb + row / args.K, k = row % args.K;
            const bool live = row < args.K * args.bb && b < args.bins;
            const int orow_g = __ldg(args.out_row + g);
            const size_t orow = (size_t(b) * args.out_rows_per_bin + orow_g) * args.K + k;
            const uint32_t tbase = tmem_base + (uint32_t(quarter * 32) << 16) + uint32_t(acc * BN);
#pragma unroll 1
            for (int kb = 0; kb < args.D / 64; ++kb, ++step) {
                const int c0 = kb * 64 + half * 32;
                float v[32];
                tmem_ld32(tbase + c0, v);
                if (kb == args.D / 64 - 1) { // accumulator drained
                    fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cl(L_tempty0 + acc * 8);
                }
                if (args.out_f && live) {
                    float* o = args.out_f + orow * args.D + c0;
#pragma unroll
                    for (int i = 0; i < 32; i += 4) *reinterpret_cast<float4*>(o + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
                }
                uint8_t* stg = smem + STG_OFF + (step & 1) * 16384;
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    uint32_t pk[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        __nv_bfloat162 p = __floats2bfloat162_rn(v[jj * 8 + 2 * q], v[jj * 8 + 2 * q + 1]);
                        pk[q] = *reinterpret_cast<uint32_t*>(&p);
                    }
                    const int j = half * 4 + jj;
                    *reinterpret_cast<uint4*>(stg + row * 128 + ((j ^ (row & 7)) * 16)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("bar.sync 1, 256;" ::: "memory");
                if (issuer) {
                    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                                     reinterpret_cast<uint64_t>(&tmO)),
                                 "r"(smem_u32(stg)), "r"(kb * 64), "r"(orow_g * args.K), "r"(mt * args.bb)
                                 : "memory");
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); // the other buffer is free
                }
                asm volatile("bar.sync 1, 256;" ::: "memory");
            }
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
        if (issuer) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    fence_before();
    cluster_sync_all(); // no CTA leaves while its peer may still signal its barriers or read its smem
    if (warp == 1) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
    }
}
constexpr int GRP2_SMEM = 6 * (BM * BK * 2 + 128 * BK * 2) + 2 * 16384 + 256 + 1024;

// ---- CTA-pair T-resident variant (single-segment groups: the normalise GEMM) --------------------
// Each CTA of a pair keeps its N-half of the group's T_alpha resident (64 KB at D = 256) and streams
// only its gathered A rows (an 8-deep ring), so per 256-row pair tile each SM pulls 64 KB instead of
// 128 KB. Work = (group, m-tile pair) units in laps over the pairs (groups are slot-major: a slot's
// edges run on neighbouring pairs at the same m-tiles and share their z~ rows through L2), the
// remaining groups split their m-tile range; a T change waits for the MMAs on the old T (t_empty).
template <typename F>
__device__ __forceinline__ void grp_lap_sweep(int worker, int workers, int groups, int msz, F&& body) {
    int g0 = 0;
    for (; groups - g0 >= workers; g0 += workers)
        for (int m = 0; m < msz; ++m) body(g0 + worker, m);
    const int rem = groups - g0;
    if (rem > 0) { // the rest as equal contiguous (group, m) ranges: one T change per worker at most
        const int tot = rem * msz;
        const int u0 = int(int64_t(worker) * tot / workers), u1 = int(int64_t(worker + 1) * tot / workers);
        for (int u = u0; u < u1; ++u) body(g0 + u / msz, u % msz);
    }
}

template <int D>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(GRP_THREADS, 1)
gemm_grp2_res_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmT,
                     const __grid_constant__ CUtensorMap tmO, const GrpArgs args) {
    constexpr int BN = D;
    constexpr int NKB = D / 64;
    constexpr int A_BYTES = BM * BK * 2;            // 16 KB: this CTA's 128 rows of a k-block
    constexpr int B_HALF = (BN / 2) * BK * 2;       // this CTA's N-half of a T k-block
    constexpr int T_OFF = 0, A_OFF = NKB * B_HALF;
    constexpr int NST = 8;
    constexpr int STG_OFF = A_OFF + NST * A_BYTES;  // 2 x 16 KB output k-block staging (SW128, TMA store)
    constexpr int BAR_OFF = STG_OFF + 2 * 16384;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + BAR_OFF);
    uint64_t* empty = full + NST;
    uint64_t* tfull = empty + NST;
    uint64_t* tempty = tfull + 2;
    uint64_t* t_full = tempty + 2;  // resident T half landed (leader copy counts both CTAs)
    uint64_t* t_empty = t_full + 1; // every MMA on the old T retired
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(t_empty + 1);
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const bool elected = elect_one_sync(); // the lane of the single-thread TMA / MMA issue loops (uniform operands)
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    const int pair = int(blockIdx.x) / 2, npairs = int(gridDim.x) / 2;
    const int mpairs = (args.mtiles + 1) / 2;

    if (threadIdx.x == 0) {
        for (int s = 0; s < NST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 2 * 8); }
        mbar_init(t_full, 1);
        mbar_init(t_empty, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    fence_before();
    cluster_sync_all();
    fence_after();
    const uint32_t tmem_base = *tmem_slot;
    griddep_wait(); // (programmatic dependent launch) inputs of the previous kernel visible
    griddep_launch_dependents();
    const int a_bytes = args.K * args.bb * 128;
    const uint32_t L_full0 = mapa_u32(smem_u32(&full[0]), 0);
    const uint32_t L_tfull = mapa_u32(smem_u32(t_full), 0);
    const uint32_t L_tempty0 = mapa_u32(smem_u32(&tempty[0]), 0);

    if (warp == 0) {
        if (elected) {
            int stage = 0, cur = -1;
            uint32_t phase = 0, teph = 0;
            grp_lap_sweep(pair, npairs, args.groups, mpairs, [&](int g, int mtp) {
                const int alpha = args.seg_alpha[g * args.max_seg];
                if (alpha != cur) { // new coefficient action: after the MMAs on the old one retired
                    if (cur >= 0) { mbar_wait(t_empty, teph); teph ^= 1; }
                    if (leader) mbar_expect_tx(t_full, 2 * NKB * B_HALF);
                    for (int kb = 0; kb < NKB; ++kb)
                        tma_load_3d_2sm(smem + T_OFF + kb * B_HALF, &tmT, L_tfull, kb * 64, int(rank) * (BN / 2), alpha);
                    cur = alpha;
                }
                const int arow = args.seg_arow[g * args.max_seg];
                const int mt = 2 * mtp + int(rank);
                for (int kb = 0; kb < NKB; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    if (leader) mbar_expect_tx(&full[stage], 2 * a_bytes);
                    asm volatile(
                        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
                            smem_u32(smem + A_OFF + stage * A_BYTES)),
                        "l"(reinterpret_cast<uint64_t>(&tmA)), "r"(L_full0 + stage * 8), "r"(kb * 64), "r"(arow * args.K), "r"(mt * args.bb)
                        : "memory");
                    if (++stage == NST) { stage = 0; phase ^= 1; }
                }
            });
        }
    } else if (warp == 1) {
        if (leader && elected) {
            constexpr uint32_t idesc = idesc_bf16(256, BN);
            int stage = 0, acc = 0, cur = -1;
            uint32_t phase = 0, acc_phase = 0, tfph = 0;
            grp_lap_sweep(pair, npairs, args.groups, mpairs, [&](int g, int) {
                const int alpha = args.seg_alpha[g * args.max_seg];
                if (alpha != cur) {
                    if (cur >= 0) mma_commit_2sm(t_empty); // fires once every MMA on the old T has completed
                    mbar_wait(t_full, tfph);
                    tfph ^= 1;
                    fence_after();
                    cur = alpha;
                }
                mbar_wait(&tempty[acc], acc_phase ^ 1);
                fence_after();
                const uint32_t d = tmem_base + uint32_t(acc * BN);
                for (int kb = 0; kb < NKB; ++kb) {
                    mbar_wait(&full[stage], phase);
                    fence_after();
                    const uint64_t da = sw128_desc(smem + A_OFF + stage * A_BYTES), db = sw128_desc(smem + T_OFF + kb * B_HALF);
#pragma unroll
                    for (int kk = 0; kk < BK / 16; ++kk)
                        mma_bf16_2sm(d, da + uint64_t(kk * 2), db + uint64_t(kk * 2), idesc, (kb | kk) != 0);
                    mma_commit_2sm(&empty[stage]);
                    if (++stage == NST) { stage = 0; phase ^= 1; }
                }
                mma_commit_2sm(&tfull[acc]);
                if (++acc == 2) { acc = 0; acc_phase ^= 1; }
            });
        }
    } else {
        // epilogue as gemm_grp2_kernel (staged SW128 k-blocks, one 3-D TMA store each)
        const int quarter = warp % 4;
        const int half = (warp - 2) / 4;
        const int row = quarter * 32 + lane;
        const bool issuer = warp == 2 && elected;
        int acc = 0, step = 0;
        uint32_t acc_phase = 0;
        grp_lap_sweep(pair, npairs, args.groups, mpairs, [&](int g, int mtp) {
            const int mt = 2 * mtp + int(rank);
            mbar_wait(&tfull[acc], acc_phase);
            fence_after();
            const int orow_g = __ldg(args.out_row + g);
            const uint32_t tbase = tmem_base + (uint32_t(quarter * 32) << 16) + uint32_t(acc * BN);
#pragma unroll 1
            for (int kb = 0; kb < NKB; ++kb, ++step) {
                float v[32];
                tmem_ld32(tbase + kb * 64 + half * 32, v);
                if (kb == NKB - 1) { // accumulator drained
                    fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cl(L_tempty0 + acc * 8);
                }
                uint8_t* stg = smem + STG_OFF + (step & 1) * 16384;
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    uint32_t pk[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        __nv_bfloat162 p = __floats2bfloat162_rn(v[jj * 8 + 2 * q], v[jj * 8 + 2 * q + 1]);
                        pk[q] = *reinterpret_cast<uint32_t*>(&p);
                    }
                    const int j = half * 4 + jj;
                    *reinterpret_cast<uint4*>(stg + row * 128 + ((j ^ (row & 7)) * 16)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("bar.sync 1, 256;" ::: "memory");
                if (issuer) {
                    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                                     reinterpret_cast<uint64_t>(&tmO)),
                                 "r"(smem_u32(stg)), "r"(kb * 64), "r"(orow_g * args.K), "r"(mt * args.bb)
                                 : "memory");
                    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                }
                asm volatile("bar.sync 1, 256;" ::: "memory");
            }
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        });
        if (issuer) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
    fence_before();
    cluster_sync_all();
    if (warp == 1) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
    }
}
template <int D>
constexpr int grp2_res_smem() { return (D / 64) * (D / 2) * 64 * 2 + 8 * BM * BK * 2 + 2 * 16384 + 256 + 1024; }

} // namespace tc
} // namespace cider
