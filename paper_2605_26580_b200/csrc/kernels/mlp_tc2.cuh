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
//
// Warp roles (640 threads): 0 weight-ring producer, 1 first-layer MMA issuer, 2-9 hidden-chunk
// epilogue (GELU, packed in place, released in 16-column groups), 10-17 final epilogue (overlaps the
// next tile's chunks; bias from SMEM; results staged in the tile's own X k-blocks in the SW128 layout),
// 18 second-layer MMA issuer, 19 row-tile (X) producer, which also TMA-stores the staged outputs and
// refills those k-blocks. The aggregator and the demix variant double-buffer their 64 KB row tile.
// EP_DEMIX (Lambda-bar -> demix -> e, hidden = the Q symbol columns) runs all 16 epilogue warps on
// the demix (16-column passes, each released to the second MMA on its own) and the final epilogue.
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
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) { // 16 columns, waited
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n\t"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]), "r"(v[1]),
                 "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
        "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
}
__device__ __forceinline__ void ld_shared_v4(const void* p, uint32_t* r) {
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(smem_u32(p)));
}
__device__ __forceinline__ void st_shared_v4(void* p, const uint32_t* r) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(smem_u32(p)), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3])
                 : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// TMA store of one box out of shared memory (bulk-group completion)
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int x, int y) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(reinterpret_cast<uint64_t>(map)),
                 "r"(smem_u32(src)), "r"(x), "r"(y)
                 : "memory");
}
// L2 prefetch of one TMA box (no shared memory, no barrier)
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int x, int y) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void ld_global_v8(const void* p, uint32_t* r) { // 32 bytes, one sector
    asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "l"(p));
}
__device__ __forceinline__ void st_global_v8(void* p, const uint32_t* r) {
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]),
                 "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}
// 64 consecutive accumulator columns of this warp's lane quarter, waited in the same statement
__device__ __forceinline__ void tmem_ld64(uint32_t taddr, float* v) {
    uint32_t r[64];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x64.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,"
        "%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,"
        "%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];\n\t"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]),
          "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]),
          "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]),
          "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]),
          "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
        : "r"(taddr)
        : "memory");
#pragma unroll
    for (int i = 0; i < 64; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void mma_commit_2sm_mask(uint64_t* bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
}
__device__ __forceinline__ void mma_commit_2sm(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(uint16_t(3))
        : "memory");
}

// tcgen05.ld of 32 columns without the wait, and the wait tied to those registers (so no use of
// them can be scheduled above it): the final epilogue loads k-block kb + 1 while it works on kb
__device__ __forceinline__ void tmem_ld32_nw(uint32_t taddr, uint32_t (&r)[32]) {
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
}
__device__ __forceinline__ void tmem_wait_ld32(uint32_t (&r)[32]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                   "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                   "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19]), "+r"(r[20]), "+r"(r[21]),
                   "+r"(r[22]), "+r"(r[23]), "+r"(r[24]), "+r"(r[25]), "+r"(r[26]), "+r"(r[27]), "+r"(r[28]),
                   "+r"(r[29]), "+r"(r[30]), "+r"(r[31])
                 :
                 : "memory");
}

constexpr int MLP2_NS_CAP = 16; // weight-ring slots at most (else as many as the shared memory holds)
template <int KIN, int D, int STGW = 4096, int EW = 8, int NXB = 1, int BIASB = 4 * D, int B1SB = 0>
struct Mlp2Layout {
    static constexpr int STG_WARP = STGW;
    static constexpr int XBUF = NXB; // row-tile buffers (2: the next tile's rows load during this tile)
    static constexpr int KB1 = KIN / 64;
    static constexpr int KB2 = MLP_HC / 64;
    static constexpr int W1_HALF = (MLP_HC / 2) * 64 * 2;   // 8 KB: this CTA's 64 rows of a W1 k-block
    static constexpr int W2_HALF = (D / 2) * 64 * 2;        // this CTA's D/2 rows of a W2 k-block
    static constexpr int SLOT = 16384;
    static constexpr int W1_PER_SLOT = SLOT / W1_HALF;       // 2
    static constexpr int X_BYTES = KB1 * 128 * 64 * 2;
    static constexpr int B1S_BYTES = B1SB;             // hidden bias [H] fp32 in shared memory (0: read by __ldg)
    static constexpr int B1S_OFF_FROM_BAR = 512 + BIASB;
    static constexpr int FIXED = 1024 + 512 + BIASB + B1SB;  // alignment slack, barriers, output bias, hidden bias
    static constexpr int BIAS_OFF_FROM_BAR = 512;      // output bias [D] fp32 right after the barriers
    // output staging for coalesced stores: one 32-row x 64-column bf16 block per epilogue warp (the
    // aggregator only; gate / fusion, KIN = 2D, need the SMEM for the weight ring and store directly)
    static constexpr int STG_BYTES = KIN == D ? EW * STGW : 0;
    static constexpr int NS_RAW = (SMEM_LIMIT - FIXED - NXB * X_BYTES - STG_BYTES) / SLOT;
    static constexpr int NS = NS_RAW > MLP2_NS_CAP ? MLP2_NS_CAP : NS_RAW;
    static constexpr int STG_OFF = NXB * X_BYTES;
    static constexpr int R_OFF = NXB * X_BYTES + STG_BYTES;
    static constexpr int BAR_OFF = R_OFF + NS * SLOT;
    static constexpr int TOTAL = BAR_OFF + 512 + BIASB + B1SB + 1024;
    static_assert(NS >= 4, "fused MLP (2-SM) does not fit in shared memory");
    static_assert((2 * NXB * KB1 + 2 * NS + 2 + 2 * 8 + 2 + 2 + NXB * (D / 64) + 1) * 8 + 4 <= 512, "barrier block");
    static_assert(D % 32 == 0 && D <= 256 && W2_HALF <= SLOT, "output width must be <= 256");
    static_assert(KB1 % W1_PER_SLOT == 0, "input width must be a multiple of 128");
};

// EP_DEMIX runs 16 epilogue warps (4 per TMEM lane quarter, 32 hidden columns each) with one
// [16][33] fp32 staging block per warp; the GELU variants run 8 with 4 KB each.
constexpr int DEMIX_STG_WARP = 16 * 33 * 4;
// 16 epilogue warps in every variant: demix = 16 warps on every phase; GELU variants = warps 2-9 on
// the hidden chunks (64 columns each) and warps 10-17 on the final epilogue (which then overlaps the
// next tile's chunks). Measured and dropped (round 1): 16 hidden-chunk warps (the 72-register cap of
// 896 threads), the aggregator's 16 warps on both phases, the gate / fusion final epilogue with the
// next TMEM load in flight, the fusion residual folded into acc2, register-direct gate / fusion
// stores, an L2 prefetch of the next row tile, a polynomial exp2 for half of the demix groups.
constexpr int MLP2_HW = 8;                                 // hidden-chunk warps of the GELU variants
constexpr int mlp2_epi_warps(int epk) { return epk == EP_DEMIX ? 16 : MLP2_HW + 8; }
constexpr int MLP2_FIN_WARP0 = 2 + MLP2_HW;
constexpr int mlp2_threads(int epk) { return (mlp2_epi_warps(epk) + 4) * 32; }
// D = 128: a hidden chunk is 1024 tensor-pipe cycles and its GELU >= 1024 MUFU cycles (16 tanh per clock
// per SM), so the hidden-chunk epilogue bounds the kernel (profiles/r2/experiments/d128_mlp_epilogue.md):
// the hidden bias is read from shared memory at the price of one weight-ring slot (aggregator 10 -> 9
// slots: -6% kernel time; gate / fusion 6 -> 5: -2.4% / -1.2%); a hidden width that does not fit runs
// on the 1-SM kernel (engine.cu mlp()). A run-time choice between the two bias sources costs the gain
// (generic loads), so it is a compile-time property of the variant. At D = 256 (the GELU has 2x slack there)
// the same trade is neutral for all three variants and is not made. Sharing one TMEM-store wait / fence /
// arrive between two 16-column groups was measured neutral and is not used.
constexpr int mlp2_b1_smem_bytes(int kin, int d, int epk) {
    return (d == 128 && epk != EP_DEMIX) ? (kin == 128 ? 4096 : 2048) : 0; // H <= 1024 (aggregator) / 512
}
// The GELU variants stage their output in the tile's own X k-blocks (no staging region); the
// aggregator (input = output width) double-buffers its row tile.
template <int KIN, int D, int EPK>
using Mlp2LayoutFor = Mlp2Layout<KIN, D, EPK == EP_DEMIX ? DEMIX_STG_WARP : 0, mlp2_epi_warps(EPK),
                                 ((KIN == D && (EPK == EP_STORE || EPK == EP_DEMIX)) || KIN <= 256) ? 2 : 1,
                                 EPK == EP_DEMIX ? 0 : 4 * D, mlp2_b1_smem_bytes(KIN, D, EPK)>;
// (KIN <= 256: the D = 128 gate / fusion row tile is 64 KB, so it double-buffers as well)

constexpr int MLP2_GG = 4; // GELU release groups per 64-column warp half (16 hidden columns = one MMA2 k-step)

// EP_DEMIX hidden phase of one epilogue warp: its 32 rows (= 32 / KK (bin, slot) groups of KK rows)
// x 32 intermediate-logit columns of a chunk, in two passes of 16 columns. Per pass the fp32
// accumulator rows go to SMEM (column-major [16][33], conflict-free both ways); each lane then takes
// one column over half of the rows and applies demix_responsibilities (denoiser.cpp:103-122): softmax
// over the KK rows of each group at 1/tau with a fixed-point normaliser (2^-22 units, rounded by the
// 2^23 magic add, summed as integers: bitwise invariant to the order of the rows), times
// S[(bin, slot)][column]. The bf16 results come back row-wise through the same SMEM block and are
// packed IN PLACE into the warp's own TMEM columns as the A operand of the V GEMM. beta S is a
// per-group constant shift of the logits and cancels inside softmax_k (not applied).
// S[(bin, slot)][column] for this lane's column and row groups of one warp chunk (both passes),
// requested one chunk ahead of its use
template <int KK>
__device__ __forceinline__ void demix_load_sv(const MlpArgs& args, int m0, int col0, int lane, float* sv) {
    constexpr int NGL = 16 / KK;
    const int cl = lane & 15, rh = lane >> 4;
#pragma unroll
    for (int p = 0; p < 2; ++p)
#pragma unroll
        for (int t = 0; t < NGL; ++t) {
            const int r0 = m0 + rh * 16 + t * KK;
            // S row stride and valid symbol count = ep.ldz (Q); hidden columns past Q (Q < 128 padded to
            // one 128-column chunk, zero rows of W and V) read S = 0, so they add nothing to e
            const int col = col0 + p * 16 + cl;
            sv[p * NGL + t] = r0 < args.ep.M && col < args.ep.ldz ? __ldg(args.ep.S + size_t(r0 / KK) * args.ep.ldz + col) : 0.0f;
        }
}

// Symbol columns past Q (Q < 128 padded to one 128-column chunk): S = 0 there, so r (x) S = 0 — the warp
// packs zeros for the second MMA (whose V rows are zero as well; TMEM garbage must not reach it) and skips
// the demix arithmetic: half of the chunk at Q = 64 (c2, c4), where the kernel is bound by this epilogue.
__device__ __forceinline__ void demix_warp_pad(uint32_t base, uint64_t* a1_full_b, uint32_t ph, uint32_t l_h_full, int lane) {
    mbar_wait(a1_full_b, ph);
    fence_after();
    const uint32_t z[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
#pragma unroll
    for (int p = 0; p < 2; ++p) tmem_st8(base + p * 8, z);
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    fence_before();
    __syncwarp();
    if (lane == 0) {
        mbar_arrive_cl(l_h_full);
        mbar_arrive_cl(l_h_full + 8);
    }
}

template <int KK>
__device__ __forceinline__ void demix_warp(const MlpArgs& args, uint8_t* stg, uint32_t base, uint64_t* a1_full_b, uint32_t ph,
                                           uint32_t l_h_full, const float* svin, int lane, long long* tr) {
    constexpr int NGL = 16 / KK; // row groups per lane (lanes 0-15: rows 0-15, lanes 16-31: rows 16-31)
    const Epi& ep = args.ep;
    float* xs = reinterpret_cast<float*>(stg); // [16 columns][33] fp32; then [32 rows][32 B] bf16
    const int cl = lane & 15, rh = lane >> 4;
    const float scale2 = ep.inv_tau * 1.4426950408889634f;
    float sv[2][NGL];
#pragma unroll
    for (int p = 0; p < 2; ++p)
#pragma unroll
        for (int t = 0; t < NGL; ++t) sv[p][t] = svin[p * NGL + t];
    if (tr) tr[2] = clock64();
    mbar_wait(a1_full_b, ph);
    fence_after();
    if (tr) tr[3] = clock64();
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        {
            float v[16];
            tmem_ld16(base + p * 16, v);
#pragma unroll
            for (int j = 0; j < 16; ++j) xs[j * 33 + lane] = v[j]; // row `lane`, column j
        }
        __syncwarp();
        float xv[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) xv[i] = xs[cl * 33 + rh * 16 + i];
        __syncwarp(); // xs is reused for the bf16 results below
        uint8_t* os = stg;
#pragma unroll
        for (int t = 0; t < NGL; ++t) {
            float mx = -INFINITY;
#pragma unroll
            for (int k = 0; k < KK; ++k) mx = fmaxf(mx, xv[t * KK + k]);
            const float nmx = -mx * scale2;
            uint32_t den = 0;
#pragma unroll
            for (int k = 0; k < KK; ++k) {
                const float e = ex2_approx(fmaf(xv[t * KK + k], scale2, nmx));
                xv[t * KK + k] = e;
                den += __float_as_uint(fmaf(e, 4194304.0f, 8388608.0f)) - 0x4B000000u; // round(e 2^22)
            }
            const float rs = (4194304.0f / float(den)) * sv[p][t];
#pragma unroll
            for (int k = 0; k < KK; ++k) {
                const int r = rh * 16 + t * KK + k;
                *reinterpret_cast<bf16*>(os + r * 32 + (((cl >> 3) ^ ((r >> 2) & 1)) * 16) + (cl & 7) * 2) =
                    __float2bfloat16_rn(xv[t * KK + k] * rs);
            }
        }
        __syncwarp();
        const uint4 p0 = *reinterpret_cast<const uint4*>(os + lane * 32 + ((0 ^ ((lane >> 2) & 1)) * 16));
        const uint4 p1 = *reinterpret_cast<const uint4*>(os + lane * 32 + ((1 ^ ((lane >> 2) & 1)) * 16));
        const uint32_t pk[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
        tmem_st8(base + p * 8, pk); // pass p's 16 columns packed in place (fp32 columns [0, 16) were read in pass 0)
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        fence_before();
        __syncwarp(); // (also: the next pass overwrites the staging block)
        if (lane == 0) mbar_arrive_cl(l_h_full + p * 8); // pass p -> MMA2 k-step 2 sub + p, as soon as it is packed
    }
    if (tr) tr[4] = clock64();
}


// warps: ring producer, MMA1 issuer, epilogue warps (2 .. EW + 1), MMA2 issuer, X producer

// EPK: final-epilogue kind (EP_STORE, EP_GATE or EP_RESID), a template parameter so each variant
// carries only the registers its epilogue needs.
// KK (EP_DEMIX only): rows per (bin, slot) group = users per bin (4 or 8), compile-time so that one demix
// body is instantiated per kernel.
template <int KIN, int D, int EPK, int KK = 0>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(mlp2_threads(EPK), 1)
mlp_tc2_kernel(const __grid_constant__ CUtensorMap tmX0, const __grid_constant__ CUtensorMap tmX1,
               const __grid_constant__ CUtensorMap tmW1, const __grid_constant__ CUtensorMap tmW2,
               const __grid_constant__ CUtensorMap tmO, const MlpArgs args_in) {
#ifdef CIDER_MLP_TRACE
    const MlpArgs& args = args_in; // diagnostic build: per-chunk clock64 stamps (tests/trace_mlp.py)
#else
    MlpArgs args = args_in; // the stamps and their predicates are compiled out (they cost 1-3% of the MLPs)
    args.trace = nullptr;
#endif
    using Lay = Mlp2LayoutFor<KIN, D, EPK>;
    constexpr int KB1 = Lay::KB1, KB2 = Lay::KB2, NS = Lay::NS;
    constexpr int EW = mlp2_epi_warps(EPK);              // epilogue warps 2 .. EW + 1
    constexpr int MMA2_WARP = EW + 2, XLOAD_WARP = EW + 3;
    constexpr int KBD = D / 64; // output k-blocks = final-epilogue steps (half h takes k-blocks h, h+2, ...)
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u); // 1 KB aligned, stays in the shared window
    uint8_t* xs = smem;
    uint8_t* ring = smem + Lay::R_OFF;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Lay::BAR_OFF);
    constexpr int NXB = Lay::XBUF;
    uint64_t* x_full = bar;             // [NXB][KB1] row-tile k-block landed (leader copy counts both CTAs)
    uint64_t* x_empty = x_full + NXB * KB1; // [NXB][KB1] k-block free: last MMA1 read it (+ final-epilogue readers)
    uint64_t* r_full = x_empty + NXB * KB1;
    uint64_t* r_empty = r_full + NS;
    uint64_t* a1_full = r_empty + NS;   // [2] first-layer accumulator ready
    constexpr int HG = 2 * MLP2_GG;     // hidden-group barriers per acc1 buffer (demix: one per 16-column pass)
    uint64_t* h_full = a1_full + 2;     // [2][HG] hidden group g of acc1[b] packed (leader copy counts both CTAs)
    uint64_t* a1_free = h_full + 2 * HG; // [2] MMA2 done reading acc1[b] (leader only)
    uint64_t* a2_full = a1_free + 2;
    uint64_t* a2_empty = a2_full + 1;
    uint64_t* o_full = a2_empty + 1;    // [NXB][KBD] output block staged in X k-block kb (4 quarter warps)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_full + NXB * KBD);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const bool elected = elect_one_sync(); // (all warps converged here) the lane of the single-thread issue loops
    const uint32_t rank = cluster_rank();
    const bool leader = rank == 0;
    const int pair = blockIdx.x / 2, npairs = gridDim.x / 2;
    const int NC = args.H / MLP_HC;
    constexpr int EPI_ARRIVALS = 2 * EW; // one elected lane per epilogue warp, both CTAs
    // hidden group g: GELU = 16 columns of both 64-column warp halves (the 8 hidden warps x 2 CTAs);
    // demix = the 32 columns of one warp per quarter (4 quarters x 2 CTAs)
    constexpr int H_ARRIVALS = EPK == EP_DEMIX ? 8 : 8 * 2;
    // Final epilogue on warps 10-17 (gate / fusion / aggregator), overlapping the next tile's chunks
    constexpr int FIN_STRIDE = 2;                                // output k-blocks between one warp's
    constexpr int A2_ARRIVALS = EPK == EP_DEMIX ? EPI_ARRIVALS : 8 * 2; // warps that drain acc2

    // Gate / fusion epilogues read z (and e) from global memory (L2: the same rows were just TMA'd
    // into X), so every X k-block is free once the tile's last MMA1 has read it and the next tile's
    // rows stream in while this tile's final epilogue runs.
    constexpr bool reads_z = EPK == EP_GATE || EPK == EP_RESID;
    constexpr bool reads_e = EPK == EP_GATE;
    // gate / fusion keep the tile's z k-blocks until the final epilogue has read them, so every chunk
    // runs over the input k-blocks starting at the second half ([e | z] order): the next tile's
    // e / acc k-blocks load during the final epilogue and the first MMA1 starts on them.
    constexpr int ROT = reads_z ? KBD : 0;
    // Issue loops run by the whole warp (bit 0: MMA1 issuer, bit 1: MMA2 issuer; lane 0 issues) or by
    // lane 0 alone, per variant (whole-warp loops: aggregator +2%, gate / fusion -10%)
    constexpr int WI = EPK == EP_DEMIX ? 3 : KIN == D ? 3 : 0; // (with elect.sync issue lanes the two forms measure equal)
    // gate / fusion: the 8 final warps walk the output k-blocks together (each warp one 32-column half
    // of every k-block), so k-block 0 is staged, stored and refilled first and the next tile's first
    // MMA1 is fed k-block by k-block instead of in two rounds
    constexpr bool KB_SEQ = reads_z;
    constexpr int O_ARRIVALS = KB_SEQ ? 8 : 4;
    if (threadIdx.x == 0) {
        // x_empty: the last MMA1 of the tile (+ the gate's 4 warps that read that e k-block); the
        // output k-blocks are refilled by the X producer itself after storing them (o_full)
        for (int kb = 0; kb < NXB * KB1; ++kb) {
            mbar_init(&x_full[kb], 1);
            mbar_init(&x_empty[kb], 1 + ((reads_e && kb % KB1 >= KBD) ? O_ARRIVALS : 0));
        }
        for (int s = 0; s < NS; ++s) { mbar_init(&r_full[s], 1); mbar_init(&r_empty[s], 1); }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&a1_full[b], 1);
            for (int g = 0; g < HG; ++g) mbar_init(&h_full[HG * b + g], H_ARRIVALS);
            mbar_init(&a1_free[b], 1);
        }
        mbar_init(a2_full, 1);
        mbar_init(a2_empty, A2_ARRIVALS);
        for (int kb = 0; kb < NXB * KBD; ++kb) mbar_init(&o_full[kb], O_ARRIVALS);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    fence_before();
    float* bias_s = reinterpret_cast<float*>(smem + Lay::BAR_OFF + Lay::BIAS_OFF_FROM_BAR); // final-epilogue bias
    if constexpr (EPK != EP_DEMIX)
        for (int i = threadIdx.x; i < D; i += blockDim.x) bias_s[i] = args.ep.bias ? args.ep.bias[i] : 0.0f;
    float* b1_s = reinterpret_cast<float*>(smem + Lay::BAR_OFF + Lay::B1S_OFF_FROM_BAR); // hidden bias (if B1S_BYTES)
    if constexpr (Lay::B1S_BYTES > 0) // (the host launches this variant only for H <= B1S_BYTES / 4)
        for (int i = threadIdx.x; i < args.H && i < Lay::B1S_BYTES / 4; i += blockDim.x) b1_s[i] = args.b1[i];
    cluster_sync_all(); // barriers of both CTAs initialised before any remote signal
    fence_after();
    const uint32_t tmem = *tmem_slot;
    griddep_wait(); // (programmatic dependent launch) inputs of the previous kernel visible
    griddep_launch_dependents();
    const uint32_t L_x_full0 = mapa_u32(smem_u32(&x_full[0]), 0);
    const uint32_t L_r_full0 = mapa_u32(smem_u32(&r_full[0]), 0);
    const uint32_t L_h_full0 = mapa_u32(smem_u32(&h_full[0]), 0);
    const uint32_t L_a2_empty = mapa_u32(smem_u32(a2_empty), 0);

    // Weight-ring sequence of one tile (the producer's order): W1(0), W1(1), then W2(c), W1(c+2) ...
    // Both MMA issuers locate their loads in it by position, so one ring serves both.
    constexpr int S1 = KB1 / Lay::W1_PER_SLOT, S2 = KB2;
    const int per_tile = NC * (S1 + S2);
    auto pos_w1 = [&](int c) { return c < 2 ? c * S1 : 2 * S1 + (c - 1) * S2 + (c - 2) * S1; };
    auto pos_w2 = [&](int c) { return 2 * S1 + c * S2 + min(c, NC - 2) * S1; };

    if (warp == 0) {
        if (elected) { // weight ring producer
            int slot = 0;
            uint32_t rph = 0;
            auto next = [&] { if (++slot == NS) { slot = 0; rph ^= 1; } };
            auto acquire = [&](uint32_t bytes_both) {
                mbar_wait(&r_empty[slot], rph ^ 1);
                if (leader) mbar_expect_tx(&r_full[slot], bytes_both); // the leader arms its own barrier
            };
            auto load_w1 = [&](int c) { // tmW1 is 3-D: {64 cols, H rows, KIN/64 k-blocks}
                for (int i = 0; i < KB1; i += Lay::W1_PER_SLOT) {
                    const int kb = (i + ROT) % KB1;
                    acquire(2 * Lay::W1_PER_SLOT * Lay::W1_HALF);
                    tma_load_3d_2sm(ring + slot * Lay::SLOT, &tmW1, L_r_full0 + slot * 8, 0,
                                    c * MLP_HC + int(rank) * (MLP_HC / 2), kb);
                    next();
                }
            };
            auto load_w2 = [&](int c) {
                for (int kb = 0; kb < KB2; ++kb) {
                    acquire(2 * Lay::W2_HALF);
                    tma_load_2d_2sm(ring + slot * Lay::SLOT, &tmW2, L_r_full0 + slot * 8, c * MLP_HC + kb * 64,
                                    int(rank) * (D / 2));
                    next();
                }
            };
            for (int tile = pair; tile < args.tiles; tile += npairs) {
                load_w1(0);
                if (NC > 1) load_w1(1);
                for (int c = 0; c < NC; ++c) {
                    load_w2(c);
                    if (c + 2 < NC) load_w1(c + 2);
                }
            }
        }
    } else if (warp == XLOAD_WARP) {
        if (elected) { // row-tile producer, one k-block at a time
            uint32_t eph = 0;
            int itx = 0;
            for (int tile = pair; tile < args.tiles; tile += npairs, ++itx) {
                const int row0 = tile * 256 + int(rank) * 128;
                const int xb = itx % NXB;
                uint8_t* xsb = xs + xb * Lay::X_BYTES;
                if (NXB > 1 && itx > 0 && xb == 0) eph ^= 1; // buffer 0's phase flips every NXB tiles
                if constexpr (EPK == EP_DEMIX) { // tmX0 is 3-D: the whole row tile in ONE box, on x_full[xb KB1]
                    if (itx >= NXB) { // this buffer holds the e tile of two tiles back: store it out first
                        const int prev_row0 = row0 - NXB * npairs * 256;
                        for (int kb = 0; kb < KBD; ++kb) {
                            mbar_wait(&o_full[xb * KBD + kb], uint32_t((itx / NXB - 1) & 1));
                            tma_store_2d(&tmO, xsb + kb * 16384, kb * 64, prev_row0);
                        }
                        bulk_commit();
                        bulk_wait_read0();
                    }
                    for (int kb = 0; kb < KB1; ++kb) mbar_wait(&x_empty[xb * KB1 + kb], eph ^ 1);
                    if (leader) mbar_expect_tx(&x_full[xb * KB1], 2 * KB1 * 16384);
                    tma_load_3d_2sm(xsb, &tmX0, L_x_full0 + xb * KB1 * 8, 0, row0, 0);
                    continue;
                }
                // The final epilogue stages the previous tile of this buffer in its k-blocks [0, KBD):
                // this thread stores them (one TMA box per k-block, two at a time as the epilogue's two
                // rounds finish) and refills them once the stores have read them out.
                const int prev_row0 = row0 - NXB * npairs * 256;
                const uint32_t oph = uint32_t((itx / NXB - 1) & 1);
                auto load_kb = [&](int kb) {
                    const int xk = xb * KB1 + kb;
                    mbar_wait(&x_empty[xk], eph ^ 1);
                    if (leader) mbar_expect_tx(&x_full[xk], 2 * 16384);
                    const int k = kb * 64;
                    if (k < args.K0) tma_load_2d_2sm(xsb + kb * 16384, &tmX0, L_x_full0 + xk * 8, k, row0);
                    else tma_load_2d_2sm(xsb + kb * 16384, &tmX1, L_x_full0 + xk * 8, k - args.K0, row0);
                };
                // by final-epilogue round (its warp halves finish output k-blocks kb0, kb0 + 1 together, and
                // the gate's e k-blocks KBD + kb0, KBD + kb0 + 1 with them): e / acc first, then the z pair
                constexpr int KSTEP = KB_SEQ ? 1 : 2;
                for (int kb0 = 0; kb0 < KBD; kb0 += KSTEP) {
                    if (KB1 > KBD)
                        for (int kb = KBD + kb0; kb < KBD + kb0 + KSTEP; ++kb) load_kb(kb);
                    if (itx >= NXB) {
                        for (int kb = kb0; kb < kb0 + KSTEP && kb < KBD; ++kb) {
                            mbar_wait(&o_full[xb * KBD + kb], oph);
                            tma_store_2d(&tmO, xsb + kb * 16384, kb * 64, prev_row0);
                        }
                        bulk_commit();
                        bulk_wait_read0();
                    }
                    for (int kb = kb0; kb < kb0 + KSTEP && kb < KBD; ++kb) load_kb(kb);
                }
                if (NXB == 1) eph ^= 1;
            }
            { // the last NXB tiles' outputs
                for (int q = 0; q < NXB; ++q) {
                    const int itl = itx - NXB + q; // tile index (per CTA) whose output is still staged
                    if (itl < 0) continue;
                    const int xb = itl % NXB;
                    const int row0 = (pair + itl * npairs) * 256 + int(rank) * 128;
                    for (int kb = 0; kb < KBD; ++kb) {
                        mbar_wait(&o_full[xb * KBD + kb], uint32_t((itl / NXB) & 1));
                        tma_store_2d(&tmO, xs + xb * Lay::X_BYTES + kb * 16384, kb * 64, row0);
                    }
                    bulk_commit();
                }
                bulk_wait_all();
            }
        }
    } else if (warp == 1 || warp == MMA2_WARP) {
        // Two MMA issuers on the leader: the tensor pipe queues only ~50 cycles of work, so every
        // barrier wait of a single issuing thread is a pipe bubble (tools/mma_bench.cu issue2_kernel:
        // 200-cycle waits per slot cost 22% with one issuer, 11% with two). Warp 1 issues the first
        // layer (acc1 buffers), warp 10 the second (acc2); a1_free orders MMA2(n) before MMA1(n+2).
        const bool el = elected;
        if (leader && (el || ((warp == 1 ? WI & 1 : WI & 2) != 0))) {
            auto ring_slot = [&](int gpos, uint32_t& ph) { ph = uint32_t(gpos / NS) & 1u; return gpos % NS; };
            const bool tr = args.trace && blockIdx.x == 0 && el;
            if (warp == 1) {
                constexpr uint32_t id1 = idesc_bf16(256, MLP_HC);
                uint32_t xph = 0, fph = 0; // fph bit b: phase of a1_free[b]
                int n = 0, it = 0;
                for (int tile = pair; tile < args.tiles; tile += npairs, ++it) {
                    const int xb = it % NXB;
                    if (NXB > 1 && it > 0 && xb == 0) xph ^= 1;
                    for (int c = 0; c < NC; ++c, ++n) {
                        const int b = n & 1;
                        if (tr && it < 4) args.trace[it * 64 + c * 8 + 6] = clock64();
                        mbar_wait(&a1_free[b], ((fph >> b) & 1u) ^ 1u); // MMA2 of the chunk two back has read acc1[b]
                        fph ^= 1u << b;
                        fence_after();
                        if (tr && it < 4) args.trace[896 + it * 8 + c] = clock64();
                        const uint32_t d = tmem + 256 + b * MLP_HC;
                        for (int sg = 0; sg < S1; ++sg) {
                            uint32_t ph;
                            const int slot = ring_slot(it * per_tile + pos_w1(c) + sg, ph);
                            if (c == 0 && EPK == EP_DEMIX && sg == 0) mbar_wait(&x_full[xb * KB1], xph); // one box
                            else if (c == 0 && EPK != EP_DEMIX) // the tile's k-blocks arrive one by one
                                for (int j = 0; j < Lay::W1_PER_SLOT; ++j) mbar_wait(&x_full[xb * KB1 + (sg * Lay::W1_PER_SLOT + j + ROT) % KB1], xph);
                            mbar_wait(&r_full[slot], ph);
                            fence_after();
#pragma unroll
                            for (int j = 0; j < Lay::W1_PER_SLOT; ++j) {
                                const int kb = (sg * Lay::W1_PER_SLOT + j + ROT) % KB1;
                                const uint64_t da = sw128_desc(xs + xb * Lay::X_BYTES + kb * 16384);
                                const uint64_t db = sw128_desc(ring + slot * Lay::SLOT + j * Lay::W1_HALF);
#pragma unroll
                                for (int kk = 0; kk < 4; ++kk)
                                    if (el) mma_bf16_2sm(d, da + uint64_t(kk * 2), db + uint64_t(kk * 2), id1, (sg | j | kk) != 0);
                            }
                            if (el) mma_commit_2sm(&r_empty[slot]);
                        }
                        if (el) mma_commit_2sm(&a1_full[b]);
                        if (c == NC - 1)
                            for (int kb = 0; kb < KB1; ++kb) if (el) mma_commit_2sm(&x_empty[xb * KB1 + kb]);
                        if (tr && it < 4) args.trace[it * 64 + c * 8 + 7] = clock64();
                    }
                    if (NXB == 1) xph ^= 1;
                }
            } else {
                constexpr uint32_t id2 = idesc_bf16(256, D);
                uint32_t hph = 0, a2ph = 0; // hph bit b: phase of h_full[b]
                int n = 0, it = 0;
                for (int tile = pair; tile < args.tiles; tile += npairs, ++it) {
                    for (int c = 0; c < NC; ++c, ++n) {
                        const int b = n & 1;
                        if (tr && it < 4) args.trace[it * 64 + c * 8 + 0] = clock64();
                        // acc2 += H(c) . W2(c)^T with A = bf16 hidden in TMEM. Hidden columns [64 kb + 16 g, +16)
                        // are GELU group g of warp-half kb, packed in place at TMEM cols 64 kb + 8 g: k-step g
                        // of W2 slot kb, issued as soon as that group lands in both CTAs.
                        const uint32_t a_base = tmem + 256 + b * MLP_HC;
                        if constexpr (EPK == EP_DEMIX) {
                            // pass j of warp group g = hidden columns [32 g + 16 j, +16), packed at TMEM columns
                            // 32 g + 8 j: every warp's first pass lands before its second, so the first
                            // pass of all four groups is issued while the second ones are still computed
#pragma unroll
                            for (int j = 0; j < 2; ++j)
#pragma unroll
                                for (int g = 0; g < MLP2_GG; ++g) {
                                    mbar_wait(&h_full[HG * b + 2 * g + j], (hph >> b) & 1u);
                                    fence_after();
                                    if (g == 0 && j == 0 && c == 0) {
                                        mbar_wait(a2_empty, a2ph ^ 1);
                                        a2ph ^= 1;
                                        fence_after();
                                    }
                                    uint32_t ph;
                                    const int slot = ring_slot(it * per_tile + pos_w2(c) + g / 2, ph);
                                    if (j == 0 && g % 2 == 0) {
                                        mbar_wait(&r_full[slot], ph);
                                        fence_after();
                                    }
                                    const uint64_t db = sw128_desc(ring + slot * Lay::SLOT);
                                    if (el) mma_bf16_2sm_ts(tmem, a_base + 32 * g + 8 * j, db + uint64_t(((g % 2) * 2 + j) * 2), id2,
                                                    (c | g | j) != 0);
                                    if (j == 1 && g % 2 == 1) if (el) mma_commit_2sm(&r_empty[slot]);
                                }
                        } else {
                        int slots[S2];
#pragma unroll
                        for (int g = 0; g < MLP2_GG; ++g) {
                            mbar_wait(&h_full[HG * b + g], (hph >> b) & 1u);
                            fence_after();
                            if (g == 0) {
                                if (tr && it < 4) args.trace[it * 64 + c * 8 + 1] = clock64();
                                if (c == 0) {
                                    mbar_wait(a2_empty, a2ph ^ 1);
                                    a2ph ^= 1;
                                    fence_after();
                                }
                            }
#pragma unroll
                            for (int kb = 0; kb < S2; ++kb) {
                                if (g == 0) {
                                    uint32_t ph;
                                    slots[kb] = ring_slot(it * per_tile + pos_w2(c) + kb, ph);
                                    mbar_wait(&r_full[slots[kb]], ph);
                                    fence_after();
                                }
                                const uint64_t db = sw128_desc(ring + slots[kb] * Lay::SLOT);
                                if (el) mma_bf16_2sm_ts(tmem, a_base + kb * 64 + g * 8, db + uint64_t(g * 2), id2, (c | kb | g) != 0);
                                if (g == MLP2_GG - 1) if (el) mma_commit_2sm(&r_empty[slots[kb]]);
                            }
                        }
                        }
                        hph ^= 1u << b;
                        if (el) mma_commit_2sm_mask(&a1_free[b], 1);
                        if (tr && it < 4) args.trace[it * 64 + c * 8 + 5] = clock64();
                    }
                    if (el) mma_commit_2sm(a2_full);
                }
            }
        }
    } else {
        // 8 epilogue warps: TMEM lane quarter = warp % 4; the two warps of a quarter own the two
        // 64-column halves of every hidden chunk, and alternate 64-column k-blocks of the output.
        const int quarter = warp % 4;
        const bool fin = EPK != EP_DEMIX && warp >= MLP2_FIN_WARP0; // final-epilogue-only warp
        const int half = fin ? (warp - MLP2_FIN_WARP0) / 4 : (warp - 2) / 4;
        const int row = quarter * 32 + lane;
        const uint32_t lane_off = uint32_t(quarter * 32) << 16;
        uint32_t e1ph = 0, e2ph = 0; // e1ph bit b: phase of a1_full[b]
        const Epi& ep = args.ep;
        auto release = [&](uint32_t leader_bar) { // elected remote arrive once the whole warp is done
            __syncwarp();
            if (lane == 0) mbar_arrive_cl(leader_bar);
        };
        int n = 0; // chunk counter across tiles: acc1 buffer = n & 1
        float svn[8]; // EP_DEMIX: the next chunk's S values
        for (int tile = pair; tile < args.tiles; tile += npairs) {
            const int it = (tile - pair) / npairs;
            if constexpr (EPK == EP_DEMIX) {
                // Module A intermediate logits -> demix -> evidence embedding (denoiser.cpp:86-139) with
                // Lambda-bar and r (x) S never leaving the chip: hidden = the Q symbol columns
                uint8_t* stg = smem + Lay::STG_OFF + (warp - 2) * Lay::STG_WARP;
                const int m0 = tile * 256 + int(rank) * 128 + quarter * 32;
                const int m0n = m0 + npairs * 256; // the next tile's rows
                if (tile == pair) { // first tile: nothing was prefetched
                    demix_load_sv<KK == 0 ? 8 : KK>(args, m0, half * 32, lane, svn);
                }
                for (int c = 0; c < NC; ++c, ++n) {
                    long long* tr = args.trace && blockIdx.x == 0 && it < 4 && warp == 2 && lane == 0 ? args.trace + it * 64 + c * 8 : nullptr;
                    const int b = n & 1;
                    const uint32_t base = tmem + lane_off + 256 + b * MLP_HC + half * 32;
                    float svc[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) svc[i] = svn[i];
                    // the next chunk's S (this tile's, or the next tile's first)
                    const int cn = c + 1 < NC ? c + 1 : 0, mn = c + 1 < NC ? m0 : m0n;
                    if (c + 1 < NC || tile + npairs < args.tiles) {
                        demix_load_sv<KK == 0 ? 8 : KK>(args, mn, cn * MLP_HC + half * 32, lane, svn);
                    }
                    if (c * MLP_HC + half * 32 >= ep.ldz) // (warp-uniform) padded symbol columns
                        demix_warp_pad(base, &a1_full[b], (e1ph >> b) & 1u, L_h_full0 + (HG * b + 2 * half) * 8, lane);
                    else
                        demix_warp<KK == 0 ? 8 : KK>(args, stg, base, &a1_full[b], (e1ph >> b) & 1u, L_h_full0 + (HG * b + 2 * half) * 8, svc, lane, tr);
                    e1ph ^= 1u << b;
                }
                const bool trf = args.trace && blockIdx.x == 0 && it < 4 && warp == 2 && lane == 0;
                if (trf) args.trace[512 + it * 4 + 0] = clock64();
                mbar_wait(a2_full, e2ph);
                e2ph ^= 1;
                fence_after();
                if (trf) args.trace[512 + it * 4 + 1] = clock64();
                {
                    // e k-block `half` of this warp's 32 rows, bf16 SW128, into the spent Z tile of this
                    // tile's buffer (MMA1 read it before MMA2 could finish); the X producer TMA-stores it
                    uint8_t* dst = xs + (it % NXB) * Lay::X_BYTES + half * 16384 + quarter * 4096;
#pragma unroll
                    for (int s2 = 0; s2 < 2; ++s2) {
                        float v[32];
                        tmem_ld32(tmem + lane_off + half * 64 + s2 * 32, v);
                        if (s2 == 1) {
                            fence_before();
                            __syncwarp();
                            if (lane == 0) mbar_arrive_cl(L_a2_empty);
                        }
#pragma unroll
                        for (int jj = 0; jj < 4; ++jj) {
                            const int j = s2 * 4 + jj;
                            uint32_t pk[4];
#pragma unroll
                            for (int t = 0; t < 4; ++t) {
                                __nv_bfloat162 b2 = __floats2bfloat162_rn(v[8 * jj + 2 * t], v[8 * jj + 2 * t + 1]);
                                pk[t] = *reinterpret_cast<uint32_t*>(&b2);
                            }
                            if (half < KBD) st_shared_v4(dst + lane * 128 + ((j ^ (lane & 7)) * 16), pk);
                        }
                    }
                    fence_proxy_async_smem();
                    __syncwarp();
                    // (D = 128: two output k-blocks; warps of halves 2, 3 only help drain acc2)
                    if (lane == 0 && half < KBD) mbar_arrive(&o_full[(it % NXB) * KBD + half]);
                }
                if (trf) args.trace[512 + it * 4 + 2] = clock64();
                continue;
            }
            if (!fin)
            for (int c = 0; c < NC; ++c, ++n) {
                const int b = n & 1;
                const float* b1 = (Lay::B1S_BYTES > 0 ? b1_s : args.b1) + c * MLP_HC + half * 64;
                const bool tr = args.trace && blockIdx.x == 0 && it < 4 && warp == 2 && lane == 0;
                if (tr) args.trace[it * 64 + c * 8 + 2] = clock64();
                mbar_wait(&a1_full[b], (e1ph >> b) & 1u);
                e1ph ^= 1u << b;
                fence_after();
                if (tr) args.trace[it * 64 + c * 8 + 3] = clock64();
                // fp32 columns [64 half, 64 half + 64) -> GELU -> bf16 pairs packed IN PLACE, group g (16
                // columns) at [8 g, 8 g + 8): every column is read (by this warp) before it is overwritten.
                const uint32_t base = tmem + lane_off + 256 + b * MLP_HC + half * 64;
#pragma unroll
                for (int g = 0; g < MLP2_GG; ++g) {
                    {
                        float4 bias4[4]; // this group's 16 hidden biases (L1-resident)
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            if constexpr (Lay::B1S_BYTES > 0) bias4[q] = *(reinterpret_cast<const float4*>(b1) + g * 4 + q); // (SMEM broadcast)
                            else bias4[q] = __ldg(reinterpret_cast<const float4*>(b1) + g * 4 + q);
                        }
                        float v[16];
                        tmem_ld16(base + g * 16, v);
                        uint32_t pk[8];
#pragma unroll
                        for (int i = 0; i < 16; i += 4) {
                            const float4 bb = bias4[i / 4];
                            pk[i / 2] = gelu2_bias_bf16(v[i], v[i + 1], bb.x, bb.y);
                            pk[i / 2 + 1] = gelu2_bias_bf16(v[i + 2], v[i + 3], bb.z, bb.w);
                        }
                        tmem_st8(base + g * 8, pk);
                        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                    }
                    fence_before();
                    release(L_h_full0 + (HG * b + g) * 8); // group g of both halves -> MMA2 k-step g
                }
                if (tr) args.trace[it * 64 + c * 8 + 4] = clock64();
            }
            if (!fin) continue;
            const int fsub = half; // first output k-block of this warp
            if (fsub >= KBD) continue;
            // final epilogue straight from TMEM: this thread's row, output k-blocks half, half + 2, ...
            // Gate / fusion read z (and e) from the tile's own X k-blocks in SMEM (X = [z | e] / [z~ | acc]:
            // they are kept until here) and write the bf16 result over the z k-block; the aggregator
            // stages in its per-warp block. Each warp's 32 x 64 result block then leaves by one TMA
            // store (SW128 box = the staging layout), so the epilogue warps never wait on HBM and the
            // write burst drains while the next tile's chunks run. A z / e k-block is handed back to the
            // X producer once the store out of it has been read.
            uint8_t* xcur = xs + (it % NXB) * Lay::X_BYTES; // this tile's row buffer
            const bool trf = args.trace && blockIdx.x == 0 && it < 4 && warp == MLP2_FIN_WARP0 + 2 && lane == 0;
            if (trf) args.trace[512 + it * 4 + 0] = clock64();
            mbar_wait(a2_full, e2ph);
            e2ph ^= 1;
            fence_after();
            if (trf) args.trace[512 + it * 4 + 1] = clock64();
#pragma unroll 1
            for (int kb = KB_SEQ ? 0 : fsub; kb < KBD; kb += KB_SEQ ? 1 : FIN_STRIDE) {
                const int n0 = kb * 64;
                // this warp's 32 rows of X k-block kb: z in (gate / fusion), the output block out (all)
                uint8_t* dst = xcur + kb * 16384 + quarter * 4096;
                const uint8_t* esrc = xcur + (KBD + kb) * 16384 + quarter * 4096;
#pragma unroll
                for (int s2i = 0; s2i < (KB_SEQ ? 1 : 2); ++s2i) { // 32-column halves of the k-block
                    const int s2 = KB_SEQ ? half : s2i;
                    float v[32];
                    tmem_ld32(tmem + lane_off + n0 + s2 * 32, v);
                    if (trf) args.trace[256 + it * 16 + (kb / 2) * 5 + 1 + s2] = clock64();
                    if (KB_SEQ ? kb == KBD - 1 : (s2 == 1 && kb + FIN_STRIDE >= KBD)) {
                        fence_before();
                        release(L_a2_empty); // accumulator drained: next tile's MMA2 may start
                    }
#pragma unroll
                    for (int i = 0; i < 32; i += 4) {
                        const float4 bb = *reinterpret_cast<const float4*>(bias_s + n0 + s2 * 32 + i); // SMEM broadcast
                        const float2 lo = __fadd2_rn(make_float2(v[i], v[i + 1]), make_float2(bb.x, bb.y));
                        const float2 hi = __fadd2_rn(make_float2(v[i + 2], v[i + 3]), make_float2(bb.z, bb.w));
                        v[i] = lo.x; v[i + 1] = lo.y; v[i + 2] = hi.x; v[i + 3] = hi.y;
                    }
#pragma unroll
                    for (int jj = 0; jj < 4; ++jj) { // 16-byte chunk j of this lane's row (SW128: at j ^ (row & 7))
                        const int j = s2 * 4 + jj;
                        const uint32_t off = uint32_t(lane * 128 + ((j ^ (lane & 7)) * 16));
                        uint32_t zq[4] = {0u, 0u, 0u, 0u}, eq[4] = {0u, 0u, 0u, 0u};
                        if (reads_z) ld_shared_v4(dst + off, zq);
                        if (reads_e) ld_shared_v4(esrc + off, eq);
                        uint32_t pk[4];
#pragma unroll
                        for (int t = 0; t < 4; ++t) {
                            const int i = jj * 8 + 2 * t;
                            float2 a = make_float2(v[i], v[i + 1]);
                            if (reads_z) {
                                const float2 z2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&zq[t]));
                                if (reads_e) {
                                    const float2 e2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&eq[t]));
                                    // g = 0.5 tanh(a / 2) + 0.5;  out = g z + (1 - g) e in the reference's form
                                    // (denoiser.cpp:156): a saturated gate passes z or e through exactly
                                    // (test_denoiser.cpp:141-159), which g (z - e) + e does not
                                    const float2 h = __fmul2_rn(a, make_float2(0.5f, 0.5f));
                                    const float2 g = __ffma2_rn(make_float2(tanh_approx(h.x), tanh_approx(h.y)), make_float2(0.5f, 0.5f),
                                                                make_float2(0.5f, 0.5f));
                                    const float2 ng = __fadd2_rn(make_float2(1.0f, 1.0f), make_float2(-g.x, -g.y));
                                    a = __ffma2_rn(g, z2, __fmul2_rn(ng, e2));
                                } else {
                                    a = __fadd2_rn(a, z2);
                                }
                            }
                            __nv_bfloat162 p = __floats2bfloat162_rn(a.x, a.y);
                            pk[t] = *reinterpret_cast<uint32_t*>(&p);
                        }
                        st_shared_v4(dst + off, pk);
                    }
                }
                if (trf) args.trace[256 + it * 16 + (kb / 2) * 5 + 3] = clock64();
                fence_proxy_async_smem(); // generic-proxy writes -> visible to the X producer's TMA store
                __syncwarp();
                if (lane == 0) {
                    if (reads_e) mbar_arrive(&x_empty[(it % NXB) * KB1 + KBD + kb]); // e k-block read: the next tile's may load
                    mbar_arrive(&o_full[(it % NXB) * KBD + kb]);   // output block staged
                }
            }
            if (trf) args.trace[512 + it * 4 + 2] = clock64();
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
