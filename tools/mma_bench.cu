// mma_bench.cu — tcgen05.mma throughput ceilings and interference, one CTA (or CTA pair) per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_bin/mma_bench tools/mma_bench.cu
// Variants: SS (A, B in SMEM) / TS (A in TMEM), N, cta_group, and concurrent noise:
//   noise=1: 8 warps hammer tcgen05.ld on a separate TMEM region (epilogue-like)
//   noise=2: 8 warps hammer ld/st.shared on a separate SMEM region
//   noise=3: 8 warps hammer tcgen05.ld + tcgen05.st
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>

#include "../paper_2605_26580_b200/csrc/kernels/mlp_tc2.cuh"

using namespace cider::tc;

__device__ __forceinline__ void mma_ts_1(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                 "r"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ CUtensorMap g_map; // set by host for NOISE==4
template <int N, int CG, bool TS, int NOISE, int ROT = 1>
__global__ void __launch_bounds__(320, 1) bench_kernel(int iters, unsigned long long* out, const __grid_constant__ CUtensorMap tmap) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint8_t* A = smem;                 // ROT x (128 x 64 bf16), 16 KB apart
    uint8_t* B = smem + 65536;         // ROT x (N(/2) x 64 bf16), 32 KB apart
    uint8_t* scratch = smem + 65536 + 131072 - 65536; // noise region overlaps the unused B tail (ROT<=2)
    static_assert(NOISE != 4 || ROT <= 2, "scratch overlaps B tiles 2-3");
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 65536 + 131072);  // [0] mma, [4..7] tma ring
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 2);
    volatile int* stop = reinterpret_cast<volatile int*>(bar + 3);
    for (int i = threadIdx.x; i < (65536 + 131072) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    const int warp = threadIdx.x / 32;
    uint32_t rank = 0;
    if (CG == 2) rank = cluster_rank();
    if (threadIdx.x == 0) { mbar_init(bar, 1); *stop = 0; asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    if (warp == 0) {
        if (CG == 1) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(slot)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(slot)));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    fence_before();
    if (CG == 2) cluster_sync_all(); else __syncthreads();
    fence_after();
    const uint32_t tmem = *slot;
    if (threadIdx.x == 0) {
        if (rank == 0) {
            const uint32_t idesc = idesc_bf16(128 * CG, N);
            long long t0 = clock64();
            for (int it = 0; it < iters; ++it) {
                const uint64_t da = sw128_desc(A + (it % ROT) * 16384), db = sw128_desc(B + (it % ROT) * 32768);
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    if (TS) {
                        if (CG == 1) mma_ts_1(tmem, tmem + 256 + kk * 8, db + kk * 2, idesc, 1);
                        else mma_bf16_2sm_ts(tmem, tmem + 256 + kk * 8, db + kk * 2, idesc, 1);
                    } else {
                        if (CG == 1) mma_bf16(tmem, da + kk * 2, db + kk * 2, idesc, 1);
                        else mma_bf16_2sm(tmem, da + kk * 2, db + kk * 2, idesc, 1);
                    }
                }
            }
            if (CG == 1) mma_commit(bar); else mma_commit_2sm(bar);
            mbar_wait(bar, 0);
            long long t1 = clock64();
            if (blockIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
        } else {
            mbar_wait(bar, 0);
        }
        *stop = 1;
    } else if (NOISE == 4 && threadIdx.x == 32) {
        // TMA stream of 16 KB boxes into a 4-slot scratch ring (64 KB), as a weight producer would
        uint64_t* tb = bar + 4;
        for (int s2 = 0; s2 < 4; ++s2) mbar_init(&tb[s2], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        uint32_t ph[4] = {0, 0, 0, 0};
        long long nbytes = 0;
        for (int i = 0; !*stop; ++i) {
            const int s2 = i % 4;
            if (i >= 4) { mbar_wait(&tb[s2], ph[s2]); ph[s2] ^= 1; }
            mbar_expect_tx(&tb[s2], 16384);
            tma_load_2d(scratch + s2 * 16384, &tmap, &tb[s2], 0, (i * 128 + blockIdx.x * 64) % 1024);
            nbytes += 16384;
        }
        for (int s2 = 0; s2 < 4; ++s2) mbar_wait(&tb[s2], ph[s2]);
        if (blockIdx.x == 0) out[1] = nbytes;
    } else if (warp >= 2 && (NOISE == 5 || NOISE == 6)) {
        // the fused MLP's hidden-chunk epilogue (TMEM ld x16 -> bias + GELU -> bf16 pack -> TMEM st x8 -> fence
        // -> arrive per 16 columns) on TMEM columns [256, 512), free-running beside the MMA stream: how many
        // elements per clock does it sustain while the tensor pipe is busy? (NOISE 6: bias in registers)
        const int quarter = warp % 4, half = (warp - 2) / 4;
        const uint32_t lane_off = uint32_t(quarter * 32) << 16;
        uint64_t* eb = bar + 8;
        if (threadIdx.x == 64) { for (int i = 0; i < 4; ++i) mbar_init(&eb[i], 8); }
        const float* b1 = reinterpret_cast<const float*>(scratch); // 0x3c003c00 pattern: small finite floats
        float4 breg[4];
        for (int q4 = 0; q4 < 4; ++q4) breg[q4] = reinterpret_cast<const float4*>(b1)[q4];
        unsigned long long groups = 0;
        int c = 0;
        while (!*stop) {
            const uint32_t base = tmem + lane_off + 256 + (c & 1) * 128 + half * 64;
            ++c;
#pragma unroll
            for (int g = 0; g < 4; ++g) {
                float4 bias4[4];
#pragma unroll
                for (int q4 = 0; q4 < 4; ++q4) bias4[q4] = NOISE == 6 ? breg[q4] : *(reinterpret_cast<const float4*>(b1) + ((c & 3) * 32 + half * 16 + g * 4 + q4));
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
                fence_before();
                __syncwarp();
                if (threadIdx.x % 32 == 0) mbar_arrive(&eb[g]);
            }
            groups += 4;
        }
        if (threadIdx.x % 32 == 0) atomicAdd(out + 1, groups * 16ull * 32ull); // elements
    } else if (warp >= 2 && NOISE && NOISE != 4) {
        const int quarter = warp % 4;
        const uint32_t ta = tmem + (uint32_t(quarter * 32) << 16) + 384;
        float v[32];
        uint32_t acc = 0;
        while (!*stop) {
            if (NOISE == 1 || NOISE == 3) {
                tmem_ld32(ta, v);
                acc += __float_as_uint(v[threadIdx.x % 32]);
                if (NOISE == 3) {
                    uint32_t pk[16];
                    for (int i = 0; i < 16; ++i) pk[i] = __float_as_uint(v[i]);
                    tmem_st16(ta + 64, pk);
                    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                }
            } else {
                uint4* p = reinterpret_cast<uint4*>(scratch) + (threadIdx.x % 256);
                uint4 x = p[0];
                x.x += 1;
                p[1024] = x;
            }
        }
        if (acc == 12345) out[1] = acc;
    }
    fence_before();
    if (CG == 2) cluster_sync_all(); else __syncthreads();
    if (warp == 0) {
        fence_after();
        if (CG == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
        else asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}


// The MLP issue pattern: per chunk 2 "W1 slots" of 8 SS MMAs (N=128 -> acc1[c&1]) and 2 "W2 slots"
// of 4 TS MMAs (N=256 -> acc2), each slot followed by a commit; COMMIT=0 drops the per-slot commits.
template <int CG, int COMMIT, int WAITS = 0, int RANDOM = 0>
__global__ void __launch_bounds__(128, 1) pattern_kernel(int chunks, unsigned long long* out) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 131072);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 8);
    for (int i = threadIdx.x; i < 131072 / 4; i += blockDim.x) {
        uint32_t h = uint32_t(i) * 2654435761u ^ (blockIdx.x * 40503u);
        h ^= h >> 15; h *= 2246822519u; h ^= h >> 13; h *= 3266489917u; h ^= h >> 16;
        // random sign / mantissa, exponent in [2^-3, 2^0]: bf16 = s eeeeeeee mmmmmmm
        const uint32_t lo = (h & 0x807fu) | ((0x7cu + ((h >> 7) & 3u)) << 7);
        const uint32_t hi = ((h >> 16) & 0x807fu) | ((0x7cu + ((h >> 23) & 3u)) << 7);
        reinterpret_cast<uint32_t*>(smem)[i] = RANDOM ? (lo | (hi << 16)) : 0x3c003c00u;
    }
    const int warp = threadIdx.x / 32;
    const uint32_t rank = CG == 2 ? cluster_rank() : 0;
    if (threadIdx.x == 0) { for (int i = 0; i < 8; ++i) mbar_init(&bar[i], 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    if (warp == 0) {
        if (CG == 1) { asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(slot))); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;"); }
        else { asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(slot))); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;"); }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    fence_before();
    if (CG == 2) cluster_sync_all(); else __syncthreads();
    fence_after();
    const uint32_t tmem = *slot;
    if (threadIdx.x == 0 && rank == 0) {
        const uint32_t id1 = idesc_bf16(128 * CG, 128), id2 = idesc_bf16(128 * CG, 256);
        if (WAITS) { mbar_arrive(&bar[6]); } // completes phase 0 of bar[6]
        long long t0 = clock64();
        int s = 0;
        for (int c = 0; c < chunks; ++c) {
            for (int w = 0; w < 2; ++w) { // W1 slots
                if (WAITS) { mbar_wait(&bar[6], 0); fence_after(); }
                const uint64_t da = sw128_desc(smem + ((c + w) % 4) * 16384), db = sw128_desc(smem + 65536 + ((c + w) % 4) * 16384);
                for (int j = 0; j < 2; ++j)
                    for (int kk = 0; kk < 4; ++kk) {
                        if (CG == 1) mma_bf16(tmem + 256 + (c & 1) * 128, da + j * 512 + kk * 2, db + j * 512 + kk * 2, id1, 1);
                        else mma_bf16_2sm(tmem + 256 + (c & 1) * 128, da + j * 512 + kk * 2, db + j * 512 + kk * 2, id1, 1);
                    }
                if (COMMIT) { if (CG == 1) mma_commit(&bar[s % 6]); else mma_commit_2sm(&bar[s % 6]); }
                ++s;
            }
            for (int w = 0; w < 2; ++w) { // W2 slots (TS)
                if (WAITS) { mbar_wait(&bar[6], 0); fence_after(); }
                const uint64_t db = sw128_desc(smem + 65536 + ((c + w) % 4) * 16384);
                for (int kk = 0; kk < 4; ++kk) {
                    if (CG == 1) mma_ts_1(tmem, tmem + 256 + ((c + 1) & 1) * 128 + w * 64 + kk * 8, db + kk * 2, id2, 1);
                    else mma_bf16_2sm_ts(tmem, tmem + 256 + ((c + 1) & 1) * 128 + w * 64 + kk * 8, db + kk * 2, id2, 1);
                }
                if (COMMIT) { if (CG == 1) mma_commit(&bar[s % 6]); else mma_commit_2sm(&bar[s % 6]); }
                ++s;
            }
        }
        uint64_t* fin = &bar[7];
        if (CG == 1) mma_commit(fin); else mma_commit_2sm(fin);
        // wait for the final commit: phase parity = number of completed phases of bar[7] so far, mod 2
        mbar_wait(fin, 0);
        long long t1 = clock64();
        if (blockIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
    }
    fence_before();
    if (CG == 2) cluster_sync_all(); else __syncthreads();
    if (warp == 0) {
        fence_after();
        if (CG == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
        else asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

template <int CG, int COMMIT, int WAITS = 0, int RANDOM = 0>
void run_pattern(int sms, const char* label, int chunks = 400) {
    unsigned long long* d;
    cudaMalloc(&d, 16);
    const int smem = 131072 + 1024 + 128;
    auto k = pattern_kernel<CG, COMMIT, WAITS, RANDOM>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sms);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CG; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k, chunks, d);
    cudaError_t err = cudaDeviceSynchronize();
    unsigned long long cyc = 0;
    cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
    const double ideal = chunks * 2048.0 * (CG == 2 ? 1.0 : 2.0); // 2-SM: 2048 clk/chunk; 1-SM: double the MMA cycles
    printf("%-40s cg=%d commit=%d: %.0f cyc/chunk (ideal %.0f) -> %.0f%%  %s\n", label, CG, COMMIT, double(cyc) / chunks,
           ideal / chunks, 100.0 * ideal / double(cyc), err == cudaSuccess ? "" : cudaGetErrorString(err));
    cudaFree(d);
}


// Two issuers: thread 0 issues the W1 slots (SS N=128 -> acc1), thread 32 the W2 slots (TS N=256 ->
// acc2); each stalls STALL cycles (spin on clock64) before every slot, as a try_wait would.
template <int ISSUERS, int STALL>
__global__ void __launch_bounds__(128, 1) issue2_kernel(int chunks, unsigned long long* out) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 131072);
    uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 16);
    for (int i = threadIdx.x; i < 131072 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    const int warp = threadIdx.x / 32;
    const uint32_t rank = cluster_rank();
    if (threadIdx.x == 0) { for (int i = 0; i < 16; ++i) mbar_init(&bar[i], 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    if (warp == 0) { asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(slot))); asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;"); }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    fence_before();
    cluster_sync_all();
    fence_after();
    const uint32_t tmem = *slot;
    auto stall = [] { if (STALL) { const long long t = clock64(); while (clock64() - t < STALL) {} } };
    const uint32_t id1 = idesc_bf16(256, 128), id2 = idesc_bf16(256, 256);
    auto w1 = [&](int c, int w) {
        const uint64_t da = sw128_desc(smem + ((c + w) % 4) * 16384), db = sw128_desc(smem + 65536 + ((c + w) % 4) * 16384);
        for (int j = 0; j < 2; ++j)
            for (int kk = 0; kk < 4; ++kk) mma_bf16_2sm(tmem + 256 + (c & 1) * 128, da + j * 512 + kk * 2, db + j * 512 + kk * 2, id1, 1);
    };
    auto w2 = [&](int c, int w) {
        const uint64_t db = sw128_desc(smem + 65536 + ((c + w) % 4) * 16384);
        for (int kk = 0; kk < 4; ++kk) mma_bf16_2sm_ts(tmem, tmem + 256 + ((c + 1) & 1) * 128 + w * 64 + kk * 8, db + kk * 2, id2, 1);
    };
    if (rank == 0 && (threadIdx.x == 0 || (ISSUERS == 2 && threadIdx.x == 32))) {
        const bool first = threadIdx.x == 0;
        long long t0 = clock64();
        int s = first ? 0 : 8;
        for (int c = 0; c < chunks; ++c) {
            if (ISSUERS == 1 || first)
                for (int w = 0; w < 2; ++w) { stall(); w1(c, w); mma_commit_2sm(&bar[s % 6]); ++s; }
            if (ISSUERS == 1 || !first)
                for (int w = 0; w < 2; ++w) { stall(); w2(c, w); mma_commit_2sm(&bar[(ISSUERS == 1 ? 0 : 8) + s % 6]); ++s; }
        }
        uint64_t* fin = &bar[first ? 7 : 15];
        mma_commit_2sm(fin);
        mbar_wait(fin, 0);
        long long t1 = clock64();
        if (blockIdx.x == 0) out[first ? 0 : 1] = (unsigned long long)(t1 - t0);
    }
    fence_before();
    cluster_sync_all();
    if (warp == 0) {
        fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    }
}

template <int ISSUERS, int STALL>
void run_issue2(int sms, const char* label) {
    unsigned long long* d;
    cudaMalloc(&d, 16);
    cudaMemset(d, 0, 16);
    const int smem = 131072 + 1024 + 256;
    auto k = issue2_kernel<ISSUERS, STALL>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int chunks = 2000;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sms);
    cfg.blockDim = dim3(128);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k, chunks, d);
    cudaError_t err = cudaDeviceSynchronize();
    unsigned long long cyc[2] = {0, 0};
    cudaMemcpy(cyc, d, 16, cudaMemcpyDeviceToHost);
    const unsigned long long c = cyc[0] > cyc[1] ? cyc[0] : cyc[1];
    printf("%-44s: %.0f cyc/chunk (ideal 2048) -> %.0f%%  %s\n", label, double(c) / chunks, 100.0 * 2048.0 * chunks / double(c),
           err == cudaSuccess ? "" : cudaGetErrorString(err));
    cudaFree(d);
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static CUtensorMap h_map;
template <int N, int CG, bool TS, int NOISE, int ROT = 1>
void run(int sms, const char* label) {
    unsigned long long* d;
    cudaMalloc(&d, 16);
    const int smem = 65536 + 131072 + 1024 + 64;
    auto k = bench_kernel<N, CG, TS, NOISE, ROT>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 2048;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sms);
    cfg.blockDim = dim3(320);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CG;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k, iters, d, h_map);
    cudaMemset(d, 0, 16);
    cudaLaunchKernelEx(&cfg, k, iters, d, h_map);
    cudaError_t err = cudaDeviceSynchronize();
    unsigned long long cyc = 0, tb = 0;
    cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(&tb, d + 1, 8, cudaMemcpyDeviceToHost);
    if (NOISE == 4) printf("   (TMA streamed %.1f B/clk/SM alongside)\n", double(tb) / double(cyc));
    if (NOISE == 5 || NOISE == 6) printf("   (GELU epilogue on 8 warps alongside: %.2f elements/clk/SM)\n", double(tb) / double(cyc) / (sms));
    const double macs = double(iters) * 4 * (128.0 * CG) * N * 16;
    printf("%-34s N=%3d cg=%d %s: %6.1f cyc/MMA  %5.0f MAC/clk/SM  (%.0f%% of 4096)\n", label, N, CG, TS ? "TS" : "SS",
           double(cyc) / (iters * 4.0), macs / CG / double(cyc), 100.0 * macs / CG / double(cyc) / 4096.0);
    if (err != cudaSuccess) printf("  error: %s\n", cudaGetErrorString(err));
    cudaFree(d);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    void* mat;
    cudaMalloc(&mat, size_t(1024) * 256 * 2);
    cudaMemset(mat, 0, size_t(1024) * 256 * 2);
    cuuint64_t dims[2] = {256, 1024};
    cuuint64_t strides[1] = {512};
    cuuint32_t box[2] = {64, 128};
    cuuint32_t es[2] = {1, 1};
    reinterpret_cast<EncodeFn>(p)(&h_map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, mat, dims, strides, box, es,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    run<128, 2, false, 5, 2>(sms, "SS N=128 2-SM + GELU epilogue");
    run<128, 2, true, 5, 2>(sms, "TS N=128 2-SM + GELU epilogue");
    run<128, 2, false, 6, 2>(sms, "SS N=128 2-SM + GELU epi (reg bias)");
    run<256, 2, true, 5, 2>(sms, "TS N=256 2-SM + GELU epilogue");
    run<128, 2, false, 0, 2>(sms, "SS N=128 2-SM quiet");
    run<128, 2, false, 2, 2>(sms, "SS N=128 2-SM + SMEM ld/st noise");
    run<128, 2, false, 4, 2>(sms, "SS N=128 2-SM + TMA stream");
    run<128, 2, false, 3, 2>(sms, "SS N=128 2-SM + TMEM ld/st noise");
    run<256, 2, false, 2, 2>(sms, "SS N=256 2-SM + SMEM ld/st noise");
    run<256, 2, false, 4, 2>(sms, "SS N=256 2-SM + TMA stream");
    run<256, 2, true, 2, 2>(sms, "TS N=256 2-SM + SMEM ld/st noise");
    return 0;
}
