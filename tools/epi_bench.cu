// Microbenchmark of the fused-MLP hidden-chunk epilogue WITHOUT the MMAs: TMEM load -> bias + GELU ->
// bf16 pack -> TMEM store -> fence -> elected mbarrier arrive, per 16-column group, over 128-row x
// 128-column chunks per SM. Reports cycles per chunk for 8 / 16 warps and variants of the loop.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o epi_bench tools/epi_bench.cu && ./epi_bench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

__device__ __forceinline__ float tanh_approx(float x) { float y; asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint32_t gelu2_bias_bf16(float x0, float x1, float b0, float b1) {
    const float2 x = __fadd2_rn(make_float2(x0, x1), make_float2(b0, b1));
    const float2 p = __ffma2_rn(__fmul2_rn(x, x), make_float2(0.0356774081f, 0.0356774081f), make_float2(0.7978845608f, 0.7978845608f));
    const float2 in = __fmul2_rn(x, p);
    const float2 y = __ffma2_rn(x, make_float2(tanh_approx(in.x), tanh_approx(in.y)), x);
    __nv_bfloat162 r = __floats2bfloat162_rn(y.x, y.y);
    return *reinterpret_cast<uint32_t*>(&r);
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n\t"
        "tcgen05.wait::ld.sync.aligned;"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr) : "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(v[0]), "r"(v[1]),
                 "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
}
// MODE bits: 1 = bias from registers (no LDG), 2 = no fence/arrive, 4 = no TMEM store, 8 = no GELU (copy), 16 = no TMEM load
template <int MODE>
__global__ void __launch_bounds__(512, 1) k(const float* bias, float* out, long long* cyc, int chunks, int warps) {
    __shared__ uint64_t bar[8];
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0)
        for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar[i])), "r"(warps / 4 * 4));
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = slot;
    const int quarter = warp % 4, cb = warp / 4, ncb = warps / 4; // column blocks of 128 / ncb columns
    const int HCW = 128 / ncb, GPW = HCW / 16;
    const uint32_t lane_off = uint32_t(quarter * 32) << 16;
    float acc = 0;
    float4 breg[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) breg[q] = reinterpret_cast<const float4*>(bias)[q];
    const long long t0 = clock64();
    for (int c = 0; c < chunks; ++c) {
        const uint32_t base = tmem + lane_off + 256 + (c & 1) * 128 + cb * HCW;
        const float* b1 = bias + (c & 3) * 128 + cb * HCW;
        for (int g = 0; g < GPW; ++g) {
            float4 bias4[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) bias4[q] = (MODE & 1) ? breg[q] : __ldg(reinterpret_cast<const float4*>(b1) + g * 4 + q);
            float v[16];
            if (MODE & 16) {
#pragma unroll
                for (int i = 0; i < 16; ++i) v[i] = acc + i;
            } else tmem_ld16(base + g * 16, v);
            uint32_t pk[8];
#pragma unroll
            for (int i = 0; i < 16; i += 4) {
                const float4 bb = bias4[i / 4];
                if (MODE & 8) {
                    pk[i / 2] = __float_as_uint(v[i] + bb.x); pk[i / 2 + 1] = __float_as_uint(v[i + 2] + bb.z);
                } else {
                    pk[i / 2] = gelu2_bias_bf16(v[i], v[i + 1], bb.x, bb.y);
                    pk[i / 2 + 1] = gelu2_bias_bf16(v[i + 2], v[i + 3], bb.z, bb.w);
                }
            }
            if (MODE & 4) {
#pragma unroll
                for (int i = 0; i < 8; ++i) acc += __uint_as_float(pk[i]);
            } else {
                tmem_st8(base + g * 8, pk);
                asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            }
            if (!(MODE & 2)) {
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar[g])) : "memory");
            }
        }
    }
    const long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}


__device__ __forceinline__ void tmem_ld16_nw(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld16(uint32_t (&r)[16]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                   "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15])
                 :: "memory");
}
// BIAS: 0 = __ldg, 1 = shared memory, 2 = registers. GW: columns per released group (16 or 32).
// PIPE: the next 16 columns' TMEM load is in flight while this group is GELU'd. NOWAITST: no wait::st
// before the fence (tcgen05.fence::before_thread_sync orders the stores)
template <int BIAS, int GW, bool PIPE, bool NOWAITST>
__global__ void __launch_bounds__(512, 1) k2(const float* bias, float* out, long long* cyc, int chunks, int warps) {
    __shared__ uint64_t bar[8];
    __shared__ uint32_t slot;
    __shared__ __align__(16) float bias_s[1024];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) bias_s[i] = bias[i];
    if (threadIdx.x == 0)
        for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar[i])), "r"(warps / 4 * 4));
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = slot;
    const int quarter = warp % 4, cb = warp / 4, ncb = warps / 4;
    const int HCW = 128 / ncb, NG16 = HCW / 16;
    const uint32_t lane_off = uint32_t(quarter * 32) << 16;
    float acc = 0;
    float4 breg[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) breg[q] = reinterpret_cast<const float4*>(bias)[q];
    const long long t0 = clock64();
    uint32_t nxt[16];
    if (PIPE) tmem_ld16_nw(tmem + lane_off + 256 + cb * HCW, nxt);
    for (int c = 0; c < chunks; ++c) {
        const uint32_t base = tmem + lane_off + 256 + (c & 1) * 128 + cb * HCW;
        const uint32_t nbase = tmem + lane_off + 256 + ((c + 1) & 1) * 128 + cb * HCW;
        const float* b1 = bias + (c & 3) * 128 + cb * HCW;
        const float* b1s = bias_s + (c & 3) * 128 + cb * HCW;
        for (int g = 0; g < NG16; ++g) {
            float4 bias4[4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
                bias4[q] = BIAS == 2 ? breg[q] : BIAS == 1 ? *(reinterpret_cast<const float4*>(b1s) + g * 4 + q) : __ldg(reinterpret_cast<const float4*>(b1) + g * 4 + q);
            float v[16];
            if (PIPE) {
                tmem_wait_ld16(nxt);
#pragma unroll
                for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(nxt[i]);
                tmem_ld16_nw(g + 1 < NG16 ? base + (g + 1) * 16 : nbase, nxt);
            } else tmem_ld16(base + g * 16, v);
            uint32_t pk[8];
#pragma unroll
            for (int i = 0; i < 16; i += 4) {
                const float4 bb = bias4[i / 4];
                pk[i / 2] = gelu2_bias_bf16(v[i], v[i + 1], bb.x, bb.y);
                pk[i / 2 + 1] = gelu2_bias_bf16(v[i + 2], v[i + 3], bb.z, bb.w);
            }
            tmem_st8(base + g * 8, pk);
            if (GW == 16 || (g & 1)) {
                if (!NOWAITST) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
                asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
                __syncwarp();
                if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar[g])) : "memory");
            }
        }
    }
    if (PIPE) tmem_wait_ld16(nxt);
    const long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc + __uint_as_float(nxt[0]);
    __syncthreads();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int BIAS, int GW, bool PIPE, bool NOWAITST>
void run2(const char* name) {
    float *out, *bias; long long* cyc;
    cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8); cudaMalloc(&bias, 4096); cudaMemset(bias, 0, 4096);
    const int chunks = 2048;
    for (int warps : {8, 16}) {
        k2<BIAS, GW, PIPE, NOWAITST><<<148, warps * 32>>>(bias, out, cyc, chunks, warps);
        k2<BIAS, GW, PIPE, NOWAITST><<<148, warps * 32>>>(bias, out, cyc, chunks, warps);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
        long long h[148]; cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
        double c = 0; for (int i = 0; i < 148; ++i) c += h[i]; c /= 148;
        printf("%-44s warps %2d: %7.0f cycles per 128x128 chunk (%5.2f elems/clk/SM)\n", name, warps, c / chunks, 16384.0 * chunks / c);
    }
    cudaFree(out); cudaFree(cyc); cudaFree(bias);
}

template <int MODE>
void run(const char* name) {
    float *out, *bias; long long* cyc;
    cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8); cudaMalloc(&bias, 4096); cudaMemset(bias, 0, 4096);
    const int chunks = 2048;
    for (int warps : {8, 16}) {
        k<MODE><<<148, warps * 32>>>(bias, out, cyc, chunks, warps);
        k<MODE><<<148, warps * 32>>>(bias, out, cyc, chunks, warps);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
        long long h[148]; cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
        double c = 0; for (int i = 0; i < 148; ++i) c += h[i]; c /= 148;
        printf("%-44s warps %2d: %7.0f cycles per 128x128 chunk (%5.2f elems/clk/SM)\n", name, warps, c / chunks, 16384.0 * chunks / c);
    }
    cudaFree(out); cudaFree(cyc); cudaFree(bias);
}

int main() {
    run<0>("full loop (as in mlp_tc2)");
    run<1>("bias in registers");
    run<2>("no fence / arrive");
    run<3>("bias in registers, no fence / arrive");
    run<4>("no TMEM store");
    run<16>("no TMEM load");
    run<8>("no GELU (ld, add, st, arrive)");
    run<1 | 2 | 4 | 16>("GELU only");
    run2<0, 16, false, false>("k2 ldg bias, 16-col groups");
    run2<1, 16, false, false>("k2 smem bias");
    run2<1, 32, false, false>("k2 smem bias, 32-col release");
    run2<1, 16, true, false>("k2 smem bias, prefetched TMEM load");
    run2<1, 32, true, false>("k2 smem bias, 32-col release, prefetch");
    run2<1, 16, false, true>("k2 smem bias, no wait::st");
    run2<1, 32, true, true>("k2 smem bias, 32-col, prefetch, no wait::st");
    run2<2, 32, true, true>("k2 reg bias, 32-col, prefetch, no wait::st");
    return 0;
}
