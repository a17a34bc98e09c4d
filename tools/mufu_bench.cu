// Microbenchmark: per-SM throughput of MUFU.TANH / MUFU.EX2 / FFMA2 / F2FP and of their mixes, with
// 4 / 8 / 16 warps per SM (one CTA per SM). Answers: what bounds the fused-MLP GELU epilogue?
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o mufu_bench tools/mufu_bench.cu && ./mufu_bench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

__device__ __forceinline__ float tanh_approx(float x) { float y; asm volatile("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float ex2_approx(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float rcp_approx(float x) { float y; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }

template <int MODE>
__global__ void k(float* out, long long* cyc, int iters) {
    float v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = threadIdx.x * 1e-3f + i * 0.1f;
    float2 a[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) a[i] = make_float2(v[2 * i], v[2 * i + 1]);
    __syncthreads();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0) { // 8 tanh
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = tanh_approx(v[i]);
        } else if (MODE == 1) { // 8 ex2
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = ex2_approx(v[i]);
        } else if (MODE == 2) { // 8 FFMA2 (16 fp32 fma per lane)
#pragma unroll
            for (int r = 0; r < 2; ++r)
#pragma unroll
                for (int i = 0; i < 4; ++i) a[i] = __ffma2_rn(a[i], make_float2(0.999f, 1.001f), make_float2(1e-3f, -1e-3f));
        } else if (MODE == 3) { // GELU mix: per pair 1 FADD2, 2 FMUL2, 2 FFMA2, 2 tanh, 1 cvt pack  (4 pairs)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float2 x = __fadd2_rn(a[i], make_float2(0.01f, 0.02f));
                const float2 p = __ffma2_rn(__fmul2_rn(x, x), make_float2(0.0356774081f, 0.0356774081f), make_float2(0.7978845608f, 0.7978845608f));
                const float2 in = __fmul2_rn(x, p);
                const float2 y = __ffma2_rn(x, make_float2(tanh_approx(in.x), tanh_approx(in.y)), x);
                __nv_bfloat162 r = __floats2bfloat162_rn(y.x, y.y);
                a[i] = make_float2(__uint_as_float(*reinterpret_cast<uint32_t*>(&r)), y.y);
            }
        } else if (MODE == 4) { // 8 tanh + 8 independent FFMA2
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = tanh_approx(v[i]);
#pragma unroll
            for (int r = 0; r < 2; ++r)
#pragma unroll
                for (int i = 0; i < 4; ++i) a[i] = __ffma2_rn(a[i], make_float2(0.999f, 1.001f), make_float2(1e-3f, -1e-3f));
        } else if (MODE == 5) { // 8 cvt packs
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                __nv_bfloat162 r = __floats2bfloat162_rn(v[i], v[(i + 1) & 7]);
                v[i] = __uint_as_float(*reinterpret_cast<uint32_t*>(&r)) + 1.0f;
            }
        } else if (MODE == 6) { // sigmoid form: ex2 + rcp per element (8 elements)
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = rcp_approx(1.0f + ex2_approx(v[i]));
        } else if (MODE == 7) { // 4 tanh + 4 (ex2 + rcp)
#pragma unroll
            for (int i = 0; i < 4; ++i) v[i] = tanh_approx(v[i]);
#pragma unroll
            for (int i = 4; i < 8; ++i) v[i] = rcp_approx(1.0f + ex2_approx(v[i]));
        }
    }
    const long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += v[i];
#pragma unroll
    for (int i = 0; i < 4; ++i) s += a[i].x + a[i].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, double elems_per_iter_lane) {
    float* out; long long* cyc;
    cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
    const int iters = 4096;
    for (int warps : {4, 8, 16, 32}) {
        k<MODE><<<148, warps * 32>>>(out, cyc, iters);
        k<MODE><<<148, warps * 32>>>(out, cyc, iters);
        cudaDeviceSynchronize();
        long long h[148]; cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
        double c = 0; for (int i = 0; i < 148; ++i) c += h[i]; c /= 148;
        printf("%-34s warps/SM %2d: %8.0f cycles, %6.2f elems/clk/SM\n", name, warps, c, elems_per_iter_lane * iters * warps * 32 / c);
    }
    cudaFree(out); cudaFree(cyc);
}

int main() {
    run<0>("MUFU.TANH", 8);
    run<1>("MUFU.EX2", 8);
    run<6>("EX2+RCP (elements)", 8);
    run<7>("4 TANH + 4 (EX2+RCP) (elements)", 8);
    run<2>("FFMA2 (fp32 fma)", 16);
    run<5>("F2FP pack (+FADD) (packs)", 8);
    run<3>("GELU mix (elements)", 8);
    run<4>("8 TANH + 8 FFMA2 (tanh)", 8);
    return 0;
}
