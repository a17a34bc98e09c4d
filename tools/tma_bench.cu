// tma_bench.cu — per-SM TMA load throughput for weight-tile boxes (L2-resident source), one
// producer thread per CTA streaming into a 12-slot ring of 16 KB.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_bin/tma_bench tools/tma_bench.cu -lcuda
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>

#include "../paper_2605_26580_b200/csrc/kernels/mlp_tc2.cuh"

using namespace cider::tc;

template <int ROWS, int PER_SLOT>
__global__ void __launch_bounds__(64, 1) tma_kernel(const __grid_constant__ CUtensorMap map, int iters, int mat_rows,
                                                    unsigned long long* out) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    constexpr int NS = 12;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + NS * 16384);
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const int box_bytes = ROWS * 128;
        long long t0 = clock64();
        uint32_t ph[NS] = {};
        for (int i = 0; i < iters; ++i) {
            const int s = i % NS;
            if (i >= NS) { mbar_wait(&full[s], ph[s]); ph[s] ^= 1; }
            mbar_expect_tx(&full[s], box_bytes * PER_SLOT);
            for (int j = 0; j < PER_SLOT; ++j) {
                const int row = ((i * PER_SLOT + j) * ROWS + blockIdx.x * 64) % mat_rows;
                tma_load_2d(smem + s * 16384 + j * box_bytes, &map, &full[s], ((i + j) % 4) * 64, row);
            }
        }
        for (int s = 0; s < NS; ++s) mbar_wait(&full[s], ph[s]);
        long long t1 = clock64();
        if (blockIdx.x == 0) out[0] = (unsigned long long)(t1 - t0);
    }
    __syncthreads();
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int ROWS, int PER_SLOT>
void run(EncodeFn enc, void* mat, int rows, int cols, int sms) {
    CUtensorMap m;
    cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
    cuuint64_t strides[1] = {cuuint64_t(cols) * 2};
    cuuint32_t box[2] = {64, ROWS};
    cuuint32_t es[2] = {1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, mat, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    unsigned long long* d;
    cudaMalloc(&d, 8);
    const int smem = 12 * 16384 + 1024 + 256;
    cudaFuncSetAttribute(tma_kernel<ROWS, PER_SLOT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 3000;
    tma_kernel<ROWS, PER_SLOT><<<sms, 64, smem>>>(m, iters, rows, d);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    tma_kernel<ROWS, PER_SLOT><<<sms, 64, smem>>>(m, iters, rows, d);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    unsigned long long cyc;
    cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = double(iters) * ROWS * 128 * PER_SLOT;
    printf("box 64x%-3d x%d per slot (%5d B/slot), row stride %5d B: %6.1f B/clk/SM, %6.1f cyc/box, chip %.2f TB/s %s\n", ROWS,
           PER_SLOT, ROWS * 128 * PER_SLOT, cols * 2, bytes / cyc, double(cyc) / (iters * PER_SLOT),
           bytes * sms / (ms * 1e-3) / 1e12, err == cudaSuccess ? "" : cudaGetErrorString(err));
    cudaFree(d);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    EncodeFn enc = reinterpret_cast<EncodeFn>(p);
    void* mat;
    cudaMalloc(&mat, size_t(1024) * 1024 * 2);
    cudaMemset(mat, 0, size_t(1024) * 1024 * 2);
    // W1-like: 1024 rows x 256 cols (512 B stride); W2-like: 256 rows x 1024 cols (2 KB stride)
    run<128, 1>(enc, mat, 1024, 256, sms);
    run<64, 2>(enc, mat, 1024, 256, sms);
    run<64, 1>(enc, mat, 1024, 256, sms);
    run<128, 1>(enc, mat, 256, 1024, sms);
    run<32, 1>(enc, mat, 1024, 256, sms);
    return 0;
}
