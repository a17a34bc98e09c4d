// engine.cu — libcider's device engine and C ABI (include/cider.h).
//
// One cider_ctx per device: it owns the weights (uploaded once, fp32 or bf16), the Tanner
// tables (edge slots, coefficient permutations, CSR lists), one CUDA stream and a chunk
// workspace sized for HBM. A forward (= StructuredDenoiser::logits, denoiser.cpp:253-259)
// is a fixed chain of GEMMs (tcgen05 in BF16 mode, SIMT in FP32 mode) and HBM-bound Tanner
// kernels; the refinement loop (refine.cpp:134-292) runs entirely on the device — reveal,
// residual forcing, the gamma=0 pass, remask selection — with no host round trip except the
// per-stage bucket sizes of threshold remasking.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <memory>
#include <atomic>
#include <mutex>
#include <string>
#include <tuple>
#include <thread>
#include <vector>

#include <nvtx3/nvToolsExt.h> // header-only NVTX3: no-ops unless a tool (ncu --nvtx, nsys) is attached

#include "host/host.hpp"
#include "kernels/common.cuh"
#include "kernels/gemm_simt.cuh"
#include "kernels/gemm_tc.cuh"
#include "kernels/mlp_tc.cuh"
#include "kernels/mlp_tc2.cuh"
#include "kernels/gemm_grp.cuh"
#include "kernels/pool_mma.cuh"
#include "kernels/wht.cuh"
#include "kernels/bp.cuh"
#include "kernels/workload.cuh"
#include "kernels/path.cuh"
#include "kernels/amp.cuh"

namespace cider {
const char* host_last_error();

namespace {

thread_local std::string g_err;
thread_local uint64_t g_err_tick = 0;

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

const double kPi = 3.14159265358979323846;
double cosine_fraction(int t, int T) { return 0.5 * (1.0 - std::cos(kPi * t / T)); }   // refine.cpp:11-15
double infer_temperature(int t, int T, double tmax, double tmin) {                       // refine.cpp:17-21
    if (T <= 1) return tmin;
    double w = 0.5 * (1.0 + std::cos(kPi * (t - 1) / (T - 1)));
    return tmax * w + tmin * (1.0 - w);
}
int remask_steps(int T, int low, int K) {                                                // refine.cpp:23-26
    int t = int((static_cast<long long>(T) * low) / K);
    return t < 1 ? 1 : t;
}

// ---- TMA descriptors -------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    if (!fn) throw CudaError("cuTensorMapEncodeTiled unavailable");
    return fn;
}

// cudaFuncSetAttribute acts on the current device's instance of a kernel: one flag per device, so that a
// process driving several GPUs (one cider_ctx per device) sets the attribute on each of them
struct PerDeviceOnce {
    std::atomic<uint64_t> done{0};
    std::mutex mu;
    template <class F>
    void run(int device, F&& f) {
        const uint64_t bit = 1ull << (unsigned(device) & 63u);
        if (done.load(std::memory_order_acquire) & bit) return;
        std::lock_guard<std::mutex> g(mu);
        if (done.load(std::memory_order_relaxed) & bit) return;
        f();
        done.fetch_or(bit, std::memory_order_release);
    }
};
inline int current_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d;
}

// bf16 row-major [rows x cols] with row stride ld (elements), box = box_rows x 64, SWIZZLE_128B
CUtensorMap make_map(const void* ptr, int64_t rows, int cols, int ld, int box_rows) {
    CUtensorMap m;
    cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
    cuuint64_t strides[1] = {cuuint64_t(ld) * 2};
    cuuint32_t box[2] = {64, cuuint32_t(box_rows)};
    cuuint32_t es[2] = {1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")");
    return m;
}

// 2-D bf16 map with an explicit box and swizzle (TMA store boxes of the fused MLP epilogues)
CUtensorMap make_map_box(const void* ptr, int64_t rows, int cols, int ld, int box_cols, int box_rows, CUtensorMapSwizzle swz) {
    CUtensorMap m;
    cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
    cuuint64_t strides[1] = {cuuint64_t(ld) * 2};
    cuuint32_t box[2] = {cuuint32_t(box_cols), cuuint32_t(box_rows)};
    cuuint32_t es[2] = {1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (box) failed (" + std::to_string(int(r)) + ")");
    return m;
}

// W1 of the 2-SM MLP as {64 cols, rows, k-blocks}: one box = box_rows rows x 2 k-blocks (16 KB)
CUtensorMap make_map_w1_3d(const void* ptr, int64_t rows, int cols, int box_rows, int box_kb = 2) {
    CUtensorMap m;
    cuuint64_t dims[3] = {64, cuuint64_t(rows), cuuint64_t(cols / 64)};
    cuuint64_t strides[2] = {cuuint64_t(cols) * 2, 128};
    cuuint32_t box[3] = {64, cuuint32_t(box_rows), cuuint32_t(box_kb)};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (3d) failed (" + std::to_string(int(r)) + ")");
    return m;
}

// Rows of a [bins][blocks][K] x cols bf16 tensor as a 3-D map {cols, blocks*K, bins}: one box =
// K rows of one block for bb consecutive bins (gemm_grp.cuh A operands).
CUtensorMap make_map_rows3d(const void* ptr, int bins, int rows_per_bin, int cols, int K, int bb) {
    CUtensorMap m;
    cuuint64_t dims[3] = {cuuint64_t(cols), cuuint64_t(rows_per_bin), cuuint64_t(bins)};
    cuuint64_t strides[2] = {cuuint64_t(cols) * 2, cuuint64_t(rows_per_bin) * cols * 2};
    cuuint32_t box[3] = {64, cuuint32_t(K), cuuint32_t(bb)};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (rows3d) failed (" + std::to_string(int(r)) + ")");
    return m;
}
// The T table [alpha][n][k] as {k, n, alpha}, box {64, 256, 1}.
CUtensorMap make_map_ttab(const void* ptr, int D, int Q, int box_rows = 0) {
    CUtensorMap m;
    cuuint64_t dims[3] = {cuuint64_t(D), cuuint64_t(D), cuuint64_t(Q)};
    cuuint64_t strides[2] = {cuuint64_t(D) * 2, cuuint64_t(D) * D * 2};
    cuuint32_t box[3] = {64, cuuint32_t(box_rows > 0 ? box_rows : D), 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (ttab) failed (" + std::to_string(int(r)) + ")");
    return m;
}

// ---- device allocations ------------------------------------------------------------------
// bumped on every device (re)allocation: captured CUDA graphs bake in device pointers
inline int64_t& alloc_generation() {
    static int64_t g = 0;
    return g;
}
struct DevBuf {
    void* p = nullptr;    // usable region
    void* base = nullptr; // allocation (p - guard)
    size_t bytes = 0, guard = 0;
    // g > 0 (debug): `g`-byte guard bands of 0xA5 before and after the usable region
    void ensure(size_t n, size_t g = 0) {
        if (n <= bytes && g == guard) return;
        release();
        ck(cudaMalloc(&base, n + 2 * g), "cudaMalloc");
        p = static_cast<char*>(base) + g;
        bytes = n;
        guard = g;
        if (g) {
            ck(cudaMemset(base, 0xA5, g), "guard");
            ck(cudaMemset(static_cast<char*>(p) + n, 0xA5, g), "guard");
            ck(cudaDeviceSynchronize(), "guard");
        }
        ++alloc_generation();
    }
    void release() {
        if (base) cudaFree(base);
        p = base = nullptr;
        bytes = guard = 0;
    }
    template <class T> T* as() const { return reinterpret_cast<T*>(p); }
};

struct LayerW {
    // matrices in the activation type (fp32 or bf16), biases fp32
    void *g1, *g2, *a1, *a2, *f1, *f2, *ak;
    float *gb1, *gb2, *ab1, *ab2, *fb1, *fb2, *aq;
    float* au; // heads x D: u_h = Wk_h^T q_h, the attention score vectors
    void* aus16; // BF16 mode, heads <= 8, D = 256: 16 x D, rows h = hi(u_h / sqrt(D/heads)), 8 + h = lo (pool_mma)
    void* aus; // BF16 mode, heads <= 16: 64 x D bf16 score matrix, rows h = hi(u_h / sqrt(D/heads)),
               // rows 16 + h = the bf16 remainder (lo), zero elsewhere: scores = N . aus^T (EP_SCORES)
};

struct Stat {
    int64_t launches = 0;
    double ms = 0.0, flops = 0.0, bytes = 0.0;
};

struct Probe;

} // namespace
} // namespace cider

using namespace cider;

struct cider_ctx {
    std::mutex mu;
    int device = 0;
    int sm_count = 148;
    cudaStream_t stream = nullptr;
    cider_model_desc md{};
    int Q = 0, D = 0, H = 0, N = 0, heads = 0;
    bool bf16 = false;
    size_t act_size = 4;
    std::unique_ptr<Gf> gf;
    std::unique_ptr<Tanner> tg;
    int L = 0, P = 0, E = 0;
    int max_check_deg = 0, min_check_deg = 1 << 30;
    // weights
    std::vector<DevBuf> wbufs;
    float* Etab = nullptr;                 // (Q+1) x D fp32
    void* Etab16 = nullptr;                // BF16 mode: the same table in bf16 (embed = one 16-byte load per store)
    void *W = nullptr, *Wt = nullptr, *Vt = nullptr;
    void *Wpad = nullptr, *Vtpad = nullptr; // BF16, Q < 128: W / V^T padded with zero symbols to 128 (demix_evid)
    std::vector<LayerW> lw;
    // Tanner tables
    int *e_slot = nullptr, *e_check = nullptr, *check_ptr = nullptr, *slot_ptr = nullptr, *slot_edge = nullptr;
    uint8_t *perm_in = nullptr, *perm_out = nullptr;
    // Q >= D path (gemm_grp.cuh): T_alpha = W^T Pi_alpha W table + group tables
    bool tpath = false;
    void* Ttab = nullptr;                          // bf16 [Q][D][D] as B tiles [alpha][n][k]
    int *gn_count = nullptr, *gn_arow = nullptr, *gn_alpha = nullptr, *gn_out = nullptr;  // per edge
    int *gm_count = nullptr, *gm_arow = nullptr, *gm_alpha = nullptr, *gm_out = nullptr;  // per slot
    int gm_max_seg = 0;
    std::vector<float> W_host; // out_proj as the device computes with it (bf16-rounded in BF16 mode)
    // workspace
    int chunk_req = 0;
    int cap_bins = 0, cap_K = 0;
    std::map<std::string, DevBuf> ws;
    size_t debug_guard = 0; // cider_set_debug_guard: guard bands around workspace buffers
    std::map<std::tuple<const void*, int64_t, int, int, int>, CUtensorMap> maps;
    // CUDA graphs of whole refinement chunks (no-remask / rank-remask passes: no host round trip),
    // keyed by shape, schedule, buffers and allocation generation; seen once eagerly, then captured
    struct GraphEntry {
        int seen = 0;
        cudaGraphExec_t exec = nullptr;
        int64_t launches = 0;
    };
    std::map<std::string, GraphEntry> graphs;
    // instrumentation
    int64_t launches = 0;
    bool profiling = false;
    std::map<std::string, Stat> stats;
    std::vector<std::tuple<std::string, cudaEvent_t, cudaEvent_t, double, double>> pending;
    std::vector<cudaEvent_t> ev_pool;
    cudaEvent_t events[64] = {};
    DevBuf flush_buf;
    // NCCL (dlopen'ed)
    void* nccl_lib = nullptr;
    void* nccl_comm = nullptr;
    // teacher-forcing probe of the running cider_refine_probe call (nullptr otherwise)
    cider::Probe* probe = nullptr;

    ~cider_ctx();
};

namespace cider {
namespace {

template <class F>
int guard(F&& f) {
    try {
        f();
        return CIDER_OK;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        g_err_tick = error_tick();
        return CIDER_EINVAL;
    } catch (const std::exception& e) {
        g_err = e.what();
        g_err_tick = error_tick();
        return CIDER_ERUNTIME;
    }
}

DevBuf& wbuf(cider_ctx& c, size_t bytes) {
    c.wbufs.emplace_back();
    c.wbufs.back().ensure(std::max<size_t>(bytes, 16));
    return c.wbufs.back();
}

float bf16_round(float v) { return __bfloat162float(__float2bfloat16_rn(v)); }

// Upload a host fp32 matrix, optionally transposed, in the activation type; `scale` (a power of two)
// multiplies it first (exact in bf16).
void* upload_mat(cider_ctx& c, const float* src, int rows, int cols, bool transpose, float scale = 1.0f) {
    const int R = transpose ? cols : rows, C = transpose ? rows : cols;
    std::vector<float> t(size_t(R) * C);
    for (int r = 0; r < rows; ++r)
        for (int q = 0; q < cols; ++q) {
            float v = src[size_t(r) * cols + q] * scale;
            if (transpose) t[size_t(q) * rows + r] = v; else t[size_t(r) * cols + q] = v;
        }
    DevBuf& b = wbuf(c, t.size() * c.act_size);
    if (c.bf16) {
        std::vector<bf16> h(t.size());
        for (size_t i = 0; i < t.size(); ++i) h[i] = __float2bfloat16_rn(t[i]);
        ck(cudaMemcpy(b.p, h.data(), h.size() * 2, cudaMemcpyHostToDevice), "upload");
    } else {
        ck(cudaMemcpy(b.p, t.data(), t.size() * 4, cudaMemcpyHostToDevice), "upload");
    }
    return b.p;
}
float* upload_vec(cider_ctx& c, const float* src, size_t n) {
    std::vector<float> t(src, src + n);
    if (c.bf16)
        for (float& v : t) v = bf16_round(v); // BF16 mode: the whole model is bf16-valued
    DevBuf& b = wbuf(c, n * 4);
    ck(cudaMemcpy(b.p, t.data(), n * 4, cudaMemcpyHostToDevice), "upload");
    return b.as<float>();
}
template <class T>
T* upload_raw(cider_ctx& c, const std::vector<T>& v) {
    DevBuf& b = wbuf(c, v.size() * sizeof(T));
    if (!v.empty()) ck(cudaMemcpy(b.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "upload");
    return b.as<T>();
}

// ---- programmatic dependent launch -----------------------------------------------------------
// The kernels of the refinement chain are launched with programmatic stream serialization: each
// calls griddep_wait() before reading anything earlier kernels produced (kernels/common.cuh), and
// the persistent ones (every CTA resident) call griddep_launch_dependents() right after, so the next
// kernel's launch and prologue (barrier init, TMEM allocation, descriptor prefetch) overlap this
// kernel's tail instead of following it. Captured into the refinement CUDA graphs as programmatic
// edges.
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    ck(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...), "cudaLaunchKernelEx");
}

// ---- launch bookkeeping --------------------------------------------------------------------
struct Launch {
    cider_ctx& c;
    std::string tag;
    double flops, bytes;
    cudaEvent_t a = nullptr, b = nullptr;
    Launch(cider_ctx& c_, const char* t, double f, double by) : c(c_), tag(t), flops(f), bytes(by) {
        ++c.launches;
        nvtxRangePushA(t); // one NVTX range per kernel class launch (ncu --nvtx --nvtx-include, nsys)
        if (c.profiling) {
            a = take();
            cudaEventRecord(a, c.stream);
        }
    }
    cudaEvent_t take() {
        if (c.ev_pool.empty()) {
            cudaEvent_t e;
            ck(cudaEventCreate(&e), "event");
            return e;
        }
        cudaEvent_t e = c.ev_pool.back();
        c.ev_pool.pop_back();
        return e;
    }
    ~Launch() {
        nvtxRangePop();
        if (c.profiling) {
            b = take();
            cudaEventRecord(b, c.stream);
            c.pending.emplace_back(tag, a, b, flops, bytes);
        }
    }
};

void resolve_stats(cider_ctx& c) {
    if (c.pending.empty()) return;
    ck(cudaStreamSynchronize(c.stream), "sync");
    for (auto& [tag, a, b, f, by] : c.pending) {
        float ms = 0.0f;
        cudaEventElapsedTime(&ms, a, b);
        Stat& s = c.stats[tag];
        s.launches++;
        s.ms += ms;
        s.flops += f;
        s.bytes += by;
        c.ev_pool.push_back(a);
        c.ev_pool.push_back(b);
    }
    c.pending.clear();
}

void check_launch(const char* what) { ck(cudaGetLastError(), what); }

inline unsigned blocks_for(int64_t n, int t = 256) { return unsigned((n + t - 1) / t); }

// ---- GEMM dispatch -------------------------------------------------------------------------
const CUtensorMap& map_for(cider_ctx& c, const void* p, int64_t rows, int cols, int ld, int box_rows) {
    auto key = std::make_tuple(p, rows, cols, ld, box_rows);
    auto it = c.maps.find(key);
    if (it != c.maps.end()) return it->second;
    return c.maps.emplace(key, make_map(p, rows, cols, ld, box_rows)).first->second;
}

template <int BN, int EPW = 4, bool BRES = false>
void launch_tc(cider_ctx& c, const CUtensorMap& a0, const CUtensorMap& a1, const CUtensorMap& b, const tc::Args& args) {
    using Lay = tc::SmemLayout<BN, EPW, BRES>;
    static PerDeviceOnce attr_set;
    attr_set.run(current_device(), [&] {
        ck(cudaFuncSetAttribute(tc::gemm_tc_kernel<BN, EPW, BRES>, cudaFuncAttributeMaxDynamicSharedMemorySize, Lay::TOTAL),
           "smem attr");
    });
    int grid = std::min(args.tiles, c.sm_count);
    launch_pdl(tc::gemm_tc_kernel<BN, EPW, BRES>, grid, 64 + 32 * EPW, Lay::TOTAL, c.stream, a0, a1, b, args);
}

// C[M x N] = [A0 (M x K0) | A1 (M x K1)] . B[N x (K0+K1)]^T, then the epilogue.
void gemm(cider_ctx& c, const char* tag, const void* A0, int K0, const void* A1, int K1, const void* B, int64_t M,
          int N, Epi ep) {
    const int K = K0 + K1;
    ep.M = int(M);
    ep.N = N;
    Launch lg(c, tag, 2.0 * double(M) * N * K, double(M) * K * c.act_size + double(N) * K * c.act_size);
    if (!c.bf16) {
        dim3 grid(unsigned((N + SG_BN - 1) / SG_BN), unsigned((M + SG_BM - 1) / SG_BM));
        gemm_simt_f32<<<grid, 256, 0, c.stream>>>(reinterpret_cast<const float*>(A0), K0 ? (A1 ? K0 : K) : K, K0 ? K0 : K,
                                                   reinterpret_cast<const float*>(A1), K1, reinterpret_cast<const float*>(B), K,
                                                   int(M), N, K, ep);
        check_launch(tag);
        return;
    }
    if (K0 % 64 || K1 % 64 || N % 64) throw InvalidInput("BF16 mode needs Q, D, H multiples of 64");
    const int BN = (N % 256 == 0) ? 256 : (N % 128 == 0) ? 128 : 64;
    if (ep.kind == EP_LOGITS && BN != N) throw InvalidInput("BF16 mode needs Q <= 256 for the fused logits epilogue");
    const CUtensorMap& a0 = map_for(c, A0, M, K0, A1 ? K0 : K, tc::BM);
    const CUtensorMap& a1 = A1 ? map_for(c, A1, M, K1, K1, tc::BM) : a0;
    const CUtensorMap& b = map_for(c, B, N, K, K, BN);
    tc::Args args;
    args.M = int(M);
    args.N = N;
    args.K = K;
    args.K0 = A1 ? K0 : K;
    args.tiles_n = N / BN;
    args.tiles = int((M + tc::BM - 1) / tc::BM) * args.tiles_n;
    args.ep = ep;
    const int epw = ep.kind == EP_DEMIX ? (BN == 64 ? 8 : 16) : 4; // the demix epilogue needs the > 4-warp staging
    if (ep.kind == EP_DEMIX && BN != 256 && BN != 64) throw InvalidInput("fused demix epilogue needs Q = 64 or Q % 256 == 0");
    // B-resident variants: one N tile, K <= 256 (W, W^T, V^T against 128-row A tiles)
    const bool bres = BN == 256 && N == 256 && K <= 256;
    // (the fused demix is epilogue-bound: it keeps 16 epilogue warps and a streamed B, measured faster
    // than 8 warps with B resident)
    if (bres && epw == 4) launch_tc<256, 4, true>(c, a0, a1, b, args);
    else if (BN == 256 && epw == 16) launch_tc<256, 16>(c, a0, a1, b, args);
    else if (BN == 256 && epw == 8) launch_tc<256, 8>(c, a0, a1, b, args);
    else if (BN == 64 && epw == 8) launch_tc<64, 8>(c, a0, a1, b, args);
    else if (BN == 256) launch_tc<256>(c, a0, a1, b, args);
    else if (BN == 128) launch_tc<128>(c, a0, a1, b, args);
    else launch_tc<64>(c, a0, a1, b, args);
    check_launch(tag);
}

Epi epi(int kind) {
    Epi e;
    std::memset(&e, 0, sizeof(e));
    e.kind = kind;
    return e;
}

void* wsbuf(cider_ctx& c, const char* name, size_t bytes);

// ---- fused two-layer maps (BF16 mode) -----------------------------------------------------------
template <int KIN, int D>
void launch_mlp(cider_ctx& c, const CUtensorMap& x0, const CUtensorMap& x1, const CUtensorMap& w1,
                const CUtensorMap& w2, const tc::MlpArgs& a) {
    using Lay = tc::MlpLayout<KIN, D>;
    static PerDeviceOnce attr_set;
    attr_set.run(current_device(), [&] {
        ck(cudaFuncSetAttribute(tc::mlp_tc_kernel<KIN, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, Lay::TOTAL),
           "smem attr");
    });
    const int grid = std::min(a.tiles, c.sm_count);
    tc::mlp_tc_kernel<KIN, D><<<grid, tc::MLP_THREADS, Lay::TOTAL, c.stream>>>(x0, x1, w1, w2, a);
}

template <int KIN, int D, int EPK, int KK = 0>
void launch_mlp2(cider_ctx& c, const CUtensorMap& x0, const CUtensorMap& x1, const CUtensorMap& w1,
                 const CUtensorMap& w2, const CUtensorMap& out, const tc::MlpArgs& a) {
    using Lay = tc::Mlp2LayoutFor<KIN, D, EPK>;
    static PerDeviceOnce attr_set;
    attr_set.run(current_device(), [&] {
        ck(cudaFuncSetAttribute(tc::mlp_tc2_kernel<KIN, D, EPK, KK>, cudaFuncAttributeMaxDynamicSharedMemorySize, Lay::TOTAL),
           "smem attr");
    });
    const int pairs = std::min(a.tiles, c.sm_count / 2);
    launch_pdl(tc::mlp_tc2_kernel<KIN, D, EPK, KK>, 2 * pairs, tc::mlp2_threads(EPK), Lay::TOTAL, c.stream, x0, x1, w1, w2, out, a);
}

// Per-chunk timelines of the fused MLPs: a diagnostic build (make EXTRA=-DCIDER_MLP_TRACE OUT=../_lib_trace,
// loaded with CIDER_LIB_DIR) run with CIDER_TRACE_MLP=1; the product build carries no stamp code.
bool mlp_trace_enabled() {
    static const bool want = std::getenv("CIDER_TRACE_MLP") != nullptr;
#ifdef CIDER_MLP_TRACE
    return want;
#else
    static bool told = false;
    if (want && !told) {
        std::fprintf(stderr, "cider: CIDER_TRACE_MLP needs the diagnostic build (make EXTRA=-DCIDER_MLP_TRACE)\n");
        told = true;
    }
    return false;
#endif
}

bool mlp_fusable(const cider_ctx& c, int Kin) {
    return c.bf16 && c.H % tc::MLP_HC == 0 && (c.D == 64 || c.D == 128 || c.D == 256) && (Kin == c.D || Kin == 2 * c.D);
}

void dump_mlp_trace(cider_ctx& c, const char* tag, int64_t M, int H, bool pair, long long* tbuf) {
    {
        long long h[1024];
        cudaMemcpyAsync(h, tbuf, sizeof(h), cudaMemcpyDeviceToHost, c.stream);
        cudaStreamSynchronize(c.stream);
        const long long t0 = h[2];
        std::fprintf(stderr, "[mlp trace %s M=%lld pair=%d] chunk: mma1_wait_free mma1_issued | mma2_wait_h mma2_got_h mma2_issued | epi_wait_a1 epi_got_a1 epi_done\n", tag, (long long)M, int(pair));
        for (int it = 0; it < (pair ? 4 : 1); ++it)
            for (int ch = 0; ch < H / tc::MLP_HC; ++ch) {
                const long long* r = h + it * 64 + ch * 8;
                std::fprintf(stderr, "  t%d c%d: %8lld %8lld | %8lld %8lld %8lld | %8lld %8lld %8lld\n", it, ch, r[6] - t0, r[7] - t0,
                             r[0] - t0, r[1] - t0, r[5] - t0, r[2] - t0, r[3] - t0, r[4] - t0);
            }
        for (int it = 0; it < (pair ? 4 : 0); ++it) {
            std::fprintf(stderr, "  t%d mma1 got_free:", it);
            for (int ch = 0; ch < H / tc::MLP_HC; ++ch) std::fprintf(stderr, " %lld", h[896 + it * 8 + ch] - t0);
            std::fprintf(stderr, "\n");
            std::fprintf(stderr, "\n");
        }
        for (int it = 0; it < (pair ? 4 : 0); ++it) {
            std::fprintf(stderr, "  t%d final epilogue: wait %lld got %lld done %lld |", it, h[512 + it * 4] - t0, h[512 + it * 4 + 1] - t0,
                         h[512 + it * 4 + 2] - t0);
            for (int k = 1; k < 10; ++k) std::fprintf(stderr, " %lld", h[256 + it * 16 + k] ? h[256 + it * 16 + k] - t0 : -1);
            std::fprintf(stderr, "\n");
        }
    }
}

// Y = ep(GELU([A0|A1] W1^T + b1) W2^T + b2); falls back to two GEMMs through the `hid` buffer.
void mlp(cider_ctx& c, const char* tag, const void* A0, int K0, const void* A1, int K1, const void* W1,
         const float* b1, const void* W2, int64_t M, Epi ep, void* hid) {
    const int Kin = K0 + K1, D = c.D, H = c.H;
    if (!mlp_fusable(c, Kin)) {
        std::string t1 = std::string(tag) + "_1", t2 = std::string(tag) + "_2";
        Epi e1 = epi(EP_GELU);
        e1.bias = b1; e1.out_t = hid; e1.ldo = H;
        gemm(c, t1.c_str(), A0, K0, A1, K1, W1, M, H, e1);
        gemm(c, t2.c_str(), hid, H, nullptr, 0, W2, M, D, ep);
        return;
    }
    ep.M = int(M);
    ep.N = D;
    // 2-SM kernel variants: aggregator (Kin = D, plain store), gate / fusion (Kin = 2D, z (e) epilogue)
    const bool pair = (D == 128 || D == 256) &&
                      ((Kin == D && ep.kind == EP_STORE) || (Kin == 2 * D && (ep.kind == EP_GATE || ep.kind == EP_RESID))) &&
                      // (D = 128 variants keep the hidden bias in shared memory: H must fit, else the 1-SM kernel)
                      (tc::mlp2_b1_smem_bytes(Kin, D, ep.kind) == 0 || H * 4 <= tc::mlp2_b1_smem_bytes(Kin, D, ep.kind));
    Launch lg(c, tag, 2.0 * double(M) * H * (Kin + D), double(M) * (Kin + D) * c.act_size);
    const CUtensorMap& x0 = map_for(c, A0, M, A1 ? K0 : Kin, A1 ? K0 : Kin, 128);
    const CUtensorMap& x1 = A1 ? map_for(c, A1, M, K1, K1, 128) : x0;
    CUtensorMap w1_3d;
    if (pair) w1_3d = make_map_w1_3d(W1, H, Kin, tc::MLP_HC / 2);
    const CUtensorMap& w1 = pair ? w1_3d : map_for(c, W1, H, Kin, Kin, tc::MLP_HC);
    const CUtensorMap& w2 = map_for(c, W2, D, H, H, pair ? D / 2 : (D > 128 ? 128 : D));
    tc::MlpArgs a;
    a.M = int(M);
    a.K0 = A1 ? K0 : Kin;
    a.H = H;
    a.tiles = int((M + (pair ? 255 : 127)) / (pair ? 256 : 128));
    a.b1 = b1;
    a.ep = ep;
    a.trace = nullptr;
    static const bool trace_on = mlp_trace_enabled();
    long long* tbuf = nullptr;
    if (trace_on) {
        tbuf = (long long*)wsbuf(c, "mlp_trace", 8 * 1024);
        cudaMemsetAsync(tbuf, 0, 8 * 1024, c.stream);
        a.trace = tbuf;
    }
    if (pair) {
        if (ep.out_f || !ep.out_t) throw InvalidInput("cider: the 2-SM MLP writes one bf16 output");
        // one TMA store box (SW128) per 128-row x 64-column output k-block staged in the tile's X
        const CUtensorMap om = make_map_box(ep.out_t, M, D, ep.ldo, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B);
        if (D == 256) {
            if (ep.kind == EP_GATE) launch_mlp2<512, 256, EP_GATE>(c, x0, x1, w1, w2, om, a);
            else if (ep.kind == EP_RESID) launch_mlp2<512, 256, EP_RESID>(c, x0, x1, w1, w2, om, a);
            else launch_mlp2<256, 256, EP_STORE>(c, x0, x1, w1, w2, om, a);
        } else {
            if (ep.kind == EP_GATE) launch_mlp2<256, 128, EP_GATE>(c, x0, x1, w1, w2, om, a);
            else if (ep.kind == EP_RESID) launch_mlp2<256, 128, EP_RESID>(c, x0, x1, w1, w2, om, a);
            else launch_mlp2<128, 128, EP_STORE>(c, x0, x1, w1, w2, om, a);
        }
    } else if (D == 256) { if (Kin == 512) launch_mlp<512, 256>(c, x0, x1, w1, w2, a); else launch_mlp<256, 256>(c, x0, x1, w1, w2, a); }
    else if (D == 128) { if (Kin == 256) launch_mlp<256, 128>(c, x0, x1, w1, w2, a); else launch_mlp<128, 128>(c, x0, x1, w1, w2, a); }
    else { if (Kin == 128) launch_mlp<128, 64>(c, x0, x1, w1, w2, a); else launch_mlp<64, 64>(c, x0, x1, w1, w2, a); }
    check_launch(tag);
    if (tbuf) dump_mlp_trace(c, tag, M, H, pair, tbuf);
}

// ---- workspace ------------------------------------------------------------------------------
struct WS {
    int* X;
    float *Zf, *lbar, *ef, *Ztf, *accf, *keys, *logits, *kappa, *k1;
    void *Zt, *Aq, *et, *hid, *Ztt, *U, *Ae, *Nn, *pooled, *mapped, *Mq, *accq, *acct;
    int *amax, *init_masked, *nlow;
    uint32_t* upd;
    float* S;  // staging for host evidence
    int* Xio;  // staging for host grids
    float* flog; // final-pass logits (internal layout), when requested
};

size_t round_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

void* wsbuf(cider_ctx& c, const char* name, size_t bytes) {
    DevBuf& b = c.ws[name];
    b.ensure(round_up(std::max<size_t>(bytes, 256), 256), c.debug_guard);
    return b.p;
}

bool pool_fast(const cider_ctx& c);

// Sizes (per bin) of the chunk workspace; rows padded to the 128-row GEMM tile.
WS workspace(cider_ctx& c, int nb, int K, bool want_flog) {
    const size_t Ms = round_up(size_t(nb) * c.L * K, 128), Me = round_up(size_t(nb) * c.E * K, 128);
    const size_t A = c.act_size, Q = c.Q, D = c.D, H = c.H;
    WS w{};
    w.X = (int*)wsbuf(c, "X", Ms * 4);
    // the fp32 residual stream exists only in FP32 mode; BF16 mode keeps it in bf16
    w.Zf = c.bf16 ? nullptr : (float*)wsbuf(c, "Zf", Ms * D * 4);
    w.lbar = (float*)wsbuf(c, "lbar", Ms * Q * 4);
    w.ef = c.bf16 ? nullptr : (float*)wsbuf(c, "ef", Ms * D * 4);
    w.Ztf = c.bf16 ? nullptr : (float*)wsbuf(c, "Ztf", Ms * D * 4);
    w.accf = (float*)wsbuf(c, "accf", Ms * D * 4);
    w.kappa = (float*)wsbuf(c, "kappa", Ms * 4);
    w.k1 = (float*)wsbuf(c, "k1", Ms * 4);
    w.amax = (int*)wsbuf(c, "amax", Ms * 4);
    w.Aq = wsbuf(c, "Aq", Ms * Q * A);
    w.hid = wsbuf(c, "hid", std::max(Ms, Me) * H * A);
    w.U = wsbuf(c, "U", Ms * Q * A);
    w.Ae = wsbuf(c, "Ae", Me * Q * A);
    w.Nn = wsbuf(c, "Nn", Me * D * A);
    w.pooled = wsbuf(c, "pooled", Me * D * A);
    w.mapped = wsbuf(c, "mapped", Me * D * A);
    w.Mq = wsbuf(c, "Mq", Me * Q * A);
    w.accq = wsbuf(c, "accq", Ms * Q * A);
    w.keys = (c.heads && !pool_fast(c)) ? (float*)wsbuf(c, "keys", Me * D * 4) : nullptr;
    w.logits = c.bf16 ? nullptr : (float*)wsbuf(c, "logits", Ms * Q * 4);
    if (c.bf16) {
        w.Zt = wsbuf(c, "Zt", Ms * D * A);
        w.et = wsbuf(c, "et", Ms * D * A);
        w.Ztt = wsbuf(c, "Ztt", Ms * D * A);
        w.acct = wsbuf(c, "acct", Ms * D * A);
    } else {
        w.Zt = w.Zf;
        w.et = w.ef;
        w.Ztt = w.Ztf;
        w.acct = w.accf;
    }
    w.init_masked = (int*)wsbuf(c, "init_masked", size_t(nb) * 4);
    w.nlow = (int*)wsbuf(c, "nlow", size_t(nb) * 4);
    w.upd = (uint32_t*)wsbuf(c, "upd", size_t(nb) * 4);
    w.S = (float*)wsbuf(c, "S", size_t(nb) * c.L * Q * 4);
    w.Xio = (int*)wsbuf(c, "Xio", size_t(nb) * c.L * K * 4);
    w.flog = want_flog ? (float*)wsbuf(c, "flog", Ms * Q * 4) : nullptr;
    return w;
}

// chunk size: explicit, or sized so the workspace stays within ~60% of free HBM
int chunk_bins(cider_ctx& c, int K) {
    if (c.chunk_req > 0) return c.chunk_req;
    const double A = double(c.act_size);
    const double Ms = double(c.L) * K, Me = double(c.E) * K;
    double per_bin = Ms * (c.D * 4.0 * 4 + c.Q * 4.0 * 2 + c.Q * A * 3 + c.D * A * 4 + 16) +
                     Me * (c.Q * A * 2 + c.D * A * 3 + (c.heads ? c.D * 4.0 : 0)) + std::max(Ms, Me) * c.H * A +
                     c.L * c.Q * 4.0;
    size_t fr = 0, tot = 0;
    ck(cudaMemGetInfo(&fr, &tot), "cudaMemGetInfo");
    double budget = 0.6 * double(fr);
    int nb = int(std::max(1.0, std::min(budget / per_bin, 65536.0)));
    return nb;
}


// ---- Tanner / demix kernel dispatch (warp-vectorised fast paths, generic fallbacks) ----------
template <typename T>
void run_demix(cider_ctx& c, const float* lbar, const float* S, int64_t slotrows, int K, T* out) {
    const int Q = c.Q;
    if (K <= 32) {
        demix_block_kernel<T><<<unsigned(slotrows), std::min(256, ((Q + 31) / 32) * 32), 0, c.stream>>>(lbar, S, K, Q, float(c.md.tau_demix), out);
    } else {
        demix_kernel<T><<<blocks_for(slotrows * Q), 256, 0, c.stream>>>(lbar, S, slotrows, K, Q, float(c.md.tau_demix), out);
    }
}
template <typename T>
void run_gather(cider_ctx& c, const T* U, int K, int64_t Me, T* Ae) {
    const int V = c.Q / 32;
    const unsigned g = blocks_for(Me * 32);
    if (c.Q % 32 == 0 && V == 8) gather_perm_warp_kernel<T, 8><<<g, 256, 0, c.stream>>>(U, c.e_slot, c.perm_in, c.L, c.E, K, c.Q, Me, Ae);
    else if (c.Q % 32 == 0 && V == 4) gather_perm_warp_kernel<T, 4><<<g, 256, 0, c.stream>>>(U, c.e_slot, c.perm_in, c.L, c.E, K, c.Q, Me, Ae);
    else if (c.Q % 32 == 0 && V == 2) gather_perm_warp_kernel<T, 2><<<g, 256, 0, c.stream>>>(U, c.e_slot, c.perm_in, c.L, c.E, K, c.Q, Me, Ae);
    else gather_perm_kernel<T><<<blocks_for(Me * c.Q), 256, 0, c.stream>>>(U, c.e_slot, c.perm_in, c.L, c.E, K, c.Q, Me, Ae);
}
template <typename T>
void run_scatter(cider_ctx& c, const T* Mq, int K, int64_t Ms, T* accq) {
    const int V = c.Q / 32;
    const unsigned g = blocks_for(Ms * 32);
    if (c.Q % 32 == 0 && V == 8) scatter_perm_warp_kernel<T, 8><<<g, 256, 0, c.stream>>>(Mq, c.slot_ptr, c.slot_edge, c.perm_out, c.L, c.E, K, c.Q, Ms, accq);
    else if (c.Q % 32 == 0 && V == 4) scatter_perm_warp_kernel<T, 4><<<g, 256, 0, c.stream>>>(Mq, c.slot_ptr, c.slot_edge, c.perm_out, c.L, c.E, K, c.Q, Ms, accq);
    else if (c.Q % 32 == 0 && V == 2) scatter_perm_warp_kernel<T, 2><<<g, 256, 0, c.stream>>>(Mq, c.slot_ptr, c.slot_edge, c.perm_out, c.L, c.E, K, c.Q, Ms, accq);
    else scatter_perm_kernel<T, T><<<blocks_for(Ms * c.Q), 256, 0, c.stream>>>(Mq, c.slot_ptr, c.slot_edge, c.perm_out, c.L, c.E, K, c.Q, Ms, accq);
}
bool pool_fast(const cider_ctx& c) {
    const int V = c.D / 32;
    if (c.D % 32 != 0 || !(V == 2 || V == 4 || V == 8)) return false; // (D < 32: V = 0 must not reach the % below)
    const bool heads_ok = c.heads == 0 || ((c.heads == 2 || c.heads == 4 || c.heads == 8 || c.heads == 16) &&
                                           (c.D / c.heads) % V == 0);
    return c.max_check_deg <= POOL_DMAX && heads_ok;
}
template <typename T, int V, int DM>
void run_pool_d(cider_ctx& c, const LayerW& lw, const T* Nn, int K, int64_t groups, T* pooled) {
    const unsigned g = blocks_for(groups * 32);
    const float* U = lw.au;
    switch (c.heads) {
        case 0: pool_warp_kernel<T, V, 0, DM><<<g, 256, 0, c.stream>>>(Nn, U, c.check_ptr, c.P, c.E, K, c.D, groups, pooled); break;
        case 2: pool_warp_kernel<T, V, 2, DM><<<g, 256, size_t(2) * c.D * 4, c.stream>>>(Nn, U, c.check_ptr, c.P, c.E, K, c.D, groups, pooled); break;
        case 4: pool_warp_kernel<T, V, 4, DM><<<g, 256, size_t(4) * c.D * 4, c.stream>>>(Nn, U, c.check_ptr, c.P, c.E, K, c.D, groups, pooled); break;
        case 8: pool_warp_kernel<T, V, 8, DM><<<g, 256, size_t(8) * c.D * 4, c.stream>>>(Nn, U, c.check_ptr, c.P, c.E, K, c.D, groups, pooled); break;
        default: pool_warp_kernel<T, V, 16, DM><<<g, 256, size_t(16) * c.D * 4, c.stream>>>(Nn, U, c.check_ptr, c.P, c.E, K, c.D, groups, pooled); break;
    }
}
template <typename T, int V, int DEG>
void run_pool_fixed(cider_ctx& c, const LayerW& lw, const T* Nn, int K, int64_t groups, T* pooled) {
    const unsigned g = blocks_for(groups * 32);
    const float* U = lw.au;
    switch (c.heads) {
        case 0: pool_warp_fixed_kernel<T, V, 0, DEG><<<g, 256, 0, c.stream>>>(Nn, U, c.check_ptr, c.P, c.E, K, c.D, groups, pooled); break;
        case 2: pool_warp_fixed_kernel<T, V, 2, DEG><<<g, 256, size_t(2) * c.D * 4, c.stream>>>(Nn, U, c.check_ptr, c.P, c.E, K, c.D, groups, pooled); break;
        case 4: pool_warp_fixed_kernel<T, V, 4, DEG><<<g, 256, size_t(4) * c.D * 4, c.stream>>>(Nn, U, c.check_ptr, c.P, c.E, K, c.D, groups, pooled); break;
        case 8: pool_warp_fixed_kernel<T, V, 8, DEG><<<g, 256, size_t(8) * c.D * 4, c.stream>>>(Nn, U, c.check_ptr, c.P, c.E, K, c.D, groups, pooled); break;
        default: pool_warp_fixed_kernel<T, V, 16, DEG><<<g, 256, size_t(16) * c.D * 4, c.stream>>>(Nn, U, c.check_ptr, c.P, c.E, K, c.D, groups, pooled); break;
    }
}
template <typename T, int V>
void run_pool_v(cider_ctx& c, const LayerW& lw, const T* Nn, int K, int64_t groups, T* pooled) {
    // check-regular codes of degree 6 (all BASELINE codes): the unrolled fixed-degree kernel
    if (c.bf16 && c.max_check_deg == 6 && c.min_check_deg == 6 && V == 8) run_pool_fixed<T, V, 6>(c, lw, Nn, K, groups, pooled);
    else if (c.max_check_deg <= 6) run_pool_d<T, V, 6>(c, lw, Nn, K, groups, pooled);
    else run_pool_d<T, V, 8>(c, lw, Nn, K, groups, pooled);
}
template <typename T>
void run_pool(cider_ctx& c, const LayerW& lw, const T* Nn, int nb, int K, T* pooled) {
    const int V = c.D / 32;
    const int64_t groups = int64_t(nb) * c.P * K;
    if (V == 8) run_pool_v<T, 8>(c, lw, Nn, K, groups, pooled);
    else if (V == 4) run_pool_v<T, 4>(c, lw, Nn, K, groups, pooled);
    else run_pool_v<T, 2>(c, lw, Nn, K, groups, pooled);
}

// BF16, check-regular degree 6, D = 256, heads in {1, 2, 4, 8}, 6K <= 48 rows per (bin, check) block (K = 4 or 8)
bool pool_mma_ok(const cider_ctx& c, const LayerW& lw, int K) {
    return c.bf16 && lw.aus16 && (c.D == 256 || c.D == 128) && c.max_check_deg == 6 && c.min_check_deg == 6 && 8 % c.heads == 0 &&
           (K == 8 || (K == 4 && c.P % 2 == 0));
}
const CUtensorMap& map_for(cider_ctx& c, const void* p, int64_t rows, int cols, int ld, int box_rows);
template <int K, int D>
void launch_pool_mma(cider_ctx& c, const LayerW& lw, const CUtensorMap& tm, int64_t blocks, void* pooled) {
    static PerDeviceOnce attr;
    attr.run(current_device(), [&] {
        ck(cudaFuncSetAttribute(pool_mma_kernel<K, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, PoolMmaLayout::TOTAL), "smem attr");
    });
    const unsigned grid = unsigned(std::min<int64_t>(blocks, int64_t(c.sm_count) * 2));
    launch_pdl(pool_mma_kernel<K, D>, grid, PM_THREADS, PoolMmaLayout::TOTAL, c.stream, tm, (const bf16*)lw.aus16, c.check_ptr, c.P, c.E,
                                                                             c.heads, blocks, (bf16*)pooled);
}
void run_pool_mma(cider_ctx& c, const LayerW& lw, const void* Nn, int64_t Me, int nb, int K, void* pooled) {
    const CUtensorMap& tm = map_for(c, Nn, Me, c.D, c.D, 48); // 48-row blocks: one check at K = 8, two at K = 4
    const int64_t blocks = int64_t(nb) * c.P / (8 / K);
    if (c.D == 256) {
        if (K == 8) launch_pool_mma<8, 256>(c, lw, tm, blocks, pooled);
        else launch_pool_mma<4, 256>(c, lw, tm, blocks, pooled);
    } else {
        if (K == 8) launch_pool_mma<8, 128>(c, lw, tm, blocks, pooled);
        else launch_pool_mma<4, 128>(c, lw, tm, blocks, pooled);
    }
}

// BF16, check-regular degree 6, D = 256, 1..16 heads dividing 32 lanes: scores from EP_SCORES
bool pool_scored(const cider_ctx& c, const LayerW& lw) {
    return c.bf16 && lw.aus && c.D == 256 && c.max_check_deg == 6 && c.min_check_deg == 6 && 32 % c.heads == 0;
}
void run_pool_scored(cider_ctx& c, const bf16* Nn, const float* sc, int nb, int K, bf16* pooled) {
    const int64_t groups = int64_t(nb) * c.P * K;
    const unsigned g = blocks_for(groups * 32);
    switch (c.heads) {
        case 1: pool_warp_scored_kernel<bf16, 8, 1, 6><<<g, 256, 0, c.stream>>>(Nn, sc, c.check_ptr, c.P, c.E, K, c.D, groups, pooled); break;
        case 2: pool_warp_scored_kernel<bf16, 8, 2, 6><<<g, 256, 0, c.stream>>>(Nn, sc, c.check_ptr, c.P, c.E, K, c.D, groups, pooled); break;
        case 4: pool_warp_scored_kernel<bf16, 8, 4, 6><<<g, 256, 0, c.stream>>>(Nn, sc, c.check_ptr, c.P, c.E, K, c.D, groups, pooled); break;
        case 8: pool_warp_scored_kernel<bf16, 8, 8, 6><<<g, 256, 0, c.stream>>>(Nn, sc, c.check_ptr, c.P, c.E, K, c.D, groups, pooled); break;
        default: pool_warp_scored_kernel<bf16, 8, 16, 6><<<g, 256, 0, c.stream>>>(Nn, sc, c.check_ptr, c.P, c.E, K, c.D, groups, pooled); break;
    }
}

// ---- grouped GEMMs of the Q >= D path ----------------------------------------------------------
void grp_gemm(cider_ctx& c, const char* tag, const void* A, int a_rows_per_bin, int nb, int K, int groups,
              const int* cnt, const int* arow, const int* alpha, int max_seg, const int* out_row, int out_rows_per_bin,
              void* out_t, float* out_f, int mean_seg) {
    const int D = c.D;
    const int bb = std::max(1, 128 / K);
    if (K > 128) throw InvalidInput("cider: K > 128 unsupported on the grouped path");
    tc::GrpArgs a;
    a.groups = groups;
    a.mtiles = (nb + bb - 1) / bb;
    a.bins = nb;
    a.K = K;
    a.bb = bb;
    a.kb_per_seg = D / 64;
    a.max_seg = max_seg;
    a.seg_count = cnt;
    a.seg_arow = arow;
    a.seg_alpha = alpha;
    a.out_rows_per_bin = out_rows_per_bin;
    a.out_row = out_row;
    a.D = D;
    a.out_t = reinterpret_cast<bf16*>(out_t);
    a.out_f = out_f;
    const double rows = double(nb) * K * groups;
    // compulsory bytes: every A row once (normalise: the site rows its edges share) + the output rows
    Launch lg(c, tag, 2.0 * rows * D * D * mean_seg, (double(nb) * K * (a_rows_per_bin + out_rows_per_bin)) * D * 2.0);
    CUtensorMap ta = make_map_rows3d(A, nb, a_rows_per_bin * K, D, K, bb);
    CUtensorMap tt = make_map_ttab(c.Ttab, D, c.Q);
    const int tiles = a.groups * a.mtiles;
    using Lay = tc::SmemLayout<256, 0>;
    if (max_seg == 1 && c.sm_count >= 2 && D == 256) {
        // single-segment groups (normalise): CTA pairs with their T halves resident, laps over the pairs
        // (c5 58.6 -> 55.7 ms, c4 45 -> 41 ms per step; at D = 128 the streamed kernel is as fast)
        static PerDeviceOnce attr_r2;
        attr_r2.run(current_device(), [&] {
            ck(cudaFuncSetAttribute(tc::gemm_grp2_res_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    tc::grp2_res_smem<256>()), "smem attr");
            ck(cudaFuncSetAttribute(tc::gemm_grp2_res_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    tc::grp2_res_smem<128>()), "smem attr");
        });
        const int mpairs = (a.mtiles + 1) / 2;
        const int grid = 2 * std::min(groups * mpairs, c.sm_count / 2);
        const CUtensorMap tt2 = make_map_ttab(c.Ttab, D, c.Q, D / 2); // N-half boxes
        if (!out_t || out_f) throw InvalidInput("cider: the paired T-resident grouped GEMM writes one bf16 output");
        const CUtensorMap to = make_map_rows3d(out_t, nb, out_rows_per_bin * K, D, K, bb);
        if (D == 256) launch_pdl(tc::gemm_grp2_res_kernel<256>, grid, tc::GRP_THREADS, tc::grp2_res_smem<256>(), c.stream, ta, tt2, to, a);
        else launch_pdl(tc::gemm_grp2_res_kernel<128>, grid, tc::GRP_THREADS, tc::grp2_res_smem<128>(), c.stream, ta, tt2, to, a);
        check_launch(tag);
        return;
    }
    if ((a.mtiles >= 2 && c.sm_count >= 2 && D == 256) || D == 128) {
        // CTA pairs, one cta_group::2 MMA over two m-tiles: each SM pulls half of every T k-block
        // (D = 128 always: the other grouped kernels are D = 256 only)
        static PerDeviceOnce attr2;
        attr2.run(current_device(), [&] {
            ck(cudaFuncSetAttribute(tc::gemm_grp2_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::GRP2_SMEM), "smem attr");
            ck(cudaFuncSetAttribute(tc::gemm_grp2_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::GRP2_SMEM), "smem attr");
        });
        const int supers = a.groups * ((a.mtiles + 1) / 2);
        const int grid = 2 * std::min(supers, c.sm_count / 2);
        const CUtensorMap tt2 = make_map_ttab(c.Ttab, D, c.Q, D / 2); // N-half boxes
        if (!out_t) throw InvalidInput("cider: the paired grouped GEMM writes a bf16 output");
        const CUtensorMap to = make_map_rows3d(out_t, nb, out_rows_per_bin * K, D, K, bb); // TMA store boxes
        if (D == 256) launch_pdl(tc::gemm_grp2_kernel<256>, grid, tc::GRP_THREADS, tc::GRP2_SMEM, c.stream, ta, tt2, to, a);
        else launch_pdl(tc::gemm_grp2_kernel<128>, grid, tc::GRP_THREADS, tc::GRP2_SMEM, c.stream, ta, tt2, to, a);
        check_launch(tag);
        return;
    }
    // a single m-tile (small batches): one CTA per (group, m-tile), T streamed
    static PerDeviceOnce attr_set;
    attr_set.run(current_device(), [&] {
        ck(cudaFuncSetAttribute(tc::gemm_grp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, Lay::TOTAL), "smem attr");
    });
    launch_pdl(tc::gemm_grp_kernel, std::min(tiles, c.sm_count), tc::GRP_THREADS, Lay::TOTAL, c.stream, ta, tt, a);
    check_launch(tag);
}

// ---- Module A evidence path in one kernel: e = (softmax_k(Z W^T / tau) (x) S) V ------------------
// (intermediate_logits + demix_responsibilities + evidence_embed, denoiser.cpp:86-139): the 2-SM
// fused two-layer kernel with hidden = the Q symbol columns and the demix as its hidden activation.
bool demix_evid_ok(const cider_ctx& c, int K) {
    return c.bf16 && (c.D == 256 || c.D == 128) && (c.Q == 256 || c.Q == 128 || c.Q == 64) && (K == 4 || K == 8);
}
void demix_evid(cider_ctx& c, const void* Zt, const float* S, int64_t Ms, int K, bf16* e_out) {
    const int D = c.D, Q = c.Q;
    const int Qp = Q < tc::MLP_HC ? tc::MLP_HC : Q; // hidden width: Q < 128 padded to one chunk (zero W / V rows)
    Epi ep = epi(EP_DEMIX);
    ep.M = int(Ms); ep.N = D; ep.out_t = e_out; ep.ldo = D; ep.S = S; ep.L = c.L; ep.K = K;
    ep.ldz = Q; // S row stride = the valid symbol columns
    ep.beta = float(c.md.evidence_scale);
    ep.inv_tau = 1.0f / float(c.md.tau_demix); // as demix_block_kernel computes it
    Launch lg(c, "demix_evid", 2.0 * double(Ms) * Q * (D + D), double(Ms) * (2 * D * c.act_size) + double(Ms / K) * Q * 4);
    const CUtensorMap x0 = make_map_w1_3d(Zt, Ms, D, 128, D / 64); // the whole 128-row tile in one box
    const void* W = Qp == Q ? c.W : c.Wpad;
    const void* Vt = Qp == Q ? c.Vt : c.Vtpad;
    const CUtensorMap w1 = make_map_w1_3d(W, Qp, D, tc::MLP_HC / 2);
    const CUtensorMap& w2 = map_for(c, Vt, D, Qp, Qp, D / 2);
    tc::MlpArgs a;
    a.M = int(Ms);
    a.K0 = D;
    a.H = Qp;
    a.tiles = int((Ms + 255) / 256);
    a.b1 = nullptr;
    a.ep = ep;
    a.trace = nullptr;
    static const bool trace_on = mlp_trace_enabled();
    if (trace_on) {
        a.trace = (long long*)wsbuf(c, "mlp_trace", 8 * 1024);
        cudaMemsetAsync(a.trace, 0, 8 * 1024, c.stream);
    }
    const CUtensorMap om = make_map_box(e_out, Ms, D, D, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B); // e k-blocks staged in X
    if (D == 256) {
        if (a.ep.K == 8) launch_mlp2<256, 256, EP_DEMIX, 8>(c, x0, x0, w1, w2, om, a);
        else launch_mlp2<256, 256, EP_DEMIX, 4>(c, x0, x0, w1, w2, om, a);
    } else {
        if (a.ep.K == 8) launch_mlp2<128, 128, EP_DEMIX, 8>(c, x0, x0, w1, w2, om, a);
        else launch_mlp2<128, 128, EP_DEMIX, 4>(c, x0, x0, w1, w2, om, a);
    }
    check_launch("demix_evid");
    if (a.trace) dump_mlp_trace(c, "demix_evid", Ms, Qp, true, a.trace);
}

// ---- one denoiser forward over nb bins (denoiser.cpp:253-259) -------------------------------
struct FwdOpts {
    float tau = 1.0f;
    float* logits_out = nullptr;  // internal-layout fp32 logits [Ms x Q] (nullable)
    float* incoming = nullptr;    // internal-layout [layers][Ms x D] (nullable)
};

struct NvtxRange { // scoped NVTX range (no-op without a tool)
    explicit NvtxRange(const char* n) { nvtxRangePushA(n); }
    ~NvtxRange() { nvtxRangePop(); }
};

void forward(cider_ctx& c, WS& w, int nb, int K, const int* X, const float* S, const FwdOpts& o) {
    NvtxRange nv("cider.forward");
    const int L = c.L, E = c.E, Q = c.Q, D = c.D, H = c.H;
    const int64_t Ms = int64_t(nb) * L * K, Me = int64_t(nb) * E * K;
    {
        Launch lg(c, "embed", 0, double(Ms) * D * (4 + c.act_size));
        if (c.bf16 && D % 8 == 0)
            launch_pdl(embed_bf16x8_kernel, blocks_for(Ms * (D / 8)), 256, 0, c.stream, X, (const bf16*)c.Etab16, Q, D, Ms, (bf16*)w.Zt);
        else if (c.bf16)
            embed_kernel<bf16><<<blocks_for(Ms * D), 256, 0, c.stream>>>(X, c.Etab, Q, D, Ms, nullptr, (bf16*)w.Zt);
        else
            embed_kernel<float><<<blocks_for(Ms * D), 256, 0, c.stream>>>(X, c.Etab, Q, D, Ms, w.Zf, nullptr);
        check_launch("embed");
    }
    for (int li = 0; li < c.N; ++li) {
        const LayerW& lw = c.lw[li];
        // Module A (denoiser.cpp:141-160)
        Epi e;
        if (demix_evid_ok(c, K)) {
            // Lambda-bar, demix and the evidence embedding in one 2-SM kernel (e is its only output)
            demix_evid(c, w.Zt, S, Ms, K, (bf16*)w.et);
        } else {
        if (c.bf16 && 32 % K == 0 && K >= 4 && (Q % 256 == 0 || Q == 64)) {
            // intermediate logits and demixing in one kernel: Lambda-bar never leaves the chip
            e = epi(EP_DEMIX);
            e.out_t = w.Aq; e.ldo = Q; e.S = S; e.L = L; e.K = K; e.beta = float(c.md.evidence_scale);
            e.inv_tau = 1.0f / float(c.md.tau_demix); // as demix_block_kernel computes it
            gemm(c, "gemm_demix", w.Zt, D, nullptr, 0, c.W, Ms, Q, e);
        } else {
        e = epi(EP_LBAR);
        e.out_f = w.lbar; e.ldo = Q; e.S = S; e.L = L; e.K = K; e.beta = float(c.md.evidence_scale);
        gemm(c, "gemm_lbar", w.Zt, D, nullptr, 0, c.W, Ms, Q, e);
        {
            Launch lg(c, "demix", 0, double(Ms) * Q * (4 + c.act_size) + double(nb) * L * Q * 4);
            if (c.bf16) run_demix<bf16>(c, w.lbar, S, int64_t(nb) * L, K, (bf16*)w.Aq);
            else run_demix<float>(c, w.lbar, S, int64_t(nb) * L, K, (float*)w.Aq);
            check_launch("demix");
        }
        }
        e = epi(EP_STORE);
        e.out_f = w.ef; e.out_t = c.bf16 ? w.et : nullptr; e.ldo = D; // (ef is null in BF16 mode)
        gemm(c, "gemm_evid", w.Aq, Q, nullptr, 0, c.Vt, Ms, D, e);
        }
        e = epi(EP_GATE);
        e.bias = lw.gb2; e.z = w.Zf; e.e = w.ef; e.zb = (const bf16*)w.Zt; e.eb = (const bf16*)w.et; e.ldz = D;
        e.out_f = w.Ztf; e.out_t = c.bf16 ? w.Ztt : nullptr; e.ldo = D;
        mlp(c, "mlp_gate", w.Zt, D, w.et, D, lw.g1, lw.gb1, lw.g2, Ms, e, w.hid);
        // Module B (denoiser.cpp:181-228)
        if (Me == 0) {
            // a code without edges (test_denoiser.cpp:249-267): no check sends anything, the fusion sees zero
            // messages — none of the edge-row kernels has a grid to launch
            ck(cudaMemsetAsync(w.acct, 0, size_t(Ms) * D * c.act_size, c.stream), "acc = 0");
            if (w.accf && w.accf != w.acct) ck(cudaMemsetAsync(w.accf, 0, size_t(Ms) * D * 4, c.stream), "acc = 0");
        } else {
        if (c.tpath) {
            // N[(b,e,k)] = z~[(b,slot_e,k)] . T_{alpha_e}
            grp_gemm(c, "grp_normalise", w.Ztt, L, nb, K, E, c.gn_count, c.gn_arow, c.gn_alpha, 1, c.gn_out, E, w.Nn,
                     nullptr, 1);
        } else {
            e = epi(EP_STORE);
            e.out_t = w.U; e.ldo = Q;
            gemm(c, "gemm_symproj", w.Ztt, D, nullptr, 0, c.W, Ms, Q, e);
            {
                Launch lg(c, "gather_perm", 0, double(Me) * Q * 2 * c.act_size);
                if (c.bf16) run_gather<bf16>(c, (const bf16*)w.U, K, Me, (bf16*)w.Ae);
                else run_gather<float>(c, (const float*)w.U, K, Me, (float*)w.Ae);
                check_launch("gather_perm");
            }
            e = epi(EP_STORE);
            e.out_t = w.Nn; e.ldo = D;
            gemm(c, "gemm_backproj", w.Ae, Q, nullptr, 0, c.Wt, Me, D, e);
        }
        if (pool_mma_ok(c, lw, K)) {
            // one pass: TMA block loads, mma.sync head scores, leave-one-out softmax pool
            Launch lg(c, "pool_attn", 2.0 * double(Me) * D * (32 + c.max_check_deg), double(Me) * D * 2 * c.act_size);
            run_pool_mma(c, lw, w.Nn, Me, nb, K, w.pooled);
            check_launch("pool");
        } else if (pool_scored(c, lw)) {
            // head scores on the tensor cores, then a streaming leave-one-out softmax pool
            float* sc = (float*)wsbuf(c, "scores", size_t(round_up(size_t(Me), 128)) * c.heads * 4);
            e = epi(EP_SCORES);
            e.out_f = sc; e.ldo = c.heads; e.K = c.heads;
            gemm(c, "gemm_scores", w.Nn, D, nullptr, 0, lw.aus, Me, 64, e);
            Launch lg(c, "pool_attn", 2.0 * double(Me) * D * c.max_check_deg, double(Me) * D * 2 * c.act_size);
            run_pool_scored(c, (const bf16*)w.Nn, sc, nb, K, (bf16*)w.pooled);
            check_launch("pool");
        } else if (pool_fast(c)) {
            Launch lg(c, c.heads ? "pool_attn" : "pool_sum", 2.0 * double(Me) * D * (c.heads + c.max_check_deg),
                      double(Me) * D * 2 * c.act_size);
            if (c.bf16) run_pool<bf16>(c, lw, (const bf16*)w.Nn, nb, K, (bf16*)w.pooled);
            else run_pool<float>(c, lw, (const float*)w.Nn, nb, K, (float*)w.pooled);
            check_launch("pool");
        } else if (c.heads) {
            e = epi(EP_STORE);
            e.out_f = w.keys; e.ldo = D;
            gemm(c, "gemm_attn_key", w.Nn, D, nullptr, 0, lw.ak, Me, D, e);
            Launch lg(c, "pool_attn_generic", 0, double(Me) * D * (2 * c.act_size + 4));
            const unsigned groups = unsigned(int64_t(nb) * c.P * K);
            if (c.bf16)
                pool_attn_kernel<bf16, bf16><<<groups, 128, 0, c.stream>>>((bf16*)w.Nn, w.keys, lw.aq, c.check_ptr, c.P, E, K, D, c.heads, (bf16*)w.pooled);
            else
                pool_attn_kernel<float, float><<<groups, 128, 0, c.stream>>>((float*)w.Nn, w.keys, lw.aq, c.check_ptr, c.P, E, K, D, c.heads, (float*)w.pooled);
            check_launch("pool_attn");
        } else {
            Launch lg(c, "pool_sum_generic", 0, double(Me) * D * 2 * c.act_size);
            if (c.bf16)
                pool_sum_kernel<bf16, bf16><<<blocks_for(Me * D), 256, 0, c.stream>>>((bf16*)w.Nn, c.e_check, c.check_ptr, E, K, D, Me, (bf16*)w.pooled);
            else
                pool_sum_kernel<float, float><<<blocks_for(Me * D), 256, 0, c.stream>>>((float*)w.Nn, c.e_check, c.check_ptr, E, K, D, Me, (float*)w.pooled);
            check_launch("pool_sum");
        }
        e = epi(EP_STORE);
        e.bias = lw.ab2; e.out_t = w.mapped; e.ldo = D;
        mlp(c, "mlp_agg", w.pooled, D, nullptr, 0, lw.a1, lw.ab1, lw.a2, Me, e, w.hid);
        if (c.tpath) {
            // acc[(b,s,k)] = sum over slot s's edges (ascending check) of mapped[(b,e,k)] . T_{alpha_e^-1}
            grp_gemm(c, "grp_message", w.mapped, E, nb, K, L, c.gm_count, c.gm_arow, c.gm_alpha, c.gm_max_seg, c.gm_out, L,
                     w.acct, o.incoming ? w.accf : nullptr, std::max(1, E / std::max(1, L)));
        } else {
            e = epi(EP_STORE);
            e.out_t = w.Mq; e.ldo = Q;
            gemm(c, "gemm_msgproj", w.mapped, D, nullptr, 0, c.W, Me, Q, e);
            {
                Launch lg(c, "scatter_perm", 0, double(Ms) * Q * c.act_size + double(Me) * Q * c.act_size);
                if (c.bf16) run_scatter<bf16>(c, (const bf16*)w.Mq, K, Ms, (bf16*)w.accq);
                else run_scatter<float>(c, (const float*)w.Mq, K, Ms, (float*)w.accq);
                check_launch("scatter_perm");
            }
            e = epi(EP_STORE);
            e.out_f = (c.bf16 && !o.incoming) ? nullptr : w.accf; e.out_t = c.bf16 ? w.acct : nullptr; e.ldo = D;
            gemm(c, "gemm_msgback", w.accq, Q, nullptr, 0, c.Wt, Ms, D, e);
        }
        } // Me > 0
        if (o.incoming)
            ck(cudaMemcpyAsync(o.incoming + size_t(li) * Ms * D, w.accf, size_t(Ms) * D * 4, cudaMemcpyDeviceToDevice, c.stream), "incoming");
        e = epi(EP_RESID);
        e.bias = lw.fb2; e.z = w.Ztf; e.zb = (const bf16*)w.Ztt; e.ldz = D; e.out_f = w.Zf; e.out_t = c.bf16 ? w.Zt : nullptr; e.ldo = D;
        mlp(c, "mlp_fuse", w.Ztt, D, w.acct, D, lw.f1, lw.fb1, lw.f2, Ms, e, w.hid);
    }
    // final logits + site statistics (denoiser.cpp:230-245, refine.cpp:61-78)
    if (c.bf16) {
        Epi e = epi(EP_LOGITS);
        e.inv_tau = 1.0f / o.tau; e.kappa = w.kappa; e.amax = w.amax; e.out_f = o.logits_out; e.ldo = Q;
        gemm(c, "gemm_logits", w.Zt, D, nullptr, 0, c.W, Ms, Q, e);
    } else {
        float* lg_buf = o.logits_out ? o.logits_out : w.logits;
        Epi e = epi(EP_STORE);
        e.out_f = lg_buf; e.ldo = Q;
        gemm(c, "gemm_logits", w.Zt, D, nullptr, 0, c.W, Ms, Q, e);
        Launch lg(c, "row_stats", 0, double(Ms) * Q * 4);
        row_stats_kernel<<<blocks_for(Ms * 32), 256, 0, c.stream>>>(lg_buf, Ms, Q, o.tau, w.kappa, w.amax);
        check_launch("row_stats");
    }
}

// ---- one pass of run_masked_loop (refine.cpp:134-195) over nb bins ------------------------------
// Device buffers of one traced pass (RefineTrace, refine.hpp:48-54): per-step reveal counts
// (nb x steps) and the sites revealed at t = 1 (nb x L*K, internal layout).
struct PassTrace {
    int* counts = nullptr;
    uint8_t* sites = nullptr;
};

// Teacher-forcing probe (cider_refine_probe): every forward's input grid and output
// logits of a few bins, plus each pass's output grid, copied to host buffers in execution order.
struct Probe {
    std::vector<int> bins; // chunk-local bin indices
    int max_rec = 0, n_rec = 0, pass = 0;
    int32_t *X = nullptr, *meta = nullptr;
    float* lg = nullptr;     // host, nullable
    float* dev_lg = nullptr; // device logits of the forward being recorded (internal layout)
};

void probe_record(cider_ctx& c, Probe& p, int K, const int* X, int t, int steps, int kind) {
    if (p.n_rec >= p.max_rec) throw InvalidInput("cider_refine_probe: more records than max_records");
    const int L = c.L, Q = c.Q, n = L * K, r = p.n_rec;
    ck(cudaStreamSynchronize(c.stream), "probe sync");
    std::vector<int> xi(n);
    std::vector<float> li(p.lg && kind < 2 ? size_t(n) * Q : 0);
    for (size_t i = 0; i < p.bins.size(); ++i) {
        const int b = p.bins[i];
        ck(cudaMemcpy(xi.data(), X + size_t(b) * n, size_t(n) * 4, cudaMemcpyDeviceToHost), "probe X");
        int32_t* xo = p.X + (i * p.max_rec + r) * size_t(n);
        for (int l = 0; l < L; ++l)
            for (int k = 0; k < K; ++k) xo[size_t(k) * L + l] = xi[size_t(l) * K + k];
        if (li.empty()) continue;
        ck(cudaMemcpy(li.data(), p.dev_lg + size_t(b) * n * Q, size_t(n) * Q * 4, cudaMemcpyDeviceToHost), "probe logits");
        float* lo = p.lg + (i * p.max_rec + r) * size_t(n) * Q;
        for (int l = 0; l < L; ++l)
            for (int k = 0; k < K; ++k)
                std::copy(li.begin() + (size_t(l) * K + k) * Q, li.begin() + (size_t(l) * K + k + 1) * Q,
                          lo + (size_t(k) * L + l) * Q);
    }
    int32_t* m = p.meta + size_t(r) * 4;
    m[0] = p.pass; m[1] = t; m[2] = steps; m[3] = kind;
    ++p.n_rec;
}

// X holds the start grid (internal layout); init_masked / upd describe it per bin.
void masked_pass(cider_ctx& c, WS& w, int nb, int K, const float* S, int* X, int steps, const cider_schedule& sc,
                 const PassTrace* pt) {
    NvtxRange nv("cider.masked_pass");
    const int n = c.L * K;
    Probe* probe = c.probe;
    // reveal keys: dynamic shared memory up to REVEAL_SMEM_SITES, else a per-bin global slice
    const int cap = reveal_key_cap(n);
    const size_t smem = cap <= REVEAL_SMEM_SITES ? size_t(cap) * 8 : 0;
    unsigned long long* gkeys = cap > REVEAL_SMEM_SITES ? (unsigned long long*)wsbuf(c, "reveal_keys", size_t(nb) * cap * 8) : nullptr;
    static PerDeviceOnce attr;
    attr.run(current_device(), [&] {
        ck(cudaFuncSetAttribute(reveal_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, REVEAL_SMEM_SITES * 8), "reveal attr");
    });
    for (int t = 1; t <= steps; ++t) {
        FwdOpts o;
        o.tau = float(infer_temperature(t, steps, sc.tau_max, sc.tau_min));
        if (probe) o.logits_out = probe->dev_lg;
        forward(c, w, nb, K, X, S, o);
        if (probe) probe_record(c, *probe, K, X, t, steps, 0);
        const bool first = t == 1 && sc.first_reveal;
        if (pt && t == 1) ck(cudaMemsetAsync(pt->sites, 0, size_t(nb) * n, c.stream), "memset");
        Launch lg(c, "reveal", 0, double(nb) * n * 12);
        launch_pdl(reveal_kernel, nb, 512, smem, c.stream, X, (const float*)w.kappa, (const int*)w.amax, c.L, K,
                   (const int*)w.init_masked, cosine_fraction(t, steps), first ? 1 : 0, pt ? pt->counts + (t - 1) : nullptr,
                   steps, pt && t == 1 ? pt->sites : nullptr, gkeys);
        check_launch("reveal");
    }
    {
        Launch lg(c, "force_residual", 0, double(nb) * n * 12);
        launch_pdl(force_residual_kernel, blocks_for(int64_t(nb) * n), 256, 0, c.stream, X, (const int*)w.amax, int64_t(nb) * n);
        check_launch("force_residual");
    }
    FwdOpts o; // the gamma = 0 pass; kappa at tau = 1 feeds MaxProbScorer (refine.cpp:218-225)
    o.tau = 1.0f;
    o.logits_out = probe ? probe->dev_lg : w.flog;
    forward(c, w, nb, K, X, S, o);
    if (probe) probe_record(c, *probe, K, X, 0, steps, 1);
    {
        Launch lg(c, "finalize", 0, double(nb) * n * 12);
        launch_pdl(finalize_kernel, blocks_for(int64_t(nb) * n), 256, 0, c.stream, X, (const int*)w.amax, (const uint32_t*)w.upd, K,
                   int64_t(nb) * n, n);
        check_launch("finalize");
        ck(cudaMemcpyAsync(w.k1, w.kappa, size_t(nb) * n * 4, cudaMemcpyDeviceToDevice, c.stream), "k1");
    }
    if (probe) {
        probe_record(c, *probe, K, X, 0, steps, 2);
        ++probe->pass;
    }
}

void validate_sched(const cider_schedule* sc, const cider_remask* rm, int K) {
    if (!sc) throw InvalidInput("run_refinement: null schedule");
    if (sc->steps < 1) throw InvalidInput("run_refinement: need T >= 1");
    if (!(sc->tau_min > 0.0) || sc->tau_max < sc->tau_min)
        throw InvalidInput("run_refinement: need tau_max >= tau_min > 0");
    if (K < 1 || K > 32) throw InvalidInput("cider: K must be in 1..32");
    if (rm && rm->mode == CIDER_REMASK_THRESHOLD) {
        if (rm->n_thresholds < 0 || rm->n_thresholds > CIDER_MAX_THRESHOLDS)
            throw InvalidInput("remask: too many thresholds");
        double prev = 1.0; // validate_remask_config (refine.cpp:48-57)
        for (int i = 0; i < rm->n_thresholds; ++i) {
            double t = rm->thresholds[i];
            if (t <= 0.0 || t >= 1.0) throw InvalidInput("remask thresholds must lie in (0,1)");
            if (t >= prev) throw InvalidInput("remask thresholds must be strictly descending");
            prev = t;
        }
    }
    if (rm && rm->mode == CIDER_REMASK_RANK && !(rm->rank_fraction >= 0.0 && rm->rank_fraction <= 1.0))
        throw InvalidInput("remask: rank_fraction must lie in [0,1]");
    if (rm && (rm->mode < 0 || rm->mode > 2)) throw InvalidInput("remask: unknown mode");
}

struct ChunkTrace {
    std::vector<int32_t> rows, steps, mask;      // per bin x CIDER_MAX_THRESHOLDS / K
    std::vector<int32_t> pass_first, n_passes;   // per bin x (1 + CIDER_MAX_THRESHOLDS) / per bin
    std::vector<int32_t> counts, n_counts;       // most recent pass: per bin x max_steps / per bin
    std::vector<uint8_t> sites;                  // most recent pass: per bin x L*K (internal layout)
    int max_steps = 0;
};

PassTrace pass_trace(cider_ctx& c, int m, int steps, int K) {
    PassTrace pt;
    pt.counts = (int*)wsbuf(c, "tr_counts", size_t(m) * steps * 4);
    pt.sites = (uint8_t*)wsbuf(c, "tr_sites", size_t(m) * c.L * K);
    return pt;
}

// fold one traced pass over m bins (bins[i] = chunk-local index, nullptr = identity) into the chunk trace
void trace_pass(cider_ctx& c, ChunkTrace& tr, const PassTrace& pt, int m, int steps, int K, const int* bins) {
    const int n = c.L * K;
    std::vector<int32_t> cnt(size_t(m) * steps);
    std::vector<uint8_t> st(size_t(m) * n);
    ck(cudaMemcpyAsync(cnt.data(), pt.counts, cnt.size() * 4, cudaMemcpyDeviceToHost, c.stream), "d2h");
    ck(cudaMemcpyAsync(st.data(), pt.sites, st.size(), cudaMemcpyDeviceToHost, c.stream), "d2h");
    ck(cudaStreamSynchronize(c.stream), "sync");
    for (int i = 0; i < m; ++i) {
        const int b = bins ? bins[i] : i;
        int& np = tr.n_passes[b];
        if (np < 1 + CIDER_MAX_THRESHOLDS) tr.pass_first[size_t(b) * (1 + CIDER_MAX_THRESHOLDS) + np] = cnt[size_t(i) * steps];
        ++np;
        tr.n_counts[b] = steps;
        for (int s = 0; s < tr.max_steps; ++s)
            tr.counts[size_t(b) * tr.max_steps + s] = s < steps ? cnt[size_t(i) * steps + s] : 0;
        std::copy(st.begin() + size_t(i) * n, st.begin() + size_t(i + 1) * n, tr.sites.begin() + size_t(b) * n);
    }
}

// gather / scatter of per-bin records for threshold-remask buckets
__global__ void gather_rows_kernel(const int* __restrict__ src, int* __restrict__ dst, const int* __restrict__ idx,
                                   int per, int64_t total) {
    int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= total) return;
    dst[i] = src[int64_t(idx[i / per]) * per + i % per];
}
__global__ void scatter_rows_kernel(const int* __restrict__ src, int* __restrict__ dst, const int* __restrict__ idx,
                                    int per, int64_t total) {
    int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= total) return;
    dst[int64_t(idx[i / per]) * per + i % per] = src[i];
}

void copy_rows(cider_ctx& c, const void* src, void* dst, const int* idx, int n, size_t per_words, bool gather) {
    int64_t total = int64_t(n) * int64_t(per_words);
    if (!total) return;
    Launch lg(c, gather ? "bin_gather" : "bin_scatter", 0, double(total) * 8);
    if (gather)
        gather_rows_kernel<<<blocks_for(total), 256, 0, c.stream>>>((const int*)src, (int*)dst, idx, int(per_words), total);
    else
        scatter_rows_kernel<<<blocks_for(total), 256, 0, c.stream>>>((const int*)src, (int*)dst, idx, int(per_words), total);
    check_launch("bin_copy");
}

// Full decode of nb bins (run_refinement / run_with_remasking, refine.cpp:199-292).
// S: device [nb x L x Q]; X: device internal grid [nb x L x K] (output).
void refine_chunk(cider_ctx& c, WS& w, int nb, int K, const float* S, int* X, const cider_schedule& sc,
                  const cider_remask* rm, ChunkTrace* tr) {
    const int n = c.L * K;
    const int64_t total = int64_t(nb) * n;
    fill_i32_kernel<<<blocks_for(total), 256, 0, c.stream>>>(X, -1, total);
    fill_i32_kernel<<<blocks_for(nb), 256, 0, c.stream>>>(w.init_masked, n, nb);
    fill_u32_kernel<<<blocks_for(nb), 256, 0, c.stream>>>(w.upd, K >= 32 ? 0xffffffffu : ((1u << K) - 1u), nb);
    c.launches += 3;
    check_launch("init");
    if (tr) {
        tr->rows.assign(size_t(nb) * CIDER_MAX_THRESHOLDS, 0);
        tr->steps.assign(size_t(nb) * CIDER_MAX_THRESHOLDS, 0);
        tr->mask.assign(size_t(nb) * K, 0);
        tr->pass_first.assign(size_t(nb) * (1 + CIDER_MAX_THRESHOLDS), 0);
        tr->n_passes.assign(nb, 0);
        tr->counts.assign(size_t(nb) * tr->max_steps, 0);
        tr->n_counts.assign(nb, 0);
        tr->sites.assign(size_t(nb) * n, 0);
    }
    {
        PassTrace pt;
        if (tr) pt = pass_trace(c, nb, sc.steps, K);
        masked_pass(c, w, nb, K, S, X, sc.steps, sc, tr ? &pt : nullptr);
        if (tr) trace_pass(c, *tr, pt, nb, sc.steps, K, nullptr);
    }
    const int mode = rm ? rm->mode : CIDER_REMASK_NONE;
    if (mode == CIDER_REMASK_RANK) {
        const int k_low = int(std::floor(rm->rank_fraction * K));
        if (k_low > 0) {
            Launch lg(c, "remask_select", 0, double(total) * 8);
            remask_select_kernel<<<nb, 128, 0, c.stream>>>(X, w.k1, c.L, K, 2, k_low, 0.0, w.upd, w.init_masked, w.nlow, nullptr);
            check_launch("remask_select");
        }
        if (k_low > 0) {
            const int T_rm = remask_steps(sc.steps, k_low, K);
            cider_schedule rs = sc;
            rs.steps = T_rm;
            PassTrace pt;
            if (tr) pt = pass_trace(c, nb, T_rm, K);
            masked_pass(c, w, nb, K, S, X, T_rm, rs, tr ? &pt : nullptr);
            if (tr) {
                trace_pass(c, *tr, pt, nb, T_rm, K, nullptr);
                std::vector<uint32_t> upd(nb);
                ck(cudaMemcpyAsync(upd.data(), w.upd, size_t(nb) * 4, cudaMemcpyDeviceToHost, c.stream), "d2h");
                ck(cudaStreamSynchronize(c.stream), "sync");
                for (int b = 0; b < nb; ++b) {
                    tr->rows[size_t(b) * CIDER_MAX_THRESHOLDS] = k_low;
                    tr->steps[size_t(b) * CIDER_MAX_THRESHOLDS] = T_rm;
                    for (int k = 0; k < K; ++k) tr->mask[size_t(b) * K + k] = (upd[b] >> k) & 1u;
                }
            }
        }
    } else if (mode == CIDER_REMASK_THRESHOLD) {
        // run_with_remasking (refine.cpp:277-292): bins diverge in |K_low| and so in T_rm; each
        // stage buckets its bins by |K_low| and runs every bucket as a compact sub-batch.
        std::vector<char> alive(nb, 1); // the reference stops a bin at its first all-clear stage
        std::vector<int> nlow(nb);
        std::vector<uint32_t> upd(nb);
        for (int s = 0; s < rm->n_thresholds; ++s) {
            {
                Launch lg(c, "remask_select", 0, double(total) * 8);
                remask_select_kernel<<<nb, 128, 0, c.stream>>>(X, w.k1, c.L, K, 1, 0, rm->thresholds[s], w.upd, w.init_masked, w.nlow, nullptr);
                check_launch("remask_select");
            }
            ck(cudaMemcpyAsync(nlow.data(), w.nlow, size_t(nb) * 4, cudaMemcpyDeviceToHost, c.stream), "d2h");
            ck(cudaMemcpyAsync(upd.data(), w.upd, size_t(nb) * 4, cudaMemcpyDeviceToHost, c.stream), "d2h");
            ck(cudaStreamSynchronize(c.stream), "sync");
            std::map<int, std::vector<int>> buckets;
            for (int b = 0; b < nb; ++b) {
                if (!alive[b]) nlow[b] = 0;
                if (nlow[b] == 0) alive[b] = 0;
                else buckets[nlow[b]].push_back(b);
            }
            // bins that are not re-decoded must keep their grid: the select kernel masked their
            // low rows only if nlow > 0, and dead bins were excluded above -> restore those
            std::vector<int> dead_masked;
            for (int b = 0; b < nb; ++b)
                if (!alive[b] && upd[b]) dead_masked.push_back(b);
            if (!dead_masked.empty()) throw std::logic_error("remask: masked rows in a finished bin");
            if (buckets.empty()) break;
            for (auto& [nl, bins] : buckets) {
                const int T_rm = remask_steps(sc.steps, nl, K);
                cider_schedule rs = sc;
                rs.steps = T_rm;
                if (tr)
                    for (int b : bins) {
                        tr->rows[size_t(b) * CIDER_MAX_THRESHOLDS + s] = nl;
                        tr->steps[size_t(b) * CIDER_MAX_THRESHOLDS + s] = T_rm;
                        for (int k = 0; k < K; ++k) tr->mask[size_t(b) * K + k] = (upd[b] >> k) & 1u;
                    }
                const int m = int(bins.size());
                PassTrace pt;
                if (tr) pt = pass_trace(c, m, T_rm, K);
                if (m == nb) {
                    masked_pass(c, w, nb, K, S, X, T_rm, rs, tr ? &pt : nullptr);
                    if (tr) trace_pass(c, *tr, pt, m, T_rm, K, nullptr);
                    continue;
                }
                // compact sub-batch in the tail of dedicated staging buffers
                int* idx = (int*)wsbuf(c, "sub_idx", size_t(m) * 4);
                ck(cudaMemcpyAsync(idx, bins.data(), size_t(m) * 4, cudaMemcpyHostToDevice, c.stream), "h2d");
                float* subS = (float*)wsbuf(c, "sub_S", size_t(m) * c.L * c.Q * 4);
                int* subX = (int*)wsbuf(c, "sub_X", size_t(m) * n * 4);
                int* keep_init = (int*)wsbuf(c, "sub_init", size_t(nb) * 4);
                uint32_t* keep_upd = (uint32_t*)wsbuf(c, "sub_upd", size_t(nb) * 4);
                float* keep_k1 = (float*)wsbuf(c, "sub_k1", size_t(nb) * n * 4);
                ck(cudaMemcpyAsync(keep_init, w.init_masked, size_t(nb) * 4, cudaMemcpyDeviceToDevice, c.stream), "d2d");
                ck(cudaMemcpyAsync(keep_upd, w.upd, size_t(nb) * 4, cudaMemcpyDeviceToDevice, c.stream), "d2d");
                ck(cudaMemcpyAsync(keep_k1, w.k1, size_t(nb) * n * 4, cudaMemcpyDeviceToDevice, c.stream), "d2d");
                copy_rows(c, S, subS, idx, m, size_t(c.L) * c.Q, true);
                copy_rows(c, X, subX, idx, m, n, true);
                copy_rows(c, keep_init, w.init_masked, idx, m, 1, true);
                copy_rows(c, keep_upd, w.upd, idx, m, 1, true);
                float* keep_flog = nullptr;
                if (w.flog) {
                    keep_flog = (float*)wsbuf(c, "sub_flog", size_t(nb) * n * c.Q * 4);
                    ck(cudaMemcpyAsync(keep_flog, w.flog, size_t(nb) * n * c.Q * 4, cudaMemcpyDeviceToDevice, c.stream), "d2d");
                }
                masked_pass(c, w, m, K, subS, subX, T_rm, rs, tr ? &pt : nullptr);
                if (tr) trace_pass(c, *tr, pt, m, T_rm, K, bins.data());
                copy_rows(c, subX, X, idx, m, n, false);
                copy_rows(c, w.k1, keep_k1, idx, m, n, false);
                ck(cudaMemcpyAsync(w.k1, keep_k1, size_t(nb) * n * 4, cudaMemcpyDeviceToDevice, c.stream), "d2d");
                ck(cudaMemcpyAsync(w.init_masked, keep_init, size_t(nb) * 4, cudaMemcpyDeviceToDevice, c.stream), "d2d");
                ck(cudaMemcpyAsync(w.upd, keep_upd, size_t(nb) * 4, cudaMemcpyDeviceToDevice, c.stream), "d2d");
                if (w.flog) {
                    copy_rows(c, w.flog, keep_flog, idx, m, size_t(n) * c.Q, false);
                    ck(cudaMemcpyAsync(w.flog, keep_flog, size_t(nb) * n * c.Q * 4, cudaMemcpyDeviceToDevice, c.stream), "d2d");
                }
            }
        }
    }
}

void upload_model(cider_ctx& c, const float* w) {
    const int Q = c.Q, D = c.D, H = c.H;
    size_t off = 0;
    auto take = [&](size_t n) { const float* p = w + off; off += n; return p; };
    const float* E = take(size_t(Q + 1) * D);
    const float* W = take(size_t(Q) * D);
    const float* V = take(size_t(Q) * D);
    c.Etab = upload_vec(c, E, size_t(Q + 1) * D);
    if (c.bf16) c.Etab16 = upload_mat(c, E, Q + 1, D, false); // (round-to-nearest-even, as the kernel's conversion)
    c.W_host.assign(W, W + size_t(Q) * D);
    if (c.bf16)
        for (float& v : c.W_host) v = bf16_round(v);
    c.W = upload_mat(c, W, Q, D, false);
    c.Wt = upload_mat(c, W, Q, D, true);
    c.Vt = upload_mat(c, V, Q, D, true);
    if (c.bf16 && Q < tc::MLP_HC) { // zero symbol rows Q..127: Lambda-bar 0, r (x) S 0 (S reads 0 there)
        std::vector<float> wp(size_t(tc::MLP_HC) * D, 0.0f), vp(size_t(tc::MLP_HC) * D, 0.0f);
        std::copy(W, W + size_t(Q) * D, wp.begin());
        std::copy(V, V + size_t(Q) * D, vp.begin());
        c.Wpad = upload_mat(c, wp.data(), tc::MLP_HC, D, false);
        c.Vtpad = upload_mat(c, vp.data(), tc::MLP_HC, D, true);
    }
    c.lw.resize(c.N);
    // BF16 mode: every GELU on the device returns 2 GELU(x) (one multiply less per element in the
    // MLP epilogues, mlp_tc.cuh) and the second-layer matrices are stored halved — both exact powers
    // of two, so the products and sums are bit-identical to unscaled ones.
    const float w2s = c.bf16 ? 0.5f : 1.0f;
    for (int l = 0; l < c.N; ++l) {
        LayerW& L = c.lw[l];
        const float* p;
        p = take(size_t(H) * 2 * D); L.g1 = upload_mat(c, p, H, 2 * D, false);
        p = take(H); L.gb1 = upload_vec(c, p, H);
        p = take(size_t(D) * H); L.g2 = upload_mat(c, p, D, H, false, w2s);
        p = take(D); L.gb2 = upload_vec(c, p, D);
        p = take(size_t(H) * D); L.a1 = upload_mat(c, p, H, D, false);
        p = take(H); L.ab1 = upload_vec(c, p, H);
        p = take(size_t(D) * H); L.a2 = upload_mat(c, p, D, H, false, w2s);
        p = take(D); L.ab2 = upload_vec(c, p, D);
        p = take(size_t(H) * 2 * D); L.f1 = upload_mat(c, p, H, 2 * D, false);
        p = take(H); L.fb1 = upload_vec(c, p, H);
        p = take(size_t(D) * H); L.f2 = upload_mat(c, p, D, H, false, w2s);
        p = take(D); L.fb2 = upload_vec(c, p, D);
        L.ak = nullptr;
        L.aq = nullptr;
        L.au = nullptr;
        L.aus = nullptr;
        L.aus16 = nullptr;
    }
    if (c.heads)
        for (int l = 0; l < c.N; ++l) {
            const float* q = take(D);
            c.lw[l].aq = upload_vec(c, q, D);
            const float* k = take(size_t(D) * D);
            c.lw[l].ak = upload_mat(c, k, D, D, false);
            // u_h[col] = sum_{t in head h} q[t] Wk[t][col], from the values the device runs with
            const int dh = D / c.heads;
            auto rv = [&](float v) { return c.bf16 ? double(bf16_round(v)) : double(v); };
            std::vector<float> u(size_t(c.heads) * D);
            for (int h = 0; h < c.heads; ++h)
                for (int col = 0; col < D; ++col) {
                    double acc = 0.0;
                    for (int t = h * dh; t < (h + 1) * dh; ++t) acc += rv(q[t]) * rv(k[size_t(t) * D + col]);
                    u[size_t(h) * D + col] = float(acc);
                }
            DevBuf& b = wbuf(c, u.size() * 4);
            ck(cudaMemcpy(b.p, u.data(), u.size() * 4, cudaMemcpyHostToDevice), "upload");
            c.lw[l].au = b.as<float>();
            if (c.bf16 && c.heads <= 16) {
                // hi + lo bf16 split: the score GEMM recovers u . n to ~2^-16 relative (fp32-grade)
                const float scale = 1.0f / std::sqrt(float(dh));
                std::vector<bf16> m(size_t(64) * D, __float2bfloat16_rn(0.0f));
                for (int h = 0; h < c.heads; ++h)
                    for (int col = 0; col < D; ++col) {
                        const float x = u[size_t(h) * D + col] * scale;
                        const bf16 hi = __float2bfloat16_rn(x);
                        m[size_t(h) * D + col] = hi;
                        m[size_t(16 + h) * D + col] = __float2bfloat16_rn(x - __bfloat162float(hi));
                    }
                DevBuf& bs = wbuf(c, m.size() * 2);
                ck(cudaMemcpy(bs.p, m.data(), m.size() * 2, cudaMemcpyHostToDevice), "upload");
                c.lw[l].aus = bs.p;
                if (c.heads <= 8) { // the same split, 16 rows: hi at h, lo at 8 + h
                    std::vector<bf16> m16(size_t(16) * D, __float2bfloat16_rn(0.0f));
                    for (int h = 0; h < c.heads; ++h)
                        for (int col = 0; col < D; ++col) {
                            m16[size_t(h) * D + col] = m[size_t(h) * D + col];
                            m16[size_t(8 + h) * D + col] = m[size_t(16 + h) * D + col];
                        }
                    DevBuf& b16 = wbuf(c, m16.size() * 2);
                    ck(cudaMemcpy(b16.p, m16.data(), m16.size() * 2, cudaMemcpyHostToDevice), "upload");
                    c.lw[l].aus16 = b16.p;
                }
            }
        }
}

void upload_code(cider_ctx& c) {
    const Tanner& t = *c.tg;
    const Gf& gf = *c.gf;
    std::vector<uint8_t> pin(size_t(t.n_edges()) * c.Q), pout(size_t(t.n_edges()) * c.Q);
    for (int e = 0; e < t.n_edges(); ++e) {
        const int a = t.coef[e], ai = gf.inv(a);
        for (int s = 0; s < c.Q; ++s) {
            pin[size_t(e) * c.Q + s] = uint8_t(gf.mul(ai, s));  // Pi_alpha(u)[s] = u[alpha^-1 s]
            pout[size_t(e) * c.Q + s] = uint8_t(gf.mul(a, s));  // Pi_alpha^-1(m)[s] = m[alpha s]
        }
    }
    c.e_slot = upload_raw(c, t.slot);
    c.e_check = upload_raw(c, t.chk);
    c.check_ptr = upload_raw(c, t.check_ptr);
    c.slot_ptr = upload_raw(c, t.slot_ptr);
    c.slot_edge = upload_raw(c, t.slot_edge);
    c.perm_in = upload_raw(c, pin);
    c.perm_out = upload_raw(c, pout);
}


// T_alpha[k][n] = sum_c W[alpha^-1 c][k] W[c][n]  (= W^T P_alpha W, the coefficient action of
// denoiser.cpp:162-179 as one D x D matrix), stored as GEMM B tiles Tt[alpha][n][k], plus the
// group tables of the two grouped GEMMs (gemm_grp.cuh). Host fp64, threaded over alpha.
void build_tpath(cider_ctx& c) {
    const int Q = c.Q, D = c.D;
    const Gf& gf = *c.gf;
    const Tanner& t = *c.tg;
    std::vector<bf16> T(size_t(Q) * D * D, __float2bfloat16_rn(0.0f));
    const float* W = c.W_host.data();
    auto work = [&](int a0, int stride) {
        std::vector<double> acc(size_t(D) * D);
        for (int alpha = a0; alpha < Q; alpha += stride) {
            if (alpha == 0) continue;
            const int ai = gf.inv(alpha);
            std::fill(acc.begin(), acc.end(), 0.0);
            for (int cc = 0; cc < Q; ++cc) {
                const float* wr = W + size_t(gf.mul(ai, cc)) * D; // W[alpha^-1 c][.]
                const float* wc = W + size_t(cc) * D;             // W[c][.]
                for (int n = 0; n < D; ++n) {
                    const double wn = wc[n];
                    double* row = &acc[size_t(n) * D];
                    for (int k = 0; k < D; ++k) row[k] += double(wr[k]) * wn;
                }
            }
            bf16* dst = &T[size_t(alpha) * D * D];
            for (size_t i = 0; i < size_t(D) * D; ++i) dst[i] = __float2bfloat16_rn(float(acc[i]));
        }
    };
    const int nt = int(std::max(1u, std::min(32u, std::thread::hardware_concurrency())));
    std::vector<std::thread> pool;
    for (int i = 0; i < nt; ++i) pool.emplace_back(work, i, nt);
    for (auto& th : pool) th.join();
    c.Ttab = upload_raw(c, T);
    // normalise GEMM: one group per edge
    // groups in slot-major edge order (slot_edge), so a slot's edges are consecutive groups
    std::vector<int> n_count(t.n_edges(), 1), n_arow(t.n_edges()), n_alpha(t.n_edges()), n_out(t.n_edges());
    for (int g = 0; g < t.n_edges(); ++g) {
        const int e = t.slot_edge[g];
        n_arow[g] = t.slot[e];
        n_alpha[g] = t.coef[e];
        n_out[g] = e;
    }
    c.gn_count = upload_raw(c, n_count);
    c.gn_arow = upload_raw(c, n_arow);
    c.gn_alpha = upload_raw(c, n_alpha);
    c.gn_out = upload_raw(c, n_out);
    // message GEMM: one group per slot, its edges in ascending check order (slot_edge order)
    int maxd = 1;
    for (int l = 0; l < t.slots; ++l) maxd = std::max(maxd, t.slot_ptr[l + 1] - t.slot_ptr[l]);
    std::vector<int> m_count(t.slots), m_arow(size_t(t.slots) * maxd, 0), m_alpha(size_t(t.slots) * maxd, 1), m_out(t.slots);
    for (int l = 0; l < t.slots; ++l) {
        m_count[l] = t.slot_ptr[l + 1] - t.slot_ptr[l];
        m_out[l] = l;
        for (int p = t.slot_ptr[l]; p < t.slot_ptr[l + 1]; ++p) {
            const int e = t.slot_edge[p];
            m_arow[size_t(l) * maxd + (p - t.slot_ptr[l])] = e;
            m_alpha[size_t(l) * maxd + (p - t.slot_ptr[l])] = gf.inv(t.coef[e]);
        }
    }
    c.gm_max_seg = maxd;
    c.gm_count = upload_raw(c, m_count);
    c.gm_arow = upload_raw(c, m_arow);
    c.gm_alpha = upload_raw(c, m_alpha);
    c.gm_out = upload_raw(c, m_out);
    c.tpath = true;
}

void require_device() {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
        throw CudaError("cider: no CUDA device (there is no CPU fallback)");
}

// NCCL, resolved at run time (dlopen) so the library never pins a second NCCL build into a
// process that already has one (PyTorch's); nccl.h supplies the types only.
void* nccl_handle() {
    static void* h = nullptr;
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) throw CudaError("libnccl.so.2 not loadable");
    return h;
}
template <class F>
F nccl_sym(const char* name) {
    void* p = dlsym(nccl_handle(), name);
    if (!p) throw CudaError(std::string("NCCL symbol missing: ") + name);
    return reinterpret_cast<F>(p);
}

} // namespace
} // namespace cider

cider_ctx::~cider_ctx() {
    if (device >= 0) cudaSetDevice(device);
    if (nccl_comm) {
        try { nccl_sym<decltype(&ncclCommDestroy)>("ncclCommDestroy")((ncclComm_t)nccl_comm); } catch (...) {}
    }
    for (auto& [k, g] : graphs)
        if (g.exec) cudaGraphExecDestroy(g.exec);
    for (auto& [k, b] : ws) b.release();
    for (auto& b : wbufs) b.release();
    flush_buf.release();
    for (auto e : ev_pool) cudaEventDestroy(e);
    for (auto& e : events)
        if (e) cudaEventDestroy(e);
    if (stream) cudaStreamDestroy(stream);
}

// ---- batched GF(Q) FFT-BP (bp.cpp:271-368) ----------------------------------
struct cider_bp_ctx {
    int device = 0, Q = 0, L = 0, P = 0, E = 0;
    std::unique_ptr<Gf> gf;
    std::unique_ptr<Tanner> tg;
    cudaStream_t stream = nullptr;
    DevBuf check_ptr, e_slot, e_coef, slot_ptr, slot_edge, mul;
    DevBuf lambda, v2c, c2v, beliefs, residual, hard, active, conv, iters, nact, grid;
    int64_t cap_bins = 0;
    std::mutex mu;
    ~cider_bp_ctx() {
        if (stream) {
            cudaStreamSynchronize(stream);
            cudaStreamDestroy(stream);
        }
    }
};

namespace {
template <typename T>
void bp_upload(cider_bp_ctx& c, DevBuf& b, const std::vector<T>& v) {
    b.ensure(std::max<size_t>(v.size() * sizeof(T), 16));
    if (!v.empty()) ck(cudaMemcpy(b.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice), "upload");
}
void bp_reserve(cider_bp_ctx& c, int64_t B, int K) {
    const size_t rq = size_t(B) * c.L * c.Q, eq = size_t(B) * c.E * c.Q;
    c.lambda.ensure(rq * 8);
    c.beliefs.ensure(rq * 8);
    c.residual.ensure(rq * 8);
    c.v2c.ensure(eq * 8);
    c.c2v.ensure(eq * 8);
    c.hard.ensure(size_t(B) * c.L * 4);
    c.active.ensure(size_t(B) * 4);
    c.conv.ensure(size_t(B) * 4);
    c.iters.ensure(size_t(B) * 4);
    c.nact.ensure(16);
    c.grid.ensure(size_t(B) * std::max(K, 1) * c.L * 4);
}
void bp_validate(const cider_bp_config* cfg) {
    if (!cfg) throw InvalidInput("bp_decode: null config");
    if (cfg->max_iters < 1) throw InvalidInput("bp_decode: need max_iters >= 1");
    if (!(cfg->message_floor > 0.0)) throw InvalidInput("bp_decode: message_floor must be positive");
}
// bp_decode over B bins whose slot beliefs are in c.lambda; leaves hard / beliefs / conv / iters
void bp_run(cider_bp_ctx& c, int64_t B, const cider_bp_config& cfg) {
    const int Q = c.Q, L = c.L, E = c.E, P = c.P;
    const int64_t rows = B * L;
    bp::bp_init_kernel<<<blocks_for(B * E * Q), 256, 0, c.stream>>>(c.lambda.as<double>(), c.e_slot.as<int>(), L, E, Q,
                                                                    B * E * Q, c.v2c.as<double>(), c.c2v.as<double>());
    std::vector<int> ones(size_t(B), 1);
    ck(cudaMemcpyAsync(c.active.p, ones.data(), size_t(B) * 4, cudaMemcpyHostToDevice, c.stream), "h2d");
    int max_deg = 0;
    for (int j = 0; j < P; ++j) max_deg = std::max(max_deg, c.tg->check_ptr[j + 1] - c.tg->check_ptr[j]);
    const size_t smem = size_t(2) * max_deg * Q * sizeof(bp::dd);
    static PerDeviceOnce attr;
    attr.run(current_device(), [&] {
        ck(cudaFuncSetAttribute(bp::bp_check_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024), "attr");
    });
    if (smem > 200 * 1024 || max_deg > 32) throw InvalidInput("bp_decode: check degree x Q too large for one CTA");
    const int rpw = 32 / bp::wht_lanes(Q);                           // edge rows per warp
    const int cthreads = 32 * std::max(1, (max_deg + rpw - 1) / rpw);
    for (int iter = 1; iter <= cfg.max_iters; ++iter) {
        ck(cudaMemsetAsync(c.nact.p, 0, 4, c.stream), "memset");
        bp::bp_check_kernel<<<unsigned(B * P), cthreads, smem, c.stream>>>(c.v2c.as<double>(), c.check_ptr.as<int>(),
                                                                          c.e_coef.as<int>(), c.mul.as<uint8_t>(), P, E, Q,
                                                                          c.active.as<int>(), c.c2v.as<double>());
        bp::bp_belief_kernel<<<unsigned((rows + 7) / 8), 256, 0, c.stream>>>(c.lambda.as<double>(), c.c2v.as<double>(),
                                                                        c.slot_ptr.as<int>(), c.slot_edge.as<int>(), L, E, Q,
                                                                        c.active.as<int>(), rows, c.beliefs.as<double>(),
                                                                        c.hard.as<int>());
        bp::bp_syndrome_kernel<<<blocks_for(B * 32), 256, 0, c.stream>>>(
            c.hard.as<int>(), c.check_ptr.as<int>(), c.e_slot.as<int>(), c.e_coef.as<int>(), c.mul.as<uint8_t>(), P, L, Q,
            iter, cfg.max_iters, cfg.early_exit, B, c.active.as<int>(), c.conv.as<int>(), c.iters.as<int>(),
            c.nact.as<int>());
        bp::bp_var_kernel<<<unsigned((rows + 7) / 8), 256, 0, c.stream>>>(c.lambda.as<double>(), c.c2v.as<double>(),
                                                                     c.slot_ptr.as<int>(), c.slot_edge.as<int>(), L, E, Q,
                                                                     cfg.message_floor, c.active.as<int>(), rows,
                                                                     c.v2c.as<double>());
        check_launch("bp iteration");
        if (iter % 4 == 0 || iter == cfg.max_iters) { // stop once every bin has exited
            int n = 0;
            ck(cudaMemcpyAsync(&n, c.nact.p, 4, cudaMemcpyDeviceToHost, c.stream), "d2h");
            ck(cudaStreamSynchronize(c.stream), "bp");
            if (n == 0) break;
        }
    }
}
} // namespace


extern "C" {

const char* cider_last_error(void) {
    if (g_err_tick >= host_error_tick()) return g_err.c_str(); // the later failure of this thread
    return host_last_error();
}

int cider_device_count(int* n) {
    return guard([&] {
        *n = 0;
        if (cudaGetDeviceCount(n) != cudaSuccess) *n = 0;
    });
}

int cider_create(const cider_model_desc* model, const float* weights, const cider_code_desc* code, int device,
                 cider_ctx** out) {
    return guard([&] {
        *out = nullptr;
        validate_model(model);
        if (!weights) throw InvalidInput("cider_create: null weights");
        auto c = std::make_unique<cider_ctx>();
        c->md = *model;
        c->gf = std::make_unique<Gf>(model->m, model->prim_poly);
        c->Q = c->gf->q;
        c->tg = std::make_unique<Tanner>(code, c->Q);
        c->D = model->dim;
        c->H = model->hidden;
        c->N = model->layers;
        c->heads = model->heads;
        c->bf16 = model->precision == CIDER_BF16;
        c->act_size = c->bf16 ? 2 : 4;
        c->L = c->tg->slots;
        c->P = c->tg->checks;
        c->E = c->tg->n_edges();
        if (c->bf16 && (c->Q % 64 || c->D % 64 || c->H % 64 || c->Q > 256))
            throw InvalidInput("BF16 mode needs Q, D, H multiples of 64 and Q <= 256");
        if (c->heads > ATT_MAXH) throw InvalidInput("cider: at most 32 attention heads");
        if (c->L > 65535) throw InvalidInput("cider: at most 65535 slots"); // 16-bit slot field of the reveal keys
        for (int j = 0; j < c->P; ++j) {
            const int dj = c->tg->check_ptr[j + 1] - c->tg->check_ptr[j];
            if (dj > ATT_MAXD) throw InvalidInput("cider: check degree above 32");
            c->max_check_deg = std::max(c->max_check_deg, dj);
            c->min_check_deg = std::min(c->min_check_deg, dj);
        }
        require_device();
        c->device = device;
        ck(cudaSetDevice(device), "cudaSetDevice");
        cudaDeviceProp prop;
        ck(cudaGetDeviceProperties(&prop, device), "props");
        if (prop.major != 10) throw CudaError("cider: needs an sm_100 (B200) device, found sm_" + std::to_string(prop.major * 10 + prop.minor));
        c->sm_count = prop.multiProcessorCount;
        ck(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "stream");
        upload_model(*c, weights);
        upload_code(*c);
        // D = 256: Module B through precomputed coefficient actions (gemm_grp.cuh). For Q < D (c4)
        // T_alpha has rank <= Q and the D x D GEMM executes 2-4x the FLOPs of the Q-space route, but
        // as one fused grouped GEMM without the projection / permutation / back-projection round trips
        // it is faster (c4: 1093 -> 1197 bins/s). Slots with no incident check (possible in external
        // codes) would make an empty group -> generic path.
        bool every_slot_checked = true;
        for (int l = 0; l < c->L; ++l) every_slot_checked &= c->tg->slot_ptr[l + 1] > c->tg->slot_ptr[l];
        if (c->bf16 && (c->D == 256 || c->D == 128) && every_slot_checked)
            build_tpath(*c);
        ck(cudaDeviceSynchronize(), "upload");
        *out = c.release();
    });
}

void cider_destroy(cider_ctx* ctx) { delete ctx; }

int cider_set_chunk(cider_ctx* ctx, int n) {
    return guard([&] {
        if (n < 0) throw InvalidInput("chunk must be >= 0");
        std::lock_guard<std::mutex> lk(ctx->mu);
        ctx->chunk_req = n;
    });
}

int cider_denoise(cider_ctx* c, int B, int K, const int32_t* X, const float* S, float* logits, float* incoming) {
    return guard([&] {
        if (!c) throw InvalidInput("null context");
        std::lock_guard<std::mutex> lk(c->mu);
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        if (B < 0 || K < 1 || K > 32) throw InvalidInput("cider_denoise: bad B/K");
        const int L = c->L, Q = c->Q, D = c->D, n = L * K;
        for (int64_t i = 0; i < int64_t(B) * n; ++i)
            if (X[i] != -1 && (X[i] < 0 || X[i] >= Q)) throw InvalidInput("embed_grid: token out of range");
        const int chunk = std::max(1, std::min(B, chunk_bins(*c, K)));
        for (int b0 = 0; b0 < B; b0 += chunk) {
            const int nb = std::min(chunk, B - b0);
            WS w = workspace(*c, nb, K, false);
            const int64_t Ms = int64_t(nb) * n;
            float* lg = (float*)wsbuf(*c, "den_logits", size_t(Ms) * Q * 4);
            float* lg_ref = (float*)wsbuf(*c, "den_logits_ref", size_t(Ms) * Q * 4);
            float* inc = incoming ? (float*)wsbuf(*c, "den_inc", size_t(Ms) * D * 4 * c->N) : nullptr;
            float* inc_ref = incoming ? (float*)wsbuf(*c, "den_inc_ref", size_t(Ms) * D * 4 * c->N) : nullptr;
            ck(cudaMemcpyAsync(w.Xio, X + size_t(b0) * n, size_t(Ms) * 4, cudaMemcpyHostToDevice, c->stream), "h2d");
            ck(cudaMemcpyAsync(w.S, S + size_t(b0) * L * Q, size_t(nb) * L * Q * 4, cudaMemcpyHostToDevice, c->stream), "h2d");
            grid_to_internal_kernel<<<blocks_for(Ms), 256, 0, c->stream>>>(w.Xio, w.X, L, K, Ms);
            ++c->launches;
            FwdOpts o;
            o.logits_out = lg;
            o.incoming = inc;
            forward(*c, w, nb, K, w.X, w.S, o);
            rows_to_ref_kernel<<<blocks_for(Ms * Q), 256, 0, c->stream>>>(lg, lg_ref, L, K, Q, Ms * Q, int64_t(n) * Q, 0);
            ++c->launches;
            if (logits)
                ck(cudaMemcpyAsync(logits + size_t(b0) * n * Q, lg_ref, size_t(Ms) * Q * 4, cudaMemcpyDeviceToHost, c->stream), "d2h");
            if (incoming) {
                for (int l = 0; l < c->N; ++l) {
                    rows_to_ref_kernel<<<blocks_for(Ms * D), 256, 0, c->stream>>>(inc + size_t(l) * Ms * D, inc_ref, L, K, D, Ms * D,
                                                                                  int64_t(c->N) * n * D, int64_t(l) * n * D);
                    ++c->launches;
                }
                ck(cudaMemcpyAsync(incoming + size_t(b0) * c->N * n * D, inc_ref, size_t(Ms) * D * c->N * 4, cudaMemcpyDeviceToHost, c->stream), "d2h");
            }
            ck(cudaStreamSynchronize(c->stream), "denoise");
        }
        resolve_stats(*c);
    });
}

// One refinement chunk through a CUDA graph: the T-step loop, residual forcing, the gamma = 0 pass and
// the rank-rule remask stage are a fixed launch sequence with no host round trip (~40 launches per
// forward), so after one eager run per key the whole chunk is captured once and replayed — the host
// no longer paces small-bin-count configurations (c2). Launches are still counted (gpu_launches).
static void refine_chunk_graphed(cider_ctx& c, WS& w, int nb, int K, const float* S, const cider_schedule& sc,
                                 const cider_remask* rm) {
    char key[256];
    // the key names every buffer the captured launches bake in, the final-logits one included
    // (a graph captured without final logits never writes them)
    std::snprintf(key, sizeof(key), "%d/%d/%p/%p/%p/%d/%.17g/%.17g/%d/%d/%.17g/%lld", nb, K, (const void*)S, (void*)w.X,
                  (void*)w.flog, sc.steps, sc.tau_max, sc.tau_min, sc.first_reveal, rm ? rm->mode : -1,
                  rm ? rm->rank_fraction : 0.0, (long long)alloc_generation());
    auto& g = c.graphs[key];
    if (g.exec) {
        ck(cudaGraphLaunch(g.exec, c.stream), "cudaGraphLaunch");
        c.launches += g.launches;
        return;
    }
    if (g.seen++ == 0) { // first time: eager (allocates, sets kernel attributes)
        refine_chunk(c, w, nb, K, S, w.X, sc, rm, nullptr);
        return;
    }
    const int64_t l0 = c.launches;
    const int64_t gen0 = alloc_generation();
    cudaGraph_t graph = nullptr;
    ck(cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal), "cudaStreamBeginCapture");
    try {
        refine_chunk(c, w, nb, K, S, w.X, sc, rm, nullptr);
    } catch (...) {
        cudaStreamEndCapture(c.stream, &graph);
        if (graph) cudaGraphDestroy(graph);
        throw;
    }
    ck(cudaStreamEndCapture(c.stream, &graph), "cudaStreamEndCapture");
    if (alloc_generation() != gen0) throw CudaError("cider: device allocation during graph capture");
    ck(cudaGraphInstantiate(&g.exec, graph, 0), "cudaGraphInstantiate");
    cudaGraphDestroy(graph);
    g.launches = c.launches - l0;
    ck(cudaGraphLaunch(g.exec, c.stream), "cudaGraphLaunch");
}

static void refine_impl(cider_ctx* c, int B, int K, const float* S, bool S_device, const cider_schedule* sched,
                        const cider_remask* rm, int32_t* grid, bool grid_device, float* final_logits, cider_trace* tr) {
    ck(cudaSetDevice(c->device), "cudaSetDevice");
    validate_sched(sched, rm, K);
    if (B < 0) throw InvalidInput("cider_refine: negative B");
    const int L = c->L, Q = c->Q, n = L * K;
    const int chunk = std::max(1, std::min(B, chunk_bins(*c, K)));
    for (int b0 = 0; b0 < B; b0 += chunk) {
        const int nb = std::min(chunk, B - b0);
        WS w = workspace(*c, nb, K, final_logits != nullptr);
        const float* Sd = S + size_t(b0) * L * Q;
        if (!S_device) {
            ck(cudaMemcpyAsync(w.S, Sd, size_t(nb) * L * Q * 4, cudaMemcpyHostToDevice, c->stream), "h2d");
            Sd = w.S;
        }
        ChunkTrace ct;
        if (tr) ct.max_steps = std::max(0, tr->max_steps);
        static const bool no_graph = std::getenv("CIDER_NO_GRAPH") != nullptr;
        const bool graphable = !tr && !c->probe && !c->profiling && !no_graph && (!rm || rm->mode != CIDER_REMASK_THRESHOLD);
        if (graphable && Sd != w.S) { // the graph reads S from the workspace: one key for every caller buffer
            ck(cudaMemcpyAsync(w.S, Sd, size_t(nb) * L * Q * 4, cudaMemcpyDeviceToDevice, c->stream), "d2d");
            Sd = w.S;
        }
        if (graphable) refine_chunk_graphed(*c, w, nb, K, Sd, *sched, rm);
        else refine_chunk(*c, w, nb, K, Sd, w.X, *sched, rm, tr ? &ct : nullptr);
        const int64_t Ms = int64_t(nb) * n;
        int* gdst = grid_device ? grid + size_t(b0) * n : w.Xio;
        grid_to_ref_kernel<<<blocks_for(Ms), 256, 0, c->stream>>>(w.X, gdst, L, K, Ms);
        ++c->launches;
        check_launch("grid_to_ref");
        if (!grid_device)
            ck(cudaMemcpyAsync(grid + size_t(b0) * n, w.Xio, size_t(Ms) * 4, cudaMemcpyDeviceToHost, c->stream), "d2h");
        if (final_logits) {
            float* ref = (float*)wsbuf(*c, "flog_ref", size_t(Ms) * Q * 4);
            rows_to_ref_kernel<<<blocks_for(Ms * Q), 256, 0, c->stream>>>(w.flog, ref, L, K, Q, Ms * Q, int64_t(n) * Q, 0);
            ++c->launches;
            ck(cudaMemcpyAsync(final_logits + size_t(b0) * n * Q, ref, size_t(Ms) * Q * 4, cudaMemcpyDeviceToHost, c->stream), "d2h");
        }
        if (tr || !grid_device || final_logits) ck(cudaStreamSynchronize(c->stream), "refine");
        if (tr) {
            constexpr int NP = 1 + CIDER_MAX_THRESHOLDS;
            for (int b = 0; b < nb; ++b) {
                const size_t B = size_t(b0 + b);
                if (tr->first_reveals) tr->first_reveals[B] = ct.pass_first[size_t(b) * NP];
                for (int s = 0; s < CIDER_MAX_THRESHOLDS; ++s) {
                    if (tr->remask_rows) tr->remask_rows[B * CIDER_MAX_THRESHOLDS + s] = ct.rows[size_t(b) * CIDER_MAX_THRESHOLDS + s];
                    if (tr->remask_steps) tr->remask_steps[B * CIDER_MAX_THRESHOLDS + s] = ct.steps[size_t(b) * CIDER_MAX_THRESHOLDS + s];
                }
                if (tr->remask_mask)
                    for (int k = 0; k < K; ++k) tr->remask_mask[B * K + k] = ct.mask[size_t(b) * K + k];
                if (tr->pass_first_reveals)
                    std::copy(ct.pass_first.begin() + size_t(b) * NP, ct.pass_first.begin() + size_t(b + 1) * NP,
                              tr->pass_first_reveals + B * NP);
                if (tr->n_passes) tr->n_passes[B] = ct.n_passes[b];
                if (tr->reveal_counts && ct.max_steps > 0)
                    std::copy(ct.counts.begin() + size_t(b) * ct.max_steps, ct.counts.begin() + size_t(b + 1) * ct.max_steps,
                              tr->reveal_counts + B * ct.max_steps);
                if (tr->n_reveal_counts) tr->n_reveal_counts[B] = ct.n_counts[b];
                if (tr->first_step_sites)
                    for (int l = 0; l < L; ++l)
                        for (int k = 0; k < K; ++k)
                            tr->first_step_sites[B * n + size_t(k) * L + l] = ct.sites[size_t(b) * n + size_t(l) * K + k];
            }
        }
    }
    if (c->profiling) resolve_stats(*c);
}

int cider_refine(cider_ctx* c, int B, int K, const float* S, const cider_schedule* sched, const cider_remask* rm,
                 int32_t* grid, float* final_logits, cider_trace* tr) {
    return guard([&] {
        if (!c) throw InvalidInput("null context");
        std::lock_guard<std::mutex> lk(c->mu);
        refine_impl(c, B, K, S, false, sched, rm, grid, false, final_logits, tr);
    });
}

int cider_refine_probe(cider_ctx* c, int B, int K, const float* S, const cider_schedule* sched, const cider_remask* rm,
                       int32_t* grid, int n_probe, const int32_t* probe_bins, int max_records, int32_t* meta,
                       int32_t* probe_X, float* probe_logits, int* n_records) {
    return guard([&] {
        if (!c) throw InvalidInput("null context");
        if (rm && rm->mode == CIDER_REMASK_THRESHOLD)
            throw InvalidInput("cider_refine_probe: threshold remasking is not supported (bins diverge into sub-batches)");
        if (n_probe < 0 || max_records < 0 || (n_probe && (!probe_bins || !probe_X)) || !meta || !n_records)
            throw InvalidInput("cider_refine_probe: bad probe arguments");
        std::lock_guard<std::mutex> lk(c->mu);
        Probe p;
        for (int i = 0; i < n_probe; ++i) {
            if (probe_bins[i] < 0 || probe_bins[i] >= B) throw InvalidInput("cider_refine_probe: probe bin out of range");
            p.bins.push_back(probe_bins[i]);
        }
        p.max_rec = max_records;
        p.X = probe_X;
        p.meta = meta;
        p.lg = probe_logits;
        p.dev_lg = (float*)wsbuf(*c, "probe_logits", size_t(round_up(size_t(B) * c->L * K, 128)) * c->Q * 4);
        const int keep_chunk = c->chunk_req;
        c->chunk_req = std::max(1, B); // one device chunk: probe bins index the whole batch
        c->probe = &p;
        try {
            refine_impl(c, B, K, S, false, sched, rm, grid, false, nullptr, nullptr);
        } catch (...) {
            c->probe = nullptr;
            c->chunk_req = keep_chunk;
            throw;
        }
        c->probe = nullptr;
        c->chunk_req = keep_chunk;
        *n_records = p.n_rec;
    });
}

// ura::remask_pass (refine.hpp:97-100, refine.cpp:238-275) with the caller's row confidences (any
// ConfidenceScorer): per bin, rows with conf < threshold are masked and re-decoded for
// remask_steps(T, n_low, K) steps (updatable = those rows), the others stay bit-identical. Bins are
// bucketed by n_low (each bucket one device batch); bins without a low row pass through untouched
// (their final_logits rows are not written, as the reference leaves final_pass_logits alone).
int cider_remask_pass(cider_ctx* c, int B, int K, const float* S, const cider_schedule* sched, const int32_t* grid_in,
                      const double* confidences, double threshold, int32_t* grid_out, float* final_logits,
                      cider_trace* tr) {
    return guard([&] {
        if (!c) throw InvalidInput("null context");
        validate_sched(sched, nullptr, K);
        if (B < 0) throw InvalidInput("remask_pass: negative B");
        if (B && (!grid_in || !grid_out || !confidences || !S)) throw InvalidInput("remask_pass: null buffer");
        std::lock_guard<std::mutex> lk(c->mu);
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        const int L = c->L, Q = c->Q, n = L * K;
        for (int64_t i = 0; i < int64_t(B) * n; ++i)
            if (grid_in[i] < 0 || grid_in[i] >= Q) throw InvalidInput("remask_pass: grid symbol out of range");
        std::copy(grid_in, grid_in + size_t(B) * n, grid_out);
        std::map<int, std::vector<int>> buckets;
        std::vector<uint32_t> low(B, 0);
        for (int b = 0; b < B; ++b) {
            for (int k = 0; k < K; ++k)
                if (confidences[size_t(b) * K + k] < threshold) low[b] |= 1u << k;
            if (low[b]) buckets[__builtin_popcount(low[b])].push_back(b);
        }
        constexpr int NP = 1 + CIDER_MAX_THRESHOLDS;
        if (tr)
            for (int b = 0; b < B; ++b) { // bins with no low row: no pass ran
                if (tr->first_reveals) tr->first_reveals[b] = 0;
                for (int s = 0; s < CIDER_MAX_THRESHOLDS; ++s) {
                    if (tr->remask_rows) tr->remask_rows[size_t(b) * CIDER_MAX_THRESHOLDS + s] = 0;
                    if (tr->remask_steps) tr->remask_steps[size_t(b) * CIDER_MAX_THRESHOLDS + s] = 0;
                }
                if (tr->remask_mask) for (int k = 0; k < K; ++k) tr->remask_mask[size_t(b) * K + k] = (low[b] >> k) & 1u;
                if (tr->pass_first_reveals) std::fill(tr->pass_first_reveals + size_t(b) * NP, tr->pass_first_reveals + size_t(b + 1) * NP, 0);
                if (tr->n_passes) tr->n_passes[b] = 0;
                if (tr->reveal_counts && tr->max_steps > 0)
                    std::fill(tr->reveal_counts + size_t(b) * tr->max_steps, tr->reveal_counts + size_t(b + 1) * tr->max_steps, 0);
                if (tr->n_reveal_counts) tr->n_reveal_counts[b] = 0;
                if (tr->first_step_sites) std::fill(tr->first_step_sites + size_t(b) * n, tr->first_step_sites + size_t(b + 1) * n, 0);
            }
        const int chunk = std::max(1, chunk_bins(*c, K));
        for (auto& [nl, bins] : buckets) {
            cider_schedule rs = *sched;
            rs.steps = remask_steps(sched->steps, nl, K);
            for (size_t i0 = 0; i0 < bins.size(); i0 += size_t(chunk)) {
                const int m = int(std::min(bins.size() - i0, size_t(chunk)));
                const int* bb = bins.data() + i0;
                WS w = workspace(*c, m, K, final_logits != nullptr);
                std::vector<float> Sh(size_t(m) * L * Q);
                std::vector<int32_t> Xh(size_t(m) * n), init(m, nl * L);
                std::vector<uint32_t> upd(m);
                for (int i = 0; i < m; ++i) {
                    const int b = bb[i];
                    std::copy(S + size_t(b) * L * Q, S + size_t(b + 1) * L * Q, Sh.begin() + size_t(i) * L * Q);
                    upd[i] = low[b];
                    for (int k = 0; k < K; ++k) // internal layout (slot, row); low rows masked
                        for (int l = 0; l < L; ++l)
                            Xh[size_t(i) * n + size_t(l) * K + k] = ((low[b] >> k) & 1u) ? -1 : grid_in[size_t(b) * n + size_t(k) * L + l];
                }
                ck(cudaMemcpyAsync(w.S, Sh.data(), Sh.size() * 4, cudaMemcpyHostToDevice, c->stream), "h2d");
                ck(cudaMemcpyAsync(w.X, Xh.data(), Xh.size() * 4, cudaMemcpyHostToDevice, c->stream), "h2d");
                ck(cudaMemcpyAsync(w.init_masked, init.data(), size_t(m) * 4, cudaMemcpyHostToDevice, c->stream), "h2d");
                ck(cudaMemcpyAsync(w.upd, upd.data(), size_t(m) * 4, cudaMemcpyHostToDevice, c->stream), "h2d");
                ChunkTrace ct;
                PassTrace pt;
                if (tr) {
                    ct.max_steps = std::max(0, tr->max_steps);
                    ct.pass_first.assign(size_t(m) * NP, 0);
                    ct.n_passes.assign(m, 0);
                    ct.counts.assign(size_t(m) * ct.max_steps, 0);
                    ct.n_counts.assign(m, 0);
                    ct.sites.assign(size_t(m) * n, 0);
                    pt = pass_trace(*c, m, rs.steps, K);
                }
                masked_pass(*c, w, m, K, w.S, w.X, rs.steps, rs, tr ? &pt : nullptr);
                if (tr) trace_pass(*c, ct, pt, m, rs.steps, K, nullptr);
                ck(cudaMemcpyAsync(Xh.data(), w.X, Xh.size() * 4, cudaMemcpyDeviceToHost, c->stream), "d2h");
                std::vector<float> fl;
                if (final_logits) {
                    fl.resize(size_t(m) * n * Q);
                    ck(cudaMemcpyAsync(fl.data(), w.flog, fl.size() * 4, cudaMemcpyDeviceToHost, c->stream), "d2h");
                }
                ck(cudaStreamSynchronize(c->stream), "remask_pass");
                for (int i = 0; i < m; ++i) {
                    const int b = bb[i];
                    for (int k = 0; k < K; ++k) {
                        if (!((low[b] >> k) & 1u)) continue; // clamped rows stay bit-identical (refine.cpp:270-273)
                        for (int l = 0; l < L; ++l) grid_out[size_t(b) * n + size_t(k) * L + l] = Xh[size_t(i) * n + size_t(l) * K + k];
                    }
                    if (final_logits)
                        for (int k = 0; k < K; ++k)
                            for (int l = 0; l < L; ++l)
                                std::copy(fl.begin() + (size_t(i) * n + size_t(l) * K + k) * Q, fl.begin() + (size_t(i) * n + size_t(l) * K + k + 1) * Q,
                                          final_logits + (size_t(b) * n + size_t(k) * L + l) * Q);
                    if (!tr) continue;
                    if (tr->first_reveals) tr->first_reveals[b] = ct.pass_first[size_t(i) * NP];
                    if (tr->remask_rows) tr->remask_rows[size_t(b) * CIDER_MAX_THRESHOLDS] = nl;
                    if (tr->remask_steps) tr->remask_steps[size_t(b) * CIDER_MAX_THRESHOLDS] = rs.steps;
                    if (tr->pass_first_reveals) tr->pass_first_reveals[size_t(b) * NP] = ct.pass_first[size_t(i) * NP];
                    if (tr->n_passes) tr->n_passes[b] = 1;
                    if (tr->reveal_counts && ct.max_steps > 0)
                        std::copy(ct.counts.begin() + size_t(i) * ct.max_steps, ct.counts.begin() + size_t(i + 1) * ct.max_steps,
                                  tr->reveal_counts + size_t(b) * ct.max_steps);
                    if (tr->n_reveal_counts) tr->n_reveal_counts[b] = ct.n_counts[i];
                    if (tr->first_step_sites)
                        for (int l = 0; l < L; ++l)
                            for (int k = 0; k < K; ++k)
                                tr->first_step_sites[size_t(b) * n + size_t(k) * L + l] = ct.sites[size_t(i) * n + size_t(l) * K + k];
                }
            }
        }
        resolve_stats(*c);
    });
}

int cider_refine_ragged(cider_ctx* c, int B, const int32_t* loads, const float* S, int k_max,
                        const cider_schedule* sched_by_load, const cider_remask* remask_by_load, int32_t* grids) {
    return guard([&] {
        if (!c) throw InvalidInput("null context");
        if (B < 0 || k_max < 1) throw InvalidInput("refine_ragged: need B >= 0 and k_max >= 1");
        if (!sched_by_load) throw InvalidInput("refine_ragged: null schedule table");
        std::vector<int64_t> off(size_t(B) + 1, 0);
        for (int b = 0; b < B; ++b) {
            if (loads[b] < 1 || loads[b] > k_max) throw InvalidInput("refine_ragged: bin load outside 1..k_max");
            off[b + 1] = off[b] + int64_t(loads[b]) * c->L;
        }
        const size_t srow = size_t(c->L) * c->Q;
        std::lock_guard<std::mutex> lk(c->mu);
        for (int k = 1; k <= k_max; ++k) { // one device batch per load (BinTask's load, protocol.hpp:32-40)
            std::vector<int> idx;
            for (int b = 0; b < B; ++b)
                if (loads[b] == k) idx.push_back(b);
            if (idx.empty()) continue;
            const int n = int(idx.size());
            std::vector<float> Sb(size_t(n) * srow);
            for (int i = 0; i < n; ++i) std::copy(S + size_t(idx[i]) * srow, S + size_t(idx[i] + 1) * srow, Sb.begin() + size_t(i) * srow);
            std::vector<int32_t> g(size_t(n) * k * c->L);
            refine_impl(c, n, k, Sb.data(), false, &sched_by_load[k - 1], remask_by_load ? &remask_by_load[k - 1] : nullptr,
                        g.data(), false, nullptr, nullptr);
            for (int i = 0; i < n; ++i) std::copy(g.begin() + size_t(i) * k * c->L, g.begin() + size_t(i + 1) * k * c->L, grids + off[idx[i]]);
        }
    });
}

int cider_refine_device(cider_ctx* c, int B, int K, const float* S_device, const cider_schedule* sched,
                        const cider_remask* rm, int32_t* grid_device) {
    return guard([&] {
        if (!c) throw InvalidInput("null context");
        std::lock_guard<std::mutex> lk(c->mu);
        refine_impl(c, B, K, S_device, true, sched, rm, grid_device, true, nullptr, nullptr);
    });
}

int cider_device_alloc(cider_ctx* c, size_t bytes, void** p) {
    return guard([&] {
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        ck(cudaMalloc(p, std::max<size_t>(bytes, 16)), "cudaMalloc");
    });
}
int cider_device_free(cider_ctx* c, void* p) {
    return guard([&] {
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        ck(cudaFree(p), "cudaFree");
    });
}
int cider_host_alloc(size_t bytes, void** p) { return guard([&] { ck(cudaMallocHost(p, std::max<size_t>(bytes, 16)), "cudaMallocHost"); }); }
int cider_host_free(void* p) { return guard([&] { ck(cudaFreeHost(p), "cudaFreeHost"); }); }
int cider_memcpy_h2d(cider_ctx* c, void* dst, const void* src, size_t n) {
    return guard([&] { ck(cudaMemcpyAsync(dst, src, n, cudaMemcpyHostToDevice, c->stream), "h2d"); });
}
int cider_memcpy_d2h(cider_ctx* c, void* dst, const void* src, size_t n) {
    return guard([&] { ck(cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, c->stream), "d2h"); });
}
int cider_synchronize(cider_ctx* c) {
    return guard([&] {
        ck(cudaStreamSynchronize(c->stream), "sync");
        resolve_stats(*c);
    });
}
int cider_flush_l2(cider_ctx* c) {
    return guard([&] {
        const size_t bytes = size_t(256) << 20; // 2x the 126 MB L2
        c->flush_buf.ensure(bytes);
        static int v = 0;
        flush_kernel<<<blocks_for(int64_t(bytes / 16)), 256, 0, c->stream>>>((int4*)c->flush_buf.p, int64_t(bytes / 16), ++v);
        check_launch("flush");
    });
}
int cider_event_record(cider_ctx* c, int slot) {
    return guard([&] {
        if (slot < 0 || slot >= 64) throw InvalidInput("event slot out of range");
        if (!c->events[slot]) ck(cudaEventCreate(&c->events[slot]), "event");
        ck(cudaEventRecord(c->events[slot], c->stream), "event record");
    });
}
int cider_event_elapsed(cider_ctx* c, int a, int b, float* ms) {
    return guard([&] {
        ck(cudaEventSynchronize(c->events[b]), "event sync");
        ck(cudaEventElapsedTime(ms, c->events[a], c->events[b]), "elapsed");
    });
}
int cider_set_profiling(cider_ctx* c, int on) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(c->mu);
        resolve_stats(*c);
        c->profiling = on != 0;
    });
}
int64_t cider_launch_count(cider_ctx* c) { return c ? c->launches : -1; }
int cider_kernel_stats(cider_ctx* c, int idx, char* name, int name_len, int64_t* launches, double* ms, double* flops,
                       double* bytes) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(c->mu);
        resolve_stats(*c);
        if (idx < 0 || idx >= int(c->stats.size())) throw InvalidInput("stat index out of range");
        auto it = c->stats.begin();
        std::advance(it, idx);
        std::snprintf(name, size_t(name_len), "%s", it->first.c_str());
        *launches = it->second.launches;
        *ms = it->second.ms;
        *flops = it->second.flops;
        *bytes = it->second.bytes;
    });
}
int cider_reset_stats(cider_ctx* c) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(c->mu);
        resolve_stats(*c);
        c->stats.clear();
        c->launches = 0;
    });
}


// Batched GF(Q) check-node update in the WHT domain (bp.cpp:128-149, 222-269):
// for each of n_checks checks with d incident edges, all d extrinsic check-to-variable messages.
int cider_check_update_wht(int m, int n_checks, int d, const double* v2c, const int32_t* coeffs, double* c2v,
                           int device) {
    return guard([&] {
        Gf gf(m, 0);
        const int Q = gf.q;
        if (n_checks < 0 || d < 1 || d > WHT_MAXD) throw InvalidInput("check_update_wht: need 1 <= d <= 32");
        for (int64_t i = 0; i < int64_t(n_checks) * d; ++i)
            if (coeffs[i] <= 0 || coeffs[i] >= Q) throw InvalidInput("coeff_map: coefficient must be a nonzero field element");
        if (n_checks == 0) return;
        require_device();
        ck(cudaSetDevice(device), "cudaSetDevice");
        std::vector<uint8_t> mul(size_t(Q) * Q);
        for (int a = 0; a < Q; ++a)
            for (int b = 0; b < Q; ++b) mul[size_t(a) * Q + b] = uint8_t(gf.mul(a, b));
        const size_t nmsg = size_t(n_checks) * d * Q;
        DevBuf din, dout, dcf, dmul;
        din.ensure(nmsg * 8);
        dout.ensure(nmsg * 8);
        dcf.ensure(size_t(n_checks) * d * 4);
        dmul.ensure(mul.size());
        cudaStream_t st;
        ck(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
        ck(cudaMemcpyAsync(din.p, v2c, nmsg * 8, cudaMemcpyHostToDevice, st), "h2d");
        ck(cudaMemcpyAsync(dcf.p, coeffs, size_t(n_checks) * d * 4, cudaMemcpyHostToDevice, st), "h2d");
        ck(cudaMemcpyAsync(dmul.p, mul.data(), mul.size(), cudaMemcpyHostToDevice, st), "h2d");
        const size_t smem = size_t(2) * d * Q * 8;
        if (smem > 200 * 1024) throw InvalidInput("check_update_wht: d * Q too large for one CTA");
        ck(cudaFuncSetAttribute(wht_check_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)), "attr");
        const int rpw = 32 / wht_lanes(Q);
        wht_check_update_kernel<<<n_checks, 32 * std::max(1, (d + rpw - 1) / rpw), smem, st>>>(
            din.as<double>(), dcf.as<int>(), dmul.as<uint8_t>(), d, Q, dout.as<double>());
        check_launch("wht_check_update");
        ck(cudaMemcpyAsync(c2v, dout.p, nmsg * 8, cudaMemcpyDeviceToHost, st), "d2h");
        ck(cudaStreamSynchronize(st), "wht");
        cudaStreamDestroy(st);
        din.release(); dout.release(); dcf.release(); dmul.release();
    });
}

int cider_bp_create(int m, uint32_t prim_poly, const cider_code_desc* code, int device, cider_bp_ctx** out) {
    return guard([&] {
        *out = nullptr;
        if (m < 1 || m > 8) throw InvalidInput("bp: GF(2^m) needs 1 <= m <= 8"); // Q <= 256 (BP_QMAX)
        auto c = std::make_unique<cider_bp_ctx>();
        c->gf = std::make_unique<Gf>(m, prim_poly);
        c->Q = c->gf->q;
        c->tg = std::make_unique<Tanner>(code, c->Q);
        c->L = c->tg->slots;
        c->P = c->tg->checks;
        c->E = c->tg->n_edges();
        require_device();
        c->device = device;
        ck(cudaSetDevice(device), "cudaSetDevice");
        ck(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "stream");
        std::vector<uint8_t> mul(size_t(c->Q) * c->Q);
        for (int a = 0; a < c->Q; ++a)
            for (int b = 0; b < c->Q; ++b) mul[size_t(a) * c->Q + b] = uint8_t(c->gf->mul(a, b));
        bp_upload(*c, c->check_ptr, c->tg->check_ptr);
        bp_upload(*c, c->e_slot, c->tg->slot);
        bp_upload(*c, c->e_coef, c->tg->coef);
        bp_upload(*c, c->slot_ptr, c->tg->slot_ptr);
        bp_upload(*c, c->slot_edge, c->tg->slot_edge);
        bp_upload(*c, c->mul, mul);
        *out = c.release();
    });
}

void cider_bp_destroy(cider_bp_ctx* c) { delete c; }

int cider_bp_decode(cider_bp_ctx* c, int B, const double* lambda, const cider_bp_config* cfg, int32_t* hard,
                    double* marginals, int32_t* converged, int32_t* iters) {
    return guard([&] {
        if (!c) throw InvalidInput("bp_decode: null context");
        bp_validate(cfg);
        if (B < 0) throw InvalidInput("bp_decode: negative batch");
        if (B == 0) return;
        std::lock_guard<std::mutex> lk(c->mu);
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        bp_reserve(*c, B, 1);
        const size_t rq = size_t(B) * c->L * c->Q;
        ck(cudaMemcpyAsync(c->lambda.p, lambda, rq * 8, cudaMemcpyHostToDevice, c->stream), "h2d");
        bp_run(*c, B, *cfg);
        ck(cudaMemcpyAsync(hard, c->hard.p, size_t(B) * c->L * 4, cudaMemcpyDeviceToHost, c->stream), "d2h");
        if (marginals) ck(cudaMemcpyAsync(marginals, c->beliefs.p, rq * 8, cudaMemcpyDeviceToHost, c->stream), "d2h");
        if (converged) ck(cudaMemcpyAsync(converged, c->conv.p, size_t(B) * 4, cudaMemcpyDeviceToHost, c->stream), "d2h");
        if (iters) ck(cudaMemcpyAsync(iters, c->iters.p, size_t(B) * 4, cudaMemcpyDeviceToHost, c->stream), "d2h");
        ck(cudaStreamSynchronize(c->stream), "bp_decode");
    });
}

int cider_sic_decode(cider_bp_ctx* c, int B, int K, const double* S, const cider_bp_config* cfg, double cancel_value,
                     int32_t* grid, int32_t* stage_converged, int32_t* stage_iters) {
    return guard([&] {
        if (!c) throw InvalidInput("sic_decode: null context");
        if (K < 1) throw InvalidInput("sic_decode: need K >= 1");
        bp_validate(cfg);
        if (B < 0) throw InvalidInput("sic_decode: negative batch");
        if (B == 0) return;
        if (std::isnan(cancel_value)) cancel_value = std::log(static_cast<double>(K) / c->Q); // bp.cpp:352-353
        std::lock_guard<std::mutex> lk(c->mu);
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        bp_reserve(*c, B, K);
        const int64_t rows = int64_t(B) * c->L;
        ck(cudaMemcpyAsync(c->residual.p, S, size_t(rows) * c->Q * 8, cudaMemcpyHostToDevice, c->stream), "h2d");
        std::vector<int32_t> conv{}, its{};
        conv.resize(static_cast<size_t>(B));
        its.resize(static_cast<size_t>(B));
        for (int stage = 0; stage < K; ++stage) {
            bp::slot_beliefs_kernel<<<blocks_for(rows, 64), 64, 0, c->stream>>>(c->residual.as<double>(), rows, c->Q,
                                                                                c->lambda.as<double>());
            bp_run(*c, B, *cfg);
            bp::sic_cancel_kernel<<<blocks_for(rows), 256, 0, c->stream>>>(c->hard.as<int>(), c->L, c->Q, cancel_value, rows,
                                                                          c->residual.as<double>(), c->grid.as<int>(), K, stage);
            check_launch("sic stage");
            if (stage_converged || stage_iters) {
                ck(cudaMemcpyAsync(conv.data(), c->conv.p, size_t(B) * 4, cudaMemcpyDeviceToHost, c->stream), "d2h");
                ck(cudaMemcpyAsync(its.data(), c->iters.p, size_t(B) * 4, cudaMemcpyDeviceToHost, c->stream), "d2h");
                ck(cudaStreamSynchronize(c->stream), "sic");
                for (int b = 0; b < B; ++b) {
                    if (stage_converged) stage_converged[size_t(b) * K + stage] = conv[b];
                    if (stage_iters) stage_iters[size_t(b) * K + stage] = its[b];
                }
            }
        }
        ck(cudaMemcpyAsync(grid, c->grid.p, size_t(B) * K * c->L * 4, cudaMemcpyDeviceToHost, c->stream), "d2h");
        ck(cudaStreamSynchronize(c->stream), "sic_decode");
    });
}

int cider_workload_bins_device(const cider_workload_desc* w, const int32_t* edges, int64_t first, int n,
                               int32_t* truth_device, float* S_device, int device) {
    return guard([&] {
        Gf gf(w->m, 0);
        const int L = w->slots, P = w->checks, K = w->k, Q = gf.q;
        if (K < 1) throw InvalidInput("sample_codewords: need K >= 1");
        if (K > wl::WL_MAXK || Q > wl::WL_MAXQ || L > wl::WL_MAXL) throw InvalidInput("workload_bins_device: shape too large");
        if (n <= 0) return;
        cider_code_desc cd{P, L, L * w->col_weight, edges};
        Tanner t(&cd, Q);
        std::vector<int> info, pivot;
        std::vector<uint8_t> red, mul(size_t(Q) * Q);
        systematic_tables(gf, t, info, pivot, red);
        for (int a = 0; a < Q; ++a)
            for (int b = 0; b < Q; ++b) mul[size_t(a) * Q + b] = uint8_t(gf.mul(a, b));
        require_device();
        ck(cudaSetDevice(device), "cudaSetDevice");
        DevBuf di, dp, dr, dm;
        auto up = [&](DevBuf& b, const void* src, size_t bytes) {
            b.ensure(std::max<size_t>(bytes, 16));
            if (bytes) ck(cudaMemcpy(b.p, src, bytes, cudaMemcpyHostToDevice), "upload");
        };
        up(di, info.data(), info.size() * 4);
        up(dp, pivot.data(), pivot.size() * 4);
        up(dr, red.data(), red.size());
        up(dm, mul.data(), mul.size());
        wl::Sys sys{int(info.size()), int(pivot.size()), di.as<int>(), dp.as<int>(), dr.as<uint8_t>(), dm.as<uint8_t>()};
        const double sigma = std::pow(10.0, -w->snr_db / 20.0);
        wl::workload_bins_kernel<<<unsigned((n + 63) / 64), 64>>>(sys, L, K, Q, sigma, w->p_erase, w->p_false,
                                                                  w->master_seed, first, n, truth_device, S_device);
        check_launch("workload_bins");
        ck(cudaDeviceSynchronize(), "workload_bins");
        di.release(); dp.release(); dr.release(); dm.release();
    });
}

int cider_grid_pack_u8(cider_ctx* c, const int32_t* grid_device, uint8_t* out_device, size_t n) {
    return guard([&] {
        if (!c) throw InvalidInput("null context");
        if (c->Q > 256) throw InvalidInput("grid_pack_u8: Q > 256");
        if ((reinterpret_cast<uintptr_t>(grid_device) & 15) || (reinterpret_cast<uintptr_t>(out_device) & 3))
            throw InvalidInput("grid_pack_u8: grid must be 16-byte and output 4-byte aligned");
        if (!n) return;
        pack_u8_kernel<<<blocks_for(int64_t((n + 3) / 4)), 256, 0, c->stream>>>(grid_device, out_device, int64_t(n));
        ++c->launches;
        check_launch("pack_u8");
    });
}

// ---- debug guard bands (an out-of-bounds write check in place of compute-sanitizer) ----------------
__global__ void guard_count_kernel(const uint8_t* __restrict__ a, size_t n, unsigned long long* bad) {
    unsigned long long c = 0;
    for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) c += a[i] != 0xA5;
    if (c) atomicAdd(bad, c); // a count, not data
}

int cider_set_debug_guard(cider_ctx* c, size_t bytes) {
    return guard([&] {
        if (!c) throw InvalidInput("null context");
        std::lock_guard<std::mutex> lk(c->mu);
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        ck(cudaStreamSynchronize(c->stream), "sync");
        for (auto& g : c->graphs)
            if (g.second.exec) cudaGraphExecDestroy(g.second.exec);
        c->graphs.clear();
        c->maps.clear();
        for (auto& kv : c->ws) kv.second.release(); // reallocated with (or without) bands on next use
        c->ws.clear();
        c->debug_guard = round_up(bytes, 256);
    });
}

int cider_debug_check(cider_ctx* c, int64_t* damaged) {
    return guard([&] {
        if (!c || !damaged) throw InvalidInput("null argument");
        std::lock_guard<std::mutex> lk(c->mu);
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        ck(cudaStreamSynchronize(c->stream), "sync");
        DevBuf cnt;
        cnt.ensure(8);
        int64_t total = 0;
        std::string names;
        for (auto& kv : c->ws) {
            const DevBuf& b = kv.second;
            if (!b.guard) continue;
            unsigned long long h = 0;
            ck(cudaMemsetAsync(cnt.p, 0, 8, c->stream), "memset");
            guard_count_kernel<<<64, 256, 0, c->stream>>>(static_cast<const uint8_t*>(b.base), b.guard, cnt.as<unsigned long long>());
            guard_count_kernel<<<64, 256, 0, c->stream>>>(static_cast<const uint8_t*>(b.p) + b.bytes, b.guard, cnt.as<unsigned long long>());
            check_launch("guard_count");
            ck(cudaMemcpyAsync(&h, cnt.p, 8, cudaMemcpyDeviceToHost, c->stream), "d2h");
            ck(cudaStreamSynchronize(c->stream), "sync");
            if (h) {
                total += int64_t(h);
                names += (names.empty() ? "" : ", ") + kv.first;
            }
        }
        cnt.release();
        *damaged = total;
        g_err = names.empty() ? std::string("guard bands intact") : "guard bands overwritten: " + names;
        g_err_tick = error_tick();
    });
}

// test-only positive control: writes one byte `offset` bytes past the end of workspace buffer `name`
int cider_debug_poke(cider_ctx* c, const char* name, int64_t offset) {
    return guard([&] {
        if (!c || !name) throw InvalidInput("null argument");
        std::lock_guard<std::mutex> lk(c->mu);
        auto it = c->ws.find(name);
        if (it == c->ws.end() || !it->second.guard) throw InvalidInput("debug_poke: no guarded buffer of that name");
        if (offset < 0 || size_t(offset) >= it->second.guard) throw InvalidInput("debug_poke: offset outside the guard band");
        ck(cudaMemsetAsync(static_cast<char*>(it->second.p) + it->second.bytes + offset, 0x00, 1, c->stream), "poke");
        ck(cudaStreamSynchronize(c->stream), "sync");
    });
}

int cider_nccl_unique_id(char out[128]) {
    return guard([&] {
        ncclUniqueId uid;
        ncclResult_t r = nccl_sym<decltype(&ncclGetUniqueId)>("ncclGetUniqueId")(&uid);
        if (r != ncclSuccess) throw CudaError("ncclGetUniqueId failed");
        std::memcpy(out, uid.internal, sizeof(uid.internal));
    });
}
int cider_nccl_init(cider_ctx* c, const char id[128], int rank, int world) {
    return guard([&] {
        if (!c) throw InvalidInput("null context");
        if (world < 1 || rank < 0 || rank >= world) throw InvalidInput("nccl: bad rank/world");
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        ncclUniqueId uid;
        std::memcpy(uid.internal, id, sizeof(uid.internal));
        ncclComm_t comm = nullptr;
        ncclResult_t r = nccl_sym<decltype(&ncclCommInitRank)>("ncclCommInitRank")(&comm, world, uid, rank);
        if (r != ncclSuccess) throw CudaError("ncclCommInitRank failed (" + std::to_string(int(r)) + ")");
        c->nccl_comm = comm;
    });
}

int cider_nccl_allgather(cider_ctx* c, const void* send, void* recv, size_t n) {
    return guard([&] {
        if (!c || !c->nccl_comm) throw InvalidInput("nccl: communicator not initialised");
        ncclResult_t r = nccl_sym<decltype(&ncclAllGather)>("ncclAllGather")(send, recv, n, ncclUint8,
                                                                            (ncclComm_t)c->nccl_comm, c->stream);
        if (r != ncclSuccess) throw CudaError("ncclAllGather failed (" + std::to_string(int(r)) + ")");
        ++c->launches;
    });
}

} // extern "C"

// ---- batched AMP slot detector (amp.cpp:63-148) ---------------------------------
struct cider_amp_ctx {
    int device = 0, L = 0, q = 0, n_s = 0;
    cudaStream_t stream = nullptr;
    cider::DevBuf At, y, S, bad;
    std::mutex mu;
    ~cider_amp_ctx() {
        if (device >= 0) cudaSetDevice(device);
        At.release(); y.release(); S.release(); bad.release();
        if (stream) cudaStreamDestroy(stream);
    }
};

using namespace cider;

int cider_amp_create(int L, int q, int n_s, const double* dicts, int device, cider_amp_ctx** out) {
    return guard([&] {
        if (!out) throw InvalidInput("amp: null output");
        *out = nullptr;
        if (L < 1 || q < 1 || n_s < 1) throw InvalidInput("amp: need L, q, n_s >= 1");
        if (n_s > q) throw InvalidInput("partial_dft: n_s must not exceed Q"); // sim.cpp:12
        if (!dicts) throw InvalidInput("amp: null dictionaries");
        require_device();
        auto c = std::make_unique<cider_amp_ctx>();
        c->device = device; c->L = L; c->q = q; c->n_s = n_s;
        ck(cudaSetDevice(device), "cudaSetDevice");
        cudaDeviceProp prop;
        ck(cudaGetDeviceProperties(&prop, device), "props");
        if (prop.major != 10) throw CudaError("cider: needs an sm_100 (B200) device, found sm_" + std::to_string(prop.major * 10 + prop.minor));
        ck(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "stream");
        // reference layout [l][col][r] -> device [l][r][col] (a thread per column reads rows coalesced)
        std::vector<double> t(size_t(L) * n_s * q * 2);
        for (int l = 0; l < L; ++l)
            for (int col = 0; col < q; ++col)
                for (int r = 0; r < n_s; ++r)
                    for (int k = 0; k < 2; ++k)
                        t[((size_t(l) * n_s + r) * q + col) * 2 + k] = dicts[((size_t(l) * q + col) * n_s + r) * 2 + k];
        c->At.ensure(t.size() * 8);
        ck(cudaMemcpy(c->At.p, t.data(), t.size() * 8, cudaMemcpyHostToDevice), "upload");
        c->bad.ensure(16);
        *out = c.release();
    });
}

void cider_amp_destroy(cider_amp_ctx* ctx) { delete ctx; }

int cider_amp_detect(cider_amp_ctx* c, int B, const double* y, const cider_amp_config* cfg, double* S) {
    return guard([&] {
        if (!c || !cfg) throw InvalidInput("amp_detect: null argument");
        if (cfg->iters < 1) throw InvalidInput("amp_detect: need at least one iteration");  // amp.cpp:66
        if (!(cfg->rho_bg > 0.0 && cfg->rho_bg < 1.0)) throw InvalidInput("amp: rho_bg must lie in (0,1)");
        if (!(cfg->sigma_u2 > 0.0)) throw InvalidInput("amp: sigma_u2 must be positive"); // amp.cpp:22-27
        if (B < 0) throw InvalidInput("amp_detect: negative batch");
        if (B == 0) return;
        std::lock_guard<std::mutex> lk(c->mu);
        ck(cudaSetDevice(c->device), "cudaSetDevice");
        const size_t ny = size_t(B) * c->L * c->n_s * 2, ns = size_t(B) * c->L * c->q;
        c->y.ensure(ny * 8);
        c->S.ensure(ns * 8);
        ck(cudaMemcpyAsync(c->y.p, y, ny * 8, cudaMemcpyHostToDevice, c->stream), "h2d");
        const int big = 1 << 30;
        ck(cudaMemcpyAsync(c->bad.p, &big, 4, cudaMemcpyHostToDevice, c->stream), "h2d");
        AmpParams p;
        p.iters = cfg->iters;
        p.rho_bg = cfg->rho_bg;
        p.sigma_u2 = cfg->sigma_u2;
        p.floor = cfg->evidence_floor;
        p.log_rho = std::log(cfg->rho_bg);
        p.log1m_rho = std::log1p(-cfg->rho_bg);
        const size_t smem = size_t(3 * c->n_s + c->q) * 16 + size_t(c->q) * 8;
        if (smem > 227 * 1024) throw InvalidInput("amp_detect: q / n_s too large for one CTA");
        if (smem > 48 * 1024)
            ck(cudaFuncSetAttribute(amp_detect_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)), "smem attr");
        amp_detect_kernel<256><<<unsigned(int64_t(B) * c->L), 256, smem, c->stream>>>(
            (const double2*)c->At.p, (const double2*)c->y.p, B, c->L, c->q, c->n_s, p, (double*)c->S.p, (int*)c->bad.p);
        check_launch("amp_detect");
        int bad = 0;
        ck(cudaMemcpyAsync(&bad, c->bad.p, 4, cudaMemcpyDeviceToHost, c->stream), "d2h");
        ck(cudaMemcpyAsync(S, c->S.p, ns * 8, cudaMemcpyDeviceToHost, c->stream), "d2h");
        ck(cudaStreamSynchronize(c->stream), "amp_detect");
        if (bad != (1 << 30)) throw std::runtime_error("amp_detect: non-finite residual at iteration " + std::to_string(bad));
    });
}
