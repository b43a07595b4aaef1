// Internal declarations shared by the translation units of libparl_gpu.so.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <utility>

#include "parl_gpu.h"

namespace parl_gpu {

using bf16 = __nv_bfloat16;

// ---------------------------------------------------------------------------
// status plumbing
struct Error {
    parl_status code;
    std::string msg;
};

#define PARL_CUDA(expr)                                                                  \
    do {                                                                                 \
        cudaError_t e_ = (expr);                                                         \
        if (e_ != cudaSuccess)                                                           \
            throw ::parl_gpu::Error{PARL_E_CUDA, std::string(#expr ": ") + cudaGetErrorString(e_)}; \
    } while (0)

#define PARL_REQUIRE(cond, code, msg)                       \
    do {                                                    \
        if (!(cond)) throw ::parl_gpu::Error{code, msg};    \
    } while (0)

// counts kernel launches per process (bench evidence: "gpu_launches") and fails
// loudly on a launch error right at its launch site (a later library call such as
// a CUB sort would otherwise consume the error and skip its own work)
extern uint64_t g_launches;
#define PARL_LAUNCHED()                                                                                  \
    do {                                                                                                 \
        ++::parl_gpu::g_launches;                                                                        \
        cudaError_t e_ = cudaPeekAtLastError();                                                          \
        if (e_ != cudaSuccess)                                                                           \
            throw ::parl_gpu::Error{PARL_E_CUDA, std::string("kernel launch at ") + __FILE__ + ":" +      \
                                                     std::to_string(__LINE__) + ": " + cudaGetErrorString(e_)}; \
    } while (0)

// ---------------------------------------------------------------------------
// Programmatic dependent launch: kernels launched with launch_pdl() may start
// while the previous kernel of the stream is still draining; they run their
// input-independent prologue, then pdl_wait() for the predecessor's completion
// (and memory) before touching its outputs.  pdl_trigger() lets the successor
// launch before this grid has fully exited.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// pull a line into L2 ahead of its load (memory-level parallelism without registers)
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

bool pdl_enabled();  // PARL_PDL=0 disables (diagnostics)

template <class... KArgs, class... Args>
void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ---------------------------------------------------------------------------
// small device helpers
template <class T>
__device__ __forceinline__ float to_f(T v);
template <>
__device__ __forceinline__ float to_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_f<bf16>(bf16 v) { return __bfloat162float(v); }

template <class T>
__device__ __forceinline__ T from_f(float v);
template <>
__device__ __forceinline__ float from_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ bf16 from_f<bf16>(float v) { return __float2bfloat16_rn(v); }

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__device__ __forceinline__ float gelu_f(float x) { return 0.5f * x * erfcf(-x * 0.70710678118654752f); }
__device__ __forceinline__ float gelu_grad_f(float x) {
    return 0.5f * erfcf(-x * 0.70710678118654752f) + x * 0.39894228040143267794f * __expf(-0.5f * x * x);
}

inline int cdiv(long a, long b) { return (int)((a + b - 1) / b); }

// ---------------------------------------------------------------------------
// GEMM: C[M x N] = sum_k A(m,k) * B(n,k), fp32 accumulation, fused epilogue.
// A(m,k) = A[m*sam + k*sak], B(n,k) = B[n*sbn + k*sbk] (either may be
// K-major or MN-major).  Output rows of C are indexed by m.
enum Epi : int {
    EPI_F32 = 0,          // Cf  = acc (+bias)
    EPI_F32_ACC = 1,      // Cf += acc                      (weight-gradient accumulate)
    EPI_ACT = 2,          // Ca  = act(acc + bias)          (bias may be null)
    EPI_RESID = 3,        // Cf  = resid + acc + bias       (fp32 residual stream)
    EPI_GELU = 4,         // Ca  = u = acc + bias; Caux = gelu(u)
    EPI_GELU_BWD = 5,     // Ca  = acc * gelu'(aux_in)
    EPI_LSE = 6,          // logits (+bias) -> per-row (max, sumexp) partials + label gather
    EPI_GELU_ACT = 7,     // Ca  = gelu(acc + bias)         (forward without an activation cache)
};

struct GemmArgs {
    int M = 0, N = 0, K = 0;
    const void* A = nullptr;
    long sam = 0, sak = 0;
    const void* B = nullptr;
    long sbn = 0, sbk = 0;
    int epi = EPI_F32;
    const float* bias = nullptr;  // [N]
    float* Cf = nullptr;          // fp32 out [M x ldc]
    long ldc = 0;
    const float* resid = nullptr; // fp32 residual [M x ldc]
    void* Ca = nullptr;           // act-dtype out [M x ldca]
    long ldca = 0;
    void* Caux = nullptr;         // second act-dtype out [M x ldca]
    const void* aux_in = nullptr; // act-dtype aux input [M x ldca] (gelu pre-activation)
    // EPI_LSE
    const int32_t* labels = nullptr;  // [M] target column per row
    float* part = nullptr;            // [M x n_parts x 2] (max, sum) partials
    float* target = nullptr;          // [M] logit at the label column
    float* logits_out = nullptr;      // optional fp32 logits store [M x ldc] (policy, for backward)
    void* logits_act = nullptr;       // optional act-dtype logits store [M x ldca]
    int n_parts = 0, part_cols = 0;   // vocab columns per partial
};

template <class T>
void gemm_simt(const GemmArgs& g, cudaStream_t st);
// tcgen05 path (bf16 only).  Returns false if the shape/layout is not supported.
bool gemm_tc(const GemmArgs& g, cudaStream_t st);
// n equal-shape GEMMs; one grouped CTA-pair launch when n is 2 or 3 and they qualify
bool gemm_tc_multi(const GemmArgs* gs, int n, cudaStream_t st);
// all weight-gradient GEMMs of a layer in one launch (MN-major A and B, shared K, fp32 accumulate)
bool gemm_tc_group_dw(const GemmArgs* gs, int n, cudaStream_t st);

}  // namespace parl_gpu
