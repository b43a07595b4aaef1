// FFMA tile GEMM with the fused epilogues of the hot path.
//
// This is the contraction kernel of the FP32 precision mode (BASELINE
// configs[0] is specified fp32; fp32 accumulation of fp32 operands keeps the
// oracle tolerance of SURVEY.md §8c, which tf32/bf16 tensor-core inputs cannot).
// In BF16 mode the tcgen05 kernel (k_gemm_tc.cu) is used instead; this kernel
// only serves BF16 shapes the tensor-core kernel does not take (tiny d).
//
// Replaces `linear` (proj/src/model.cpp:301-314) and the dX/dW loops of
// `backward` (model.cpp:652-817).
#include "internal.cuh"

namespace parl_gpu {

namespace {

constexpr int BM = 64, BN = 64, BK = 16, NT = 256;

template <class T>
__device__ __forceinline__ void load_tile(float (*S)[BM + 4], const T* __restrict__ X, long s_row, long s_k,
                                          int row0, int k0, int rows, int K) {
    const int tid = threadIdx.x;
#pragma unroll
    for (int i = 0; i < (BM * BK) / NT; ++i) {
        const int e = tid + i * NT;
        int r, k;
        if (s_k == 1) {  // K-major: consecutive threads walk k
            r = e / BK;
            k = e % BK;
        } else {  // MN-major: consecutive threads walk rows
            k = e / BM;
            r = e % BM;
        }
        const int gr = row0 + r, gk = k0 + k;
        float v = 0.f;
        if (gr < rows && gk < K) v = to_f<T>(X[(long)gr * s_row + (long)gk * s_k]);
        S[k][r] = v;
    }
}

template <class T>
__global__ void __launch_bounds__(NT) gemm_simt_kernel(GemmArgs g) {
    __shared__ float As[2][BK][BM + 4];
    __shared__ float Bs[2][BK][BN + 4];
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    const int tid = threadIdx.x, ty = tid / 16, tx = tid % 16;
    const T* A = static_cast<const T*>(g.A);
    const T* B = static_cast<const T*>(g.B);

    float acc[4][4] = {};
    int buf = 0;
    load_tile<T>(As[0], A, g.sam, g.sak, m0, 0, g.M, g.K);
    load_tile<T>(Bs[0], B, g.sbn, g.sbk, n0, 0, g.N, g.K);
    __syncthreads();
    for (int k0 = 0; k0 < g.K; k0 += BK) {
        if (k0 + BK < g.K) {
            load_tile<T>(As[buf ^ 1], A, g.sam, g.sak, m0, k0 + BK, g.M, g.K);
            load_tile<T>(Bs[buf ^ 1], B, g.sbn, g.sbk, n0, k0 + BK, g.N, g.K);
        }
#pragma unroll
        for (int k = 0; k < BK; ++k) {
            float a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[buf][k][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Bs[buf][k][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
        buf ^= 1;
    }

#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int m = m0 + ty * 4 + i;
        if (m >= g.M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int n = n0 + tx * 4 + j;
            if (n >= g.N) continue;
            float v = acc[i][j];
            switch (g.epi) {
                case EPI_F32:
                    if (g.bias) v += g.bias[n];
                    g.Cf[(long)m * g.ldc + n] = v;
                    break;
                case EPI_F32_ACC:
                    g.Cf[(long)m * g.ldc + n] += v;
                    break;
                case EPI_ACT:
                    if (g.bias) v += g.bias[n];
                    static_cast<T*>(g.Ca)[(long)m * g.ldca + n] = from_f<T>(v);
                    break;
                case EPI_RESID:
                    if (g.bias) v += g.bias[n];
                    g.Cf[(long)m * g.ldc + n] = g.resid[(long)m * g.ldc + n] + v;
                    break;
                case EPI_GELU: {
                    if (g.bias) v += g.bias[n];
                    const T u = from_f<T>(v);
                    static_cast<T*>(g.Ca)[(long)m * g.ldca + n] = u;
                    static_cast<T*>(g.Caux)[(long)m * g.ldca + n] = from_f<T>(gelu_f(to_f<T>(u)));
                    break;
                }
                case EPI_GELU_ACT: {
                    if (g.bias) v += g.bias[n];
                    static_cast<T*>(g.Ca)[(long)m * g.ldca + n] = from_f<T>(gelu_f(to_f<T>(from_f<T>(v))));
                    break;
                }
                case EPI_GELU_BWD: {
                    const float u = to_f<T>(static_cast<const T*>(g.aux_in)[(long)m * g.ldca + n]);
                    static_cast<T*>(g.Ca)[(long)m * g.ldca + n] = from_f<T>(v * gelu_grad_f(u));
                    break;
                }
                default:
                    break;
            }
        }
    }
}

}  // namespace

template <class T>
void gemm_simt(const GemmArgs& g, cudaStream_t st) {
    if (g.M <= 0 || g.N <= 0) return;
    dim3 grid(cdiv(g.N, BN), cdiv(g.M, BM));
    gemm_simt_kernel<T><<<grid, NT, 0, st>>>(g);
    PARL_LAUNCHED();
}

template void gemm_simt<float>(const GemmArgs&, cudaStream_t);
template void gemm_simt<bf16>(const GemmArgs&, cudaStream_t);

}  // namespace parl_gpu
