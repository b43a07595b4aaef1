// Microbenchmark: per-SM throughput of single-CTA tcgen05.mma (kind::f16, bf16 in, fp32 TMEM
// accumulate) in the shapes the attention kernels issue: SS (both operands from shared memory)
// and TS (A from TMEM), M = 128, N = 64 / 128 / 256, K = 16 per instruction, 128B-swizzled
// K-major operands as the attention tiles are laid out.  One CTA per SM, one issuing thread,
// back-to-back MMAs on one accumulator; clock64 around ITERS x 4 MMAs + commit + wait.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2511_18871_b200/csrc mma_bench.cu
#include <cstdint>
#include <cstdio>

#include "tc_util.cuh"

using namespace parl_gpu;

template <int N, bool TS, int BMN = 0>
__global__ void __launch_bounds__(128, 1) k(unsigned long long* out, int iters) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* A = smem;                 // 128 x 64 bf16, SW128 K-major: 16 KB
    uint8_t* B = smem + 16384;         // N x 64 bf16: up to 32 KB
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase_s;
    for (int i = threadIdx.x; i < (16384 + N * 128) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
    if (threadIdx.x == 0) {
        tc::mbar_init(&bar, 1);
        tc::fence_barrier_init();
    }
    if (threadIdx.x < 32) tc::tmem_alloc<512>(&tbase_s);
    tc::fence_async_smem();
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tb = tbase_s;
    if (threadIdx.x == 0) {
        constexpr uint32_t id = tc::idesc_bf16(128, N, 0, BMN);
        const uint32_t a0 = tc::smem_u32(A), b0 = tc::smem_u32(B);
        const unsigned long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {  // K = 64: four K = 16 steps inside the 128-byte swizzle atom
                // B MN-major (N contiguous): K = 16 rows of 128 B per step, as the backward's dV / dK B operands
                const uint64_t bd = BMN ? tc::sdesc(b0 + ks * 2048, 128 * 128, 1024) : tc::sdesc(b0 + ks * 32, 16, 1024);
                if (TS) tc::mma_bf16_ts(tb, tb + 256 + ks * 8, bd, id, 1);
                else tc::mma_bf16(tb, tc::sdesc(a0 + ks * 32, 16, 1024), bd, id, 1);
            }
        }
        tc::mma_commit(&bar);
        tc::mbar_wait(&bar, 0);
        const unsigned long long t1 = clock64();
        if (blockIdx.x == 0) out[0] = t1 - t0;
    }
    tc::tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        tc::tc_fence_after();
        tc::tmem_dealloc<512>(tb);
    }
}

template <int N, bool TS, int BMN = 0>
void run(const char* name, unsigned long long* d, int sms) {
    const int iters = 4096, smem = 16384 + 32768 + 1024;
    cudaFuncSetAttribute(k<N, TS, BMN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k<N, TS, BMN><<<sms, 128, smem>>>(d, 16);  // warm-up
    k<N, TS, BMN><<<sms, 128, smem>>>(d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long clk = 0;
    cudaMemcpy(&clk, d, 8, cudaMemcpyDeviceToHost);
    const double flop = 2.0 * 128 * N * 64 * iters;  // per CTA (= per SM)
    printf("%-28s %s  %8.1f flop/clk/SM  (%.1f clk per 128x%dx16 MMA)\n", name, cudaGetErrorString(e), flop / clk,
           (double)clk / (4.0 * iters), N);
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 8);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<64, false>("SS M=128 N=64", d, sms);
    run<128, false>("SS M=128 N=128", d, sms);
    run<256, false>("SS M=128 N=256", d, sms);
    run<64, true>("TS M=128 N=64", d, sms);
    run<128, true>("TS M=128 N=128", d, sms);
    run<256, true>("TS M=128 N=256", d, sms);
    run<64, true, 1>("TS M=128 N=64 B MN-major", d, sms);
    run<128, true, 1>("TS M=128 N=128 B MN-major", d, sms);
    run<64, false, 1>("SS M=128 N=64 B MN-major", d, sms);
    return 0;
}
