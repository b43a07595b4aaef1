// Microbenchmark: SM throughput of ex2.approx.f32 vs ex2.approx.f16x2 vs ex2.approx.ftz.bf16x2
// and of a degree-3 FMA-pipe exp2 (per-SM results per clock).  nvcc -arch=sm_100a mufu_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_fp16.h>

template <int MODE>
__global__ void k(float* out, int iters, float seed) {
    float a[8];
    uint32_t h[8];
    for (int i = 0; i < 8; ++i) a[i] = -(seed + 0.01f * i + 0.001f * threadIdx.x);
    for (int i = 0; i < 8; ++i) {
        __half2 t = __floats2half2_rn(a[i], a[i] * 0.5f);
        h[i] = *reinterpret_cast<uint32_t*>(&t);
    }
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0) {
                asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
            } else if (MODE == 1) {
                asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h[i]));
            } else if (MODE == 2) {
                asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h[i]));
            } else if (MODE == 4) {  // fp32 pair -> bf16x2 (the P pack of the softmax)
                asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(h[i]) : "f"(a[i]), "f"(a[(i + 1) & 7]));
                a[i] = __uint_as_float(h[i]) * 0.5f;
            } else if (MODE == 5) {  // 3-input max
                a[i] = fmaxf(fmaxf(a[i], a[(i + 3) & 7]), a[(i + 5) & 7]);
            } else {  // FMA-pipe exp2: Cody-Waite split + degree-3 polynomial
                float x = fmaxf(a[i], -127.f);
                float fi = floorf(x);
                float f = x - fi;
                float p = fmaf(fmaf(fmaf(0.0555041f, f, 0.2402265f), f, 0.6931472f), f, 1.0f);
                a[i] = __int_as_float(__float_as_int(p) + ((int)fi << 23)) - 1.0f;
            }
        }
    }
    long long t1 = clock64();
    float s = 0;
    for (int i = 0; i < 8; ++i) s += a[i] + __uint_as_float(h[i]);
    if (threadIdx.x == 0 && blockIdx.x == 0) out[1] = (float)(t1 - t0);
    out[2 + blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    float* d;
    cudaMalloc(&d, (2 + 148 * 1024) * sizeof(float));
    const int iters = 4096;
    const char* names[] = {"ex2.f32", "ex2.f16x2", "ex2.bf16x2", "fma-poly exp2", "cvt bf16x2", "fmax3(+fmul)"};
    for (int mode = 0; mode < 6; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            if (mode == 0) k<0><<<148 * 2, 512>>>(d, iters, 0.5f);
            if (mode == 1) k<1><<<148 * 2, 512>>>(d, iters, 0.5f);
            if (mode == 2) k<2><<<148 * 2, 512>>>(d, iters, 0.5f);
            if (mode == 3) k<3><<<148 * 2, 512>>>(d, iters, 0.5f);
            if (mode == 4) k<4><<<148 * 2, 512>>>(d, iters, 0.5f);
            if (mode == 5) k<5><<<148 * 2, 512>>>(d, iters, 0.5f);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            float clk;
            cudaMemcpy(&clk, d + 1, 4, cudaMemcpyDeviceToHost);
            const double ops = 148.0 * 2 * 512 * iters * 8 * (mode == 1 || mode == 2 ? 2 : 1);
            if (rep == 1 && mode >= 4) printf("(ops = instructions)\n");
            if (rep == 1)
                printf("%-14s  %.3f ms  %.1f exp/clk/SM (clock64 of block 0: %.0f clk, %.1f exp/clk/SM)\n", names[mode],
                       ms, ops / 148 / (ms * 1e-3 * 1.9e9), clk, 2 * 512.0 * iters * 8 * (mode == 1 || mode == 2 ? 2 : 1) / clk);
        }
    }
    return 0;
}
