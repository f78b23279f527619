// Microbenchmark: FFMA vs FFMA2 (broadcast scalar) throughput on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(float* out, float a, int iters) {
    float2 x[8];
    float y[16];
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
#pragma unroll
    for (int i = 0; i < 16; ++i) y[i] = threadIdx.x * 1e-3f + i;
    float b = a * 0.999f;
    for (int it = 0; it < iters; ++it) {
        if (MODE == 0) {
#pragma unroll
            for (int i = 0; i < 16; ++i) y[i] = fmaf(a, y[i], b);
        } else if (MODE == 1) {
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = __ffma2_rn(make_float2(a, a), x[i], make_float2(b, b));
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = __ffma2_rn(make_float2(a, a), x[i], x[(i + 1) & 7]);
        }
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += x[i].x + x[i].y;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += y[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
    float* out;
    cudaMalloc(&out, 148 * 64 * 1024 * sizeof(float));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    for (int mode = 0; mode < 3; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (mode == 0) k<0><<<148 * 8, 256>>>(out, 1.0001f, iters);
            if (mode == 1) k<1><<<148 * 8, 256>>>(out, 1.0001f, iters);
            if (mode == 2) k<2><<<148 * 8, 256>>>(out, 1.0001f, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            double fmas = 148.0 * 8 * 256 * iters * 16;  // 16 FMAs per thread-iteration in all modes
            if (rep) printf("mode %d: %.3f ms  %.1f TFMA/s  (%.1f TFLOP/s)\n", mode, ms, fmas / ms / 1e9, 2 * fmas / ms / 1e9);
        }
    }
    return 0;
}
