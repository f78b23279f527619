// Microbenchmark: FFMA2 throughput when all three operands are registers
// (Ra.F32 broadcast scalar, Rb/Rc float2 pairs) vs constant-bank scalar.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(float* out, float a0, int iters) {
    float2 x[8], c[8];
    float s[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        x[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
        c[i] = make_float2(1e-3f * i * threadIdx.x, 2e-3f * i + threadIdx.y);
        s[i] = a0 + 1e-4f * i * threadIdx.x;  // distinct registers
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0) x[i] = __ffma2_rn(make_float2(s[i], s[i]), x[i], c[i]);         // R, R2, R2
            else if (MODE == 1) x[i] = __ffma2_rn(make_float2(a0, a0), x[i], c[i]);        // c[], R2, R2
            else if (MODE == 2) x[i] = __ffma2_rn(make_float2(s[i], s[i]), x[i], x[(i + 1) & 7]);
            else if (MODE == 3) { x[i].x = fmaf(s[i], x[i].x, c[i].x); x[i].y = fmaf(s[i], x[i].y, c[i].y); }  // 2 FFMA
            else if (MODE == 4) { x[i].x = fmaf(s[i], c[i].x, x[i].x); x[i].y = fmaf(s[(i + 1) & 7], c[i].y, x[i].y); }  // accumulate form
            else { x[i].x = fmaf(-s[i], c[i].x, x[i].x); x[i].y = fmaf(-s[(i + 1) & 7], c[i].y, x[i].y); }  // negated operand
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) s[i] = __int_as_float(__float_as_int(s[i]) ^ (it & 1));  // keep s live in regs
    }
    float r = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) r += x[i].x + x[i].y + s[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
int main() {
    float* out;
    cudaMalloc(&out, 148 * 64 * 1024 * sizeof(float));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    for (int wps : {64, 16, 12, 8})
    for (int mode = 3; mode < 6; ++mode)
        for (int rep = 0; rep < 2; ++rep) {
            const int blocks = 148 * wps / 2, threads = 64;
            cudaEventRecord(e0);
            if (mode == 0) k<0><<<blocks, threads>>>(out, 0.999f, iters);
            if (mode == 1) k<1><<<blocks, threads>>>(out, 0.999f, iters);
            if (mode == 2) k<2><<<blocks, threads>>>(out, 0.999f, iters);
            if (mode == 3) k<3><<<blocks, threads>>>(out, 0.999f, iters);
            if (mode == 4) k<4><<<blocks, threads>>>(out, 0.999f, iters);
            if (mode == 5) k<5><<<blocks, threads>>>(out, 0.999f, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double fma = 16.0 * iters * blocks * threads;
            if (rep) printf("warps/SM %d mode %d: %.2f TFMA/s\n", wps, mode, fma / (ms * 1e-3) / 1e12);
        }
    return 0;
}
