// Microbenchmark: cycles per hop of the chained kernels' unit carry
// (x <- Phi_l x + z_l over tapes staged in shared memory, chain.cuh
// unit_carry_fwd) against variants of the state broadcast, one warp per SM.
//   MODE 0  as chain.cuh: state through shared memory (STS, warp sync, 6 x LDS.128),
//           the global record store per hop, next row prefetched
//   MODE 1  MODE 0 without the global store
//   MODE 2  state broadcast by 22 warp shuffles (no shared memory round trip)
//   MODE 3  MODE 2 with the hop loop unrolled by 2 (no register copies of the row)
//   MODE 4  no broadcast: the dot over the lane's own x (the FMA chain alone)
//   MODE 5  the 22 shuffles alone (summed, no dot)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 carry_hop.cu -o carry_hop
#include <cstdio>
#include <cuda_runtime.h>

constexpr int M = 22, MP4 = 24, L = 32;

__device__ __forceinline__ float dot(const float (&w)[MP4], const float (&x)[MP4], float z) {
    float q0 = z, q1 = 0.f, q2 = 0.f, q3 = 0.f;
#pragma unroll
    for (int c = 0; c < M; ++c) {
        switch (c & 3) {
            case 0: q0 = fmaf(w[c], x[c], q0); break;
            case 1: q1 = fmaf(w[c], x[c], q1); break;
            case 2: q2 = fmaf(w[c], x[c], q2); break;
            default: q3 = fmaf(w[c], x[c], q3); break;
        }
    }
    return (q0 + q1) + (q2 + q3);
}

template <int MODE>
__global__ void khop(float* gx, long long* cyc, int reps) {
    extern __shared__ __align__(16) float dyn[];
    float* tz = dyn;                                  // [L][M+1][MP4]
    float* xb = tz + L * (M + 1) * MP4;               // [64]
    float* xs = xb + 64;                              // [(L+1)][MP4]
    const int lane = threadIdx.x;
    for (int i = lane; i < L * (M + 1) * MP4; i += 32) tz[i] = 0.01f * ((i * 13) % 7 - 3);
    __syncwarp();
    const int r = lane < M ? lane : 0;
    float x = lane < M ? 1.f : 0.f;
    float* xg = gx + blockIdx.x * (L * MP4);
    long long t0 = clock64();
    for (int rep = 0; rep < reps; ++rep) {
        float w[MP4], wn[MP4];
#pragma unroll
        for (int c = 0; c < MP4; ++c) w[c] = tz[(1 + r) * MP4 + c];
        float zr = tz[r];
        if constexpr (MODE == 4 || MODE == 5) {
            for (int l = 0; l < L; ++l) {
                float xv[MP4];
                if constexpr (MODE == 4) {
#pragma unroll
                    for (int c = 0; c < MP4; ++c) xv[c] = x;
                    x = dot(w, xv, zr);
                } else {
                    float acc = zr;
#pragma unroll
                    for (int c = 0; c < M; ++c) acc += __shfl_sync(0xffffffffu, x, c);
                    x = acc * 0.01f;
                }
            }
        } else if constexpr (MODE <= 2) {
            for (int l = 0; l < L; ++l) {
                const float* tn = tz + (l + 1 < L ? l + 1 : l) * (M + 1) * MP4;
#pragma unroll
                for (int c = 0; c < MP4; ++c) wn[c] = tn[(1 + r) * MP4 + c];
                const float zn = tn[r];
                float xv[MP4];
                if constexpr (MODE <= 1) {
                    if (lane < M) {
                        xs[l * MP4 + lane] = x;
                        if (MODE == 0) xg[l * MP4 + lane] = x;
                    }
                    float* b = xb + (l & 1) * 32;
                    b[lane] = lane < M ? x : 0.f;
                    __syncwarp();
#pragma unroll
                    for (int c = 0; c < MP4; ++c) xv[c] = b[c];
                } else {
                    if (lane < M) xs[l * MP4 + lane] = x;
#pragma unroll
                    for (int c = 0; c < MP4; ++c) xv[c] = __shfl_sync(0xffffffffu, x, c < M ? c : 0);
                }
                x = dot(w, xv, zr);
#pragma unroll
                for (int c = 0; c < MP4; ++c) w[c] = wn[c];
                zr = zn;
            }
        } else {
            for (int l = 0; l < L; l += 2) {
                const float* t1 = tz + (l + 1) * (M + 1) * MP4;
#pragma unroll
                for (int c = 0; c < MP4; ++c) wn[c] = t1[(1 + r) * MP4 + c];
                const float z1 = t1[r];
                float xv[MP4];
                if (lane < M) xs[l * MP4 + lane] = x;
#pragma unroll
                for (int c = 0; c < MP4; ++c) xv[c] = __shfl_sync(0xffffffffu, x, c < M ? c : 0);
                x = dot(w, xv, zr);
                const float* t2 = tz + (l + 2 < L ? l + 2 : l) * (M + 1) * MP4;
#pragma unroll
                for (int c = 0; c < MP4; ++c) w[c] = t2[(1 + r) * MP4 + c];
                zr = t2[r];
                if (lane < M) xs[(l + 1) * MP4 + lane] = x;
#pragma unroll
                for (int c = 0; c < MP4; ++c) xv[c] = __shfl_sync(0xffffffffu, x, c < M ? c : 0);
                x = dot(wn, xv, z1);
            }
        }
    }
    long long t1 = clock64();
    if (lane < M) gx[blockIdx.x * (L * MP4) + lane] += x + xs[lane];
    if (lane == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run() {
    float* gx;
    long long* cyc;
    cudaMalloc(&gx, 148 * L * MP4 * 4);
    cudaMalloc(&cyc, 148 * 8);
    const int sm = (L * (M + 1) * MP4 + 64 + (L + 1) * MP4) * 4;
    cudaFuncSetAttribute(khop<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    khop<MODE><<<148, 32, sm>>>(gx, cyc, 100);
    khop<MODE><<<148, 32, sm>>>(gx, cyc, 100);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (long long v : h) mx = v > mx ? v : mx;
    printf("MODE %d: %.1f cycles/hop (%s)\n", MODE, (double)mx / (100.0 * L), cudaGetErrorString(e));
}

int main() {
    run<0>();
    run<1>();
    run<2>();
    run<3>();
    run<4>();
    run<5>();
    return 0;
}
