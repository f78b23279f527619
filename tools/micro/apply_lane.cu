// Microbenchmark: cycles per sample of the lane-per-sub-chunk recursion
// (unit_fwd_pass's inner loop) with rows already in shared memory, for
//   MODE 0  the product formulation: row t loaded one step ahead, 4 partial
//           sums over lags M..2 (oldest first), then the lag-1 FMA
//   MODE 1  two-step lookahead: Q(t+2) = e - sum_{i>=3} a s is accumulated
//           two samples early, P(t+1) = Q(t+1) - a2 s(t-1) one sample early,
//           so a sample's critical path is the single lag-1 FMA
//   MODE 2  MODE 0 plus the per-window bookkeeping of the product kernel
//           (output box store, async-proxy fence, warp syncs)
//   MODE 3  MODE 1 plus the same bookkeeping
// at 1, 2, 4 and 8 resident warps per SM (one warp = one independent lane set).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 apply_lane.cu -o apply_lane
#include <cstdio>
#include <cuda_runtime.h>

constexpr int M = 22;
constexpr int W = 8;                        // rows per window
constexpr int AROW = 180;                   // floats per lane row block (odd 16-B granules: 45)
constexpr int XROW = 12;
constexpr int MR = 24;                      // ring of 3 windows (no rotation)

template <int MODE>
__global__ void kapply(float* out, long long* cyc, int nwin) {
    extern __shared__ __align__(16) float sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float* A = sm + warp * (32 * AROW + 32 * XROW + 32 * W);
    float* E = A + 32 * AROW;
    float* O = E + 32 * XROW;
    for (int i = lane; i < 32 * AROW; i += 32) A[i] = 0.02f * (float)((i * 7) % 13 - 6) / 6.f;
    for (int i = lane; i < 32 * XROW; i += 32) E[i] = 0.1f * (float)(i % 5);
    __syncwarp();
    const float* Ar = A + lane * AROW;
    const float* er = E + lane * XROW;
    float R[MR];
#pragma unroll
    for (int i = 0; i < MR; ++i) R[i] = 0.f;
    long long t0 = clock64();
    if constexpr (MODE == 0 || MODE == 2) {
        float an[M];
#pragma unroll
        for (int i = 0; i < M; ++i) an[i] = Ar[i];
        for (int k = 0; k < nwin; k += 3) {
#pragma unroll
          for (int w3 = 0; w3 < 3; ++w3) {
            float ev[W];
#pragma unroll
            for (int u = 0; u < W; ++u) ev[u] = er[u];
#pragma unroll
            for (int uu = 0; uu < W; ++uu) {
                const int u = w3 * W + uu;
                float a[M];
#pragma unroll
                for (int i = 0; i < M; ++i) a[i] = an[i];
                const int un = (uu + 1) % W;
#pragma unroll
                for (int i = 0; i < M; ++i) an[i] = Ar[un * M + i];
                float p0 = 0.f, p1 = 0.f, p2 = 0.f, p3 = 0.f;
#pragma unroll
                for (int i = M; i >= 2; --i) {
                    const float x = R[(u - i + 2 * MR) % MR];
                    switch (i & 3) {
                        case 0: p0 = fmaf(a[i - 1], x, p0); break;
                        case 1: p1 = fmaf(a[i - 1], x, p1); break;
                        case 2: p2 = fmaf(a[i - 1], x, p2); break;
                        default: p3 = fmaf(a[i - 1], x, p3); break;
                    }
                }
                const float v = fmaf(-a[0], R[(u - 1 + 2 * MR) % MR], ev[uu] - ((p0 + p1) + (p2 + p3)));
                R[u % MR] = v;
                if (MODE == 2) O[lane * W + uu] = v;
            }
            if (MODE == 2) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                __syncwarp();
            }
          }
        }
    } else {
        // lookahead: P1 = P(t), Q2 = Q(t+1) (excl. lag 2 term), rows t+1, t+2 held partly
        // R ring: R[(u - i) mod M] = s(t - i) at step u (t = window position)
        float P = 0.f, Qn = 0.f, a2n = 0.f, a1n = 0.f, a1 = 0.f;
        for (int k = 0; k < nwin; k += 3) {
#pragma unroll
          for (int w3 = 0; w3 < 3; ++w3) {
            float ev[W + 2];
#pragma unroll
            for (int u = 0; u < W + 2; ++u) ev[u] = er[u];
#pragma unroll
            for (int uu = 0; uu < W; ++uu) {
                const int u = w3 * W + uu;
                // s(t) = P(t) - a_{t,1} s(t-1)
                const float s1 = R[(u - 1 + 2 * MR) % MR];
                const float v = fmaf(-a1, s1, P);
                // P(t+1) = Q(t+1) - a_{t+1,2} s(t-1)
                const float Pn = fmaf(-a2n, s1, Qn);
                // Q(t+2) = e(t+2) - sum_{i=3..M} a_{t+2,i} s(t+2-i), lag i -> s(t+2-i)
                float r[M];
                const int u2 = (uu + 2) % W;
#pragma unroll
                for (int i = 0; i < M; ++i) r[i] = Ar[u2 * M + i];
                float q0 = ev[uu + 2], q1 = 0.f, q2 = 0.f, q3 = 0.f;
#pragma unroll
                for (int i = M; i >= 3; --i) {
                    const float x = R[(u + 2 - i + 2 * MR) % MR];  // s(t+2-i), i >= 3 -> <= t-1
                    switch (i & 3) {
                        case 0: q0 = fmaf(-r[i - 1], x, q0); break;
                        case 1: q1 = fmaf(-r[i - 1], x, q1); break;
                        case 2: q2 = fmaf(-r[i - 1], x, q2); break;
                        default: q3 = fmaf(-r[i - 1], x, q3); break;
                    }
                }
                R[u % MR] = v;
                if (MODE == 3) O[lane * W + uu] = v;
                P = Pn;
                a1 = a1n;
                a1n = r[0];
                a2n = r[1];
                Qn = (q0 + q1) + (q2 + q3);
            }
            if (MODE == 3) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                __syncwarp();
                __syncwarp();
            }
          }
        }
    }
    long long t1 = clock64();
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < MR; ++i) acc += R[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (lane == 0) cyc[blockIdx.x * 32 + warp] = t1 - t0;
}

template <int MODE>
void run(int wpsm, int nsm) {
    const int nwin = 201;
    const int threads = 32 * wpsm;
    const size_t smem = (size_t)wpsm * (32 * AROW + 32 * XROW + 32 * W) * 4;
    cudaFuncSetAttribute(kapply<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    float* out;
    long long* cyc;
    cudaMalloc(&out, nsm * threads * 4);
    cudaMalloc(&cyc, nsm * 32 * 8);
    kapply<MODE><<<nsm, threads, smem>>>(out, cyc, nwin);
    kapply<MODE><<<nsm, threads, smem>>>(out, cyc, nwin);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[32 * 148];
    cudaMemcpy(h, cyc, nsm * 32 * 8, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int b = 0; b < nsm; ++b)
        for (int w = 0; w < wpsm; ++w) mx = mx > h[b * 32 + w] ? mx : (double)h[b * 32 + w];
    printf("MODE %d warps/SM %d: %.1f cycles/sample (%s)\n", MODE, wpsm, mx / (nwin * W),
           cudaGetErrorString(e));
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    for (int w : {1, 2, 4, 8}) {
        run<0>(w, 148);
        run<1>(w, 148);
        run<2>(w, 148);
        run<3>(w, 148);
    }
    return 0;
}
