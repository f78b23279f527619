// Microbenchmark: cycles per warp-step of the packed-chain basis step
// (k_basis2's inner loop) vs warps per SM, for the step-structure variants.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2406_05128_b200/csrc basis_step.cu
#include <cstdio>
#include "lp_scan.cuh"
using namespace tvlp;
constexpr int M = 22;

template <int MODE>
__global__ void __launch_bounds__(64, 10) kb(float* out, int nwin, int lim) {
    __shared__ __align__(16) float rows[M * M];
    for (int i = threadIdx.x; i < M * M; i += blockDim.x) rows[i] = 0.01f * ((i % 7) - 3);
    __syncthreads();
    const int q = threadIdx.x & 15;
    float2 R[M];
#pragma unroll
    for (int p = 0; p < M; ++p) R[p] = make_float2(p == q ? 1.f : 0.f, p == q + 1 ? 1.f : 0.f);
    float ati[M];
#pragma unroll
    for (int i = 0; i < M; ++i) ati[i] = 0.f;
    const bool zsx = q == 11, zsy = false;
    float ec0 = 0.5f + q, ec1 = 0.25f * q;
    for (int k = 0; k < nwin; ++k) {
        if constexpr (MODE == 2) {
            basis3_full<M, false>(std::make_integer_sequence<int, (M + kBasisGroup - 1) / kBasisGroup>{},
                                  R, rows, rows + 7, ati, zsx, zsy, lim);
        } else if constexpr (MODE == 3) {
            // dependent FFMA2 chain (latency probe)
#pragma unroll
            for (int i = 0; i < M; ++i) R[0] = __ffma2_rn(make_float2(rows[0], rows[0]), R[0], R[1]);
        } else if constexpr (MODE == 0) {
            basis2_full<M, false>(std::make_integer_sequence<int, M>{}, R, rows, ati, ec0, ec1, zsx,
                                  zsy, lim);
        } else {
            basis2_partial<M, false>(std::make_integer_sequence<int, M>{}, R, rows, ati, ec0, ec1,
                                     zsx, zsy, lim);
        }
        ec0 += 1.f;
    }
    float s = 0.f;
#pragma unroll
    for (int p = 0; p < M; ++p) s += R[p].x + R[p].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    float* out;
    cudaMalloc(&out, 148 * 64 * 1024 * sizeof(float));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int nwin = 400;
    for (int mode = 0; mode < 4; ++mode) {
        for (int wps : {2, 4, 8, 12, 16, 20, 24}) {
            const int blocks = 148 * wps / 2;
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(e0);
                if (mode == 0) kb<0><<<blocks, 64>>>(out, nwin, M);
                else if (mode == 1) kb<1><<<blocks, 64>>>(out, nwin, 0);
                else if (mode == 2) kb<2><<<blocks, 64>>>(out, nwin, M);
                else kb<3><<<blocks, 64>>>(out, nwin, M);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (rep == 1) {
                    const double steps_per_smsp = (double)wps / 4 * nwin * M;
                    printf("mode %d warps/SM %2d: %.3f ms, %.1f cycles per warp-step per SMSP (at %d MHz)\n",
                           mode, wps, ms, ms * 1e-3 * clk * 1e3 / steps_per_smsp, clk / 1000);
                }
            }
        }
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
