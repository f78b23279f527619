// Microbenchmark: the k_basis4 step structure (3 scalar chains per lane, ring
// of M registers, per-step coefficient row) in isolation, TI flavour
// (coefficients in registers).  Reports TFMA/s vs chains-per-lane layout.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 basis_ti.cu
#include <cstdio>
#include <utility>
#include <cuda_runtime.h>
constexpr int M = 22;

template <int C, int U, bool TV>
__device__ __forceinline__ void step(float (&R)[C][M], const float (&ati)[M], const float* rows,
                                     float ev) {
    float a[M];
#pragma unroll
    for (int i = 0; i < M; ++i) a[i] = TV ? rows[U * M + i] : ati[i];
    float c[C];
#pragma unroll
    for (int j = 0; j < C; ++j) c[j] = j == 0 ? ev : 0.f;
#pragma unroll
    for (int i = M; i >= 2; --i) {
        const int r = (U - i + 2 * M) % M;
#pragma unroll
        for (int j = 0; j < C; ++j) c[j] = fmaf(-a[i - 1], R[j][r], c[j]);
    }
#pragma unroll
    for (int j = 0; j < C; ++j) R[j][U % M] = fmaf(-a[0], R[j][(U - 1 + M) % M], c[j]);
}
template <int C, bool TV, int GS, int G, int... V>
__device__ __forceinline__ void group(std::integer_sequence<int, V...>, float (&R)[C][M],
                                      const float (&a)[M], const float* rows, const float* es) {
    ((G * GS + V < M ? step<C, (G * GS + V) % M, TV>(R, a, rows, es[(G * GS + V) % M]) : void()),
     ...);
}
template <int C, bool TV, int GS, int... G>
__device__ __forceinline__ void window(std::integer_sequence<int, G...>, float (&R)[C][M],
                                       const float (&a)[M], const float* rows, const float* es,
                                       int lim) {
    if constexpr (GS >= M) {
        (group<C, TV, GS, G>(std::make_integer_sequence<int, GS>{}, R, a, rows, es), ...);
    } else {
        ((G * GS < lim ? group<C, TV, GS, G>(std::make_integer_sequence<int, GS>{}, R, a, rows, es)
                       : void()),
         ...);
    }
}

template <int C, bool TV, int GS>
__global__ void __launch_bounds__(64, 1) kb(float* out, int nwin, int lim) {
    __shared__ float es[32];
    __shared__ __align__(16) float rows[M * M];
    if (threadIdx.x < 32) es[threadIdx.x] = 1e-3f * threadIdx.x;
    for (int i = threadIdx.x; i < M * M; i += 64) rows[i] = ((i % 5) - 2) * 1e-2f;
    __syncthreads();
    float a[M];
#pragma unroll
    for (int i = 0; i < M; ++i) a[i] = (i % 5 - 2) * 1e-2f + threadIdx.x * 1e-6f;
    float R[C][M];
#pragma unroll
    for (int j = 0; j < C; ++j)
#pragma unroll
        for (int p = 0; p < M; ++p) R[j][p] = (p == j) ? 1.f : 0.f;
    for (int k = 0; k < nwin; ++k)
        window<C, TV, GS>(std::make_integer_sequence<int, (M + GS - 1) / GS>{}, R, a, rows, es, lim);
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < C; ++j)
#pragma unroll
        for (int p = 0; p < M; ++p) s += R[j][p];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int C, bool TV, int GS>
void run(float* out, int wps) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int nwin = 200, blocks = 148 * wps / 2;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        kb<C, TV, GS><<<blocks, 64>>>(out, nwin, M);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double fma = (double)blocks * 64 * nwin * M * M * C;
        if (rep) printf("%s G=%d chains/lane %d warps/SM %2d: %.2f TFMA/s\n", TV ? "TV" : "TI", GS, C, wps, fma / (ms * 1e-3) / 1e12);
    }
}
int main() {
    float* out;
    cudaMalloc(&out, 148 * 64 * 64 * sizeof(float));
    for (int wps : {12}) {
        run<3, false, 22>(out, wps);
        run<3, false, 2>(out, wps);
        run<3, true, 1>(out, wps);
        run<3, true, 2>(out, wps);
        run<3, true, 3>(out, wps);
        run<3, true, 4>(out, wps);
        run<2, true, 2>(out, wps);
        run<4, true, 2>(out, wps);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
