// stepup.cu -- reflection -> direct-form rows (the step-up recursion) and its
// VJP, SURVEY.md §8(f) rank 2 (params.py:43-97).  Frame-rate work (F x M per
// sequence): one thread per row, float64 internally like the reference
// (params.py:64 casts to float64), with the reference's exact operation order
// (separate multiply and add, numpy's pairwise summation for the VJP's dot),
// so the fp64 results are bit-identical to tvlp's.
#include "common.cuh"

namespace tvlp {

constexpr int kStepMax = 30;  // largest order (the scan kernels' limit)

// numpy's pairwise sum for n <= 128 (loops_utils.h.src): plain loop below 8,
// else 8 interleaved partial sums combined as ((0+1)+(2+3))+((4+5)+(6+7)).
__device__ __forceinline__ double np_pairwise(const double* x, int n) {
    if (n < 8) {
        double r = 0.0;
        for (int i = 0; i < n; ++i) r = __dadd_rn(r, x[i]);
        return r;
    }
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = x[j];
    int i = 8;
    for (; i < n - (n % 8); i += 8)
        for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], x[i + j]);
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, x[i]);
    return res;
}

// a_m = [a_{m-1} + k_{m-1} * reverse(a_{m-1}), k_{m-1}]  (params.py:43-53)
// one thread per row, 32 per CTA: the rows spread over every SM (at 128 per
// CTA a decoder step's 6.4 k rows sat on 51 SMs, and the VJP's per-thread
// stage arrays -- 3.5 KB of local memory each -- thrashed their L1)
constexpr int kStepThreads = 32;

template <typename IO>
__global__ void __launch_bounds__(kStepThreads)
k_step_up(const IO* __restrict__ k, IO* __restrict__ a, int64_t rows, int M,
          int* __restrict__ bad) {
    grid_dep_wait();
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const IO* kr = k + r * M;
    double cur[kStepMax], nxt[kStepMax];
    bool ok = true;
    for (int i = 0; i < M; ++i) ok &= fabs((double)kr[i]) < 1.0;
    if (!ok && bad != nullptr) atomicOr(bad, 1);
    cur[0] = (double)kr[0];
    for (int m = 2; m <= M; ++m) {
        const double km = (double)kr[m - 1];
        for (int i = 0; i < m - 1; ++i) nxt[i] = __dadd_rn(cur[i], __dmul_rn(km, cur[m - 2 - i]));
        nxt[m - 1] = km;
        for (int i = 0; i < m; ++i) cur[i] = nxt[i];
    }
    for (int i = 0; i < M; ++i) a[r * M + i] = (IO)cur[i];
}

// params.py:74-84: g = grad_a; for m = M..2: grad_k[m-1] = g[m-1] +
// sum(g[:m-1] * reverse(stage_{m-1})); g = g[:m-1] + k[m-1] * reverse(g[:m-1]).
template <typename IO>
__global__ void __launch_bounds__(kStepThreads)
k_step_up_vjp(const IO* __restrict__ grad_a, const IO* __restrict__ k, IO* __restrict__ grad_k,
              int64_t rows, int M) {
    grid_dep_wait();
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const IO* kr = k + r * M;
    // stages[m-2] (length m-1) packed: offset (m-2)(m-1)/2
    double stages[kStepMax * (kStepMax - 1) / 2];
    double cur[kStepMax], nxt[kStepMax];
    cur[0] = (double)kr[0];
    for (int m = 2; m <= M; ++m) {
        double* st = stages + (m - 2) * (m - 1) / 2;
        for (int i = 0; i < m - 1; ++i) st[i] = cur[i];
        const double km = (double)kr[m - 1];
        for (int i = 0; i < m - 1; ++i) nxt[i] = __dadd_rn(cur[i], __dmul_rn(km, cur[m - 2 - i]));
        nxt[m - 1] = km;
        for (int i = 0; i < m; ++i) cur[i] = nxt[i];
    }
    double g[kStepMax], gk[kStepMax], prod[kStepMax];
    for (int i = 0; i < M; ++i) g[i] = (double)grad_a[r * M + i];
    for (int m = M; m >= 2; --m) {
        const double* prev = stages + (m - 2) * (m - 1) / 2;
        for (int i = 0; i < m - 1; ++i) prod[i] = __dmul_rn(g[i], prev[m - 2 - i]);
        gk[m - 1] = __dadd_rn(g[m - 1], np_pairwise(prod, m - 1));
        const double km = (double)kr[m - 1];
        for (int i = 0; i < m - 1; ++i) nxt[i] = __dadd_rn(g[i], __dmul_rn(km, g[m - 2 - i]));
        for (int i = 0; i < m - 1; ++i) g[i] = nxt[i];
    }
    gk[0] = g[0];
    for (int i = 0; i < M; ++i) grad_k[r * M + i] = (IO)gk[i];
}

// float32 rows (the decoder): one warp per row, lane i holds component i in
// float64 registers; the reversed-coefficient reads are warp shuffles, the
// VJP's stage vectors stay in registers (no 3.5 KB local array per row) and
// its dot products are warp sums (not numpy's pairwise order: the float64
// entry point keeps the bit-exact kernel above).
__global__ void __launch_bounds__(128)
k_step_up_vjp_warp(const float* __restrict__ grad_a, const float* __restrict__ k,
                   float* __restrict__ grad_k, int64_t rows, int M) {
    grid_dep_wait();
    const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (r >= rows) return;
    const float* kr = k + r * M;
    const double kl = lane < M ? (double)kr[lane] : 0.0;
    // forward: stage m-1 (length m-1) kept per lane: st[m] = component `lane` of
    // the stage entering step m (valid for lane < m - 1)
    double st[kStepMax];
    const double k0 = __shfl_sync(0xffffffffu, kl, 0);
    double cur = lane == 0 ? k0 : 0.0;
#pragma unroll
    for (int m = 2; m <= kStepMax; ++m) {
        if (m > M) break;
        st[m - 2] = cur;
        const double km = __shfl_sync(0xffffffffu, kl, m - 1);
        const int src = m - 2 - lane;
        const double rev = __shfl_sync(0xffffffffu, cur, src >= 0 ? src : 0);
        double nxt = cur;
        if (lane < m - 1) nxt = __dadd_rn(cur, __dmul_rn(km, rev));
        else if (lane == m - 1) nxt = km;
        cur = nxt;
    }
    double g = lane < M ? (double)grad_a[r * M + lane] : 0.0;
    double gk = 0.0;
#pragma unroll
    for (int m = kStepMax; m >= 2; --m) {
        if (m > M) continue;
        // gk[m-1] = g[m-1] + sum_{i < m-1} g[i] * stage[m-2-i]
        const int src = m - 2 - lane;
        const double prev = __shfl_sync(0xffffffffu, st[m - 2], src >= 0 ? src : 0);
        double prod = lane < m - 1 ? g * prev : 0.0;
#pragma unroll
        for (int o = 16; o; o >>= 1) prod += __shfl_xor_sync(0xffffffffu, prod, o);
        const double gm1 = __shfl_sync(0xffffffffu, g, m - 1);
        if (lane == m - 1) gk = gm1 + prod;
        // g[i] <- g[i] + k[m-1] g[m-2-i] for i < m-1
        const double km = __shfl_sync(0xffffffffu, kl, m - 1);
        const double rev = __shfl_sync(0xffffffffu, g, src >= 0 ? src : 0);
        if (lane < m - 1) g = __dadd_rn(g, __dmul_rn(km, rev));
    }
    if (lane == 0) gk = g;
    if (lane < M) grad_k[r * M + lane] = (float)gk;
}

template <typename IO>
cudaError_t launch_step_up(const IO* k, IO* a, int64_t rows, int M, int* bad, cudaStream_t st) {
    if (M < 1 || M > kStepMax) return cudaErrorInvalidValue;
    launch_pdl(k_step_up<IO>, (unsigned)((rows + kStepThreads - 1) / kStepThreads), kStepThreads,
               0, st, k, a, rows, M, bad);
    return cudaGetLastError();
}
template <typename IO>
cudaError_t launch_step_up_vjp(const IO* ga, const IO* k, IO* gk, int64_t rows, int M,
                               cudaStream_t st) {
    if (M < 1 || M > kStepMax) return cudaErrorInvalidValue;
    if constexpr (std::is_same<IO, float>::value) {
        launch_pdl(k_step_up_vjp_warp, (unsigned)((rows * 32 + 127) / 128), 128, 0, st, ga, k, gk,
                   rows, M);
        return cudaGetLastError();
    }
    launch_pdl(k_step_up_vjp<IO>, (unsigned)((rows + kStepThreads - 1) / kStepThreads),
               kStepThreads, 0, st, ga, k, gk, rows, M);
    return cudaGetLastError();
}
template cudaError_t launch_step_up<float>(const float*, float*, int64_t, int, int*, cudaStream_t);
template cudaError_t launch_step_up<double>(const double*, double*, int64_t, int, int*,
                                            cudaStream_t);
template cudaError_t launch_step_up_vjp<float>(const float*, const float*, float*, int64_t, int,
                                               cudaStream_t);
template cudaError_t launch_step_up_vjp<double>(const double*, const double*, double*, int64_t,
                                                int, cudaStream_t);

}  // namespace tvlp
