// framewise.cu -- frame-wise time-invariant LP with overlap-add (GOLF-ff).
//
// Reference: pkg/src/tvlp/params.py:152-217 (FramePlan), 220-239
// (_framewise_forward), 259-273 (_framewise_vjp), lpc.py:50-61/176-195.
//
// Every frame f in [-n_lead, F) is an independent zero-state TI recursion of
// `size` samples over window[k] * e[f*hop + k] with coefficient row
// frames[max(f,0)].  One lane per frame (frames of a sequence are contiguous
// lanes), all lanes step through k together: the window value is a broadcast
// and the per-frame outputs seg[b, k, fi] are written as coalesced 128-B rows.
// Overlap-add and the frame-row reduction are deterministic gathers in frame
// order (the reference's accumulation order).
#include "common.cuh"
#include "framewise_launch.cuh"

#ifndef TVLP_FW_PREFETCH
#define TVLP_FW_PREFETCH 16
#endif

namespace tvlp {

template <int M>
struct FwGeo {
    static constexpr int L = clcm(M, 4);  // unrolled body; ring positions static
    static constexpr int RS = (M + TVLP_FW_PREFETCH + 3) / 4 * 4;  // backward ring: M live + prefetch slots
};

// One warp = 32 consecutive frames of one sequence (grid: B x ceil(nfr/32),
// so every SM gets work).  The excitation span those frames read,
// [f0*hop, (f0+31)*hop + size), and the window are staged in shared memory
// once (coalesced) when they fit; the per-step reads are then shared-memory
// hits instead of 32 scattered global loads.
template <typename IO>
struct FwStage {
    static __host__ __device__ int64_t span(int size, int hop) { return 31LL * hop + size; }
    static __host__ __device__ size_t bytes(int size, int hop) {
        return (size_t)(span(size, hop) + size) * sizeof(IO);
    }
};
constexpr size_t kFwStageMax = 200 * 1024;

// dst[i] = src[t0 + i] (/ div), zero outside [0, n_src); one warp, 16 loads in
// flight per lane so the copy is bandwidth-, not latency-bound
template <typename IO, bool DIV>
__device__ __forceinline__ void stage_span(IO* __restrict__ dst, const IO* __restrict__ src,
                                           int64_t t0, int64_t n, int64_t n_src, IO div) {
    constexpr int U = 64;  // loads in flight per lane (staging is latency-bound)
    const int lane = threadIdx.x & 31;
    for (int64_t i0 = lane; i0 < n; i0 += 32 * U) {
        IO v[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const int64_t i = i0 + 32 * j, t = t0 + i;
            v[j] = (i < n && t >= 0 && t < n_src) ? src[t] : (IO)0;
        }
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const int64_t i = i0 + 32 * j;
            if (i < n) dst[i] = DIV ? v[j] / div : v[j];
        }
    }
}

template <typename IO, int M, bool STAGED>
__global__ void __launch_bounds__(32)
k_fw_forward(const IO* __restrict__ e, const IO* __restrict__ frames, const IO* __restrict__ win,
             IO* __restrict__ seg, int64_t B, int64_t T, int F, int nfr, int size, int hop,
             int n_lead) {
    grid_dep_wait();
    constexpr int L = FwGeo<M>::L;
    extern __shared__ __align__(16) unsigned char fw_smem[];
    const int lane = threadIdx.x;
    const int64_t b = blockIdx.y;
    const int fi0 = blockIdx.x * 32;
    const int fi = fi0 + lane;
    const bool active = fi < nfr;
    const int f = fi - n_lead;
    const int row = f > 0 ? f : 0;
    const int64_t start = (int64_t)f * hop;
    const int64_t span0 = (int64_t)(fi0 - n_lead) * hop;  // time of the staged span's first sample
    const IO* eb = e + b * T;
    IO* es = reinterpret_cast<IO*>(fw_smem);
    IO* ws = es + FwStage<IO>::span(size, hop);
    if (STAGED) {
        stage_span<IO, false>(es, eb, span0, FwStage<IO>::span(size, hop), T, (IO)1);
        stage_span<IO, false>(ws, win, 0, size, size, (IO)1);
        __syncwarp();
    }
    IO a[M];
#pragma unroll
    for (int i = 0; i < M; ++i) a[i] = active ? frames[(b * F + row) * M + i] : (IO)0;
    IO R[M];
#pragma unroll
    for (int p = 0; p < M; ++p) R[p] = (IO)0;
    IO* sb = seg + b * (int64_t)size * nfr + fi;
    const IO* el = es + (int64_t)lane * hop;  // this frame's excitation in the staged span
    for (int k0 = 0; k0 < size; k0 += L) {
#pragma unroll
        for (int u = 0; u < L; ++u) {
            const int k = k0 + u;
            if (k < size) {
                IO xin;
                if (STAGED) {
                    xin = el[k] * ws[k];
                } else {
                    const int64_t t = start + k;
                    xin = ((active && t >= 0 && t < T) ? eb[t] : (IO)0) * win[k];
                }
                IO p0 = (IO)0, p1 = (IO)0, p2 = (IO)0, p3 = (IO)0;
#pragma unroll
                for (int i = M; i >= 2; --i) {
                    const IO x = R[(u - i + 2 * M) % M];
                    switch (i & 3) {
                        case 0: p0 = fma(a[i - 1], x, p0); break;
                        case 1: p1 = fma(a[i - 1], x, p1); break;
                        case 2: p2 = fma(a[i - 1], x, p2); break;
                        default: p3 = fma(a[i - 1], x, p3); break;
                    }
                }
                const IO v = fma(-a[0], R[(u - 1 + M) % M], xin - ((p0 + p1) + (p2 + p3)));
                R[u % M] = v;
                if (active) sb[(int64_t)k * nfr] = v;
            }
        }
    }
}

// out[t] = (sum over frames covering t, in frame order, of seg) / cola
template <typename IO>
__global__ void k_fw_ola(const IO* __restrict__ seg, IO* __restrict__ out, int64_t B, int64_t T,
                         int nfr, int size, int hop, int n_lead, IO cola) {
    grid_dep_wait();
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= B * T) return;
    const int64_t b = idx / T, t = idx % T;
    // frames f with f*hop <= t < f*hop + size
    int64_t fhi = t / hop;
    int64_t flo = (t - size) >= 0 ? (t - size) / hop + 1 : -((size - t - 1) / hop);
    if (flo < -n_lead) flo = -n_lead;
    if (fhi > nfr - n_lead - 1) fhi = nfr - n_lead - 1;
    IO acc = (IO)0;
    const IO* sb = seg + b * (int64_t)size * nfr;
    for (int64_t f = flo; f <= fhi; ++f) {
        const int64_t k = t - f * hop;
        acc += sb[k * nfr + (f + n_lead)];
    }
    out[idx] = acc / cola;
}

// Adjoint per frame, reverse k:  lambda_0 += g(start+k)/cola (masked);
// ge_f(k) = lambda_0;  lambda = C^T lambda;  ga += ge_f(k) * s_f(k-1-c).
// Same warp/frame mapping and staging as the forward (g/cola staged).
template <typename IO, int M, bool STAGED>
__global__ void __launch_bounds__(32, 1)
k_fw_backward(const IO* __restrict__ gout, const IO* __restrict__ frames,
              const IO* __restrict__ win, const IO* __restrict__ seg, IO* __restrict__ gew,
              IO* __restrict__ gapart, int64_t B, int64_t T, int F, int nfr, int size, int hop,
              int n_lead, IO cola) {
    grid_dep_wait();

    extern __shared__ __align__(16) unsigned char fw_smem[];
    const int lane = threadIdx.x;
    const int64_t b = blockIdx.y;
    const int fi0 = blockIdx.x * 32;
    const int fi = fi0 + lane;
    const bool active = fi < nfr;
    const int f = fi - n_lead;
    const int row = f > 0 ? f : 0;
    const int64_t start = (int64_t)f * hop;
    const int64_t span0 = (int64_t)(fi0 - n_lead) * hop;
    const IO* gb = gout + b * T;
    IO* gs = reinterpret_cast<IO*>(fw_smem);
    IO* ws = gs + FwStage<IO>::span(size, hop);
    if (STAGED) {
        stage_span<IO, true>(gs, gb, span0, FwStage<IO>::span(size, hop), T, cola);
        stage_span<IO, false>(ws, win, 0, size, size, (IO)1);
        __syncwarp();
    }
    IO a[M];
#pragma unroll
    for (int i = 0; i < M; ++i) a[i] = active ? frames[(b * F + row) * M + i] : (IO)0;
    const int64_t gid = b * nfr + fi;
    const IO* sb = seg + b * (int64_t)size * nfr + fi;
    IO* ob = gew + b * (int64_t)size * nfr + fi;
    const IO* gl = gs + (int64_t)lane * hop;
    // ring of past outputs: R[k' mod RS] = s_f(k').  At step k it holds
    // s_f(k-1 .. k-RS); the slot freed by s_f(k-1) is refilled with
    // s_f(k-1-RS), which is first needed RS - M steps later, so the global
    // load has that many steps to land (a ring of exactly M slots exposed the
    // full memory latency every step).
    constexpr int RS = FwGeo<M>::RS;
    const int K0 = (size + RS - 1) / RS * RS;
    IO R[RS];
#pragma unroll
    for (int i = 0; i < RS; ++i) {
        const int kp = K0 - 2 - i;  // K0 % RS == 0, so the slot of s_f(kp) is static
        R[(2 * RS - 2 - i) % RS] =
            (active && kp >= 0 && kp < size) ? sb[(int64_t)kp * nfr] : (IO)0;
    }
    IO lam[M];
    IO ga[M];
#pragma unroll
    for (int i = 0; i < M; ++i) {
        lam[i] = (IO)0;
        ga[i] = (IO)0;
    }
    for (int kb = K0 - RS; kb >= 0; kb -= RS) {
#pragma unroll
        for (int u = RS - 1; u >= 0; --u) {
            const int k = kb + u;
            if (k < size) {
                IO gv, wk;
                if (STAGED) {
                    gv = gl[k];
                    wk = ws[k];
                } else {
                    const int64_t t = start + k;
                    gv = (active && t >= 0 && t < T) ? gb[t] / cola : (IO)0;
                    wk = win[k];
                }
                const IO l0 = lam[0] + gv;
                if (active) ob[(int64_t)k * nfr] = l0 * wk;
#pragma unroll
                for (int c = 0; c < M; ++c) ga[c] = fma(R[(u - 1 - c + 2 * RS) % RS], l0, ga[c]);
#pragma unroll
                for (int i = 0; i < M - 1; ++i) lam[i] = fma(-a[i], l0, lam[i + 1]);
                lam[M - 1] = -a[M - 1] * l0;
            }
            const int kp = k - 1 - RS;
            R[(u - 1 + 2 * RS) % RS] =
                (active && kp >= 0 && kp < size) ? sb[(int64_t)kp * nfr] : (IO)0;
        }
    }
    if (active) {
#pragma unroll
        for (int c = 0; c < M; ++c) gapart[gid * M + c] = -ga[c];
    }
}

// grad_e[t] = sum over covering frames (frame order) of gew;  grad_frames[row]
// = sum over frames mapping to row (lead-in frames hold row 0).
template <typename IO>
__global__ void k_fw_gather_ge(const IO* __restrict__ gew, IO* __restrict__ ge, int64_t B,
                               int64_t T, int nfr, int size, int hop, int n_lead) {
    grid_dep_wait();
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= B * T) return;
    const int64_t b = idx / T, t = idx % T;
    int64_t fhi = t / hop;
    int64_t flo = (t - size) >= 0 ? (t - size) / hop + 1 : -((size - t - 1) / hop);
    if (flo < -n_lead) flo = -n_lead;
    if (fhi > nfr - n_lead - 1) fhi = nfr - n_lead - 1;
    IO acc = (IO)0;
    const IO* gb = gew + b * (int64_t)size * nfr;
    for (int64_t f = flo; f <= fhi; ++f) acc += gb[(t - f * hop) * nfr + (f + n_lead)];
    ge[idx] = acc;
}

template <typename IO>
__global__ void k_fw_rows(const IO* __restrict__ gapart, IO* __restrict__ gf, int64_t B, int F,
                          int nfr, int M, int n_lead) {
    grid_dep_wait();
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= B * (int64_t)F * M) return;
    const int c = (int)(idx % M);
    const int64_t br = idx / M;
    const int r = (int)(br % F);
    const int64_t b = br / F;
    IO acc = (IO)0;
    if (r == 0) {
        for (int fi = 0; fi <= n_lead; ++fi) acc += gapart[(b * nfr + fi) * M + c];
    } else {
        acc = (IO)0 + gapart[(b * nfr + r + n_lead) * M + c];
    }
    gf[idx] = acc;
}

#define TVLP_FW_DISPATCH(Mp, ...)                          \
    switch (Mp) {                                          \
        case 2: { constexpr int M_ = 2; __VA_ARGS__ }      \
        case 4: { constexpr int M_ = 4; __VA_ARGS__ }      \
        case 6: { constexpr int M_ = 6; __VA_ARGS__ }      \
        case 8: { constexpr int M_ = 8; __VA_ARGS__ }      \
        case 12: { constexpr int M_ = 12; __VA_ARGS__ }    \
        case 16: { constexpr int M_ = 16; __VA_ARGS__ }    \
        case 22: { constexpr int M_ = 22; __VA_ARGS__ }    \
        case 24: { constexpr int M_ = 24; __VA_ARGS__ }    \
        case 30: { constexpr int M_ = 30; __VA_ARGS__ }    \
        default: return cudaErrorInvalidValue;             \
    }

template <typename IO>
cudaError_t launch_fw_forward(int Mp, const IO* e, const IO* frames, const IO* win, IO* seg,
                              IO* out, const FwArgs& a, cudaStream_t st) {
    const dim3 grid((unsigned)((a.nfr + 31) / 32), (unsigned)a.B);
    const size_t sm = FwStage<IO>::bytes(a.size, a.hop);
    const bool staged = sm <= kFwStageMax;
    TVLP_FW_DISPATCH(Mp, {
        if (staged) {
            auto k = k_fw_forward<IO, M_, true>;
            cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   (int)sm);
            if (err != cudaSuccess) return err;
            launch_pdl(k, grid, 32, sm, st, e, frames, win, seg, a.B, a.T, a.F, a.nfr, a.size,
                       a.hop, a.n_lead);
        } else {
            launch_pdl(k_fw_forward<IO, M_, false>, grid, 32, 0, st, e, frames, win, seg, a.B,
                       a.T, a.F, a.nfr, a.size, a.hop, a.n_lead);
        }
        break;
    })
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) return err;
    const int64_t n = a.B * a.T;
    launch_pdl(k_fw_ola<IO>, (unsigned)((n + 255) / 256), 256, 0, st, seg, out, a.B, a.T, a.nfr, a.size,
                                                              a.hop, a.n_lead, (IO)a.cola);
    return cudaGetLastError();
}

template <typename IO>
cudaError_t launch_fw_backward(int Mp, int M, const IO* gout, const IO* frames, const IO* win,
                               const IO* seg, IO* gew, IO* gapart, IO* ge, IO* gf,
                               const FwArgs& a, cudaStream_t st) {
    const dim3 grid((unsigned)((a.nfr + 31) / 32), (unsigned)a.B);
    const size_t sm = FwStage<IO>::bytes(a.size, a.hop);
    const bool staged = sm <= kFwStageMax;
    TVLP_FW_DISPATCH(Mp, {
        if (staged) {
            auto k = k_fw_backward<IO, M_, true>;
            cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   (int)sm);
            if (err != cudaSuccess) return err;
            launch_pdl(k, grid, 32, sm, st, gout, frames, win, seg, gew, gapart, a.B, a.T, a.F,
                       a.nfr, a.size, a.hop, a.n_lead, (IO)a.cola);
        } else {
            launch_pdl(k_fw_backward<IO, M_, false>, grid, 32, 0, st, gout, frames, win, seg, gew,
                       gapart, a.B, a.T, a.F, a.nfr, a.size, a.hop, a.n_lead, (IO)a.cola);
        }
        break;
    })
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) return err;
    const int64_t n = a.B * a.T;
    launch_pdl(k_fw_gather_ge<IO>, (unsigned)((n + 255) / 256), 256, 0, st, gew, ge, a.B, a.T, a.nfr,
                                                                    a.size, a.hop, a.n_lead);
    err = cudaGetLastError();
    if (err != cudaSuccess) return err;
    const int64_t nr = a.B * (int64_t)a.F * Mp;
    launch_pdl(k_fw_rows<IO>, (unsigned)((nr + 255) / 256), 256, 0, st, gapart, gf, a.B, a.F, a.nfr, Mp,
                                                                a.n_lead);
    (void)M;
    return cudaGetLastError();
}

template cudaError_t launch_fw_forward<float>(int, const float*, const float*, const float*,
                                              float*, float*, const FwArgs&, cudaStream_t);
template cudaError_t launch_fw_forward<double>(int, const double*, const double*, const double*,
                                               double*, double*, const FwArgs&, cudaStream_t);
template cudaError_t launch_fw_backward<float>(int, int, const float*, const float*, const float*,
                                               const float*, float*, float*, float*, float*,
                                               const FwArgs&, cudaStream_t);
template cudaError_t launch_fw_backward<double>(int, int, const double*, const double*,
                                                const double*, const double*, double*, double*,
                                                double*, double*, const FwArgs&, cudaStream_t);

}  // namespace tvlp
