// framewise.cu -- frame-wise time-invariant LP with overlap-add (GOLF-ff).
//
// Reference: pkg/src/tvlp/params.py:152-217 (FramePlan), 220-239
// (_framewise_forward), 259-273 (_framewise_vjp), lpc.py:50-61/176-195.
//
// Every frame f in [-n_lead, F) is an independent zero-state TI recursion of
// `size` samples over window[k] * e[f*hop + k] with coefficient row
// frames[max(f,0)].  Overlap-add and the frame-row reduction are
// deterministic gathers in frame order (the reference's accumulation order).
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include <cudaTypedefs.h>

#include "common.cuh"
#include "framewise_launch.cuh"


namespace tvlp {

// ============================================================================
// Layout: seg and the per-frame gradient contributions gew are [B][nfr][size]
// (frame-major: row fi is frame fi's output, like the reference's list of
// seg_outputs).  One warp = 32 consecutive frames of one sequence (lane =
// frame); every lane steps through k = 0..size-1 together.  Rows of 32
// frames x W steps leave (forward) or arrive (backward) as ONE 2-D tensor
// copy (box {W, 32}; the last block of a sequence uses a box of its
// remaining rows so it never touches the next sequence's frames).  The
// excitation / gradient span the 32 frames read is staged once in shared
// memory with one pad word per hop (lane f reads index f*(hop+1) + ..., 32
// distinct banks).  Overlap-add and the grad_e gather then read the
// frame-major rows with consecutive samples on consecutive threads.
// ============================================================================
constexpr int kFwW = 8;        // steps per compute window
constexpr int kFwOut = 2;      // output box stages
// output boxes: rows of 128 B (32 fp32 / 16 fp64 steps), 128B-swizzled in
// shared memory (conflict-free row writes): one proxy fence + tensor store
// per 128 B of steps instead of per compute window
template <typename IO>
struct FwOut {
    static constexpr int OW = 128 / (int)sizeof(IO);  // steps per output box
    // shared-memory element (row r, step c) of a 128B-swizzled [32][128 B] box
    static __device__ __forceinline__ int at(int r, int c) {
        const int byte = c * (int)sizeof(IO);
        return (r * 128 + ((((byte >> 4) ^ (r & 7)) << 4) | (byte & 15))) / (int)sizeof(IO);
    }
};

// backward: windows of saved outputs below the current one that the lags reach
template <int M>
struct FwLag {
    static constexpr int NB = (M + 1 + kFwW - 1) / kFwW;
    static constexpr int SW = (NB + 1) * kFwW;  // register window of saved outputs
    static constexpr int NS = NB + 10;          // stages of the saved-output ring (1 KB each)
};
constexpr int kFwSegStages = FwLag<30>::NS;  // shared-memory ring slots (the largest order)

struct FwMaps {
    CUtensorMap seg[2];   // [B*nfr][size] box {W, 32} / {W, nfr % 32} (backward loads)
    CUtensorMap segw[2];  // same rows, box {128 B, 32 / nfr % 32}, 128B swizzle (stores)
    CUtensorMap gew[2];   // gew rows, stores like segw
    void* segp;           // the seg / gew rows themselves: lanes store their windows directly
    void* gewp;
};

// W outputs of a lane's frame row from registers as 16-byte vectors (n valid:
// a multiple of the vector width, frame sizes are multiples of 4); see
// store_window in lp_scan.cuh for why there is no output box.
template <typename IO, int W>
__device__ __forceinline__ void fw_store_window(IO* dst, const IO (&v)[W], int n) {
    constexpr int V = 16 / (int)sizeof(IO);
#pragma unroll
    for (int q = 0; q < W / V; ++q) {
        if (q * V < n) {
            if constexpr (sizeof(IO) == 4)
                __stcs(reinterpret_cast<float4*>(dst) + q,
                       make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
            else
                __stcs(reinterpret_cast<double2*>(dst) + q, make_double2(v[2 * q], v[2 * q + 1]));
        }
    }
}

// The staged span keeps hop-blocks at a stride of fw_stride(hop) elements:
// blocks start 16-byte aligned (one bulk copy each) and lane f's reads land
// in different banks for 8 consecutive lanes.
template <typename IO>
__host__ __device__ __forceinline__ int fw_stride(int hop) {
    constexpr int q = 16 / (int)sizeof(IO);  // elements per 16 bytes
    int s = (hop + q - 1) / q * q;
    if (((s / q) & 1) == 0) s += q;
    return s;
}

template <typename IO>
struct FwSmem {
    static __host__ __device__ int span(int size, int hop) { return 31 * hop + size; }
    static __host__ __device__ int blocks(int size, int hop) { return (span(size, hop) + hop - 1) / hop; }
    static __host__ __device__ int padded(int size, int hop) {
        return blocks(size, hop) * fw_stride<IO>(hop);
    }
    static constexpr int OUT = 32 * 128;  // one output box: 32 rows x 128 B
    static constexpr int SEGW = 32 * kFwW * (int)sizeof(IO);  // one window of 32 rows
    // [span (padded)][window][out boxes][seg ring][barriers]
    static __host__ __device__ size_t off_win(int size, int hop) {
        return (size_t)padded(size, hop) * sizeof(IO);
    }
    static __host__ __device__ size_t off_out(int size, int hop) {
        // (128B-swizzled boxes need 1024-byte alignment)
        return (off_win(size, hop) + (size_t)size * sizeof(IO) + 1023) / 1024 * 1024;
    }
    static __host__ __device__ size_t off_seg(int size, int hop) {
        return off_out(size, hop) + kFwOut * OUT;
    }
    static __host__ __device__ size_t off_bar(int size, int hop, bool bwd) {
        return off_seg(size, hop) + (bwd ? kFwSegStages * SEGW : 0);
    }
    static size_t bytes(int size, int hop, bool bwd) {
        return off_bar(size, hop, bwd) + 8 * (kFwSegStages + 1);
    }
};

// Stage hop-blocks q = 0..nblk-1 of src (block q: times t0 + q*hop + [0, hop))
// at dst + q*stride, zero outside [0, n_src): blocks inside [0, n_src) with
// 16-byte aligned sources travel as one bulk copy each (lane 0, completing on
// `bar`), the rest by warp loads; with DIV the span is then divided by `div`
// in place (the reference's g = grad / cola, params.py:263).
template <typename IO, bool DIV>
__device__ __forceinline__ void fw_stage(IO* __restrict__ dst, const IO* __restrict__ src,
                                         int64_t t0, int nblk, int64_t n_src, int hop, IO div,
                                         uint64_t* bar) {
    const int lane = threadIdx.x & 31;
    const int st = fw_stride<IO>(hop);
    const uint32_t bbytes = (uint32_t)hop * sizeof(IO);
    auto bulk_ok = [&](int q) {
        const int64_t t = t0 + (int64_t)q * hop;
        return t >= 0 && t + hop <= n_src && bbytes % 16 == 0 &&
               ((reinterpret_cast<uintptr_t>(src + t) & 15) == 0);
    };
    if (lane == 0) {
        uint32_t tx = 0;
        for (int q = 0; q < nblk; ++q) tx += bulk_ok(q) ? bbytes : 0;
        mbar_init(bar, 1);
        fence_mbar_init();
        mbar_arrive_expect_tx(bar, tx);
        for (int q = 0; q < nblk; ++q)
            if (bulk_ok(q)) tma_load_1d(dst + q * st, src + t0 + (int64_t)q * hop, bbytes, bar);
    }
    for (int q = 0; q < nblk; ++q) {
        if (bulk_ok(q)) continue;  // warp-uniform
        for (int r = lane; r < hop; r += 32) {
            const int64_t t = t0 + (int64_t)q * hop + r;
            dst[q * st + r] = (t >= 0 && t < n_src) ? src[t] : (IO)0;
        }
    }
    __syncwarp();
    mbar_wait(bar, 0);
    if (DIV) {
        for (int q = 0; q < nblk; ++q)
            for (int r = lane; r < hop; r += 32) dst[q * st + r] = dst[q * st + r] / div;
        __syncwarp();
    }
}

// Forward per frame (params.py:230-237): zero-state TI recursion of
// window[k] * e[f*hop + k] with row frames[max(f, 0)] (lpc.py:50-61), in the
// same arithmetic as the TI/TV lane kernels (the reference's single
// rectangular frame == lp_forward_ti holds bit-exactly).
template <typename IO, int M>
__global__ void __launch_bounds__(32)
k_fw_forward(const __grid_constant__ FwMaps maps, const IO* __restrict__ e,
             const IO* __restrict__ frames, const IO* __restrict__ win, int64_t T, int F,
             int nfr, int size, int hop, int n_lead) {
    grid_dep_wait();
    using S = FwSmem<IO>;
    constexpr int W = kFwW;
    constexpr int L = (M + W - 1) / W * W;  // ring (>= M) = unrolled body: positions static
    extern __shared__ __align__(128) unsigned char fw_smem[];
    const int lane = threadIdx.x;
    const int64_t b = blockIdx.y;
    const int fi0 = blockIdx.x * 32;
    const int fi = fi0 + lane;
    const bool active = fi < nfr;
    const int rows = min(32, nfr - fi0);
    const int f = fi - n_lead;
    const int row = f > 0 ? f : 0;
    IO* es = reinterpret_cast<IO*>(fw_smem);
    IO* ws = reinterpret_cast<IO*>(fw_smem + S::off_win(size, hop));
    uint64_t* sbar = reinterpret_cast<uint64_t*>(fw_smem + S::off_bar(size, hop, false));
    fw_stage<IO, false>(es, e + b * T, (int64_t)(fi0 - n_lead) * hop, S::blocks(size, hop), T, hop,
                        (IO)1, sbar);
    for (int i = lane; i < size; i += 32) ws[i] = win[i];
    __syncwarp();
    IO a[M];
#pragma unroll
    for (int i = 0; i < M; ++i) a[i] = active ? frames[(b * F + row) * M + i] : (IO)0;
    IO R[L];
#pragma unroll
    for (int p = 0; p < L; ++p) R[p] = (IO)0;
    const int hst = fw_stride<IO>(hop);
    const int base = lane * hst;  // staged index of this frame's first sample
    const int nw = (size + W - 1) / W;
    const int64_t grow = b * nfr + fi0;
    for (int k0 = 0; k0 < nw * W; k0 += L) {
#pragma unroll
        for (int wi = 0; wi < L / W; ++wi) {
            const int kw = k0 + wi * W;  // window start
            if (kw < size) {
                // staged index of sample k (one division per window)
                const int kq = kw / hop, kr = kw - kq * hop;
                IO xv[W];
#pragma unroll
                for (int u = 0; u < W; ++u) {
                    const int k = kw + u;
                    const int pk = base + kq * hst + kr + u + (kr + u >= hop ? hst - hop : 0);
                    xv[u] = k < size ? es[pk] * ws[k] : (IO)0;
                }
                IO ov[W];
#pragma unroll
                for (int u = 0; u < W; ++u) {
                    const int pos = wi * W + u;  // position in the unrolled body
                    IO p0 = (IO)0, p1 = (IO)0, p2 = (IO)0, p3 = (IO)0;
#pragma unroll
                    for (int i = M; i >= 2; --i) {
                        const IO x = R[(pos - i + 2 * L) % L];
                        switch (i & 3) {
                            case 0: p0 = fma(a[i - 1], x, p0); break;
                            case 1: p1 = fma(a[i - 1], x, p1); break;
                            case 2: p2 = fma(a[i - 1], x, p2); break;
                            default: p3 = fma(a[i - 1], x, p3); break;
                        }
                    }
                    const IO v = fma(-a[0], R[(pos - 1 + L) % L], xv[u] - ((p0 + p1) + (p2 + p3)));
                    R[pos % L] = v;
                    ov[u] = v;
                }
                if (active)
                    fw_store_window<IO, W>(static_cast<IO*>(maps.segp) + (grow + lane) * size + kw,
                                           ov, size - kw);
            }
        }
    }
}

// sum over the frames f = q - j covering sample r of hop-block q, in frame
// order (j descending), of row (f + n_lead) at k = r + j*hop; the loads of a
// group of four are issued before the adds (a serial load-add chain was
// latency-bound: 4 dependent L2 trips per sample)
template <typename IO>
__device__ __forceinline__ IO fw_gather_sum(const IO* __restrict__ sb, int q, int r, int size,
                                            int hop, int n_lead, int flo, int fhi) {
    IO acc = (IO)0;
    for (int j0 = (size - 1 - r) / hop; j0 >= 0; j0 -= 4) {
        IO v[4];
#pragma unroll
        for (int d = 0; d < 4; ++d) {
            const int j = j0 - d, f = q - j;
            v[d] = (j >= 0 && f >= flo && f <= fhi) ? sb[(int64_t)(f + n_lead) * size + r + j * hop]
                                                     : (IO)0;
        }
#pragma unroll
        for (int d = 0; d < 4; ++d)
            if (j0 - d >= 0 && q - (j0 - d) >= flo && q - (j0 - d) <= fhi) acc += v[d];
    }
    return acc;
}

// Vector form of k_fw_ola / k_fw_gather_ge (fp32, hop % 4 == 0, T % 4 == 0):
// one thread per 4 consecutive samples, one 16-byte load per covering frame
// (the four samples share their frame range: r % 4 == 0 and hop % 4 == 0),
// summed per element in the same frame order.  DIV: / cola (the OLA).
template <bool DIV>
__global__ void k_fw_gather4(const float* __restrict__ rows, float* __restrict__ out, int64_t B,
                             int64_t T, int nfr, int size, int hop, int n_lead, float cola) {
    grid_dep_wait();
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t T4 = T / 4;
    if (idx >= B * T4) return;
    const int64_t b = idx / T4;
    const int t = (int)(idx - b * T4) * 4;
    const int q = t / hop, r = t - q * hop;
    const float* sb = rows + b * (int64_t)nfr * size;
    const int flo = -n_lead, fhi = nfr - n_lead - 1;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int j0 = (size - 1 - r) / hop; j0 >= 0; j0 -= 4) {
        float4 v[4];
#pragma unroll
        for (int d = 0; d < 4; ++d) {
            const int j = j0 - d, f = q - j;
            v[d] = (j >= 0 && f >= flo && f <= fhi)
                       ? __ldcs(reinterpret_cast<const float4*>(sb + (f + n_lead) * size + r +
                                                                j * hop))
                       : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int d = 0; d < 4; ++d) {
            const int j = j0 - d, f = q - j;
            if (j >= 0 && f >= flo && f <= fhi) {
                acc.x += v[d].x;
                acc.y += v[d].y;
                acc.z += v[d].z;
                acc.w += v[d].w;
            }
        }
    }
    if (DIV) {
        acc.x = acc.x / cola;
        acc.y = acc.y / cola;
        acc.z = acc.z / cola;
        acc.w = acc.w / cola;
    }
    reinterpret_cast<float4*>(out + b * T)[t / 4] = acc;
}

// out[t] = (sum over the frames covering t, in frame order, of seg) / cola
// (params.py:236-239).  Block (q, b) covers t = q*hop + r: the frames f =
// q-j (j descending, so frames ascend) contribute seg row f at k = r + j*hop;
// consecutive threads read consecutive samples of a row.
template <typename IO>
__global__ void k_fw_ola(const IO* __restrict__ seg, IO* __restrict__ out, int64_t T, int nfr,
                         int size, int hop, int n_lead, IO cola) {
    grid_dep_wait();
    const int64_t b = blockIdx.y;
    const int q = blockIdx.x;
    const IO* sb = seg + b * (int64_t)nfr * size;
    const int flo_all = -n_lead, fhi_all = nfr - n_lead - 1;
    for (int r = threadIdx.x; r < hop; r += blockDim.x) {
        const int64_t t = (int64_t)q * hop + r;
        if (t >= T) return;
        out[b * T + t] = fw_gather_sum<IO>(sb, q, r, size, hop, n_lead, flo_all, fhi_all) / cola;
    }
}

// Adjoint per frame (params.py:259-273 with lpc.py:176-195), reverse k:
//   lambda_0 += g(start + k) / cola;  ge_f(k) = lambda_0;  lambda = C^T lambda;
//   ga[c] += ge_f(k) s_f(k-1-c);  gew_f(k) = window[k] ge_f(k).
// The saved rows s_f stream in (reverse windows) through a ring of tensor
// copies; each window's steps read s_f(k-1-c) from a register window of the
// saved outputs, refreshed by one row load per window.
template <typename IO, int M>
__global__ void __launch_bounds__(32)
k_fw_backward(const __grid_constant__ FwMaps maps, const IO* __restrict__ gout,
              const IO* __restrict__ frames, const IO* __restrict__ win, IO* __restrict__ gapart,
              int64_t T, int F, int nfr, int size, int hop, int n_lead, IO cola) {
    grid_dep_wait();
    using S = FwSmem<IO>;
    constexpr int W = kFwW;
    constexpr int NB = FwLag<M>::NB, SW = FwLag<M>::SW, NS = FwLag<M>::NS;
    extern __shared__ __align__(128) unsigned char fw_smem[];
    const int lane = threadIdx.x;
    const int64_t b = blockIdx.y;
    const int fi0 = blockIdx.x * 32;
    const int fi = fi0 + lane;
    const bool active = fi < nfr;
    const int rows = min(32, nfr - fi0);
    const int mi = rows == 32 ? 0 : 1;
    const int f = fi - n_lead;
    const int row = f > 0 ? f : 0;
    IO* gs = reinterpret_cast<IO*>(fw_smem);
    IO* ws = reinterpret_cast<IO*>(fw_smem + S::off_win(size, hop));
    unsigned char* segs = fw_smem + S::off_seg(size, hop);
    uint64_t* bars = reinterpret_cast<uint64_t*>(fw_smem + S::off_bar(size, hop, true));
    const int nw = (size + W - 1) / W;
    const int64_t grow = b * nfr + fi0;
    const uint32_t tx = (uint32_t)rows * W * sizeof(IO);
    if (lane == 0) {
        prefetch_tmap(&maps.seg[mi]);
        for (int i = 0; i < NS; ++i) mbar_init(&bars[i], 1);
        fence_mbar_init();
    }
    __syncwarp();
    // loads run from the top window down: window w is the o-th load
    // (o = nw-1-w) and lives in stage o % NS, completing that stage's
    // (o / NS)-th phase
    auto issue = [&](int w) {
        if (lane == 0 && w >= 0) {
            const int st = (nw - 1 - w) % NS;
            mbar_arrive_expect_tx(&bars[st], tx);
            tma_load_2d(segs + st * S::SEGW, &maps.seg[mi], w * W, (int)grow, &bars[st]);
        }
    };
    for (int i = 0; i < NS; ++i) issue(nw - 1 - i);
    fw_stage<IO, true>(gs, gout + b * T, (int64_t)(fi0 - n_lead) * hop, S::blocks(size, hop), T, hop,
                       cola, bars + NS);
    for (int i = lane; i < size; i += 32) ws[i] = win[i];
    __syncwarp();
    IO a[M];
#pragma unroll
    for (int i = 0; i < M; ++i) a[i] = active ? frames[(b * F + row) * M + i] : (IO)0;
    IO lam[M], ga[M];
#pragma unroll
    for (int i = 0; i < M; ++i) {
        lam[i] = (IO)0;
        ga[i] = (IO)0;
    }
    // window w's saved row of this lane, 0 below window 0 (s(<0) = 0: zi = 0)
    auto seg_row = [&](int w, IO* dst) {
        if (w < 0) {
#pragma unroll
            for (int u = 0; u < W; ++u) dst[u] = (IO)0;
            return;
        }
        const int o = nw - 1 - w;
        mbar_wait(&bars[o % NS], (uint32_t)((o / NS) & 1));
        const IO* src = reinterpret_cast<const IO*>(segs + (o % NS) * S::SEGW) + lane * W;
#pragma unroll
        for (int u = 0; u < W; ++u) dst[u] = src[u];
    };
    IO sv[SW];  // sv[i] = s(kw - NB*W + i) for the current window start kw
#pragma unroll
    for (int j = 0; j <= NB; ++j) seg_row(nw - 1 - j, sv + (NB - j) * W);
    const int hst = fw_stride<IO>(hop);
    const int base = lane * hst;  // staged index of this frame's first sample
    for (int wv = nw - 1; wv >= 0; --wv) {
        const int kw = wv * W;
        IO gv[W], wk[W], ov[W];
        const int kq = kw / hop, kr = kw - kq * hop;
#pragma unroll
        for (int u = 0; u < W; ++u) {
            const int k = kw + u;
            const int pk = base + kq * hst + kr + u + (kr + u >= hop ? hst - hop : 0);
            gv[u] = k < size ? gs[pk] : (IO)0;
            wk[u] = k < size ? ws[k] : (IO)0;
        }
#pragma unroll
        for (int u = W - 1; u >= 0; --u) {
            const IO l0 = lam[0] + gv[u];
            ov[u] = l0 * wk[u];
#pragma unroll
            for (int c = 0; c < M; ++c) ga[c] = fma(sv[NB * W + u - 1 - c], l0, ga[c]);
#pragma unroll
            for (int i = 0; i < M - 1; ++i) lam[i] = fma(-a[i], l0, lam[i + 1]);
            lam[M - 1] = -a[M - 1] * l0;
        }
        if (active)
            fw_store_window<IO, W>(static_cast<IO*>(maps.gewp) + (grow + lane) * size + kw, ov,
                                   size - kw);
        // the stage of window wv is no longer needed: refill it NS windows down
        __syncwarp();
        issue(wv - NS);
        // slide the register window down by W
#pragma unroll
        for (int i = SW - 1; i >= W; --i) sv[i] = sv[i - W];
        seg_row(wv - NB - 1, sv);
    }
    if (active) {
#pragma unroll
        for (int c = 0; c < M; ++c) gapart[(b * nfr + fi) * M + c] = -ga[c];
    }
}

// grad_e[t] = sum over the frames covering t (frame order) of gew rows
// (same block geometry as k_fw_ola)
template <typename IO>
__global__ void k_fw_gather_ge(const IO* __restrict__ gew, IO* __restrict__ ge, int64_t T, int nfr,
                               int size, int hop, int n_lead) {
    grid_dep_wait();
    const int64_t b = blockIdx.y;
    const int q = blockIdx.x;
    const IO* gb = gew + b * (int64_t)nfr * size;
    const int flo_all = -n_lead, fhi_all = nfr - n_lead - 1;
    for (int r = threadIdx.x; r < hop; r += blockDim.x) {
        const int64_t t = (int64_t)q * hop + r;
        if (t >= T) return;
        ge[b * T + t] = fw_gather_sum<IO>(gb, q, r, size, hop, n_lead, flo_all, fhi_all);
    }
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

#include "framewise_pieces.cuh"

namespace {
// piece kernels for the plans they serve ($TVLP_FW_PIECES=0: one lane per frame)
bool fw_pieces(const FwArgs& a) {
    static const int on = [] {
        const char* v = std::getenv("TVLP_FW_PIECES");
        return (v != nullptr && v[0] != 0) ? std::atoi(v) : 1;
    }();
    return on != 0 && fwp_supported(a.size, a.hop);
}
// the vector OLA / grad_e gather applies (fp32, 16-byte aligned rows and outputs)
template <typename IO>
bool fw_gather4(const FwArgs& a, const void* rows, const void* out) {
    return sizeof(IO) == 4 && a.hop % 4 == 0 && a.T % 4 == 0 && a.size % 4 == 0 &&
           (reinterpret_cast<uintptr_t>(rows) & 15) == 0 &&
           (reinterpret_cast<uintptr_t>(out) & 15) == 0;
}
}  // namespace

// impulse-response tails the piece kernels exchange between forward and
// backward: [B][nfr][2 Mp] (0: the plan does not use the piece kernels)
int64_t fw_aux_elems(const FwArgs& a, int Mp) {
    return fw_pieces(a) ? a.B * (int64_t)a.nfr * 2 * Mp : 0;
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

namespace {
PFN_cuTensorMapEncodeTiled_v12000 fw_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}
// frame rows [B*nfr][size] of `base`, box {box0, rows}
cudaError_t fw_view(CUtensorMap* m, const void* base, int sz, const FwArgs& a, uint32_t box0,
                    uint32_t rows, bool swz) {
    std::memset(m, 0, sizeof(*m));
    auto fn = fw_encode();
    if (!fn) return cudaErrorNotSupported;
    cuuint64_t gdim[2] = {(cuuint64_t)a.size, (cuuint64_t)(a.B * a.nfr)};
    cuuint64_t gstr[1] = {(cuuint64_t)a.size * sz};
    cuuint32_t box[2] = {box0, rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = fn(m, sz == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                    2, const_cast<void*>(base), gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}
template <typename IO>
cudaError_t fw_maps(FwMaps& m, const IO* seg, const IO* gew, const FwArgs& a) {
    const uint32_t rem = (uint32_t)(a.nfr % 32 == 0 ? 32 : a.nfr % 32);
    const uint32_t box[2] = {32u, rem};
    const uint32_t ow = (uint32_t)FwOut<IO>::OW;
    for (int i = 0; i < 2; ++i) {
        cudaError_t err = fw_view(&m.seg[i], seg, (int)sizeof(IO), a, kFwW, box[i], false);
        if (err == cudaSuccess) err = fw_view(&m.segw[i], seg, (int)sizeof(IO), a, ow, box[i], true);
        if (err != cudaSuccess) return err;
        if (gew != nullptr) {
            err = fw_view(&m.gew[i], gew, (int)sizeof(IO), a, ow, box[i], true);
            if (err != cudaSuccess) return err;
        } else {
            std::memset(&m.gew[i], 0, sizeof(m.gew[i]));
        }
    }
    m.segp = const_cast<IO*>(seg);
    m.gewp = const_cast<IO*>(gew);
    return cudaSuccess;
}
}  // namespace

// frame sizes whose staged span fits the shared memory (the C ABI checks)
bool fw_supported(int Mp, int size, int hop, int elem) {
    if (Mp > 30 || size % 4 != 0 || hop < 1) return false;  // rows: 16-byte strides
    const size_t b = elem == 8 ? FwSmem<double>::bytes(size, hop, true)
                               : FwSmem<float>::bytes(size, hop, true);
    return b <= 220 * 1024;
}

template <typename IO>
cudaError_t launch_fw_forward(int Mp, const IO* e, const IO* frames, const IO* win, IO* seg,
                              IO* out, const FwArgs& a, cudaStream_t st, IO* aux) {
    if (!fw_supported(Mp, a.size, a.hop, (int)sizeof(IO))) return cudaErrorInvalidValue;
    const dim3 grid((unsigned)((a.nfr + 31) / 32), (unsigned)a.B);
    cudaError_t err = cudaSuccess;
    if (fw_pieces(a)) {
        const size_t sm = FwpSmem<IO>::bytes(a.size, a.hop);
        TVLP_FW_DISPATCH(Mp, {
            auto k = k_fwp_forward<IO, M_>;
            err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            if (err != cudaSuccess) return err;
            launch_pdl(k, dim3((unsigned)((a.nfr + kFwpFrames - 1) / kFwpFrames), (unsigned)a.B),
                       kFwpThreads, sm, st, seg, e, frames, win, a.T, a.F, a.nfr, a.size, a.hop,
                       a.n_lead, aux);
            break;
        })
    } else {
    const size_t sm = FwSmem<IO>::bytes(a.size, a.hop, false);
    FwMaps maps;
    err = fw_maps<IO>(maps, seg, nullptr, a);
    if (err != cudaSuccess) return err;
    TVLP_FW_DISPATCH(Mp, {
        auto k = k_fw_forward<IO, M_>;
        err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (err != cudaSuccess) return err;
        launch_pdl(k, grid, 32, sm, st, maps, e, frames, win, a.T, a.F, a.nfr, a.size, a.hop,
                   a.n_lead);
        break;
    })
    }
    err = cudaGetLastError();
    if (err != cudaSuccess) return err;
    if (fw_gather4<IO>(a, seg, out)) {
        const int64_t n = a.B * (a.T / 4);
        launch_pdl(k_fw_gather4<true>, (unsigned)((n + 255) / 256), 256, 0, st,
                   reinterpret_cast<const float*>(seg), reinterpret_cast<float*>(out), a.B, a.T,
                   a.nfr, a.size, a.hop, a.n_lead, (float)a.cola);
        return cudaGetLastError();
    }
    const dim3 og((unsigned)((a.T + a.hop - 1) / a.hop), (unsigned)a.B);
    launch_pdl(k_fw_ola<IO>, og, (unsigned)std::min(a.hop, 256), 0, st, seg, out, a.T, a.nfr,
               a.size, a.hop, a.n_lead, (IO)a.cola);
    return cudaGetLastError();
}

template <typename IO>
cudaError_t launch_fw_backward(int Mp, int M, const IO* gout, const IO* frames, const IO* win,
                               const IO* seg, IO* gew, IO* gapart, IO* ge, IO* gf,
                               const FwArgs& a, cudaStream_t st, const IO* aux) {
    if (!fw_supported(Mp, a.size, a.hop, (int)sizeof(IO))) return cudaErrorInvalidValue;
    const dim3 grid((unsigned)((a.nfr + 31) / 32), (unsigned)a.B);
    cudaError_t err = cudaSuccess;
    if (fw_pieces(a)) {
        const size_t sm = FwpSmem<IO>::bytes(a.size, a.hop);
        TVLP_FW_DISPATCH(Mp, {
            auto k = aux != nullptr ? k_fwp_backward<IO, M_, true> : k_fwp_backward<IO, M_, false>;
            err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
            if (err != cudaSuccess) return err;
            launch_pdl(k, dim3((unsigned)((a.nfr + kFwpFrames - 1) / kFwpFrames), (unsigned)a.B),
                       kFwpThreads, sm, st, gew, gapart, seg, gout, frames, win, a.T, a.F, a.nfr,
                       a.size, a.hop, a.n_lead, (IO)a.cola, aux);
            break;
        })
    } else {
    const size_t sm = FwSmem<IO>::bytes(a.size, a.hop, true);
    FwMaps maps;
    err = fw_maps<IO>(maps, seg, gew, a);
    if (err != cudaSuccess) return err;
    TVLP_FW_DISPATCH(Mp, {
        auto k = k_fw_backward<IO, M_>;
        err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
        if (err != cudaSuccess) return err;
        launch_pdl(k, grid, 32, sm, st, maps, gout, frames, win, gapart, a.T, a.F, a.nfr, a.size,
                   a.hop, a.n_lead, (IO)a.cola);
        break;
    })
    }
    err = cudaGetLastError();
    if (err != cudaSuccess) return err;
    if (fw_gather4<IO>(a, gew, ge)) {
        const int64_t n = a.B * (a.T / 4);
        launch_pdl(k_fw_gather4<false>, (unsigned)((n + 255) / 256), 256, 0, st,
                   reinterpret_cast<const float*>(gew), reinterpret_cast<float*>(ge), a.B, a.T,
                   a.nfr, a.size, a.hop, a.n_lead, 1.f);
    } else {
        const dim3 og((unsigned)((a.T + a.hop - 1) / a.hop), (unsigned)a.B);
        launch_pdl(k_fw_gather_ge<IO>, og, (unsigned)std::min(a.hop, 256), 0, st, gew, ge, a.T,
                   a.nfr, a.size, a.hop, a.n_lead);
    }
    err = cudaGetLastError();
    if (err != cudaSuccess) return err;
    const int64_t nr = a.B * (int64_t)a.F * Mp;
    launch_pdl(k_fw_rows<IO>, (unsigned)((nr + 255) / 256), 256, 0, st, gapart, gf, a.B, a.F,
               a.nfr, Mp, a.n_lead);
    (void)M;
    return cudaGetLastError();
}

template cudaError_t launch_fw_forward<float>(int, const float*, const float*, const float*,
                                              float*, float*, const FwArgs&, cudaStream_t, float*);
template cudaError_t launch_fw_forward<double>(int, const double*, const double*, const double*,
                                               double*, double*, const FwArgs&, cudaStream_t,
                                               double*);
template cudaError_t launch_fw_backward<float>(int, int, const float*, const float*, const float*,
                                               const float*, float*, float*, float*, float*,
                                               const FwArgs&, cudaStream_t, const float*);
template cudaError_t launch_fw_backward<double>(int, int, const double*, const double*,
                                                const double*, const double*, double*, double*,
                                                double*, double*, const FwArgs&, cudaStream_t,
                                                const double*);

}  // namespace tvlp
