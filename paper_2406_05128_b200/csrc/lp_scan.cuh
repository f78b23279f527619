// lp_scan.cuh -- chunked-scan kernels for the sample-wise (TV) and
// time-invariant (TI) all-pole recursion and its adjoint.
//
// Reference path: pkg/src/tvlp/lpc.py:36-47 (_lp_kernel_tv), 101-117
// (lp_forward_tv), 152-173 (lp_backward_tv), 50-61/82-98/176-195 (TI).
//
// Notation.  s(t) = e(t) - sum_{i=1..M} A[t,i-1] s(t-i).  State x(t) =
// [s(t), s(t-1), ..., s(t-M+1)];  x(t) = C(t) x(t-1) + u0 e(t) with C(t) the
// companion matrix of row A[t].  A sequence of T samples is cut into
// sub-chunks of Ls samples.  For sub-chunk j = [t0, t1]:
//   Phi_j = C(t1)...C(t0)              (M x M, "basis" kernel, M unit chains)
//   z_j   = zero-state final state     (one more chain driven by e)
//   x_in(j+1) = Phi_j x_in(j) + z_j    ("carry" kernel, serial per sequence)
// then every sub-chunk re-runs the recursion from x_in(j) ("apply" kernel,
// one lane per sub-chunk).  The adjoint lambda(t) = C(t+1)^T lambda(t+1) +
// u0 g_s(t), g_e(t) = lambda(t)_0, uses the same Phi_j transposed:
//   mu(j-1) = Phi_j^T mu(j) + nu_j     (nu_j: zero-state adjoint of sub-chunk j)
// The adjoint reads row A[t] at step t (transposed state form), so every
// sub-chunk only touches its own rows.  g_A[t,i-1] = -g_e(t) s(t-i).
//
// Data layout in HBM (all row-major, batch-major):
//   e, s, g_s, g_e : [B, T]          A, g_A : [B, T, M]     zi : [B, M]
//   PhiZ : [B*nsub, M+1, M]          (row c < M: column c of Phi_j; row M: z_j)
//   Xin, Nu, Mu : [B*nsub, M]        (all in the I/O dtype)
// Preconditions (enforced by the C ABI, which pads otherwise): Ls % 8 == 0,
// T % Ls == 0 (all sub-chunks full), all pointers 16-byte aligned.
#pragma once
#include "common.cuh"
#include "scan_launch.cuh"

#ifndef TVLP_BASIS_CHAINS
#define TVLP_BASIS_CHAINS 3
#endif
#ifndef TVLP_BASIS4_PIPE
#define TVLP_BASIS4_PIPE 0
#endif
#ifndef TVLP_BASIS4_MINB
#define TVLP_BASIS4_MINB 1
#endif
#ifndef TVLP_BASIS4_WARPS
#define TVLP_BASIS4_WARPS 2
#endif
#ifndef TVLP_BASIS4_STAGES
#define TVLP_BASIS4_STAGES 2
#endif
#ifndef TVLP_BASIS_GROUP
#define TVLP_BASIS_GROUP 2
#endif

namespace tvlp {

#ifndef TVLP_LANE_WIN
#define TVLP_LANE_WIN 8
#endif
constexpr int kLaneWin = TVLP_LANE_WIN;  // rows per TMA window in the lane-per-sub-chunk kernels
#ifndef TVLP_LANE_STAGES
#define TVLP_LANE_STAGES 3
#endif
constexpr int kLaneStages = TVLP_LANE_STAGES;  // input stages (per warp)
constexpr int kOutStages = 2;
#ifndef TVLP_GRAD_A_VEC
#define TVLP_GRAD_A_VEC 1
#endif   // output staging slots

template <int M>
struct Geo {
    static constexpr int WR = clcm(M, 4);          // basis window rows (multiple of M)
    static constexpr int LsUnit = clcm(WR, kLaneWin);  // Ls granularity
};

struct ScanArgs {
    int64_t B, T;
    int Ls, nsub;
};

// Carry tape of one sub-chunk (I/O dtype), rows padded to MP4 = round_up(M,4):
//   rows 0..M-1   W[c] = column c of Phi_j      (read by the adjoint carry)
//   row  M        z_j  (zero-state final state) (forward carry)
//   rows M+1..2M  R[i] = row i of Phi_j         (forward carry)
template <int M>
struct Tape {
    static constexpr int MP4 = (M + 3) / 4 * 4;
    static constexpr int Z_ROW = M;
    static constexpr int R_ROW = M + 1;
    static constexpr int SIZE = (2 * M + 1) * MP4;
};

// ============================================================================
// Basis kernel: one warp per sub-chunk; lane c < M runs the unit chain c,
// lane M runs the zero-state chain driven by e.  ACC is the chain precision
// (double by default: fp32 chains lose ~1e-3 relative on resonant filters,
// see DESIGN.md "precision").  Rows stream through shared memory in windows
// of WR rows by 1-D bulk TMA; the M-sample state lives in a register ring
// whose positions are compile-time (the unrolled body covers WR = k*M rows).
// ============================================================================
template <typename IO, typename ACC, int M, bool TI, int NW>
struct BasisSmem {
    static constexpr int WR = Geo<M>::WR;
    static constexpr int NSTB = 2;
    static constexpr bool CONV = !std::is_same<IO, ACC>::value;
    static constexpr int A_BYTES = TI ? 0 : WR * M * (int)sizeof(IO);
    static constexpr int E_BYTES = WR * (int)sizeof(IO);
    static constexpr int STAGE_BYTES = (A_BYTES + E_BYTES + 15) / 16 * 16;
    static constexpr int CONV_BYTES = CONV ? ((TI ? 0 : WR * M * (int)sizeof(ACC)) +
                                              WR * (int)sizeof(ACC) + 15) / 16 * 16
                                           : 0;
    static constexpr int WARP_BYTES = NSTB * STAGE_BYTES + CONV_BYTES;
    static constexpr int BYTES = NW * WARP_BYTES + NW * NSTB * 8;
};

template <typename IO, typename ACC, int M, bool TI, int NW>
__global__ void __launch_bounds__(NW * 32)
k_basis(const IO* __restrict__ e, const IO* __restrict__ A, IO* __restrict__ PhiZ,
        ScanArgs g) {
    grid_dep_wait();
    using S = BasisSmem<IO, ACC, M, TI, NW>;
    constexpr int WR = S::WR;
    constexpr int NSTB = S::NSTB;
    static_assert(M + 1 <= 32, "order M must be <= 31");
    extern __shared__ __align__(128) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char* wbase = smem + warp * S::WARP_BYTES;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NW * S::WARP_BYTES) + warp * NSTB;

    const int64_t gid = (int64_t)blockIdx.x * NW + warp;
    const int64_t nsc = g.B * g.nsub;
    if (gid >= nsc) return;  // warp-uniform
    const int64_t b = gid / g.nsub;
    const int j = (int)(gid % g.nsub);
    const int64_t t0 = (int64_t)j * g.Ls;
    const int len = (int)(int64_t)min((int64_t)(g.Ls), (int64_t)(g.T - t0));
    const int nwin = (len + WR - 1) / WR;
    const int64_t row0 = b * g.T + t0;

    if (lane == 0) {
        for (int s = 0; s < NSTB; ++s) mbar_init(&bars[s], 1);
        fence_mbar_init();
    }
    __syncwarp();

    auto stage_ptr = [&](int st) { return wbase + st * S::STAGE_BYTES; };
    auto issue = [&](int k) {
        if (k >= nwin) return;
        const int st = k % NSTB;
        const int rows = min(WR, len - k * WR);
        if (lane == 0) {
            const uint32_t bytes = rows * (TI ? 0 : M) * (int)sizeof(IO) + rows * (int)sizeof(IO);
            mbar_arrive_expect_tx(&bars[st], bytes);
            const int64_t r = row0 + (int64_t)k * WR;
            unsigned char* p = stage_ptr(st);
            if (!TI) tma_load_1d(p, A + r * M, rows * M * (int)sizeof(IO), &bars[st]);
            tma_load_1d(p + S::A_BYTES, e + r, rows * (int)sizeof(IO), &bars[st]);
        }
    };
#pragma unroll
    for (int k = 0; k < NSTB; ++k) issue(k);

    // TI: constant row in registers (the same A pointer holds a [B, M])
    ACC ati[M];
    if (TI) {
#pragma unroll
        for (int i = 0; i < M; ++i) ati[i] = (ACC)A[b * M + i];
    }

    // ring: R[p] holds s(t) for local step tau with tau mod M == p.
    ACC R[M];
#pragma unroll
    for (int p = 0; p < M; ++p) R[p] = (lane < M && (M - 1 - p) == lane) ? (ACC)1 : (ACC)0;
    const ACC emask = (lane == M) ? (ACC)1 : (ACC)0;

    for (int k = 0; k < nwin; ++k) {
        const int st = k % NSTB;
        mbar_wait(&bars[st], (uint32_t)((k / NSTB) & 1));
        const int rows = min(WR, len - k * WR);
        const ACC* Ar;
        const ACC* er;
        if constexpr (S::CONV) {
            ACC* cA = reinterpret_cast<ACC*>(wbase + NSTB * S::STAGE_BYTES);
            ACC* ce = cA + (TI ? 0 : WR * M);
            const IO* rawA = reinterpret_cast<const IO*>(stage_ptr(st));
            const IO* rawe = reinterpret_cast<const IO*>(stage_ptr(st) + S::A_BYTES);
            __syncwarp();
            if (!TI)
                for (int idx = lane; idx < rows * M; idx += 32) cA[idx] = (ACC)rawA[idx];
            for (int idx = lane; idx < rows; idx += 32) ce[idx] = (ACC)rawe[idx];
            __syncwarp();
            issue(k + NSTB);  // raw stage consumed
            Ar = cA;
            er = ce;
        } else {
            Ar = reinterpret_cast<const ACC*>(stage_ptr(st));
            er = reinterpret_cast<const ACC*>(stage_ptr(st) + S::A_BYTES);
        }
        const int tau0 = k * WR;
#pragma unroll
        for (int u = 0; u < WR; ++u) {
            ACC a[M];
            if constexpr (TI) {
#pragma unroll
                for (int i = 0; i < M; ++i) a[i] = ati[i];
            } else {
                load_row_at<ACC, M>(Ar + u * M, a, u * M * (int)sizeof(ACC));
            }
            const ACC ein = er[u] * emask;
            // terms i >= 2 first (older samples), freshest term last
            ACC p0 = (ACC)0, p1 = (ACC)0, p2 = (ACC)0, p3 = (ACC)0;
#pragma unroll
            for (int i = M; i >= 2; --i) {
                const ACC x = R[(u - i + 2 * M) % M];
                switch (i & 3) {
                    case 0: p0 = fma(a[i - 1], x, p0); break;
                    case 1: p1 = fma(a[i - 1], x, p1); break;
                    case 2: p2 = fma(a[i - 1], x, p2); break;
                    default: p3 = fma(a[i - 1], x, p3); break;
                }
            }
            const ACC part = ein - ((p0 + p1) + (p2 + p3));
            const ACC v = fma(-a[0], R[(u - 1 + M) % M], part);
            R[u % M] = (u < rows) ? v : R[u % M];
        }
        (void)tau0;
        if constexpr (!S::CONV) {
            __syncwarp();
            issue(k + NSTB);
        }
    }

    // final state x[i] = s(t1 - i) = R[(len-1-i) mod M]; runtime rotation.
    if (lane <= M) {
        ACC tmp[M];
#pragma unroll
        for (int p = 0; p < M; ++p) tmp[p] = R[p];
        IO* tape = PhiZ + gid * Tape<M>::SIZE;
        IO* out = tape + lane * Tape<M>::MP4;  // W[lane] (or z for lane M)
        const int last = (len - 1) % M;
        for (int i = 0; i < M; ++i) {
            const IO v = (IO)tmp[(last - i + M) % M];
            out[i] = v;
            if (lane < M) tape[(Tape<M>::R_ROW + i) * Tape<M>::MP4 + lane] = v;  // R[i][lane]
        }
    }
}

// ============================================================================
// fp32 basis, three chains per lane (scalar FFMA).  A sub-chunk takes
// P = ceil((M+1)/3) lanes (M = 22: 8 lanes, 24 slots for the M unit chains and
// the zero-state chain), a warp packs S = 32/P sub-chunks and is independent
// of every other warp (warp-level sync only).  Each lane's coefficient row
// loads (7 LDS per step for M = 22) are shared by its three chains, and the
// three chains are independent FMA streams (ILP) within the step.
// ============================================================================
// ---------------------------------------------------------------- frame-rate rows
// One formula for every kernel (the basis, apply and adjoint passes must see
// bit-identical rows): w = r * (1/hop), row = fa + w (fb - fa) (one FMA per
// coefficient; the last anchor has fb = fa, i.e. w = 0 as in params.py:116).
template <typename IO, int M>
__device__ __forceinline__ void frame_row_store(const FrameSrc<IO>& fs, int64_t b, int64_t t,
                                                IO inv_hop, IO* dst) {
    if (t >= fs.Tv) {
#pragma unroll
        for (int i = 0; i < M; ++i) dst[i] = (IO)0;
        return;
    }
    const int tt = (int)t;
    int f0 = tt / fs.hop;
    const int r = tt - f0 * fs.hop;
    if (f0 > fs.nF - 1) f0 = (int)fs.nF - 1;
    const int f1 = min(f0 + 1, (int)fs.nF - 1);
    const IO w = (IO)r * inv_hop;
    const IO* pa = fs.frames + ((int64_t)b * fs.nF + f0) * fs.Mf;
    const IO* pb = fs.frames + ((int64_t)b * fs.nF + f1) * fs.Mf;
    if constexpr (std::is_same<IO, float>::value && M % 2 == 0) {
        // unpadded even order (the decoder's 22): rows are 8-byte aligned,
        // read as float2 (half the load instructions; same values)
        if (fs.Mf == M && ((reinterpret_cast<uintptr_t>(pa) | reinterpret_cast<uintptr_t>(pb)) & 7) == 0) {
#pragma unroll
            for (int i = 0; i < M; i += 2) {
                const float2 a2 = __ldg(reinterpret_cast<const float2*>(pa + i));
                const float2 b2 = __ldg(reinterpret_cast<const float2*>(pb + i));
                dst[i] = fma(w, b2.x - a2.x, a2.x);
                dst[i + 1] = fma(w, b2.y - a2.y, a2.y);
            }
            return;
        }
    }
#pragma unroll
    for (int i = 0; i < M; ++i) {
        const IO fa = i < fs.Mf ? __ldg(pa + i) : (IO)0;
        const IO fb = i < fs.Mf ? __ldg(pb + i) : (IO)0;
        dst[i] = fma(w, fb - fa, fa);
    }
}
// Rows of one window of W consecutive times for one lane.  Interval changes
// (multiples of hop) fall on window boundaries because hop % W == 0 (the C
// ABI materialises A otherwise), so the frame rows are (re)loaded once per
// window at most and kept as (fa, fb - fa) in registers; per step one FMA per
// coefficient.  Keeping the reload out of the unrolled steps keeps the
// kernel's code small (a per-step reload thrashed the instruction cache).
template <typename IO, int M>
struct FrameCursor {
    int f0 = -1, r0 = 0;
    int64_t t = 0;
    IO fa[M], d[M];
    __device__ __forceinline__ void window(const FrameSrc<IO>& fs, int64_t b, int64_t t_first) {
        t = t_first;
        const int tt = (int)min(t_first, fs.Tv - 1);
        const int f = tt / fs.hop;
        r0 = (int)(t_first - (int64_t)f * fs.hop);
        if (f != f0 && t_first < fs.Tv) {
            f0 = f;
            const int g1 = min(f + 1, (int)fs.nF - 1);
            const IO* pa = fs.frames + ((int64_t)b * fs.nF + f) * fs.Mf;
            const IO* pb = fs.frames + ((int64_t)b * fs.nF + g1) * fs.Mf;
#pragma unroll
            for (int i = 0; i < M; ++i) {
                const IO x = i < fs.Mf ? __ldg(pa + i) : (IO)0;
                const IO y = i < fs.Mf ? __ldg(pb + i) : (IO)0;
                fa[i] = x;
                d[i] = y - x;
            }
        }
    }
    __device__ __forceinline__ void row(const FrameSrc<IO>& fs, IO inv_hop, int u,
                                        IO (&a)[M]) const {
        const IO w = (IO)(r0 + u) * inv_hop;
        const bool valid = t + u < fs.Tv;
#pragma unroll
        for (int i = 0; i < M; ++i) a[i] = valid ? fma(w, d[i], fa[i]) : (IO)0;
    }
};

// steps per basic block in full windows: steps of a group interleave; the
// group boundary bounds how far the scheduler runs ahead (register pressure)
constexpr int kBasisGroup = TVLP_BASIS_GROUP;
// independent scalar chains per lane (3: M = 22 -> 8 lanes per sub-chunk)
constexpr int kChains = TVLP_BASIS_CHAINS;
constexpr bool kBasisPipe = TVLP_BASIS4_PIPE;

template <int M, bool TI>
struct Basis4Cfg {
    static_assert(M % 2 == 0, "even orders only (odd orders are padded)");
    static constexpr int P = (M + kChains) / kChains;  // ceil((M + 1) / kChains)
    static constexpr int S = 32 / P;
    static constexpr int NW = TVLP_BASIS4_WARPS;  // independent warps per CTA
    static constexpr int NSTB = TVLP_BASIS4_STAGES;  // coefficient windows in flight per sub-chunk
    static constexpr int ROWS_BYTES = TI ? 0 : (M * M * 4 + 15) / 16 * 16;
    static constexpr int E_OFF = ROWS_BYTES;
    static constexpr int STAGE = ROWS_BYTES + 128;  // + the window's excitation (<= 28 floats)
    // after the scan a sub-chunk's region holds half of its tape at a time
    // (W + z rows, then R rows) for the bulk store
    static constexpr int OUT_BYTES = (M + 1) * Tape<M>::MP4 * 4;
    static constexpr int SUB_BYTES = NSTB * STAGE > OUT_BYTES ? NSTB * STAGE : OUT_BYTES;
    static constexpr int WARP_BYTES = S * SUB_BYTES;
    static constexpr int BAR_OFF = NW * WARP_BYTES;
    static constexpr int BYTES = BAR_OFF + NW * S * NSTB * 8;
};

// SPL: partial sums per chain (the 21 older-lag terms of a chain are a serial
// FMA dependency; SPL interleaved partial sums shorten it SPL-fold, for
// warps that must hide FMA latency alone -- the persistent chained forward)
template <int M, bool TI, int U, int SPL>
__device__ __forceinline__ void basis4_step(float (&R)[kChains][M], const float* __restrict__ Ar,
                                            const float* __restrict__ es, const float (&ati)[M],
                                            float (&ac)[M], int zs) {
    float a[M];
    if constexpr (TI) {
#pragma unroll
        for (int i = 0; i < M; ++i) a[i] = ati[i];
    } else if constexpr (kBasisPipe) {
        // row U was loaded one step ahead into ac; fetch row U+1 now so its
        // shared-memory latency hides behind this step's FMAs
#pragma unroll
        for (int i = 0; i < M; ++i) a[i] = ac[i];
        if constexpr (U + 1 < M) load_row_at<float, M>(Ar + (U + 1) * M, ac, (U + 1) * M * 4);
    } else {
        load_row_at<float, M>(Ar + U * M, a, U * M * 4);
    }
    const float ev = es[U];
    float c[kChains][SPL];
#pragma unroll
    for (int j = 0; j < kChains; ++j) {
        c[j][0] = zs == j ? ev : 0.f;
#pragma unroll
        for (int q = 1; q < SPL; ++q) c[j][q] = 0.f;
    }
#pragma unroll
    for (int i = M; i >= 2; --i) {  // lags M..2, oldest first
        const int r = (U - i + 2 * M) % M;
        const float na = -a[i - 1];
#pragma unroll
        for (int j = 0; j < kChains; ++j) c[j][i % SPL] = fmaf(na, R[j][r], c[j][i % SPL]);
    }
    const int r1 = (U - 1 + M) % M;
#pragma unroll
    for (int j = 0; j < kChains; ++j) {
        float t = c[j][0];
        if constexpr (SPL == 2) t = c[j][0] + c[j][1];
        if constexpr (SPL == 4) t = (c[j][0] + c[j][1]) + (c[j][2] + c[j][3]);
        R[j][U % M] = fmaf(-a[0], R[j][r1], t);
    }
}
template <int M, bool TI, int SPL, int G, int... V>
__device__ __forceinline__ void basis4_group(std::integer_sequence<int, V...>,
                                             float (&R)[kChains][M],
                                             const float* __restrict__ Ar,
                                             const float* __restrict__ es, const float (&ati)[M],
                                             float (&ac)[M], int zs) {
    ((G * kBasisGroup + V < M
          ? basis4_step<M, TI, (G * kBasisGroup + V) % M, SPL>(R, Ar, es, ati, ac, zs)
          : void()),
     ...);
}
template <int M, bool TI, int SPL, int... G>
__device__ __forceinline__ void basis4_full(std::integer_sequence<int, G...>,
                                            float (&R)[kChains][M],
                                            const float* __restrict__ Ar,
                                            const float* __restrict__ es, const float (&ati)[M],
                                            float (&ac)[M], int zs, int lim) {
    if constexpr (TI) {
        // no row loads to keep in place: one straight-line window
        (basis4_group<M, TI, SPL, G>(std::make_integer_sequence<int, kBasisGroup>{}, R, Ar, es,
                                     ati, ac, zs),
         ...);
    } else {
        ((G * kBasisGroup < lim
              ? basis4_group<M, TI, SPL, G>(std::make_integer_sequence<int, kBasisGroup>{}, R, Ar,
                                            es, ati, ac, zs)
              : void()),
         ...);
    }
}
template <int M, bool TI, int SPL, int... U>
__device__ __forceinline__ void basis4_partial(std::integer_sequence<int, U...>,
                                               float (&R)[kChains][M],
                                               const float* __restrict__ Ar,
                                               const float* __restrict__ es,
                                               const float (&ati)[M], float (&ac)[M], int zs,
                                               int u0) {
    ((U >= u0 ? basis4_step<M, TI, U, SPL>(R, Ar, es, ati, ac, zs) : void()), ...);
}

// One warp's basis work: lane (sub-chunk slot sc = lane / P, chain group
// q = lane % P) computes the chains of global sub-chunk `gid` (valid lanes)
// into the carry tape.  wbase: the warp's WARP_BYTES of shared memory; bars:
// the warp's S * NSTB mbarriers.  Used by k_basis4 (one sub-chunk group per
// warp) and by the persistent chained forward (a ticket loop of groups).
template <int M, bool TI, bool FR, int SPL = 1>
__device__ __forceinline__ void basis4_warp(const float* __restrict__ e,
                                            const float* __restrict__ A,
                                            float* __restrict__ PhiZ, const ScanArgs& g,
                                            const FrameSrc<float>& fs, int64_t gid, bool valid,
                                            unsigned char* wbase, uint64_t* wbars,
                                            int64_t tgid = -1) {
    using C = Basis4Cfg<M, TI>;
    constexpr int P = C::P, S = C::S, NSTB = C::NSTB;
    static_assert(M + 1 <= 32, "order M must be <= 31");
    const int lane = threadIdx.x & 31;
    const int q = lane % P;
    const bool lane_used = lane / P < S;
    const int sc = lane_used ? lane / P : S - 1;
    const int64_t nsc = g.B * g.nsub;
    const int64_t gg = gid < nsc ? gid : nsc - 1;
    const int64_t b = gg / g.nsub;
    const int j = (int)(gg % g.nsub);
    const int len = g.Ls;  // all sub-chunks are full (T % Ls == 0)
    const int u0 = (M - len % M) % M;  // the first window covers ring positions u0..M-1
    const int nwin = (len + u0) / M;
    const int64_t row0 = b * g.T + (int64_t)j * g.Ls;
    const float* eb = e + row0;
    unsigned char* sbase = wbase + sc * C::SUB_BYTES;
    auto stage = [&](int st) { return sbase + st * C::STAGE; };
    uint64_t* bars = wbars + sc * NSTB;
    const bool leader = valid && q == 0;

    // Window k covers ring positions first..M-1 = times k*M - u0 + (first..M-1).
    // Its coefficient rows and its excitation both arrive by bulk copy on the
    // stage's mbarrier; the excitation copy starts at the 16-byte boundary at
    // or below the window's first time (row0 is a multiple of 8 samples) and
    // ends at the next boundary at or above its end (never past the sub-chunk,
    // whose end is the end of the last window), so es = base + eoff.
    auto e_lo = [&](int k) {
        const int first = k == 0 ? u0 : 0;
        return (k * M - u0 + first) & ~3;
    };
    auto issue = [&](int k) {
        if (!leader || k >= nwin) return;
        const int st = k % NSTB;
        const int first = k == 0 ? u0 : 0;
        const int64_t tstart = (int64_t)k * M - u0 + first;
        const int rows = M - first;
        const int elo = e_lo(k), ehi = (k * M - u0 + M + 3) & ~3;
        const uint32_t ebytes = (uint32_t)(ehi - elo) * 4;
        mbar_arrive_expect_tx(&bars[st], ((TI || FR) ? 0 : rows * M * 4) + ebytes);
        if (!TI && !FR)
            tma_load_1d(stage(st) + first * M * 4, A + (row0 + tstart) * M, rows * M * 4,
                        &bars[st]);
        tma_load_1d(stage(st) + C::E_OFF, eb + elo, ebytes, &bars[st]);
    };
    if (leader) {
        for (int st = 0; st < NSTB; ++st) mbar_init(&bars[st], 1);
        fence_mbar_init();
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < NSTB; ++k) issue(k);

    float ati[M];
    if (TI) {
#pragma unroll
        for (int i = 0; i < M; ++i) ati[i] = A[b * M + i];
    }
    const int c0 = kChains * q;  // chains c0 .. c0+kChains-1 (chain M: the zero-state chain)
    const int zs = M - c0;       // which of the lane's chains is the zero-state one, if any
    float R[kChains][M];
    float ac[M];  // coefficient row of the next step (pipelined loads)
#pragma unroll
    for (int p = 0; p < M; ++p) {
        const int c = ((u0 - 1 - p) % M + M) % M;  // state component held at ring position p
#pragma unroll
        for (int j = 0; j < kChains; ++j) R[j][p] = c == c0 + j ? 1.f : 0.f;
    }

    const float inv_hop = FR ? 1.f / (float)fs.hop : 0.f;
    for (int k = 0; k < nwin; ++k) {
        const int st = k % NSTB;
        if constexpr (FR) {
            // the window's coefficient rows, interpolated from the frame rows by
            // the sub-chunk's lanes into the stage (ring position U = row U)
            if (lane_used) {
                float* rows_out = reinterpret_cast<float*>(stage(st));
                const int first = k == 0 ? u0 : 0;
                for (int U = first + q; U < M; U += P)
                    frame_row_store<float, M>(fs, b, (int64_t)j * g.Ls + k * M - u0 + U, inv_hop,
                                              rows_out + U * M);
            }
            __syncwarp();
        }
        if (valid) mbar_wait(&bars[st], (uint32_t)((k / NSTB) & 1));
        const float* Ar = reinterpret_cast<const float*>(stage(st));
        const float* es =
            reinterpret_cast<const float*>(stage(st) + C::E_OFF) + (k * M - u0 - e_lo(k));
        if (!TI && kBasisPipe) {  // first row of the window (later rows are fetched a step ahead)
            const int first = (k == 0) ? u0 : 0;
            load_row_at<float, M>(Ar + first * M, ac, first * M * 4);
        }
        if (k == 0 && u0 != 0)
            basis4_partial<M, TI, SPL>(std::make_integer_sequence<int, M>{}, R, Ar, es, ati, ac, zs,
                                       u0);
        else
            basis4_full<M, TI, SPL>(std::make_integer_sequence<int, (M + kBasisGroup - 1) / kBasisGroup>{},
                               R, Ar, es, ati, ac, zs, len);
        __syncwarp();  // the warp is done with stage st (generic reads before the async refill
                       // are ordered by this sync; no proxy fence is needed for WAR)
        issue(k + NSTB);
    }

    // Final states -> tape through shared memory: the tape rows of a sub-chunk
    // are assembled in its (now idle) stage region and leave as two bulk
    // stores (W + z rows, then the transposed R rows) instead of 132 scattered
    // 4-byte stores per lane.
    constexpr int MP4 = Tape<M>::MP4;
    float* buf = reinterpret_cast<float*>(sbase);
    // (grouped launches: e/A index the lane's group, the tape the whole launch)
    float* tape = PhiZ + (tgid >= 0 ? tgid : gg) * Tape<M>::SIZE;
    __syncwarp();
    if (lane_used) {
#pragma unroll
        for (int i = 0; i < M; ++i) {
#pragma unroll
            for (int c = 0; c < kChains; ++c)
                if (c0 + c <= M) buf[(c0 + c) * MP4 + i] = R[c][M - 1 - i];  // W column / z row
        }
#pragma unroll
        for (int c = 0; c < kChains; ++c)
            if (c0 + c <= M)
                for (int i = M; i < MP4; ++i) buf[(c0 + c) * MP4 + i] = 0.f;
    }
    fence_proxy_async();
    __syncwarp();
    if (leader) {
        tma_store_1d(tape, buf, (M + 1) * MP4 * 4);
        bulk_commit();
        bulk_wait_read<0>();
    }
    __syncwarp();
    if (lane_used) {
#pragma unroll
        for (int i = 0; i < M; ++i) {
#pragma unroll
            for (int c = 0; c < kChains; ++c)
                if (c0 + c < M) buf[i * MP4 + c0 + c] = R[c][M - 1 - i];  // R row i
        }
        if (zs >= 0 && zs < kChains)  // the zero-state lane pads the R rows
            for (int i = 0; i < M; ++i)
                for (int c = M; c < MP4; ++c) buf[i * MP4 + c] = 0.f;
    }
    fence_proxy_async();
    __syncwarp();
    if (leader) {
        tma_store_1d(tape + Tape<M>::R_ROW * MP4, buf, M * MP4 * 4);
        bulk_commit();
        bulk_wait<0>();
    }
}

template <int M, bool TI, bool FR = false>
__global__ void __launch_bounds__(Basis4Cfg<M, TI>::NW * 32, TVLP_BASIS4_MINB)
k_basis4(const float* __restrict__ e, const float* __restrict__ A, float* __restrict__ PhiZ,
         ScanArgs g, const FrameSrc<float> fs) {
    grid_dep_wait();
    using C = Basis4Cfg<M, TI>;
    extern __shared__ __align__(128) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool lane_used = lane / C::P < C::S;
    const int sc = lane_used ? lane / C::P : C::S - 1;
    const int64_t gid = ((int64_t)blockIdx.x * C::NW + warp) * C::S + sc;
    const bool valid = lane_used && gid < g.B * g.nsub;  // idle lanes compute on garbage, never wait
    basis4_warp<M, TI, FR>(e, A, PhiZ, g, fs, gid, valid, smem + warp * C::WARP_BYTES,
                           reinterpret_cast<uint64_t*>(smem + C::BAR_OFF) + warp * C::S * C::NSTB);
}

// ============================================================================
// Carry kernels: one warp per segment of consecutive sub-chunks (a whole
// sequence, or a group in the two-level scheme), lane r holds component r.
// The chain is latency-bound (one M x M mat-vec per sub-chunk): the tape rows
// it needs stream into a kCS-deep shared-memory ring by bulk TMA (one copy per
// sub-chunk, issued kCS steps ahead), the lane's matrix row and the broadcast
// state are read as 16-byte vectors, and the dot product runs on 4 partial
// accumulators.
// ============================================================================
#ifndef TVLP_CARRY_CB
#define TVLP_CARRY_CB 8
#endif
#ifndef TVLP_CARRY_CS
#define TVLP_CARRY_CS 4
#endif
// sub-chunks per carry ring stage (one wait / copy per stage; 8 measured
// better than 4: 20.8 -> 18.8 us fwd, 25.0 -> 22.9 us bwd at config 3)
constexpr int kCB = TVLP_CARRY_CB;
constexpr int kCS = TVLP_CARRY_CS;   // carry ring stages (kCB*kCS sub-chunks in flight)

template <typename CT, int N>
__device__ __forceinline__ void load_vec(const CT* p, CT (&v)[N]) {
    static_assert(N % 4 == 0, "padded rows");
    if constexpr (sizeof(CT) == 4) {
#pragma unroll
        for (int i = 0; i < N; i += 4) {
            const float4 q = *reinterpret_cast<const float4*>(p + i);
            v[i] = q.x;
            v[i + 1] = q.y;
            v[i + 2] = q.z;
            v[i + 3] = q.w;
        }
    } else {
#pragma unroll
        for (int i = 0; i < N; i += 2) {
            const double2 q = *reinterpret_cast<const double2*>(p + i);
            v[i] = q.x;
            v[i + 1] = q.y;
        }
    }
}

template <int M, typename CT>
__device__ __forceinline__ CT dot_rows(const CT (&w)[Tape<M>::MP4], const CT (&x)[Tape<M>::MP4],
                                       CT init) {
    CT q0 = init, q1 = (CT)0, q2 = (CT)0, q3 = (CT)0;
#pragma unroll
    for (int c = 0; c < M; ++c) {
        switch (c & 3) {
            case 0: q0 = fma(w[c], x[c], q0); break;
            case 1: q1 = fma(w[c], x[c], q1); break;
            case 2: q2 = fma(w[c], x[c], q2); break;
            default: q3 = fma(w[c], x[c], q3); break;
        }
    }
    return (q0 + q1) + (q2 + q3);
}

template <int M, typename CT, int CBW = kCB>
struct CarrySmem {
    static constexpr int MP4 = Tape<M>::MP4;
    static constexpr int SUB = Tape<M>::SIZE * (int)sizeof(CT);  // one sub-chunk's tape
    // as many tapes per stage as requested while the ring stays under ~200 KB
    // (fp64 tapes and high orders are larger)
    static constexpr int CB_FIT = (200 * 1024) / (kCS * (SUB + MP4 * (int)sizeof(CT)));
    static constexpr int CB = CBW < CB_FIT ? CBW : (CB_FIT > 0 ? CB_FIT : 1);
    static constexpr int STAGE = CB * SUB;
    static constexpr int NU = CB * MP4 * (int)sizeof(CT);        // bwd: nu of the stage
    static constexpr int BYTES = kCS * (STAGE + NU) + 64 * (int)sizeof(CT) + kCS * 8;
};

// Arguments of the carry recurrences.  A "segment" is a run of consecutive
// sub-chunks (or groups) of one sequence: the whole sequence in the one-level
// scheme, one group in the expansion step of the hierarchical scheme.
template <typename CT>
struct CarryArgs {
    // 3-D view [tapes][2M+1 rows][MP4] of `tape` (use_tmap): each ring stage
    // is ONE tensor copy of just the rows the chain reads (z + R rows forward,
    // W rows backward) -- a single CTA's bulk copies stream at ~24 GB/s, so
    // the carry chains were bound by the tape bytes they moved (measured)
    alignas(64) CUtensorMap tmap;
    int use_tmap;
    const CT* tape;      // [B*nsub][Tape<M>::SIZE]
    const CT* force;     // fwd: nullable override of the tape's z rows; bwd: nu. [B*nsub][MP4]
    const CT* x0;        // nullable initial state per segment (fwd: left end, bwd: right end)
    int64_t x0_stride;
    CT* X;               // nullable: fwd state at each sub-chunk start / bwd carry into each sub-chunk
    CT* tail;            // nullable: state past the segment (fwd: after its last sub-chunk,
                         // bwd: left of its first sub-chunk), one row per segment
    int64_t tail_stride;
    int64_t nseg;
    int seglen, nsub;
    unsigned* dstat;     // fwd only: zeroed per sequence (defect statistics of "auto")
    int* fflags;         // fwd only: zeroed per sequence (forward refinement flags)
    const int* only;     // nullable: per-sequence flags; other sequences' segments return
};

// Forward carry: x(k0) = x0 (or zero), x(k+1) = Phi_k x(k) + z_k.  One warp per
// segment (one CTA); whole tapes of SM::CB consecutive sub-chunks per bulk copy.
template <int M, typename CT, int CBW = kCB, bool TM = false>
__global__ void __launch_bounds__(32)
k_carry_fwd(const __grid_constant__ CarryArgs<CT> a) {
    grid_dep_wait();
    using TP = Tape<M>;
    using SM = CarrySmem<M, CT, CBW>;
    constexpr int MP4 = TP::MP4;
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x;
    CT* xs = reinterpret_cast<CT*>(smem + kCS * (SM::STAGE + SM::NU));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kCS * (SM::STAGE + SM::NU) + 64 * sizeof(CT));
    const int64_t sidx = blockIdx.x;
    if (sidx >= a.nseg) return;
    const int nper = (a.nsub + a.seglen - 1) / a.seglen;  // segments per sequence
    const int64_t b = sidx / nper;
    if (a.only != nullptr && a.only[b] == 0) return;
    const int k0 = (int)(sidx % nper) * a.seglen;
    const int n = min(a.seglen, a.nsub - k0);
    const int64_t base = b * a.nsub + k0;
    const int r = lane < M ? lane : 0;
    const int nsteps = a.tail != nullptr ? n : n - 1;  // mat-vecs needed
    const int nst = (nsteps + SM::CB - 1) / SM::CB;
    if (lane == 0) {
        for (int i = 0; i < kCS; ++i) mbar_init(&bars[i], 1);
        fence_mbar_init();
    }
    __syncwarp();
    auto issue = [&](int sg) {  // stage sg: sub-chunks sg*SM::CB .. +SM::CB-1
        if (lane == 0 && sg < nst) {
            const int st = sg % kCS;
            const int cnt = min(SM::CB, nsteps - sg * SM::CB);
            unsigned char* dst = smem + st * (SM::STAGE + SM::NU);
            if (TM) {  // z + R rows of SM::CB tapes: box [CB][M+1][MP4]
                mbar_arrive_expect_tx(&bars[st], SM::CB * (M + 1) * MP4 * (int)sizeof(CT) +
                                                     (a.force ? cnt * MP4 * (int)sizeof(CT) : 0));
                tma_load_3d(dst, &a.tmap, 0, TP::Z_ROW, (int)(base + sg * SM::CB), &bars[st]);
            } else {
                mbar_arrive_expect_tx(&bars[st],
                                      cnt * (SM::SUB + (a.force ? MP4 * (int)sizeof(CT) : 0)));
                tma_load_1d(dst, a.tape + (base + sg * SM::CB) * TP::SIZE, cnt * SM::SUB,
                            &bars[st]);
            }
            if (a.force)
                tma_load_1d(dst + SM::STAGE, a.force + (base + sg * SM::CB) * MP4,
                            cnt * MP4 * sizeof(CT), &bars[st]);
        }
    };
    for (int i = 0; i < kCS; ++i) issue(i);
    if (lane == 0 && k0 == 0) {
        if (a.dstat != nullptr) {
            a.dstat[2 * b] = 0u;
            a.dstat[2 * b + 1] = 0u;
        }
        if (a.fflags != nullptr) a.fflags[b] = 0;  // set by k_refine_fwd in precision "auto"
    }
    CT x = (a.x0 != nullptr && lane < M) ? a.x0[sidx * a.x0_stride + lane] : (CT)0;
    for (int sg = 0; sg < nst; ++sg) {
        const int st = sg % kCS;
        mbar_wait(&bars[st], (uint32_t)((sg / kCS) & 1));
        const unsigned char* dst = smem + st * (SM::STAGE + SM::NU);
        const CT* sgb = reinterpret_cast<const CT*>(dst);
        const CT* fgb = reinterpret_cast<const CT*>(dst + SM::STAGE);
#pragma unroll
        for (int u = 0; u < SM::CB; ++u) {
            const int i = sg * SM::CB + u;
            if (i < nsteps) {
                // the matrix row does not depend on x: load it before the
                // broadcast so only STS -> LDS -> FMA chain is serial
                // tensor-copied stage: tape u is [z row, R rows] at stride (M+1) MP4
                const CT* tp = TM ? sgb + u * (M + 1) * MP4 - TP::Z_ROW * MP4
                                  : sgb + u * TP::SIZE;
                CT w[MP4], xv[MP4];
                load_vec<CT, MP4>(tp + (TP::R_ROW + r) * MP4, w);
                const CT zr = a.force ? fgb[u * MP4 + r] : tp[TP::Z_ROW * MP4 + r];
                if (a.X != nullptr && lane < M) a.X[(base + i) * MP4 + lane] = x;
                // two broadcast buffers alternate, so one warp sync per step
                // orders both the write-after-read and the read-after-write
                CT* xb = xs + (i & 1) * 32;
                xb[lane] = lane < M ? x : (CT)0;
                __syncwarp();
                load_vec<CT, MP4>(xb, xv);
                x = dot_rows<M, CT>(w, xv, zr);
            }
        }
        __syncwarp();
        issue(sg + kCS);
    }
    if (lane < M) {
        if (a.tail != nullptr)
            a.tail[sidx * a.tail_stride + lane] = x;
        else if (a.X != nullptr)
            a.X[(base + n - 1) * MP4 + lane] = x;
    }
}

// Adjoint carry (right to left): mu(k_last) = x0 (or zero),
// mu(k-1) = Phi_k^T mu(k) + nu_k.  X[k] = carry into sub-chunk k from the right.
template <int M, typename CT, int CBW = kCB, bool TM = false>
__global__ void __launch_bounds__(32)
k_carry_bwd(const __grid_constant__ CarryArgs<CT> a) {
    grid_dep_wait();
    using TP = Tape<M>;
    using SM = CarrySmem<M, CT, CBW>;
    constexpr int MP4 = TP::MP4;
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x;
    CT* ms = reinterpret_cast<CT*>(smem + kCS * (SM::STAGE + SM::NU));
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kCS * (SM::STAGE + SM::NU) + 64 * sizeof(CT));
    const int64_t sidx = blockIdx.x;
    if (sidx >= a.nseg) return;
    const int nper = (a.nsub + a.seglen - 1) / a.seglen;
    const int64_t b = sidx / nper;
    if (a.only != nullptr && a.only[b] == 0) return;
    const int k0 = (int)(sidx % nper) * a.seglen;
    const int n = min(a.seglen, a.nsub - k0);
    const int64_t base = b * a.nsub + k0;
    const int r = lane < M ? lane : 0;
    // mat-vec i uses sub-chunk kk = n-1-i (kk >= 1, or >= 0 with a tail);
    // stage sg holds sub-chunks kk = n-1-sg*SM::CB-u (descending), i.e. the
    // contiguous range [hi-cnt+1, hi] with hi = n-1-sg*SM::CB.
    const int nsteps = a.tail != nullptr ? n : n - 1;
    const int nst = (nsteps + SM::CB - 1) / SM::CB;
    if (lane == 0) {
        for (int i = 0; i < kCS; ++i) mbar_init(&bars[i], 1);
        fence_mbar_init();
    }
    __syncwarp();
    auto issue = [&](int sg) {
        if (lane == 0 && sg < nst) {
            const int st = sg % kCS;
            const int cnt = min(SM::CB, nsteps - sg * SM::CB);
            const int lo = n - sg * SM::CB - cnt;  // lowest sub-chunk of the stage
            unsigned char* dst = smem + st * (SM::STAGE + SM::NU);
            if (TM) {  // W rows of SM::CB tapes from the stage's lowest: box [CB][M][MP4]
                mbar_arrive_expect_tx(&bars[st], SM::CB * M * MP4 * (int)sizeof(CT) +
                                                     cnt * MP4 * (int)sizeof(CT));
                tma_load_3d(dst, &a.tmap, 0, 0, (int)(base + lo), &bars[st]);
            } else {
                mbar_arrive_expect_tx(&bars[st], cnt * (SM::SUB + MP4 * (int)sizeof(CT)));
                tma_load_1d(dst, a.tape + (base + lo) * TP::SIZE, cnt * SM::SUB, &bars[st]);
            }
            tma_load_1d(dst + SM::STAGE, a.force + (base + lo) * MP4, cnt * MP4 * sizeof(CT),
                        &bars[st]);
        }
    };
    for (int i = 0; i < kCS; ++i) issue(i);
    CT mu = (a.x0 != nullptr && lane < M) ? a.x0[sidx * a.x0_stride + lane] : (CT)0;
    for (int sg = 0; sg < nst; ++sg) {
        const int st = sg % kCS;
        mbar_wait(&bars[st], (uint32_t)((sg / kCS) & 1));
        const unsigned char* dst = smem + st * (SM::STAGE + SM::NU);
        const int cnt = min(SM::CB, nsteps - sg * SM::CB);
#pragma unroll
        for (int u = 0; u < SM::CB; ++u) {
            const int i = sg * SM::CB + u;
            if (i < nsteps) {
                const int kk = n - 1 - i;
                const int slot = cnt - 1 - u;  // position of kk inside the stage
                const CT* tp = reinterpret_cast<const CT*>(dst) + slot * (TM ? M * MP4 : TP::SIZE);
                const CT* nu = reinterpret_cast<const CT*>(dst + SM::STAGE) + slot * MP4;
                CT w[MP4], mv[MP4];
                load_vec<CT, MP4>(tp + r * MP4, w);
                const CT nur = nu[r];
                if (a.X != nullptr && lane < M) a.X[(base + kk) * MP4 + lane] = mu;
                CT* mb = ms + (i & 1) * 32;
                mb[lane] = lane < M ? mu : (CT)0;
                __syncwarp();
                load_vec<CT, MP4>(mb, mv);
                mu = dot_rows<M, CT>(w, mv, nur);
            }
        }
        __syncwarp();
        issue(sg + kCS);
    }
    if (lane < M) {
        if (a.tail != nullptr)
            a.tail[sidx * a.tail_stride + lane] = mu;
        else if (a.X != nullptr)
            a.X[base * MP4 + lane] = mu;
    }
}

// Group product for the hierarchical carry: P_g = Phi_{k1-1} ... Phi_{k0} over
// a group of G consecutive sub-chunks, written in the tape layout (W rows =
// columns, R rows = rows; the z row is filled by a k_carry_fwd tail pass).
// One warp per group; lane c < M owns column c of the running product, the
// factor's rows are broadcast from a shared-memory ring.
template <int M, typename CT>
__global__ void __launch_bounds__(32)
k_group_P(const CT* __restrict__ tape, CT* __restrict__ gtape, int64_t ngroups, int G, int nsub,
          const int* __restrict__ only) {
    grid_dep_wait();
    using TP = Tape<M>;
    using SM = CarrySmem<M, CT, 4>;
    constexpr int MP4 = TP::MP4;
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kCS * (SM::STAGE + SM::NU) + 64 * sizeof(CT));
    const int64_t gi = blockIdx.x;
    if (gi >= ngroups) return;
    const int ng = (nsub + G - 1) / G;
    const int64_t b = gi / ng;
    if (only != nullptr && only[b] == 0) return;
    const int k0 = (int)(gi % ng) * G;
    const int n = min(G, nsub - k0);
    const int64_t base = b * nsub + k0;
    const int nst = (n + SM::CB - 1) / SM::CB;
    if (lane == 0) {
        for (int i = 0; i < kCS; ++i) mbar_init(&bars[i], 1);
        fence_mbar_init();
    }
    __syncwarp();
    auto issue = [&](int sg) {
        if (lane == 0 && sg < nst) {
            const int st = sg % kCS;
            const int cnt = min(SM::CB, n - sg * SM::CB);
            mbar_arrive_expect_tx(&bars[st], cnt * SM::SUB);
            tma_load_1d(smem + st * (SM::STAGE + SM::NU), tape + (base + sg * SM::CB) * TP::SIZE,
                        cnt * SM::SUB, &bars[st]);
        }
    };
    for (int i = 0; i < kCS; ++i) issue(i);
    CT col[M];
#pragma unroll
    for (int i = 0; i < M; ++i) col[i] = (lane == i) ? (CT)1 : (CT)0;
    for (int sg = 0; sg < nst; ++sg) {
        const int st = sg % kCS;
        mbar_wait(&bars[st], (uint32_t)((sg / kCS) & 1));
        const CT* sgb = reinterpret_cast<const CT*>(smem + st * (SM::STAGE + SM::NU));
        const int cnt = min(SM::CB, n - sg * SM::CB);
        for (int u = 0; u < cnt; ++u) {
            const CT* R = sgb + u * TP::SIZE + TP::R_ROW * MP4;
            CT nc[M];
#pragma unroll
            for (int i = 0; i < M; ++i) {
                CT row[MP4];
                load_vec<CT, MP4>(R + i * MP4, row);  // broadcast: all lanes read row i
                CT q0 = (CT)0, q1 = (CT)0;
#pragma unroll
                for (int c = 0; c < M; ++c) {
                    if (c & 1)
                        q1 = fma(row[c], col[c], q1);
                    else
                        q0 = fma(row[c], col[c], q0);
                }
                nc[i] = q0 + q1;
            }
#pragma unroll
            for (int i = 0; i < M; ++i) col[i] = nc[i];
        }
        __syncwarp();
        issue(sg + kCS);
    }
    if (lane < M) {
        CT* gt = gtape + gi * TP::SIZE;
        for (int i = 0; i < M; ++i) {
            gt[lane * MP4 + i] = col[i];                // W[lane] = column lane
            gt[(TP::R_ROW + i) * MP4 + lane] = col[i];  // R[i][lane]
        }
    }
}

// Group products as a tree: one CTA per group loads the G transition
// matrices (R rows) with bulk copies and multiplies neighbours level by level
// in shared memory (slot i <- slot i+s x slot i; later sub-chunks on the
// left), so a group costs log2(G) dependent mat-mats instead of G (k_group_P:
// one warp, 32 serial mat-mats per group, 83 us at config 4).  Lane j of a
// warp forms column j of a product from its own column of the right factor
// (registers) and broadcast rows of the left one; the result overwrites the
// right factor in place (column j is only read by lane j).
constexpr int kTreeWarps = 8;
template <int M, typename CT>
__global__ void __launch_bounds__(kTreeWarps * 32)
k_group_P_tree(const CT* __restrict__ tape, CT* __restrict__ gtape, int64_t ngroups, int G,
               int nsub, const int* __restrict__ only) {
    grid_dep_wait();
    using TP = Tape<M>;
    constexpr int MP4 = TP::MP4;
    constexpr int MAT = M * MP4;  // one matrix: M rows of MP4
    extern __shared__ __align__(128) unsigned char smem[];
    CT* slots = reinterpret_cast<CT*>(smem);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + (size_t)G * MAT * sizeof(CT));
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t gi = blockIdx.x;
    if (gi >= ngroups) return;
    const int ng = (nsub + G - 1) / G;
    const int64_t b = gi / ng;
    if (only != nullptr && only[b] == 0) return;
    const int k0 = (int)(gi % ng) * G;
    const int n = min(G, nsub - k0);
    const int64_t base = b * nsub + k0;
    if (tid == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
        mbar_arrive_expect_tx(bar, (uint32_t)(n * MAT * sizeof(CT)));
        for (int t = 0; t < n; ++t)
            tma_load_1d(slots + t * MAT, tape + (base + t) * TP::SIZE + TP::R_ROW * MP4,
                        (uint32_t)(MAT * sizeof(CT)), bar);
    }
    __syncthreads();
    mbar_wait(bar, 0);
    for (int st = 1; st < n; st *= 2) {
        const int npair = (n - st + 2 * st - 1) / (2 * st);  // pairs (i, i+st), i = 2*st*q
        for (int q = warp; q < npair; q += kTreeWarps) {
            CT* R = slots + (2 * st * q) * MAT;   // right factor, overwritten
            const CT* L = R + st * MAT;           // left factor
            if (lane < M) {
                CT col[MP4];
#pragma unroll
                for (int k = 0; k < MP4; ++k) col[k] = k < M ? R[k * MP4 + lane] : (CT)0;
                // outer-product order: one accumulator per row, a 4-wide slice
                // of every row of L per step -- 22 independent FMA chains
                CT out[M];
#pragma unroll
                for (int r = 0; r < M; ++r) out[r] = (CT)0;
#pragma unroll
                for (int kb = 0; kb < MP4; kb += 4) {
#pragma unroll
                    for (int r = 0; r < M; ++r) {
                        CT v[4];
                        load_vec<CT, 4>(L + r * MP4 + kb, v);
#pragma unroll
                        for (int d = 0; d < 4; ++d)
                            if (kb + d < M) out[r] = fma(v[d], col[kb + d], out[r]);
                    }
                }
#pragma unroll
                for (int r = 0; r < M; ++r) R[r * MP4 + lane] = out[r];
            }
        }
        __syncthreads();
    }
    CT* gt = gtape + gi * TP::SIZE;
    for (int idx = tid; idx < M * M; idx += blockDim.x) {
        const int r = idx / M, c = idx - r * M;
        const CT v = slots[r * MP4 + c];
        gt[(TP::R_ROW + r) * MP4 + c] = v;  // R[r][c] = P[r][c]
        gt[c * MP4 + r] = v;                // W[c] = column c
    }
}

// ============================================================================
// Lane-per-sub-chunk streaming kernels (apply fwd, adjoint zero-state, apply
// bwd).  One warp = 32 consecutive sub-chunks; lane l runs the recursion of
// sub-chunk g0+l.  Sub-chunks are full and uniformly strided (the C ABI picks
// Ls | T or pads T), so the inputs of one window (W rows of all 32 lanes) are
// ONE 2-D box of the view [B*nsub, Ls*M] (resp. [B*nsub, Ls]) and arrive with
// a single tensor TMA per operand; outputs leave the same way.  Box rows are
// padded to an odd number of 16-byte granules so the 32 lanes' vector reads of
// the same row offset hit distinct bank groups (the pad columns are the next
// window's first values, or zero-filled past the sub-chunk end).
// ============================================================================
template <typename IO, int M, bool TI>
struct LaneSmem {
    static constexpr int W = kLaneWin;
    static constexpr int SZ = (int)sizeof(IO);
    static constexpr int AROW = TI ? 0 : odd16_stride(W * M * SZ) / SZ;  // elements per lane
    static constexpr int XROW = odd16_stride(W * SZ) / SZ;
    static constexpr int A_BYTES = (32 * AROW * SZ + 127) / 128 * 128;
    static constexpr int X_BYTES = (32 * XROW * SZ + 127) / 128 * 128;
    static constexpr int STAGE = A_BYTES + X_BYTES;
    static constexpr int OUT = (32 * W * SZ + 127) / 128 * 128;
    static constexpr int BYTES = kLaneStages * STAGE + kOutStages * OUT + 128;
    static constexpr uint32_t TX = 32u * (AROW + XROW) * SZ;  // bytes landed per stage
};

struct LaneMaps {
    CUtensorMap A;  // [B*nsub, Ls*M] box {AROW, 32}   (unused for TI)
    CUtensorMap X;  // [B*nsub, Ls]   box {XROW, 32}   (e or g_s)
    CUtensorMap O;  // [B*nsub, Ls]   box {W, 32}      (s or g_e; unused by the lane passes)
    void* o;        // the same rows: lanes store their output windows directly
};

// A lane's W outputs of one window, stored straight from registers as 16-byte
// vectors: W consecutive values of the lane's own sub-chunk row are whole
// 32-byte sectors, and without an output box there is no async-proxy fence,
// warp sync or bulk-store wait per window (tools/micro/apply_lane.cu: the
// fence + syncs of a boxed TMA store cost ~50 cycles per sample at one warp
// per SM, more than the recursion itself at ~39).
template <typename IO, int W>
__device__ __forceinline__ void store_window(IO* dst, const IO (&v)[W]) {
    constexpr int V = 16 / (int)sizeof(IO);
    static_assert(W % V == 0, "windows are whole 16-byte vectors");
#pragma unroll
    for (int q = 0; q < W / V; ++q) {
        if constexpr (sizeof(IO) == 4)
            __stcs(reinterpret_cast<float4*>(dst) + q,
                   make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
        else
            __stcs(reinterpret_cast<double2*>(dst) + q, make_double2(v[2 * q], v[2 * q + 1]));
    }
}

// ---------------------------------------------------------------- fused refinement
constexpr float kDefectTol = 2e-5f;     // forward: relative to max |x| (samples of s)
constexpr float kDefectTolBwd = 2e-5f;  // adjoint: relative to max |lambda_0| (= |grad_e|)

static __device__ unsigned long long g_refined_sequences = 0;  // launched from scan_kernels.cu only


// Prologue of the fused re-apply: for every flagged sequence among the warp's
// 32 sub-chunks the warp runs the correction recurrence of k_refine_fwd/bwd
// (same arithmetic, same order) up to its own sub-chunks and hands each lane
// the correction of its carry-in state.  Returns false when no sequence of the
// warp is flagged (the warp then exits: its first-pass outputs stand).  sm:
// 32 + 32 M scratch values (the idle stage memory).
template <int M, typename CT>
__device__ bool refine_prologue(const RefineSrc<CT>& rf, bool fwd, const CT* __restrict__ X,
                                const ScanArgs& g, int64_t g0, CT* sm, CT (&corr)[M]) {
    using TP = Tape<M>;
    constexpr int MP4 = TP::MP4;
    const int lane = threadIdx.x & 31;
    const int64_t nsc = g.B * g.nsub;
    const int64_t glast = (g0 + 31 < nsc ? g0 + 31 : nsc - 1);
    const int64_t b0 = g0 / g.nsub, b1 = glast / g.nsub;
    CT* es = sm;
    CT* E = sm + 32;  // E[lane][i]: correction of the lane's carry-in state
#pragma unroll
    for (int i = 0; i < M; ++i) E[lane * M + i] = (CT)0;
    __syncwarp();
    bool any = false;
    const int r = lane < M ? lane : 0;
    for (int64_t b = b0; b <= b1; ++b) {
        const float dmax = __uint_as_float(rf.dstat[2 * b]);
        const float xmax = __uint_as_float(rf.dstat[2 * b + 1]);
        const bool bad = fwd ? dmax > kDefectTol * xmax
                             : (dmax > kDefectTolBwd * xmax ||
                                (rf.inherit != nullptr && rf.inherit[b] != 0));
        if (!bad) continue;
        any = true;
        const int64_t base = b * g.nsub;
        if (lane == 0) {
            if (fwd && rf.flags != nullptr) rf.flags[b] = 1;
            if (base >= g0) atomicAdd(&g_refined_sequences, 1ull);  // one warp per sequence
        }
        const int jlo = (int)(g0 > base ? g0 - base : 0);
        const int jhi = (int)(glast - base < g.nsub - 1 ? glast - base : g.nsub - 1);
        CT e = (CT)0;
        if (fwd) {
            for (int j = 0; j < jhi; ++j) {  // e_{j+1} = Phi_j e_j + d_j
                const CT* t = rf.tape + (base + j) * TP::SIZE;
                es[lane] = lane < M ? e : (CT)0;
                __syncwarp();
                CT w[MP4], ev[MP4];
                load_vec<CT, MP4>(t + (TP::R_ROW + r) * MP4, w);
                load_vec<CT, MP4>(es, ev);
                const CT d = lane < M ? rf.K[(base + j) * MP4 + r] - X[(base + j + 1) * MP4 + r]
                                      : (CT)0;
                const CT en = dot_rows<M, CT>(w, ev, d);
                __syncwarp();
                e = en;
                if (j + 1 >= jlo && lane < M) E[(base + j + 1 - g0) * M + lane] = e;
            }
        } else {
            for (int j = g.nsub - 1; j > jlo; --j) {  // e_{j-1} = Phi_j^T e_j + d_j
                const CT* t = rf.tape + (base + j) * TP::SIZE;
                es[lane] = lane < M ? e : (CT)0;
                __syncwarp();
                CT w[MP4], ev[MP4];
                load_vec<CT, MP4>(t + r * MP4, w);
                load_vec<CT, MP4>(es, ev);
                const CT d = lane < M ? rf.K[(base + j) * MP4 + r] - X[(base + j - 1) * MP4 + r]
                                      : (CT)0;
                const CT en = dot_rows<M, CT>(w, ev, d);
                __syncwarp();
                e = en;
                if (j - 1 <= jhi && lane < M) E[(base + j - 1 - g0) * M + lane] = e;
            }
        }
    }
    if (!any) return false;
    __syncwarp();
#pragma unroll
    for (int i = 0; i < M; ++i) corr[i] = E[lane * M + i];
    __syncwarp();  // the scratch is stage memory: read out before the first bulk copy
    return true;
}

// ---------------------------------------------------------------- apply fwd
// One lane re-runs the recursion of its sub-chunk from x_in.  The state lives
// in a register ring of MR = round_up(M, W) slots (slot p holds s at local
// step tau with tau mod MR == p); the unrolled body covers MR/W windows so
// every ring index is a compile-time constant.
template <typename IO, int M, bool TI, bool FR = false, bool RF = false>
__global__ void __launch_bounds__(32)
k_apply_fwd(const __grid_constant__ LaneMaps maps, const IO* __restrict__ ati_ptr,
            const IO* __restrict__ Xin, int* __restrict__ flag, IO* __restrict__ Xend,
            unsigned* __restrict__ dstat, const int* __restrict__ only, ScanArgs g,
            const FrameSrc<IO> fs, const RefineSrc<IO> rf) {
    grid_dep_wait();
    using S = LaneSmem<IO, M, TI || FR>;
    // the refinement ("auto") exists for fp32 I/O only
    static_assert(!RF || (32 + 32 * M) * S::SZ <= kLaneStages * S::STAGE, "refinement scratch");
    constexpr int W = S::W;
    constexpr int MR = (M + W - 1) / W * W;
    constexpr int WPB = MR / W;
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kLaneStages * S::STAGE + kOutStages * S::OUT);
    const int64_t nsc = g.B * g.nsub;
    const int g0 = blockIdx.x * 32;
    const int64_t gid = (int64_t)g0 + lane;
    const bool active = gid < nsc;
    const int nwin = g.Ls / W;
    // refinement pass: only warps holding a flagged sequence recompute (the
    // others would reproduce their first-pass outputs bit-for-bit)
    if (only != nullptr && !__any_sync(0xffffffffu, active && only[gid / g.nsub] != 0)) return;
    // RF: the re-apply launch of precision "auto" with the refine step folded in
    IO corr[M];
    if constexpr (RF) {
        if (!refine_prologue<M, IO>(rf, true, Xin, g, g0, reinterpret_cast<IO*>(smem), corr))
            return;
    }

    if (lane == 0) {
        if (!TI && !FR) prefetch_tmap(&maps.A);
        prefetch_tmap(&maps.X);

        for (int st = 0; st < kLaneStages; ++st) mbar_init(&bars[st], 1);
        fence_mbar_init();
    }
    __syncwarp();
    auto issue = [&](int k) {
        if (k < nwin && lane == 0) {
            const int st = k % kLaneStages;
            unsigned char* base = smem + st * S::STAGE;
            mbar_arrive_expect_tx(&bars[st], S::TX);
            if (!TI && !FR) tma_load_2d(base, &maps.A, k * W * M, g0, &bars[st]);
            tma_load_2d(base + S::A_BYTES, &maps.X, k * W, g0, &bars[st]);
        }
    };
#pragma unroll
    for (int k = 0; k < kLaneStages; ++k) issue(k);

    IO ati[M];
    if (TI) {
        const int64_t b = active ? gid / g.nsub : 0;
#pragma unroll
        for (int i = 0; i < M; ++i) ati[i] = active ? ati_ptr[b * M + i] : (IO)0;
    }
    IO R[MR];
#pragma unroll
    for (int p = 0; p < MR; ++p) R[p] = (IO)0;
#pragma unroll
    for (int i = 0; i < M; ++i) {
        if constexpr (RF)
            R[MR - 1 - i] = active ? Xin[gid * Tape<M>::MP4 + i] + corr[i] : (IO)0;
        else
            R[MR - 1 - i] = active ? Xin[gid * Tape<M>::MP4 + i] : (IO)0;
    }
    bool finite = true;
    // frame-rate rows (FR): the lane walks its sub-chunk forward in time
    const int64_t fb_b = active ? gid / g.nsub : 0;
    const IO inv_hop = FR ? (IO)1 / (IO)fs.hop : (IO)0;
    FrameCursor<IO, FR ? M : 1> cur;
    const int64_t ft0 = active ? (gid % g.nsub) * (int64_t)g.Ls : 0;

    for (int kb = 0; kb < nwin; kb += WPB) {
#pragma unroll
        for (int w = 0; w < WPB; ++w) {
            const int k = kb + w;
            if (k < nwin) {
                const int st = k % kLaneStages;
                mbar_wait(&bars[st], (uint32_t)((k / kLaneStages) & 1));
                const unsigned char* base = smem + st * S::STAGE;
                const IO* Ar = reinterpret_cast<const IO*>(base) + lane * S::AROW;
                const IO* er = reinterpret_cast<const IO*>(base + S::A_BYTES) + lane * S::XROW;
                IO ev[W], ov[W];
#pragma unroll
                for (int u = 0; u < W; ++u) ev[u] = er[u];
                if constexpr (FR) cur.window(fs, fb_b, ft0 + (int64_t)k * W);
#pragma unroll
                for (int u = 0; u < W; ++u) {
                    const int pos = w * W + u;  // compile-time after unrolling
                    IO a[M];
                    if constexpr (TI) {
#pragma unroll
                        for (int i = 0; i < M; ++i) a[i] = ati[i];
                    } else if constexpr (FR) {
                        cur.row(fs, inv_hop, u, a);
                    } else {
                        load_row_at<IO, M>(Ar + u * M, a, (lane * S::AROW + u * M) * S::SZ);
                    }
                    IO p0 = (IO)0, p1 = (IO)0, p2 = (IO)0, p3 = (IO)0;
#pragma unroll
                    for (int i = M; i >= 2; --i) {
                        const IO x = R[(pos - i + 2 * MR) % MR];
                        switch (i & 3) {
                            case 0: p0 = fma(a[i - 1], x, p0); break;
                            case 1: p1 = fma(a[i - 1], x, p1); break;
                            case 2: p2 = fma(a[i - 1], x, p2); break;
                            default: p3 = fma(a[i - 1], x, p3); break;
                        }
                    }
                    const IO v =
                        fma(-a[0], R[(pos - 1 + MR) % MR], ev[u] - ((p0 + p1) + (p2 + p3)));
                    R[pos % MR] = v;
                    ov[u] = v;
                    finite &= is_finite_val(v);
                }
                TVLP_ASSERT(!active || (gid < nsc && k * W + W <= g.Ls));
                if (active)
                    store_window<IO, W>(static_cast<IO*>(maps.o) + gid * (int64_t)g.Ls + k * W, ov);
                __syncwarp();  // every lane is done with the stage: refill it
                issue(k + kLaneStages);
            }
        }
    }
    if (flag != nullptr) {
        // a non-finite output means non-finite input or overflow; the host
        // tells them apart (overflow of an unstable filter is legitimate).
        const unsigned bad = __ballot_sync(0xffffffffu, active && !finite);
        if (bad && lane == 0) atomicOr(flag, 1);
    }
    if (!RF && Xend != nullptr && active) {
        // end state x[i] = s(t1 - i): the defect check compares it with the
        // carry's x_in of the next sub-chunk
        IO tmp[MR];
#pragma unroll
        for (int p = 0; p < MR; ++p) tmp[p] = R[p];
        const int last = (g.Ls - 1) % MR;
        const bool has_next = (gid % g.nsub) + 1 < g.nsub;
        float dm = 0.f, xm = 0.f;
        for (int i = 0; i < M; ++i) {
            const IO v = tmp[(last - i + MR) % MR];
            Xend[gid * Tape<M>::MP4 + i] = v;
            if (has_next) {
                const IO xn = Xin[(gid + 1) * Tape<M>::MP4 + i];
                dm = fmaxf(dm, (float)fabs(v - xn));
                xm = fmaxf(xm, fmaxf((float)fabs(v), (float)fabs(xn)));
            }
        }
        if (has_next && dstat != nullptr) {
            const int64_t b = gid / g.nsub;
            if (!(dm == dm)) dm = __int_as_float(0x7f800000);  // NaN -> +inf: always refine
            atomicMax(&dstat[2 * b], __float_as_uint(dm));
            atomicMax(&dstat[2 * b + 1], __float_as_uint(xm));
        }
    }
}

// ---------------------------------------------------------------- adjoint
// MODE 0: zero-state adjoint per sub-chunk -> Nu.  MODE 1: apply from Mu,
// write g_e.  Reverse time; row A[t] is used at step t:
//   lambda += u0 g_s(t);  g_e(t) = lambda_0;  lambda = C(t)^T lambda.
// The transposed-state update shifts lambda inside its FMAs (no moves).
template <typename IO, int M, bool TI, int MODE, bool FR = false, bool RF = false>
__global__ void __launch_bounds__(32)
k_adjoint(const __grid_constant__ LaneMaps maps, const IO* __restrict__ ati_ptr,
          const IO* __restrict__ Mu, IO* __restrict__ Nu, unsigned* __restrict__ dstat,
          const int* __restrict__ only, ScanArgs g, const FrameSrc<IO> fs,
          const RefineSrc<IO> rf) {
    grid_dep_wait();
    using S = LaneSmem<IO, M, TI || FR>;
    // the refinement ("auto") exists for fp32 I/O only
    static_assert(!RF || (32 + 32 * M) * S::SZ <= kLaneStages * S::STAGE, "refinement scratch");
    constexpr int W = S::W;
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kLaneStages * S::STAGE + kOutStages * S::OUT);
    const int64_t nsc = g.B * g.nsub;
    const int g0 = blockIdx.x * 32;
    const int64_t gid = (int64_t)g0 + lane;
    const bool active = gid < nsc;
    const int nwin = g.Ls / W;
    if (only != nullptr && !__any_sync(0xffffffffu, active && only[gid / g.nsub] != 0)) return;
    IO corr[M];
    if constexpr (RF) {
        static_assert(MODE == 1, "the refinement re-applies the adjoint from Mu");
        if (!refine_prologue<M, IO>(rf, false, Mu, g, g0, reinterpret_cast<IO*>(smem), corr))
            return;
    }

    if (lane == 0) {
        if (!TI && !FR) prefetch_tmap(&maps.A);
        prefetch_tmap(&maps.X);

        for (int st = 0; st < kLaneStages; ++st) mbar_init(&bars[st], 1);
        fence_mbar_init();
    }
    __syncwarp();
    // reverse window k covers rows [Ls-(k+1)W, Ls-kW)
    auto issue = [&](int k) {
        if (k < nwin && lane == 0) {
            const int st = k % kLaneStages;
            unsigned char* base = smem + st * S::STAGE;
            const int wr = nwin - 1 - k;
            mbar_arrive_expect_tx(&bars[st], S::TX);
            if (!TI && !FR) tma_load_2d(base, &maps.A, wr * W * M, g0, &bars[st]);
            tma_load_2d(base + S::A_BYTES, &maps.X, wr * W, g0, &bars[st]);
        }
    };
#pragma unroll
    for (int k = 0; k < kLaneStages; ++k) issue(k);

    IO ati[M];
    if (TI) {
        const int64_t b = active ? gid / g.nsub : 0;
#pragma unroll
        for (int i = 0; i < M; ++i) ati[i] = active ? ati_ptr[b * M + i] : (IO)0;
    }
    IO lam[M];
#pragma unroll
    for (int i = 0; i < M; ++i) {
        if constexpr (RF)
            lam[i] = active ? Mu[gid * Tape<M>::MP4 + i] + corr[i] : (IO)0;
        else
            lam[i] = (MODE == 1 && active) ? Mu[gid * Tape<M>::MP4 + i] : (IO)0;
    }
    // frame-rate rows (FR): the lane walks its sub-chunk backward in time
    const int64_t fb_b = active ? gid / g.nsub : 0;
    const IO inv_hop = FR ? (IO)1 / (IO)fs.hop : (IO)0;
    FrameCursor<IO, FR ? M : 1> cur;
    const int64_t ft0 = active ? (gid % g.nsub) * (int64_t)g.Ls : 0;

    float gmx = 0.f;  // MODE 1: max |grad_e| over the lane's samples (defect scale)
    for (int k = 0; k < nwin; ++k) {
        const int st = k % kLaneStages;
        mbar_wait(&bars[st], (uint32_t)((k / kLaneStages) & 1));
        const unsigned char* base = smem + st * S::STAGE;
        const IO* Ar = reinterpret_cast<const IO*>(base) + lane * S::AROW;
        const IO* xr = reinterpret_cast<const IO*>(base + S::A_BYTES) + lane * S::XROW;
        IO gv[W], ov[W];
#pragma unroll
        for (int u = 0; u < W; ++u) gv[u] = xr[u];
        if constexpr (FR) cur.window(fs, fb_b, ft0 + (int64_t)(nwin - 1 - k) * W);
#pragma unroll
        for (int u = W - 1; u >= 0; --u) {
            IO a[M];
            if constexpr (TI) {
#pragma unroll
                for (int i = 0; i < M; ++i) a[i] = ati[i];
            } else if constexpr (FR) {
                cur.row(fs, inv_hop, u, a);
            } else {
                load_row_at<IO, M>(Ar + u * M, a, (lane * S::AROW + u * M) * S::SZ);
            }
            const IO l0 = lam[0] + gv[u];
            ov[u] = l0;
            if (MODE == 1) gmx = fmaxf(gmx, (float)fabs(l0));
#pragma unroll
            for (int i = 0; i < M - 1; ++i) lam[i] = fma(-a[i], l0, lam[i + 1]);
            lam[M - 1] = -a[M - 1] * l0;
        }
        TVLP_ASSERT(!(MODE == 1 && active) || (gid < nsc && (nwin - k) * W <= g.Ls));
        if (MODE == 1 && active)
            store_window<IO, W>(static_cast<IO*>(maps.o) + gid * (int64_t)g.Ls + (nwin - 1 - k) * W,
                                ov);
        __syncwarp();  // every lane is done with the stage: refill it
        issue(k + kLaneStages);
    }
    // MODE 0: Nu = zero-state carry-out.  MODE 1: Nu (if given) = the carry-out
    // C(t0)^T lambda(t0) obtained from Mu, which the defect check compares with
    // the carry chain's Mu of the previous sub-chunk.
    if (active && Nu != nullptr) {
#pragma unroll
        for (int i = 0; i < M; ++i) Nu[gid * Tape<M>::MP4 + i] = lam[i];
        if (MODE == 1 && dstat != nullptr && (gid % g.nsub) > 0) {
            // scale: |grad_e| = |lambda_0|, over the sub-chunk's samples and the
            // boundary.  The other adjoint components are coefficient-weighted
            // sums of future grad_e and can be orders larger on resonant rows,
            // while a defect in component i reaches grad_e unamplified i steps
            // later (it shifts into lambda_0); the parity metric is relative to
            // the sequence's max |grad_e|, which the boundary value alone can
            // understate by orders (false flags on loss gradients).
            float dm = 0.f;
            const IO mp0 = Mu[(gid - 1) * Tape<M>::MP4];
            const float xm = fmaxf(gmx, fmaxf((float)fabs(lam[0]), (float)fabs(mp0)));
#pragma unroll
            for (int i = 0; i < M; ++i) {
                const IO mp = Mu[(gid - 1) * Tape<M>::MP4 + i];
                dm = fmaxf(dm, (float)fabs(lam[i] - mp));
            }
            const int64_t b = gid / g.nsub;
            if (!(dm == dm)) dm = __int_as_float(0x7f800000);
            atomicMax(&dstat[2 * b], __float_as_uint(dm));
            atomicMax(&dstat[2 * b + 1], __float_as_uint(xm));
        }
    }
}

// ---------------------------------------------------------------- refinement
// A-posteriori check of the fp32-chain carries (precision "auto").  For a
// sequence, d_j = Xend_j - Xin_{j+1} is the boundary defect between the state
// the apply pass actually reached at the end of sub-chunk j (a plain fp32
// recursion from Xin_j) and the carry's prediction for sub-chunk j+1.  With
// exact carries d_j is fp32 rounding noise.  If max|d| > tau * max|x| the
// carries are corrected by e_{j+1} = Phi_j e_j + d_j (e_0 = 0, Xin += e): the
// correction is linear and small, so the fp32 Phi_j (relative error ~1e-5
// after cancellation) contracts the error by ~1e-4 per pass.
// (kDefectTol / kDefectTolBwd are defined with the fused refinement prologue
// above the apply kernels)

template <typename CT>
__device__ __forceinline__ CT warp_max(CT v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}


template <int M, typename CT>
__global__ void __launch_bounds__(32)
k_refine_fwd(const CT* __restrict__ tape, CT* __restrict__ Xin, const CT* __restrict__ Xend,
             const unsigned* __restrict__ dstat, int* __restrict__ flags, int nsub, int64_t B) {
    grid_dep_wait();
    using TP = Tape<M>;
    constexpr int MP4 = TP::MP4;
    __shared__ __align__(16) CT es[32];
    const int lane = threadIdx.x;
    const int64_t b = blockIdx.x;
    if (b >= B) return;
    const float dmax = __uint_as_float(dstat[2 * b]), xmax = __uint_as_float(dstat[2 * b + 1]);
    const bool bad = dmax > kDefectTol * xmax;
    if (lane == 0) {
        flags[b] = bad ? 1 : 0;
        if (bad) atomicAdd(&g_refined_sequences, 1ull);
    }
    if (!bad) return;
    const int64_t base = b * nsub;
    const int r = lane < M ? lane : 0;
    CT e = (CT)0;  // correction of Xin_j, component r
    for (int j = 0; j + 1 < nsub; ++j) {
        const CT* t = tape + (base + j) * TP::SIZE;
        es[lane] = lane < M ? e : (CT)0;
        __syncwarp();
        CT w[MP4], ev[MP4];
        load_vec<CT, MP4>(t + (TP::R_ROW + r) * MP4, w);
        load_vec<CT, MP4>(es, ev);
        const CT d = lane < M ? Xend[(base + j) * MP4 + r] - Xin[(base + j + 1) * MP4 + r] : (CT)0;
        const CT en = dot_rows<M, CT>(w, ev, d);
        __syncwarp();
        e = en;
        if (lane < M) Xin[(base + j + 1) * MP4 + r] += e;
    }
}

// Adjoint analogue: K_j = carry-out of sub-chunk j computed by the apply pass
// from Mu_j; d_j = K_j - Mu_{j-1};  e_{j-1} = Phi_j^T e_j + d_j (e_last = 0).
template <int M, typename CT>
__global__ void __launch_bounds__(32)
k_refine_bwd(const CT* __restrict__ tape, CT* __restrict__ Mu, const CT* __restrict__ K,
             const unsigned* __restrict__ dstat, int* __restrict__ flags, int nsub, int64_t B,
             const int* __restrict__ fflags) {
    grid_dep_wait();
    using TP = Tape<M>;
    constexpr int MP4 = TP::MP4;
    __shared__ __align__(16) CT es[32];
    const int lane = threadIdx.x;
    const int64_t b = blockIdx.x;
    if (b >= B) return;
    const float dmax = __uint_as_float(dstat[2 * b]), xmax = __uint_as_float(dstat[2 * b + 1]);
    // a sequence whose forward carries needed refinement has ill-conditioned
    // transition matrices; its adjoint carries are refined too (defects of the
    // adjoint can be amplified by the resonance before they reach grad_e)
    const bool bad = dmax > kDefectTolBwd * xmax || (fflags != nullptr && fflags[b] != 0);
    if (lane == 0) {
        flags[b] = bad ? 1 : 0;
        if (bad) atomicAdd(&g_refined_sequences, 1ull);
    }
    if (!bad) return;
    const int64_t base = b * nsub;
    const int r = lane < M ? lane : 0;
    CT e = (CT)0;
    for (int j = nsub - 1; j >= 1; --j) {
        const CT* t = tape + (base + j) * TP::SIZE;
        es[lane] = lane < M ? e : (CT)0;
        __syncwarp();
        CT w[MP4], ev[MP4];
        load_vec<CT, MP4>(t + r * MP4, w);
        load_vec<CT, MP4>(es, ev);
        const CT d = lane < M ? K[(base + j) * MP4 + r] - Mu[(base + j - 1) * MP4 + r] : (CT)0;
        const CT en = dot_rows<M, CT>(w, ev, d);
        __syncwarp();
        e = en;
        if (lane < M) Mu[(base + j - 1) * MP4 + r] += e;
    }
}

// ---------------------------------------------------------------- hierarchical refinement helpers
// Per-sequence decision of precision "auto" (the long-sequence path; the
// short path decides inside k_refine_fwd/bwd).
static __global__ void k_refine_decide(const unsigned* __restrict__ dstat, int* __restrict__ flags,
                                const int* __restrict__ inherit, float tol, int64_t B) {
    grid_dep_wait();
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    const float d = __uint_as_float(dstat[2 * b]), x = __uint_as_float(dstat[2 * b + 1]);
    const bool bad = d > tol * x || (inherit != nullptr && inherit[b] != 0);
    flags[b] = bad ? 1 : 0;
    if (bad) atomicAdd(&g_refined_sequences, 1ull);
}

// D[j] = forcing of the correction recurrence.  fwd: Xend[j] - Xin[j+1]
// (zero for the last sub-chunk); bwd: K[j] - Mu[j-1] (zero for j = 0).
template <typename CT>
__global__ void k_defects(const CT* __restrict__ P, const CT* __restrict__ Q, CT* __restrict__ D,
                          int nsub, int mp4, int M, bool fwd, const int* __restrict__ only,
                          int64_t B) {
    grid_dep_wait();
    const int64_t n = B * (int64_t)nsub * mp4;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(i % mp4);
        const int64_t g = i / mp4;
        const int j = (int)(g % nsub);
        const int64_t b = g / nsub;
        CT v = (CT)0;
        if (c < M && (only == nullptr || only[b])) {
            if (fwd && j + 1 < nsub) v = P[g * mp4 + c] - Q[(g + 1) * mp4 + c];
            if (!fwd && j > 0) v = P[g * mp4 + c] - Q[(g - 1) * mp4 + c];
        }
        D[i] = v;
    }
}

template <typename CT>
__global__ void k_add_rows(CT* __restrict__ X, const CT* __restrict__ E, int nsub, int mp4,
                           const int* __restrict__ only, int64_t B) {
    grid_dep_wait();
    const int64_t n = B * (int64_t)nsub * mp4;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = i / ((int64_t)nsub * mp4);
        if (only == nullptr || only[b]) X[i] += E[i];
    }
}

// ---------------------------------------------------------------- g_A
// g_A[b,t,c] = -g_e[b,t] * s(t-c-1), s(<0) from zi (lpc.py:138-149, 172).
// A block stages s[tlo-M, tlo+RT) and g_e[tlo, tlo+RT) in shared memory and
// writes its RT*M contiguous outputs with coalesced stores.
template <typename IO, int M>
__global__ void __launch_bounds__(256)
k_grad_A(const IO* __restrict__ ge, const IO* __restrict__ s, const IO* __restrict__ zi,
         IO* __restrict__ gA, int64_t T) {
    grid_dep_wait();
    constexpr int RT = 256;
    __shared__ IO sh_s[RT + M];
    __shared__ IO sh_g[RT];
    const int64_t b = blockIdx.y;
    const int64_t tlo = (int64_t)blockIdx.x * RT;
    const int rows = (int)(int64_t)min((int64_t)RT, T - tlo);
    const IO* sb = s + b * T;
    for (int i = threadIdx.x; i < RT + M; i += 256) {
        const int64_t tau = tlo - M + i;
        IO v = (IO)0;
        if (tau >= 0) {
            if (tau < T) v = sb[tau];
        } else if (zi) {
            v = zi[b * M + (-tau - 1)];
        }
        sh_s[i] = v;
    }
    for (int i = threadIdx.x; i < RT; i += 256) sh_g[i] = i < rows ? ge[b * T + tlo + i] : (IO)0;
    __syncthreads();
    IO* out = gA + (b * T + tlo) * M;
    const int n = rows * M;
    if constexpr (sizeof(IO) == 4 && TVLP_GRAD_A_VEC) {
        // 16-byte stores: the block's output span starts 16B-aligned
        // (T % 4 == 0 and RT * M * 4 % 16 == 0); rows*M % 4 == 0 as rows % 4 == 0
        for (int q = threadIdx.x * 4; q < n; q += 256 * 4) {
            float r4[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int idx = q + e;
                const int r = idx / M;
                const int c = idx - r * M;
                r4[e] = (-sh_g[r]) * sh_s[M + r - c - 1];
            }
            *reinterpret_cast<float4*>(out + q) = make_float4(r4[0], r4[1], r4[2], r4[3]);
        }
    } else {
        for (int idx = threadIdx.x; idx < n; idx += 256) {
            const int r = idx / M;
            const int c = idx - r * M;
            out[idx] = (-sh_g[r]) * sh_s[M + r - c - 1];
        }
    }
}

// g_a[b,c] = -sum_t s(t-c-1) g_e(t): partial sums per (b, chunk), then a
// fixed-order sum over chunks (deterministic).
template <typename IO>
__global__ void k_grad_a_partial(const IO* __restrict__ ge, const IO* __restrict__ s,
                                 const IO* __restrict__ zi, IO* __restrict__ part,
                                 int64_t T, int M, int nchunk) {
    grid_dep_wait();
    const int64_t b = blockIdx.y;
    const int chunk = blockIdx.x;
    const int64_t len = (T + nchunk - 1) / nchunk;
    const int64_t lo = chunk * len, hi = min(T, lo + len);
    __shared__ double red[32][33];
    for (int c0 = 0; c0 < M; c0 += 32) {
        const int c = c0 + (threadIdx.x & 31);
        double acc = 0.0;
        if (c < M) {
            for (int64_t t = lo + (threadIdx.x >> 5); t < hi; t += blockDim.x >> 5) {
                const int64_t src = t - c - 1;
                IO lag;
                if (src >= 0)
                    lag = s[b * T + src];
                else
                    lag = zi ? zi[b * M + (c - t)] : (IO)0;
                acc += (double)(lag * ge[b * T + t]);
            }
        }
        red[threadIdx.x >> 5][threadIdx.x & 31] = acc;
        __syncthreads();
        if (threadIdx.x < 32 && c0 + (int)threadIdx.x < M) {
            double tot = 0.0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w][threadIdx.x];
            part[((int64_t)b * nchunk + chunk) * M + c0 + threadIdx.x] = (IO)tot;
        }
        __syncthreads();
    }
}

template <typename IO>
__global__ void k_grad_a_final(const IO* __restrict__ part, IO* __restrict__ ga, int64_t B, int M,
                               int nchunk) {
    grid_dep_wait();
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= B * M) return;
    const int64_t b = idx / M;
    const int c = (int)(idx % M);
    double tot = 0.0;
    for (int k = 0; k < nchunk; ++k) tot += (double)part[(b * nchunk + k) * M + c];
    ga[idx] = (IO)(-tot);
}

// ---------------------------------------------------------------- frame-rate helpers
// A[b, t, :] for t < T (rows past Tv zero), padded to Mp columns.
template <typename IO, int M>
__global__ void __launch_bounds__(256)
k_upsample(const FrameSrc<IO> fs, IO* __restrict__ A, int64_t B, int64_t T) {
    grid_dep_wait();
    const IO inv_hop = (IO)1 / (IO)fs.hop;
    const int64_t n = B * T;
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x)
        frame_row_store<IO, M>(fs, r / T, r % T, inv_hop, A + r * M);
}

// grad_frames[b, f, c] = sum_{t: f0(t)=f} (1-w) gA(t,c) + sum_{t: f1(t)=f} w gA(t,c),
// gA(t, c) = -grad_e(t) s(t-1-c), s(<0) = zi (params.py:135-145 over lpc.py:172).
// One CTA per (sequence, kFramesPerCta consecutive frames).  The weighted
// adjoints p0(t) = (1-w)(-grad_e), p1(t) = w(-grad_e) and s over the frames'
// support (plus lags) are staged in shared memory; thread (frame, 4 lags,
// part) runs one interval with a sliding register window over s (one shared
// load of p and one of s per 4 FMAs), the two parts are added at the end.
constexpr int kFramesPerCta = 8;
template <typename IO>
__global__ void __launch_bounds__(kFramesPerCta * 16)
k_grad_frames(const FrameSrc<IO> fs, const IO* __restrict__ ge, const IO* __restrict__ s,
              const IO* __restrict__ zi, int Mzi, IO* __restrict__ gF, int64_t T) {
    grid_dep_wait();
    extern __shared__ __align__(16) unsigned char gf_smem[];
    __shared__ IO red[kFramesPerCta][32];
    const int64_t b = blockIdx.y;
    const int64_t fbase = (int64_t)blockIdx.x * kFramesPerCta;
    const int hop = fs.hop;
    constexpr int LAG = 32;  // staged lags (>= Mf)
    // support of frames fbase..fbase+K-1: t in [(fbase-1) hop, (fbase+K) hop)
    const int64_t tlo = (fbase - 1) * hop;
    const int span = (kFramesPerCta + 1) * hop;
    // -grad_e(t), t = tlo + i (the interval weights (1 - w), w are applied in
    // the reduction: two staged arrays instead of three keep the grid in one
    // wave -- 12 CTAs per SM instead of 8 at hop 240)
    IO* gn = reinterpret_cast<IO*>(gf_smem);
    IO* ss = gn + span;                        // s(tlo - LAG + i)
    const IO* gb = ge + b * T;
    const IO* sb = s + b * T;
    const IO inv_hop = (IO)1 / (IO)hop;
    // staging: 8 independent global loads in flight per thread and pass
    constexpr int U = 8;
    for (int i0 = threadIdx.x; i0 < span + LAG; i0 += U * blockDim.x) {
        IO v[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const int i = i0 + j * blockDim.x;
            const int64_t u = tlo - LAG + i;  // s index
            v[j] = (IO)0;
            if (i < span + LAG) {
                if (u >= 0)
                    v[j] = u < fs.Tv ? sb[u] : (IO)0;
                else if (zi != nullptr && -u - 1 < fs.Mf)
                    v[j] = zi[b * Mzi + (-u - 1)];
            }
        }
#pragma unroll
        for (int j = 0; j < U; ++j)
            if (i0 + j * (int)blockDim.x < span + LAG) ss[i0 + j * blockDim.x] = v[j];
    }
    for (int i0 = threadIdx.x; i0 < span; i0 += U * blockDim.x) {
        IO v[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const int i = i0 + j * blockDim.x;
            const int64_t t = tlo + i;
            v[j] = (i < span && t >= 0 && t < fs.Tv) ? -gb[t] : (IO)0;
        }
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const int i = i0 + j * blockDim.x;
            if (i < span) gn[i] = v[j];
        }
    }
    __syncthreads();
    const int k = threadIdx.x >> 4;          // frame in the CTA
    const int c0 = ((threadIdx.x >> 1) & 7) * 4;  // first of 4 lags
    const int part = threadIdx.x & 1;        // 0: f0(t) = f, 1: f1(t) = f
    const int64_t f = fbase + k;
    // part 0: t in [f hop, (f+1) hop) -> local i = (k+1) hop + r, weight p0
    // part 1: t in [(f-1) hop, f hop) -> local i = k hop + r, weight p1 (f >= 1)
    const int i0 = (k + 1 - part) * hop;
    // the interval's weight of frame f: part 0 (its own interval, frame f):
    // 1 - w, w = r / hop (0 in the held last interval); part 1 (interval of
    // frame f - 1, never the last): w -- the same products as staging them
    const bool held = part == 0 && !(f < fs.nF - 1);
    IO acc[4] = {(IO)0, (IO)0, (IO)0, (IO)0};
    if (f < fs.nF && (part == 0 || f >= 1)) {
        // x[j] = s(t - 1 - c0 - j) at the current t (ss index LAG + i - 1 - c0 - j)
        const IO* sp = ss + LAG + i0 - 1 - c0;
        IO x0 = sp[0], x1 = sp[-1], x2 = sp[-2], x3 = sp[-3];
#pragma unroll 4
        for (int r = 0; r < hop; ++r) {
            const IO w = held ? (IO)0 : (IO)r * inv_hop;
            const IO pv = (part == 0 ? (IO)1 - w : w) * gn[i0 + r];
            acc[0] = fma(pv, x0, acc[0]);
            acc[1] = fma(pv, x1, acc[1]);
            acc[2] = fma(pv, x2, acc[2]);
            acc[3] = fma(pv, x3, acc[3]);
            x3 = x2;
            x2 = x1;
            x1 = x0;
            x0 = sp[r + 1];
        }
    }
    if (part == 1) {
#pragma unroll
        for (int j = 0; j < 4; ++j) red[k][c0 + j] = acc[j];
    }
    __syncthreads();
    if (part == 0 && f < fs.nF) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (c0 + j < fs.Mf) gF[(b * fs.nF + f) * fs.Mf + c0 + j] = acc[j] + red[k][c0 + j];
    }
}

}  // namespace tvlp
