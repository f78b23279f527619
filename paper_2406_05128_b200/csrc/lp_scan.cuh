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
// Preconditions (enforced by the C ABI, which pads otherwise): T % 4 == 0,
// Ls % lcm(M,4,8) == 0, all pointers 16-byte aligned.
#pragma once
#include "common.cuh"

namespace tvlp {

constexpr int kLaneWin = 8;     // rows per TMA window in the lane-per-sub-chunk kernels
constexpr int kLaneStages = 3;  // input stages (per warp)
constexpr int kOutStages = 2;   // output staging slots

template <int M>
struct Geo {
    static constexpr int WR = clcm(M, 4);          // basis window rows (multiple of M)
    static constexpr int LsUnit = clcm(WR, kLaneWin);  // Ls granularity
};

struct ScanArgs {
    int64_t B, T;
    int Ls, nsub;
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
            fence_proxy_async();
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
            fence_proxy_async();
            issue(k + NSTB);
        }
    }

    // final state x[i] = s(t1 - i) = R[(len-1-i) mod M]; runtime rotation.
    if (lane <= M) {
        ACC tmp[M];
#pragma unroll
        for (int p = 0; p < M; ++p) tmp[p] = R[p];
        IO* out = PhiZ + (gid * (M + 1) + lane) * M;
        const int last = (len - 1) % M;
        for (int i = 0; i < M; ++i) out[i] = (IO)tmp[(last - i + M) % M];
    }
}

// ============================================================================
// Carry kernels: one warp per sequence, lane r holds component r.  The chain
// is latency-bound (one M x M mat-vec per sub-chunk), so the next sub-chunks'
// matrix rows are prefetched into registers (distance kPF) while the current
// mat-vec runs; the state is broadcast through shared memory.
// ============================================================================
constexpr int kPF = 4;

template <int M, typename ACC, typename CT>
__global__ void __launch_bounds__(128)
k_carry_fwd(const CT* __restrict__ PhiZ, const CT* __restrict__ zi, CT* __restrict__ Xin,
            ScanArgs g) {
    __shared__ ACC xs[4][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t b = (int64_t)blockIdx.x * 4 + warp;
    if (b >= g.B) return;
    const int r = lane < M ? lane : 0;
    ACC x = (ACC)0;
    if (zi != nullptr && lane < M) x = (ACC)zi[b * M + lane];
    const int64_t g0 = b * g.nsub;
    const int nstep = g.nsub - 1;
    // ring of prefetched rows: w[k][c] = Phi_j[r][c] (c < M), w[k][M] = z_j[r]
    CT w[kPF][M + 1];
#pragma unroll
    for (int k = 0; k < kPF; ++k) {
        if (k < nstep) {
            const CT* W = PhiZ + (g0 + k) * (M + 1) * M;
#pragma unroll
            for (int c = 0; c <= M; ++c) w[k][c] = W[c * M + r];
        }
    }
    for (int j0 = 0; j0 <= nstep; j0 += kPF) {
#pragma unroll
        for (int k = 0; k < kPF; ++k) {
            const int j = j0 + k;
            if (j <= nstep) {
                if (lane < M) Xin[(g0 + j) * M + lane] = (CT)x;
                if (j < nstep) {
                    xs[warp][lane] = x;
                    __syncwarp();
                    ACC q0 = (ACC)w[k][M], q1 = (ACC)0, q2 = (ACC)0, q3 = (ACC)0;
#pragma unroll
                    for (int c = 0; c < M; ++c) {
                        const ACC xc = xs[warp][c];
                        switch (c & 3) {
                            case 0: q0 = fma((ACC)w[k][c], xc, q0); break;
                            case 1: q1 = fma((ACC)w[k][c], xc, q1); break;
                            case 2: q2 = fma((ACC)w[k][c], xc, q2); break;
                            default: q3 = fma((ACC)w[k][c], xc, q3); break;
                        }
                    }
                    __syncwarp();
                    if (lane < M) x = (q0 + q1) + (q2 + q3);
                    const int jn = j + kPF;
                    if (jn < nstep) {
                        const CT* W = PhiZ + (g0 + jn) * (M + 1) * M;
#pragma unroll
                        for (int c = 0; c <= M; ++c) w[k][c] = W[c * M + r];
                    }
                }
            }
        }
    }
}

// mu(j-1) = Phi_j^T mu(j) + nu_j ;  Mu[j] = carry into sub-chunk j from the right.
template <int M, typename ACC, typename CT>
__global__ void __launch_bounds__(128)
k_carry_bwd(const CT* __restrict__ PhiZ, const CT* __restrict__ Nu, CT* __restrict__ Mu,
            ScanArgs g) {
    __shared__ ACC ms[4][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t b = (int64_t)blockIdx.x * 4 + warp;
    if (b >= g.B) return;
    const int r = lane < M ? lane : 0;
    ACC mu = (ACC)0;
    const int64_t g0 = b * g.nsub;
    const int nstep = g.nsub - 1;  // steps j = nsub-1 .. 1
    // w[k][c] = Phi_j^T[r][c] = W_j[r][c]; w[k][M] = nu_j[r]
    CT w[kPF][M + 1];
#pragma unroll
    for (int k = 0; k < kPF; ++k) {
        const int j = g.nsub - 1 - k;
        if (j >= 1) {
            const CT* W = PhiZ + (g0 + j) * (M + 1) * M + r * M;
#pragma unroll
            for (int c = 0; c < M; ++c) w[k][c] = W[c];
            w[k][M] = Nu[(g0 + j) * M + r];
        }
    }
    for (int i0 = 0; i0 < g.nsub; i0 += kPF) {
#pragma unroll
        for (int k = 0; k < kPF; ++k) {
            const int j = g.nsub - 1 - (i0 + k);
            if (j >= 0) {
                if (lane < M) Mu[(g0 + j) * M + lane] = (CT)mu;
                if (j >= 1) {
                    ms[warp][lane] = mu;
                    __syncwarp();
                    ACC q0 = (ACC)w[k][M], q1 = (ACC)0, q2 = (ACC)0, q3 = (ACC)0;
#pragma unroll
                    for (int c = 0; c < M; ++c) {
                        const ACC mc = ms[warp][c];
                        switch (c & 3) {
                            case 0: q0 = fma((ACC)w[k][c], mc, q0); break;
                            case 1: q1 = fma((ACC)w[k][c], mc, q1); break;
                            case 2: q2 = fma((ACC)w[k][c], mc, q2); break;
                            default: q3 = fma((ACC)w[k][c], mc, q3); break;
                        }
                    }
                    __syncwarp();
                    if (lane < M) mu = (q0 + q1) + (q2 + q3);
                    const int jn = j - kPF;
                    if (jn >= 1) {
                        const CT* W = PhiZ + (g0 + jn) * (M + 1) * M + r * M;
#pragma unroll
                        for (int c = 0; c < M; ++c) w[k][c] = W[c];
                        w[k][M] = Nu[(g0 + jn) * M + r];
                    }
                }
            }
        }
    }
}

// ============================================================================
// Lane-per-sub-chunk streaming kernels (apply fwd, adjoint zero-state, apply
// bwd).  One warp = 32 consecutive sub-chunks; lane l streams its own rows in
// windows of W = 8 through a 3-stage shared ring (each lane issues its own
// 1-D bulk copies; the stage mbarrier expects the warp's total bytes).
// Outputs are staged per lane and written back by bulk TMA stores.
// ============================================================================
template <typename IO, int M, bool TI>
struct LaneSmem {
    static constexpr int W = kLaneWin;
    static constexpr int ASTR = TI ? 0 : odd16_stride(W * M * (int)sizeof(IO));
    static constexpr int XSTR = odd16_stride(W * (int)sizeof(IO));
    static constexpr int STAGE = 32 * (ASTR + XSTR);
    static constexpr int OSTR = odd16_stride(W * (int)sizeof(IO));
    static constexpr int OUT = 32 * OSTR;
    static constexpr int BYTES = kLaneStages * STAGE + kOutStages * OUT + kLaneStages * 8;
};

// direction: +1 forward windows from t0, -1 reverse windows from t1.
template <typename IO, int M, bool TI, int DIR>
struct LaneStream {
    using S = LaneSmem<IO, M, TI>;
    static constexpr int W = S::W;
    unsigned char* base;
    uint64_t* bars;
    int lane;
    bool active;
    int len;
    int64_t row0;  // flat row of t0
    int nwin;

    __device__ __forceinline__ unsigned char* A_slot(int st) const {
        return base + st * S::STAGE + lane * S::ASTR;
    }
    __device__ __forceinline__ unsigned char* X_slot(int st) const {
        return base + st * S::STAGE + 32 * S::ASTR + lane * S::XSTR;
    }
    __device__ __forceinline__ unsigned char* O_slot(int so) const {
        return base + kLaneStages * S::STAGE + so * S::OUT + lane * S::OSTR;
    }
    // window k: rows [lo, lo+rows) relative to t0
    __device__ __forceinline__ void window(int k, int& lo, int& rows) const {
        if (DIR > 0) {
            lo = k * W;
            rows = active ? max(0, min(W, len - lo)) : 0;
        } else {
            const int hi = len - k * W;
            lo = max(0, hi - W);
            rows = active ? max(0, hi - lo) : 0;
        }
    }
    __device__ __forceinline__ void issue(int k, int nwin_max, const IO* A, const IO* X) {
        if (k >= nwin_max) return;
        const int st = k % kLaneStages;
        int lo, rows;
        window(k, lo, rows);
        const uint32_t mine = rows * ((TI ? 0 : M) + 1) * (uint32_t)sizeof(IO);
        const uint32_t tot = warp_sum_u32(mine);
        if (lane == 0) mbar_arrive_expect_tx(&bars[st], tot);
        __syncwarp();
        if (rows > 0) {
            const int64_t r = row0 + lo;
            // reverse windows may be short at t0: place rows at the window end
            const int pad = (DIR > 0) ? 0 : (W - rows);
            if (!TI)
                tma_load_1d(A_slot(st) + pad * M * (int)sizeof(IO), A + r * M,
                            rows * M * (uint32_t)sizeof(IO), &bars[st]);
            tma_load_1d(X_slot(st) + pad * (int)sizeof(IO), X + r, rows * (uint32_t)sizeof(IO),
                        &bars[st]);
        }
    }
};

// ---------------------------------------------------------------- apply fwd
// One lane re-runs the recursion of its sub-chunk from x_in.  The state lives
// in a register ring of MR = round_up(M, W) slots (slot p holds s at local
// step tau with tau mod MR == p); the unrolled body covers MR/W windows so
// every ring index is a compile-time constant.  Full windows take a
// predicate-free path; only the last window of a sequence can be partial.
template <typename IO, int M, bool TI>
__global__ void __launch_bounds__(32)
k_apply_fwd(const IO* __restrict__ e, const IO* __restrict__ A, const IO* __restrict__ Xin,
            IO* __restrict__ s, int* __restrict__ flag, ScanArgs g) {
    using S = LaneSmem<IO, M, TI>;
    using LS = LaneStream<IO, M, TI, +1>;
    constexpr int W = S::W;
    constexpr int MR = (M + W - 1) / W * W;
    constexpr int WPB = MR / W;
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x;
    LS ls;
    ls.base = smem;
    ls.bars = reinterpret_cast<uint64_t*>(smem + kLaneStages * S::STAGE + kOutStages * S::OUT);
    ls.lane = lane;
    const int64_t nsc = g.B * g.nsub;
    const int64_t gid = (int64_t)blockIdx.x * 32 + lane;
    ls.active = gid < nsc;
    const int64_t b = ls.active ? gid / g.nsub : 0;
    const int j = ls.active ? (int)(gid % g.nsub) : 0;
    const int64_t t0 = (int64_t)j * g.Ls;
    ls.len = ls.active ? (int)(int64_t)min((int64_t)(g.Ls), (int64_t)(g.T - t0)) : 0;
    ls.row0 = b * g.T + t0;
    const int nwin_max = (g.Ls + W - 1) / W;

    if (lane == 0) {
        for (int st = 0; st < kLaneStages; ++st) mbar_init(&ls.bars[st], 1);
        fence_mbar_init();
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < kLaneStages; ++k) ls.issue(k, nwin_max, A, e);

    IO ati[M];
    if (TI) {
#pragma unroll
        for (int i = 0; i < M; ++i) ati[i] = ls.active ? A[b * M + i] : (IO)0;
    }
    IO R[MR];
#pragma unroll
    for (int p = 0; p < MR; ++p) R[p] = (IO)0;
#pragma unroll
    for (int i = 0; i < M; ++i) R[MR - 1 - i] = ls.active ? Xin[gid * M + i] : (IO)0;
    bool finite = true;

    for (int kb = 0; kb < nwin_max; kb += WPB) {
#pragma unroll
        for (int w = 0; w < WPB; ++w) {
            const int k = kb + w;
            if (k < nwin_max) {
                const int st = k % kLaneStages;
                mbar_wait(&ls.bars[st], (uint32_t)((k / kLaneStages) & 1));
                int lo, rows;
                ls.window(k, lo, rows);
                const IO* Ar = reinterpret_cast<const IO*>(ls.A_slot(st));
                const IO* er = reinterpret_cast<const IO*>(ls.X_slot(st));
                const int so = k % kOutStages;
                IO* ob = reinterpret_cast<IO*>(ls.O_slot(so));
                if (k >= kOutStages) bulk_wait_read<kOutStages - 1>();
                IO ev[W];
#pragma unroll
                for (int u = 0; u < W; ++u) ev[u] = er[u];
                const bool full = rows == W;
#pragma unroll
                for (int u = 0; u < W; ++u) {
                    if (full || u < rows) {
                        const int pos = w * W + u;  // compile-time after unrolling
                        IO a[M];
                        if constexpr (TI) {
#pragma unroll
                            for (int i = 0; i < M; ++i) a[i] = ati[i];
                        } else {
                            load_row_at<IO, M>(Ar + u * M, a, u * M * (int)sizeof(IO));
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
                        const IO v = fma(-a[0], R[(pos - 1 + MR) % MR], ev[u] - ((p0 + p1) + (p2 + p3)));
                        R[pos % MR] = v;
                        ob[u] = v;
                        finite &= is_finite_val(v);
                    }
                }
                __syncwarp();
                fence_proxy_async();
                if (rows > 0) tma_store_1d(s + ls.row0 + lo, ob, rows * (uint32_t)sizeof(IO));
                bulk_commit();
                ls.issue(k + kLaneStages, nwin_max, A, e);
            }
        }
    }
    bulk_wait<0>();
    if (flag != nullptr) {
        // a non-finite output means non-finite input or overflow; the host
        // tells them apart (overflow of an unstable filter is legitimate).
        const unsigned bad = __ballot_sync(0xffffffffu, !finite);
        if (bad && lane == 0) atomicOr(flag, 1);
    }
}

// ---------------------------------------------------------------- adjoint
// MODE 0: zero-state adjoint per sub-chunk -> Nu.  MODE 1: apply from Mu,
// write g_e.  Reverse time; row A[t] is used at step t:
//   lambda += u0 g_s(t);  g_e(t) = lambda_0;  lambda = C(t)^T lambda.
// The transposed-state update shifts lambda inside its FMAs (no moves).
template <typename IO, int M, bool TI, int MODE>
__global__ void __launch_bounds__(32)
k_adjoint(const IO* __restrict__ gs, const IO* __restrict__ A, const IO* __restrict__ Mu,
          IO* __restrict__ Nu, IO* __restrict__ ge, ScanArgs g) {
    using S = LaneSmem<IO, M, TI>;
    using LS = LaneStream<IO, M, TI, -1>;
    constexpr int W = S::W;
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x;
    LS ls;
    ls.base = smem;
    ls.bars = reinterpret_cast<uint64_t*>(smem + kLaneStages * S::STAGE + kOutStages * S::OUT);
    ls.lane = lane;
    const int64_t nsc = g.B * g.nsub;
    const int64_t gid = (int64_t)blockIdx.x * 32 + lane;
    ls.active = gid < nsc;
    const int64_t b = ls.active ? gid / g.nsub : 0;
    const int j = ls.active ? (int)(gid % g.nsub) : 0;
    const int64_t t0 = (int64_t)j * g.Ls;
    ls.len = ls.active ? (int)(int64_t)min((int64_t)(g.Ls), (int64_t)(g.T - t0)) : 0;
    ls.row0 = b * g.T + t0;
    const int nwin_max = (g.Ls + W - 1) / W;

    if (lane == 0) {
        for (int st = 0; st < kLaneStages; ++st) mbar_init(&ls.bars[st], 1);
        fence_mbar_init();
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < kLaneStages; ++k) ls.issue(k, nwin_max, A, gs);

    IO ati[M];
    if (TI) {
#pragma unroll
        for (int i = 0; i < M; ++i) ati[i] = ls.active ? A[b * M + i] : (IO)0;
    }
    IO lam[M];
#pragma unroll
    for (int i = 0; i < M; ++i)
        lam[i] = (MODE == 1 && ls.active) ? Mu[gid * M + i] : (IO)0;

    // reverse windows of a sub-chunk whose length is not a multiple of W:
    // window k covers [max(0, len-(k+1)W), len-kW); slots are right-aligned.
    for (int k = 0; k < nwin_max; ++k) {
        const int st = k % kLaneStages;
        mbar_wait(&ls.bars[st], (uint32_t)((k / kLaneStages) & 1));
        int lo, rows;
        ls.window(k, lo, rows);
        const IO* Ar = reinterpret_cast<const IO*>(ls.A_slot(st));
        const IO* xr = reinterpret_cast<const IO*>(ls.X_slot(st));
        const int so = k % kOutStages;
        IO* ob = reinterpret_cast<IO*>(ls.O_slot(so));
        if (MODE == 1 && k >= kOutStages) bulk_wait_read<kOutStages - 1>();
        IO gv[W];
#pragma unroll
        for (int u = 0; u < W; ++u) gv[u] = xr[u];
        const bool full = rows == W;
#pragma unroll
        for (int u = W - 1; u >= 0; --u) {
            if (full || u >= W - rows) {
                IO a[M];
                if constexpr (TI) {
#pragma unroll
                    for (int i = 0; i < M; ++i) a[i] = ati[i];
                } else {
                    load_row_at<IO, M>(Ar + u * M, a, u * M * (int)sizeof(IO));
                }
                const IO l0 = lam[0] + gv[u];
                if (MODE == 1) ob[u] = l0;
#pragma unroll
                for (int i = 0; i < M - 1; ++i) lam[i] = fma(-a[i], l0, lam[i + 1]);
                lam[M - 1] = -a[M - 1] * l0;
            }
        }
        if (MODE == 1) {
            __syncwarp();
            fence_proxy_async();
            if (rows > 0)
                tma_store_1d(ge + ls.row0 + lo, ob + (W - rows), rows * (uint32_t)sizeof(IO));
            bulk_commit();
        }
        ls.issue(k + kLaneStages, nwin_max, A, gs);
    }
    if (MODE == 1) bulk_wait<0>();
    if (MODE == 0 && ls.active) {
#pragma unroll
        for (int i = 0; i < M; ++i) Nu[gid * M + i] = lam[i];
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
    for (int idx = threadIdx.x; idx < n; idx += 256) {
        const int r = idx / M;
        const int c = idx - r * M;
        out[idx] = (-sh_g[r]) * sh_s[M + r - c - 1];
    }
}

// g_a[b,c] = -sum_t s(t-c-1) g_e(t): partial sums per (b, chunk), then a
// fixed-order sum over chunks (deterministic).
template <typename IO>
__global__ void k_grad_a_partial(const IO* __restrict__ ge, const IO* __restrict__ s,
                                 const IO* __restrict__ zi, IO* __restrict__ part,
                                 int64_t T, int M, int nchunk) {
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
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= B * M) return;
    const int64_t b = idx / M;
    const int c = (int)(idx % M);
    double tot = 0.0;
    for (int k = 0; k < nchunk; ++k) tot += (double)part[(b * nchunk + k) * M + c];
    ga[idx] = (IO)(-tot);
}

}  // namespace tvlp
