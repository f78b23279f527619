// chain.cuh -- single-pass chunked scans with chained carries (fp32 I/O).
//
// Reference path: pkg/src/tvlp/lpc.py:36-47 / 101-117 (forward) and 152-173
// (backward).  Same algorithm as lp_scan.cuh (sub-chunk transition matrices,
// carries, re-application), restructured so that one persistent launch does
// the whole forward (or the adjoint passes of the whole backward) and the
// serial carries leave the critical path:
//
//   * A sequence's sub-chunks are grouped into UNITS of U consecutive
//     sub-chunks (the last unit of a sequence may be shorter).  A unit is the
//     work item of one warp in the lane-per-sub-chunk passes; units of one
//     sequence are chained: unit r needs the carry state published by unit
//     r-1 (forward) or r+1 (adjoint).  Work is handed out by atomic tickets in
//     unit-column order (all sequences' unit 0, then unit 1, ...), and a warp
//     only ever waits for a unit with a SMALLER ticket, which some running warp
//     already holds -- the chain cannot deadlock whatever the residency.
//   * Forward (k_fwd_chain): basis warps and an apply warp share each CTA.
//     Basis warps take tickets of 4-sub-chunk groups and write the transition
//     tapes (the k_basis4 code); the apply warp takes unit tickets, waits until
//     its unit's tapes are complete (a per-unit counter the basis warps
//     release), runs the unit's carries from the state the previous unit
//     published, publishes the state past its unit, and re-runs the
//     recursion of its sub-chunks (one lane each).  The compute-bound basis
//     and the memory-bound apply of different units overlap on every SM.
//   * Backward (k_bwd_chain): per unit the zero-state adjoint, the carry
//     (waiting for the unit to the right), the adjoint re-application.  The
//     second read of the unit's coefficient rows follows the first within a
//     few microseconds, so it is served from L2 (the first read keeps the
//     lines with an evict_last policy, the second releases them).
//   * Precision "auto": every unit records its boundary defects (lp_scan.cuh
//     "refinement"); the unit that completes a sequence (per-sequence done
//     counter) applies the correction recurrence to that sequence and
//     re-runs it when the defect check failed -- no extra launch when nothing
//     is flagged.
#pragma once
#include "chain_launch.cuh"
#include "lp_scan.cuh"

#ifndef TVLP_CHAIN_BASIS_WARPS
// 0: the forward's transition tapes come from k_basis4 (a separate launch) and
// k_fwd_chain runs the carries and re-application only; > 0: that many basis
// warps share each persistent CTA with one apply warp
#define TVLP_CHAIN_BASIS_WARPS 0
#endif
#ifndef TVLP_CHAIN_FWD_UNIT
#define TVLP_CHAIN_FWD_UNIT (TVLP_CHAIN_BASIS_WARPS > 0 ? 16 : 32)
#endif
#ifndef TVLP_CHAIN_BWD_ZS
// 1: the chained backward also runs the zero-state adjoint of each unit (the
// second read of A then often hits L2); 0: the zero-state pass is the
// separate streaming kernel k_adjoint<MODE 0> and the chained kernel reads nu
#define TVLP_CHAIN_BWD_ZS 0
#endif
#ifndef TVLP_CHAIN_BWD_UNIT
#define TVLP_CHAIN_BWD_UNIT (TVLP_CHAIN_BWD_ZS ? 16 : 32)
#endif
#ifndef TVLP_CHAIN_BASIS_SPLIT
#define TVLP_CHAIN_BASIS_SPLIT 2
#endif
#ifndef TVLP_CHAIN_FWD_STAGES
#define TVLP_CHAIN_FWD_STAGES (TVLP_CHAIN_BASIS_WARPS > 0 ? 2 : 3)
#endif
#ifndef TVLP_CHAIN_BWD_STAGES
#define TVLP_CHAIN_BWD_STAGES (TVLP_CHAIN_BWD_ZS ? 8 : 3)
#endif

namespace tvlp {

static __device__ unsigned long long g_chain_refined = 0;  // sequences refined (diagnostic)

// Optional per-work-item timeline (tools/chain_trace.py): 8 u64 per record,
// [kind | sm << 8 | ticket << 32, t0, t1, t2, t3, t4, 0, 0] in globaltimer ns.
struct ChainTrace {
    unsigned long long* buf;  // nullable
    unsigned cap;             // records
};
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned smid() {
    unsigned r;
    asm volatile("mov.u32 %0, %smid;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void trace_rec(const ChainTrace& tr, unsigned slot, unsigned kind,
                                          unsigned ticket, const unsigned long long (&t)[5]) {
    if (tr.buf == nullptr || slot >= tr.cap || (threadIdx.x & 31) != 0) return;
    unsigned long long* r = tr.buf + (size_t)slot * 8;
    r[0] = (unsigned long long)kind | ((unsigned long long)smid() << 8) |
           ((unsigned long long)ticket << 32);
    for (int i = 0; i < 5; ++i) r[1 + i] = t[i];
}

// ---------------------------------------------------------------- signalling
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release_add_u32(unsigned* p, unsigned v) {
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// A published state component: the value's bits and a ready flag in one
// 64-bit word, so a reader that sees the flag also sees the value.
__device__ __forceinline__ void st_state(unsigned long long* p, float v) {
    const unsigned long long w = (1ull << 32) | (unsigned long long)__float_as_uint(v);
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
}
__device__ __forceinline__ bool ld_state(const unsigned long long* p, float& v) {
    unsigned long long w;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
    v = __uint_as_float((unsigned)w);
    return (w >> 32) != 0;
}
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ unsigned warp_ticket(unsigned* ctr) {
    unsigned t = 0;
    if ((threadIdx.x & 31) == 0) t = atomicAdd(ctr, 1u);
    return __shfl_sync(0xffffffffu, t, 0);
}
// lanes < M return component `lane` of the state published at p
template <int M>
__device__ __forceinline__ float wait_state(const unsigned long long* p) {
    const int lane = threadIdx.x & 31;
    float v = 0.f;
    if (lane < M) {
        unsigned ns = 32;
        while (!ld_state(p + lane, v)) {
            __nanosleep(ns);
            if (ns < 512) ns <<= 1;
        }
    }
    __syncwarp();
    return v;
}
__device__ __forceinline__ void wait_count(const unsigned* p, unsigned need) {
    if ((threadIdx.x & 31) == 0) {
        unsigned ns = 64;
        while (ld_acquire_u32(p) < need) {
            __nanosleep(ns);
            if (ns < 1024) ns <<= 1;
        }
        fence_proxy_async_global();  // TMA reads of data released by other SMs follow
    }
    __syncwarp();
}

// L2 policies for tensor loads: a first read that will be repeated shortly
// keeps its lines, the repeat releases them.
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void tma_load_2d_hint(void* dst, const CUtensorMap* map, int c0, int c1,
                                                 uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
        "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

// Lane-view tensor maps, box rows U ([0]) and rem ([1]): A [B*nsub, Ls*M],
// signal in (e or g_s) [B*nsub, Ls], signal out (s or g_e) [B*nsub, Ls].
struct UnitMaps {
    CUtensorMap A[2];
    CUtensorMap X[2];
    CUtensorMap O[2];
    float* o;  // the output rows ([B*nsub][Ls]): lanes store their windows directly
};

template <int M, int U, int NST>
struct UnitLane {
    static constexpr int W = kLaneWin;
    static constexpr int AROW = odd16_stride(W * M * 4) / 4;
    static constexpr int XROW = odd16_stride(W * 4) / 4;
    static constexpr int A_BYTES = (U * AROW * 4 + 127) / 128 * 128;
    static constexpr int X_BYTES = (U * XROW * 4 + 127) / 128 * 128;
    static constexpr int STAGE = A_BYTES + X_BYTES;
    static constexpr int BYTES = NST * STAGE;  // + the caller's barriers
    __device__ static uint32_t tx(int L) { return (uint32_t)L * (AROW + XROW) * 4u; }
};

// ---------------------------------------------------------------- forward lane pass
// Lanes l < L re-run the recursion of sub-chunk g0 + l from xin[l] (shared,
// rows of MP4), write s through the unit's output box, and return the end
// state in `xe` (registers, x[i] = s(t1 - i)).
// FR: frame-rate rows interpolated in registers by
// a FrameCursor (lp_scan.cuh) instead of streamed; fs the frame source, fb the
// sequence within it, tl0 the time of the unit's first sub-chunk.
template <int M, int U, int NST, bool TI, bool FR = false>
__device__ __forceinline__ void unit_fwd_pass(const UnitMaps& mp, int which, int64_t g0, int L,
                                              int nwin, unsigned char* sm, uint64_t* bars,
                                              const float* xin, float (&xe)[M], bool& finite,
                                              const float* ati,
                                              const FrameSrc<float>* fs = nullptr, int64_t fb = 0,
                                              int64_t tl0 = 0) {
    using S = UnitLane<M, U, NST>;
    constexpr int W = S::W;
    constexpr int MR = (M + W - 1) / W * W;
    constexpr int WPB = MR / W;
    constexpr int MP4 = Tape<M>::MP4;
    const int lane = threadIdx.x & 31;
    const int ln = lane < U ? lane : U - 1;  // lanes past the unit read a valid row, never write
    const bool active = lane < L;
    const uint32_t tx = (TI || FR) ? (uint32_t)L * S::XROW * 4u : S::tx(L);
    FrameCursor<float, FR ? M : 1> cur;
    const float inv_hop = FR ? 1.f / (float)fs->hop : 0.f;
    const int64_t tlane = tl0 + (int64_t)lane * (nwin * W);  // this lane's sub-chunk start
    const uint64_t pol = policy_evict_first();
    float ar[TI ? M : 1];  // TI: the sequence's constant row
    if constexpr (TI) {
#pragma unroll
        for (int i = 0; i < M; ++i) ar[i] = ati[i];
    }
    if (lane == 0) {
        for (int st = 0; st < NST; ++st) mbar_init(&bars[st], 1);
        fence_mbar_init();
    }
    __syncwarp();
    auto issue = [&](int k) {
        if (k < nwin && lane == 0) {
            const int st = k % NST;
            unsigned char* base = sm + st * S::STAGE;
            mbar_arrive_expect_tx(&bars[st], tx);
            if (!TI && !FR)
                tma_load_2d_hint(base, &mp.A[which], k * W * M, (int)g0, &bars[st], pol);
            tma_load_2d_hint(base + S::A_BYTES, &mp.X[which], k * W, (int)g0, &bars[st], pol);
        }
    };
#pragma unroll
    for (int k = 0; k < NST; ++k) issue(k);
    float R[MR];
#pragma unroll
    for (int p = 0; p < MR; ++p) R[p] = 0.f;
#pragma unroll
    for (int i = 0; i < M; ++i) R[MR - 1 - i] = active ? xin[lane * MP4 + i] : 0.f;
    for (int kb = 0; kb < nwin; kb += WPB) {
#pragma unroll
        for (int w = 0; w < WPB; ++w) {
            const int k = kb + w;
            if (k < nwin) {
                const int st = k % NST;
                TVLP_ASSERT(k < nwin && ln < U && L <= U);
                mbar_wait(&bars[st], (uint32_t)((k / NST) & 1));
                const unsigned char* base = sm + st * S::STAGE;
                const float* Ar = reinterpret_cast<const float*>(base) + ln * S::AROW;
                const float* er = reinterpret_cast<const float*>(base + S::A_BYTES) + ln * S::XROW;
                float ev[W], ov[W];
#pragma unroll
                for (int u = 0; u < W; ++u) ev[u] = er[u];
                if constexpr (FR) cur.window(*fs, fb, tlane + (int64_t)k * W);
                // rows are loaded one step ahead (issued before this step's
                // output store, so no shared-memory ordering holds them back)
                float an[M];
                if constexpr (!TI && !FR) load_row_at<float, M>(Ar, an, (ln * S::AROW) * 4);
#pragma unroll
                for (int u = 0; u < W; ++u) {
                    const int pos = w * W + u;
                    float a[M];
                    if constexpr (FR) {
                        cur.row(*fs, inv_hop, u, a);
                    } else {
#pragma unroll
                        for (int i = 0; i < M; ++i) a[i] = TI ? ar[TI ? i : 0] : an[i];
                    }
                    if (!TI && !FR && u + 1 < W)
                        load_row_at<float, M>(Ar + (u + 1) * M, an, (ln * S::AROW + (u + 1) * M) * 4);
                    float p0 = 0.f, p1 = 0.f, p2 = 0.f, p3 = 0.f;
#pragma unroll
                    for (int i = M; i >= 2; --i) {
                        const float x = R[(pos - i + 2 * MR) % MR];
                        switch (i & 3) {
                            case 0: p0 = fmaf(a[i - 1], x, p0); break;
                            case 1: p1 = fmaf(a[i - 1], x, p1); break;
                            case 2: p2 = fmaf(a[i - 1], x, p2); break;
                            default: p3 = fmaf(a[i - 1], x, p3); break;
                        }
                    }
                    const float v = fmaf(-a[0], R[(pos - 1 + MR) % MR], ev[u] - ((p0 + p1) + (p2 + p3)));
                    R[pos % MR] = v;
                    ov[u] = v;
                    finite &= !active || isfinite(v);
                }
                if (active) store_window<float, W>(mp.o + (g0 + lane) * (int64_t)(nwin * W) + k * W, ov);
                __syncwarp();  // every lane is done with the stage: refill it
                issue(k + NST);
            }
        }
    }
    const int last = (nwin * W - 1) % MR;
#pragma unroll
    for (int i = 0; i < M; ++i) {
        float v = 0.f;
#pragma unroll
        for (int p = 0; p < MR; ++p)
            if (p == (last - i + MR) % MR) v = R[p];
        xe[i] = v;
    }
}

// ---------------------------------------------------------------- adjoint lane pass
// MODE 0: zero-state adjoint of sub-chunk g0 + l (lam starts at 0), returns
// nu_l in lam.  MODE 1: from lam (the carry into the sub-chunk from the
// right), writes grad_e through the unit's output box; returns the carry-out.
template <int M, int U, int NST, int MODE, bool TI, bool FR = false>
__device__ __forceinline__ void unit_adj_pass(const UnitMaps& mp, int which, int64_t g0, int L,
                                              int nwin, unsigned char* sm, uint64_t* bars,
                                              float (&lam)[M], const float* ati,
                                              float* gmax = nullptr,
                                              const FrameSrc<float>* fs = nullptr, int64_t fb = 0,
                                              int64_t tl0 = 0) {
    using S = UnitLane<M, U, NST>;
    constexpr int W = S::W;
    const int lane = threadIdx.x & 31;
    const int ln = lane < U ? lane : U - 1;  // lanes past the unit read a valid row, never write
    const uint32_t tx = (TI || FR) ? (uint32_t)L * S::XROW * 4u : S::tx(L);
    FrameCursor<float, FR ? M : 1> cur;
    const float inv_hop = FR ? 1.f / (float)fs->hop : 0.f;
    const int64_t tlane = tl0 + (int64_t)lane * (nwin * W);  // this lane's sub-chunk start
    const uint64_t pol = MODE == 0 ? policy_evict_last() : policy_evict_first();
    float ar[TI ? M : 1];  // TI: the sequence's constant row
    if constexpr (TI) {
#pragma unroll
        for (int i = 0; i < M; ++i) ar[i] = ati[i];
    }
    if (lane == 0) {
        for (int st = 0; st < NST; ++st) mbar_init(&bars[st], 1);
        fence_mbar_init();
    }
    __syncwarp();
    auto issue = [&](int k) {
        if (k < nwin && lane == 0) {
            const int st = k % NST;
            unsigned char* base = sm + st * S::STAGE;
            const int wr = nwin - 1 - k;
            mbar_arrive_expect_tx(&bars[st], tx);
            if (!TI && !FR)
                tma_load_2d_hint(base, &mp.A[which], wr * W * M, (int)g0, &bars[st], pol);
            tma_load_2d_hint(base + S::A_BYTES, &mp.X[which], wr * W, (int)g0, &bars[st], pol);
        }
    };
#pragma unroll
    for (int k = 0; k < NST; ++k) issue(k);
    float gm = 0.f;  // MODE 1: max |grad_e| over the lane's samples
    for (int k = 0; k < nwin; ++k) {
        const int st = k % NST;
        TVLP_ASSERT(k < nwin && ln < U && L <= U);
        mbar_wait(&bars[st], (uint32_t)((k / NST) & 1));
        const unsigned char* base = sm + st * S::STAGE;
        const float* Ar = reinterpret_cast<const float*>(base) + ln * S::AROW;
        const float* xr = reinterpret_cast<const float*>(base + S::A_BYTES) + ln * S::XROW;
        float gv[W], ov[W];
#pragma unroll
        for (int u = 0; u < W; ++u) gv[u] = xr[u];
        if constexpr (FR) cur.window(*fs, fb, tlane + (int64_t)(nwin - 1 - k) * W);
        // rows are loaded one step ahead (issued before this step's output
        // store, so no shared-memory ordering holds them back)
        float an[M];
        if constexpr (!TI && !FR)
            load_row_at<float, M>(Ar + (W - 1) * M, an, (ln * S::AROW + (W - 1) * M) * 4);
#pragma unroll
        for (int u = W - 1; u >= 0; --u) {
            float a[M];
            if constexpr (FR) {
                cur.row(*fs, inv_hop, u, a);
            } else {
#pragma unroll
                for (int i = 0; i < M; ++i) a[i] = TI ? ar[TI ? i : 0] : an[i];
            }
            if (!TI && !FR && u > 0)
                load_row_at<float, M>(Ar + (u - 1) * M, an, (ln * S::AROW + (u - 1) * M) * 4);
            const float l0 = lam[0] + gv[u];
            ov[u] = l0;
            if (MODE == 1) gm = fmaxf(gm, fabsf(l0));
#pragma unroll
            for (int i = 0; i < M - 1; ++i) lam[i] = fmaf(-a[i], l0, lam[i + 1]);
            lam[M - 1] = -a[M - 1] * l0;
        }
        if (MODE == 1 && lane < L)
            store_window<float, W>(mp.o + (g0 + lane) * (int64_t)(nwin * W) + (nwin - 1 - k) * W, ov);
        __syncwarp();  // every lane is done with the stage: refill it
        issue(k + NST);
    }
    if (gmax != nullptr) *gmax = lane < L ? gm : 0.f;
}

// ---------------------------------------------------------------- carries of a unit
// fwd: x(l+1) = R_l x(l) + z_l over the unit's tapes staged in shared memory
// as [l][M+1][MP4] (z row, then the M rows of Phi); records x(l) in xs[l].
template <int M>
__device__ __forceinline__ float unit_carry_fwd(const float* tz, int L, float x, float* xs,
                                                float* xg, float* xb) {
    constexpr int MP4 = Tape<M>::MP4;
    const int lane = threadIdx.x & 31;
    const int r = lane < M ? lane : 0;
    // row r of Phi_l and z_l are independent of the state: loaded one hop
    // ahead, so a hop's critical path is the state broadcast + one dot
    float w[MP4], wn[MP4];
    load_vec<float, MP4>(tz + (1 + r) * MP4, w);
    float zr = tz[r];
    for (int l = 0; l < L; ++l) {
        const float* tn = tz + (l + 1 < L ? l + 1 : l) * (M + 1) * MP4;
        load_vec<float, MP4>(tn + (1 + r) * MP4, wn);
        const float zn = tn[r];
        if (lane < M) {
            xs[l * MP4 + lane] = x;
            xg[l * MP4 + lane] = x;
        }
        float* b = xb + (l & 1) * 32;
        b[lane] = lane < M ? x : 0.f;
        __syncwarp();
        float xv[MP4];
        load_vec<float, MP4>(b, xv);
        x = dot_rows<M, float>(w, xv, zr);
#pragma unroll
        for (int c = 0; c < MP4; ++c) w[c] = wn[c];
        zr = zn;
    }
    return x;
}
// bwd: mu(l-1) = W_l^T mu(l) + nu_l over the unit's W rows staged as
// [l][M][MP4] (row c = column c of Phi_l); records mu(l) in xs[l].
template <int M>
__device__ __forceinline__ float unit_carry_bwd(const float* tw, const float* nu, int L, float mu,
                                                float* xs, float* xg, float* xb) {
    constexpr int MP4 = Tape<M>::MP4;
    const int lane = threadIdx.x & 31;
    const int r = lane < M ? lane : 0;
    float w[MP4], wn[MP4];
    load_vec<float, MP4>(tw + ((L - 1) * M + r) * MP4, w);
    float nr = nu[(L - 1) * MP4 + r];
    for (int l = L - 1; l >= 0; --l) {
        const int ln = l > 0 ? l - 1 : 0;
        load_vec<float, MP4>(tw + (ln * M + r) * MP4, wn);
        const float nn = nu[ln * MP4 + r];
        if (lane < M) {
            xs[l * MP4 + lane] = mu;
            xg[l * MP4 + lane] = mu;
        }
        float* b = xb + (l & 1) * 32;
        b[lane] = lane < M ? mu : 0.f;
        __syncwarp();
        float mv[MP4];
        load_vec<float, MP4>(b, mv);
        mu = dot_rows<M, float>(w, mv, nr);
#pragma unroll
        for (int c = 0; c < MP4; ++c) w[c] = wn[c];
        nr = nn;
    }
    return mu;
}

// max over the warp's lanes (defect statistics of a unit: one sequence)
__device__ __forceinline__ float warp_fmax(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// ---------------------------------------------------------------- arguments
// Grouped launches (tvlp_lp_*_tv_grouped): up to kMaxGroups independent
// batches with their own buffers and the same (T, M) share one launch;
// sequence b of the launch is sequence b - gB0[g] of group g.
struct GroupIdx {
    int64_t gB0[kMaxGroups + 1];  // first sequence of each group (gB0[ng] = total B)
    int ng;
    __device__ __forceinline__ int of(int64_t b) const {
        int g = 0;
#pragma unroll
        for (int i = 1; i < kMaxGroups; ++i)
            if (i < ng && b >= gB0[i]) g = i;
        return g;
    }
};

struct ChainFwdArgs {
    UnitMaps mp[kMaxGroups];  // A, e, s lane views of each group
    FrameSrc<float> fs;       // FR: the frame rows (one group)
    GroupIdx gi;
    const float* Ag[kMaxGroups];  // TI: the constant rows [B_g][Mp] of each group
    const float* zig[kMaxGroups]; // nullable initial states [B_g][zs]
    CUtensorMap Tz;        // carry tape, 3-D [ntapes][2M+1][MP4], box [8][M+1][MP4] from row M
    const float* e;        // (basis role: one group)
    const float* A;
    int zs;
    float* tape;           // carry tape [B*nsub][Tape::SIZE] + per-sequence flags after it
    int* fflags;           // per-sequence refinement flags (the backward inherits them)
    float* Xin;            // [B*nsub][MP4]
    float* Xend;           // [B*nsub][MP4]
    int* nonfinite;        // nullable
    unsigned* ticket;      // [0] basis groups, [1] units
    unsigned* cnt;         // [B*nu] sub-chunks whose tapes are complete
    unsigned* done;        // [B] units finished
    unsigned* dstat;       // [3B] per sequence: max defect, max |x|, max ||Phi_j||_inf
    unsigned long long* pub;  // [B*nu][MP4] state published past each unit
    int refine;            // precision "auto": check + refine
    float tol;             // boundary-defect tolerance relative to max |x|
    ScanArgs g;
    UnitGeo u;
    ChainTrace tr;         // records: basis groups [0, B*ngrp), then units
};

struct ChainBwdArgs {
    UnitMaps mp[kMaxGroups];  // A, g_s, g_e lane views of each group
    FrameSrc<float> fs;       // FR: the frame rows (one group)
    GroupIdx gi;
    const float* Ag[kMaxGroups];  // TI: the constant rows [B_g][Mp]
    CUtensorMap Tw;        // carry tape, box [8][M][MP4] from row 0 (W rows)
    const float* Nu;       // [B*nsub][MP4] zero-state adjoints (kernels without the pass)
    const float* tape;
    const int* inherit;    // nullable: the forward's refinement flags
    float* Mu;             // [B*nsub][MP4] carry into each sub-chunk from the right
    float* Kout;           // [B*nsub][MP4] carry-out of each sub-chunk (apply pass)
    unsigned* ticket;
    unsigned* done;
    unsigned* dstat;
    unsigned long long* pub;
    int refine;
    float tol;             // relative to max |grad_e| at the boundaries
    ScanArgs g;
    UnitGeo u;
    ChainTrace tr;
};

template <int M, int NWB, int NST>
struct FwdChainSmem {
    using BC = Basis4Cfg<M, false>;
    static constexpr int MP4 = Tape<M>::MP4;
    static constexpr int U = TVLP_CHAIN_FWD_UNIT;
    static constexpr int BASIS = NWB * BC::WARP_BYTES;
    static constexpr int BBARS = (NWB * BC::S * BC::NSTB * 8 + 15) / 16 * 16;
    static constexpr int TZ = ((U + 7) / 8 * 8) * (M + 1) * MP4 * 4;  // staged z + R rows
    static constexpr int LANE = UnitLane<M, U, NST>::BYTES;
    static constexpr int APPLY = TZ > LANE ? TZ : LANE;
    static constexpr int XS = (U + 1) * MP4 * 4;
    static constexpr int OFF_APPLY = BASIS;
    static constexpr int OFF_XS = OFF_APPLY + APPLY;
    static constexpr int OFF_XB = OFF_XS + XS;
    static constexpr int OFF_BB = OFF_XB + 64 * 4;
    static constexpr int OFF_AB = OFF_BB + BBARS;
    static constexpr int BYTES = OFF_AB + (NST + 1) * 8;
};

template <int M, int NST, bool ZS>
struct BwdChainSmem {
    static constexpr int MP4 = Tape<M>::MP4;
    static constexpr int U = TVLP_CHAIN_BWD_UNIT;
    static constexpr int LANE = UnitLane<M, U, NST>::BYTES;
    static constexpr int TW = ((U + 7) / 8 * 8) * M * MP4 * 4;  // staged W rows
    static constexpr int NU = U * MP4 * 4;
    static constexpr int XS = U * MP4 * 4;
    // with the zero-state pass the W rows land during it (own region);
    // without it they share the lane stages (the carry precedes the pass)
    static constexpr int OFF_TW = ZS ? LANE : 0;
    static constexpr int REGION = ZS ? LANE + TW : (LANE > TW ? LANE : TW);
    static constexpr int OFF_NU = REGION;
    static constexpr int OFF_XS = OFF_NU + NU;
    static constexpr int OFF_XB = OFF_XS + XS;
    static constexpr int OFF_BAR = OFF_XB + 64 * 4;
    static constexpr int BYTES = OFF_BAR + (NST + 1) * 8;
};

// ---------------------------------------------------------------- refinement of one sequence
// Forward: e_{j+1} = Phi_j e_j + d_j, d_j = Xend_j - Xin_{j+1} (k_refine_fwd),
// Xin += e; then every unit of the sequence is re-applied, recording the new
// end states.  The correction uses the fp32 transition matrices, so it is
// repeated (up to kRefineIters passes) until the boundary defects are at the
// float32 rounding level (kRefineTarget of max |x|): residual defects of a
// resonant row are carried undamped through the rest of the sequence, so the
// detection threshold (tol) is far too loose a stopping point.  One warp.
constexpr int kRefineIters = 4;
constexpr float kRefineTarget = 3e-7f;
template <int M, int NST, bool TI, bool FR>
__device__ bool refine_sequence_fwd(const ChainFwdArgs& a, int64_t b, unsigned char* sm,
                                    uint64_t* bars, float* xs, float* xb, bool force,
                                    float xmax) {
    using TP = Tape<M>;
    constexpr int MP4 = TP::MP4;
    constexpr int U = TVLP_CHAIN_FWD_UNIT;
    const int lane = threadIdx.x & 31;
    const int r = lane < M ? lane : 0;
    const int nsub = a.g.nsub;
    const int64_t base = b * nsub;
    const int nwin = a.g.Ls / kLaneWin;
    const int grp = a.gi.of(b);
    const int64_t vbase = (b - a.gi.gB0[grp]) * nsub;  // the group's lane-view rows
    const float* arow = TI ? a.Ag[grp] + (b - a.gi.gB0[grp]) * M : nullptr;
    for (int it = 0; it < kRefineIters; ++it) {
        float e = 0.f, emax = 0.f;
        for (int j = 0; j + 1 < nsub; ++j) {
            const float* t = a.tape + (base + j) * TP::SIZE;
            xb[lane] = lane < M ? e : 0.f;
            __syncwarp();
            float w[MP4], ev[MP4];
            load_vec<float, MP4>(t + (TP::R_ROW + r) * MP4, w);
            load_vec<float, MP4>(xb, ev);
            const float d = lane < M ? a.Xend[(base + j) * MP4 + r] -
                                           a.Xin[(base + j + 1) * MP4 + r]
                                     : 0.f;
            const float en = dot_rows<M, float>(w, ev, d);
            __syncwarp();
            e = en;
            emax = fmaxf(emax, fabsf(e));
            if (lane < M) a.Xin[(base + j + 1) * MP4 + r] += e;
        }
        __syncwarp();
        // the corrections are the carries' accumulated error: small ones
        // (damped rows) leave the first pass's outputs within tolerance
        emax = warp_fmax(emax);
        if (it == 0 && !force && emax <= a.tol * xmax) return false;
        float dm = 0.f, xm = 0.f;
        for (int ru = 0; ru < a.u.nu; ++ru) {
            const int L = a.u.len(ru);
            const int64_t g0 = base + (int64_t)ru * U;
            for (int i = lane; i < L * MP4; i += 32) xs[i] = a.Xin[g0 * MP4 + i];
            __syncwarp();
            float xe[M];
            bool fin = true;
            unit_fwd_pass<M, U, NST, TI, FR>(a.mp[grp], L == U ? 0 : 1, vbase + (int64_t)ru * U, L,
                                             nwin, sm, bars, xs, xe, fin, arow, &a.fs,
                                             b - a.gi.gB0[grp], (int64_t)ru * U * a.g.Ls);
            if (lane < L) {
                const bool has_next = ru * U + lane + 1 < nsub;
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    a.Xend[(g0 + lane) * MP4 + i] = xe[i];
                    if (has_next) {
                        const float xn = a.Xin[(g0 + lane + 1) * MP4 + i];
                        dm = fmaxf(dm, fabsf(xe[i] - xn));
                        xm = fmaxf(xm, fmaxf(fabsf(xe[i]), fabsf(xn)));
                    }
                }
            }
            __syncwarp();
        }
        dm = warp_fmax(dm);
        xm = warp_fmax(xm);
        if (dm <= kRefineTarget * xm) break;  // (NaN defects keep refining)
    }
    return true;
}

// Backward: e_{j-1} = Phi_j^T e_j + d_j, d_j = K_j - Mu_{j-1} (k_refine_bwd),
// Mu += e; then the adjoint re-application of every unit of the sequence,
// repeated like the forward.
template <int M, int NST, bool TI, bool FR>
__device__ bool refine_sequence_bwd(const ChainBwdArgs& a, int64_t b, unsigned char* sm,
                                    uint64_t* bars, float* xb, bool force, float xmax) {
    using TP = Tape<M>;
    constexpr int MP4 = TP::MP4;
    constexpr int U = TVLP_CHAIN_BWD_UNIT;
    const int lane = threadIdx.x & 31;
    const int r = lane < M ? lane : 0;
    const int nsub = a.g.nsub;
    const int64_t base = b * nsub;
    const int nwin = a.g.Ls / kLaneWin;
    const int grp = a.gi.of(b);
    const int64_t vbase = (b - a.gi.gB0[grp]) * nsub;
    const float* arow = TI ? a.Ag[grp] + (b - a.gi.gB0[grp]) * M : nullptr;
    for (int it = 0; it < kRefineIters; ++it) {
        float e = 0.f, emax = 0.f;
        for (int j = nsub - 1; j >= 1; --j) {
            const float* t = a.tape + (base + j) * TP::SIZE;
            xb[lane] = lane < M ? e : 0.f;
            __syncwarp();
            float w[MP4], ev[MP4];
            load_vec<float, MP4>(t + r * MP4, w);
            load_vec<float, MP4>(xb, ev);
            const float d = lane < M ? a.Kout[(base + j) * MP4 + r] -
                                           a.Mu[(base + j - 1) * MP4 + r]
                                     : 0.f;
            const float en = dot_rows<M, float>(w, ev, d);
            __syncwarp();
            e = en;
            // component 0 reaches grad_e directly; the others after shifting
            emax = fmaxf(emax, fabsf(e));
            if (lane < M) a.Mu[(base + j - 1) * MP4 + r] += e;
        }
        __syncwarp();
        emax = warp_fmax(emax);
        if (it == 0 && !force && emax <= a.tol * xmax) return false;
        float dm = 0.f, xm = 0.f;
        for (int ru = 0; ru < a.u.nu; ++ru) {
            const int L = a.u.len(ru);
            const int64_t g0 = base + (int64_t)ru * U;
            float lam[M];
#pragma unroll
            for (int i = 0; i < M; ++i) lam[i] = lane < L ? a.Mu[(g0 + lane) * MP4 + i] : 0.f;
            unit_adj_pass<M, U, NST, 1, TI, FR>(a.mp[grp], L == U ? 0 : 1, vbase + (int64_t)ru * U, L,
                                                nwin, sm, bars, lam, arow, nullptr, &a.fs,
                                                b - a.gi.gB0[grp], (int64_t)ru * U * a.g.Ls);
            if (lane < L) {
                const bool has_prev = ru * U + lane > 0;
                const float* prev = a.Mu + (g0 + lane - 1) * MP4;
                if (has_prev) xm = fmaxf(xm, fmaxf(fabsf(lam[0]), fabsf(prev[0])));
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    a.Kout[(g0 + lane) * MP4 + i] = lam[i];
                    if (has_prev) dm = fmaxf(dm, fabsf(lam[i] - prev[i]));
                }
            }
            __syncwarp();
        }
        dm = warp_fmax(dm);
        xm = warp_fmax(xm);
        if (dm <= kRefineTarget * xm) break;
    }
    return true;
}

// ---------------------------------------------------------------- grouped streaming passes
// The transition tapes of every group's sequences in ONE k_basis4-shaped
// launch: a lane's global sub-chunk selects its group's e and A (a warp may
// straddle two groups; the tape is indexed by the global sub-chunk).
struct GroupSrc {
    const float* x[kMaxGroups];  // e (fwd) or g_s (bwd)
    const float* A[kMaxGroups];
    GroupIdx gi;
};
template <int M, bool TI>
__global__ void __launch_bounds__(Basis4Cfg<M, TI>::NW * 32, TVLP_BASIS4_MINB)
k_basis4_groups(const __grid_constant__ GroupSrc gs, float* __restrict__ PhiZ, ScanArgs g) {
    grid_dep_wait();
    using C = Basis4Cfg<M, TI>;
    extern __shared__ __align__(128) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool lane_used = lane / C::P < C::S;
    const int sc = lane_used ? lane / C::P : C::S - 1;
    const int64_t gid = ((int64_t)blockIdx.x * C::NW + warp) * C::S + sc;
    const int64_t nsc = g.B * g.nsub;
    const int64_t gq = gid < nsc ? gid : nsc - 1;
    const int64_t b = gq / g.nsub;
    const int grp = gs.gi.of(b);
    const int64_t b0 = gs.gi.gB0[grp];
    ScanArgs gl = g;
    gl.B = gs.gi.gB0[grp + 1] - b0;
    const FrameSrc<float> fs{};
    basis4_warp<M, TI, false>(gs.x[grp], gs.A[grp], PhiZ, gl, fs, gq - b0 * g.nsub,
                              lane_used && gid < nsc, smem + warp * C::WARP_BYTES,
                              reinterpret_cast<uint64_t*>(smem + C::BAR_OFF) +
                                  warp * C::S * C::NSTB,
                              gq);
}

// Zero-state adjoints of every group's sub-chunks in one launch: one warp per
// unit (units never straddle sequences, so a unit is in one group's lane
// views); nu of sub-chunk g0 + l goes to Nu[global sub-chunk].
template <int M, int U, int NST, bool TI>
__global__ void __launch_bounds__(32)
k_adj_zs_units(const __grid_constant__ ChainBwdArgs a) {
    grid_dep_wait();
    constexpr int MP4 = Tape<M>::MP4;
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int64_t t = blockIdx.x;
    const int nu = a.u.nu, nsub = a.g.nsub;
    if (t >= a.g.B * nu) return;
    const int64_t b = t / nu;
    const int ru = (int)(t % nu);
    const int L = a.u.len(ru);
    const int grp = a.gi.of(b);
    const int64_t bl = b - a.gi.gB0[grp];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + UnitLane<M, U, NST>::BYTES);
    float lam[M];
#pragma unroll
    for (int i = 0; i < M; ++i) lam[i] = 0.f;
    unit_adj_pass<M, U, NST, 0, TI>(a.mp[grp], L == U ? 0 : 1, bl * nsub + (int64_t)ru * U, L,
                                    a.g.Ls / kLaneWin, smem, bars, lam,
                                    TI ? a.Ag[grp] + bl * M : nullptr);
    if (lane < L) {
        float* out = const_cast<float*>(a.Nu) + (b * nsub + (int64_t)ru * U + lane) * MP4;
#pragma unroll
        for (int i = 0; i < M; ++i) out[i] = lam[i];
#pragma unroll
        for (int i = M; i < MP4; ++i) out[i] = 0.f;
    }
}

// ---------------------------------------------------------------- forward kernel
template <int M, int NWB, int NST, bool TI, bool FR = false>
__global__ void __launch_bounds__((NWB + 1) * 32, NWB > 0 ? 1 : 2)
k_fwd_chain(const __grid_constant__ ChainFwdArgs a) {
    grid_dep_wait();
    using SM = FwdChainSmem<M, NWB, NST>;
    using BC = Basis4Cfg<M, false>;
    using TP = Tape<M>;
    constexpr int MP4 = TP::MP4;
    constexpr int U = SM::U;
    static_assert(U % BC::S == 0 && U <= 32, "units hold whole basis groups");
    extern __shared__ __align__(128) unsigned char smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t B = a.g.B;
    const int nsub = a.g.nsub;
    static_assert(!(TI && NWB > 0), "TI: the transition tapes come from k_basis4");
    if (NWB > 0 && warp < NWB) {
        // ------------------------------------------------ basis role
        const int ngrp = (nsub + BC::S - 1) / BC::S;  // 4-sub-chunk groups per sequence
        const bool lane_used = lane / BC::P < BC::S;
        const int sc = lane_used ? lane / BC::P : BC::S - 1;
        unsigned char* wbase = smem + warp * BC::WARP_BYTES;
        uint64_t* wbars = reinterpret_cast<uint64_t*>(smem + SM::OFF_BB) + warp * BC::S * BC::NSTB;
        const FrameSrc<float> fs{};
        for (;;) {
            const unsigned t = warp_ticket(a.ticket);
            if ((int64_t)t >= B * ngrp) break;
            unsigned long long tt[5] = {gtime(), 0, 0, 0, 0};
            const int q = (int)(t / B);
            const int64_t b = t % B;
            const int j = q * BC::S + sc;
            const bool valid = lane_used && j < nsub;
            basis4_warp<M, false, false, TVLP_CHAIN_BASIS_SPLIT>(
                a.e, a.A, a.tape, a.g, fs, b * nsub + (valid ? j : 0), valid, wbase, wbars);
            fence_proxy_async_global();  // leaders: their completed tape stores, generic-visible
            __syncwarp();
            if (lane == 0) {
                __threadfence();
                const int j0 = q * BC::S;
                red_release_add_u32(&a.cnt[b * a.u.nu + j0 / U], (unsigned)min(BC::S, nsub - j0));
            }
            tt[1] = gtime();
            trace_rec(a.tr, t, 1, t, tt);
        }
        return;
    }
    // ---------------------------------------------------- apply role
    unsigned char* sa = smem + SM::OFF_APPLY;
    float* xs = reinterpret_cast<float*>(smem + SM::OFF_XS);
    float* xb = reinterpret_cast<float*>(smem + SM::OFF_XB);
    uint64_t* abars = reinterpret_cast<uint64_t*>(smem + SM::OFF_AB);  // NST lane stages + tz
    const int nwin = a.g.Ls / kLaneWin;
    const int nu = a.u.nu;
    bool finite = true;
    for (;;) {
        const unsigned t = warp_ticket(a.ticket + 1);
        if ((int64_t)t >= B * nu) break;
        const int ru = (int)(t / B);
        const int64_t b = t % B;
        const int L = a.u.len(ru);
        const int64_t g0 = b * nsub + (int64_t)ru * U;
        const int grp = a.gi.of(b);
        const int64_t bl = b - a.gi.gB0[grp];              // sequence within its group
        const int64_t r0 = bl * nsub + (int64_t)ru * U;    // row of the group's lane views
        TVLP_ASSERT(ru < nu && b < B && L >= 1 && L <= U && g0 + L <= B * nsub);
        TVLP_ASSERT(grp < a.gi.ng && bl >= 0 && bl < a.gi.gB0[grp + 1] - a.gi.gB0[grp]);
        unsigned long long tt[5] = {gtime(), 0, 0, 0, 0};
        // 1. tapes of the unit complete? (NWB == 0: a previous launch wrote them)
        if constexpr (NWB > 0) wait_count(&a.cnt[b * nu + ru], (unsigned)L);
        tt[1] = gtime();
        // 2. stage the z and R rows of its L tapes
        uint64_t* tb = abars + NST;
        const int nb8 = (L + 7) / 8;
        if (lane == 0) {
            mbar_init(tb, 1);
            fence_mbar_init();
            mbar_arrive_expect_tx(tb, (uint32_t)nb8 * 8 * (M + 1) * MP4 * 4);
            for (int k = 0; k < nb8; ++k)
                tma_load_3d(sa + k * 8 * (M + 1) * MP4 * 4, &a.Tz, 0, TP::Z_ROW, (int)(g0 + 8 * k),
                            tb);
        }
        // 3. state entering the unit
        float x = 0.f;
        if (ru == 0) {
            if (a.zig[grp] != nullptr && lane < M) x = a.zig[grp][bl * a.zs + lane];
            __syncwarp();
        } else {
            TVLP_ASSERT(b * nu + ru - 1 < B * nu);
            x = wait_state<M>(a.pub + (b * nu + ru - 1) * MP4);
        }
        if (ru == 0 && lane == 0) a.fflags[b] = 0;
        mbar_wait(tb, 0);
        tt[2] = gtime();
        // 4. carries through the unit, publish the state past it
        x = unit_carry_fwd<M>(reinterpret_cast<const float*>(sa), L, x, xs, a.Xin + g0 * MP4, xb);
        if (ru + 1 < nu && lane < M) st_state(a.pub + (b * nu + ru) * MP4 + lane, x);
        if (lane < M) xs[L * MP4 + lane] = x;
        __syncwarp();
        tt[3] = gtime();
        // 5. re-run the unit's sub-chunks from their carried-in states
        float xe[M];
        unit_fwd_pass<M, U, NST, TI, FR>(a.mp[grp], L == U ? 0 : 1, r0, L, nwin, sa, abars, xs, xe,
                                         finite, TI ? a.Ag[grp] + bl * M : nullptr, &a.fs, bl,
                                         (int64_t)ru * U * a.g.Ls);
        tt[4] = gtime();
        trace_rec(a.tr, (NWB > 0 ? (unsigned)(B * ((nsub + BC::S - 1) / BC::S)) : 0u) + t, 2, t, tt);
        // 6. boundary defects (precision "auto")
        if (a.refine) {
            float dm = 0.f, xm = 0.f;
            const bool chk = lane < L && (lane + 1 < L || ru + 1 < nu);
            if (lane < L) {
#pragma unroll
                for (int i = 0; i < M; ++i) a.Xend[(g0 + lane) * MP4 + i] = xe[i];
            }
            if (chk) {
#pragma unroll
                for (int i = 0; i < M; ++i) {
                    const float xn = xs[(lane + 1) * MP4 + i];
                    dm = fmaxf(dm, fabsf(xe[i] - xn));
                    xm = fmaxf(xm, fmaxf(fabsf(xe[i]), fabsf(xn)));
                }
                if (!(dm == dm)) dm = __int_as_float(0x7f800000);
            }
            dm = warp_fmax(dm);
            xm = warp_fmax(xm);
            if (lane == 0) {
                atomicMax(&a.dstat[3 * b], __float_as_uint(dm));
                atomicMax(&a.dstat[3 * b + 1], __float_as_uint(xm));
            }
            // 7. the unit completing a sequence refines it when the check failed
            unsigned old = 0;
            if (lane == 0) {
                __threadfence();
                old = atomicAdd(&a.done[b], 1u);
            }
            old = __shfl_sync(0xffffffffu, old, 0);
            if (old == (unsigned)nu - 1) {
                __threadfence();
                const float dmax = __uint_as_float(ld_acquire_u32(&a.dstat[3 * b]));
                const float xmax = __uint_as_float(ld_acquire_u32(&a.dstat[3 * b + 1]));
                // defects above tol are refined (the boundary-defect check)
                if (dmax > a.tol * xmax) {
                    const bool done = refine_sequence_fwd<M, NST, TI, FR>(
                        a, b, sa, abars, xs, xb, dmax > a.tol * xmax, xmax);
                    if (done && lane == 0) {
                        a.fflags[b] = 1;
                        atomicAdd(&g_chain_refined, 1ull);
                    }
                }
            }
        }
        __syncwarp();
    }
    if (a.nonfinite != nullptr) {
        const unsigned bad = __ballot_sync(0xffffffffu, !finite);
        if (bad && lane == 0) atomicOr(a.nonfinite, 1);
    }
}

// ---------------------------------------------------------------- backward kernel
template <int M, int NST, bool ZS, bool TI, bool FR = false>
__global__ void __launch_bounds__(32)
k_bwd_chain(const __grid_constant__ ChainBwdArgs a) {
    grid_dep_wait();
    using SM = BwdChainSmem<M, NST, ZS>;
    constexpr int MP4 = Tape<M>::MP4;
    constexpr int U = SM::U;
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    unsigned char* sl = smem;
    float* tw = reinterpret_cast<float*>(smem + SM::OFF_TW);
    float* nus = reinterpret_cast<float*>(smem + SM::OFF_NU);
    float* xs = reinterpret_cast<float*>(smem + SM::OFF_XS);
    float* xb = reinterpret_cast<float*>(smem + SM::OFF_XB);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + SM::OFF_BAR);
    const int64_t B = a.g.B;
    const int nsub = a.g.nsub;
    const int nu = a.u.nu;
    const int nwin = a.g.Ls / kLaneWin;
    for (;;) {
        const unsigned t = warp_ticket(a.ticket);
        if ((int64_t)t >= B * nu) break;
        const int ru = nu - 1 - (int)(t / B);  // right to left
        const int64_t b = t % B;
        unsigned long long tt[5] = {gtime(), 0, 0, 0, 0};
        const int L = a.u.len(ru);
        const int which = L == U ? 0 : 1;
        const int64_t g0 = b * nsub + (int64_t)ru * U;
        const int grp = a.gi.of(b);
        const int64_t bl = b - a.gi.gB0[grp];
        const int64_t r0 = bl * nsub + (int64_t)ru * U;
        TVLP_ASSERT(ru >= 0 && ru < nu && b < B && L >= 1 && L <= U && g0 + L <= B * nsub);
        TVLP_ASSERT(grp < a.gi.ng && bl >= 0 && bl < a.gi.gB0[grp + 1] - a.gi.gB0[grp]);
        const float* arow = TI ? a.Ag[grp] + bl * M : nullptr;
        // W rows of the unit's tapes (read by the carry), staged during the
        // zero-state pass
        uint64_t* tb = bars + NST;
        const int nb8 = (L + 7) / 8;
        if (lane == 0) {
            mbar_init(tb, 1);
            fence_mbar_init();
            mbar_arrive_expect_tx(tb, (uint32_t)nb8 * 8 * M * MP4 * 4 +
                                          (ZS ? 0u : (uint32_t)L * MP4 * 4));
            for (int k = 0; k < nb8; ++k)
                tma_load_3d(tw + k * 8 * M * MP4, &a.Tw, 0, 0, (int)(g0 + 8 * k), tb);
            if (!ZS) tma_load_1d(nus, a.Nu + g0 * MP4, (uint32_t)L * MP4 * 4, tb);
        }
        float lam[M];
        if constexpr (ZS) {
            // 1. zero-state adjoint -> nu
#pragma unroll
            for (int i = 0; i < M; ++i) lam[i] = 0.f;
            unit_adj_pass<M, U, NST, 0, TI, FR>(a.mp[grp], which, r0, L, nwin, sl, bars, lam, arow,
                                                nullptr, &a.fs, bl, (int64_t)ru * U * a.g.Ls);
            if (lane < L) {
#pragma unroll
                for (int i = 0; i < M; ++i) nus[lane * MP4 + i] = lam[i];
            }
        }
        tt[1] = gtime();
        // 2. carry from the right
        float mu = 0.f;
        if (ru + 1 < nu) mu = wait_state<M>(a.pub + (b * nu + ru + 1) * MP4);
        mbar_wait(tb, 0);
        __syncwarp();
        tt[2] = gtime();
        mu = unit_carry_bwd<M>(tw, nus, L, mu, xs, a.Mu + g0 * MP4, xb);
        if (ru > 0 && lane < M) st_state(a.pub + (b * nu + ru) * MP4 + lane, mu);
        tt[3] = gtime();
        __syncwarp();
        // 3. adjoint re-application from the carried-in states
#pragma unroll
        for (int i = 0; i < M; ++i) lam[i] = lane < L ? xs[lane * MP4 + i] : 0.f;
        // keep the unit's left carry for lane 0's defect check (nus is free now)
        if (lane < M) nus[lane] = mu;
        __syncwarp();
        float gmx = 0.f;
        unit_adj_pass<M, U, NST, 1, TI, FR>(a.mp[grp], which, r0, L, nwin, sl, bars, lam, arow,
                                            &gmx, &a.fs, bl, (int64_t)ru * U * a.g.Ls);
        tt[4] = gtime();
        trace_rec(a.tr, t, 3, t, tt);
        if (a.refine) {
            float dm = 0.f, xm = 0.f;
            if (lane < L) {
#pragma unroll
                for (int i = 0; i < M; ++i) a.Kout[(g0 + lane) * MP4 + i] = lam[i];
            }
            const bool chk = lane < L && (lane > 0 || ru > 0);
            // scale: max |grad_e| over the unit's samples (the parity metric is
            // relative to the sequence's max |grad_e|; the boundary values of
            // lambda_0 alone can be far smaller and flag rounding-level defects)
            xm = gmx;
            if (chk) {
                const float* prev = lane > 0 ? xs + (lane - 1) * MP4 : nus;
                xm = fmaxf(xm, fmaxf(fabsf(lam[0]), fabsf(prev[0])));
#pragma unroll
                for (int i = 0; i < M; ++i) dm = fmaxf(dm, fabsf(lam[i] - prev[i]));
                if (!(dm == dm)) dm = __int_as_float(0x7f800000);
            }
            dm = warp_fmax(dm);
            xm = warp_fmax(xm);
            if (lane == 0) {
                atomicMax(&a.dstat[3 * b], __float_as_uint(dm));
                atomicMax(&a.dstat[3 * b + 1], __float_as_uint(xm));
            }
            unsigned old = 0;
            if (lane == 0) {
                __threadfence();
                old = atomicAdd(&a.done[b], 1u);
            }
            old = __shfl_sync(0xffffffffu, old, 0);
            if (old == (unsigned)nu - 1) {
                __threadfence();
                const float dmax = __uint_as_float(ld_acquire_u32(&a.dstat[3 * b]));
                const float xmax = __uint_as_float(ld_acquire_u32(&a.dstat[3 * b + 1]));
                const bool bad = dmax > a.tol * xmax ||
                                 (a.inherit != nullptr && a.inherit[b] != 0);
                if (bad) {
                    const bool done =
                        refine_sequence_bwd<M, NST, TI, FR>(a, b, sl, bars, xb, bad, xmax);
                    if (done && lane == 0) atomicAdd(&g_chain_refined, 1ull);
                }
            }
        }
        __syncwarp();
    }
}

}  // namespace tvlp
