// framewise_pieces.cuh -- frame-wise TI LP with every frame cut into P pieces
// (included by framewise.cu; same contract as k_fw_forward / k_fw_backward).
//
// Reference: params.py:220-239 (_framewise_forward), 259-273 (_framewise_vjp),
// lpc.py:50-61 / 176-195 (the TI recursion and its adjoint).
//
// One lane per frame leaves 6500 chains for config 2 (B=32, T=48000, hop 240,
// frame 960): 1.5 warps per SM, each issuing at ~1 instruction per 3 cycles
// (ncu: 54 instructions and ~170 cycles per sample).  A frame is a
// time-invariant recursion, so it splits like the sample-wise scan but
// with ONE transition for all of its pieces:
//
//   pass 1   every piece runs its recursion from a zero state (its exit
//            state z_p = the last M outputs) and, interleaved for ILP, the
//            frame's impulse response h(n) = delta(n) - sum_i a_i h(n-i);
//   carry    the exit of piece p from entry x is Z(x) + z_p, where the
//            zero-input response of an entry state x over n >= 0 is
//              y(n) = sum_{k=1..M} q_k h(n + k),
//              q_k  = x(-k) + sum_{i=1..M-k} a_i x(-k-i)
//            (the entry state acts as an input pulse train at -M..-1), so
//            Z needs only h(L-M+1 .. L+M-1); P-1 steps through the P lanes
//            of a frame by warp shuffles;
//   pass 2   every piece re-runs its recursion from its carried-in entry
//            state and writes its outputs.
//
// The adjoint of a TI all-pole filter is the same all-pole filter on
// reversed time (ge(k) = g(k) - sum_i a_i ge(k+i), lpc.py:176-195), so the
// backward runs passes 1 and carry on the reversed pieces with the same
// impulse response (the forward saves its tail per frame in the caller's
// aux buffer, so the backward's pass 1 runs one chain); its pass 2 is the
// push-form adjoint (as k_fw_backward),
// which also accumulates ga[c] = sum_k ge(k) s(k-1-c) against the saved
// frame outputs and writes gew = window * ge.
//
// Lanes: lane = kFwP * (frame within the warp) + piece, a CTA of 128
// threads covers 128 / kFwP consecutive frames of one sequence (the staged span of
// k_fw_forward).  Arithmetic differs from the one-lane-per-frame kernels (the
// carry adds one rounding level), so the plans that must stay bit-identical
// to lp_forward_ti (one rectangular frame) keep those kernels.

// TVLP_FW_P: pieces per frame (4; 8 is faster but its longer fp32 carry
// chain misses the parity bar on a resonant golden frame).  TVLP_FW_CARRY64:
// 1 = the carry's dot products in fp64, 2 = only its exit sums (both pass
// at P=8 and are slower than P=4 in fp32: measured).
#ifndef TVLP_FW_P
#define TVLP_FW_P 4
#endif
#ifndef TVLP_FW_CARRY64
#define TVLP_FW_CARRY64 0
#endif
constexpr int kFwP = TVLP_FW_P;  // pieces per frame (lanes per frame)
static_assert(kFwP == 2 || kFwP == 4 || kFwP == 8, "a frame's lanes share a warp");
constexpr int kFwpThreads = 128;                 // CTA
constexpr int kFwpFrames = kFwpThreads / kFwP;   // consecutive frames per CTA

// hop-blocks of the span the CTA's frames read
__host__ __device__ __forceinline__ int fwp_blocks(int size, int hop) {
    return ((kFwpFrames - 1) * hop + size + hop - 1) / hop;
}

template <typename IO>
__host__ __device__ __forceinline__ int fwp_lpad(int L) {
    // window blocks of the P pieces at an odd number of 16-byte granules
    constexpr int q = 16 / (int)sizeof(IO);
    int s = (L + q - 1) / q * q;
    if (((s / q) & 1) == 0) s += q;
    return s;
}

template <typename IO>
struct FwpSmem {
    static __host__ __device__ size_t off_win(int size, int hop) {
        return ((size_t)fwp_blocks(size, hop) * fw_stride<IO>(hop) * sizeof(IO) + 15) / 16 *
               16;
    }
    static __host__ __device__ size_t off_bar(int size, int hop) {
        return (off_win(size, hop) + (size_t)kFwP * fwp_lpad<IO>(size / kFwP) * sizeof(IO) + 15) /
               16 * 16;
    }
    static size_t bytes(int size, int hop) { return off_bar(size, hop) + 16; }
};

// the plans served by the piece kernels
inline bool fwp_supported(int size, int hop) {
    return size % (kFwP * kFwW) == 0 && size >= 128 && hop >= kFwW;
}

// CTA-wide staging of the span of 32 frames (hop-blocks at stride
// fw_stride, as fw_stage) and of the window in kFwP blocks of lp elements:
// one thread issues the bulk copies of every whole, aligned block, all
// threads fill the rest, then everyone waits on the barrier.  DIV: g / cola
// in place afterwards (params.py:263).
template <typename IO, bool DIV>
__device__ __forceinline__ void fwp_stage(IO* __restrict__ es, const IO* __restrict__ src,
                                          int64_t t0, int nblk, int64_t n_src, int hop, IO div,
                                          IO* __restrict__ ws, const IO* __restrict__ win, int L,
                                          int lp, uint64_t* bar) {
    const int tid = threadIdx.x, nt = blockDim.x;
    const int st = fw_stride<IO>(hop);
    const uint32_t bbytes = (uint32_t)hop * sizeof(IO);
    auto bulk_ok = [&](int q) {
        const int64_t t = t0 + (int64_t)q * hop;
        return t >= 0 && t + hop <= n_src && bbytes % 16 == 0 &&
               ((reinterpret_cast<uintptr_t>(src + t) & 15) == 0);
    };
    const bool wok = ((uint32_t)L * sizeof(IO)) % 16 == 0 &&
                     (reinterpret_cast<uintptr_t>(win) & 15) == 0;
    if (tid == 0) {
        uint32_t tx = wok ? (uint32_t)(kFwP * L * sizeof(IO)) : 0u;
        for (int q = 0; q < nblk; ++q) tx += bulk_ok(q) ? bbytes : 0;
        mbar_init(bar, 1);
        fence_mbar_init();
        mbar_arrive_expect_tx(bar, tx);
        for (int q = 0; q < nblk; ++q)
            if (bulk_ok(q)) tma_load_1d(es + q * st, src + t0 + (int64_t)q * hop, bbytes, bar);
        if (wok)
            for (int p = 0; p < kFwP; ++p)
                tma_load_1d(ws + p * lp, win + p * L, (uint32_t)(L * sizeof(IO)), bar);
    }
    for (int q = 0; q < nblk; ++q) {
        if (bulk_ok(q)) continue;  // block-uniform
        for (int r = tid; r < hop; r += nt) {
            const int64_t t = t0 + (int64_t)q * hop + r;
            es[q * st + r] = (t >= 0 && t < n_src) ? src[t] : (IO)0;
        }
    }
    if (!wok)
        for (int i = tid; i < kFwP * L; i += nt) ws[(i / L) * lp + i % L] = win[i];
    __syncthreads();  // the barrier's init and the thread-filled blocks
    mbar_wait(bar, 0);
    if (DIV) {
        for (int q = 0; q < nblk; ++q)
            for (int r = tid; r < hop; r += nt) es[q * st + r] = es[q * st + r] / div;
        __syncthreads();
    }
}

// Pass 1 of one piece: L steps of the zero-state recursion over the inputs
// x(n) = in(n) (in(kw, xv) fills window kw, in processing order) and of the
// impulse response, then M more impulse-response steps.  Returns the exit
// state z[i] = y(L-1-i) and ht[t] = h(L-M+t), t = 0..2M-1.
template <typename IO, int M, typename In, bool WITH_H = true>
__device__ __forceinline__ void fwp_pass1(const IO (&a)[M], int L, In in, IO (&z)[M],
                                          IO (&ht)[2 * M]) {
    constexpr int W = kFwW;
    constexpr int MR = (M + W - 1) / W * W;
    constexpr int WPB = MR / W;
    IO R[MR], H[MR];
#pragma unroll
    for (int p = 0; p < MR; ++p) {
        R[p] = (IO)0;
        H[p] = (IO)0;
    }
    const int nwin = L / W;
    for (int kb = 0; kb < nwin; kb += WPB) {
#pragma unroll
        for (int w = 0; w < WPB; ++w) {
            const int k = kb + w;
            if (k < nwin) {
                IO xv[W];
                in(k * W, xv);
#pragma unroll
                for (int u = 0; u < W; ++u) {
                    const int pos = w * W + u;
                    IO p0 = (IO)0, p1 = (IO)0, p2 = (IO)0, p3 = (IO)0;
                    IO h0 = (IO)0, h1 = (IO)0, h2 = (IO)0, h3 = (IO)0;
#pragma unroll
                    for (int i = M; i >= 2; --i) {
                        const IO x = R[(pos - i + 2 * MR) % MR];
                        const IO hx = H[(pos - i + 2 * MR) % MR];
                        switch (i & 3) {
                            case 0: p0 = fma(a[i - 1], x, p0); h0 = fma(a[i - 1], hx, h0); break;
                            case 1: p1 = fma(a[i - 1], x, p1); h1 = fma(a[i - 1], hx, h1); break;
                            case 2: p2 = fma(a[i - 1], x, p2); h2 = fma(a[i - 1], hx, h2); break;
                            default: p3 = fma(a[i - 1], x, p3); h3 = fma(a[i - 1], hx, h3); break;
                        }
                    }
                    R[pos % MR] =
                        fma(-a[0], R[(pos - 1 + MR) % MR], xv[u] - ((p0 + p1) + (p2 + p3)));
                    if constexpr (WITH_H) {
                        const IO d = (kb == 0 && pos == 0) ? (IO)1 : (IO)0;
                        H[pos % MR] =
                            fma(-a[0], H[(pos - 1 + MR) % MR], d - ((h0 + h1) + (h2 + h3)));
                    }
                }
            }
        }
    }
    {
        // ring slots of the last steps (runtime L): through a local copy
        IO Rl[MR], Hl[MR];
#pragma unroll
        for (int p = 0; p < MR; ++p) {
            Rl[p] = R[p];
            Hl[p] = H[p];
        }
#pragma unroll
        for (int i = 0; i < M; ++i) {
            z[i] = Rl[(L - 1 - i) % MR];
            if (WITH_H) ht[i] = Hl[(L - M + i) % MR];
        }
    }
    if constexpr (!WITH_H) return;
    // h(L .. L+M-1): zero input
#pragma unroll
    for (int n = 0; n < M; ++n) {
        IO acc = (IO)0;
#pragma unroll
        for (int i = 1; i <= M; ++i) acc = fma(a[i - 1], ht[M + n - i], acc);
        ht[M + n] = -acc;
    }
}

// exit state of a piece entered in state x (x[i] = y(-1-i)): Z(x) + z
template <typename IO, int M>
__device__ __forceinline__ void fwp_exit(const IO (&a)[M], const IO (&ht)[2 * M], const IO (&z)[M],
                                         const IO (&x)[M], IO (&out)[M]) {
#if TVLP_FW_CARRY64 == 1
    using AC = double;  // the carry's dot products in fp64 (one rounding per exit)
#else
    using AC = IO;
#endif
#if TVLP_FW_CARRY64 == 2
    using AS = double;  // only the exit sums in fp64
#else
    using AS = AC;
#endif
    AC q[M];
#pragma unroll
    for (int k = 1; k <= M; ++k) {
        AC v = (AC)x[k - 1];
#pragma unroll
        for (int i = 1; i <= M - k; ++i) v = fma((AC)a[i - 1], (AC)x[k - 1 + i], v);
        q[k - 1] = v;
    }
#pragma unroll
    for (int j = 0; j < M; ++j) {
        AS v = (AS)z[j];
#pragma unroll
        for (int k = 1; k <= M; ++k) v = fma((AS)q[k - 1], (AS)ht[M - 1 - j + k], v);
        out[j] = (IO)v;
    }
}

// Entry states of the P pieces of each frame (lanes 4f .. 4f+3): piece 0
// (forward) or P-1 (reverse) starts from zero; the others receive their
// neighbour's exit through shuffles, one piece per step.
template <typename IO, int M, bool REV>
__device__ __forceinline__ void fwp_carry(const IO (&a)[M], const IO (&ht)[2 * M],
                                          const IO (&z)[M], int p, IO (&xe)[M]) {
    IO xo[M];
#pragma unroll
    for (int i = 0; i < M; ++i) {
        xe[i] = (IO)0;
        xo[i] = z[i];  // exit of a piece entered at rest
    }
#pragma unroll 1
    for (int s = 1; s < kFwP; ++s) {
        const int tgt = REV ? kFwP - 1 - s : s;  // the piece whose entry is settled now
#pragma unroll
        for (int i = 0; i < M; ++i) {
            const IO c = REV ? __shfl_down_sync(0xffffffffu, xo[i], 1)
                             : __shfl_up_sync(0xffffffffu, xo[i], 1);
            if (p == tgt) xe[i] = c;
        }
        if (s + 1 < kFwP && p == tgt) fwp_exit<IO, M>(a, ht, z, xe, xo);
    }
}

template <typename IO, int M>
__global__ void __launch_bounds__(kFwpThreads)
k_fwp_forward(IO* __restrict__ seg, const IO* __restrict__ e, const IO* __restrict__ frames,
              const IO* __restrict__ win, int64_t T, int F, int nfr, int size, int hop,
              int n_lead, IO* __restrict__ aux) {
    grid_dep_wait();
    using S = FwpSmem<IO>;
    constexpr int W = kFwW;
    constexpr int MR = (M + W - 1) / W * W;
    constexpr int WPB = MR / W;
    extern __shared__ __align__(128) unsigned char fw_smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int p = lane & (kFwP - 1);
    const int fc = tid / kFwP;  // frame within the CTA (kFwP lanes each)
    const int64_t b = blockIdx.y;
    const int fi0 = blockIdx.x * kFwpFrames;
    const int fi = fi0 + fc;
    const bool active = fi < nfr;
    const int L = size / kFwP;
    const int hst = fw_stride<IO>(hop);
    const int lp = fwp_lpad<IO>(L);
    IO* es = reinterpret_cast<IO*>(fw_smem);
    IO* ws = reinterpret_cast<IO*>(fw_smem + S::off_win(size, hop));
    uint64_t* sbar = reinterpret_cast<uint64_t*>(fw_smem + S::off_bar(size, hop));
    const int row = max(fi - n_lead, 0);
    IO a[M];
#pragma unroll
    for (int i = 0; i < M; ++i) a[i] = active ? frames[(b * F + row) * M + i] : (IO)0;
    fwp_stage<IO, false>(es, e + b * T, (int64_t)(fi0 - n_lead) * hop,
                         fwp_blocks(size, hop), T, hop, (IO)1, ws, win, L, lp, sbar);
    (void)warp;
    // input of window kw of this piece: window * e over the staged span
    const IO* wsp = ws + p * lp;
    const int nspan = fwp_blocks(size, hop) * hst;  // staged elements
    auto in = [&](int kw, IO (&xv)[W]) {
        const int o0 = fc * hop + p * L + kw;  // span offset of the window's first sample
        const int q0 = o0 / hop, r0 = o0 - q0 * hop;
#pragma unroll
        for (int u = 0; u < W; ++u) {
            const int r = r0 + u;
            const int ix = q0 * hst + r + (r >= hop ? hst - hop : 0);
            TVLP_ASSERT(ix >= 0 && ix < nspan && kw + u < L);
            xv[u] = es[ix] * wsp[kw + u];
        }
    };
    IO z[M], ht[2 * M], xe[M];
    fwp_pass1<IO, M>(a, L, in, z, ht);
    // the frame's impulse-response tail, for the backward (same row, same L)
    if (aux != nullptr && active && p == 0) {
        IO* dst = aux + (b * nfr + fi) * (int64_t)(2 * M);
#pragma unroll
        for (int i = 0; i < 2 * M; ++i) dst[i] = ht[i];
    }
    fwp_carry<IO, M, false>(a, ht, z, p, xe);
    // pass 2: from the carried-in state, outputs to the frame's row
    IO R[MR];
#pragma unroll
    for (int q = 0; q < MR; ++q) R[q] = (IO)0;
#pragma unroll
    for (int i = 0; i < M; ++i) R[MR - 1 - i] = xe[i];
    IO* out = seg + ((b * nfr + fi) * (int64_t)size + p * L);
    const int nwin = L / W;
    for (int kb = 0; kb < nwin; kb += WPB) {
#pragma unroll
        for (int w = 0; w < WPB; ++w) {
            const int k = kb + w;
            if (k < nwin) {
                IO xv[W], ov[W];
                in(k * W, xv);
#pragma unroll
                for (int u = 0; u < W; ++u) {
                    const int pos = w * W + u;
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
                        fma(-a[0], R[(pos - 1 + MR) % MR], xv[u] - ((p0 + p1) + (p2 + p3)));
                    R[pos % MR] = v;
                    ov[u] = v;
                }
                TVLP_ASSERT(!active || p * L + k * W + W <= size);
                if (active) fw_store_window<IO, W>(out + k * W, ov, W);
            }
        }
    }
}

template <typename IO, int M, bool HT = false>
__global__ void __launch_bounds__(kFwpThreads)
k_fwp_backward(IO* __restrict__ gew, IO* __restrict__ gapart, const IO* __restrict__ seg,
               const IO* __restrict__ gout, const IO* __restrict__ frames,
               const IO* __restrict__ win, int64_t T, int F, int nfr, int size, int hop,
               int n_lead, IO cola, const IO* __restrict__ aux) {
    grid_dep_wait();
    using S = FwpSmem<IO>;
    constexpr int W = kFwW;
    constexpr int NBK = (M + 1 + W - 1) / W;  // blocks below the window that the lags reach
    constexpr int NRB = NBK + 1;              // those and the window's own
    constexpr int SR = NRB * W;
    extern __shared__ __align__(128) unsigned char fw_smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int p = lane & (kFwP - 1);
    const int fc = tid / kFwP;
    const int64_t b = blockIdx.y;
    const int fi0 = blockIdx.x * kFwpFrames;
    const int fi = fi0 + fc;
    const bool active = fi < nfr;
    const int L = size / kFwP;
    const int hst = fw_stride<IO>(hop);
    const int lp = fwp_lpad<IO>(L);
    IO* gs = reinterpret_cast<IO*>(fw_smem);
    IO* ws = reinterpret_cast<IO*>(fw_smem + S::off_win(size, hop));
    uint64_t* sbar = reinterpret_cast<uint64_t*>(fw_smem + S::off_bar(size, hop));
    const int row = max(fi - n_lead, 0);
    IO a[M];
#pragma unroll
    for (int i = 0; i < M; ++i) a[i] = active ? frames[(b * F + row) * M + i] : (IO)0;
    fwp_stage<IO, true>(gs, gout + b * T, (int64_t)(fi0 - n_lead) * hop,
                        fwp_blocks(size, hop), T, hop, cola, ws, win, L, lp, sbar);
    (void)warp;
    const int kend = (p + 1) * L;  // the piece covers k in [kend - L, kend), walked downward
    // pass 1 input, reversed time m: g(kend - 1 - m)
    const int nspan = fwp_blocks(size, hop) * hst;  // staged elements
    auto in = [&](int mw, IO (&xv)[W]) {
        const int o0 = fc * hop + kend - 1 - mw;  // span offset of the window's first (top) sample
        const int q0 = o0 / hop, r0 = o0 - q0 * hop;
#pragma unroll
        for (int u = 0; u < W; ++u) {
            const int r = r0 - u;
            const int ix = q0 * hst + r - (r < 0 ? hst - hop : 0);
            TVLP_ASSERT(ix >= 0 && ix < nspan);
            xv[u] = gs[ix];
        }
    };
    IO z[M], ht[2 * M], xe[M];
    if constexpr (HT) {
        // the forward saved this frame's impulse-response tail: one chain here
#pragma unroll
        for (int i = 0; i < 2 * M; ++i)
            ht[i] = active ? aux[(b * nfr + fi) * (int64_t)(2 * M) + i] : (IO)0;
        fwp_pass1<IO, M, decltype(in), false>(a, L, in, z, ht);
    } else {
        fwp_pass1<IO, M>(a, L, in, z, ht);
    }
    fwp_carry<IO, M, true>(a, ht, z, p, xe);
    // pass 2 (push form): lam[i] = -sum_{j > i} a_j ge(k + j - i) entering
    // step k, from the entry state xe[i] = ge(kend + i)
    IO lam[M], ga[M];
#pragma unroll
    for (int i = 0; i < M; ++i) {
        IO v = (IO)0;
#pragma unroll
        for (int j = i + 1; j <= M; ++j) v = fma(-a[j - 1], xe[j - i - 1], v);
        lam[i] = v;
        ga[i] = (IO)0;
    }
    const IO* srow = seg + (b * nfr + fi) * (int64_t)size;  // this frame's saved outputs
    IO* grow = gew + (b * nfr + fi) * (int64_t)size;
    const IO* wsp = ws + p * lp;
    // saved outputs s(k) for 0 <= k < size (zero below: frames start at rest)
    auto sload = [&](int k0, IO (&v)[W]) {
        TVLP_ASSERT(k0 + W <= size);
        if (k0 >= 0 && active) {
            constexpr int V = 16 / (int)sizeof(IO);
#pragma unroll
            for (int q = 0; q < W / V; ++q) {
                if constexpr (sizeof(IO) == 4) {
                    const float4 t = __ldcs(reinterpret_cast<const float4*>(srow + k0) + q);
                    v[4 * q] = t.x; v[4 * q + 1] = t.y; v[4 * q + 2] = t.z; v[4 * q + 3] = t.w;
                } else {
                    const double2 t = __ldcs(reinterpret_cast<const double2*>(srow + k0) + q);
                    v[2 * q] = t.x; v[2 * q + 1] = t.y;
                }
            }
        } else {
#pragma unroll
            for (int u = 0; u < W; ++u) v[u] = (IO)0;
        }
    };
    // ring of NRB W-blocks of saved outputs: the current window's and the NBK
    // below it (the lags reach M samples down); block j below the top window
    // lives in ring block (NBK - j) mod NRB, so with NRB windows unrolled
    // every index is static.  The block that replaces a finished window is
    // prefetched one window ahead.
    // sv[i] = s(kw - NBK*W + i): the current window's saved outputs and the
    // NBK blocks below (the lags reach M samples down), a shift register
    // moved down one block per window (one window of code: it stays in the
    // instruction cache); the next two blocks below are prefetched
    IO sv[SR];
    const int nwin = L / W;
    const int kw0 = kend - W;  // top window
    {
        IO t[W];
#pragma unroll
        for (int j = 0; j <= NBK; ++j) {
            sload(kw0 - j * W, t);
#pragma unroll
            for (int u = 0; u < W; ++u) sv[(NBK - j) * W + u] = t[u];
        }
    }
    IO pf0[W], pf1[W];
    sload(kw0 - NRB * W, pf0);
    sload(kw0 - (NRB + 1) * W, pf1);
#pragma unroll 1
    for (int wi = 0; wi < nwin; ++wi) {
        const int kw = kw0 - wi * W;
        IO gv[W], wk[W], ov[W];
        {
            const int o0 = fc * hop + kw;
            const int q0 = o0 / hop, r0 = o0 - q0 * hop;
#pragma unroll
            for (int u = 0; u < W; ++u) {
                const int r = r0 + u;
                gv[u] = gs[q0 * hst + r + (r >= hop ? hst - hop : 0)];
                wk[u] = wsp[kw - p * L + u];
            }
        }
#pragma unroll
        for (int u = W - 1; u >= 0; --u) {
            const IO l0 = lam[0] + gv[u];
            ov[u] = l0 * wk[u];
#pragma unroll
            for (int c = 0; c < M; ++c) ga[c] = fma(sv[NBK * W + u - 1 - c], l0, ga[c]);
#pragma unroll
            for (int i = 0; i < M - 1; ++i) lam[i] = fma(-a[i], l0, lam[i + 1]);
            lam[M - 1] = -a[M - 1] * l0;
        }
        TVLP_ASSERT(kw >= 0 && kw + W <= size && kw - p * L >= 0 && kw - p * L + W <= L);
        if (active) fw_store_window<IO, W>(grow + kw, ov, W);
#pragma unroll
        for (int i = SR - 1; i >= W; --i) sv[i] = sv[i - W];
#pragma unroll
        for (int u = 0; u < W; ++u) {
            sv[u] = pf0[u];
            pf0[u] = pf1[u];
        }
        sload(kw - (NRB + 2) * W, pf1);
    }
    // the frame's partial correlations, summed in piece order
#pragma unroll
    for (int c = 0; c < M; ++c) {
        IO v = ga[c];
#pragma unroll
        for (int d = 1; d < kFwP; ++d) v += __shfl_down_sync(0xffffffffu, ga[c], d);
        ga[c] = v;
    }
    if (active && p == 0) {
#pragma unroll
        for (int c = 0; c < M; ++c) gapart[(b * nfr + fi) * M + c] = -ga[c];
    }
}
