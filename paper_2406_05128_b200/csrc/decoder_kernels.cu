// decoder_kernels.cu -- the decoder pieces around the LP that profiled hot
// in the config-5 step, float32.
// First the two that took ~2.6 of the torch step's 6.2 ms (a float64
// cumsum, table gathers, the x4 decimation conv and its dgrad, the depthwise
// global FIR and its backward); further down the MSS framing and loss
// terms, the noise shaping's framing / overlap-add / spectra product and the
// HpN source pair:
//
//  * the wavetable oscillator (source.py:224-318): the table phase in float64
//    (the frame-rate f0 track is linear inside a frame, so its running sum is a
//    per-frame prefix plus a closed-form quadratic -- no sequential scan), the
//    bilinear table read and the x`OS` windowed-sinc decimation in ONE kernel:
//    the oversampled track only ever lives in shared memory.  Its VJP to the
//    table-position frames (the only trainable input; f0 is not
//    differentiated, source.py:301-303) recomputes the row difference and
//    folds the transposed decimation, the read's VJP and the upsample VJP
//    (params.py:135-145) into per-frame block sums, then one 2-term combine.
//  * the per-item causal global FIR (source.py:445-466, y[n] = sum_k h[k]
//    x[n-k]) and its VJP (grad_x: the correlation with h; grad_h[k] = sum_n
//    g[n] x[n-k], per-tile partials reduced in a fixed order).
//
// Roofline: all of it is a few hundred MB of HBM per step and < 2 GFLOP of
// FFMA; the kernels are sized so neither the gathers nor shared memory
// bandwidth dominate (register-blocked FIR tiles: 31 LDS per 128 FFMA).
#include <algorithm>

#include "common.cuh"
#include "decoder_launch.cuh"

namespace tvlp {

// ---------------------------------------------------------------- oscillator

// sum over frame g's hop_os samples of the linear f0 track (params.py:107-117:
// w = n / hop_os, the last frame held)
__device__ __forceinline__ double frame_sum(const double* f0, int64_t F, int64_t g, int hop_os) {
    const double a = f0[g], b = g + 1 < F ? f0[g + 1] : a;
    return (double)hop_os * a + (b - a) * (0.5 * (double)(hop_os - 1));
}

// sum_{h < g} frame_sum(h), by one full warp
__device__ double frame_prefix(const double* f0, int64_t F, int64_t g, int hop_os) {
    const int lane = threadIdx.x & 31;
    double s = 0.0;
#pragma unroll 8
    for (int64_t h = lane; h < g; h += 32) s += frame_sum(f0, F, h, hop_os);
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
}

// phase (periods, mod 1, rounded to float32 like the torch path's .to(f32))
// of oversampled sample n inside frame g whose prefix is P
__device__ __forceinline__ float osc_phase(const double* f0, const OscGeo& g_, int64_t fr,
                                           int n, double P) {
    const double a = f0[fr];
    const double d = fr + 1 < g_.F ? f0[fr + 1] - a : 0.0;
    const double nn = (double)n;
    const double cum = P + (nn + 1.0) * a + d * (nn * (nn + 1.0) * 0.5) * g_.inv_hop;
    const double ph = cum * g_.inv_rate;
    return (float)(ph - floor(ph));
}

// bilinear read (source.py:241-262, decoder._WavetableRead) -> (out, high - low)
__device__ __forceinline__ float2 table_read(const float* __restrict__ tab, int K, int L,
                                             float pos, float ph) {
    const float p = fminf(fmaxf(pos, 0.f), (float)(K - 1));
    const int r0 = min((int)floorf(p), K - 1);
    const int r1 = min(r0 + 1, K - 1);
    const float wr = __fsub_rn(p, (float)r0);
    const float x = __fmul_rn(ph, (float)L);
    const float fx = floorf(x);
    int i0 = (int)fx;  // x in [0, L]: the phase is in [0, 1]
    if (i0 >= L) i0 -= L;
    const int i1 = i0 + 1 == L ? 0 : i0 + 1;
    const float wi = __fsub_rn(x, fx), wi1 = __fsub_rn(1.f, wi);
    const float low = __fadd_rn(__fmul_rn(wi1, __ldg(tab + r0 * L + i0)),
                                __fmul_rn(wi, __ldg(tab + r0 * L + i1)));
    const float high = __fadd_rn(__fmul_rn(wi1, __ldg(tab + r1 * L + i0)),
                                 __fmul_rn(wi, __ldg(tab + r1 * L + i1)));
    return make_float2(__fadd_rn(__fmul_rn(__fsub_rn(1.f, wr), low), __fmul_rn(wr, high)),
                       __fsub_rn(high, low));
}

// the upsampled position track (decoder._Upsample forward)
__device__ __forceinline__ float pos_track(const float* pos, const OscGeo& g_, int64_t fr, int n) {
    const float w = fr == g_.F - 1 ? 0.f : __fmul_rn((float)n, g_.inv_hop_f);
    const float a = pos[fr], b = fr + 1 < g_.F ? pos[fr + 1] : a;
    return __fadd_rn(__fmul_rn(__fsub_rn(1.f, w), a), __fmul_rn(w, b));
}

constexpr int kOscThreads = 256;

__host__ __device__ __forceinline__ int osc_taps_u4(int nt, int os) {
    return ((nt + os - 1) / os + 3) & ~3;
}
// polyphase columns of one CTA's span: outputs t < hop read columns t + u, u < U4
__host__ __device__ __forceinline__ int osc_span_cols(int hop, int u4) { return hop + u4; }

// frames one CTA's oversampled span (at most NR samples) can touch
__host__ __device__ __forceinline__ int osc_span_frames(int NR, int hop_os) {
    return (NR / hop_os + 3) & ~1;  // even: the float rows after it stay 16-byte aligned
}

// One CTA per (frame f, item b): output samples [f*hop, f*hop + hop) need the
// oversampled samples [OS*m0 + gd - (nt-1), OS*(m1-1) + gd]; they are computed
// into shared memory in polyphase order (raw[r][v] = sample OS*v + r of the
// span) so the decimation dot reads consecutive words across the warp.
template <int OS>
__global__ void __launch_bounds__(kOscThreads)
k_osc_fwd(const double* __restrict__ f0, const float* __restrict__ pos,
          const float* __restrict__ tab, const float* __restrict__ taps, float* __restrict__ sig,
          OscGeo g) {
    extern __shared__ __align__(16) unsigned char osc_sm[];
    grid_dep_wait();
    const int64_t f = blockIdx.x, b = blockIdx.y;
    const int64_t m0 = f * g.hop;
    const int nm = (int)min((int64_t)g.hop, g.n_out - m0);
    if (nm <= 0) return;
    const int64_t ilo = OS * m0 + g.gd - (g.nt - 1);
    const int NR = OS * (nm - 1) + g.nt;
    const int NRmax = OS * (g.hop - 1) + g.nt;
    const int U4 = osc_taps_u4(g.nt, OS);           // taps per phase, padded to 4
    const int NVp = osc_span_cols(g.hop, U4);        // columns per phase (zero padded)
    double* Pf = reinterpret_cast<double*>(osc_sm);
    float* hq = reinterpret_cast<float*>(Pf + osc_span_frames(NRmax, g.hop_os));  // [OS][U4]
    float* raw = hq + OS * U4;                                                     // [OS][NVp]
    const double* f0b = f0 + b * g.F;
    const float* posb = pos + b * g.F;
    const int64_t ia = ilo > 0 ? ilo : (int64_t)0, ib = min((int64_t)ilo + NR, g.n_os) - 1;
    const int64_t gl = ia / g.hop_os, gh = ib / g.hop_os;
    TVLP_ASSERT(gh - gl + 1 <= osc_span_frames(NRmax, g.hop_os));
    if (threadIdx.x < 32) {
        const double P0 = frame_prefix(f0b, g.F, gl, g.hop_os);
        if (threadIdx.x == 0) {
            double P = P0;
            for (int64_t h = gl; h <= gh; ++h) {
                Pf[h - gl] = P;
                P += frame_sum(f0b, g.F, h, g.hop_os);
            }
        }
    }
    // polyphase taps: hq[r][u] = h[nt-1-(OS u + r)] (0 past the end)
    for (int j = threadIdx.x; j < OS * U4; j += blockDim.x) {
        const int r = j / U4, u = j % U4, q = OS * u + r;
        hq[j] = q < g.nt ? taps[g.nt - 1 - q] : 0.f;
    }
    __syncthreads();
    const int64_t gbase = gl * g.hop_os;
    for (int idx = threadIdx.x; idx < OS * NVp; idx += blockDim.x) {
        const int64_t i = ilo + idx;
        float v = 0.f;
        if (idx < NR && i >= 0 && i < g.n_os) {
            const int loc = (int)(i - gbase);
            const int k = loc / g.hop_os;
            const int n = loc - k * g.hop_os;
            const float ph = osc_phase(f0b, g, gl + k, n, Pf[k]);
            v = table_read(tab, g.K, g.L, pos_track(posb, g, gl + k, n), ph).x;
        }
        raw[(idx % OS) * NVp + idx / OS] = v;
    }
    __syncthreads();
    // sig[m0 + t] = sum_j h[j] raw_full[gd + OS(m0+t) - j] = sum_q h[nt-1-q] span[OS t + q]
    //             = sum_r sum_u hq[r][u] raw[r][t + u]
    for (int t = threadIdx.x; t < nm; t += blockDim.x) {
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int r = 0; r < OS; ++r) {
            const float* hr = hq + r * U4;
            const float* xr = raw + r * NVp + t;
            for (int u = 0; u < U4; u += 4) {
                const float4 h4 = *reinterpret_cast<const float4*>(hr + u);
                acc[0] = fmaf(h4.x, xr[u], acc[0]);
                acc[1] = fmaf(h4.y, xr[u + 1], acc[1]);
                acc[2] = fmaf(h4.z, xr[u + 2], acc[2]);
                acc[3] = fmaf(h4.w, xr[u + 3], acc[3]);
            }
        }
        sig[b * g.n_out + m0 + t] = (acc[0] + acc[1]) + (acc[2] + acc[3]);
    }
}

// VJP: one CTA per (frame f, item b) over the frame's oversampled samples i:
// gr[i] = sum_m g[m] h[gd + OS m - i] (the transposed decimation,
// source.py:285-291), times the row difference, reduced into the two block
// sums of the upsample VJP: part[b][f] = (sum (1-w) gr*d, sum w gr*d).
template <int OS>
__global__ void __launch_bounds__(kOscThreads)
k_osc_vjp(const double* __restrict__ f0, const float* __restrict__ pos,
          const float* __restrict__ tab, const float* __restrict__ taps,
          const float* __restrict__ gsig, float* __restrict__ part, OscGeo g) {
    extern __shared__ __align__(16) unsigned char osc_sm[];
    __shared__ float red[2][kOscThreads / 32];
    __shared__ double Psh;
    grid_dep_wait();
    const int64_t f = blockIdx.x, b = blockIdx.y;
    const int64_t i0 = f * g.hop_os;
    const int ni = (int)min((int64_t)g.hop_os, g.n_os - i0);
    const int U4 = osc_taps_u4(g.nt, OS);
    // [OS][U4 + 4]: hp[j0][u] = h[j0 + OS u]; the lanes of a warp read OS rows
    // at once, so rows are skewed by 4 words (distinct banks for LDS.128)
    const int HS = U4 + 4;
    float* hp = reinterpret_cast<float*>(osc_sm);
    float* gs = hp + OS * HS;
    const double* f0b = f0 + b * g.F;
    const float* posb = pos + b * g.F;
    // m range: floor((i0 - gd) / OS) .. (i0 + ni - 1 - gd + nt - 1) / OS
    const int64_t d0 = i0 - g.gd;
    const int64_t mb = d0 >= 0 ? d0 / OS : -((-d0 + OS - 1) / OS);
    const int NG = (int)((i0 + ni - 1 - g.gd + g.nt - 1 - mb * OS) / OS) + 1;
    if (threadIdx.x < 32) {
        const double P = frame_prefix(f0b, g.F, f, g.hop_os);
        if (threadIdx.x == 0) Psh = P;
    }
    for (int j = threadIdx.x; j < OS * U4; j += blockDim.x) {
        const int q = (j / U4) + OS * (j % U4);
        hp[(j / U4) * HS + j % U4] = q < g.nt ? taps[q] : 0.f;
    }
    for (int v = threadIdx.x; v < NG + U4; v += blockDim.x) {
        const int64_t m = mb + v;
        gs[v] = (m >= 0 && m < g.n_out) ? gsig[b * g.n_out + m] : 0.f;
    }
    __syncthreads();
    const double P = Psh;
    float sa = 0.f, sb = 0.f;
    for (int n = threadIdx.x; n < ni; n += blockDim.x) {
        const int64_t d = i0 + n - g.gd;
        const int64_t mf = d >= 0 ? (d + OS - 1) / OS : -((-d) / OS);  // ceil(d / OS)
        const int j0 = (int)(mf * OS - d);                               // in [0, OS)
        const int v0 = (int)(mf - mb);
        float acc = 0.f;
        const float* hr = hp + j0 * HS;
        const float* gr = gs + v0;
        float a4[4] = {0.f, 0.f, 0.f, 0.f};
        for (int u = 0; u < U4; u += 4) {
            const float4 h4 = *reinterpret_cast<const float4*>(hr + u);
            a4[0] = fmaf(h4.x, gr[u], a4[0]);
            a4[1] = fmaf(h4.y, gr[u + 1], a4[1]);
            a4[2] = fmaf(h4.z, gr[u + 2], a4[2]);
            a4[3] = fmaf(h4.w, gr[u + 3], a4[3]);
        }
        acc = (a4[0] + a4[1]) + (a4[2] + a4[3]);
        const float ph = osc_phase(f0b, g, f, n, P);
        const float dl = table_read(tab, g.K, g.L, pos_track(posb, g, f, n), ph).y;
        const float gp = __fmul_rn(acc, dl);
        const float w = f == g.F - 1 ? 0.f : __fmul_rn((float)n, g.inv_hop_f);
        sa = fmaf(__fsub_rn(1.f, w), gp, sa);
        sb = fmaf(w, gp, sb);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        sa += __shfl_xor_sync(0xffffffffu, sa, o);
        sb += __shfl_xor_sync(0xffffffffu, sb, o);
    }
    const int wid = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        red[0][wid] = sa;
        red[1][wid] = sb;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        float a = 0.f, c = 0.f;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
            a += red[0][w];
            c += red[1][w];
        }
        part[(b * g.F + f) * 2 + 0] = a;
        part[(b * g.F + f) * 2 + 1] = c;
    }
}

// grad_pos[b][f] = part[b][f].a + part[b][f-1].b  (decoder._Upsample backward)
__global__ void k_osc_combine(const float* __restrict__ part, float* __restrict__ gpos,
                              int64_t B, int64_t F) {
    grid_dep_wait();
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= B * F) return;
    const int64_t f = r % F;
    gpos[r] = part[2 * r] + (f > 0 ? part[2 * (r - 1) + 1] : 0.f);
}

inline size_t osc_fwd_smem(const OscGeo& g, int os) {
    const int NR = os * (g.hop - 1) + g.nt;
    const int u4 = osc_taps_u4(g.nt, os);
    return osc_span_frames(NR, g.hop_os) * sizeof(double) +
           ((size_t)os * u4 + (size_t)os * osc_span_cols(g.hop, u4)) * sizeof(float);
}
inline size_t osc_vjp_smem(const OscGeo& g, int os) {
    const int u4 = osc_taps_u4(g.nt, os);
    const int NG = (g.hop_os + g.nt + 2 * os) / os + 2 + u4;
    return ((size_t)os * (u4 + 4) + (size_t)NG) * sizeof(float);
}

// ---------------------------------------------------------------- FIR rows
// Per-row FIRs: the decoder's global FIR (source.py:445-466, one 128-tap
// filter per item) and the noise shaping's frame FIRs (source.py:367-428,
// one 510-tap filter per 960-sample frame) share these kernels:
//   y[n] = sum_{k<m} h[k] x[n + off - k],  n in [0, ny),  x = 0 outside [0, nx)
// (global FIR: off 0, nx = ny = n; noise frames: off = the FIR's 255-sample
// delay, nx = ny = frame size), its adjoint to x (ADJ, off 0) and the tap
// gradient grad_h[k] = sum_n g[n] x[n + off - k].
constexpr int kFirThreads = 128;
constexpr int kFirKB = 8;                        // taps per register block
constexpr int kFirMaxTaps = 1024;
template <int J>
struct FirTile {
    static constexpr int TILE = kFirThreads * J;  // outputs per CTA (J = 16: 2048, 8: 1024)
};

// shared-memory skew: one pad word per 16 (thread t's rows start 17t apart:
// conflict-free across the warp)
__device__ __forceinline__ int skew(int y) { return y + (y >> 4); }

template <bool ADJ, int J>
__global__ void __launch_bounds__(kFirThreads)
k_fir(const float* __restrict__ x, const float* __restrict__ taps, float* __restrict__ y,
      int64_t n, int m, int off) {
    extern __shared__ __align__(16) float fir_sm[];
    grid_dep_wait();
    constexpr int TILE = FirTile<J>::TILE;
    const int mp = (m + kFirKB - 1) / kFirKB * kFirKB;
    const int64_t b = blockIdx.y, n0 = (int64_t)blockIdx.x * TILE;
    float* hs = fir_sm;           // [mp]
    float* xs = fir_sm + mp;      // skewed [TILE + mp]
    const float* xb = x + b * n;
    const float* hb = taps + b * m;
    for (int k = threadIdx.x; k < mp; k += blockDim.x) hs[k] = k < m ? hb[k] : 0.f;
    const int NX = TILE + mp;
    const int64_t s0 = ADJ ? n0 : n0 + off - (mp - 1);   // first staged sample
    for (int e = threadIdx.x; e < NX; e += blockDim.x) {
        const int64_t idx = s0 + e;
        xs[skew(e)] = (idx >= 0 && idx < n) ? xb[idx] : 0.f;
    }
    __syncthreads();
    const int base = threadIdx.x * J;
    float acc[J];
#pragma unroll
    for (int j = 0; j < J; ++j) acc[j] = 0.f;
    for (int kb = 0; kb < mp; kb += kFirKB) {
        float hv[kFirKB];
#pragma unroll
        for (int kk = 0; kk < kFirKB; ++kk) hv[kk] = hs[kb + kk];
        float xr[J + kFirKB - 1];
        // fwd: staged index of x[n0+base+j+off-k] = base + j - k + mp - 1, k = kb + kk
        //      = (base + mp - kb - KB) + (j - kk + KB - 1)
        // adj: staged index of x[n0+base+j+k] = base + kb + (j + kk)
        const int e0 = ADJ ? base + kb : base + mp - kb - kFirKB;
#pragma unroll
        for (int e = 0; e < J + kFirKB - 1; ++e) xr[e] = xs[skew(e0 + e)];
#pragma unroll
        for (int kk = 0; kk < kFirKB; ++kk)
#pragma unroll
            for (int j = 0; j < J; ++j)
                acc[j] = fmaf(hv[kk], xr[ADJ ? j + kk : j - kk + kFirKB - 1], acc[j]);
    }
    float* yb = y + b * n + n0 + base;
    if (n0 + base + J <= n && ((reinterpret_cast<uintptr_t>(yb) & 15) == 0)) {
#pragma unroll
        for (int j = 0; j < J; j += 4)
            *reinterpret_cast<float4*>(yb + j) = make_float4(acc[j], acc[j + 1], acc[j + 2],
                                                             acc[j + 3]);
    } else {
#pragma unroll
        for (int j = 0; j < J; ++j)
            if (n0 + base + j < n) yb[j] = acc[j];
    }
}

// grad_h partials: part[b][tile][k] = sum_{n in tile} g[n] x[n + off - k].
// Thread t: taps [16 kb, 16 kb + 16) (kb = t % 8) over n-slice t / 8 of
// TILE/16 samples; the 16 slices are summed in shared memory in a fixed
// order; taps beyond 128 loop the k window.
constexpr int kTapJ = 16, kTapSlices = kFirThreads / 8, kTapWin = 128;
template <int J>
__global__ void __launch_bounds__(kFirThreads)
k_fir_taps_part(const float* __restrict__ g, const float* __restrict__ x, float* __restrict__ part,
                int64_t n, int m, int off, int ntiles) {
    extern __shared__ __align__(16) float fir_sm[];
    grid_dep_wait();
    constexpr int TILE = FirTile<J>::TILE, SLICE = TILE / kTapSlices;
    const int64_t b = blockIdx.y, n0 = (int64_t)blockIdx.x * TILE;
    const int mw = kTapWin;
    float* gs = fir_sm;                       // skewed [TILE]
    float* xs = gs + skew(TILE) + 1;          // skewed [TILE + mw]
    float* red = xs + skew(TILE + mw) + 1;    // [kTapSlices][mw]
    const int kb = threadIdx.x % 8, sl = threadIdx.x / 8;
    for (int e = threadIdx.x; e < TILE; e += blockDim.x) {
        const int64_t idx = n0 + e;
        gs[skew(e)] = idx < n ? g[b * n + idx] : 0.f;
    }
    for (int k0 = 0; k0 < m; k0 += mw) {
        __syncthreads();
        // staged x[n0 + off - k0 - mw + e], e in [0, TILE + mw)
        for (int e = threadIdx.x; e < TILE + mw; e += blockDim.x) {
            const int64_t idx = n0 + off - k0 - mw + e;
            xs[skew(e)] = (idx >= 0 && idx < n) ? x[b * n + idx] : 0.f;
        }
        __syncthreads();
        float acc[kTapJ];
#pragma unroll
        for (int j = 0; j < kTapJ; ++j) acc[j] = 0.f;
        for (int s = 0; s < SLICE; s += 8) {
            const int nl = sl * SLICE + s;   // local n of this 8-block
            float gv[8], xr[8 + kTapJ - 1];
#pragma unroll
            for (int q = 0; q < 8; ++q) gv[q] = gs[skew(nl + q)];
            // x[n + off - k] for n = n0 + nl + q, k = k0 + 16 kb + j: staged e = nl + q - 16 kb - j + mw
            const int e0 = nl + mw - 16 * kb - (kTapJ - 1);
#pragma unroll
            for (int e = 0; e < 8 + kTapJ - 1; ++e) xr[e] = xs[skew(e0 + e)];
#pragma unroll
            for (int q = 0; q < 8; ++q)
#pragma unroll
                for (int j = 0; j < kTapJ; ++j)
                    acc[j] = fmaf(gv[q], xr[q - j + kTapJ - 1], acc[j]);
        }
#pragma unroll
        for (int j = 0; j < kTapJ; ++j) red[sl * mw + 16 * kb + j] = acc[j];
        __syncthreads();
        for (int k = threadIdx.x; k < mw; k += blockDim.x) {
            float s = 0.f;
            for (int q = 0; q < kTapSlices; ++q) s += red[q * mw + k];
            if (k0 + k < m) part[(b * ntiles + blockIdx.x) * (int64_t)m + k0 + k] = s;
        }
    }
}

__global__ void k_fir_taps_reduce(const float* __restrict__ part, float* __restrict__ gh,
                                  int64_t B, int m, int ntiles) {
    grid_dep_wait();
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= B * m) return;
    const int64_t b = r / m, k = r % m;
    float s = 0.f;
    for (int t = 0; t < ntiles; ++t) s += part[(b * ntiles + t) * (int64_t)m + k];
    gh[r] = s;
}

// ---------------------------------------------------------------- launchers
namespace {
template <typename K>
cudaError_t allow_smem(K kernel, size_t bytes) {
    if (bytes > 227 * 1024) return cudaErrorInvalidValue;  // (very long hops)
    return bytes > 48 * 1024 ? cudaFuncSetAttribute(kernel,
                                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                    (int)bytes)
                             : cudaSuccess;
}
}  // namespace

cudaError_t launch_osc_fwd(const double* f0, const float* pos, const float* tab,
                           const float* taps, float* sig, const OscGeo& g, int os,
                           cudaStream_t st) {
    if (os != 4) return cudaErrorInvalidValue;
    const size_t sm = osc_fwd_smem(g, os);
    cudaError_t e = allow_smem(k_osc_fwd<4>, sm);
    if (e != cudaSuccess) return e;
    e = launch_pdl(k_osc_fwd<4>, dim3((unsigned)g.F, (unsigned)g.B), kOscThreads, sm, st, f0, pos,
                   tab, taps, sig, g);
    return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_osc_vjp(const double* f0, const float* pos, const float* tab,
                           const float* taps, const float* gsig, float* part, float* gpos,
                           const OscGeo& g, int os, cudaStream_t st) {
    if (os != 4) return cudaErrorInvalidValue;
    const size_t sm = osc_vjp_smem(g, os);
    cudaError_t e = allow_smem(k_osc_vjp<4>, sm);
    if (e != cudaSuccess) return e;
    e = launch_pdl(k_osc_vjp<4>, dim3((unsigned)g.F, (unsigned)g.B), kOscThreads, sm, st, f0, pos,
                   tab, taps, gsig, part, g);
    if (e != cudaSuccess) return e;
    const int64_t rows = g.B * g.F;
    e = launch_pdl(k_osc_combine, dim3((unsigned)((rows + 255) / 256)), 256, 0, st,
                   (const float*)part, gpos, g.B, g.F);
    return e != cudaSuccess ? e : cudaGetLastError();
}

// rows up to 1024 samples (the noise frames) use the 1024-output tile
int fir_j(int64_t n) { return n <= 1024 ? 8 : 16; }
int fir_tiles(int64_t n) {
    const int tile = kFirThreads * fir_j(n);
    return (int)((n + tile - 1) / tile);
}

template <bool ADJ, int J>
cudaError_t launch_fir_j(const float* x, const float* taps, float* y, int64_t B, int64_t n, int m,
                         int off, cudaStream_t st) {
    const int mp = (m + kFirKB - 1) / kFirKB * kFirKB;
    const int NX = FirTile<J>::TILE + mp;
    const size_t sm = (mp + NX + NX / 16 + 1) * sizeof(float);
    cudaError_t e = allow_smem(k_fir<ADJ, J>, sm);
    if (e == cudaSuccess)
        e = launch_pdl(k_fir<ADJ, J>, dim3((unsigned)fir_tiles(n), (unsigned)B), kFirThreads, sm,
                       st, x, taps, y, n, m, off);
    return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_fir(const float* x, const float* taps, float* y, int64_t B, int64_t n, int m,
                       bool adj, int off, cudaStream_t st) {
    if (m < 1 || m > kFirMaxTaps || (adj && off != 0)) return cudaErrorInvalidValue;
    if (fir_j(n) == 8)
        return adj ? launch_fir_j<true, 8>(x, taps, y, B, n, m, off, st)
                   : launch_fir_j<false, 8>(x, taps, y, B, n, m, off, st);
    return adj ? launch_fir_j<true, 16>(x, taps, y, B, n, m, off, st)
               : launch_fir_j<false, 16>(x, taps, y, B, n, m, off, st);
}

size_t fir_taps_part_elems(int64_t B, int64_t n, int m) { return (size_t)B * fir_tiles(n) * m; }

template <int J>
cudaError_t launch_fir_taps_j(const float* g, const float* x, float* part, int64_t B, int64_t n,
                              int m, int off, cudaStream_t st) {
    constexpr int TILE = FirTile<J>::TILE;
    const size_t sm = ((TILE + TILE / 16 + 1) + (TILE + kTapWin + (TILE + kTapWin) / 16 + 1) +
                       kTapSlices * kTapWin) * sizeof(float);
    cudaError_t e = allow_smem(k_fir_taps_part<J>, sm);
    if (e == cudaSuccess)
        e = launch_pdl(k_fir_taps_part<J>, dim3((unsigned)fir_tiles(n), (unsigned)B), kFirThreads,
                       sm, st, g, x, part, n, m, off, fir_tiles(n));
    return e;
}

cudaError_t launch_fir_taps(const float* g, const float* x, float* part, float* gh, int64_t B,
                            int64_t n, int m, int off, cudaStream_t st) {
    if (m < 1 || m > kFirMaxTaps) return cudaErrorInvalidValue;
    cudaError_t e = fir_j(n) == 8 ? launch_fir_taps_j<8>(g, x, part, B, n, m, off, st)
                                  : launch_fir_taps_j<16>(g, x, part, B, n, m, off, st);
    if (e == cudaSuccess)
        e = launch_pdl(k_fir_taps_reduce, dim3((unsigned)((B * m + 255) / 256)), 256, 0, st,
                       (const float*)part, gh, B, m, fir_tiles(n));
    return e != cudaSuccess ? e : cudaGetLastError();
}

// ---------------------------------------------------------------- MSS loss terms
// One FFT size of the multi-resolution spectral loss (loss.py:105-126) from
// the one-sided spectra X (signal, differentiated) and Y (target), complex
// [B][n] interleaved (n = frames x bins per item):
//   term_b = sqrt(sum (|X|-|Y|)^2) / max(sqrt(sum |Y|^2), 1e-12)
//          + mean |log(|X| + eps) - log(|Y| + eps)|
// and its VJP to X: g_b [ (|X|-|Y|) / (sqrt(S1) ynorm) + sgn(lx - ly) /
// (n (|X| + eps)) ] X / |X|  (0 where |X| = 0, like the reference's phase
// mask, loss.py:71-73).  Replaces ~25 elementwise passes of the torch graph
// (magnitudes, the two norms, logs, the absolute mean and their backward) by
// one reduction pass and one gradient pass.
constexpr int kMssThreads = 256;

__device__ __forceinline__ float mss_mag(float2 z) { return sqrtf(z.x * z.x + z.y * z.y); }

__global__ void __launch_bounds__(kMssThreads)
k_mss_reduce(const float2* __restrict__ X, const float2* __restrict__ Y, int64_t n, float eps,
             float* __restrict__ part, int nchunk) {
    grid_dep_wait();
    const int64_t b = blockIdx.y;
    const int64_t lo = n * blockIdx.x / nchunk, hi = n * (blockIdx.x + 1) / nchunk;
    const float2* xb = X + b * n;
    const float2* yb = Y + b * n;
    // four independent elements per iteration (the loop was latency-bound:
    // IPC 1.1 with one dependent load pair in flight per thread)
    float s1 = 0.f, s2 = 0.f, s3 = 0.f;
    const int64_t step = blockDim.x;
    int64_t i = lo + threadIdx.x;
    for (; i + 3 * step < hi; i += 4 * step) {
        float2 xv[4], yv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            xv[u] = xb[i + u * step];
            yv[u] = yb[i + u * step];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const float mx = mss_mag(xv[u]), my = mss_mag(yv[u]);
            const float d = mx - my;
            s1 = fmaf(d, d, s1);
            s2 = fmaf(my, my, s2);
            s3 += fabsf(__logf(mx + eps) - __logf(my + eps));  // (MUFU: ~1e-6 absolute)
        }
    }
    for (; i < hi; i += step) {
        const float mx = mss_mag(xb[i]), my = mss_mag(yb[i]);
        const float d = mx - my;
        s1 = fmaf(d, d, s1);
        s2 = fmaf(my, my, s2);
        s3 += fabsf(__logf(mx + eps) - __logf(my + eps));
    }
    __shared__ float red[3][kMssThreads / 32];
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
        s3 += __shfl_xor_sync(0xffffffffu, s3, o);
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        red[0][w] = s1;
        red[1][w] = s2;
        red[2][w] = s3;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        float t = 0.f;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += red[threadIdx.x][k];
        part[(b * nchunk + blockIdx.x) * 3 + threadIdx.x] = t;
    }
}

// per item, chunks summed in a fixed order (double): term[b]; aux[b] =
// (sqrt(S1), ynorm, n, 0) for the VJP
__global__ void k_mss_finish(const float* __restrict__ part, int nchunk, int64_t B, int64_t n,
                             float* __restrict__ term, float* __restrict__ aux) {
    grid_dep_wait();
    const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    double s1 = 0.0, s2 = 0.0, s3 = 0.0;
    for (int c = 0; c < nchunk; ++c) {
        const float* q = part + (b * nchunk + c) * 3;
        s1 += q[0];
        s2 += q[1];
        s3 += q[2];
    }
    const double r1 = sqrt(s1), yn = fmax(sqrt(s2), 1e-12);
    term[b] = (float)(r1 / yn + s3 / (double)n);
    aux[b * 4 + 0] = (float)r1;
    aux[b * 4 + 1] = (float)yn;
    aux[b * 4 + 2] = (float)n;
    aux[b * 4 + 3] = 0.f;
}

__global__ void __launch_bounds__(kMssThreads)
k_mss_grad(const float2* __restrict__ X, const float2* __restrict__ Y,
           const float* __restrict__ aux, const float* __restrict__ gterm, int64_t B, int64_t n,
           float eps, float2* __restrict__ gX) {
    grid_dep_wait();
    const int64_t b = blockIdx.x;   // grid: (items, element blocks of 4 x 256): no division
    const float g = gterm[b];
    const float r1 = aux[b * 4 + 0], yn = aux[b * 4 + 1];
    // per-item factors; two reciprocals per element instead of four divisions
    const float c_la = g / (float)n, c_sc = r1 > 0.f ? g / (r1 * yn) : 0.f;
    const int64_t k0 = (int64_t)blockIdx.y * 4 * blockDim.x + threadIdx.x;
    float2 xv[4], yv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {   // four independent elements in flight
        const int64_t k = k0 + u * blockDim.x;
        xv[u] = k < n ? X[b * n + k] : make_float2(0.f, 0.f);
        yv[u] = k < n ? Y[b * n + k] : make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int64_t k = k0 + u * blockDim.x;
        if (k >= n) break;
        const float mx = mss_mag(xv[u]), my = mss_mag(yv[u]);
        const float dl = __logf(mx + eps) - __logf(my + eps);
        const float sg = dl > 0.f ? 1.f : (dl < 0.f ? -1.f : 0.f);
        const float gm = fmaf(c_sc, mx - my, c_la * sg * __frcp_rn(mx + eps));
        const float q = mx > 0.f ? gm * __frcp_rn(mx) : 0.f;
        gX[b * n + k] = make_float2(q * xv[u].x, q * xv[u].y);
    }
}

int mss_chunks(int64_t n) { return (int)std::min<int64_t>(64, std::max<int64_t>(1, n / 4096)); }

size_t mss_part_floats(int64_t B, int64_t n) { return (size_t)B * mss_chunks(n) * 3; }

cudaError_t launch_mss_terms(const float* X, const float* Y, int64_t B, int64_t n, float eps,
                             float* term, float* aux, float* part, cudaStream_t st) {
    const int nc = mss_chunks(n);
    cudaError_t e = launch_pdl(k_mss_reduce, dim3((unsigned)nc, (unsigned)B), kMssThreads, 0, st,
                               reinterpret_cast<const float2*>(X),
                               reinterpret_cast<const float2*>(Y), n, eps, part, nc);
    if (e == cudaSuccess)
        e = launch_pdl(k_mss_finish, dim3((unsigned)((B + 127) / 128)), 128, 0, st,
                       (const float*)part, nc, B, n, term, aux);
    return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_mss_terms_vjp(const float* X, const float* Y, const float* aux,
                                 const float* gterm, int64_t B, int64_t n, float eps, float* gX,
                                 cudaStream_t st) {
    cudaError_t e = launch_pdl(k_mss_grad,
                               dim3((unsigned)B, (unsigned)((n + 4 * kMssThreads - 1) / (4 * kMssThreads))),
                               kMssThreads, 0, st, reinterpret_cast<const float2*>(X),
                               reinterpret_cast<const float2*>(Y), aux, gterm, B, n, eps,
                               reinterpret_cast<float2*>(gX));
    return e != cudaSuccess ? e : cudaGetLastError();
}

// ---------------------------------------------------------------- STFT frames
// stft_mag's framing (loss.py:46-63): reflect-padded by N/2, frames of N at
// `hop`, times the window -- one pass writing the FFT input (the torch graph
// pads, unfolds and multiplies: three), and its adjoint: each signal sample
// gathers, in a fixed order, the windowed frame gradients of the padded
// positions that map to it (itself and its reflections in the pads,
// loss.py:81-86), scaled by `scale` (the caller's inverse-FFT normalisation).
__device__ __forceinline__ int64_t reflect_index(int64_t i, int64_t n) {
    if (i < 0) i = -i;
    if (i >= n) i = 2 * (n - 1) - i;
    return i;
}

// grid: (frames, column blocks, items) -- no division per element (a 64-bit
// division per thread made these kernels issue-bound: ~16 us of 27 per call)
__global__ void k_stft_frames(const float* __restrict__ x, const float* __restrict__ win,
                              float* __restrict__ fr, int64_t B, int64_t n, int N, int hop,
                              int64_t nfr) {
    grid_dep_wait();
    const int64_t f = blockIdx.x, b = blockIdx.z;
    const int64_t row = b * nfr + f;
    const int64_t t0 = f * hop - N / 2;
    // 4 columns per thread (independent loads in flight)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int j = (blockIdx.y * 4 + q) * blockDim.x + threadIdx.x;
        if (j < N) fr[row * N + j] = x[b * n + reflect_index(t0 + j, n)] * win[j];
    }
}

// grad of padded position p: sum over frames f with 0 <= p - f hop < N of
// win[j] (scale gframe[f][j] + dc_scale dc[f])  (dc: nullable per-frame term)
__device__ __forceinline__ float stft_pad_grad(const float* __restrict__ gfb,
                                               const float* __restrict__ win,
                                               const float* __restrict__ dcb, int64_t dcs,
                                               float scale, float dc_scale, int p, int N,
                                               int hop, int nfr) {
    int f1 = p / hop;
    if (f1 > nfr - 1) f1 = nfr - 1;
    int f0 = p - (N - 1);
    f0 = f0 <= 0 ? 0 : (f0 + hop - 1) / hop;
    float s = 0.f;
    for (int f = f0; f <= f1; ++f) {
        const int j = p - f * hop;
        float v = gfb[(int64_t)f * N + j] * scale;
        if (dcb != nullptr) v = fmaf(dc_scale, dcb[f * dcs], v);
        s = fmaf(v, win[j], s);
    }
    return s;
}

__global__ void k_stft_frames_vjp(const float* __restrict__ gfr, const float* __restrict__ win,
                                  float* __restrict__ gx, int64_t B, int64_t n, int N, int hop,
                                  int64_t nfr, float scale, const float* __restrict__ dc,
                                  int64_t dcs, float dc_scale) {
    grid_dep_wait();
    const int64_t b = blockIdx.x;
    const int t = blockIdx.y * blockDim.x + threadIdx.x;   // (n < 2^31: 32-bit index math)
    if (t >= n) return;
    const int64_t i = b * n + t;
    const int pad = N / 2, nn = (int)n, nf = (int)nfr;
    const float* gfb = gfr + b * nfr * N;
    const float* dcb = dc == nullptr ? nullptr : dc + b * nfr * dcs;
    // padded positions mapping to t: t + pad; pad - t (left mirror, 1 <= t <= pad);
    // pad + 2(n-1) - t (right mirror, n-1-pad <= t <= n-2)
    float s = stft_pad_grad(gfb, win, dcb, dcs, scale, dc_scale, t + pad, N, hop, nf);
    if (t >= 1 && t <= pad)
        s += stft_pad_grad(gfb, win, dcb, dcs, scale, dc_scale, pad - t, N, hop, nf);
    if (t <= nn - 2 && t >= nn - 1 - pad)
        s += stft_pad_grad(gfb, win, dcb, dcs, scale, dc_scale, pad + 2 * (nn - 1) - t, N, hop,
                           nf);
    gx[i] = s;
}

cudaError_t launch_stft_frames(const float* x, const float* win, float* fr, int64_t B, int64_t n,
                               int N, int hop, cudaStream_t st) {
    const int64_t nfr = 1 + (n + 2 * (N / 2) - N) / hop;
    cudaError_t e = launch_pdl(k_stft_frames, dim3((unsigned)nfr, (unsigned)((N + 1023) / 1024), (unsigned)B),
                               256, 0, st, x, win, fr, B, n, N, hop, nfr);
    return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_stft_frames_vjp(const float* gfr, const float* win, float* gx, int64_t B,
                                   int64_t n, int N, int hop, float scale, const float* dc,
                                   int64_t dcs, float dc_scale, cudaStream_t st) {
    const int64_t nfr = 1 + (n + 2 * (N / 2) - N) / hop;
    cudaError_t e = launch_pdl(k_stft_frames_vjp, dim3((unsigned)B, (unsigned)((n + 255) / 256)),
                               256, 0, st, gfr, win, gx, B, n, N, hop, nfr, scale, dc, dcs,
                               dc_scale);
    return e != cudaSuccess ? e : cudaGetLastError();
}

// ---------------------------------------------------------------- noise frames
// shape_noise's framing and overlap-add (source.py:367-428) for hop-spaced
// frames (frame i starts at sample s_i = start0 + i hop; samples outside
// [0, n) are zero / dropped):
//   frames[b][i][j] = noise[b][s_i + j] win[j] for j < size, 0 up to nfft
//     (the FFT input, zero-padded in the same pass);
//   out[b][t] = inv_cola sum_{i: 0 <= t - s_i < size} y[b][i][t - s_i + delay]
//     (a fixed-order gather: no scatter, no atomics) and its adjoint.
__global__ void k_noise_frames(const float* __restrict__ noise, const float* __restrict__ win,
                               float* __restrict__ fr, int64_t B, int64_t n, int64_t nfr,
                               int size, int nfft, int64_t start0, int hop) {
    grid_dep_wait();
    const int64_t f = blockIdx.x, b = blockIdx.z;           // grid: (frames, columns, items)
    const int64_t row = b * nfr + f;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int j = (blockIdx.y * 4 + q) * blockDim.x + threadIdx.x;
        if (j >= nfft) break;
        const int64_t t = start0 + f * hop + j;
        fr[row * nfft + j] = (j < size && t >= 0 && t < n) ? noise[b * n + t] * win[j] : 0.f;
    }
}

__global__ void k_frame_ola(const float* __restrict__ y, float* __restrict__ out, int64_t B,
                            int64_t n, int64_t nfr, int size, int ld, int delay, int64_t start0,
                            int hop, float inv_cola) {
    grid_dep_wait();
    const int64_t b = blockIdx.x;                            // grid: (items, samples)
    const int64_t t = (int64_t)blockIdx.y * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const int64_t i = b * n + t;
    // frames with 0 <= t - start0 - f hop < size
    const int64_t u = t - start0;
    int64_t f1 = u / hop;
    if (f1 > nfr - 1) f1 = nfr - 1;
    int64_t f0 = u - (size - 1);
    f0 = f0 <= 0 ? 0 : (f0 + hop - 1) / hop;
    float s = 0.f;
    const float* yb = y + b * nfr * ld;
    for (int64_t f = f0; f <= f1; ++f) s += yb[f * ld + (u - f * hop) + delay];
    out[i] = s * inv_cola;
}

__global__ void k_frame_ola_vjp(const float* __restrict__ g, float* __restrict__ gy, int64_t B,
                                int64_t n, int64_t nfr, int size, int ld, int delay,
                                int64_t start0, int hop, float inv_cola) {
    grid_dep_wait();
    const int64_t f = blockIdx.x, b = blockIdx.z;          // grid: (frames, columns, items)
    const int64_t row = b * nfr + f;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int jc = (blockIdx.y * 4 + q) * blockDim.x + threadIdx.x;
        if (jc >= ld) break;
        const int j = jc - delay;
        const int64_t t = start0 + f * hop + j;
        gy[row * ld + jc] = (j >= 0 && j < size && t >= 0 && t < n) ? g[b * n + t] * inv_cola : 0.f;
    }
}

cudaError_t launch_noise_frames(const float* noise, const float* win, float* fr, int64_t B,
                                int64_t n, int64_t nfr, int size, int nfft, int64_t start0, int hop,
                                cudaStream_t st) {
    cudaError_t e = launch_pdl(k_noise_frames,
                               dim3((unsigned)nfr, (unsigned)((nfft + 1023) / 1024), (unsigned)B), 256, 0,
                               st, noise, win, fr, B, n, nfr, size, nfft, start0, hop);
    return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_frame_ola(const float* y, float* out, int64_t B, int64_t n, int64_t nfr,
                             int size, int ld, int delay, int64_t start0, int hop, float inv_cola,
                             bool adj, cudaStream_t st) {
    cudaError_t e;
    if (!adj)
        e = launch_pdl(k_frame_ola, dim3((unsigned)B, (unsigned)((n + 255) / 256)), 256, 0, st, y,
                       out, B, n, nfr, size, ld, delay, start0, hop, inv_cola);
    else
        e = launch_pdl(k_frame_ola_vjp, dim3((unsigned)nfr, (unsigned)((ld + 1023) / 1024), (unsigned)B),
                       256, 0, st, y, out, B, n, nfr, size, ld, delay, start0, hop, inv_cola);
    return e != cudaSuccess ? e : cudaGetLastError();
}

// ---------------------------------------------------------------- noise spectra
// The frame FIRs' spectra applied to the noise frames' spectra
// (source.py:404-412, FFT convolution): P[b][i] = S[b][i] * H[b][rows[i]]
// (complex, K bins; rows[i] = the frame's FIR row, lead-in frames share row
// 0) without materialising H[:, rows]; the VJP to H sums, in frame order,
// gP * conj(S) over the frames that use each row (rows is nondecreasing, so
// row f's frames are the contiguous range first[f] .. first[f+1]-1).
__global__ void k_spec_mul(const float2* __restrict__ S, const float2* __restrict__ H,
                           const int* __restrict__ rows, float2* __restrict__ P, int64_t nfr,
                           int64_t F, int K) {
    grid_dep_wait();
    const int64_t i = blockIdx.x, b = blockIdx.z;        // grid: (frames, bins, items)
    const int k = blockIdx.y * blockDim.x + threadIdx.x;
    if (k >= K) return;
    const float2 s = S[(b * nfr + i) * K + k];
    const float2 h = H[(b * F + rows[i]) * K + k];
    P[(b * nfr + i) * K + k] = make_float2(s.x * h.x - s.y * h.y, s.x * h.y + s.y * h.x);
}

__global__ void k_spec_mul_vjp(const float2* __restrict__ gP, const float2* __restrict__ S,
                               const int* __restrict__ first, float2* __restrict__ gH,
                               int64_t nfr, int64_t F, int K) {
    grid_dep_wait();
    const int64_t f = blockIdx.x, b = blockIdx.z;        // grid: (rows, bins, items)
    const int k = blockIdx.y * blockDim.x + threadIdx.x;
    if (k >= K) return;
    float2 acc = make_float2(0.f, 0.f);
    for (int i = first[f]; i < first[f + 1]; ++i) {
        const float2 g = gP[(b * nfr + i) * K + k];
        const float2 s = S[(b * nfr + i) * K + k];
        // g * conj(s)
        acc.x += g.x * s.x + g.y * s.y;
        acc.y += g.y * s.x - g.x * s.y;
    }
    gH[(b * F + f) * K + k] = acc;
}

cudaError_t launch_spec_mul(const float* S, const float* H, const int* rows, const int* first,
                            float* out, int64_t B, int64_t nfr, int64_t F, int K, bool adj,
                            cudaStream_t st) {
    cudaError_t e;
    if (!adj)
        e = launch_pdl(k_spec_mul, dim3((unsigned)nfr, (unsigned)((K + 255) / 256), (unsigned)B),
                       256, 0, st, reinterpret_cast<const float2*>(S),
                       reinterpret_cast<const float2*>(H), rows, reinterpret_cast<float2*>(out), nfr,
                       F, K);
    else  // S: the output gradient gP, H: the noise spectra S
        e = launch_pdl(k_spec_mul_vjp, dim3((unsigned)F, (unsigned)((K + 255) / 256), (unsigned)B),
                       256, 0, st, reinterpret_cast<const float2*>(S),
                       reinterpret_cast<const float2*>(H), first, reinterpret_cast<float2*>(out),
                       nfr, F, K);
    return e != cudaSuccess ? e : cudaGetLastError();
}

// ---------------------------------------------------------------- HpN source pair
// The HpN decoder's two LP inputs (synth.py:264-273 with the paper's C(z),
// decoder.Decoder.render) in one pass: rows b < B: H(t) (sig(t) V(t)), rows
// B + b: noise(t) G(t), zero from T1 to Tp = F hop, where V, G, H are the
// upsampled gain frames (params.py:107-132: w = j / hop, held last frame) --
// instead of three upsampled tracks, three products and the stacking copy.
// The VJP writes grad_sig, grad_noise and, per (item, frame block), the six
// weighted block sums of the three gain tracks' gradients; a combine adds
// each frame's two intervals (params.py:135-145).
__device__ __forceinline__ float gain_at(const float* __restrict__ fr, int64_t F, int64_t f,
                                         float w) {
    const float a = fr[f];
    const float b = f + 1 < F ? fr[f + 1] : a;
    return __fadd_rn(__fmul_rn(__fsub_rn(1.f, w), a), __fmul_rn(w, b));
}

__global__ void k_source_pair(const float* __restrict__ sig, const float* __restrict__ noise,
                              const float* __restrict__ vg, const float* __restrict__ ng,
                              const float* __restrict__ hg, float* __restrict__ out, int64_t B,
                              int64_t T1, int64_t F, int hop, int64_t Tp) {
    grid_dep_wait();
    const int64_t f = blockIdx.x, b = blockIdx.y;   // grid: (frame blocks, items)
    const float inv_hop = 1.f / (float)hop;
    for (int j = threadIdx.x; j < hop; j += blockDim.x) {
        const int64_t t = f * hop + j;
        if (t >= Tp) break;
        float o0 = 0.f, o1 = 0.f;
        if (t < T1) {
            const float w = f == F - 1 ? 0.f : __fmul_rn((float)j, inv_hop);
            const float V = gain_at(vg + b * F, F, f, w), H = gain_at(hg + b * F, F, f, w);
            const float G = gain_at(ng + b * F, F, f, w);
            o0 = __fmul_rn(H, __fmul_rn(sig[b * T1 + t], V));
            o1 = __fmul_rn(noise[b * T1 + t], G);
        }
        out[b * Tp + t] = o0;
        out[(B + b) * Tp + t] = o1;
    }
}

__global__ void k_source_pair_vjp(const float* __restrict__ g, const float* __restrict__ sig,
                                  const float* __restrict__ noise, const float* __restrict__ vg,
                                  const float* __restrict__ ng, const float* __restrict__ hg,
                                  float* __restrict__ gsig, float* __restrict__ gnoise,
                                  float* __restrict__ part, int64_t B, int64_t T1, int64_t F,
                                  int hop, int64_t Tp) {
    grid_dep_wait();
    const int64_t f = blockIdx.x, b = blockIdx.y;
    const float inv_hop = 1.f / (float)hop;
    float acc[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // (1-w), w sums of dV, dH, dG
    for (int j = threadIdx.x; j < hop; j += blockDim.x) {
        const int64_t t = f * hop + j;
        if (t >= T1) break;
        const float w = f == F - 1 ? 0.f : __fmul_rn((float)j, inv_hop);
        const float V = gain_at(vg + b * F, F, f, w), H = gain_at(hg + b * F, F, f, w);
        const float G = gain_at(ng + b * F, F, f, w);
        const float gt = g[b * Tp + t], gb = g[(B + b) * Tp + t];
        const float sv = sig[b * T1 + t], nv = noise[b * T1 + t];
        const float sV = __fmul_rn(sv, V);
        gsig[b * T1 + t] = __fmul_rn(__fmul_rn(gt, H), V);
        gnoise[b * T1 + t] = __fmul_rn(gb, G);
        const float dV = __fmul_rn(__fmul_rn(gt, H), sv), dH = __fmul_rn(gt, sV);
        const float dG = __fmul_rn(gb, nv);
        const float w1 = __fsub_rn(1.f, w);
        acc[0] = fmaf(w1, dV, acc[0]);
        acc[1] = fmaf(w, dV, acc[1]);
        acc[2] = fmaf(w1, dH, acc[2]);
        acc[3] = fmaf(w, dH, acc[3]);
        acc[4] = fmaf(w1, dG, acc[4]);
        acc[5] = fmaf(w, dG, acc[5]);
    }
    __shared__ float red[6][8];
#pragma unroll
    for (int q = 0; q < 6; ++q)
#pragma unroll
        for (int o = 16; o; o >>= 1) acc[q] += __shfl_xor_sync(0xffffffffu, acc[q], o);
    const int wid = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0)
#pragma unroll
        for (int q = 0; q < 6; ++q) red[q][wid] = acc[q];
    __syncthreads();
    if (threadIdx.x < 6) {
        float tsum = 0.f;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) tsum += red[threadIdx.x][k];
        part[(b * F + f) * 6 + threadIdx.x] = tsum;
    }
}

// grad of gain frames: X[b][f] = part[b][f].(1-w)X + part[b][f-1].wX
__global__ void k_source_pair_combine(const float* __restrict__ part, float* __restrict__ gv,
                                      float* __restrict__ gh, float* __restrict__ gn, int64_t B,
                                      int64_t F) {
    grid_dep_wait();
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= B * F) return;
    const int64_t f = r % F;
    const float* p = part + r * 6;
    const float* q = f > 0 ? part + (r - 1) * 6 : nullptr;
    gv[r] = p[0] + (q ? q[1] : 0.f);
    gh[r] = p[2] + (q ? q[3] : 0.f);
    gn[r] = p[4] + (q ? q[5] : 0.f);
}

cudaError_t launch_source_pair(const float* sig, const float* noise, const float* vg,
                               const float* ng, const float* hg, float* out, int64_t B, int64_t T1,
                               int64_t F, int hop, int64_t Tp, cudaStream_t st) {
    cudaError_t e = launch_pdl(k_source_pair, dim3((unsigned)F, (unsigned)B), 256, 0, st, sig, noise,
                               vg, ng, hg, out, B, T1, F, hop, Tp);
    return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_source_pair_vjp(const float* g, const float* sig, const float* noise,
                                   const float* vg, const float* ng, const float* hg, float* gsig,
                                   float* gnoise, float* gvg, float* gng, float* ghg, float* part,
                                   int64_t B, int64_t T1, int64_t F, int hop, int64_t Tp,
                                   cudaStream_t st) {
    cudaError_t e = launch_pdl(k_source_pair_vjp, dim3((unsigned)F, (unsigned)B), 256, 0, st, g, sig,
                               noise, vg, ng, hg, gsig, gnoise, part, B, T1, F, hop, Tp);
    if (e == cudaSuccess)
        e = launch_pdl(k_source_pair_combine, dim3((unsigned)((B * F + 255) / 256)), 256, 0, st,
                       (const float*)part, gvg, ghg, gng, B, F);
    return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace tvlp
