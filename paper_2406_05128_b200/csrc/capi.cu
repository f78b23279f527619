// capi.cu -- the C ABI (include/tvlp.h): argument checks, workspace carving,
// layout normalisation (T padded to a multiple of 4, M padded to a compiled
// order, 16-byte alignment) and the launch sequences of each operation.
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/tvlp.h"
#include "chain_launch.cuh"
#include "decoder_launch.cuh"
#include "framewise_launch.cuh"
#include "lp_scan.cuh"

namespace tvlp {
template <typename IO>
cudaError_t launch_step_up(const IO* k, IO* a, int64_t rows, int M, int* bad, cudaStream_t st);
template <typename IO>
cudaError_t launch_step_up_vjp(const IO* ga, const IO* k, IO* gk, int64_t rows, int M,
                               cudaStream_t st);
}  // namespace tvlp
#include "scan_launch.cuh"

namespace tvlp {
namespace {

thread_local int g_last_cuda = 0;

inline int fail_cuda(cudaError_t e) {
    g_last_cuda = (int)e;
    return TVLP_ERR_CUDA;
}
#define TVLP_CK(x)                                   \
    do {                                             \
        cudaError_t e__ = (x);                       \
        if (e__ != cudaSuccess) return fail_cuda(e__); \
    } while (0)

constexpr int kMaxOrder = 30;

// ---------------------------------------------------------------- instrumentation
std::atomic<int64_t> g_launches{0};
std::atomic<int> g_prof_on{0};
struct ProfRec {
    const char* name;
    cudaEvent_t a, b;
};
std::mutex g_prof_mu;
std::vector<ProfRec> g_prof;

// Run a launcher, count its kernels and (if enabled) bracket it with events.
template <typename F>
cudaError_t tracked(const char* name, int nkernels, cudaStream_t st, F&& launch) {
    g_launches += nkernels;
    if (!g_prof_on.load()) return launch();
    ProfRec r{name, nullptr, nullptr};
    cudaEventCreate(&r.a);
    cudaEventCreate(&r.b);
    cudaEventRecord(r.a, st);
    cudaError_t err = launch();
    cudaEventRecord(r.b, st);
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof.push_back(r);
    return err;
}
#define TVLP_RUN(name, nk, st, call) TVLP_CK(tracked(name, nk, st, [&]() { return (call); }))

// ---------------------------------------------------------------- geometry
struct Plan {
    int64_t B = 0, T = 0, Tp = 0;
    int M = 0, Mp = 0;
    int Ls = 0, nsub = 0;
};

// Sub-chunk length: a multiple of 8 dividing T (so all sub-chunks are full and
// uniformly strided for the 2-D tensor TMA), closest to the target (512, or
// $TVLP_SUBCHUNK); if T has no such divisor, T is padded up to a multiple.
// Sub-chunk length: a multiple of 8 dividing T, closest to the target.  The
// target is ~512 (one basis wave at config 3 and 100-step carry chains),
// smaller when the batch has too few sub-chunks to fill the GPU: the
// per-sub-chunk passes are then latency-bound and scale with Ls while the
// serial carries scale with T/Ls.  Measured with the chained kernels (us per
// fwd+bwd, tools/r2_ls_small.sh): config 1 (96 k samples) Ls 480 151, 320
// 125, 240 115, 200 114, 160 113, 120 121; config 3's 8- and 4-way shares
// (384 k / 768 k samples) flat within 2% over 240-320.
int64_t choose_ls(int64_t B, int64_t T, int64_t* Tp, bool frames) {
    int64_t target = B * T >= (int64_t)4096 * 512 ? 512 : (B * T >= 200000 ? 320 : 200);
    // frame-rate rows: the lane passes interpolate rows instead of streaming
    // them and are latency-bound, so more (shorter) sub-chunks pay for the
    // longer carry chains (config 3 measured: Ls 480 396 us, 240 354 us)
    if (frames) target = B * T >= (int64_t)4096 * 512 ? 240 : 160;
    if (const char* env = std::getenv("TVLP_SUBCHUNK")) {
        const long v = std::atol(env);
        if (v >= 8) target = v;
    }
    if (T >= 256) {
        int64_t best = -1;
        for (int64_t d = 96; d <= 1024; d += 8)
            if (T % d == 0 && (best < 0 || std::llabs(d - target) < std::llabs(best - target)))
                best = d;
        if (best > 0) {
            *Tp = T;
            return best;
        }
        const int64_t Ls = (target + 7) / 8 * 8;
        *Tp = (T + Ls - 1) / Ls * Ls;
        return Ls;
    }
    const int64_t Ls = (T + 7) / 8 * 8;
    *Tp = Ls;
    return Ls;
}

bool make_plan(int64_t B, int64_t T, int M, Plan& p, bool frames = false) {
    if (B < 1 || T < 1 || M < 1 || M > kMaxOrder) return false;
    p.B = B;
    p.T = T;
    p.M = M;
    p.Mp = padded_order(M);
    p.Ls = (int)choose_ls(B, T, &p.Tp, frames);
    p.nsub = (int)(p.Tp / p.Ls);
    return true;
}

ScanArgs scan_args(const Plan& p) {
    ScanArgs g;
    g.B = p.B;
    g.T = p.Tp;
    g.Ls = p.Ls;
    g.nsub = p.nsub;
    return g;
}

// carry tape: per-sub-chunk tapes followed by one forward-refinement flag per
// sequence (an int stored in the first bytes of a B-element trailing region)
int64_t tape_body(const Plan& p) { return p.B * (int64_t)p.nsub * tape_elems(p.Mp); }
inline int64_t mp4(const Plan& p) { return (p.Mp + 3) / 4 * 4; }

// Hierarchical carry: chains longer than kSerialMax sub-chunks are cut into
// groups of kGroup whose products P_g form the next level (SURVEY.md §5 "long
// context"), recursively.  Level-l group tapes live in the carry tape after
// the level-0 tapes and the per-sequence flag slots, so the backward reuses
// the forward's group products.
int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return (v != nullptr && v[0] != 0) ? std::atoi(v) : dflt;
}
// tuning knobs (read once per process): the longest serial carry chain and
// the group length of the hierarchical scheme
const int kSerialMax = env_int("TVLP_CARRY_SERIAL_MAX", 256);
const int kGroup = env_int("TVLP_CARRY_GROUP", 32);
// single-level "auto" refinement folded into the re-apply launch (1) or as a
// separate per-sequence refine kernel before it (0)
const int kFusedRefine = env_int("TVLP_FUSED_REFINE", 1);
// frame-rate rows in the chained forward (k_fwd_chain<..., FR>): correct but
// measured slower than basis -> carry -> apply at config 5 (88 vs 79 us; the
// interpolating cursor costs registers: 255/thread); the chained adjoint with
// frame-rate rows is the faster one (74 vs 87 us) and is the default
const int kFrFwdChain = env_int("TVLP_FR_FWD_CHAIN", 0);
struct Levels {
    int L = 1;
    int64_t n[8] = {};
    int64_t off[8] = {};  // element offset of level-l tapes in the carry tape
};
Levels make_levels(const Plan& p) {
    Levels v;
    v.n[0] = p.nsub;
    v.off[0] = 0;
    int64_t cur = tape_body(p) + (p.B + 3) / 4 * 4;  // group tapes stay 16-B aligned
    while (v.n[v.L - 1] > kSerialMax && v.L < 8) {
        v.n[v.L] = (v.n[v.L - 1] + kGroup - 1) / kGroup;
        v.off[v.L] = cur;
        cur += p.B * v.n[v.L] * tape_elems(p.Mp);
        ++v.L;
    }
    return v;
}
int64_t carry_elems(const Plan& p) {
    const Levels v = make_levels(p);
    if (v.L == 1) return tape_body(p) + p.B;
    return v.off[v.L - 1] + p.B * v.n[v.L - 1] * tape_elems(p.Mp);
}

template <typename IO>
struct Hier {
    const Plan* p;
    Levels lv;
    IO* tape;           // carry tape base
    IO* U[8] = {};      // per level >= 1: group forcing / tails
    IO* V[8] = {};      // per level >= 1: group states
    const int* only = nullptr;
    cudaStream_t st = nullptr;

    IO* tape_l(int l) const { return tape + lv.off[l]; }
    CarryArgs<IO> args(int l) const {
        CarryArgs<IO> a{};
        a.tape = tape_l(l);
        a.nsub = (int)lv.n[l];
        a.only = only;
        return a;
    }
    // x(k+1) = Phi_k x(k) + f_k on level l (f = tape z rows if force == null)
    cudaError_t fwd(int l, const IO* force, const IO* x0, int64_t x0s, IO* X, unsigned* dstat,
                    int* fflags) const {
        const int64_t B = p->B;
        if (l == lv.L - 1) {
            CarryArgs<IO> a = args(l);
            a.force = force;
            a.x0 = x0;
            a.x0_stride = x0s;
            a.X = X;
            a.nseg = B;
            a.seglen = a.nsub;
            a.dstat = dstat;
            a.fflags = fflags;
            return launch_carry_fwd<IO>(p->Mp, a, st);
        }
        const int TS = tape_elems(p->Mp);
        CarryArgs<IO> t = args(l);  // group tails (zero-state group outputs)
        t.force = force;
        t.nseg = B * lv.n[l + 1];
        t.seglen = kGroup;
        t.dstat = dstat;
        t.fflags = fflags;
        if (force == nullptr) {
            t.tail = tape_l(l + 1) + (int64_t)p->Mp * mp4(*p);  // z row (Tape::Z_ROW = M)
            t.tail_stride = TS;
        } else {
            t.tail = U[l + 1];
            t.tail_stride = mp4(*p);
        }
        cudaError_t err = launch_carry_fwd<IO>(p->Mp, t, st);
        if (err != cudaSuccess) return err;
        err = fwd(l + 1, force == nullptr ? nullptr : U[l + 1], x0, x0s, V[l + 1], nullptr, nullptr);
        if (err != cudaSuccess) return err;
        CarryArgs<IO> e = args(l);  // expansion inside each group
        e.force = force;
        e.x0 = V[l + 1];
        e.x0_stride = mp4(*p);
        e.X = X;
        e.nseg = B * lv.n[l + 1];
        e.seglen = kGroup;
        return launch_carry_fwd<IO>(p->Mp, e, st);
    }
    // mu(k-1) = Phi_k^T mu(k) + nu_k on level l
    // x0 (nullable, [B][mp4]): adjoint state entering each sequence from the
    // right (a later time segment held elsewhere, longseq.py)
    cudaError_t bwd(int l, const IO* nu, IO* X, const IO* x0 = nullptr) const {
        const int64_t B = p->B;
        if (l == lv.L - 1) {
            CarryArgs<IO> a = args(l);
            a.force = nu;
            a.X = X;
            a.nseg = B;
            a.seglen = a.nsub;
            a.x0 = x0;
            a.x0_stride = mp4(*p);
            return launch_carry_bwd<IO>(p->Mp, a, st);
        }
        CarryArgs<IO> t = args(l);
        t.force = nu;
        t.tail = U[l + 1];
        t.tail_stride = mp4(*p);
        t.nseg = B * lv.n[l + 1];
        t.seglen = kGroup;
        cudaError_t err = launch_carry_bwd<IO>(p->Mp, t, st);
        if (err != cudaSuccess) return err;
        err = bwd(l + 1, U[l + 1], V[l + 1], x0);
        if (err != cudaSuccess) return err;
        CarryArgs<IO> e = args(l);
        e.force = nu;
        e.x0 = V[l + 1];
        e.x0_stride = mp4(*p);
        e.X = X;
        e.nseg = B * lv.n[l + 1];
        e.seglen = kGroup;
        return launch_carry_bwd<IO>(p->Mp, e, st);
    }
    cudaError_t compose() const {  // group products of every level
        for (int l = 0; l + 1 < lv.L; ++l) {
            cudaError_t err = launch_group_P<IO>(p->Mp, tape_l(l), tape_l(l + 1),
                                                 p->B * lv.n[l + 1], kGroup, (int)lv.n[l], only, st);
            if (err != cudaSuccess) return err;
        }
        return cudaSuccess;
    }
};

// bump allocator over the caller's workspace (nullptr base = sizing pass)
struct Carver {
    unsigned char* base;
    size_t used = 0;
    explicit Carver(void* b) : base(static_cast<unsigned char*>(b)) {}
    void* take(size_t bytes) {
        used = (used + 255) / 256 * 256;
        void* p = base ? base + used : nullptr;
        used += bytes;
        return p;
    }
};

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
inline bool base_ok(const void* p) { return p != nullptr; }

// ---------------------------------------------------------------- pack kernels
// dst[b, t, c] (Tp x Mp, zero-filled) <- src[b, t, c] (T x M)
template <typename IO>
__global__ void k_pack(const IO* __restrict__ src, IO* __restrict__ dst, int64_t B, int64_t T,
                       int M, int64_t Tp, int Mp) {
    grid_dep_wait();
    const int64_t n = B * Tp * Mp;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(i % Mp);
        const int64_t bt = i / Mp;
        const int64_t t = bt % Tp, b = bt / Tp;
        dst[i] = (t < T && c < M) ? src[(b * T + t) * M + c] : (IO)0;
    }
}
template <typename IO>
__global__ void k_unpack(const IO* __restrict__ src, IO* __restrict__ dst, int64_t B, int64_t T,
                         int M, int64_t Tp, int Mp) {
    grid_dep_wait();
    const int64_t n = B * T * M;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(i % M);
        const int64_t bt = i / M;
        const int64_t t = bt % T, b = bt / T;
        dst[i] = src[(b * Tp + t) * Mp + c];
    }
}
inline unsigned grid_for(int64_t n) {
    int64_t g = (n + 255) / 256;
    if (g > 148 * 64) g = 148 * 64;
    if (g < 1) g = 1;
    return (unsigned)g;
}
template <typename IO>
cudaError_t pack(const void* src, void* dst, int64_t B, int64_t T, int M, int64_t Tp, int Mp,
                 cudaStream_t st) {
    g_launches += 1;
    launch_pdl(k_pack<IO>, grid_for(B * Tp * Mp), 256, 0, st, static_cast<const IO*>(src),
                                                       static_cast<IO*>(dst), B, T, M, Tp, Mp);
    return cudaGetLastError();
}
template <typename IO>
cudaError_t unpack(const void* src, void* dst, int64_t B, int64_t T, int M, int64_t Tp, int Mp,
                   cudaStream_t st) {
    g_launches += 1;
    launch_pdl(k_unpack<IO>, grid_for(B * T * M), 256, 0, st, static_cast<const IO*>(src),
                                                       static_cast<IO*>(dst), B, T, M, Tp, Mp);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- small ops
template <typename IO>
__global__ void k_shift(const IO* __restrict__ A, IO* __restrict__ out, int64_t B, int64_t T,
                        int M) {
    grid_dep_wait();
    const int64_t n = B * T * M;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(i % M);
        const int64_t bt = i / M;
        const int64_t t = bt % T, b = bt / T;
        const int64_t src = t + c + 1;  // A_hat[t, i-1] = A[t+i, i-1], i = c+1
        out[i] = src < T ? A[(b * T + src) * M + c] : (IO)0;
    }
}
template <typename IO>
__global__ void k_lag(const IO* __restrict__ s, const IO* __restrict__ zi, IO* __restrict__ out,
                      int64_t B, int64_t T, int M) {
    grid_dep_wait();
    const int64_t n = B * T * M;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(i % M);
        const int64_t bt = i / M;
        const int64_t t = bt % T, b = bt / T;
        const int64_t src = t - c - 1;
        out[i] = src >= 0 ? s[b * T + src] : (zi ? zi[b * M + (c - t)] : (IO)0);
    }
}

// Phi[b][i][c] = R rows of a product tape (Tape layout: rows R_ROW + i).
template <typename IO>
__global__ void k_extract_phi(const IO* __restrict__ tape, IO* __restrict__ Phi, int64_t B, int M,
                              int mp4, int tsize, int rrow) {
    grid_dep_wait();
    const int64_t n = B * M * M;
    for (int64_t x = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int c = (int)(x % M);
        const int i = (int)((x / M) % M);
        const int64_t b = x / ((int64_t)M * M);
        Phi[x] = tape[b * tsize + (int64_t)(rrow + i) * mp4 + c];
    }
}

// Transition of a whole sequence (segment): the product of its sub-chunk
// transitions Phi_{n-1} ... Phi_0, from the top level of the carry tape.
template <typename IO>
int segment_transition_impl(const void* carry_v, const Plan& p, void* Phi, void* ws,
                            size_t ws_bytes, cudaStream_t st, size_t* need) {
    const size_t sz = sizeof(IO);
    const int TS = tape_elems(p.Mp);
    Carver c(ws);
    IO* out = static_cast<IO*>(c.take(p.B * (int64_t)TS * sz));
    if (need) {
        *need = c.used;
        return TVLP_OK;
    }
    if (ws_bytes < c.used) return TVLP_ERR_WORKSPACE;
    const Levels lv = make_levels(p);
    const IO* top = static_cast<const IO*>(carry_v) + lv.off[lv.L - 1];
    const int n = (int)lv.n[lv.L - 1];
    TVLP_CK(launch_group_P<IO>(p.Mp, top, out, p.B, n, n, nullptr, st));
    g_launches += 1;
    const int64_t tot = p.B * (int64_t)p.M * p.M;
    launch_pdl(k_extract_phi<IO>, grid_for(tot), 256, 0, st, out, static_cast<IO*>(Phi), p.B, p.M,
               (int)mp4(p), TS, p.Mp + 1);
    TVLP_CK(cudaGetLastError());
    return TVLP_OK;
}

// ---------------------------------------------------------------- TV / TI
template <typename IO>
int forward_impl(bool ti, const void* e, const void* A, const void* zi, void* s, const Plan& p,
                 void* carry_v, int prec, void* ws, size_t ws_bytes, int32_t* nonfinite,
                 cudaStream_t st, size_t* need, const FrameSrc<IO>* fr = nullptr) {
    const size_t sz = sizeof(IO);
    IO* carry = static_cast<IO*>(carry_v);
    // TVLP_CARRY_REUSE: the caller's tape already holds Phi_j and z_j for the
    // same (e, A); only zi is new, so the basis (and compose) passes are skipped
    const bool reuse_tape = (prec & TVLP_CARRY_REUSE) && carry != nullptr;
    prec &= ~TVLP_CARRY_REUSE;
    // frame-rate coefficients: rows interpolated inside the fp32 scan kernels,
    // else (fp64 I/O or fp64 chains) materialised once into the workspace
    const bool frames = fr != nullptr;
    // (frame intervals must fall on the lane kernels' 8-row windows)
    const bool native_fr = frames && std::is_same<IO, float>::value && prec != kPrecF64Chains &&
                           fr->hop % kLaneWin == 0;
    const bool packed = p.Tp != p.T || (!frames && (p.Mp != p.M || !aligned16(A))) ||
                        !aligned16(e) || !aligned16(s) || (zi && !aligned16(zi));
    const int64_t nsc = p.B * p.nsub;
    const int64_t mp = mp4(p);
    Hier<IO> h;
    h.p = &p;
    h.lv = make_levels(p);
    h.st = st;
    Carver c(ws);
    IO* phiz = carry ? carry : static_cast<IO*>(c.take(carry_elems(p) * sz));
    h.tape = phiz;
    IO* xin = static_cast<IO*>(c.take(nsc * mp * sz));
    for (int l = 1; l < h.lv.L; ++l) {
        h.U[l] = static_cast<IO*>(c.take(p.B * h.lv.n[l] * mp * sz));
        h.V[l] = static_cast<IO*>(c.take(p.B * h.lv.n[l] * mp * sz));
    }
    // precision "auto": fp32 chains + boundary-defect check + refinement (long,
    // hierarchical chains are always checked: their group products are fp32)
    const bool hier = h.lv.L > 1;
    const bool refine = sizeof(IO) == 4 && (prec == kPrecAuto || hier);
    // the chained single-pass forward (chain.cuh): fp32 I/O, sample-rate rows
    // or frame-rate rows interpolated in the kernels, one carry level, fp32
    // chains
    const bool f32 = std::is_same<IO, float>::value;
    const bool chain = f32 && (!frames || (native_fr && kFrFwdChain)) && !reuse_tape && !hier &&
                       (prec == kPrecAuto || prec == kPrecF32Chains) && chain_supported(p.Mp);
    IO* xend = (refine || (f32 && need) || chain) ? static_cast<IO*>(c.take(nsc * mp * sz)) : nullptr;
    void* ctl = (f32 && (need || chain)) ? c.take(chain_ctl_bytes(p.B, p.nsub, p.Mp)) : nullptr;
    int* fflags = reinterpret_cast<int*>(phiz + tape_body(p));  // flag slots in the carry tape
    int* flags = refine ? fflags : nullptr;
    unsigned* dstat = refine ? static_cast<unsigned*>(c.take(p.B * 2 * sizeof(unsigned))) : nullptr;
    IO* D0 = (refine && hier) ? static_cast<IO*>(c.take(nsc * mp * sz)) : nullptr;
    IO* E0 = (refine && hier) ? static_cast<IO*>(c.take(nsc * mp * sz)) : nullptr;
    const IO* e_p = static_cast<const IO*>(e);
    const IO* A_p = static_cast<const IO*>(A);
    const IO* zi_p = static_cast<const IO*>(zi);
    IO* s_p = static_cast<IO*>(s);
    void *pe = nullptr, *pA = nullptr, *ps = nullptr, *pz = nullptr;
    if (packed) {
        pe = c.take(p.B * p.Tp * sz);
        if (!frames) pA = c.take((ti ? p.B : p.B * p.Tp) * p.Mp * sz);
        ps = c.take(p.B * p.Tp * sz);
        if (zi) pz = c.take(p.B * p.Mp * sz);
    }
    // (the sizing pass reserves the materialised rows whatever the precision)
    if (frames && (!native_fr || need)) pA = c.take(p.B * p.Tp * p.Mp * sz);
    // frames mode does not pack for M != Mp, but the carry reads Mp state
    // components per row: an initial state of a padded order is zero-padded
    // into its own buffer (the sizing pass's packed layout already covers it)
    void* pz_only = (frames && zi && !packed && p.Mp != p.M) ? c.take(p.B * p.Mp * sz) : nullptr;
    if (need) {
        *need = c.used;
        return TVLP_OK;
    }
    if (ws_bytes < c.used) return TVLP_ERR_WORKSPACE;
    const ScanArgs g = scan_args(p);
    if (pz_only) {
        TVLP_CK(pack<IO>(zi, pz_only, p.B, 1, p.M, 1, p.Mp, st));
        zi_p = static_cast<const IO*>(pz_only);
    }
    if (packed) {
        TVLP_CK(pack<IO>(e, pe, p.B, p.T, 1, p.Tp, 1, st));
        if (!frames) {
            if (ti)
                TVLP_CK(pack<IO>(A, pA, p.B, 1, p.M, 1, p.Mp, st));
            else
                TVLP_CK(pack<IO>(A, pA, p.B, p.T, p.M, p.Tp, p.Mp, st));
            A_p = static_cast<const IO*>(pA);
        }
        if (zi) TVLP_CK(pack<IO>(zi, pz, p.B, 1, p.M, 1, p.Mp, st));
        e_p = static_cast<const IO*>(pe);
        zi_p = static_cast<const IO*>(pz);
        s_p = static_cast<IO*>(ps);
    }
    if (frames && !native_fr) {
        TVLP_RUN("upsample", 1, st, (launch_upsample<IO>(p.Mp, *fr, static_cast<IO*>(pA), p.B,
                                                          p.Tp, st)));
        A_p = static_cast<const IO*>(pA);
    }
    const FrameSrc<IO>* frk = native_fr ? fr : nullptr;
    if constexpr (std::is_same<IO, float>::value) {
        if (chain) {
            ChainFwdCall cc{ti, 1, {}, p.Mp, phiz, fflags, xin, xend,
                            nonfinite, ctl, prec == kPrecAuto ? 1 : 0, g};
            cc.grp[0] = ChainGroup{e_p, frames ? nullptr : A_p, zi_p, s_p, p.B};
            cc.fr = frames ? fr : nullptr;
            TVLP_RUN("basis", 2, st, (launch_fwd_chain(p.Mp, cc, st, 0)));
            TVLP_RUN("fwd_chain", 1, st, (launch_fwd_chain(p.Mp, cc, st, 1)));
            if (packed) TVLP_CK(unpack<IO>(ps, s, p.B, p.T, 1, p.Tp, 1, st));
            return TVLP_OK;
        }
    }
    const int bprec = (prec == kPrecAuto || prec == kPrecF32Chains) ? prec : kPrecF64Chains;
    if (!reuse_tape) {
        TVLP_RUN("basis", 1, st, (launch_basis<IO>(p.Mp, ti, bprec, e_p, A_p, phiz, g, st, frk)));
        if (hier) TVLP_RUN("compose", h.lv.L - 1, st, (h.compose()));
    }
    TVLP_RUN("carry_fwd", 1, st, (h.fwd(0, nullptr, zi_p, p.Mp, xin, dstat, fflags)));
    TVLP_RUN("apply_fwd", 1, st,
             (launch_apply_fwd<IO>(p.Mp, ti, e_p, A_p, xin, s_p, nonfinite, xend, dstat, nullptr, g,
                                   st, frk)));
    if (refine && !hier && kFusedRefine) {
        // flagged sequences: correction recurrence + re-apply in one launch
        RefineSrc<IO> rf;
        rf.tape = phiz;
        rf.K = xend;
        rf.dstat = dstat;
        rf.flags = flags;
        TVLP_RUN("apply_fwd_refined", 1, st,
                 (launch_apply_fwd<IO>(p.Mp, ti, e_p, A_p, xin, s_p, nullptr, nullptr, nullptr,
                                       nullptr, g, st, frk, &rf)));
    } else if (refine) {
        if (!hier) {
            TVLP_RUN("refine_fwd", 1, st,
                     (launch_refine<IO>(p.Mp, true, phiz, xin, xend, dstat, flags, nullptr, g, st)));
        } else {
            // decide, defects D = Xend - Xin(next), corrections E through the
            // same hierarchy (forced by D), Xin += E -- flagged sequences only
            TVLP_RUN("refine_fwd", 4, st, ([&]() -> cudaError_t {
                cudaError_t err = launch_refine_helpers<IO>(0, p.Mp, nullptr, nullptr, nullptr,
                                                            p.nsub, true, nullptr, flags, dstat,
                                                            nullptr, kDefectTol, p.B, st);
                if (err != cudaSuccess) return err;
                err = launch_refine_helpers<IO>(1, p.Mp, xend, xin, D0, p.nsub, true, flags,
                                                nullptr, nullptr, nullptr, 0.f, p.B, st);
                if (err != cudaSuccess) return err;
                Hier<IO> hr = h;
                hr.only = flags;
                err = hr.fwd(0, D0, nullptr, 0, E0, nullptr, nullptr);
                if (err != cudaSuccess) return err;
                return launch_refine_helpers<IO>(2, p.Mp, xin, E0, nullptr, p.nsub, true, flags,
                                                 nullptr, nullptr, nullptr, 0.f, p.B, st);
            }()));
        }
        TVLP_RUN("apply_fwd_refined", 1, st,
                 (launch_apply_fwd<IO>(p.Mp, ti, e_p, A_p, xin, s_p, nullptr, nullptr, nullptr, flags,
                                       g, st, frk)));
    }
    if (packed) TVLP_CK(unpack<IO>(ps, s, p.B, p.T, 1, p.Tp, 1, st));
    return TVLP_OK;
}

inline int grad_a_chunks(const Plan& p) {
    int64_t n = p.Tp / 2048;
    if (n < 1) n = 1;
    if (n > 256) n = 256;
    return (int)n;
}

template <typename IO>
int backward_impl(bool ti, const void* gs, const void* A, const void* s, const void* zi, void* ge,
                  void* gA, const Plan& p, const void* carry_v, int prec, void* ws,
                  size_t ws_bytes, cudaStream_t st, size_t* need,
                  const FrameSrc<IO>* fr = nullptr, const void* mu_in = nullptr,
                  void* grad_zi = nullptr) {
    // frames mode: A is the frame-rate source fr, gA receives grad_frames [B][F][M]
    const size_t sz = sizeof(IO);
    const IO* carry = static_cast<const IO*>(carry_v);
    const bool frames = fr != nullptr;
    // (without the forward's tape the basis is recomputed; the frame-rate
    // basis has fp32 chains only)
    const bool native_fr = frames && std::is_same<IO, float>::value &&
                           (carry != nullptr || prec == kPrecF32Chains) &&
                           fr->hop % kLaneWin == 0;
    const bool packed = p.Tp != p.T ||
                        (!frames && (p.Mp != p.M || !aligned16(A) || (!ti && !aligned16(gA)))) ||
                        !aligned16(gs) || !aligned16(s) || !aligned16(ge) ||
                        (zi && !aligned16(zi));
    const int64_t nsc = p.B * p.nsub;
    const int64_t mp = mp4(p);
    Hier<IO> h;
    h.p = &p;
    h.lv = make_levels(p);
    h.st = st;
    const bool hier = h.lv.L > 1;
    Carver c(ws);
    IO* phiz_own = carry ? nullptr : static_cast<IO*>(c.take(carry_elems(p) * sz));
    IO* nu = static_cast<IO*>(c.take(nsc * mp * sz));
    IO* mu = static_cast<IO*>(c.take(nsc * mp * sz));
    for (int l = 1; l < h.lv.L; ++l) {
        h.U[l] = static_cast<IO*>(c.take(p.B * h.lv.n[l] * mp * sz));
        h.V[l] = static_cast<IO*>(c.take(p.B * h.lv.n[l] * mp * sz));
    }
    // without the forward's tape (and its per-sequence refinement flags) the
    // backward recomputes the transition matrices with fp64 chains
    if (carry == nullptr && prec == kPrecAuto) prec = kPrecF64Chains;
    const bool refine = sizeof(IO) == 4 && (prec == kPrecAuto || hier);
    // the chained single-pass adjoint (chain.cuh): fp32, sample-rate rows, one
    // carry level, the forward's tape, no segment boundary terms
    const bool f32 = std::is_same<IO, float>::value;
    const bool chain = f32 && (!frames || native_fr) && carry != nullptr && !hier && !mu_in && !grad_zi &&
                       (prec == kPrecAuto || prec == kPrecF32Chains) && chain_supported(p.Mp);
    IO* kout = (refine || grad_zi || need || chain) ? static_cast<IO*>(c.take(nsc * mp * sz))
                                                    : nullptr;
    void* ctl = (f32 && (need || chain)) ? c.take(chain_ctl_bytes(p.B, p.nsub, p.Mp)) : nullptr;
    IO* mu_in_p = (mu_in || need) ? static_cast<IO*>(c.take(p.B * mp * sz)) : nullptr;
    int* flags = refine ? static_cast<int*>(c.take(p.B * sizeof(int))) : nullptr;
    unsigned* dstat = refine ? static_cast<unsigned*>(c.take(p.B * 2 * sizeof(unsigned))) : nullptr;
    IO* D0 = (refine && hier) ? static_cast<IO*>(c.take(nsc * mp * sz)) : nullptr;
    IO* E0 = (refine && hier) ? static_cast<IO*>(c.take(nsc * mp * sz)) : nullptr;
    const int nchunk = grad_a_chunks(p);
    IO* part = ti ? static_cast<IO*>(c.take(p.B * (int64_t)nchunk * p.Mp * sz)) : nullptr;
    IO* ga_p = (ti && p.Mp != p.M) ? static_cast<IO*>(c.take(p.B * p.Mp * sz)) : nullptr;
    const IO* gs_p = static_cast<const IO*>(gs);
    const IO* A_p = static_cast<const IO*>(A);
    const IO* s_p = static_cast<const IO*>(s);
    const IO* zi_p = static_cast<const IO*>(zi);
    IO* ge_p = static_cast<IO*>(ge);
    IO* gA_p = static_cast<IO*>(gA);
    void *pgs = nullptr, *pA = nullptr, *ps = nullptr, *pz = nullptr, *pge = nullptr,
         *pgA = nullptr;
    if (packed) {
        pgs = c.take(p.B * p.Tp * sz);
        if (!frames) pA = c.take((ti ? p.B : p.B * p.Tp) * p.Mp * sz);
        ps = c.take(p.B * p.Tp * sz);
        if (zi) pz = c.take(p.B * p.Mp * sz);
        pge = c.take(p.B * p.Tp * sz);
        if (!ti && !frames) pgA = c.take(p.B * p.Tp * p.Mp * sz);
    }
    // (the sizing pass reserves the materialised rows whatever the precision)
    if (frames && (!native_fr || need)) pA = c.take(p.B * p.Tp * p.Mp * sz);
    if (need) {
        *need = c.used;
        return TVLP_OK;
    }
    if (ws_bytes < c.used) return TVLP_ERR_WORKSPACE;
    const ScanArgs g = scan_args(p);
    if (packed) {
        TVLP_CK(pack<IO>(gs, pgs, p.B, p.T, 1, p.Tp, 1, st));
        if (!frames) {
            if (ti)
                TVLP_CK(pack<IO>(A, pA, p.B, 1, p.M, 1, p.Mp, st));
            else
                TVLP_CK(pack<IO>(A, pA, p.B, p.T, p.M, p.Tp, p.Mp, st));
            A_p = static_cast<const IO*>(pA);
            gA_p = static_cast<IO*>(pgA);
        }
        TVLP_CK(pack<IO>(s, ps, p.B, p.T, 1, p.Tp, 1, st));
        if (zi) TVLP_CK(pack<IO>(zi, pz, p.B, 1, p.M, 1, p.Mp, st));
        gs_p = static_cast<const IO*>(pgs);
        s_p = static_cast<const IO*>(ps);
        zi_p = static_cast<const IO*>(pz);
        ge_p = static_cast<IO*>(pge);
    }
    if (frames && !native_fr) {
        TVLP_RUN("upsample", 1, st, (launch_upsample<IO>(p.Mp, *fr, static_cast<IO*>(pA), p.B,
                                                          p.Tp, st)));
        A_p = static_cast<const IO*>(pA);
    }
    const FrameSrc<IO>* frk = native_fr ? fr : nullptr;
    h.tape = carry ? const_cast<IO*>(carry) : phiz_own;
    if (!carry) {
        // transition matrices only (the zero-state row is unused here; s is a
        // valid stand-in for e of the same shape)
        TVLP_RUN("basis", 1, st,
                 (launch_basis<IO>(p.Mp, ti, prec, s_p, A_p, phiz_own, g, st, frk)));
        if (hier) TVLP_RUN("compose", h.lv.L - 1, st, (h.compose()));
    }
    bool chained = false;
    if constexpr (std::is_same<IO, float>::value) {
        if (chain) {
            const int* inherit = reinterpret_cast<const int*>(carry + tape_body(p));
            ChainBwdCall cc{ti, 1, {}, h.tape, inherit, nu, mu, kout, ctl,
                            prec == kPrecAuto ? 1 : 0, g};
            cc.grp[0] = ChainGroup{gs_p, frames ? nullptr : A_p, nullptr, ge_p, p.B};
            cc.fr = frk;
            TVLP_RUN("adjoint_zs", 2, st, (launch_bwd_chain(p.Mp, cc, st, 0)));
            TVLP_RUN("bwd_chain", 1, st, (launch_bwd_chain(p.Mp, cc, st, 1)));
            chained = true;
        }
    }
    if (!chained) {
    TVLP_RUN("adjoint_zs", 1, st,
             (launch_adjoint<IO>(p.Mp, ti, 0, gs_p, A_p, nullptr, nu, nullptr, nullptr, nullptr, g,
                                 st, frk)));
    if (dstat) TVLP_CK(cudaMemsetAsync(dstat, 0, p.B * 2 * sizeof(unsigned), st));
    if (mu_in) {  // [B][M] -> [B][mp4] (zero padded)
        TVLP_CK(cudaMemsetAsync(mu_in_p, 0, p.B * mp * sz, st));
        TVLP_CK(cudaMemcpy2DAsync(mu_in_p, mp * sz, mu_in, p.M * sz, p.M * sz, p.B,
                                  cudaMemcpyDeviceToDevice, st));
    }
    TVLP_RUN("carry_bwd", 1, st, (h.bwd(0, nu, mu, mu_in ? mu_in_p : nullptr)));
    TVLP_RUN("adjoint_apply", 1, st,
             (launch_adjoint<IO>(p.Mp, ti, 1, gs_p, A_p, mu, kout, ge_p, dstat, nullptr, g, st,
                                 frk)));
    if (refine && !hier && kFusedRefine && !grad_zi) {
        // (grad_zi re-writes the carry-outs the recurrence reads: separate kernels)
        RefineSrc<IO> rf;
        rf.tape = h.tape;
        rf.K = kout;
        rf.dstat = dstat;
        rf.inherit = carry ? reinterpret_cast<const int*>(carry + tape_body(p)) : nullptr;
        TVLP_RUN("adjoint_apply_refined", 1, st,
                 (launch_adjoint<IO>(p.Mp, ti, 1, gs_p, A_p, mu, nullptr, ge_p, nullptr, nullptr,
                                     g, st, frk, &rf)));
    } else if (refine) {
        const int* inherit = carry ? reinterpret_cast<const int*>(carry + tape_body(p)) : nullptr;
        if (!hier) {
            TVLP_RUN("refine_bwd", 1, st,
                     (launch_refine<IO>(p.Mp, false, h.tape, mu, kout, dstat, flags, inherit, g,
                                        st)));
        } else {
            TVLP_RUN("refine_bwd", 4, st, ([&]() -> cudaError_t {
                cudaError_t err = launch_refine_helpers<IO>(0, p.Mp, nullptr, nullptr, nullptr,
                                                            p.nsub, false, nullptr, flags, dstat,
                                                            inherit, kDefectTolBwd, p.B, st);
                if (err != cudaSuccess) return err;
                err = launch_refine_helpers<IO>(1, p.Mp, kout, mu, D0, p.nsub, false, flags,
                                                nullptr, nullptr, nullptr, 0.f, p.B, st);
                if (err != cudaSuccess) return err;
                Hier<IO> hr = h;
                hr.only = flags;
                err = hr.bwd(0, D0, E0);
                if (err != cudaSuccess) return err;
                return launch_refine_helpers<IO>(2, p.Mp, mu, E0, nullptr, p.nsub, false, flags,
                                                 nullptr, nullptr, nullptr, 0.f, p.B, st);
            }()));
        }
        TVLP_RUN("adjoint_apply_refined", 1, st,
                 (launch_adjoint<IO>(p.Mp, ti, 1, gs_p, A_p, mu, grad_zi ? kout : nullptr, ge_p,
                                     nullptr, flags, g, st, frk)));
    }
    }  // !chained
    if (grad_zi) {  // adjoint at the segment's left boundary: carry-out of sub-chunk 0
        TVLP_CK(cudaMemcpy2DAsync(grad_zi, p.M * sz, kout, p.nsub * mp * sz, p.M * sz, p.B,
                                  cudaMemcpyDeviceToDevice, st));
    }
    if (frames) {
        TVLP_RUN("grad_frames", 1, st,
                 (launch_grad_frames<IO>(*fr, ge_p, s_p, zi_p, zi_p == zi ? p.M : p.Mp,
                                         static_cast<IO*>(gA), p.B, p.Tp, st)));
    } else if (ti) {
        IO* ga_out = ga_p ? ga_p : static_cast<IO*>(gA);
        TVLP_RUN("grad_a", 2, st,
                 (launch_grad_a<IO>(p.Mp, ge_p, s_p, zi_p, part, ga_out, p.B, p.Tp, nchunk, st)));
        if (ga_p) TVLP_CK(unpack<IO>(ga_p, gA, p.B, 1, p.M, 1, p.Mp, st));
    } else {
        TVLP_RUN("grad_A", 1, st, (launch_grad_A<IO>(p.Mp, ge_p, s_p, zi_p, gA_p, p.B, p.Tp, st)));
    }
    if (packed) {
        TVLP_CK(unpack<IO>(pge, ge, p.B, p.T, 1, p.Tp, 1, st));
        if (!ti && !frames) TVLP_CK(unpack<IO>(pgA, gA, p.B, p.T, p.M, p.Tp, p.Mp, st));
    }
    return TVLP_OK;
}

// ---------------------------------------------------------------- frame-wise
bool fw_args(int64_t B, int64_t T, int64_t F, int M, int size, int hop, double cola, FwArgs& a) {
    if (B < 1 || T < 1 || M < 1 || M > kMaxOrder || size < 1 || hop < 1) return false;
    // (frame sizes whose staged span fits shared memory; fp64 bound is the tighter)
    if (!fw_supported(padded_order(M), size, hop, 8)) return false;
    if (F != (T - 1) / hop + 1) return false;  // params.py:223-227
    a.B = B;
    a.T = T;
    a.F = (int)F;
    a.size = size;
    a.hop = hop;
    a.n_lead = (size - 1) / hop;  // params.py:203-207
    a.nfr = (int)(F + a.n_lead);
    a.cola = cola;
    return true;
}

template <typename IO>
int fw_forward_impl(const void* e, const void* frames, const void* win, void* out, void* seg,
                    const FwArgs& a, int M, void* ws, size_t ws_bytes, cudaStream_t st,
                    size_t* need, void* aux = nullptr) {
    const int Mp = padded_order(M);
    Carver c(ws);
    void* fp = (Mp != M) ? c.take(a.B * (int64_t)a.F * Mp * sizeof(IO)) : nullptr;
    if (need) {
        *need = c.used;
        return TVLP_OK;
    }
    if (ws_bytes < c.used) return TVLP_ERR_WORKSPACE;
    const IO* fr = static_cast<const IO*>(frames);
    if (fp) {
        TVLP_CK(pack<IO>(frames, fp, a.B, a.F, M, a.F, Mp, st));
        fr = static_cast<const IO*>(fp);
    }
    TVLP_RUN("fw_forward", 2, st,
             (launch_fw_forward<IO>(Mp, static_cast<const IO*>(e), fr, static_cast<const IO*>(win),
                                    static_cast<IO*>(seg), static_cast<IO*>(out), a, st,
                                    static_cast<IO*>(aux))));
    return TVLP_OK;
}

template <typename IO>
int fw_backward_impl(const void* gout, const void* frames, const void* win, const void* seg,
                     void* ge, void* gf, const FwArgs& a, int M, void* ws, size_t ws_bytes,
                     cudaStream_t st, size_t* need, const void* aux = nullptr) {
    const int Mp = padded_order(M);
    Carver c(ws);
    void* fp = (Mp != M) ? c.take(a.B * (int64_t)a.F * Mp * sizeof(IO)) : nullptr;
    void* gfp = (Mp != M) ? c.take(a.B * (int64_t)a.F * Mp * sizeof(IO)) : nullptr;
    IO* gew = static_cast<IO*>(c.take(a.B * (int64_t)a.size * a.nfr * sizeof(IO)));
    IO* gap = static_cast<IO*>(c.take(a.B * (int64_t)a.nfr * Mp * sizeof(IO)));
    if (need) {
        *need = c.used;
        return TVLP_OK;
    }
    if (ws_bytes < c.used) return TVLP_ERR_WORKSPACE;
    const IO* fr = static_cast<const IO*>(frames);
    if (fp) {
        TVLP_CK(pack<IO>(frames, fp, a.B, a.F, M, a.F, Mp, st));
        fr = static_cast<const IO*>(fp);
    }
    IO* gf_out = gfp ? static_cast<IO*>(gfp) : static_cast<IO*>(gf);
    TVLP_RUN("fw_backward", 3, st,
             (launch_fw_backward<IO>(Mp, M, static_cast<const IO*>(gout), fr,
                                     static_cast<const IO*>(win), static_cast<const IO*>(seg), gew,
                                     gap, static_cast<IO*>(ge), gf_out, a, st,
                                     static_cast<const IO*>(aux))));
    if (gfp) TVLP_CK(unpack<IO>(gfp, gf, a.B, a.F, M, a.F, Mp, st));
    return TVLP_OK;
}

// ---------------------------------------------------------------- grouped
// The chained kernels take the groups' own buffers (per-group tensor maps):
// fp32, one carry level, a compiled order equal to M, T a multiple of the
// sub-chunk length and 16-byte aligned arrays.  Otherwise the groups are
// concatenated into workspace, filtered as one batch and split back.
template <typename IO>
bool grouped_direct(const Plan& p, int prec, bool aligned) {
    return std::is_same<IO, float>::value && make_levels(p).L == 1 &&
           (prec == kPrecAuto || prec == kPrecF32Chains) && chain_supported(p.Mp) &&
           p.Tp == p.T && p.Mp == p.M && aligned;
}

template <typename IO>
int grouped_forward_impl(int n, const tvlp_lp_fwd_group* gr, const Plan& p, void* carry_v,
                         int prec, void* ws, size_t ws_bytes, int32_t* nonfinite,
                         cudaStream_t st, size_t* need) {
    const size_t sz = sizeof(IO);
    bool al = true, any_zi = false;
    for (int i = 0; i < n && !need; ++i) {
        al = al && aligned16(gr[i].e) && aligned16(gr[i].A) && aligned16(gr[i].s) &&
             (!gr[i].zi || aligned16(gr[i].zi));
        any_zi = any_zi || gr[i].zi != nullptr;
    }
    const bool direct = !need && grouped_direct<IO>(p, prec, al);
    const int64_t nsc = p.B * p.nsub, mp = mp4(p);
    Carver c(ws);
    IO* carry = carry_v ? static_cast<IO*>(carry_v) : static_cast<IO*>(c.take(carry_elems(p) * sz));
    if (direct) {
        IO* xin = static_cast<IO*>(c.take(nsc * mp * sz));
        IO* xend = static_cast<IO*>(c.take(nsc * mp * sz));
        void* ctl = c.take(chain_ctl_bytes(p.B, p.nsub, p.Mp));
        if (ws_bytes < c.used) return TVLP_ERR_WORKSPACE;
        if constexpr (std::is_same<IO, float>::value) {
            const ScanArgs g = scan_args(p);
            ChainFwdCall cc{false, n, {}, p.Mp, carry,
                            reinterpret_cast<int*>(carry + tape_body(p)), xin, xend, nonfinite,
                            ctl, prec == kPrecAuto ? 1 : 0, g};
            for (int i = 0; i < n; ++i)
                cc.grp[i] = ChainGroup{static_cast<const float*>(gr[i].e),
                                       static_cast<const float*>(gr[i].A),
                                       static_cast<const float*>(gr[i].zi),
                                       static_cast<float*>(gr[i].s), gr[i].B};
            TVLP_RUN("basis", 1 + n, st, (launch_fwd_chain(p.Mp, cc, st, 0)));
            TVLP_RUN("fwd_chain", 1, st, (launch_fwd_chain(p.Mp, cc, st, 1)));
        }
        return TVLP_OK;
    }
    // concatenation fallback
    IO* ce = static_cast<IO*>(c.take(p.B * p.T * sz));
    IO* cA = static_cast<IO*>(c.take(p.B * p.T * p.M * sz));
    IO* cz = static_cast<IO*>(c.take(p.B * p.M * sz));
    IO* cs = static_cast<IO*>(c.take(p.B * p.T * sz));
    size_t inner = 0;
    const void* any16 = reinterpret_cast<const void*>(uintptr_t(256));  // sizing: aligned, non-null
    forward_impl<IO>(false, any16, any16, any16, (void*)any16, p, nullptr, prec, nullptr, 0, nullptr,
                     st, &inner);
    void* iws = c.take(inner);
    if (need) {
        *need = c.used;
        return TVLP_OK;
    }
    if (ws_bytes < c.used) return TVLP_ERR_WORKSPACE;
    int64_t off = 0;
    if (any_zi) TVLP_CK(cudaMemsetAsync(cz, 0, p.B * p.M * sz, st));
    for (int i = 0; i < n; ++i) {
        const int64_t B = gr[i].B;
        TVLP_CK(cudaMemcpyAsync(ce + off * p.T, gr[i].e, B * p.T * sz, cudaMemcpyDeviceToDevice, st));
        TVLP_CK(cudaMemcpyAsync(cA + off * p.T * p.M, gr[i].A, B * p.T * p.M * sz,
                                cudaMemcpyDeviceToDevice, st));
        if (gr[i].zi)
            TVLP_CK(cudaMemcpyAsync(cz + off * p.M, gr[i].zi, B * p.M * sz,
                                    cudaMemcpyDeviceToDevice, st));
        off += B;
    }
    const int rc = forward_impl<IO>(false, ce, cA, any_zi ? cz : nullptr, cs, p, carry, prec, iws,
                                    inner, nonfinite, st, nullptr);
    if (rc != TVLP_OK) return rc;
    off = 0;
    for (int i = 0; i < n; ++i) {
        TVLP_CK(cudaMemcpyAsync(gr[i].s, cs + off * p.T, gr[i].B * p.T * sz,
                                cudaMemcpyDeviceToDevice, st));
        off += gr[i].B;
    }
    return TVLP_OK;
}

template <typename IO>
int grouped_backward_impl(int n, const tvlp_lp_bwd_group* gr, const Plan& p, const void* carry_v,
                          int prec, void* ws, size_t ws_bytes, cudaStream_t st, size_t* need) {
    const size_t sz = sizeof(IO);
    bool al = true, any_zi = false;
    for (int i = 0; i < n && !need; ++i) {
        al = al && aligned16(gr[i].grad_s) && aligned16(gr[i].A) && aligned16(gr[i].s) &&
             aligned16(gr[i].grad_e) && aligned16(gr[i].grad_A) &&
             (!gr[i].zi || aligned16(gr[i].zi));
        any_zi = any_zi || gr[i].zi != nullptr;
    }
    const bool direct = !need && carry_v != nullptr && grouped_direct<IO>(p, prec, al);
    const int64_t nsc = p.B * p.nsub, mp = mp4(p);
    Carver c(ws);
    if (direct) {
        IO* nu = static_cast<IO*>(c.take(nsc * mp * sz));
        IO* mu = static_cast<IO*>(c.take(nsc * mp * sz));
        IO* kout = static_cast<IO*>(c.take(nsc * mp * sz));
        void* ctl = c.take(chain_ctl_bytes(p.B, p.nsub, p.Mp));
        if (ws_bytes < c.used) return TVLP_ERR_WORKSPACE;
        if constexpr (std::is_same<IO, float>::value) {
            const float* carry = static_cast<const float*>(carry_v);
            const ScanArgs g = scan_args(p);
            ChainBwdCall cc{false, n, {}, carry,
                            reinterpret_cast<const int*>(carry + tape_body(p)), nu, mu, kout, ctl,
                            prec == kPrecAuto ? 1 : 0, g};
            for (int i = 0; i < n; ++i)
                cc.grp[i] = ChainGroup{static_cast<const float*>(gr[i].grad_s),
                                       static_cast<const float*>(gr[i].A), nullptr,
                                       static_cast<float*>(gr[i].grad_e), gr[i].B};
            TVLP_RUN("adjoint_zs", 1 + n, st, (launch_bwd_chain(p.Mp, cc, st, 0)));
            TVLP_RUN("bwd_chain", 1, st, (launch_bwd_chain(p.Mp, cc, st, 1)));
            for (int i = 0; i < n; ++i)
                TVLP_RUN("grad_A", 1, st,
                         (launch_grad_A<IO>(p.Mp, static_cast<const IO*>(gr[i].grad_e),
                                            static_cast<const IO*>(gr[i].s),
                                            static_cast<const IO*>(gr[i].zi),
                                            static_cast<IO*>(gr[i].grad_A), gr[i].B, p.T, st)));
        }
        return TVLP_OK;
    }
    IO* cg = static_cast<IO*>(c.take(p.B * p.T * sz));
    IO* cA = static_cast<IO*>(c.take(p.B * p.T * p.M * sz));
    IO* cs = static_cast<IO*>(c.take(p.B * p.T * sz));
    IO* cz = static_cast<IO*>(c.take(p.B * p.M * sz));
    IO* cge = static_cast<IO*>(c.take(p.B * p.T * sz));
    IO* cgA = static_cast<IO*>(c.take(p.B * p.T * p.M * sz));
    size_t inner = 0;
    const void* any16 = reinterpret_cast<const void*>(uintptr_t(256));  // sizing: aligned, non-null
    backward_impl<IO>(false, any16, any16, any16, any16, (void*)any16, (void*)any16, p, nullptr,
                      prec, nullptr, 0, st, &inner);
    void* iws = c.take(inner);
    if (need) {
        *need = c.used;
        return TVLP_OK;
    }
    if (ws_bytes < c.used) return TVLP_ERR_WORKSPACE;
    if (any_zi) TVLP_CK(cudaMemsetAsync(cz, 0, p.B * p.M * sz, st));
    int64_t off = 0;
    for (int i = 0; i < n; ++i) {
        const int64_t B = gr[i].B;
        TVLP_CK(cudaMemcpyAsync(cg + off * p.T, gr[i].grad_s, B * p.T * sz,
                                cudaMemcpyDeviceToDevice, st));
        TVLP_CK(cudaMemcpyAsync(cA + off * p.T * p.M, gr[i].A, B * p.T * p.M * sz,
                                cudaMemcpyDeviceToDevice, st));
        TVLP_CK(cudaMemcpyAsync(cs + off * p.T, gr[i].s, B * p.T * sz, cudaMemcpyDeviceToDevice,
                                st));
        if (gr[i].zi)
            TVLP_CK(cudaMemcpyAsync(cz + off * p.M, gr[i].zi, B * p.M * sz,
                                    cudaMemcpyDeviceToDevice, st));
        off += B;
    }
    const int rc = backward_impl<IO>(false, cg, cA, cs, any_zi ? cz : nullptr, cge, cgA, p,
                                     carry_v, prec, iws, inner, st, nullptr);
    if (rc != TVLP_OK) return rc;
    off = 0;
    for (int i = 0; i < n; ++i) {
        const int64_t B = gr[i].B;
        TVLP_CK(cudaMemcpyAsync(gr[i].grad_e, cge + off * p.T, B * p.T * sz,
                                cudaMemcpyDeviceToDevice, st));
        TVLP_CK(cudaMemcpyAsync(gr[i].grad_A, cgA + off * p.T * p.M, B * p.T * p.M * sz,
                                cudaMemcpyDeviceToDevice, st));
        off += B;
    }
    return TVLP_OK;
}

}  // namespace
}  // namespace tvlp

using namespace tvlp;

bool frame_src_ok(int64_t T, int64_t F, int32_t hop) {
    return hop >= 1 && T >= 1 && F == (T - 1) / hop + 1;  // params.py:102-117 (T = T1 - 1)
}

template <typename IO>
FrameSrc<IO> frame_src(const void* frames, int64_t T, int32_t M, int64_t F, int32_t hop) {
    FrameSrc<IO> fs;
    fs.frames = static_cast<const IO*>(frames);
    fs.nF = F;
    fs.Tv = T;
    fs.hop = hop;
    fs.Mf = M;
    return fs;
}

extern "C" {

int tvlp_abi_version(void) { return TVLP_ABI_VERSION; }

const char* tvlp_status_string(int status) {
    switch (status) {
        case TVLP_OK: return "ok";
        case TVLP_ERR_ARG: return "invalid argument";
        case TVLP_ERR_ORDER: return "unsupported filter order";
        case TVLP_ERR_WORKSPACE: return "workspace too small";
        case TVLP_ERR_CUDA: return cudaGetErrorString((cudaError_t)g_last_cuda);
        default: return "unknown status";
    }
}

int tvlp_last_cuda_error(void) { return g_last_cuda; }

int32_t tvlp_max_order(void) { return kMaxOrder; }

int64_t tvlp_launch_count(void) { return g_launches.load(); }

// ---------------------------------------------------------------- decoder pieces
static int osc_geo(const double* f0, const float* pos, const float* tab, int32_t K, int32_t L,
                   const float* taps, int32_t nt, int64_t B, int64_t n_out, int64_t F,
                   int32_t hop, int32_t os, double fs, OscGeo* g) {
    if (!f0 || !pos || !tab || !taps || K < 1 || L < 2 || nt < 1 || (nt % 2) == 0 || B < 0 ||
        n_out < 1 || hop < 1 || os != 4 || !(fs > 0.0))
        return TVLP_ERR_ARG;
    const int64_t n_os = n_out * os, hop_os = (int64_t)hop * os;
    if (F != (n_os - 1) / hop_os + 1 || hop_os > (1 << 20) || nt > 4096) return TVLP_ERR_ARG;
    *g = OscGeo{B, n_out, F, n_os, hop, (int)hop_os, K, L, nt, (nt - 1) / 2, 1.0 / (fs * os),
                1.0 / (double)hop_os, 1.0f / (float)hop_os};
    return TVLP_OK;
}

int tvlp_wavetable_osc(const double* f0_frames, const float* pos_frames, const float* tables,
                       int32_t K, int32_t L, const float* taps, int32_t ntaps, float* sig,
                       int64_t B, int64_t n_out, int64_t F, int32_t hop, int32_t oversample,
                       double fs, void* stream) {
    OscGeo g;
    int rc = osc_geo(f0_frames, pos_frames, tables, K, L, taps, ntaps, B, n_out, F, hop,
                     oversample, fs, &g);
    if (rc != TVLP_OK) return rc;
    if (!sig) return TVLP_ERR_ARG;
    if (B == 0) return TVLP_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    TVLP_CK(tracked("osc_fwd", 1, st, [&] {
        return launch_osc_fwd(f0_frames, pos_frames, tables, taps, sig, g, oversample, st);
    }));
    return TVLP_OK;
}

int tvlp_wavetable_osc_vjp(const double* f0_frames, const float* pos_frames, const float* tables,
                           int32_t K, int32_t L, const float* taps, int32_t ntaps,
                           const float* grad_sig, float* grad_pos, float* workspace, int64_t B,
                           int64_t n_out, int64_t F, int32_t hop, int32_t oversample, double fs,
                           void* stream) {
    OscGeo g;
    int rc = osc_geo(f0_frames, pos_frames, tables, K, L, taps, ntaps, B, n_out, F, hop,
                     oversample, fs, &g);
    if (rc != TVLP_OK) return rc;
    if (!grad_sig || !grad_pos || !workspace) return TVLP_ERR_ARG;
    if (B == 0) return TVLP_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    TVLP_CK(tracked("osc_vjp", 2, st, [&] {
        return launch_osc_vjp(f0_frames, pos_frames, tables, taps, grad_sig, workspace, grad_pos,
                              g, oversample, st);
    }));
    return TVLP_OK;
}

int tvlp_global_fir(const float* x, const float* taps, float* y, int64_t B, int64_t n, int32_t m,
                    void* stream) {
    if (!x || !taps || !y || B < 0 || n < 0 || m < 1 || m > 1024) return TVLP_ERR_ARG;
    if (B == 0 || n == 0) return TVLP_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    TVLP_CK(tracked("global_fir", 1, st, [&] { return launch_fir(x, taps, y, B, n, m, false, 0, st); }));
    return TVLP_OK;
}

static bool noise_geo_ok(int64_t B, int64_t n, int64_t nfr, int32_t size, int32_t ld,
                         int32_t delay, int32_t hop) {
    // (grid y covers one item's samples / one frame row in blocks of 256)
    return B >= 0 && B <= 65535 && n >= 1 && n <= (1 << 24) && nfr >= 1 && nfr < (1 << 30) &&
           size >= 1 && hop >= 1 && delay >= 0 && ld >= size + delay && ld <= (1 << 24);
}

int tvlp_noise_frames(const float* noise, const float* window, float* frames, int64_t B,
                      int64_t n, int64_t nframes, int32_t size, int32_t nfft, int64_t start0,
                      int32_t hop, void* stream) {
    if (!noise || !window || !frames || !noise_geo_ok(B, n, nframes, size, nfft, 0, hop))
        return TVLP_ERR_ARG;
    if (B == 0) return TVLP_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    TVLP_CK(tracked("noise_frames", 1, st, [&] {
        return launch_noise_frames(noise, window, frames, B, n, nframes, size, nfft, start0, hop,
                                   st);
    }));
    return TVLP_OK;
}

int tvlp_frame_ola(const float* y, float* out, int64_t B, int64_t n, int64_t nframes, int32_t size,
                   int32_t ld, int32_t delay, int64_t start0, int32_t hop, float scale,
                   int32_t adjoint, void* stream) {
    if (!y || !out || !noise_geo_ok(B, n, nframes, size, ld, delay, hop)) return TVLP_ERR_ARG;
    if (B == 0) return TVLP_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    TVLP_CK(tracked(adjoint ? "frame_ola_vjp" : "frame_ola", 1, st, [&] {
        return launch_frame_ola(y, out, B, n, nframes, size, ld, delay, start0, hop, scale,
                                adjoint != 0, st);
    }));
    return TVLP_OK;
}

int tvlp_spectra_mul(const float* S, const float* H, const int32_t* rows, float* P, int64_t B,
                     int64_t nframes, int64_t F, int32_t K, void* stream) {
    if (!S || !H || !rows || !P || B < 0 || B > 65535 || nframes < 1 || F < 1 || K < 1)
        return TVLP_ERR_ARG;
    if (B == 0) return TVLP_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    TVLP_CK(tracked("spectra_mul", 1, st, [&] {
        return launch_spec_mul(S, H, rows, nullptr, P, B, nframes, F, K, false, st);
    }));
    return TVLP_OK;
}

int tvlp_spectra_mul_vjp(const float* grad_P, const float* S, const int32_t* first, float* grad_H,
                         int64_t B, int64_t nframes, int64_t F, int32_t K, void* stream) {
    if (!grad_P || !S || !first || !grad_H || B < 0 || B > 65535 || nframes < 1 || F < 1 || K < 1)
        return TVLP_ERR_ARG;
    if (B == 0) return TVLP_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    TVLP_CK(tracked("spectra_mul_vjp", 1, st, [&] {
        return launch_spec_mul(grad_P, S, nullptr, first, grad_H, B, nframes, F, K, true, st);
    }));
    return TVLP_OK;
}

static bool source_geo_ok(int64_t B, int64_t T1, int64_t F, int32_t hop, int64_t Tp) {
    return B >= 0 && B <= 65535 && T1 >= 1 && hop >= 1 && F == (T1 - 1) / hop + 1 &&
           Tp >= T1 && Tp <= F * hop;
}

int tvlp_source_pair(const float* sig, const float* noise, const float* voiced_gain,
                     const float* noise_gain, const float* h_gain, float* out, int64_t B,
                     int64_t T1, int64_t F, int32_t hop, int64_t Tp, void* stream) {
    if (!sig || !noise || !voiced_gain || !noise_gain || !h_gain || !out ||
        !source_geo_ok(B, T1, F, hop, Tp))
        return TVLP_ERR_ARG;
    if (B == 0) return TVLP_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    TVLP_CK(tracked("source_pair", 1, st, [&] {
        return launch_source_pair(sig, noise, voiced_gain, noise_gain, h_gain, out, B, T1, F, hop,
                                  Tp, st);
    }));
    return TVLP_OK;
}

int tvlp_source_pair_vjp(const float* grad_out, const float* sig, const float* noise,
                         const float* voiced_gain, const float* noise_gain, const float* h_gain,
                         float* grad_sig, float* grad_noise, float* grad_voiced_gain,
                         float* grad_noise_gain, float* grad_h_gain, float* workspace, int64_t B,
                         int64_t T1, int64_t F, int32_t hop, int64_t Tp, void* stream) {
    if (!grad_out || !sig || !noise || !voiced_gain || !noise_gain || !h_gain || !grad_sig ||
        !grad_noise || !grad_voiced_gain || !grad_noise_gain || !grad_h_gain || !workspace ||
        !source_geo_ok(B, T1, F, hop, Tp))
        return TVLP_ERR_ARG;
    if (B == 0) return TVLP_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    TVLP_CK(tracked("source_pair_vjp", 2, st, [&] {
        return launch_source_pair_vjp(grad_out, sig, noise, voiced_gain, noise_gain, h_gain,
                                      grad_sig, grad_noise, grad_voiced_gain, grad_noise_gain,
                                      grad_h_gain, workspace, B, T1, F, hop, Tp, st);
    }));
    return TVLP_OK;
}

int64_t tvlp_stft_nframes(int64_t n, int32_t N, int32_t hop) {
    if (n < 1 || n > (1 << 24) || N < 2 || hop < 1 || n < N || N / 2 >= n) return 0;
    return 1 + (n + 2 * (N / 2) - N) / hop;
}

int tvlp_stft_frames(const float* x, const float* window, float* frames, int64_t B, int64_t n,
                     int32_t N, int32_t hop, void* stream) {
    if (!x || !window || !frames || B < 0 || B > 65535 || tvlp_stft_nframes(n, N, hop) == 0)
        return TVLP_ERR_ARG;
    if (B == 0) return TVLP_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    TVLP_CK(tracked("stft_frames", 1, st,
                    [&] { return launch_stft_frames(x, window, frames, B, n, N, hop, st); }));
    return TVLP_OK;
}

int tvlp_stft_frames_vjp(const float* grad_frames, const float* window, float* grad_x, int64_t B,
                         int64_t n, int32_t N, int32_t hop, float scale, const float* dc,
                         int64_t dc_stride, float dc_scale, void* stream) {
    if (!grad_frames || !window || !grad_x || B < 0 || tvlp_stft_nframes(n, N, hop) == 0 ||
        (dc && dc_stride < 1))
        return TVLP_ERR_ARG;
    if (B == 0) return TVLP_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    TVLP_CK(tracked("stft_frames_vjp", 1, st, [&] {
        return launch_stft_frames_vjp(grad_frames, window, grad_x, B, n, N, hop, scale, dc,
                                      dc_stride, dc_scale, st);
    }));
    return TVLP_OK;
}

size_t tvlp_mss_terms_workspace(int64_t B, int64_t n) {
    if (B < 0 || n < 1) return 0;
    return mss_part_floats(B, n) * sizeof(float);
}

int tvlp_mss_terms(const float* X, const float* Y, int64_t B, int64_t n, float eps, float* term,
                   float* aux, void* workspace, size_t workspace_bytes, void* stream) {
    if (!X || !Y || !term || !aux || B < 0 || n < 1 || n > (1 << 24) || !(eps >= 0.f))
        return TVLP_ERR_ARG;
    if (B == 0) return TVLP_OK;
    if (!workspace || workspace_bytes < tvlp_mss_terms_workspace(B, n)) return TVLP_ERR_WORKSPACE;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    TVLP_CK(tracked("mss_terms", 2, st, [&] {
        return launch_mss_terms(X, Y, B, n, eps, term, aux, static_cast<float*>(workspace), st);
    }));
    return TVLP_OK;
}

int tvlp_mss_terms_vjp(const float* X, const float* Y, const float* aux, const float* grad_term,
                       float* grad_X, int64_t B, int64_t n, float eps, void* stream) {
    if (!X || !Y || !aux || !grad_term || !grad_X || B < 0 || n < 1 || n > (1 << 24))
        return TVLP_ERR_ARG;
    if (B == 0) return TVLP_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    TVLP_CK(tracked("mss_terms_vjp", 1, st, [&] {
        return launch_mss_terms_vjp(X, Y, aux, grad_term, B, n, eps, grad_X, st);
    }));
    return TVLP_OK;
}

size_t tvlp_global_fir_workspace(int64_t B, int64_t n, int32_t m) {
    if (B < 0 || n < 0 || m < 1) return 0;
    return fir_taps_part_elems(B, n, m) * sizeof(float);
}

int tvlp_global_fir_vjp(const float* grad_y, const float* x, const float* taps, float* grad_x,
                        float* grad_taps, void* workspace, size_t workspace_bytes, int64_t B,
                        int64_t n, int32_t m, void* stream) {
    if (!grad_y || !x || !taps || B < 0 || n < 0 || m < 1 || m > 1024) return TVLP_ERR_ARG;
    if (B == 0) return TVLP_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (n == 0) {
        if (grad_taps) TVLP_CK(cudaMemsetAsync(grad_taps, 0, B * m * sizeof(float), st));
        return TVLP_OK;
    }
    if (grad_x)
        TVLP_CK(tracked("global_fir_vjp_x", 1, st,
                        [&] { return launch_fir(grad_y, taps, grad_x, B, n, m, true, 0, st); }));
    if (grad_taps) {
        if (!workspace || workspace_bytes < tvlp_global_fir_workspace(B, n, m))
            return TVLP_ERR_WORKSPACE;
        TVLP_CK(tracked("global_fir_vjp_taps", 2, st, [&] {
            return launch_fir_taps(grad_y, x, static_cast<float*>(workspace), grad_taps, B, n, m,
                                   0, st);
        }));
    }
    return TVLP_OK;
}

int64_t tvlp_refined_sequences(void) {
    return (int64_t)(refined_sequences() + chain_refined_sequences());
}

void tvlp_profile_enable(int32_t on) { g_prof_on.store(on ? 1 : 0); }

void tvlp_chain_trace(void* buf, size_t bytes) { chain_set_trace(buf, bytes); }

int32_t tvlp_profile_dump(char* buf, int32_t buflen) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    std::vector<std::string> names;
    std::vector<double> ms;
    std::vector<long> cnt;
    for (auto& r : g_prof) {
        cudaEventSynchronize(r.b);
        float t = 0.f;
        cudaEventElapsedTime(&t, r.a, r.b);
        size_t k = 0;
        while (k < names.size() && names[k] != r.name) ++k;
        if (k == names.size()) {
            names.emplace_back(r.name);
            ms.push_back(0.0);
            cnt.push_back(0);
        }
        ms[k] += t;
        cnt[k] += 1;
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    g_prof.clear();
    std::string out;
    char line[160];
    for (size_t k = 0; k < names.size(); ++k) {
        std::snprintf(line, sizeof(line), "%s %ld %.6f\n", names[k].c_str(), cnt[k], ms[k]);
        out += line;
    }
    if (buf && buflen > 0) {
        const int n = (int)std::min<size_t>(out.size(), (size_t)buflen - 1);
        std::memcpy(buf, out.data(), n);
        buf[n] = 0;
        return n;
    }
    return (int32_t)out.size();
}

int64_t tvlp_carry_elems(int64_t B, int64_t T, int32_t M) {
    Plan p;
    if (!make_plan(B, T, M, p)) return -1;
    return carry_elems(p);
}

int64_t tvlp_carry_elems_frames(int64_t B, int64_t T, int32_t M) {
    Plan p;
    if (!make_plan(B, T, M, p, true)) return -1;
    return carry_elems(p);
}

int64_t tvlp_subchunk_len(int64_t B, int64_t T, int32_t M) {
    Plan p;
    if (!make_plan(B, T, M, p)) return -1;
    return p.Ls;
}

int64_t tvlp_framewise_nframes(int64_t T, int64_t F, int32_t frame_size, int32_t hop) {
    FwArgs a;
    if (!fw_args(1, T, F, 1, frame_size, hop, 1.0, a)) return -1;
    return a.nfr;
}

static int check_common(int32_t dtype, int32_t M) {
    if (dtype != TVLP_F32 && dtype != TVLP_F64) return TVLP_ERR_ARG;
    if (M < 1 || M > kMaxOrder) return TVLP_ERR_ORDER;
    return TVLP_OK;
}

size_t tvlp_workspace_bytes(int32_t op, int32_t dtype, int64_t B, int64_t T, int32_t M,
                            int64_t F, int32_t frame_size, int32_t hop) {
    if (check_common(dtype, M) != TVLP_OK) return 0;
    size_t need = 0;
    const bool f64 = dtype == TVLP_F64;
    // sizing pass: fake non-null, unaligned pointers force the packed layout
    const void* any = reinterpret_cast<const void*>(uintptr_t(1));
    if (op <= TVLP_OP_BWD_TI) {
        Plan p;
        if (!make_plan(B, T, M, p)) return 0;
        const bool ti = op == TVLP_OP_FWD_TI || op == TVLP_OP_BWD_TI;
        if (op == TVLP_OP_FWD_TV || op == TVLP_OP_FWD_TI) {
            if (f64)
                forward_impl<double>(ti, any, any, any, (void*)any, p, nullptr, kPrecAuto, nullptr,
                                     0, nullptr, 0, &need);
            else
                forward_impl<float>(ti, any, any, any, (void*)any, p, nullptr, kPrecAuto, nullptr,
                                    0, nullptr, 0, &need);
        } else {
            if (f64)
                backward_impl<double>(ti, any, any, any, any, (void*)any, (void*)any, p, nullptr,
                                      kPrecAuto, nullptr, 0, 0, &need);
            else
                backward_impl<float>(ti, any, any, any, any, (void*)any, (void*)any, p, nullptr,
                                     kPrecAuto, nullptr, 0, 0, &need);
        }
        return need;
    }
    if (op == TVLP_OP_BWD_TV_EX || op == TVLP_OP_SEGMENT_TRANSITION) {
        Plan p;
        if (!make_plan(B, T, M, p)) return 0;
        if (op == TVLP_OP_SEGMENT_TRANSITION) {
            if (f64)
                segment_transition_impl<double>(any, p, (void*)any, nullptr, 0, 0, &need);
            else
                segment_transition_impl<float>(any, p, (void*)any, nullptr, 0, 0, &need);
        } else if (f64) {
            backward_impl<double>(false, any, any, any, any, (void*)any, (void*)any, p, nullptr,
                                  kPrecAuto, nullptr, 0, 0, &need, nullptr, any, (void*)any);
        } else {
            backward_impl<float>(false, any, any, any, any, (void*)any, (void*)any, p, nullptr,
                                 kPrecAuto, nullptr, 0, 0, &need, nullptr, any, (void*)any);
        }
        return need;
    }
    if (op == TVLP_OP_FWD_TV_FRAMES || op == TVLP_OP_BWD_TV_FRAMES) {
        Plan p;
        if (!make_plan(B, T, M, p, true) || !frame_src_ok(T, F, hop)) return 0;
        if (op == TVLP_OP_FWD_TV_FRAMES) {
            if (f64) {
                const FrameSrc<double> fs = frame_src<double>(any, T, M, F, hop);
                forward_impl<double>(false, any, any, any, (void*)any, p, nullptr, kPrecAuto,
                                     nullptr, 0, nullptr, 0, &need, &fs);
            } else {
                const FrameSrc<float> fs = frame_src<float>(any, T, M, F, hop);
                forward_impl<float>(false, any, any, any, (void*)any, p, nullptr, kPrecAuto,
                                    nullptr, 0, nullptr, 0, &need, &fs);
            }
        } else {
            if (f64) {
                const FrameSrc<double> fs = frame_src<double>(any, T, M, F, hop);
                backward_impl<double>(false, any, any, any, any, (void*)any, (void*)any, p,
                                      nullptr, kPrecAuto, nullptr, 0, 0, &need, &fs);
            } else {
                const FrameSrc<float> fs = frame_src<float>(any, T, M, F, hop);
                backward_impl<float>(false, any, any, any, any, (void*)any, (void*)any, p,
                                     nullptr, kPrecAuto, nullptr, 0, 0, &need, &fs);
            }
        }
        return need;
    }
    FwArgs a;
    if (!fw_args(B, T, F, M, frame_size, hop, 1.0, a)) return 0;
    if (op == TVLP_OP_FW_FWD) {
        if (f64)
            fw_forward_impl<double>(any, any, any, (void*)any, (void*)any, a, M, nullptr, 0, 0,
                                    &need);
        else
            fw_forward_impl<float>(any, any, any, (void*)any, (void*)any, a, M, nullptr, 0, 0,
                                   &need);
    } else if (op == TVLP_OP_FW_BWD) {
        if (f64)
            fw_backward_impl<double>(any, any, any, any, (void*)any, (void*)any, a, M, nullptr, 0,
                                     0, &need);
        else
            fw_backward_impl<float>(any, any, any, any, (void*)any, (void*)any, a, M, nullptr, 0,
                                    0, &need);
    }
    return need;
}

static int fwd_entry(bool ti, int32_t dtype, const void* e, const void* A, const void* zi,
                     void* s, int64_t B, int64_t T, int32_t M, void* carry, int32_t prec,
                     void* ws, size_t ws_bytes, int32_t* nonfinite, void* stream) {
    int rc = check_common(dtype, M);
    if (rc != TVLP_OK) return rc;
    if (!e || !A || !s) return TVLP_ERR_ARG;
    Plan p;
    if (!make_plan(B, T, M, p)) return TVLP_ERR_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (dtype == TVLP_F64)
        return forward_impl<double>(ti, e, A, zi, s, p, carry,
                                    TVLP_CARRY_F64 | (prec & TVLP_CARRY_REUSE), ws, ws_bytes,
                                    nonfinite, st, nullptr);
    return forward_impl<float>(ti, e, A, zi, s, p, carry, prec, ws, ws_bytes, nonfinite, st,
                               nullptr);
}

static int bwd_entry(bool ti, int32_t dtype, const void* gs, const void* A, const void* s,
                     const void* zi, void* ge, void* gA, int64_t B, int64_t T, int32_t M,
                     const void* carry, int32_t prec, void* ws, size_t ws_bytes, void* stream) {
    int rc = check_common(dtype, M);
    if (rc != TVLP_OK) return rc;
    if (!gs || !A || !s || !ge || !gA) return TVLP_ERR_ARG;
    Plan p;
    if (!make_plan(B, T, M, p)) return TVLP_ERR_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (dtype == TVLP_F64)
        return backward_impl<double>(ti, gs, A, s, zi, ge, gA, p, carry, TVLP_CARRY_F64, ws,
                                     ws_bytes, st, nullptr);
    return backward_impl<float>(ti, gs, A, s, zi, ge, gA, p, carry, prec, ws, ws_bytes, st,
                                nullptr);
}

int tvlp_lp_forward_tv(int32_t dtype, const void* e, const void* A, const void* zi, void* s,
                       int64_t B, int64_t T, int32_t M, void* carry, int32_t carry_prec,
                       void* workspace, size_t workspace_bytes, int32_t* nonfinite, void* stream) {
    return fwd_entry(false, dtype, e, A, zi, s, B, T, M, carry, carry_prec, workspace,
                     workspace_bytes, nonfinite, stream);
}

int tvlp_lp_backward_tv(int32_t dtype, const void* grad_s, const void* A, const void* s,
                        const void* zi, void* grad_e, void* grad_A, int64_t B, int64_t T,
                        int32_t M, const void* carry, int32_t carry_prec, void* workspace,
                        size_t workspace_bytes, void* stream) {
    return bwd_entry(false, dtype, grad_s, A, s, zi, grad_e, grad_A, B, T, M, carry, carry_prec,
                     workspace, workspace_bytes, stream);
}

int tvlp_lp_forward_tv_frames(int32_t dtype, const void* e, const void* frames, const void* zi,
                              void* s, int64_t B, int64_t T, int32_t M, int64_t F, int32_t hop,
                              void* carry, int32_t carry_prec, void* workspace,
                              size_t workspace_bytes, int32_t* nonfinite, void* stream) {
    int rc = check_common(dtype, M);
    if (rc != TVLP_OK) return rc;
    if (!e || !frames || !s || !frame_src_ok(T, F, hop)) return TVLP_ERR_ARG;
    Plan p;
    if (!make_plan(B, T, M, p, true)) return TVLP_ERR_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (dtype == TVLP_F64) {
        const FrameSrc<double> fs = frame_src<double>(frames, T, M, F, hop);
        return forward_impl<double>(false, e, frames, zi, s, p, carry, TVLP_CARRY_F64, workspace,
                                    workspace_bytes, nonfinite, st, nullptr, &fs);
    }
    const FrameSrc<float> fs = frame_src<float>(frames, T, M, F, hop);
    return forward_impl<float>(false, e, frames, zi, s, p, carry, carry_prec, workspace,
                               workspace_bytes, nonfinite, st, nullptr, &fs);
}

int tvlp_lp_backward_tv_frames(int32_t dtype, const void* grad_s, const void* frames,
                               const void* s, const void* zi, void* grad_e, void* grad_frames,
                               int64_t B, int64_t T, int32_t M, int64_t F, int32_t hop,
                               const void* carry, int32_t carry_prec, void* workspace,
                               size_t workspace_bytes, void* stream) {
    int rc = check_common(dtype, M);
    if (rc != TVLP_OK) return rc;
    if (!grad_s || !frames || !s || !grad_e || !grad_frames || !frame_src_ok(T, F, hop))
        return TVLP_ERR_ARG;
    Plan p;
    if (!make_plan(B, T, M, p, true)) return TVLP_ERR_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (dtype == TVLP_F64) {
        const FrameSrc<double> fs = frame_src<double>(frames, T, M, F, hop);
        return backward_impl<double>(false, grad_s, frames, s, zi, grad_e, grad_frames, p, carry,
                                     TVLP_CARRY_F64, workspace, workspace_bytes, st, nullptr,
                                     &fs);
    }
    const FrameSrc<float> fs = frame_src<float>(frames, T, M, F, hop);
    return backward_impl<float>(false, grad_s, frames, s, zi, grad_e, grad_frames, p, carry,
                                carry_prec, workspace, workspace_bytes, st, nullptr, &fs);
}

int tvlp_reflection_to_lpc(int32_t dtype, const void* k, void* a, int64_t rows, int32_t M,
                           int32_t* bad, void* stream) {
    int rc = check_common(dtype, M);
    if (rc != TVLP_OK) return rc;
    if (!k || !a || rows < 0) return TVLP_ERR_ARG;
    if (rows == 0) return TVLP_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    g_launches += 1;
    cudaError_t err = dtype == TVLP_F64
                          ? launch_step_up<double>(static_cast<const double*>(k),
                                                   static_cast<double*>(a), rows, M, bad, st)
                          : launch_step_up<float>(static_cast<const float*>(k),
                                                  static_cast<float*>(a), rows, M, bad, st);
    return err == cudaSuccess ? TVLP_OK : TVLP_ERR_CUDA;
}

int tvlp_reflection_to_lpc_vjp(int32_t dtype, const void* grad_a, const void* k, void* grad_k,
                               int64_t rows, int32_t M, void* stream) {
    int rc = check_common(dtype, M);
    if (rc != TVLP_OK) return rc;
    if (!grad_a || !k || !grad_k || rows < 0) return TVLP_ERR_ARG;
    if (rows == 0) return TVLP_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    g_launches += 1;
    cudaError_t err =
        dtype == TVLP_F64
            ? launch_step_up_vjp<double>(static_cast<const double*>(grad_a),
                                         static_cast<const double*>(k),
                                         static_cast<double*>(grad_k), rows, M, st)
            : launch_step_up_vjp<float>(static_cast<const float*>(grad_a),
                                        static_cast<const float*>(k),
                                        static_cast<float*>(grad_k), rows, M, st);
    return err == cudaSuccess ? TVLP_OK : TVLP_ERR_CUDA;
}

int tvlp_lp_backward_tv_ex(int32_t dtype, const void* grad_s, const void* A, const void* s,
                           const void* zi, void* grad_e, void* grad_A, int64_t B, int64_t T,
                           int32_t M, const void* carry, int32_t carry_prec, const void* mu_in,
                           void* grad_zi, void* workspace, size_t workspace_bytes, void* stream) {
    int rc = check_common(dtype, M);
    if (rc != TVLP_OK) return rc;
    if (!grad_s || !A || !s || !grad_e || !grad_A) return TVLP_ERR_ARG;
    Plan p;
    if (!make_plan(B, T, M, p)) return TVLP_ERR_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (dtype == TVLP_F64)
        return backward_impl<double>(false, grad_s, A, s, zi, grad_e, grad_A, p, carry,
                                     TVLP_CARRY_F64, workspace, workspace_bytes, st, nullptr,
                                     nullptr, mu_in, grad_zi);
    return backward_impl<float>(false, grad_s, A, s, zi, grad_e, grad_A, p, carry, carry_prec,
                                workspace, workspace_bytes, st, nullptr, nullptr, mu_in, grad_zi);
}

int tvlp_segment_transition(int32_t dtype, const void* carry, int64_t B, int64_t T, int32_t M,
                            void* Phi, void* workspace, size_t workspace_bytes, void* stream) {
    int rc = check_common(dtype, M);
    if (rc != TVLP_OK) return rc;
    if (!carry || !Phi) return TVLP_ERR_ARG;
    Plan p;
    if (!make_plan(B, T, M, p)) return TVLP_ERR_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (dtype == TVLP_F64)
        return segment_transition_impl<double>(carry, p, Phi, workspace, workspace_bytes, st,
                                               nullptr);
    return segment_transition_impl<float>(carry, p, Phi, workspace, workspace_bytes, st, nullptr);
}

static int grouped_plan(int32_t dtype, int32_t n, const int64_t* Bs, int64_t T, int32_t M,
                        Plan& p) {
    int rc = check_common(dtype, M);
    if (rc != TVLP_OK) return rc;
    if (n < 1 || n > TVLP_MAX_GROUPS || n > kMaxGroups || T < 1) return TVLP_ERR_ARG;
    int64_t Bt = 0;
    for (int i = 0; i < n; ++i) {
        if (Bs[i] < 1) return TVLP_ERR_ARG;
        Bt += Bs[i];
    }
    return make_plan(Bt, T, M, p) ? TVLP_OK : TVLP_ERR_ARG;
}

int tvlp_lp_forward_tv_grouped(int32_t dtype, int32_t n, const tvlp_lp_fwd_group* groups,
                               int64_t T, int32_t M, void* carry, int32_t carry_prec,
                               void* workspace, size_t workspace_bytes, int32_t* nonfinite,
                               void* stream) {
    if (!groups || n < 1 || n > TVLP_MAX_GROUPS) return TVLP_ERR_ARG;
    int64_t Bs[TVLP_MAX_GROUPS];
    for (int i = 0; i < n; ++i) {
        if (!groups[i].e || !groups[i].A || !groups[i].s) return TVLP_ERR_ARG;
        Bs[i] = groups[i].B;
    }
    Plan p;
    int rc = grouped_plan(dtype, n, Bs, T, M, p);
    if (rc != TVLP_OK) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (dtype == TVLP_F64)
        return grouped_forward_impl<double>(n, groups, p, carry, TVLP_CARRY_F64, workspace,
                                            workspace_bytes, nonfinite, st, nullptr);
    return grouped_forward_impl<float>(n, groups, p, carry, carry_prec, workspace,
                                       workspace_bytes, nonfinite, st, nullptr);
}

int tvlp_lp_backward_tv_grouped(int32_t dtype, int32_t n, const tvlp_lp_bwd_group* groups,
                                int64_t T, int32_t M, const void* carry, int32_t carry_prec,
                                void* workspace, size_t workspace_bytes, void* stream) {
    if (!groups || n < 1 || n > TVLP_MAX_GROUPS) return TVLP_ERR_ARG;
    int64_t Bs[TVLP_MAX_GROUPS];
    for (int i = 0; i < n; ++i) {
        const tvlp_lp_bwd_group& g = groups[i];
        if (!g.grad_s || !g.A || !g.s || !g.grad_e || !g.grad_A) return TVLP_ERR_ARG;
        Bs[i] = g.B;
    }
    Plan p;
    int rc = grouped_plan(dtype, n, Bs, T, M, p);
    if (rc != TVLP_OK) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (dtype == TVLP_F64)
        return grouped_backward_impl<double>(n, groups, p, carry, TVLP_CARRY_F64, workspace,
                                             workspace_bytes, st, nullptr);
    return grouped_backward_impl<float>(n, groups, p, carry, carry_prec, workspace,
                                        workspace_bytes, st, nullptr);
}

size_t tvlp_workspace_bytes_grouped(int32_t op, int32_t dtype, int32_t n, const int64_t* B,
                                    int64_t T, int32_t M) {
    if (!B || n < 1 || n > TVLP_MAX_GROUPS) return 0;
    Plan p;
    if (grouped_plan(dtype, n, B, T, M, p) != TVLP_OK) return 0;
    size_t need = 0;
    // the sizing pass covers the concatenation fallback (a superset of the
    // direct path's buffers)
    if (op == TVLP_OP_FWD_TV) {
        if (dtype == TVLP_F64)
            grouped_forward_impl<double>(n, nullptr, p, nullptr, TVLP_CARRY_F64, nullptr, 0,
                                         nullptr, 0, &need);
        else
            grouped_forward_impl<float>(n, nullptr, p, nullptr, TVLP_CARRY_AUTO, nullptr, 0,
                                        nullptr, 0, &need);
    } else if (op == TVLP_OP_BWD_TV) {
        if (dtype == TVLP_F64)
            grouped_backward_impl<double>(n, nullptr, p, nullptr, TVLP_CARRY_F64, nullptr, 0, 0,
                                          &need);
        else
            grouped_backward_impl<float>(n, nullptr, p, nullptr, TVLP_CARRY_AUTO, nullptr, 0, 0,
                                         &need);
    }
    const size_t direct = 3 * (size_t)p.B * p.nsub * mp4(p) * 8 +
                          chain_ctl_bytes(p.B, p.nsub, p.Mp) + 4096;
    return need > direct ? need : direct;
}

int tvlp_lp_forward_ti(int32_t dtype, const void* e, const void* a, const void* zi, void* s,
                       int64_t B, int64_t T, int32_t M, void* carry, int32_t carry_prec,
                       void* workspace, size_t workspace_bytes, int32_t* nonfinite, void* stream) {
    return fwd_entry(true, dtype, e, a, zi, s, B, T, M, carry, carry_prec, workspace,
                     workspace_bytes, nonfinite, stream);
}

int tvlp_lp_backward_ti(int32_t dtype, const void* grad_s, const void* a, const void* s,
                        const void* zi, void* grad_e, void* grad_a, int64_t B, int64_t T,
                        int32_t M, const void* carry, int32_t carry_prec, void* workspace,
                        size_t workspace_bytes, void* stream) {
    return bwd_entry(true, dtype, grad_s, a, s, zi, grad_e, grad_a, B, T, M, carry, carry_prec,
                     workspace, workspace_bytes, stream);
}

int tvlp_shift_coeffs(int32_t dtype, const void* A, void* out, int64_t B, int64_t T, int32_t M,
                      void* stream) {
    if (dtype != TVLP_F32 && dtype != TVLP_F64) return TVLP_ERR_ARG;
    if (!A || !out || B < 1 || T < 1 || M < 1) return TVLP_ERR_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const unsigned grid = grid_for(B * T * M);
    if (dtype == TVLP_F64)
        launch_pdl(k_shift<double>, grid, 256, 0, st, static_cast<const double*>(A),
                                              static_cast<double*>(out), B, T, M);
    else
        launch_pdl(k_shift<float>, grid, 256, 0, st, static_cast<const float*>(A),
                                             static_cast<float*>(out), B, T, M);
    TVLP_CK(cudaGetLastError());
    return TVLP_OK;
}

int tvlp_lagged_signal_matrix(int32_t dtype, const void* s, const void* zi, void* out, int64_t B,
                              int64_t T, int32_t M, void* stream) {
    if (dtype != TVLP_F32 && dtype != TVLP_F64) return TVLP_ERR_ARG;
    if (!s || !out || B < 1 || T < 1 || M < 1) return TVLP_ERR_ARG;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const unsigned grid = grid_for(B * T * M);
    if (dtype == TVLP_F64)
        launch_pdl(k_lag<double>, grid, 256, 0, st, static_cast<const double*>(s),
                                            static_cast<const double*>(zi),
                                            static_cast<double*>(out), B, T, M);
    else
        launch_pdl(k_lag<float>, grid, 256, 0, st, static_cast<const float*>(s),
                                           static_cast<const float*>(zi),
                                           static_cast<float*>(out), B, T, M);
    TVLP_CK(cudaGetLastError());
    return TVLP_OK;
}

int tvlp_framewise_forward_ex(int32_t dtype, const void* e, const void* frames,
                              const void* window, double cola, void* out, void* seg, void* aux,
                              int64_t B, int64_t T, int64_t F, int32_t M, int32_t frame_size,
                              int32_t hop, void* workspace, size_t workspace_bytes,
                              void* stream) {
    int rc = check_common(dtype, M);
    if (rc != TVLP_OK) return rc;
    if (!e || !frames || !window || !out || !seg) return TVLP_ERR_ARG;
    FwArgs a;
    if (!fw_args(B, T, F, M, frame_size, hop, cola, a)) return TVLP_ERR_ARG;
    if (fw_aux_elems(a, padded_order(M)) == 0) aux = nullptr;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (dtype == TVLP_F64)
        return fw_forward_impl<double>(e, frames, window, out, seg, a, M, workspace,
                                       workspace_bytes, st, nullptr, aux);
    return fw_forward_impl<float>(e, frames, window, out, seg, a, M, workspace, workspace_bytes,
                                  st, nullptr, aux);
}

int tvlp_framewise_forward(int32_t dtype, const void* e, const void* frames, const void* window,
                           double cola, void* out, void* seg, int64_t B, int64_t T, int64_t F,
                           int32_t M, int32_t frame_size, int32_t hop, void* workspace,
                           size_t workspace_bytes, void* stream) {
    return tvlp_framewise_forward_ex(dtype, e, frames, window, cola, out, seg, nullptr, B, T, F,
                                     M, frame_size, hop, workspace, workspace_bytes, stream);
}

int tvlp_framewise_backward_ex(int32_t dtype, const void* grad_out, const void* frames,
                               const void* window, double cola, const void* seg,
                               const void* aux, void* grad_e, void* grad_frames, int64_t B,
                               int64_t T, int64_t F, int32_t M, int32_t frame_size, int32_t hop,
                               void* workspace, size_t workspace_bytes, void* stream) {
    int rc = check_common(dtype, M);
    if (rc != TVLP_OK) return rc;
    if (!grad_out || !frames || !window || !seg || !grad_e || !grad_frames) return TVLP_ERR_ARG;
    FwArgs a;
    if (!fw_args(B, T, F, M, frame_size, hop, cola, a)) return TVLP_ERR_ARG;
    if (fw_aux_elems(a, padded_order(M)) == 0) aux = nullptr;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (dtype == TVLP_F64)
        return fw_backward_impl<double>(grad_out, frames, window, seg, grad_e, grad_frames, a, M,
                                        workspace, workspace_bytes, st, nullptr, aux);
    return fw_backward_impl<float>(grad_out, frames, window, seg, grad_e, grad_frames, a, M,
                                   workspace, workspace_bytes, st, nullptr, aux);
}

int tvlp_framewise_backward(int32_t dtype, const void* grad_out, const void* frames,
                            const void* window, double cola, const void* seg, void* grad_e,
                            void* grad_frames, int64_t B, int64_t T, int64_t F, int32_t M,
                            int32_t frame_size, int32_t hop, void* workspace,
                            size_t workspace_bytes, void* stream) {
    return tvlp_framewise_backward_ex(dtype, grad_out, frames, window, cola, seg, nullptr, grad_e,
                                      grad_frames, B, T, F, M, frame_size, hop, workspace,
                                      workspace_bytes, stream);
}

int64_t tvlp_framewise_aux_elems(int64_t B, int64_t T, int64_t F, int32_t M, int32_t frame_size,
                                 int32_t hop) {
    FwArgs a;
    if (M < 1 || M > kMaxOrder || !fw_args(B, T, F, M, frame_size, hop, 1.0, a)) return 0;
    return fw_aux_elems(a, padded_order(M));
}

}  // extern "C"
