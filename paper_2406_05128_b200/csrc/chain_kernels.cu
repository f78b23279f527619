// chain_kernels.cu -- instantiations and launchers of the chained single-pass
// scans (chain.cuh).
#include <cstdlib>
#include <cstring>

#include <cudaTypedefs.h>

#include "chain.cuh"
#include "chain_launch.cuh"
#include "scan_launch.cuh"

namespace tvlp {
UnitGeo chain_units_n(int nsub, int U);
namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode() {
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

// 2-D row-major fp32 view [dim1, dim0], box {box0, box1}
cudaError_t view2d(CUtensorMap* m, const void* base, uint64_t dim0, uint64_t dim1, uint32_t box0,
                   uint32_t box1) {
    std::memset(m, 0, sizeof(*m));
    if (base == nullptr) return cudaSuccess;  // (TI: no coefficient stream)
    auto fn = encode();
    if (!fn) return cudaErrorNotSupported;
    cuuint64_t gdim[2] = {dim0, dim1};
    cuuint64_t gstr[1] = {dim0 * 4};
    cuuint32_t box[2] = {box0, box1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), gdim, gstr, box,
                    es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// 3-D view [ntapes][2M+1][MP4] of the carry tape, box [8][rows][MP4]
cudaError_t view_tapes(CUtensorMap* m, const void* base, int M, int mp4, int tsize,
                       uint64_t ntapes, uint32_t rows) {
    std::memset(m, 0, sizeof(*m));
    auto fn = encode();
    if (!fn) return cudaErrorNotSupported;
    cuuint64_t gdim[3] = {(cuuint64_t)mp4, (cuuint64_t)(2 * M + 1), ntapes};
    cuuint64_t gstr[2] = {(cuuint64_t)mp4 * 4, (cuuint64_t)tsize * 4};
    cuuint32_t box[3] = {(cuuint32_t)mp4, rows, 8};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), gdim, gstr, box,
                    es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int M, int U, int NST>
cudaError_t unit_maps(UnitMaps& mp, const float* A, const float* X, const float* O,
                      const ScanArgs& g, const UnitGeo& u) {
    using S = UnitLane<M, U, NST>;
    const uint64_t rows = (uint64_t)g.B * g.nsub;
    const uint32_t box[2] = {(uint32_t)u.U, (uint32_t)u.rem};
    for (int i = 0; i < 2; ++i) {
        cudaError_t err = view2d(&mp.A[i], A, (uint64_t)g.Ls * M, rows, S::AROW, box[i]);
        if (err == cudaSuccess) err = view2d(&mp.X[i], X, (uint64_t)g.Ls, rows, S::XROW, box[i]);
        if (err == cudaSuccess) err = view2d(&mp.O[i], O, (uint64_t)g.Ls, rows, S::W, box[i]);
        if (err != cudaSuccess) return err;
    }
    mp.o = const_cast<float*>(O);
    return cudaSuccess;
}

int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return (v != nullptr && v[0] != 0) ? std::atoi(v) : dflt;
}

int sm_count() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 1)
            n = 148;
    }
    return n;
}

template <typename K>
cudaError_t set_smem(K kernel, int bytes) {
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

ChainTrace g_trace{nullptr, 0};

// Persistent-style grid for `units` equal work items: as many warps as fit
// (or $env), then evened out so every round is full (a last round of a few
// items would run at a fraction of the machine).
template <typename K>
int64_t balanced_grid(int64_t units, K kernel, int threads, int smem, const char* env) {
    int per_sm = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem) !=
            cudaSuccess ||
        per_sm < 1)
        per_sm = 1;
    int64_t g0 = env_int(env, sm_count() * per_sm);
    if (g0 < 1) g0 = 1;
    if (units <= g0) return units;
    const int64_t rounds = units / g0;  // >= 1
    return (units + rounds - 1) / rounds;
}

// Control words of a chained launch, zeroed by a kernel launched ahead of
// the pass that precedes the chained kernel: unlike a memset node it
// keeps the stream's programmatic dependent launches chained.
__global__ void k_zero_ctl(uint4* p, size_t n16) {
    grid_dep_wait();
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16;
         i += (size_t)gridDim.x * blockDim.x)
        p[i] = make_uint4(0u, 0u, 0u, 0u);
}
cudaError_t zero_ctl(void* p, size_t bytes, cudaStream_t st) {
    const size_t n16 = bytes / 16;
    unsigned grid = (unsigned)((n16 + 255) / 256);
    if (grid > 148) grid = 148;
    if (grid < 1) grid = 1;
    launch_pdl(k_zero_ctl, grid, 256, 0, st, static_cast<uint4*>(p), n16);
    return cudaGetLastError();
}

// Boundary-defect tolerance of precision "auto".  Unrefined defects add up
// over a sequence's boundaries (undamped on near-unit-circle rows), so the
// chained path detects at half the single-level path's 2e-5 (lp_scan.cuh
// kDefectTol): measured on config 3, D1 defects stay below 4e-6 of max|x|
// (nothing refined), while resonant rows whose 2e-5-level defects had summed
// to 1.6e-4 in the output are caught (tools/stress_prec.py).
// $TVLP_DEFECT_TOL overrides (experiments).
float defect_tol(int nsub, bool fwd) {
    (void)nsub;
    static const char* env = std::getenv("TVLP_DEFECT_TOL");
    if (env != nullptr && env[0] != 0) return (float)std::atof(env);
    return 0.5f * (fwd ? kDefectTol : kDefectTolBwd);
}

struct CtlLayout {
    size_t ticket, cnt, done, dstat, pub, bytes;
};
CtlLayout ctl_layout(int64_t B, const UnitGeo& u, int mp4) {
    CtlLayout c;
    size_t o = 0;
    auto take = [&](size_t n) {
        o = (o + 15) / 16 * 16;
        const size_t at = o;
        o += n;
        return at;
    };
    c.ticket = take(2 * sizeof(unsigned));
    c.cnt = take((size_t)B * u.nu * sizeof(unsigned));
    c.done = take((size_t)B * sizeof(unsigned));
    c.dstat = take((size_t)B * 3 * sizeof(unsigned));
    c.pub = take((size_t)B * u.nu * mp4 * sizeof(unsigned long long));
    c.bytes = (o + 255) / 256 * 256;
    return c;
}

GroupIdx group_index(int ng, const ChainGroup* grp) {
    GroupIdx gi;
    std::memset(&gi, 0, sizeof(gi));
    gi.ng = ng;
    int64_t acc = 0;
    for (int i = 0; i < ng; ++i) {
        gi.gB0[i] = acc;
        acc += grp[i].B;
    }
    for (int i = ng; i <= kMaxGroups; ++i) gi.gB0[i] = acc;
    return gi;
}

// a group's own ScanArgs (its B) for the per-group streaming launches
ScanArgs group_args(const ScanArgs& g, int64_t B) {
    ScanArgs s = g;
    s.B = B;
    return s;
}

template <int M, bool TI>
cudaError_t fwd_chain_impl(const ChainFwdCall& c, cudaStream_t st, int phase) {
    constexpr int NWB = TVLP_CHAIN_BASIS_WARPS, NST = TVLP_CHAIN_FWD_STAGES;
    using SM = FwdChainSmem<M, NWB, NST>;
    constexpr int MP4 = Tape<M>::MP4;
    const bool fr = c.fr != nullptr;  // frame-rate rows (TV, one group)
    auto k = fr ? k_fwd_chain<M, NWB, NST, false, true> : k_fwd_chain<M, NWB, NST, TI && NWB == 0>;
    if (fr && (TI || c.ng != 1 || NWB > 0)) return cudaErrorInvalidValue;
    cudaError_t err = set_smem(k, SM::BYTES);
    if (err != cudaSuccess) return err;
    if (c.ng < 1 || c.ng > kMaxGroups || (NWB > 0 && c.ng != 1)) return cudaErrorInvalidValue;
    const UnitGeo u = chain_units(c.g.nsub, true);
    const CtlLayout L = ctl_layout(c.g.B, u, MP4);
    unsigned char* ctl = static_cast<unsigned char*>(c.ctl);
    if (phase == 0) {
        // the control words, then the transition tapes (k_basis4, one launch
        // per group: each fills its own sequences' tapes)
        err = zero_ctl(ctl, L.bytes, st);
        if (err != cudaSuccess || NWB > 0) return err;
        if (c.ng == 1)
            return launch_basis<float>(M, TI, kPrecF32Chains, c.grp[0].x, c.grp[0].A, c.tape, c.g,
                                       st, c.fr);
        // groups: one launch over all of them (each lane picks its group)
        using BC = Basis4Cfg<M, TI>;
        auto kb = k_basis4_groups<M, TI>;
        err = set_smem(kb, BC::BYTES);
        if (err != cudaSuccess) return err;
        GroupSrc gs;
        std::memset(&gs, 0, sizeof(gs));
        gs.gi = group_index(c.ng, c.grp);
        for (int i = 0; i < c.ng; ++i) {
            gs.x[i] = c.grp[i].x;
            gs.A[i] = c.grp[i].A;
        }
        const int64_t per = (int64_t)BC::S * BC::NW;
        launch_pdl(kb, (unsigned)((c.g.B * c.g.nsub + per - 1) / per), BC::NW * 32, BC::BYTES, st,
                   gs, c.tape, c.g);
        return cudaGetLastError();
    }
    ChainFwdArgs a;
    std::memset(&a, 0, sizeof(a));
    a.gi = group_index(c.ng, c.grp);
    for (int i = 0; i < c.ng; ++i) {
        const ScanArgs gg = group_args(c.g, c.grp[i].B);
        err = unit_maps<M, SM::U, NST>(a.mp[i], (TI || fr) ? nullptr : c.grp[i].A, c.grp[i].x,
                                       c.grp[i].y, gg, u);
        if (err != cudaSuccess) return err;
        a.Ag[i] = c.grp[i].A;
        a.zig[i] = c.grp[i].zi;
    }
    if (fr) a.fs = *c.fr;
    err = view_tapes(&a.Tz, c.tape, M, MP4, Tape<M>::SIZE, (uint64_t)c.g.B * c.g.nsub, M + 1);
    if (err != cudaSuccess) return err;
    a.e = c.grp[0].x;
    a.A = c.grp[0].A;
    a.zs = c.zs;
    a.tape = c.tape;
    a.fflags = c.fflags;
    a.Xin = c.Xin;
    a.Xend = c.Xend;
    a.nonfinite = c.nonfinite;
    a.ticket = reinterpret_cast<unsigned*>(ctl + L.ticket);
    a.cnt = reinterpret_cast<unsigned*>(ctl + L.cnt);
    a.done = reinterpret_cast<unsigned*>(ctl + L.done);
    a.dstat = reinterpret_cast<unsigned*>(ctl + L.dstat);
    a.pub = reinterpret_cast<unsigned long long*>(ctl + L.pub);
    a.refine = c.refine;
    a.tol = defect_tol(c.g.nsub, true);
    a.g = c.g;
    a.u = u;
    a.tr = g_trace;
    int64_t grid;
    if constexpr (NWB > 0) {
        // persistent: one CTA per SM (the shared memory allows no second)
        const int64_t groups = c.g.B * ((c.g.nsub + 3) / 4);
        grid = env_int("TVLP_CHAIN_FWD_CTAS", sm_count());
        const int64_t need = (groups + NWB - 1) / NWB;
        if (grid > need) grid = need;
    } else {
        // the chained carries and re-application over the units of every group
        grid = balanced_grid(c.g.B * u.nu, k, (NWB + 1) * 32, SM::BYTES, "TVLP_CHAIN_FWD_CTAS");
    }
    if (grid < 1) grid = 1;
    launch_pdl(k, (unsigned)grid, (NWB + 1) * 32, SM::BYTES, st, a);
    return cudaGetLastError();
}

template <int M, bool TI>
cudaError_t bwd_chain_impl(const ChainBwdCall& c, cudaStream_t st, int phase) {
    constexpr int NST = TVLP_CHAIN_BWD_STAGES;
    constexpr bool ZS = TVLP_CHAIN_BWD_ZS != 0;
    using SM = BwdChainSmem<M, NST, ZS>;
    constexpr int MP4 = Tape<M>::MP4;
    const bool fr = c.fr != nullptr;  // frame-rate rows (TV, one group)
    auto k = fr ? k_bwd_chain<M, NST, ZS, false, true> : k_bwd_chain<M, NST, ZS, TI>;
    if (fr && (TI || c.ng != 1)) return cudaErrorInvalidValue;
    cudaError_t err = set_smem(k, SM::BYTES);
    if (err != cudaSuccess) return err;
    if (c.ng < 1 || c.ng > kMaxGroups) return cudaErrorInvalidValue;
    const UnitGeo u = chain_units(c.g.nsub, false);
    const CtlLayout L = ctl_layout(c.g.B, u, MP4);
    unsigned char* ctl = static_cast<unsigned char*>(c.ctl);
    if (phase == 0) {
        err = zero_ctl(ctl, L.bytes, st);
        if (err != cudaSuccess) return err;
        if constexpr (!ZS) {
            // the zero-state adjoints: the streaming k_adjoint<MODE 0> for one
            // group; for several, one launch of unit warps over all of them
            if (c.ng == 1)
                return launch_adjoint<float>(M, TI, 0, c.grp[0].x, c.grp[0].A, nullptr, c.Nu,
                                             nullptr, nullptr, nullptr, c.g, st, c.fr);
            constexpr int UZ = 32, NZ = 3;
            const UnitGeo uz = chain_units_n(c.g.nsub, UZ);
            ChainBwdArgs z;
            std::memset(&z, 0, sizeof(z));
            z.gi = group_index(c.ng, c.grp);
            for (int i = 0; i < c.ng; ++i) {
                err = unit_maps<M, UZ, NZ>(z.mp[i], TI ? nullptr : c.grp[i].A, c.grp[i].x,
                                           c.grp[i].y, group_args(c.g, c.grp[i].B), uz);
                if (err != cudaSuccess) return err;
                z.Ag[i] = c.grp[i].A;
            }
            z.Nu = c.Nu;
            z.g = c.g;
            z.u = uz;
            auto kz = k_adj_zs_units<M, UZ, NZ, TI>;
            const int smz = UnitLane<M, UZ, NZ>::BYTES + NZ * 8;
            err = set_smem(kz, smz);
            if (err != cudaSuccess) return err;
            launch_pdl(kz, (unsigned)(c.g.B * uz.nu), 32, smz, st, z);
            return cudaGetLastError();
        }
        return cudaSuccess;
    }
    ChainBwdArgs a;
    std::memset(&a, 0, sizeof(a));
    a.gi = group_index(c.ng, c.grp);
    for (int i = 0; i < c.ng; ++i) {
        err = unit_maps<M, SM::U, NST>(a.mp[i], (TI || fr) ? nullptr : c.grp[i].A, c.grp[i].x,
                                       c.grp[i].y, group_args(c.g, c.grp[i].B), u);
        if (err != cudaSuccess) return err;
        a.Ag[i] = c.grp[i].A;
    }
    if (fr) a.fs = *c.fr;
    err = view_tapes(&a.Tw, c.tape, M, MP4, Tape<M>::SIZE, (uint64_t)c.g.B * c.g.nsub, M);
    if (err != cudaSuccess) return err;
    a.Nu = c.Nu;
    a.tape = c.tape;
    a.inherit = c.inherit;
    a.Mu = c.Mu;
    a.Kout = c.Kout;
    a.ticket = reinterpret_cast<unsigned*>(ctl + L.ticket);
    a.done = reinterpret_cast<unsigned*>(ctl + L.done);
    a.dstat = reinterpret_cast<unsigned*>(ctl + L.dstat);
    a.pub = reinterpret_cast<unsigned long long*>(ctl + L.pub);
    a.refine = c.refine;
    a.tol = defect_tol(c.g.nsub, false);
    a.g = c.g;
    a.u = u;
    a.tr = g_trace;
    const int64_t grid = balanced_grid(c.g.B * u.nu, k, 32, SM::BYTES, "TVLP_CHAIN_BWD_CTAS");
    launch_pdl(k, (unsigned)grid, 32, SM::BYTES, st, a);
    return cudaGetLastError();
}

}  // namespace

UnitGeo chain_units_n(int nsub, int U) {
    UnitGeo u;
    u.U = U;
    u.nu = (nsub + u.U - 1) / u.U;
    u.rem = nsub - (u.nu - 1) * u.U;
    return u;
}

UnitGeo chain_units(int nsub, bool fwd) {
    return chain_units_n(nsub, fwd ? TVLP_CHAIN_FWD_UNIT : TVLP_CHAIN_BWD_UNIT);
}

bool chain_supported(int Mp) {
    static const int on = env_int("TVLP_CHAIN", 1);
    return on != 0 && Mp == 22;
}

size_t chain_ctl_bytes(int64_t B, int nsub, int Mp) {
    const int mp4 = (Mp + 3) / 4 * 4;
    const size_t f = ctl_layout(B, chain_units(nsub, true), mp4).bytes;
    const size_t b = ctl_layout(B, chain_units(nsub, false), mp4).bytes;
    return f > b ? f : b;
}

cudaError_t launch_fwd_chain(int Mp, const ChainFwdCall& c, cudaStream_t st, int phase) {
    switch (Mp) {
        case 22:
            return c.ti ? fwd_chain_impl<22, true>(c, st, phase)
                        : fwd_chain_impl<22, false>(c, st, phase);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_bwd_chain(int Mp, const ChainBwdCall& c, cudaStream_t st, int phase) {
    switch (Mp) {
        case 22:
            return c.ti ? bwd_chain_impl<22, true>(c, st, phase)
                        : bwd_chain_impl<22, false>(c, st, phase);
        default: return cudaErrorInvalidValue;
    }
}

void chain_set_trace(void* buf, size_t bytes) {
    g_trace.buf = static_cast<unsigned long long*>(buf);
    g_trace.cap = buf ? (unsigned)(bytes / 64) : 0u;
}

unsigned long long chain_refined_sequences() {
    unsigned long long v = 0;
    cudaMemcpyFromSymbol(&v, g_chain_refined, sizeof(v));
    return v;
}

}  // namespace tvlp
