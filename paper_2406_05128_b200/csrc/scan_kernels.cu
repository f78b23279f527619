#include <cstdlib>
// scan_kernels.cu -- instantiations and launchers of the chunked-scan kernels.
#include <cstring>

#include <cudaTypedefs.h>

#include "lp_scan.cuh"
#include "scan_launch.cuh"

namespace tvlp {

namespace {

template <typename K>
cudaError_t ensure_smem(K kernel, int bytes) {
    if (bytes <= 48 * 1024) return cudaSuccess;
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

#ifndef TVLP_BASIS_WARPS
#define TVLP_BASIS_WARPS 4
#endif
constexpr int kBasisWarps = TVLP_BASIS_WARPS;

template <typename IO, typename ACC, int M, bool TI>
cudaError_t basis_impl(const IO* e, const IO* A, IO* PhiZ, const ScanArgs& g,
                       cudaStream_t st) {
    using S = BasisSmem<IO, ACC, M, TI, kBasisWarps>;
    auto k = k_basis<IO, ACC, M, TI, kBasisWarps>;
    cudaError_t err = ensure_smem(k, S::BYTES);
    if (err != cudaSuccess) return err;
    const int64_t nsc = g.B * g.nsub;
    const int64_t blocks = (nsc + kBasisWarps - 1) / kBasisWarps;
    launch_pdl(k, (unsigned)blocks, kBasisWarps * 32, S::BYTES, st, e, A, PhiZ, g);
    return cudaGetLastError();
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
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

// 2-D row-major view [dim1, dim0] of `base`, box {box0, box1}
cudaError_t map2d(CUtensorMap* m, const void* base, int sz, uint64_t dim0, uint64_t dim1,
                  uint32_t box0, uint32_t box1) {
    std::memset(m, 0, sizeof(*m));
    if (base == nullptr) return cudaSuccess;
    auto fn = encode_fn();
    if (!fn) return cudaErrorNotSupported;
    cuuint64_t gdim[2] = {dim0, dim1};
    cuuint64_t gstr[1] = {dim0 * (uint64_t)sz};
    cuuint32_t box[2] = {box0, box1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = fn(m, sz == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                    2, const_cast<void*>(base), gdim, gstr, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// 3-D view [ntapes][rows][MP4] of a carry tape array, box [cb][box_rows][MP4]
cudaError_t map_tapes(CUtensorMap* m, const void* base, int sz, int mp4, int rows,
                      uint64_t ntapes, int tape_elems_, uint32_t box_rows, uint32_t cb) {
    std::memset(m, 0, sizeof(*m));
    auto fn = encode_fn();
    if (!fn) return cudaErrorNotSupported;
    cuuint64_t gdim[3] = {(cuuint64_t)mp4, (cuuint64_t)rows, ntapes};
    cuuint64_t gstr[2] = {(cuuint64_t)mp4 * sz, (cuuint64_t)tape_elems_ * sz};
    cuuint32_t box[3] = {(cuuint32_t)mp4, box_rows, cb};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = fn(m, sz == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                    3, const_cast<void*>(base), gdim, gstr, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <typename IO, int M, bool TI>
cudaError_t lane_maps(LaneMaps& mp, const IO* A, const IO* X, const IO* O, const ScanArgs& g) {
    using S = LaneSmem<IO, M, TI>;
    const uint64_t rows = (uint64_t)g.B * g.nsub;
    cudaError_t err = cudaSuccess;
    if (!TI) err = map2d(&mp.A, A, S::SZ, (uint64_t)g.Ls * M, rows, S::AROW, 32);
    else std::memset(&mp.A, 0, sizeof(mp.A));
    if (err == cudaSuccess) err = map2d(&mp.X, X, S::SZ, (uint64_t)g.Ls, rows, S::XROW, 32);
    if (err == cudaSuccess) err = map2d(&mp.O, O, S::SZ, (uint64_t)g.Ls, rows, S::W, 32);
    mp.o = const_cast<IO*>(O);
    return err;
}

template <int M, bool TI, bool FR = false>
cudaError_t basis4_impl(const float* e, const float* A, float* PhiZ, const ScanArgs& g,
                        cudaStream_t st, const FrameSrc<float>* fr = nullptr) {
    using C = Basis4Cfg<M, TI>;
    auto k = k_basis4<M, TI, FR>;
    cudaError_t err = ensure_smem(k, C::BYTES);
    if (err != cudaSuccess) return err;
    const int64_t nsc = g.B * g.nsub;
    const int64_t per = (int64_t)C::S * C::NW;
    const FrameSrc<float> fs = fr ? *fr : FrameSrc<float>{};
    launch_pdl(k, (unsigned)((nsc + per - 1) / per), C::NW * 32, C::BYTES, st, e, A, PhiZ, g, fs);
    return cudaGetLastError();
}

template <typename IO, int M, bool TI, bool FR = false>
cudaError_t apply_impl(const IO* e, const IO* A, const IO* Xin, IO* s, int* flag, IO* Xend,
                       unsigned* dstat, const int* only, const ScanArgs& g, cudaStream_t st,
                       const FrameSrc<IO>* fr = nullptr, const RefineSrc<IO>* rf = nullptr) {
    using S = LaneSmem<IO, M, TI || FR>;
    auto k = k_apply_fwd<IO, M, TI, FR>;
    if constexpr (sizeof(IO) == 4)  // precision "auto" (fp32 I/O only)
        if (rf != nullptr && rf->tape != nullptr) k = k_apply_fwd<IO, M, TI, FR, true>;
    cudaError_t err = ensure_smem(k, S::BYTES);
    if (err != cudaSuccess) return err;
    LaneMaps mp;
    err = lane_maps<IO, M, TI || FR>(mp, (TI || FR) ? nullptr : A, e, s, g);
    if (err != cudaSuccess) return err;
    const int64_t nsc = g.B * g.nsub;
    const FrameSrc<IO> fs = fr ? *fr : FrameSrc<IO>{};
    const RefineSrc<IO> rs = rf ? *rf : RefineSrc<IO>{};
    launch_pdl(k, (unsigned)((nsc + 31) / 32), 32, S::BYTES, st, mp, TI ? A : nullptr, Xin, flag,
               Xend, dstat, only, g, fs, rs);
    return cudaGetLastError();
}

template <typename IO, int M, bool TI, int MODE, bool FR = false>
cudaError_t adjoint_impl(const IO* gs, const IO* A, const IO* Mu, IO* Nu, IO* ge,
                         unsigned* dstat, const int* only, const ScanArgs& g, cudaStream_t st,
                         const FrameSrc<IO>* fr = nullptr, const RefineSrc<IO>* rf = nullptr) {
    using S = LaneSmem<IO, M, TI || FR>;
    auto k = k_adjoint<IO, M, TI, MODE, FR>;
    if constexpr (sizeof(IO) == 4 && MODE == 1)
        if (rf != nullptr && rf->tape != nullptr) k = k_adjoint<IO, M, TI, MODE, FR, true>;
    cudaError_t err = ensure_smem(k, S::BYTES);
    if (err != cudaSuccess) return err;
    LaneMaps mp;
    err = lane_maps<IO, M, TI || FR>(mp, (TI || FR) ? nullptr : A, gs, MODE == 1 ? ge : nullptr,
                                     g);
    if (err != cudaSuccess) return err;
    const int64_t nsc = g.B * g.nsub;
    const FrameSrc<IO> fs = fr ? *fr : FrameSrc<IO>{};
    const RefineSrc<IO> rs = rf ? *rf : RefineSrc<IO>{};
    launch_pdl(k, (unsigned)((nsc + 31) / 32), 32, S::BYTES, st, mp, TI ? A : nullptr, Mu, Nu,
               dstat, only, g, fs, rs);
    return cudaGetLastError();
}

#define TVLP_DISPATCH_M(Mp, ...)                           \
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

}  // namespace

template <typename IO>
cudaError_t launch_basis(int Mp, bool ti, int prec, const IO* e, const IO* A, IO* PhiZ,
                         const ScanArgs& g, cudaStream_t st, const FrameSrc<IO>* fr) {
    TVLP_DISPATCH_M(Mp, {
        if constexpr (std::is_same<IO, float>::value) {
            if (fr != nullptr)  // frame-rate rows: fp32 chains, TV only (the caller checks)
                return basis4_impl<M_, false, true>(e, A, PhiZ, g, st, fr);
            if (prec == kPrecF32Chains || prec == kPrecAuto)
                return ti ? basis4_impl<M_, true>(e, A, PhiZ, g, st)
                          : basis4_impl<M_, false>(e, A, PhiZ, g, st);
        }
        return ti ? basis_impl<IO, double, M_, true>(e, A, PhiZ, g, st)
                  : basis_impl<IO, double, M_, false>(e, A, PhiZ, g, st);
    })
}

int tape_elems(int Mp) {
    switch (Mp) {
#define TVLP_TE(m) \
    case m: return Tape<m>::SIZE;
        TVLP_TE(2) TVLP_TE(4) TVLP_TE(6) TVLP_TE(8) TVLP_TE(12) TVLP_TE(16) TVLP_TE(22) TVLP_TE(24)
        TVLP_TE(30)
#undef TVLP_TE
        default: return -1;
    }
}

// Few long chains (one per sequence) want deep bulk copies (8 tapes per
// stage); many short segments (the hierarchy's groups) want small rings so
// several segments share an SM.
template <int M, typename IO, int CBW>
cudaError_t carry_tmap(CarryArgs<IO>& a, bool fwd) {
    using SM = CarrySmem<M, IO, CBW>;
    const int64_t nper = (a.nsub + a.seglen - 1) / a.seglen;
    const uint64_t ntapes = (uint64_t)(a.nseg / nper) * a.nsub;
    a.use_tmap = 1;
    return map_tapes(&a.tmap, a.tape, (int)sizeof(IO), Tape<M>::MP4, 2 * M + 1, ntapes,
                     Tape<M>::SIZE, fwd ? M + 1 : M, SM::CB);
}

template <int M, typename IO, int CBW>
cudaError_t carry_fwd_cb(const CarryArgs<IO>& a0, cudaStream_t st) {
    using SM = CarrySmem<M, IO, CBW>;
    auto k = k_carry_fwd<M, IO, CBW, (CBW < kCB)>;
    cudaError_t err = ensure_smem(k, SM::BYTES);
    if (err != cudaSuccess) return err;
    CarryArgs<IO> a = a0;
    if (CBW < kCB) {  // many short segments: tensor copies of the needed rows (measured
                      // faster there; one 1-D copy of whole tapes is faster for long chains)
        err = carry_tmap<M, IO, CBW>(a, true);
        if (err != cudaSuccess) return err;
    }
    launch_pdl(k, (unsigned)a.nseg, 32, SM::BYTES, st, a);
    return cudaGetLastError();
}
template <int M, typename IO>
cudaError_t carry_fwd_impl(const CarryArgs<IO>& a, cudaStream_t st) {
    return a.nseg <= 296 ? carry_fwd_cb<M, IO, kCB>(a, st) : carry_fwd_cb<M, IO, 2>(a, st);
}

template <int M, typename IO, int CBW>
cudaError_t carry_bwd_cb(const CarryArgs<IO>& a0, cudaStream_t st) {
    using SM = CarrySmem<M, IO, CBW>;
    auto k = k_carry_bwd<M, IO, CBW, (CBW < kCB)>;
    cudaError_t err = ensure_smem(k, SM::BYTES);
    if (err != cudaSuccess) return err;
    CarryArgs<IO> a = a0;
    if (CBW < kCB) {
        err = carry_tmap<M, IO, CBW>(a, false);
        if (err != cudaSuccess) return err;
    }
    launch_pdl(k, (unsigned)a.nseg, 32, SM::BYTES, st, a);
    return cudaGetLastError();
}
template <int M, typename IO>
cudaError_t carry_bwd_impl(const CarryArgs<IO>& a, cudaStream_t st) {
    return a.nseg <= 296 ? carry_bwd_cb<M, IO, kCB>(a, st) : carry_bwd_cb<M, IO, 2>(a, st);
}

template <int M, typename IO>
cudaError_t group_P_impl(const IO* tape, IO* gtape, int64_t ngroups, int G, int nsub,
                         const int* only, cudaStream_t st) {
    // product tree (default) or one warp of serial mat-mats ($TVLP_COMPOSE_TREE=0)
    static const int tree = [] {
        const char* v = std::getenv("TVLP_COMPOSE_TREE");
        return (v != nullptr && v[0] != 0) ? std::atoi(v) : 1;
    }();
    const size_t tb = (size_t)G * M * Tape<M>::MP4 * sizeof(IO) + 16;
    if (tree && tb <= 220 * 1024) {
        auto kt = k_group_P_tree<M, IO>;
        cudaError_t err = ensure_smem(kt, (int)tb);
        if (err != cudaSuccess) return err;
        launch_pdl(kt, (unsigned)ngroups, kTreeWarps * 32, tb, st, tape, gtape, ngroups, G, nsub,
                   only);
        return cudaGetLastError();
    }
    using SM = CarrySmem<M, IO, 4>;
    auto k = k_group_P<M, IO>;
    cudaError_t err = ensure_smem(k, SM::BYTES);
    if (err != cudaSuccess) return err;
    launch_pdl(k, (unsigned)ngroups, 32, SM::BYTES, st, tape, gtape, ngroups, G, nsub, only);
    return cudaGetLastError();
}

template <typename IO>
cudaError_t launch_carry_fwd(int Mp, const CarryArgs<IO>& a, cudaStream_t st) {
    TVLP_DISPATCH_M(Mp, { return carry_fwd_impl<M_, IO>(a, st); })
}

unsigned long long refined_sequences() {
    unsigned long long v = 0;
    cudaMemcpyFromSymbol(&v, g_refined_sequences, sizeof(v));
    return v;
}

template <typename IO>
cudaError_t launch_carry_bwd(int Mp, const CarryArgs<IO>& a, cudaStream_t st) {
    TVLP_DISPATCH_M(Mp, { return carry_bwd_impl<M_, IO>(a, st); })
}

template <typename IO>
cudaError_t launch_group_P(int Mp, const IO* tape, IO* gtape, int64_t ngroups, int G, int nsub,
                           const int* only, cudaStream_t st) {
    TVLP_DISPATCH_M(Mp, { return group_P_impl<M_, IO>(tape, gtape, ngroups, G, nsub, only, st); })
}

// what: 0 = decide, 1 = defects, 2 = add (X=P as mutable, E=Q)
template <typename IO>
cudaError_t launch_refine_helpers(int what, int Mp, const IO* P, const IO* Q, IO* D, int nsub,
                                  bool fwd, const int* only, int* flags, const unsigned* dstat,
                                  const int* inherit, float tol, int64_t B, cudaStream_t st) {
    const int mp4 = (Mp + 3) / 4 * 4;
    const int64_t n = B * (int64_t)nsub * mp4;
    int64_t grid = (n + 255) / 256;
    if (grid > 148 * 32) grid = 148 * 32;
    if (grid < 1) grid = 1;
    if (what == 0)
        launch_pdl(k_refine_decide, (unsigned)((B + 127) / 128), 128, 0, st, dstat, flags, inherit, tol, B);
    else if (what == 1)
        launch_pdl(k_defects<IO>, (unsigned)grid, 256, 0, st, P, Q, D, nsub, mp4, Mp, fwd, only, B);
    else
        launch_pdl(k_add_rows<IO>, (unsigned)grid, 256, 0, st, const_cast<IO*>(P), Q, nsub, mp4, only, B);
    return cudaGetLastError();
}

template <typename IO>
cudaError_t launch_apply_fwd(int Mp, bool ti, const IO* e, const IO* A, const IO* Xin, IO* s,
                             int* flag, IO* Xend, unsigned* dstat, const int* only,
                             const ScanArgs& g, cudaStream_t st, const FrameSrc<IO>* fr,
                             const RefineSrc<IO>* rf) {
    TVLP_DISPATCH_M(Mp, {
        if constexpr (std::is_same<IO, float>::value) {
            if (fr != nullptr)
                return apply_impl<IO, M_, false, true>(e, A, Xin, s, flag, Xend, dstat, only, g,
                                                       st, fr, rf);
        }
        return ti ? apply_impl<IO, M_, true>(e, A, Xin, s, flag, Xend, dstat, only, g, st,
                                             nullptr, rf)
                  : apply_impl<IO, M_, false>(e, A, Xin, s, flag, Xend, dstat, only, g, st,
                                              nullptr, rf);
    })
}

template <typename IO>
cudaError_t launch_refine(int Mp, bool fwd, const IO* tape, IO* X, const IO* Xend,
                          const unsigned* dstat, int* flags, const int* fflags, const ScanArgs& g,
                          cudaStream_t st) {
    TVLP_DISPATCH_M(Mp, {
        if (fwd)
            launch_pdl(k_refine_fwd<M_, IO>, (unsigned)g.B, 32, 0, st, tape, X, Xend, dstat, flags, g.nsub,
                                                               g.B);
        else
            launch_pdl(k_refine_bwd<M_, IO>, (unsigned)g.B, 32, 0, st, tape, X, Xend, dstat, flags, g.nsub,
                                                               g.B, fflags);
        return cudaGetLastError();
    })
}

template <typename IO>
cudaError_t launch_adjoint(int Mp, bool ti, int mode, const IO* gs, const IO* A, const IO* Mu,
                           IO* Nu, IO* ge, unsigned* dstat, const int* only, const ScanArgs& g,
                           cudaStream_t st, const FrameSrc<IO>* fr, const RefineSrc<IO>* rf) {
    TVLP_DISPATCH_M(Mp, {
        if constexpr (std::is_same<IO, float>::value) {
            if (fr != nullptr)
                return mode == 0 ? adjoint_impl<IO, M_, false, 0, true>(gs, A, Mu, Nu, ge, dstat,
                                                                        only, g, st, fr, rf)
                                 : adjoint_impl<IO, M_, false, 1, true>(gs, A, Mu, Nu, ge, dstat,
                                                                        only, g, st, fr, rf);
        }
        if (mode == 0)
            return ti ? adjoint_impl<IO, M_, true, 0>(gs, A, Mu, Nu, ge, dstat, only, g, st,
                                                      nullptr, rf)
                      : adjoint_impl<IO, M_, false, 0>(gs, A, Mu, Nu, ge, dstat, only, g, st,
                                                       nullptr, rf);
        return ti ? adjoint_impl<IO, M_, true, 1>(gs, A, Mu, Nu, ge, dstat, only, g, st, nullptr,
                                                  rf)
                  : adjoint_impl<IO, M_, false, 1>(gs, A, Mu, Nu, ge, dstat, only, g, st, nullptr,
                                                   rf);
    })
}

template <typename IO>
cudaError_t launch_upsample(int Mp, const FrameSrc<IO>& fr, IO* A, int64_t B, int64_t T,
                            cudaStream_t st) {
    int64_t blocks = (B * T + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    TVLP_DISPATCH_M(Mp, {
        launch_pdl(k_upsample<IO, M_>, (unsigned)blocks, 256, 0, st, fr, A, B, T);
        return cudaGetLastError();
    })
}

template <typename IO>
cudaError_t launch_grad_frames(const FrameSrc<IO>& fr, const IO* ge, const IO* s, const IO* zi,
                               int Mzi, IO* gF, int64_t B, int64_t T, cudaStream_t st) {
    if (fr.Mf > 32) return cudaErrorInvalidValue;
    const size_t sm = (size_t)(2 * (kFramesPerCta + 1) * fr.hop + 32) * sizeof(IO);
    if (sm > 200 * 1024) return cudaErrorInvalidValue;
    auto k = k_grad_frames<IO>;
    cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (err != cudaSuccess) return err;
    launch_pdl(k, dim3((unsigned)((fr.nF + kFramesPerCta - 1) / kFramesPerCta), (unsigned)B),
               kFramesPerCta * 16, sm, st, fr, ge, s, zi, Mzi, gF, T);
    return cudaGetLastError();
}

template <typename IO>
cudaError_t launch_grad_A(int Mp, const IO* ge, const IO* s, const IO* zi, IO* gA, int64_t B,
                          int64_t T, cudaStream_t st) {
    dim3 grid((unsigned)((T + 255) / 256), (unsigned)B);
    TVLP_DISPATCH_M(Mp, {
        launch_pdl(k_grad_A<IO, M_>, grid, 256, 0, st, ge, s, zi, gA, T);
        return cudaGetLastError();
    })
}

template <typename IO>
cudaError_t launch_grad_a(int M, const IO* ge, const IO* s, const IO* zi, IO* part, IO* ga,
                          int64_t B, int64_t T, int nchunk, cudaStream_t st) {
    dim3 grid((unsigned)nchunk, (unsigned)B);
    launch_pdl(k_grad_a_partial<IO>, grid, 256, 0, st, ge, s, zi, part, T, M, nchunk);
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) return err;
    launch_pdl(k_grad_a_final<IO>, (unsigned)((B * M + 127) / 128), 128, 0, st, part, ga, B, M, nchunk);
    return cudaGetLastError();
}

#define TVLP_INST(IO)                                                                            \
    template cudaError_t launch_basis<IO>(int, bool, int, const IO*, const IO*, IO*,             \
                                          const ScanArgs&, cudaStream_t, const FrameSrc<IO>*);   \
    template cudaError_t launch_carry_fwd<IO>(int, const CarryArgs<IO>&, cudaStream_t);          \
    template cudaError_t launch_carry_bwd<IO>(int, const CarryArgs<IO>&, cudaStream_t);          \
    template cudaError_t launch_group_P<IO>(int, const IO*, IO*, int64_t, int, int, const int*,  \
                                            cudaStream_t);                                       \
    template cudaError_t launch_refine_helpers<IO>(int, int, const IO*, const IO*, IO*, int,     \
                                                   bool, const int*, int*, const unsigned*,      \
                                                   const int*, float, int64_t, cudaStream_t);    \
    template cudaError_t launch_apply_fwd<IO>(int, bool, const IO*, const IO*, const IO*, IO*,   \
                                              int*, IO*, unsigned*, const int*, const ScanArgs&, \
                                              cudaStream_t, const FrameSrc<IO>*,                 \
                                              const RefineSrc<IO>*);                             \
    template cudaError_t launch_adjoint<IO>(int, bool, int, const IO*, const IO*, const IO*,     \
                                            IO*, IO*, unsigned*, const int*, const ScanArgs&,    \
                                            cudaStream_t, const FrameSrc<IO>*,                   \
                                            const RefineSrc<IO>*);                               \
    template cudaError_t launch_refine<IO>(int, bool, const IO*, IO*, const IO*,                 \
                                           const unsigned*, int*, const int*, const ScanArgs&,   \
                                           cudaStream_t);                                        \
    template cudaError_t launch_upsample<IO>(int, const FrameSrc<IO>&, IO*, int64_t, int64_t,      \
                                             cudaStream_t);                                       \
    template cudaError_t launch_grad_frames<IO>(const FrameSrc<IO>&, const IO*, const IO*,         \
                                                const IO*, int, IO*, int64_t, int64_t,            \
                                                cudaStream_t);                                    \
    template cudaError_t launch_grad_A<IO>(int, const IO*, const IO*, const IO*, IO*, int64_t,   \
                                           int64_t, cudaStream_t);                               \
    template cudaError_t launch_grad_a<IO>(int, const IO*, const IO*, const IO*, IO*, IO*,       \
                                           int64_t, int64_t, int, cudaStream_t);
TVLP_INST(float)
TVLP_INST(double)

}  // namespace tvlp
