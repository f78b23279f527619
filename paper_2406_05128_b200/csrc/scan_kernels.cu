// scan_kernels.cu -- instantiations and launchers of the chunked-scan kernels.
#include "lp_scan.cuh"
#include "scan_launch.cuh"

namespace tvlp {

namespace {

template <typename K>
cudaError_t ensure_smem(K kernel, int bytes) {
    if (bytes <= 48 * 1024) return cudaSuccess;
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
}

constexpr int kBasisWarps = 4;

template <typename IO, typename ACC, int M, bool TI>
cudaError_t basis_impl(const IO* e, const IO* A, IO* PhiZ, const ScanArgs& g,
                       cudaStream_t st) {
    using S = BasisSmem<IO, ACC, M, TI, kBasisWarps>;
    auto k = k_basis<IO, ACC, M, TI, kBasisWarps>;
    cudaError_t err = ensure_smem(k, S::BYTES);
    if (err != cudaSuccess) return err;
    const int64_t nsc = g.B * g.nsub;
    const int64_t blocks = (nsc + kBasisWarps - 1) / kBasisWarps;
    k<<<(unsigned)blocks, kBasisWarps * 32, S::BYTES, st>>>(e, A, PhiZ, g);
    return cudaGetLastError();
}

template <typename IO, int M, bool TI>
cudaError_t apply_impl(const IO* e, const IO* A, const IO* Xin, IO* s, int* flag,
                       const ScanArgs& g, cudaStream_t st) {
    using S = LaneSmem<IO, M, TI>;
    auto k = k_apply_fwd<IO, M, TI>;
    cudaError_t err = ensure_smem(k, S::BYTES);
    if (err != cudaSuccess) return err;
    const int64_t nsc = g.B * g.nsub;
    k<<<(unsigned)((nsc + 31) / 32), 32, S::BYTES, st>>>(e, A, Xin, s, flag, g);
    return cudaGetLastError();
}

template <typename IO, int M, bool TI, int MODE>
cudaError_t adjoint_impl(const IO* gs, const IO* A, const IO* Mu, IO* Nu, IO* ge,
                         const ScanArgs& g, cudaStream_t st) {
    using S = LaneSmem<IO, M, TI>;
    auto k = k_adjoint<IO, M, TI, MODE>;
    cudaError_t err = ensure_smem(k, S::BYTES);
    if (err != cudaSuccess) return err;
    const int64_t nsc = g.B * g.nsub;
    k<<<(unsigned)((nsc + 31) / 32), 32, S::BYTES, st>>>(gs, A, Mu, Nu, ge, g);
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

int ls_unit(int Mp) {
    switch (Mp) {
#define TVLP_LSU(m) \
    case m: return Geo<m>::LsUnit;
        TVLP_LSU(2) TVLP_LSU(4) TVLP_LSU(6) TVLP_LSU(8) TVLP_LSU(12) TVLP_LSU(16) TVLP_LSU(22)
        TVLP_LSU(24) TVLP_LSU(30)
#undef TVLP_LSU
        default: return -1;
    }
}

template <typename IO>
cudaError_t launch_basis(int Mp, bool ti, int prec, const IO* e, const IO* A, IO* PhiZ,
                         const ScanArgs& g, cudaStream_t st) {
    TVLP_DISPATCH_M(Mp, {
        if constexpr (std::is_same<IO, float>::value) {
            if (prec == kPrecF32Chains)
                return ti ? basis_impl<IO, float, M_, true>(e, A, PhiZ, g, st)
                          : basis_impl<IO, float, M_, false>(e, A, PhiZ, g, st);
        }
        return ti ? basis_impl<IO, double, M_, true>(e, A, PhiZ, g, st)
                  : basis_impl<IO, double, M_, false>(e, A, PhiZ, g, st);
    })
}

template <typename IO>
cudaError_t launch_carry_fwd(int Mp, const IO* PhiZ, const IO* zi, IO* Xin, const ScanArgs& g,
                             cudaStream_t st) {
    TVLP_DISPATCH_M(Mp, {
        k_carry_fwd<M_, double, IO><<<(unsigned)((g.B + 3) / 4), 128, 0, st>>>(PhiZ, zi, Xin, g);
        return cudaGetLastError();
    })
}

template <typename IO>
cudaError_t launch_carry_bwd(int Mp, const IO* PhiZ, const IO* Nu, IO* Mu, const ScanArgs& g,
                             cudaStream_t st) {
    TVLP_DISPATCH_M(Mp, {
        k_carry_bwd<M_, double, IO><<<(unsigned)((g.B + 3) / 4), 128, 0, st>>>(PhiZ, Nu, Mu, g);
        return cudaGetLastError();
    })
}

template <typename IO>
cudaError_t launch_apply_fwd(int Mp, bool ti, const IO* e, const IO* A, const IO* Xin, IO* s,
                             int* flag, const ScanArgs& g, cudaStream_t st) {
    TVLP_DISPATCH_M(Mp, {
        return ti ? apply_impl<IO, M_, true>(e, A, Xin, s, flag, g, st)
                  : apply_impl<IO, M_, false>(e, A, Xin, s, flag, g, st);
    })
}

template <typename IO>
cudaError_t launch_adjoint(int Mp, bool ti, int mode, const IO* gs, const IO* A, const IO* Mu,
                           IO* Nu, IO* ge, const ScanArgs& g, cudaStream_t st) {
    TVLP_DISPATCH_M(Mp, {
        if (mode == 0)
            return ti ? adjoint_impl<IO, M_, true, 0>(gs, A, Mu, Nu, ge, g, st)
                      : adjoint_impl<IO, M_, false, 0>(gs, A, Mu, Nu, ge, g, st);
        return ti ? adjoint_impl<IO, M_, true, 1>(gs, A, Mu, Nu, ge, g, st)
                  : adjoint_impl<IO, M_, false, 1>(gs, A, Mu, Nu, ge, g, st);
    })
}

template <typename IO>
cudaError_t launch_grad_A(int Mp, const IO* ge, const IO* s, const IO* zi, IO* gA, int64_t B,
                          int64_t T, cudaStream_t st) {
    dim3 grid((unsigned)((T + 255) / 256), (unsigned)B);
    TVLP_DISPATCH_M(Mp, {
        k_grad_A<IO, M_><<<grid, 256, 0, st>>>(ge, s, zi, gA, T);
        return cudaGetLastError();
    })
}

template <typename IO>
cudaError_t launch_grad_a(int M, const IO* ge, const IO* s, const IO* zi, IO* part, IO* ga,
                          int64_t B, int64_t T, int nchunk, cudaStream_t st) {
    dim3 grid((unsigned)nchunk, (unsigned)B);
    k_grad_a_partial<IO><<<grid, 256, 0, st>>>(ge, s, zi, part, T, M, nchunk);
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) return err;
    k_grad_a_final<IO><<<(unsigned)((B * M + 127) / 128), 128, 0, st>>>(part, ga, B, M, nchunk);
    return cudaGetLastError();
}

#define TVLP_INST(IO)                                                                            \
    template cudaError_t launch_basis<IO>(int, bool, int, const IO*, const IO*, IO*,             \
                                          const ScanArgs&, cudaStream_t);                        \
    template cudaError_t launch_carry_fwd<IO>(int, const IO*, const IO*, IO*, const ScanArgs&,   \
                                              cudaStream_t);                                     \
    template cudaError_t launch_carry_bwd<IO>(int, const IO*, const IO*, IO*, const ScanArgs&,   \
                                              cudaStream_t);                                     \
    template cudaError_t launch_apply_fwd<IO>(int, bool, const IO*, const IO*, const IO*, IO*,   \
                                              int*, const ScanArgs&, cudaStream_t);              \
    template cudaError_t launch_adjoint<IO>(int, bool, int, const IO*, const IO*, const IO*,     \
                                            IO*, IO*, const ScanArgs&, cudaStream_t);            \
    template cudaError_t launch_grad_A<IO>(int, const IO*, const IO*, const IO*, IO*, int64_t,   \
                                           int64_t, cudaStream_t);                               \
    template cudaError_t launch_grad_a<IO>(int, const IO*, const IO*, const IO*, IO*, IO*,       \
                                           int64_t, int64_t, int, cudaStream_t);
TVLP_INST(float)
TVLP_INST(double)

}  // namespace tvlp
