// scan_launch.cuh -- host launchers for the chunked-scan kernels (internal).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tvlp {

struct ScanArgs;

// Orders with compiled kernels; other orders are zero-padded up to the next
// one by the C ABI (exact: padded coefficients are 0).
constexpr int kNumOrders = 9;
constexpr int kOrders[kNumOrders] = {2, 4, 6, 8, 12, 16, 22, 24, 30};
inline int padded_order(int M) {
    for (int i = 0; i < kNumOrders; ++i)
        if (kOrders[i] >= M) return kOrders[i];
    return -1;
}

enum Prec : int { kPrecF64Chains = 0, kPrecF32Chains = 1 };

template <typename IO>
cudaError_t launch_basis(int Mp, bool ti, int prec, const IO* e, const IO* A, IO* PhiZ,
                         const ScanArgs& g, cudaStream_t st);
int tape_elems(int Mp);  // carry-tape elements per sub-chunk
template <typename CT>
struct CarryArgs;
// x(k+1) = Phi_k x(k) + z_k over segments (see CarryArgs in lp_scan.cuh)
template <typename IO>
cudaError_t launch_carry_fwd(int Mp, const CarryArgs<IO>& a, cudaStream_t st);
// mu(k-1) = Phi_k^T mu(k) + nu_k over segments
template <typename IO>
cudaError_t launch_carry_bwd(int Mp, const CarryArgs<IO>& a, cudaStream_t st);
// group products P_g of G consecutive tapes (hierarchical carry)
template <typename IO>
cudaError_t launch_group_P(int Mp, const IO* tape, IO* gtape, int64_t ngroups, int G, int nsub,
                           const int* only, cudaStream_t st);
template <typename IO>
cudaError_t launch_refine_helpers(int what, int Mp, const IO* P, const IO* Q, IO* D, int nsub,
                                  bool fwd, const int* only, int* flags, const unsigned* dstat,
                                  const int* inherit, float tol, int64_t B, cudaStream_t st);
unsigned long long refined_sequences();  // diagnostic counter (synchronising read)
enum Prec2 : int { kPrecAuto = 2 };
template <typename IO>
cudaError_t launch_apply_fwd(int Mp, bool ti, const IO* e, const IO* A, const IO* Xin, IO* s,
                             int* flag, IO* Xend, unsigned* dstat, const int* only,
                             const ScanArgs& g, cudaStream_t st);
template <typename IO>
cudaError_t launch_adjoint(int Mp, bool ti, int mode, const IO* gs, const IO* A, const IO* Mu,
                           IO* Nu, IO* ge, unsigned* dstat, const int* only, const ScanArgs& g,
                           cudaStream_t st);
template <typename IO>
cudaError_t launch_refine(int Mp, bool fwd, const IO* tape, IO* X, const IO* Xend,
                          const unsigned* dstat, int* flags, const int* fflags, const ScanArgs& g,
                          cudaStream_t st);
template <typename IO>
cudaError_t launch_grad_A(int Mp, const IO* ge, const IO* s, const IO* zi, IO* gA, int64_t B,
                          int64_t T, cudaStream_t st);
template <typename IO>
cudaError_t launch_grad_a(int M, const IO* ge, const IO* s, const IO* zi, IO* part, IO* ga,
                          int64_t B, int64_t T, int nchunk, cudaStream_t st);

}  // namespace tvlp
