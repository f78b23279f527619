// scan_launch.cuh -- host launchers for the chunked-scan kernels (internal).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tvlp {

struct ScanArgs;

// Frame-rate coefficient source (upsample_linear,
// params.py:107-132, fused into the scan kernels).  Row t of A is
// (1-w) F[f0] + w F[f1] with f0 = t/hop, w = (t - f0*hop)/hop, f1 = f0+1,
// held (w = 0) on the last anchor; rows at or past Tv (padding) are zero and
// columns at or past Mf (padded orders) are zero.
template <typename IO>
struct FrameSrc {
    const IO* frames;  // [B][nF][Mf]
    int64_t nF;        // frames per sequence: (T - 1) / hop + 1 (params.py:102-104)
    int64_t Tv;        // valid samples per sequence
    int hop;
    int Mf;
};

// Inputs of the refinement folded into the re-apply launch (precision "auto",
// single-level carries; see k_refine_fwd/bwd below for the recurrence).  With
// tape == nullptr the lane kernels run unchanged.
template <typename CT>
struct RefineSrc {
    const CT* tape = nullptr;        // carry tape (Phi_j rows/columns)
    const CT* K = nullptr;           // fwd: Xend (apply's end states); bwd: the carry-outs
    const unsigned* dstat = nullptr; // per-sequence defect statistics of the first pass
    int* flags = nullptr;            // fwd: forward refinement flags (set to 1 when refined)
    const int* inherit = nullptr;    // bwd: the forward's flags (refine those sequences too)
};

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
                         const ScanArgs& g, cudaStream_t st, const FrameSrc<IO>* fr = nullptr);
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
                             const ScanArgs& g, cudaStream_t st,
                             const FrameSrc<IO>* fr = nullptr,
                             const RefineSrc<IO>* rf = nullptr);
template <typename IO>
cudaError_t launch_adjoint(int Mp, bool ti, int mode, const IO* gs, const IO* A, const IO* Mu,
                           IO* Nu, IO* ge, unsigned* dstat, const int* only, const ScanArgs& g,
                           cudaStream_t st, const FrameSrc<IO>* fr = nullptr,
                           const RefineSrc<IO>* rf = nullptr);
// A[b, t, :] = the frame-rate rows upsampled (params.py:120-132), [B][T][Mp]
template <typename IO>
cudaError_t launch_upsample(int Mp, const FrameSrc<IO>& fr, IO* A, int64_t B, int64_t T,
                            cudaStream_t st);
// grad_frames[b, f, c] = sum_t dA[t, c]/dF[f, c] * (-grad_e(t) s(t-1-c))
// (params.py:135-145 composed with lpc.py:172), without materialising grad_A
template <typename IO>
cudaError_t launch_grad_frames(const FrameSrc<IO>& fr, const IO* ge, const IO* s, const IO* zi,
                               int Mzi, IO* gF, int64_t B, int64_t T, cudaStream_t st);
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
