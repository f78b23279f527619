// chain_launch.cuh -- host interface of the chained single-pass scans
// (chain.cuh; internal to the library).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "scan_launch.cuh"

namespace tvlp {

struct ScanArgs;

// Units of consecutive sub-chunks: the lane-pass work item of one warp.
struct UnitGeo {
    int U;    // sub-chunks per unit (lanes)
    int nu;   // units per sequence
    int rem;  // sub-chunks of the last unit (1..U)
    __host__ __device__ int len(int r) const { return r == nu - 1 ? rem : U; }
};

// Grouped launches: up to kMaxGroups batches with their own buffers and the
// same (T, M) in one launch (the HpN synthesiser's H(z) and C(z) filters).
constexpr int kMaxGroups = 4;
struct ChainGroup {
    const float* x;    // fwd: e [B,T]; bwd: grad_s [B,T]
    const float* A;    // [B,T,Mp] (TI: [B,Mp])
    const float* zi;   // fwd, nullable: [B][zs] (padded components zero)
    float* y;          // fwd: s [B,T]; bwd: grad_e [B,T]
    int64_t B;
};

struct ChainFwdCall {
    bool ti;           // time-invariant: A is one row [B][Mp] per sequence
    int ng;            // groups (1 for the plain batched call)
    ChainGroup grp[kMaxGroups];
    int zs;
    float* tape;       // carry tape of all groups' sequences (group after group)
    int* fflags;       // per-sequence refinement flags (in the carry tape)
    float* Xin;
    float* Xend;
    int* nonfinite;
    void* ctl;         // chain_ctl_bytes() of workspace (zeroed by the launcher)
    int refine;
    const ScanArgs& g; // g.B: the total over the groups
    const FrameSrc<float>* fr = nullptr;  // frame-rate rows interpolated in the kernels
};

struct ChainBwdCall {
    bool ti;
    int ng;
    ChainGroup grp[kMaxGroups];
    const float* tape;
    const int* inherit;  // nullable
    float* Nu;           // zero-state adjoints (written by the launch when the chained
                         // kernel does not run that pass itself)
    float* Mu;
    float* Kout;
    void* ctl;
    int refine;
    const ScanArgs& g;
    const FrameSrc<float>* fr = nullptr;  // frame-rate rows interpolated in the kernels
};

UnitGeo chain_units(int nsub, bool fwd);
bool chain_supported(int Mp);
size_t chain_ctl_bytes(int64_t B, int nsub, int Mp);
// phase 0: zero the control words and run the streaming pass the chained
// kernel consumes (fwd: k_basis4 tapes; bwd: k_adjoint<MODE 0> nu);
// phase 1: the chained kernel.  Stream-ordered: call 0 then 1.
cudaError_t launch_fwd_chain(int Mp, const ChainFwdCall& c, cudaStream_t st, int phase);
cudaError_t launch_bwd_chain(int Mp, const ChainBwdCall& c, cudaStream_t st, int phase);
unsigned long long chain_refined_sequences();
void chain_set_trace(void* buf, size_t bytes);  // diagnostics (tools/chain_trace.py)

}  // namespace tvlp
