// chain_launch.cuh -- host interface of the chained single-pass scans
// (chain.cuh; internal to the library).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace tvlp {

struct ScanArgs;

// Units of consecutive sub-chunks: the lane-pass work item of one warp.
struct UnitGeo {
    int U;    // sub-chunks per unit (lanes)
    int nu;   // units per sequence
    int rem;  // sub-chunks of the last unit (1..U)
    __host__ __device__ int len(int r) const { return r == nu - 1 ? rem : U; }
};

struct ChainFwdCall {
    bool ti;           // time-invariant: A is one row [B][Mp] per sequence
    const float* e;
    const float* A;
    const float* zi;   // nullable, [B][zs] with zs >= Mp (padded components zero)
    int zs;
    float* s;
    float* tape;       // carry tape
    int* fflags;       // per-sequence refinement flags (in the carry tape)
    float* Xin;
    float* Xend;
    int* nonfinite;
    void* ctl;         // chain_ctl_bytes() of workspace (zeroed by the launcher)
    int refine;
    const ScanArgs& g;
};

struct ChainBwdCall {
    bool ti;
    const float* gs;
    const float* A;
    float* ge;
    const float* tape;
    const int* inherit;  // nullable
    float* Nu;           // zero-state adjoints (written by the launch when the chained
                         // kernel does not run that pass itself)
    float* Mu;
    float* Kout;
    void* ctl;
    int refine;
    const ScanArgs& g;
};

UnitGeo chain_units(int nsub, bool fwd);
bool chain_supported(int Mp);
size_t chain_ctl_bytes(int64_t B, int nsub, int Mp);
cudaError_t launch_fwd_chain(int Mp, const ChainFwdCall& c, cudaStream_t st);
cudaError_t launch_bwd_chain(int Mp, const ChainBwdCall& c, cudaStream_t st);
unsigned long long chain_refined_sequences();
void chain_set_trace(void* buf, size_t bytes);  // diagnostics (tools/chain_trace.py)

}  // namespace tvlp
