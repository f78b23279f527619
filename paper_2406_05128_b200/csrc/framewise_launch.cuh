// framewise_launch.cuh -- host launchers for the frame-wise LP kernels (internal).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tvlp {

struct FwArgs {
    int64_t B, T;
    int F, nfr, size, hop, n_lead;
    double cola;
};

// frame sizes / orders / element sizes the kernels handle
bool fw_supported(int Mp, int size, int hop, int elem);
// seg: [B, nfr, size] saved frame outputs (frame-major); out: [B, T];
// aux (nullable): [B, nfr, 2 Mp] the frames' impulse-response tails, written
// by the forward's piece kernels and read by the backward's (fw_aux_elems)
template <typename IO>
cudaError_t launch_fw_forward(int Mp, const IO* e, const IO* frames, const IO* win, IO* seg,
                              IO* out, const FwArgs& a, cudaStream_t st, IO* aux = nullptr);
// gew: [B, nfr, size] scratch, gapart: [B, nfr, Mp] scratch; ge: [B, T]; gf: [B, F, Mp]
template <typename IO>
cudaError_t launch_fw_backward(int Mp, int M, const IO* gout, const IO* frames, const IO* win,
                               const IO* seg, IO* gew, IO* gapart, IO* ge, IO* gf,
                               const FwArgs& a, cudaStream_t st, const IO* aux = nullptr);
int64_t fw_aux_elems(const FwArgs& a, int Mp);

}  // namespace tvlp
