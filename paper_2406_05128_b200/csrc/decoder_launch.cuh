// decoder_launch.cuh -- launchers of decoder_kernels.cu (the oscillator and
// the global FIR around the LP; include/tvlp.h tvlp_wavetable_osc*,
// tvlp_global_fir*).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tvlp {

struct OscGeo {
    int64_t B, n_out, F, n_os;
    int hop, hop_os, K, L, nt, gd;
    double inv_rate;  // 1 / (fs * oversample)
    double inv_hop;   // 1 / hop_os
    float inv_hop_f;
};
cudaError_t launch_osc_fwd(const double* f0, const float* pos, const float* tab,
                           const float* taps, float* sig, const OscGeo& g, int os,
                           cudaStream_t st);
cudaError_t launch_osc_vjp(const double* f0, const float* pos, const float* tab,
                           const float* taps, const float* gsig, float* part, float* gpos,
                           const OscGeo& g, int os, cudaStream_t st);
cudaError_t launch_fir(const float* x, const float* taps, float* y, int64_t B, int64_t n, int m,
                       bool adj, int off, cudaStream_t st);
size_t fir_taps_part_elems(int64_t B, int64_t n, int m);
cudaError_t launch_fir_taps(const float* g, const float* x, float* part, float* gh, int64_t B,
                            int64_t n, int m, int off, cudaStream_t st);
int mss_chunks(int64_t n);
size_t mss_part_floats(int64_t B, int64_t n);
cudaError_t launch_mss_terms(const float* X, const float* Y, int64_t B, int64_t n, float eps,
                             float* term, float* aux, float* part, cudaStream_t st);
cudaError_t launch_mss_terms_vjp(const float* X, const float* Y, const float* aux,
                                 const float* gterm, int64_t B, int64_t n, float eps, float* gX,
                                 cudaStream_t st);
cudaError_t launch_stft_frames(const float* x, const float* win, float* fr, int64_t B, int64_t n,
                               int N, int hop, cudaStream_t st);
cudaError_t launch_stft_frames_vjp(const float* gfr, const float* win, float* gx, int64_t B,
                                   int64_t n, int N, int hop, float scale, const float* dc,
                                   int64_t dcs, float dc_scale, cudaStream_t st);
cudaError_t launch_noise_frames(const float* noise, const float* win, float* fr, int64_t B,
                                int64_t n, int64_t nfr, int size, int nfft, int64_t start0, int hop,
                                cudaStream_t st);
cudaError_t launch_frame_ola(const float* y, float* out, int64_t B, int64_t n, int64_t nfr,
                             int size, int ld, int delay, int64_t start0, int hop, float inv_cola,
                             bool adj, cudaStream_t st);
cudaError_t launch_spec_mul(const float* S, const float* H, const int* rows, const int* first,
                            float* out, int64_t B, int64_t nfr, int64_t F, int K, bool adj,
                            cudaStream_t st);
cudaError_t launch_source_pair(const float* sig, const float* noise, const float* vg,
                               const float* ng, const float* hg, float* out, int64_t B, int64_t T1,
                               int64_t F, int hop, int64_t Tp, cudaStream_t st);
cudaError_t launch_source_pair_vjp(const float* g, const float* sig, const float* noise,
                                   const float* vg, const float* ng, const float* hg, float* gsig,
                                   float* gnoise, float* gvg, float* gng, float* ghg, float* part,
                                   int64_t B, int64_t T1, int64_t F, int hop, int64_t Tp,
                                   cudaStream_t st);
}  // namespace tvlp
