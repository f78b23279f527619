/*
 * tvlp.h -- C ABI of the B200-native differentiable linear-prediction kernels
 * (libtvlp_b200.so).  Plain pointers and sizes only; every pointer is a CUDA
 * device pointer unless stated otherwise; `stream` is a cudaStream_t (NULL =
 * legacy default stream).  All calls are asynchronous on `stream`, never
 * synchronise the host, and return a TVLP_* status (TVLP_ERR_CUDA carries a
 * launch error; see tvlp_last_cuda_error()).
 *
 * Each entry point replaces one function of the reference tvlp 0.1.0 LP path
 * (files under pkg/src/tvlp/ of arxiv/paper_2406_05128), with a leading batch
 * axis added (the reference is 1-D only):
 *
 *   tvlp_lp_forward_tv       lpc.py:101-117  lp_forward_tv(e, A, zi)   (+ _lp_kernel_tv lpc.py:36-47)
 *   tvlp_lp_backward_tv      lpc.py:152-173  lp_backward_tv(grad_s, A, s, zi)
 *   tvlp_lp_forward_ti       lpc.py:82-98    lp_forward_ti(e, a, zi)   (+ _lp_kernel_ti lpc.py:50-61)
 *   tvlp_lp_backward_ti      lpc.py:176-195  lp_backward_ti(grad_s, a, s, zi)
 *   tvlp_shift_coeffs        lpc.py:120-135  shift_coeffs(A)
 *   tvlp_lagged_signal_matrix lpc.py:138-149 lagged_signal_matrix(s, M, zi)
 *   tvlp_framewise_forward   params.py:220-239 _framewise_forward(e, frames, plan)
 *   tvlp_framewise_backward  params.py:259-273 _framewise_vjp(grad, e, frames, plan, segs)
 *
 * The tape-op contract of lpc.py:202-223 (forward saves the output s and A,
 * backward returns (grad_e, grad_A), no gradient for zi) is kept: the forward
 * may additionally emit the "carry tape" (the per-sub-chunk transition
 * matrices, in the I/O dtype) that the backward reuses instead of recomputing.
 *
 * Layouts (C-contiguous): e, s, grad_s, grad_e [B, T]; A, grad_A [B, T, M];
 * zi [B, M] (nullable = zeros); a, grad_a [B, M]; frames, grad_frames
 * [B, F, M]; window [frame_size] (the reference's float64 window cast to the
 * I/O dtype); seg [B, n_frames, frame_size] (frame-major, like the
 * reference's list of per-frame seg_outputs).  dtype: TVLP_F32 or TVLP_F64 for
 * every floating-point array of the call.
 */
#ifndef TVLP_B200_H
#define TVLP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TVLP_ABI_VERSION 1

#define TVLP_F32 0
#define TVLP_F64 1

#define TVLP_OK 0
#define TVLP_ERR_ARG 1       /* bad shape / null pointer / unsupported dtype */
#define TVLP_ERR_ORDER 2     /* M outside [1, tvlp_max_order()] */
#define TVLP_ERR_WORKSPACE 3 /* workspace smaller than tvlp_workspace_bytes() */
#define TVLP_ERR_CUDA 4      /* a CUDA launch failed */

/* precision of the sub-chunk transition matrices ("carries") */
#define TVLP_CARRY_F64 0 /* fp64 chains: matches the fp64 oracle to 1e-4 on resonant tracks */
#define TVLP_CARRY_F32 1 /* fp32 chains: faster, ~1e-3 relative on near-unit-circle poles */
#define TVLP_CARRY_AUTO 2 /* fp32 chains + boundary-defect check + device-side refinement of the
                             sequences whose carries fail it (fp32 I/O; fp64 I/O uses fp64) */
/* OR-ed into carry_prec of a forward: `carry` already holds the tape of a
 * forward over the same (e, A, B, T, M) -- the tape does not depend on zi --
 * so the transition pass is skipped and only the carry and apply passes run
 * (a new initial state, longseq.py). */
#define TVLP_CARRY_REUSE 16

/* workspace op codes */
#define TVLP_OP_FWD_TV 0
#define TVLP_OP_BWD_TV 1
#define TVLP_OP_FWD_TI 2
#define TVLP_OP_BWD_TI 3
#define TVLP_OP_FW_FWD 4
#define TVLP_OP_FW_BWD 5
#define TVLP_OP_FWD_TV_FRAMES 6
#define TVLP_OP_BWD_TV_FRAMES 7
#define TVLP_OP_BWD_TV_EX 8
#define TVLP_OP_SEGMENT_TRANSITION 9

int tvlp_abi_version(void);
const char* tvlp_status_string(int status);
int tvlp_last_cuda_error(void);
int32_t tvlp_max_order(void);

/* Number of elements (of the call dtype) of the carry tape for (B, T, M). */
int64_t tvlp_carry_elems(int64_t B, int64_t T, int32_t M);
/* Same for tvlp_lp_forward_tv_frames (its plan uses shorter sub-chunks). */
int64_t tvlp_carry_elems_frames(int64_t B, int64_t T, int32_t M);
/* Sub-chunk length used for (B, T, M) (diagnostics / tests; small batches use
 * shorter sub-chunks to fill the GPU). */
int64_t tvlp_subchunk_len(int64_t B, int64_t T, int32_t M);
/* Device workspace bytes needed by `op`; F/frame_size/hop only for frame-wise ops. */
size_t tvlp_workspace_bytes(int32_t op, int32_t dtype, int64_t B, int64_t T, int32_t M, int64_t F,
                            int32_t frame_size, int32_t hop);
/* Number of frames (lead-in included) of the frame-wise plan (params.py:203-217). */
int64_t tvlp_framewise_nframes(int64_t T, int64_t F, int32_t frame_size, int32_t hop);

/* s = LP_A(e).  carry (nullable): receives tvlp_carry_elems() values for the
 * backward.  nonfinite (nullable, device int32): OR-ed with 1 when e or A holds
 * a non-finite value (lpc.py:64-70, 111-112 reject those; the flag lets the
 * caller raise without a synchronising check inside the call). */
int tvlp_lp_forward_tv(int32_t dtype, const void* e, const void* A, const void* zi, void* s,
                       int64_t B, int64_t T, int32_t M, void* carry, int32_t carry_prec,
                       void* workspace, size_t workspace_bytes, int32_t* nonfinite, void* stream);

/* (grad_e, grad_A) of lp_forward_tv given the saved output s.  carry: the
 * tape written by the forward for the same (A, B, T, M), or NULL to recompute. */
int tvlp_lp_backward_tv(int32_t dtype, const void* grad_s, const void* A, const void* s,
                        const void* zi, void* grad_e, void* grad_A, int64_t B, int64_t T,
                        int32_t M, const void* carry, int32_t carry_prec, void* workspace,
                        size_t workspace_bytes, void* stream);

/* Frame-rate coefficients: the TV filter with
 * A = upsample_linear(frames, hop, T - 1) (params.py:107-132; the synthesiser's
 * call site synth.py:268-273) without materialising A: frames [B, F, M],
 * F = (T - 1) / hop + 1, rows interpolated inside the scan kernels (fp32; fp64
 * I/O or fp64 carries materialise A in the workspace).  Replaces the pair of
 * tape ops upsample_linear -> lp_tv (params.py:337-345, lpc.py:202-213). */
int tvlp_lp_forward_tv_frames(int32_t dtype, const void* e, const void* frames, const void* zi,
                              void* s, int64_t B, int64_t T, int32_t M, int64_t F, int32_t hop,
                              void* carry, int32_t carry_prec, void* workspace,
                              size_t workspace_bytes, int32_t* nonfinite, void* stream);
/* (grad_e, grad_frames) of lp_forward_tv_frames: the VJP chain lpc.py:152-173
 * then params.py:135-145, with grad_A never written (grad_frames [B, F, M]). */
int tvlp_lp_backward_tv_frames(int32_t dtype, const void* grad_s, const void* frames,
                               const void* s, const void* zi, void* grad_e, void* grad_frames,
                               int64_t B, int64_t T, int32_t M, int64_t F, int32_t hop,
                               const void* carry, int32_t carry_prec, void* workspace,
                               size_t workspace_bytes, void* stream);

/* Reflection rows -> direct-form rows by the step-up recursion (params.py:43-71,
 * reflection_to_lpc): k, a [rows, M]; float64
 * arithmetic in the reference's order (bit-identical in fp64).  bad (nullable,
 * device int32) is OR-ed with 1 when some |k| >= 1 (params.py:67-68 raise). */
int tvlp_reflection_to_lpc(int32_t dtype, const void* k, void* a, int64_t rows, int32_t M,
                           int32_t* bad, void* stream);
/* grad_k of reflection_to_lpc (params.py:74-84, _reflection_to_lpc_vjp). */
int tvlp_reflection_to_lpc_vjp(int32_t dtype, const void* grad_a, const void* k, void* grad_k,
                               int64_t rows, int32_t M, void* stream);

/* Time segments of one long sequence on several GPUs (the
 * exchange step; host side paper_2406_05128_b200/longseq.py):
 * tvlp_lp_backward_tv_ex = tvlp_lp_backward_tv with mu_in (nullable, [B, M]):
 * the adjoint of the state at the segment's end contributed by later segments,
 * and grad_zi (nullable, [B, M]): dL/dzi, the adjoint leaving through the
 * segment's initial state.  tvlp_segment_transition: Phi [B, M, M] (row-major)
 * = the product of all sub-chunk transitions of each sequence, from the carry
 * tape a tvlp_lp_forward_tv call filled; x_end = Phi zi + (zero-state end). */
int tvlp_lp_backward_tv_ex(int32_t dtype, const void* grad_s, const void* A, const void* s,
                           const void* zi, void* grad_e, void* grad_A, int64_t B, int64_t T,
                           int32_t M, const void* carry, int32_t carry_prec, const void* mu_in,
                           void* grad_zi, void* workspace, size_t workspace_bytes, void* stream);
int tvlp_segment_transition(int32_t dtype, const void* carry, int64_t B, int64_t T, int32_t M,
                            void* Phi, void* workspace, size_t workspace_bytes, void* stream);

/* Grouped launch (north star (3); SURVEY.md §8(b) "grouped variant"): n
 * independent batches with their OWN buffers and the same (T, M) -- the
 * GOLF HpN synthesiser's H(z) filter on the glottal source and its C(z) filter
 * on the noise (synth.py:264-273 records them as separate lp_tv tape ops) --
 * filtered by ONE launch sequence, without concatenating the inputs.  Each
 * group is exactly tvlp_lp_forward_tv / tvlp_lp_backward_tv on its own
 * arrays.  carry: tvlp_carry_elems(sum of B, T, M) values shared by the
 * groups (the backward reads the forward's).  Workspace:
 * tvlp_workspace_bytes_grouped().  n <= 4. */
typedef struct tvlp_lp_fwd_group {
    const void* e;  /* [B, T] */
    const void* A;  /* [B, T, M] */
    const void* zi; /* [B, M] or NULL */
    void* s;        /* [B, T] out */
    int64_t B;
} tvlp_lp_fwd_group;
typedef struct tvlp_lp_bwd_group {
    const void* grad_s; /* [B, T] */
    const void* A;      /* [B, T, M] */
    const void* s;      /* [B, T] the forward's output */
    const void* zi;     /* [B, M] or NULL */
    void* grad_e;       /* [B, T] out */
    void* grad_A;       /* [B, T, M] out */
    int64_t B;
} tvlp_lp_bwd_group;
#define TVLP_MAX_GROUPS 4
int tvlp_lp_forward_tv_grouped(int32_t dtype, int32_t n, const tvlp_lp_fwd_group* groups,
                               int64_t T, int32_t M, void* carry, int32_t carry_prec,
                               void* workspace, size_t workspace_bytes, int32_t* nonfinite,
                               void* stream);
int tvlp_lp_backward_tv_grouped(int32_t dtype, int32_t n, const tvlp_lp_bwd_group* groups,
                                int64_t T, int32_t M, const void* carry, int32_t carry_prec,
                                void* workspace, size_t workspace_bytes, void* stream);
/* op: TVLP_OP_FWD_TV or TVLP_OP_BWD_TV; B: the n batch sizes (host array). */
size_t tvlp_workspace_bytes_grouped(int32_t op, int32_t dtype, int32_t n, const int64_t* B,
                                    int64_t T, int32_t M);

/* Time-invariant special case: a [B, M] constant row per sequence. */
int tvlp_lp_forward_ti(int32_t dtype, const void* e, const void* a, const void* zi, void* s,
                       int64_t B, int64_t T, int32_t M, void* carry, int32_t carry_prec,
                       void* workspace, size_t workspace_bytes, int32_t* nonfinite, void* stream);
int tvlp_lp_backward_ti(int32_t dtype, const void* grad_s, const void* a, const void* s,
                        const void* zi, void* grad_e, void* grad_a, int64_t B, int64_t T,
                        int32_t M, const void* carry, int32_t carry_prec, void* workspace,
                        size_t workspace_bytes, void* stream);

int tvlp_shift_coeffs(int32_t dtype, const void* A, void* out, int64_t B, int64_t T, int32_t M,
                      void* stream);
int tvlp_lagged_signal_matrix(int32_t dtype, const void* s, const void* zi, void* out, int64_t B,
                              int64_t T, int32_t M, void* stream);

/* Frame-wise TI LP with overlap-add.  cola = window.sum()/hop (params.py:199-201).
 * seg [B, tvlp_framewise_nframes(), frame_size] receives the per-frame outputs
 * (the reference's seg_outputs), which the backward consumes.  frame_size must
 * be a multiple of 4 whose staged span fits shared memory (hop 240 / frame 960:
 * yes); other plans return TVLP_ERR_ARG. */
int tvlp_framewise_forward(int32_t dtype, const void* e, const void* frames, const void* window,
                           double cola, void* out, void* seg, int64_t B, int64_t T, int64_t F,
                           int32_t M, int32_t frame_size, int32_t hop, void* workspace,
                           size_t workspace_bytes, void* stream);
int tvlp_framewise_backward(int32_t dtype, const void* grad_out, const void* frames,
                            const void* window, double cola, const void* seg, void* grad_e,
                            void* grad_frames, int64_t B, int64_t T, int64_t F, int32_t M,
                            int32_t frame_size, int32_t hop, void* workspace,
                            size_t workspace_bytes, void* stream);
/* The same pair with an auxiliary buffer the forward fills and the backward
 * reads: [B, n_frames, 2 * padded M] values of the I/O dtype, each frame's
 * impulse-response tail (the frames-in-pieces kernels' carry needs it in both
 * directions; the backward then skips recomputing it).
 * tvlp_framewise_aux_elems() gives its size, 0 for plans that do not use it
 * (aux is then ignored).  aux NULL == the plain entry points. */
int64_t tvlp_framewise_aux_elems(int64_t B, int64_t T, int64_t F, int32_t M, int32_t frame_size,
                                 int32_t hop);
int tvlp_framewise_forward_ex(int32_t dtype, const void* e, const void* frames,
                              const void* window, double cola, void* out, void* seg, void* aux,
                              int64_t B, int64_t T, int64_t F, int32_t M, int32_t frame_size,
                              int32_t hop, void* workspace, size_t workspace_bytes, void* stream);
int tvlp_framewise_backward_ex(int32_t dtype, const void* grad_out, const void* frames,
                               const void* window, double cola, const void* seg, const void* aux,
                               void* grad_e, void* grad_frames, int64_t B, int64_t T, int64_t F,
                               int32_t M, int32_t frame_size, int32_t hop, void* workspace,
                               size_t workspace_bytes, void* stream);

/* The decoder pieces around the LP, float32.
 *
 * tvlp_wavetable_osc: the wavetable oscillator of source.py:224-318
 * (oscillator_phase -> upsample_linear(pos, hop*os) -> wavetable_read ->
 * decimate_fir) in one kernel; replaces the four taped ops of
 * source.py:294-318 (wavetable_osc).  f0_frames [B, F] float64 (validated by
 * the caller: 0 <= f0 < fs/2, source.py:230-233), pos_frames [B, F] table
 * positions (clipped to [0, K-1] inside), tables [K, L], taps [ntaps] (the
 * odd-length decimation lowpass, design_lowpass), sig [B, n_out];
 * F = (n_out*os - 1) / (hop*os) + 1; os = 4 (the reference default).
 * tvlp_wavetable_osc_vjp: grad_pos [B, F] from grad_sig [B, n_out] (f0 is not
 * differentiated, source.py:301-303); workspace: 2*B*F floats. */
int tvlp_wavetable_osc(const double* f0_frames, const float* pos_frames, const float* tables,
                       int32_t K, int32_t L, const float* taps, int32_t ntaps, float* sig,
                       int64_t B, int64_t n_out, int64_t F, int32_t hop, int32_t oversample,
                       double fs, void* stream);
int tvlp_wavetable_osc_vjp(const double* f0_frames, const float* pos_frames, const float* tables,
                           int32_t K, int32_t L, const float* taps, int32_t ntaps,
                           const float* grad_sig, float* grad_pos, float* workspace, int64_t B,
                           int64_t n_out, int64_t F, int32_t hop, int32_t oversample, double fs,
                           void* stream);
/* The per-item causal global FIR (source.py:445-466, _fw_global_fir /
 * _vjp_global_fir): y[b, n] = sum_{k<m} taps[b, k] x[b, n-k]; x, y [B, n],
 * taps [B, m], 1 <= m <= 1024.  The VJP writes grad_x [B, n] and/or
 * grad_taps [B, m] (either nullable); workspace: tvlp_global_fir_workspace
 * bytes (the per-tile tap partials, reduced in a fixed order). */
int tvlp_global_fir(const float* x, const float* taps, float* y, int64_t B, int64_t n, int32_t m,
                    void* stream);
size_t tvlp_global_fir_workspace(int64_t B, int64_t n, int32_t m);
int tvlp_global_fir_vjp(const float* grad_y, const float* x, const float* taps, float* grad_x,
                        float* grad_taps, void* workspace, size_t workspace_bytes, int64_t B,
                        int64_t n, int32_t m, void* stream);

/* shape_noise's framing and overlap-add (source.py:367-428) for hop-spaced
 * frames: frame i starts at sample start0 + i hop (samples outside [0, n)
 * read as 0 / are dropped).  tvlp_noise_frames: frames [B, nframes, nfft] =
 * noise [B, n] times window [size], zero-padded to nfft (the FFT input).
 * tvlp_frame_ola: out [B, n] = scale * sum over frames of y [B, nframes, ld]
 * read from column `delay` on (adjoint = 0), or its adjoint (adjoint = 1:
 * y is the output gradient [B, n], out the frame gradient [B, nframes, ld],
 * zero outside the read columns).  Fixed-order gathers, no atomics. */
int tvlp_noise_frames(const float* noise, const float* window, float* frames, int64_t B,
                      int64_t n, int64_t nframes, int32_t size, int32_t nfft, int64_t start0,
                      int32_t hop, void* stream);
int tvlp_frame_ola(const float* y, float* out, int64_t B, int64_t n, int64_t nframes, int32_t size,
                   int32_t ld, int32_t delay, int64_t start0, int32_t hop, float scale,
                   int32_t adjoint, void* stream);

/* The noise shaping's FFT-convolution product (source.py:404-412):
 * P[b][i] = S[b][i] * H[b][rows[i]] over K complex bins (interleaved float
 * pairs; S [B, nframes, K], H [B, F, K], rows [nframes] device int32,
 * nondecreasing), and its VJP to H: grad_H[b][f] = sum over the frames i
 * with rows[i] = f (i in [first[f], first[f+1]), first [F+1]) of
 * grad_P[b][i] * conj(S[b][i]), in frame order. */
int tvlp_spectra_mul(const float* S, const float* H, const int32_t* rows, float* P, int64_t B,
                     int64_t nframes, int64_t F, int32_t K, void* stream);
int tvlp_spectra_mul_vjp(const float* grad_P, const float* S, const int32_t* first, float* grad_H,
                         int64_t B, int64_t nframes, int64_t F, int32_t K, void* stream);

/* The HpN decoder's two LP inputs in one pass (synth.py:264-273 with the
 * paper's C(z) LP; decoder.Decoder.render): out [2B, Tp] = rows
 * h_gain(t) (sig(t) voiced_gain(t)) then noise(t) noise_gain(t), zero from T1
 * to Tp, the gains [B, F] upsampled at `hop` (params.py:107-132; F = (T1-1)/hop
 * + 1, T1 <= Tp <= F hop); sig, noise [B, T1].  The VJP writes grad_sig,
 * grad_noise [B, T1] and the three gain-frame gradients [B, F]; workspace:
 * 6 B F floats. */
int tvlp_source_pair(const float* sig, const float* noise, const float* voiced_gain,
                     const float* noise_gain, const float* h_gain, float* out, int64_t B,
                     int64_t T1, int64_t F, int32_t hop, int64_t Tp, void* stream);
int tvlp_source_pair_vjp(const float* grad_out, const float* sig, const float* noise,
                         const float* voiced_gain, const float* noise_gain, const float* h_gain,
                         float* grad_sig, float* grad_noise, float* grad_voiced_gain,
                         float* grad_noise_gain, float* grad_h_gain, float* workspace, int64_t B,
                         int64_t T1, int64_t F, int32_t hop, int64_t Tp, void* stream);

/* stft_mag's framing (loss.py:46-63): x [B, n] reflect-padded by N/2, frames
 * of N samples every `hop`, times window [N] -> frames [B, nframes, N]
 * (nframes = tvlp_stft_nframes(n, N, hop); 0 = invalid: n < N or
 * N/2 >= n); the VJP overlap-adds the windowed frame gradients back through
 * the pads (loss.py:81-86), each frame's value taken as scale * grad_frames +
 * dc_scale * dc[frame * dc_stride] (dc nullable: the one-sided spectrum's DC
 * correction when grad_frames is a plain inverse FFT of the spectrum's
 * gradient, odd N). */
int64_t tvlp_stft_nframes(int64_t n, int32_t N, int32_t hop);
int tvlp_stft_frames(const float* x, const float* window, float* frames, int64_t B, int64_t n,
                     int32_t N, int32_t hop, void* stream);
int tvlp_stft_frames_vjp(const float* grad_frames, const float* window, float* grad_x, int64_t B,
                         int64_t n, int32_t N, int32_t hop, float scale, const float* dc,
                         int64_t dc_stride, float dc_scale, void* stream);

/* One FFT size of the multi-resolution spectral loss (loss.py:105-126) from
 * one-sided spectra (the caller's FFTs): X (signal) and Y (target) complex
 * [B][n] as interleaved float pairs, n = frames x bins per item.
 * term[b] = ||(|X|-|Y|)|| / max(||Y||, 1e-12) + mean |log(|X|+eps) -
 * log(|Y|+eps)|; aux [B][4] keeps what the VJP needs; workspace:
 * tvlp_mss_terms_workspace bytes.  The VJP writes grad_X (complex [B][n])
 * from grad_term [B] (the stft_mag VJP's phase mask, loss.py:71-73). */
size_t tvlp_mss_terms_workspace(int64_t B, int64_t n);
int tvlp_mss_terms(const float* X, const float* Y, int64_t B, int64_t n, float eps, float* term,
                   float* aux, void* workspace, size_t workspace_bytes, void* stream);
int tvlp_mss_terms_vjp(const float* X, const float* Y, const float* aux, const float* grad_term,
                       float* grad_X, int64_t B, int64_t n, float eps, void* stream);

/* Instrumentation (bench.py): number of kernels this library has launched,
 * and optional CUDA-event timing of every launch (off by default; when on,
 * each launch is bracketed by two events on its stream).  tvlp_profile_dump
 * writes "name launches total_ms" lines (it synchronises on the recorded
 * events) and resets the table; returns the number of bytes written. */
int64_t tvlp_launch_count(void);
/* Sequences whose fp32 carries failed the boundary-defect check and were
 * refined (precision TVLP_CARRY_AUTO), cumulative; synchronises the device. */
int64_t tvlp_refined_sequences(void);
void tvlp_profile_enable(int32_t on);
/* Diagnostics: a device buffer (NULL = off) that the chained single-pass
 * kernels fill with one 64-byte timeline record per work item (globaltimer
 * ns; tools/chain_trace.py decodes it). */
void tvlp_chain_trace(void* buf, size_t bytes);
int32_t tvlp_profile_dump(char* buf, int32_t buflen);

#ifdef __cplusplus
}
#endif
#endif /* TVLP_B200_H */
