/*
 * libmixgraph_b200 — C ABI of the B200 (sm_100a) console render + backward.
 *
 * The reference (arXiv 2509.15948, /root/reference/pkg) is pure Python; its
 * operator boundary is the Python call surface listed in SURVEY.md §8(b).
 * Each entry point below replaces one of those calls; the Python mirror in
 * paper_2509_15948_b200/ binds them with ctypes (INTEGRATION.md shows the
 * binding a reference maintainer would add).
 *
 * Conventions
 *  - every pointer is a DEVICE pointer unless stated; the caller allocates
 *    everything (outputs and workspaces); nothing allocates inside;
 *  - every call is asynchronous on the given cudaStream_t (passed as void*)
 *    and returns 0 on success, 1 = bad argument, 2 = launch failure;
 *  - signals are float32 stereo rows laid out (2, L) (left then right);
 *    parameter banks, dry/wet weights, gradient banks and all scalar
 *    reductions are float64;
 *  - tables are immutable per device after mgb_init(); kernels keep no other
 *    global state, so calls are reentrant per stream.
 */
#ifndef MIXGRAPH_B200_H
#define MIXGRAPH_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MGB_ABI_VERSION 4

/* One homogeneous schedule level (Algorithm 1 step) of B same-type nodes.
 * Replaces processors.KERNELS[tag](u, p) + drywet_wrap(ybar, u, w)
 * (mg/processors.py:61-73, :97-329) as called from execute_batched
 * (mg/scheduler.py:247-262), and their tape adjoints (mg/engine.py:100-112). */
typedef struct MgbLevel {
  char tag;                     /* 'g','s','e','r','c','n','d' */
  int B;                        /* nodes in the level */
  int L;                        /* samples per channel */
  const float* const* u_rows;   /* [B] ptrs to (2,L) inputs (gathered + fan-in summed) */
  const float* const* gy_rows;  /* [B] ptrs to (2,L) dLoss/dy (backward only) */
  const double* bank;           /* (N_t, P_t) parameter bank of this type */
  const int* prow;              /* [B] bank row per level row (plan.pslice / type_perm) */
  const int* widx;              /* [B] processor index per level row (plan.weight_idx) */
  const double* w;              /* [P] effective dry/wet weights sigma(raw)*mask; NULL => wet only */
  const double* greg;           /* scalar dLoss/d(reg) (backward); NULL => 0 */
  float* y;                     /* (B,2,L) output after dry/wet */
  float* ybar;                  /* (B,2,L) wet output (required for e,r,d) */
  float* aux;                   /* c,n: (B,L) envelope store; otherwise unused */
  double* reg;                  /* [B] gain-staging term per row (e,r,d); may be NULL */
  float* gu;                    /* (B,2,L) dLoss/du (backward); NULL = not requested (a level
                                   reading only the stems): the input-gradient work is skipped */
  double* gbank;                /* (N_t,P_t) gradient bank; rows prow[] are written */
  double* gw;                   /* [P] dLoss/dw; entries widx[] are written */
  void* ws;                     /* per-level workspace, persistent between fwd and bwd */
  size_t ws_bytes;
} MgbLevel;

/* Initialise per-device tables (twiddles, reverb noise spectra, windows).
 * reverb_spec: host pointer to 2 x 313 x 193 complex128 (mid, side) noise STFTs
 * and reverb_wss: host pointer to 60000 float64 OLA normaliser, both computed on
 * the host by the reference's table recipe (mg/processors.py:127-145).
 * Call once per device before any other call (not during stream capture). */
int mgb_init(const double* reverb_spec_host, const double* reverb_wss_host, void* stream);

/* Bytes of workspace one level of (tag, B, L) needs for mgb_level_forward/backward. */
size_t mgb_level_workspace(char tag, int B, int L);

/* Forward of one level: y = drywet(KERNELS[tag](u, bank[prow]), u, w[widx]);
 * also writes ybar / aux / reg as the tag requires. */
int mgb_level_forward(const MgbLevel* level, void* stream);

/* Backward of one level: consumes gy_rows (and greg), writes gu (unless NULL),
 * gbank rows, gw entries.  Must follow mgb_level_forward on the same workspace. */
int mgb_level_backward(const MgbLevel* level, void* stream);

/* The same two calls split in phases so a caller can overlap the
 * parameter-only work with other levels on a second stream:
 *   forward  phase 1: FIR synthesis and FIR spectra (e, r, d), ballistics
 *                     parameter blocks (c, n); depends on bank/prow only;
 *                     no-op for g, s;
 *            phase 2: the signal pass: y and ybar;
 *            phase 3: the gain-staging norms and term (reg) of e, r, d, read by
 *                     the backward and by the caller's reg (no-op otherwise;
 *                     a forward-only caller that ignores reg may skip it).
 *   backward phase 1: the signal adjoint gu, plus the per-CTA parameter
 *                     partials and (e, r, d) the FIR-gradient spectra, kept in the
 *                     workspace;
 *            phase 2: everything written to gbank and gw: the per-node
 *                     reductions of those partials and the FIR adjoint (e, r, d).
 *                     Nothing downstream of the level's gu needs it.
 * mgb_level_forward == phases 1, 2, 3 on one stream; mgb_level_backward == 1, 2.
 * Within one level the phases must be ordered (1 before 2, forward before
 * backward); phase 2 of the backward may run concurrently with other levels. */
int mgb_level_forward_phase(const MgbLevel* level, int phase, void* stream);
int mgb_level_backward_phase(const MgbLevel* level, int phase, void* stream);

/* Number of kernel launches this library has enqueued so far (host counter,
 * atomic across host threads; a launch captured into a CUDA graph counts once,
 * at capture). */
long long mgb_launch_count(void);

/* Profiling: *dst = the GPU's global nanosecond timer when the stream reaches this point
 * (a one-thread kernel; usable inside a captured CUDA graph, where timing events are not). */
int mgb_timestamp(unsigned long long* dst, void* stream);

/* cudaMemsetAsync(ptr, 0, bytes) on the stream (not a kernel; e.g. the warm-up part of dL/dy). */
int mgb_zero(void* ptr, size_t bytes, void* stream);

/* A new non-blocking CUDA stream on the current device, owned by the caller
 * (NULL on failure); mgb_stream_destroy releases it.  Concurrent song searches
 * give every host thread its own streams (torch hands out pooled streams, which
 * two threads could share while one of them is capturing a CUDA graph). */
void* mgb_stream_create(void);
int mgb_stream_destroy(void* stream);
/* The same with a priority: level > 0 the device's greatest, < 0 the least, 0 default
 * (a step's critical-path stream high, its side streams low; graph captures keep it). */
void* mgb_stream_create_priority(int level);

/* Effective dry/wet weights w = sigmoid(raw) * mask (mg/scheduler.py:218-222).
 * mask may be NULL. */
int mgb_weights(const double* raw, const double* mask, double* w, int P, void* stream);

/* Fan-in aggregation for mix/output nodes (mg/engine.py:439-450 segment_sum):
 * out[s] = sum_{i in [seg_off[s], seg_off[s+1])} in_rows[i], each row (2,L). */
int mgb_bus_sum(const float* const* in_rows, const int* seg_off, float* out, int S, int L, void* stream);

/* Segment gather for a training step (mg/optimizer.py:97-105 sample_segment):
 * dst[r][0:len] = src[r][song_off[row_song[r]] : + len] for r < rows; src, dst
 * and row_song are device arrays of rows entries, song_off a device array of
 * per-song sample offsets (rewritten between steps; a captured step replays with
 * the new values).  Used by the batched multi-song trainer. */
int mgb_gather_rows(const float* const* src, float* const* dst, const int* row_song, const long long* song_off,
                    int rows, int len, void* stream);

/* Batched complex FFT, natural order, unnormalised except for `scale`.
 * in/out: batch x 2^log2n complex64; tmp: batch x 2^log2n (only for log2n > 13). */
int mgb_fft(const void* in, void* out, void* tmp, int batch, int log2n, int inverse, float scale, void* stream);

/* ---- multi-resolution STFT loss (mg/losses.py:104-170) ---------------- */

/* One resolution's constant tables, built on the host from the reference's
 * mel_filterbank / a_weight_gains recipe (mg/losses.py:51-101). */
typedef struct MgbLossRes {
  int n_fft;                    /* power of two, 256..8192 */
  int hop;                      /* n_fft / 4 */
  int frames;                   /* 1 + Ls / hop */
  int n_mels;
  const int* band_start;        /* [n_mels] first bin of band j */
  const int* band_len;          /* [n_mels] bins in band j */
  const int* band_off;          /* [n_mels] offset of band j's weights in band_w */
  const double* band_w;         /* concatenated band weights (A-weight x mel) */
  const int* bin_start;         /* [n_bins] offset into bin_band/bin_w */
  const int* bin_len;           /* [n_bins] */
  const int* bin_band;          /* transposed (CSC) band indices */
  const double* bin_w;          /* transposed weights */
  double* tmel;                 /* (frames, n_mels, 4 groups) target mel */
  double* tlog;                 /* (frames, n_mels, 4) log(target mel + 1e-7) */
  double* mel;                  /* (frames, n_mels, 4) estimate mel (fwd -> bwd) */
  double* part;                 /* (frames, 4, 3) per-frame partial sums */
  float* gframes;               /* (frames, 2, n_fft): the forward's frame spectra, then the backward's
                                   frame adjoints; NULL for a forward-only loss */
} MgbLossRes;

typedef struct MgbLoss {
  int n_res;
  MgbLossRes res[8];
  int Ls;                       /* scored length */
  double group_w[4];            /* [lr/2, lr/2, mid, side] */
  double* stats;                /* [batch][n_res*4*4] fp64: tnorm, slog, sdiff2, sc (per res, group) */
  double* loss;                 /* device [batch]: L_a per signal */
  int batch;                    /* signals per call (0 or 1: one); the per-signal buffers of every
                                   resolution (tmel, tlog, mel, part, gframes) hold batch copies,
                                   signal-major */
  long long sig_stride;         /* floats from one signal's left channel to the next signal's (input,
                                   target and gradient pointers alike; batch > 1 only) */
} MgbLoss;

/* Target spectra for a (2, Ls) target whose channels start at tgt_l / tgt_r
 * (prepare_target, mg/losses.py:130-140).  With batch > 1 the three calls below
 * process batch independent signals (songs) at once: signal q's pointers are the
 * given ones plus q * sig_stride. */
int mgb_mrstft_target(const MgbLoss* loss, const float* tgt_l, const float* tgt_r, void* stream);
/* L_a for the (2, Ls) estimate; writes *loss->loss (mg/losses.py:143-170). */
int mgb_mrstft_forward(const MgbLoss* loss, const float* y_l, const float* y_r, void* stream);
/* dL_a/dy into g_l, g_r (Ls each, overwritten).  Must follow mgb_mrstft_forward on the
 * same estimate: the forward leaves each frame's spectrum in gframes (when gframes is
 * set) and its mel / stats, the backward reads them and overwrites gframes with the
 * frame adjoints. */
int mgb_mrstft_backward(const MgbLoss* loss, const float* y_l, const float* y_r, float* g_l, float* g_r,
                        void* stream);

/* ---- optimiser (mg/optimizer.py:82-137) --------------------------------- */

/* step_scalars (device, float64[8]): [lr, b1, b2, eps, wd, c1, c2, alpha_p].
 * One fused AdamW over the flat parameter vector p (n values, banks then raw
 * weights); before it, the delay rule (mg/optimizer.py:108-124) rewrites the
 * d-bank z gradients (rows of 880 at [d_off, d_off + 880*d_rows)); after it,
 * the unit-disk projection (mg/optimizer.py:127-137).  The raw-weight
 * gradient is assembled from dL/dw: g_raw = gw * mask * s(1-s) + alpha_p s(1-s)
 * over [w_off, w_off + P).  If loss_guard (device scalar, this step's total
 * loss) is non-finite the parameters and moments are left untouched
 * (NonFiniteLoss, mg/optimizer.py:164-171).  halt (device scalar, may be NULL)
 * makes that sticky for a run of steps: a non-finite loss_guard sets *halt = 1,
 * and while *halt != 0 no step updates anything (the reference stops the run at
 * the first non-finite loss, mg/optimizer.py:170-171, 208-215).  The caller
 * zeroes *halt when a run starts. */
int mgb_adamw_step(double* p, double* g, double* m, double* v, long long n, long long d_off, int d_rows,
                   long long w_off, int P, const double* gw, const double* mask, const double* step_scalars,
                   const double* loss_guard, double* halt, void* stream);

/* ---- post-hoc song metrics (mg/metrics.py:45-112, mg/cli.py:55-63) --------- */

/* Workspace bytes of mgb_song_metrics for (L, seg). */
size_t mgb_metrics_workspace(int L, int seg);

/* Metrics of a rendered match yh against its target y, both (2, L) float32:
 *  seg_stats [L/seg][10] float64: per seg-sample segment (split_segments), for y
 *            then yh: sum mid^2, max|mid|, sum side^2, sum l^2, sum r^2;
 *  dots      [5] float64: s.s, s_hat.s, alpha = (s_hat.s)/(s.s), sum (alpha s)^2,
 *            sum (s_hat - alpha s)^2 over the 2L samples (si_sdr);
 *  bark_y, bark_yh [L/seg][n_bands] float64: log10(sum of |rfft(mid)|^2 over the
 *            bins of Zwicker band j + 1e-12), bark_edges (device, n_bands + 1 Hz)
 *            at sample rate sr (feature_bark_spectrum; the non-power-of-two rfft by
 *            Bluestein on the float32 FFT).
 * Segments require L >= seg; with L < seg only dots is written. */
int mgb_song_metrics(const float* y, const float* yh, int L, int seg, const double* bark_edges, int n_bands,
                     double sr, double* seg_stats, double* dots, double* bark_y, double* bark_yh, void* ws,
                     size_t ws_bytes, void* stream);

/* Loss assembly of n signals (songs) (mg/optimizer.py:156-162):
 * vals[q] = [L_a + gain_w * L_g + (alpha_p > 0 ? alpha_p * L_p : 0), L_a, L_g, L_p] with
 * L_a = la[q], L_g = sum of reg[reg_idx[i]] for i in [reg_off[q], reg_off[q+1]) (reg_idx NULL:
 * reg[i]; reg_off NULL: 0), L_p = sparsity[q], alpha_p = step_scalars[7]; guard (may be NULL)
 * = sum of the totals (the mgb_adamw_step loss guard).  n <= 1024. */
int mgb_loss_assembly(const double* la, const double* reg, const int* reg_off, const int* reg_idx,
                      const double* sparsity, const double* step_scalars, double gain_w, int n, double* vals,
                      double* guard, void* stream);

/* sum over the P effective weights' sigmoid (sparsity term, mg/losses.py:181-183) */
int mgb_sparsity(const double* raw, int P, double* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif
