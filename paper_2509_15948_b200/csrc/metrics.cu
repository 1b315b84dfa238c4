// Post-hoc song metrics on device (mg/metrics.py:45-112): the per-segment MIR
// features of a rendered match against its target (RMS, crest factor, stereo
// width, stereo imbalance, Bark-band log spectrum) and the scale-invariant SDR.
//
// * k_seg_stats: per 8-second segment (the reference's split_segments), float64
//   block partials of sum(mid^2), max|mid|, sum(side^2), sum(l^2), sum(r^2) of
//   both signals, and the SI-SDR dot products s.s and s_hat.s over the whole
//   (2, L) signals; a one-CTA pass sums the partials in a fixed order.
// * SI-SDR's error energy sum((s_hat - a s)^2) is a second pass once a = (s_hat.s)/(s.s)
//   is known (the reference forms the error explicitly; so does this).
// * Bark spectrum: |rfft(mid)|^2 of a 240,000-sample segment (not a power of two)
//   by Bluestein's chirp-z on the library's power-of-two FFT (mgb_fft_c2c, 2^19
//   points): chirps computed in float64 from n^2 mod 2N, band energies summed in
//   float64, log10(energy + 1e-12) per Zwicker band.
#include "common.cuh"
#include "mgb_internal.h"

namespace {

constexpr int MT = 256;
constexpr int MBLK = 64;  // partial blocks per segment

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ double block_max(double v, double* scratch) {
  v = warp_max(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  double r = 0.0;
  if (wid == 0) {
    r = (lane < (int)((blockDim.x + 31) >> 5)) ? scratch[lane] : 0.0;
    r = warp_max(r);
  }
  return r;
}

// partials[m][blk][12]: per signal (y, yh): sum mid^2, max |mid|, sum side^2, sum l^2, sum r^2; then s.s, sh.s
__global__ void __launch_bounds__(MT) k_seg_stats(const float* __restrict__ y, const float* __restrict__ yh, int L,
                                                  int seg, double* __restrict__ part) {
  mgb_pdl_entry();
  __shared__ double red[32];
  const int m = blockIdx.y;
  const long long base = (long long)m * seg;
  double acc[12];
#pragma unroll
  for (int i = 0; i < 12; ++i) acc[i] = 0.0;
  for (int i = blockIdx.x * MT + threadIdx.x; i < seg; i += MBLK * MT) {
    const long long n = base + i;
    const double l = y[n], r = y[L + n], hl = yh[n], hr = yh[L + n];
    const double mid = l + r, side = l - r, hmid = hl + hr, hside = hl - hr;
    acc[0] += mid * mid;
    acc[1] = fmax(acc[1], fabs(mid));
    acc[2] += side * side;
    acc[3] += l * l;
    acc[4] += r * r;
    acc[5] += hmid * hmid;
    acc[6] = fmax(acc[6], fabs(hmid));
    acc[7] += hside * hside;
    acc[8] += hl * hl;
    acc[9] += hr * hr;
  }
  double* out = part + ((size_t)m * MBLK + blockIdx.x) * 12;
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    const double v = (i == 1 || i == 6) ? block_max(acc[i], red) : block_sum(acc[i], red);
    if (threadIdx.x == 0) out[i] = v;
    __syncthreads();
  }
}

// the SI-SDR dot products over all 2L samples (the reference ravels both channels)
__global__ void __launch_bounds__(MT) k_sisdr_dots(const float* __restrict__ y, const float* __restrict__ yh, long long n2,
                                                   const double* __restrict__ alpha, double* __restrict__ part) {
  mgb_pdl_entry();
  __shared__ double red[32];
  double a0 = 0.0, a1 = 0.0;
  const double al = alpha ? *alpha : 0.0;
  for (long long i = (long long)blockIdx.x * MT + threadIdx.x; i < n2; i += (long long)gridDim.x * MT) {
    const double s = y[i], sh = yh[i];
    if (alpha) {
      const double t = al * s, e = sh - t;
      a0 += t * t;
      a1 += e * e;
    } else {
      a0 += s * s;
      a1 += sh * s;
    }
  }
  a0 = block_sum(a0, red);
  __syncthreads();
  a1 = block_sum(a1, red);
  if (threadIdx.x == 0) {
    part[blockIdx.x * 2] = a0;
    part[blockIdx.x * 2 + 1] = a1;
  }
}

// fixed-order reduction of the per-block partials: out[m][10] (segment stats) or out[2] (dots)
__global__ void k_stats_final(const double* __restrict__ part, int nseg, double* __restrict__ out) {
  mgb_pdl_entry();
  const int m = blockIdx.x, i = threadIdx.x;
  if (i >= 10) return;
  double v = 0.0;
  for (int b = 0; b < MBLK; ++b) {
    const double p = part[((size_t)m * MBLK + b) * 12 + i];
    v = (i == 1 || i == 6) ? fmax(v, p) : v + p;
  }
  out[m * 10 + i] = v;
}

__global__ void k_dots_final(const double* __restrict__ part, int nblk, double* __restrict__ out, int set_alpha) {
  mgb_pdl_entry();
  if (threadIdx.x) return;
  double a0 = 0.0, a1 = 0.0;
  for (int b = 0; b < nblk; ++b) {
    a0 += part[b * 2];
    a1 += part[b * 2 + 1];
  }
  out[0] = a0;
  out[1] = a1;
  if (set_alpha) out[2] = a0 != 0.0 ? a1 / a0 : 0.0;  // alpha = (sh.s)/(s.s)
}

// Bluestein: w_n = exp(-i pi n^2 / N), phases from n^2 mod 2N in exact integer arithmetic
__device__ __forceinline__ float2 chirp(long long n, long long N, bool conj) {
  const long long q = (n * n) % (2 * N);
  double s, c;
  sincospi((double)q / (double)N, &s, &c);
  return make_float2((float)c, conj ? (float)s : (float)-s);
}

// a[m][n] = mid[n] * w_n (n < N), 0 up to M
__global__ void k_blue_a(const float* __restrict__ y, int L, int N, long long M, float2* __restrict__ a) {
  mgb_pdl_entry();
  const int m = blockIdx.y;
  float2* am = a + (size_t)m * M;
  const long long base = (long long)m * N;
  for (long long n = (long long)blockIdx.x * blockDim.x + threadIdx.x; n < M; n += (long long)gridDim.x * blockDim.x) {
    float2 v = make_float2(0.f, 0.f);
    if (n < N) {
      const float mid = y[base + n] + y[L + base + n];
      const float2 w = chirp(n, N, false);
      v = make_float2(mid * w.x, mid * w.y);
    }
    am[n] = v;
  }
}

// b[n] = conj(w_n) for n < N and b[M - n] = conj(w_n) for 0 < n < N (circular), else 0
__global__ void k_blue_b(int N, long long M, float2* __restrict__ b) {
  mgb_pdl_entry();
  for (long long n = (long long)blockIdx.x * blockDim.x + threadIdx.x; n < M; n += (long long)gridDim.x * blockDim.x) {
    long long k = -1;
    if (n < N) k = n;
    else if (n > M - N) k = M - n;
    b[n] = k >= 0 ? chirp(k, N, true) : make_float2(0.f, 0.f);
  }
}

__global__ void k_cmul_rows(float2* __restrict__ a, const float2* __restrict__ B, long long M) {
  mgb_pdl_entry();
  float2* am = a + (size_t)blockIdx.y * M;
  for (long long n = (long long)blockIdx.x * blockDim.x + threadIdx.x; n < M; n += (long long)gridDim.x * blockDim.x) {
    const float2 x = am[n], h = B[n];
    am[n] = make_float2(x.x * h.x - x.y * h.y, x.x * h.y + x.y * h.x);
  }
}

// X_k = w_k * conv_k (k <= N/2): band energies sum |X_k|^2 over the bins whose
// frequency k * sr / N lies in [edge_j, edge_j+1), float64; per-block partials
__global__ void __launch_bounds__(MT) k_blue_bands(const float2* __restrict__ conv, int N, long long M,
                                                   const double* __restrict__ edges, int nb, double sr,
                                                   double* __restrict__ part) {
  mgb_pdl_entry();
  __shared__ double red[32];
  __shared__ double ed[32];
  const int m = blockIdx.y;
  if (threadIdx.x <= nb) ed[threadIdx.x] = edges[threadIdx.x];
  __syncthreads();
  const float2* cm = conv + (size_t)m * M;
  const int nbins = N / 2 + 1;
  for (int j = 0; j < nb; ++j) {
    // bins of band j: k in [ceil(e_j N / sr), ceil(e_{j+1} N / sr))
    const long long k0 = (long long)ceil(ed[j] * N / sr), k1 = (long long)ceil(ed[j + 1] * N / sr);
    double s = 0.0;
    for (long long k = k0 + (long long)blockIdx.x * MT + threadIdx.x; k < k1 && k < nbins;
         k += (long long)gridDim.x * MT) {
      const float2 w = chirp(k, N, false), c = cm[k];
      const double xr = (double)w.x * c.x - (double)w.y * c.y, xi = (double)w.x * c.y + (double)w.y * c.x;
      s += xr * xr + xi * xi;
    }
    s = block_sum(s, red);
    if (threadIdx.x == 0) part[((size_t)m * nb + j) * gridDim.x + blockIdx.x] = s;
    __syncthreads();
  }
}

__global__ void k_bands_final(const double* __restrict__ part, int nb, int nblk, double scale,
                              double* __restrict__ out) {
  mgb_pdl_entry();
  const int m = blockIdx.x, j = threadIdx.x;
  if (j >= nb) return;
  double s = 0.0;
  for (int b = 0; b < nblk; ++b) s += part[((size_t)m * nb + j) * nblk + b];
  out[m * nb + j] = log10(s * scale + 1e-12);
}

}  // namespace

extern "C" size_t mgb_metrics_workspace(int L, int seg) {
  if (L <= 0 || seg <= 0) return 0;
  const int nseg = L / seg;
  const long long M = 1LL << mgb_log2_ceil(2LL * seg - 1);
  size_t b = 0;
  b += mgb_align(sizeof(double) * (size_t)(nseg > 0 ? nseg : 1) * MBLK * 12);  // segment partials
  b += mgb_align(sizeof(double) * 148 * 2 * 2);                                 // dot partials
  b += mgb_align(sizeof(float2) * (size_t)M * (nseg + 2));                      // Bluestein a rows, b, tmp
  b += mgb_align(sizeof(double) * (size_t)(nseg > 0 ? nseg : 1) * 32 * 64);     // band partials
  return b;
}

extern "C" int mgb_song_metrics(const float* y, const float* yh, int L, int seg, const double* bark_edges, int n_bands,
                                double sr, double* seg_stats, double* dots, double* bark_y, double* bark_yh, void* ws,
                                size_t ws_bytes, void* stream) {
  if (!y || !yh || L <= 0 || seg <= 0 || n_bands <= 0 || n_bands > 31) return 1;
  if (ws_bytes < mgb_metrics_workspace(L, seg)) return 1;
  cudaStream_t st = (cudaStream_t)stream;
  const int nseg = L / seg;
  const long long M = 1LL << mgb_log2_ceil(2LL * seg - 1);
  const int logM = mgb_log2_ceil(M);
  if (logM > 21) return 1;
  MgbArena a{(char*)ws, 0};
  double* spart = a.take<double>((size_t)(nseg > 0 ? nseg : 1) * MBLK * 12);
  double* dpart = a.take<double>(148 * 2 * 2);
  float2* rows = a.take<float2>((size_t)M * (nseg + 2));
  double* bpart = a.take<double>((size_t)(nseg > 0 ? nseg : 1) * 32 * 64);
  float2* bch = rows + (size_t)M * nseg;
  float2* tmp = bch + M;
  // SI-SDR over the whole signals: dots, alpha, then the explicit error energy
  const long long n2 = 2LL * L;
  mgb_launch(k_sisdr_dots, dim3(148), dim3(MT), 0, st, y, yh, n2, (const double*)nullptr, dpart);
  MGB_CHECK_LAUNCH();
  mgb_launch(k_dots_final, dim3(1), dim3(32), 0, st, (const double*)dpart, 148, dots, 1);
  MGB_CHECK_LAUNCH();
  mgb_launch(k_sisdr_dots, dim3(148), dim3(MT), 0, st, y, yh, n2, (const double*)(dots + 2), dpart);
  MGB_CHECK_LAUNCH();
  mgb_launch(k_dots_final, dim3(1), dim3(32), 0, st, (const double*)dpart, 148, dots + 3, 0);
  MGB_CHECK_LAUNCH();
  if (nseg < 1) return 0;  // shorter than one segment: the reference raises TooShort for the MIR features
  mgb_launch(k_seg_stats, dim3(MBLK, nseg), dim3(MT), 0, st, y, yh, L, seg, spart);
  MGB_CHECK_LAUNCH();
  mgb_launch(k_stats_final, dim3(nseg), dim3(32), 0, st, (const double*)spart, nseg, seg_stats);
  MGB_CHECK_LAUNCH();
  // Bluestein band spectra of both signals' mid channels
  mgb_launch(k_blue_b, dim3(592), dim3(256), 0, st, seg, M, bch);
  MGB_CHECK_LAUNCH();
  if (int rc = mgb_fft_c2c(bch, bch, tmp, 1, logM, 0, 1.f, st)) return rc;
  for (int which = 0; which < 2; ++which) {
    const float* x = which ? yh : y;
    double* out = which ? bark_yh : bark_y;
    mgb_launch(k_blue_a, dim3(592, nseg), dim3(256), 0, st, x, L, seg, M, rows);
    MGB_CHECK_LAUNCH();
    for (int m = 0; m < nseg; ++m)
      if (int rc = mgb_fft_c2c(rows + (size_t)m * M, rows + (size_t)m * M, tmp, 1, logM, 0, 1.f, st)) return rc;
    mgb_launch(k_cmul_rows, dim3(592, nseg), dim3(256), 0, st, rows, (const float2*)bch, M);
    MGB_CHECK_LAUNCH();
    for (int m = 0; m < nseg; ++m)
      if (int rc = mgb_fft_c2c(rows + (size_t)m * M, rows + (size_t)m * M, tmp, 1, logM, 1, 1.f / (float)M, st))
        return rc;
    mgb_launch(k_blue_bands, dim3(64, nseg), dim3(MT), 0, st, (const float2*)rows, seg, M, bark_edges, n_bands, sr,
               bpart);
    MGB_CHECK_LAUNCH();
    mgb_launch(k_bands_final, dim3(nseg), dim3(32), 0, st, (const double*)bpart, n_bands, 64, 1.0, out);
    MGB_CHECK_LAUNCH();
  }
  return 0;
}
