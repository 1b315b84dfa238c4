// Multi-resolution STFT loss (mg/losses.py:104-170), forward and backward.
//
// Per resolution n (hop n/4, reflect pad n/2, periodic Hann), one CTA per
// frame: both output channels ride one complex float64 FFT (left + i*right)
// in shared memory; the four groups [L, R, L+R, L-R] are separated from the
// spectrum by linearity; |X| x (A-weight * HTK mel) is applied as a banded
// (CSR) product; log-mel L1 and spectral-convergence partial sums are reduced
// per frame (float64) and combined by a one-CTA finalize.
// Backward recomputes the frame spectrum, forms dmel, d|X| (CSC), dX, packs
// the two channels' Hermitian adjoint spectra into one inverse FFT, and
// writes per-frame adjoints; a gather kernel overlap-adds them (with the
// reflect-pad adjoint) across all resolutions into dL/dy, without atomics.
// float64 is used throughout because the 1e-5 loss gate is tighter than an
// fp32 STFT of quiet mel bands allows; the loss is a small share of the step.
#include "common.cuh"
#include "mgb_internal.h"

namespace {

constexpr double LOG_EPS = 1e-7;

__device__ __forceinline__ long long reflect_idx(long long i, long long n) {
  if (n == 1) return 0;
  const long long period = 2 * (n - 1);
  long long a = i < 0 ? -i : i;
  a %= period;
  return a >= n ? period - a : a;
}

template <int N>
struct LossCfg {
  static constexpr int NT = N >= 4096 ? 512 : 256;
  static constexpr int NB = N / 2 + 1;
  static constexpr size_t SMEM = sizeof(double2) * padded_len<N>() + 64;  // padded FFT buffer
};

// load windowed frame f of (xl, xr) into s (complex double) and FFT it
template <int N>
__device__ __forceinline__ void load_fft(double2* s, const float* __restrict__ xl, const float* __restrict__ xr,
                                         int Ls, int hop, int f) {
  constexpr int NT = LossCfg<N>::NT;
  for (int t = threadIdx.x; t < N; t += NT) {
    const long long idx = reflect_idx((long long)f * hop + t - N / 2, Ls);
    const double win = 0.5 - 0.5 * cospi(2.0 * t / (double)N);
    s[pidx<true>(t)] = make_double2((double)xl[idx] * win, (double)xr[idx] * win);
  }
  smem_fft<double, N, 1, NT, N, 1, false, true>(s, false);
}

// per-bin group spectra from the packed spectrum
__device__ __forceinline__ void groups_at(const double2* s, int n, int k, double2 X[4]) {
  const double2 zk = s[pidx<true>(k)], zp = s[pidx<true>((n - k) & (n - 1))];
  const double2 a = make_double2(0.5 * (zk.x + zp.x), 0.5 * (zk.y - zp.y));
  const double2 d = make_double2(0.5 * (zk.x - zp.x), 0.5 * (zk.y + zp.y));
  const double2 b = make_double2(d.y, -d.x);
  X[0] = a;
  X[1] = b;
  X[2] = make_double2(a.x + b.x, a.y + b.y);
  X[3] = make_double2(a.x - b.x, a.y - b.y);
}

// Replace the spectrum in s by the 4 group magnitudes mag[g*NB + k] (double view).
template <int N>
__device__ __forceinline__ void spectrum_to_mags(double2* s) {
  constexpr int NT = LossCfg<N>::NT, NB = LossCfg<N>::NB;
  constexpr int PER = (NB + NT - 1) / NT;
  double m[PER][4];
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int k = threadIdx.x + i * NT;
    if (k < NB) {
      double2 X[4];
      groups_at(s, N, k, X);
#pragma unroll
      for (int g = 0; g < 4; ++g) m[i][g] = sqrt(X[g].x * X[g].x + X[g].y * X[g].y);
    }
  }
  __syncthreads();
  double* md = reinterpret_cast<double*>(s);
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int k = threadIdx.x + i * NT;
    if (k < NB) {
#pragma unroll
      for (int g = 0; g < 4; ++g) md[g * NB + k] = m[i][g];
    }
  }
  __syncthreads();
}

// mode 0: target (write tmel, tlog, part[.,g,0] = sum mel^2)
// mode 1: estimate (write mel, part[.,g,0] = sum |dlog|, part[.,g,1] = sum (mel - tmel)^2)
template <int N>
__global__ void __launch_bounds__(LossCfg<N>::NT) k_mr_fwd(MgbLossRes r, const float* __restrict__ xl,
                                                           const float* __restrict__ xr, int Ls, int mode) {
  constexpr int NT = LossCfg<N>::NT, NB = LossCfg<N>::NB;
  extern __shared__ __align__(16) unsigned char smraw[];
  double2* s = reinterpret_cast<double2*>(smraw);
  __shared__ double red[32];
  __shared__ double acc[4][2];
  const int f = blockIdx.x;
  load_fft<N>(s, xl, xr, Ls, r.hop, f);
  spectrum_to_mags<N>(s);
  const double* md = reinterpret_cast<const double*>(s);
  if (threadIdx.x < 8) (&acc[0][0])[threadIdx.x] = 0.0;
  __syncthreads();
  const int nm = r.n_mels;
  double a0[4] = {0, 0, 0, 0}, a1[4] = {0, 0, 0, 0};
  for (int q = threadIdx.x; q < 4 * nm; q += NT) {
    const int g = q / nm, j = q % nm;
    const int k0 = r.band_start[j], len = r.band_len[j], off = r.band_off[j];
    double mel = 0.0;
    for (int i = 0; i < len; ++i) mel = fma(md[g * NB + k0 + i], r.band_w[off + i], mel);
    const size_t o = ((size_t)g * r.frames + f) * nm + j;
    if (mode == 0) {
      r.tmel[o] = mel;
      r.tlog[o] = log(mel + LOG_EPS);
      a0[g] += mel * mel;
    } else {
      r.mel[o] = mel;
      const double dlog = log(mel + LOG_EPS) - r.tlog[o];
      const double dm = mel - r.tmel[o];
      a0[g] += fabs(dlog);
      a1[g] += dm * dm;
    }
  }
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    const double t0 = block_sum(a0[g], red);
    __syncthreads();
    const double t1 = block_sum(a1[g], red);
    __syncthreads();
    if (threadIdx.x == 0) {
      r.part[((size_t)f * 4 + g) * 3 + 0] = t0;
      r.part[((size_t)f * 4 + g) * 3 + 1] = t1;
    }
  }
}

// stats layout per (res, group): [tnorm, slog, sdiff2, dn]
// one CTA per (resolution, group)
__global__ void k_mr_finalize(MgbLoss L, int mode) {
  __shared__ double red[32];
  const int ri = blockIdx.x >> 2, g = blockIdx.x & 3;
  const MgbLossRes& r = L.res[ri];
  double s0 = 0.0, s1 = 0.0;
  for (int f = threadIdx.x; f < r.frames; f += blockDim.x) {
    s0 += r.part[((size_t)f * 4 + g) * 3 + 0];
    s1 += r.part[((size_t)f * 4 + g) * 3 + 1];
  }
  s0 = block_sum(s0, red);
  __syncthreads();
  s1 = block_sum(s1, red);
  if (threadIdx.x == 0) {
    double* st = L.stats + ((size_t)ri * 4 + g) * 4;
    if (mode == 0) {
      st[0] = fmax(sqrt(s0), 1e-12);
    } else {
      st[1] = s0;
      st[2] = s1;
      st[3] = sqrt(s1);
    }
  }
}

// L_a = sum over (res, group) of w_g (slog / frames + dn / tnorm), in a fixed order
__global__ void k_mr_total(MgbLoss L) {
  if (threadIdx.x) return;
  double tot = 0.0;
  for (int ri = 0; ri < L.n_res; ++ri)
    for (int g = 0; g < 4; ++g) {
      const double* st = L.stats + ((size_t)ri * 4 + g) * 4;
      tot += L.group_w[g] * (st[1] / (double)L.res[ri].frames + st[3] / st[0]);
    }
  *L.loss = tot;
}

template <int N>
__global__ void __launch_bounds__(LossCfg<N>::NT) k_mr_bwd(MgbLossRes r, const double* __restrict__ stats,
                                                           MgbLoss L, const float* __restrict__ xl,
                                                           const float* __restrict__ xr, int Ls) {
  constexpr int NT = LossCfg<N>::NT, NB = LossCfg<N>::NB;
  extern __shared__ __align__(16) unsigned char smraw[];
  double2* s = reinterpret_cast<double2*>(smraw);
  __shared__ double dmel[4][128];
  const int f = blockIdx.x;
  const int nm = r.n_mels;
  // dL/dmel
  for (int q = threadIdx.x; q < 4 * nm; q += NT) {
    const int g = q / nm, j = q % nm;
    const size_t o = ((size_t)g * r.frames + f) * nm + j;
    const double mel = r.mel[o];
    const double dlog = log(mel + LOG_EPS) - r.tlog[o];
    const double sg = (dlog > 0.0) ? 1.0 : (dlog < 0.0 ? -1.0 : 0.0);
    const double* st = stats + (size_t)g * 4;
    const double dn = st[3], tn = st[0];
    double v = sg / ((double)r.frames * (mel + LOG_EPS));
    if (dn > 0.0) v += (mel - r.tmel[o]) / (dn * tn);
    dmel[g][j] = L.group_w[g] * v;
  }
  load_fft<N>(s, xl, xr, Ls, r.hop, f);
  // per bin: dX_l, dX_r from the four groups, stored as Hermitian packs
  constexpr int PER = (NB + NT - 1) / NT;
  double2 dl[PER], dr[PER];
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int k = threadIdx.x + i * NT;
    dl[i] = dr[i] = make_double2(0.0, 0.0);
    if (k < NB) {
      double2 X[4];
      groups_at(s, N, k, X);
      double2 dX[4];
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        double dm = 0.0;
        const int b0 = r.bin_start[k], bl = r.bin_len[k];
        for (int e = 0; e < bl; ++e) dm = fma(dmel[g][r.bin_band[b0 + e]], r.bin_w[b0 + e], dm);
        const double mag = sqrt(X[g].x * X[g].x + X[g].y * X[g].y);
        const double den = mag == 0.0 ? 1.0 : mag;
        dX[g] = make_double2(dm * X[g].x / den, dm * X[g].y / den);
      }
      dl[i] = make_double2(dX[0].x + dX[2].x + dX[3].x, dX[0].y + dX[2].y + dX[3].y);
      dr[i] = make_double2(dX[1].x + dX[2].x - dX[3].x, dX[1].y + dX[2].y - dX[3].y);
    }
  }
  __syncthreads();
  // P[k] = Hl[k] + i Hr[k]; Hc[k] = dXc/2 (0<k<N/2), Hc[N-k] = conj(dXc)/2, Hc[0]/Hc[N/2] = Re dXc
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int k = threadIdx.x + i * NT;
    if (k < NB) {
      if (k == 0 || k == N / 2) {
        s[pidx<true>(k)] = make_double2(dl[i].x, dr[i].x);
      } else {
        const double2 hl = make_double2(0.5 * dl[i].x, 0.5 * dl[i].y);
        const double2 hr = make_double2(0.5 * dr[i].x, 0.5 * dr[i].y);
        s[pidx<true>(k)] = make_double2(hl.x - hr.y, hl.y + hr.x);         // hl + i hr
        s[pidx<true>(N - k)] = make_double2(hl.x + hr.y, -hl.y + hr.x);    // conj(hl) + i conj(hr)
      }
    }
  }
  smem_fft<double, N, 1, NT, N, 1, false, true>(s, true);
  float* gf = r.gframes + (size_t)f * 2 * N;
  for (int t = threadIdx.x; t < N; t += NT) {
    const double win = 0.5 - 0.5 * cospi(2.0 * t / (double)N);
    const double2 v = s[pidx<true>(t)];
    gf[t] = (float)(v.x * win);
    gf[N + t] = (float)(v.y * win);
  }
}

__global__ void k_mr_ola(MgbLoss L, float* __restrict__ gl, float* __restrict__ gr) {
  const int Ls = L.Ls;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < Ls; t += (long long)gridDim.x * blockDim.x) {
    double al = 0.0, ar = 0.0;
    for (int ri = 0; ri < L.n_res; ++ri) {
      const MgbLossRes& r = L.res[ri];
      const int n = r.n_fft, hop = r.hop, pad = n / 2;
      long long P[3];
      int np = 0;
      P[np++] = t + pad;
      if (t >= 1 && t <= pad) P[np++] = pad - t;
      if (t >= Ls - 1 - pad && t <= Ls - 2) P[np++] = 2LL * (Ls - 1) - t + pad;
      for (int q = 0; q < np; ++q) {
        const long long p = P[q];
        long long fhi = p / hop;
        if (fhi > r.frames - 1) fhi = r.frames - 1;
        long long flo = (p - n + hop) / hop;  // ceil((p - n + 1) / hop) for p >= n - 1
        if (p - n + 1 <= 0) flo = 0;
        for (long long f = flo; f <= fhi; ++f) {
          const long long o = p - f * hop;
          if (o < 0 || o >= n) continue;
          al += r.gframes[(size_t)f * 2 * n + o];
          ar += r.gframes[(size_t)f * 2 * n + n + o];
        }
      }
    }
    gl[t] = (float)al;
    gr[t] = (float)ar;
  }
}

template <int N>
int launch_fwd(const MgbLossRes& r, const float* xl, const float* xr, int Ls, int mode, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_mr_fwd<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LossCfg<N>::SMEM);
    cudaFuncSetAttribute(k_mr_bwd<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LossCfg<N>::SMEM);
    attr = true;
  }
  k_mr_fwd<N><<<r.frames, LossCfg<N>::NT, LossCfg<N>::SMEM, st>>>(r, xl, xr, Ls, mode);
  MGB_CHECK_LAUNCH();
  return 0;
}

template <int N>
int launch_bwd(const MgbLossRes& r, const double* stats, const MgbLoss& L, const float* xl, const float* xr,
               int Ls, cudaStream_t st) {
  k_mr_bwd<N><<<r.frames, LossCfg<N>::NT, LossCfg<N>::SMEM, st>>>(r, stats, L, xl, xr, Ls);
  MGB_CHECK_LAUNCH();
  return 0;
}

int dispatch_fwd(const MgbLossRes& r, const float* xl, const float* xr, int Ls, int mode, cudaStream_t st) {
  switch (r.n_fft) {
    case 256: return launch_fwd<256>(r, xl, xr, Ls, mode, st);
    case 512: return launch_fwd<512>(r, xl, xr, Ls, mode, st);
    case 1024: return launch_fwd<1024>(r, xl, xr, Ls, mode, st);
    case 2048: return launch_fwd<2048>(r, xl, xr, Ls, mode, st);
    case 4096: return launch_fwd<4096>(r, xl, xr, Ls, mode, st);
    case 8192: return launch_fwd<8192>(r, xl, xr, Ls, mode, st);
    default: return 1;
  }
}

int dispatch_bwd(const MgbLossRes& r, const double* stats, const MgbLoss& L, const float* xl, const float* xr,
                 int Ls, cudaStream_t st) {
  switch (r.n_fft) {
    case 256: return launch_bwd<256>(r, stats, L, xl, xr, Ls, st);
    case 512: return launch_bwd<512>(r, stats, L, xl, xr, Ls, st);
    case 1024: return launch_bwd<1024>(r, stats, L, xl, xr, Ls, st);
    case 2048: return launch_bwd<2048>(r, stats, L, xl, xr, Ls, st);
    case 4096: return launch_bwd<4096>(r, stats, L, xl, xr, Ls, st);
    case 8192: return launch_bwd<8192>(r, stats, L, xl, xr, Ls, st);
    default: return 1;
  }
}

int check_loss(const MgbLoss* L) {
  if (!L || L->n_res <= 0 || L->n_res > 8 || L->Ls <= 0) return 1;
  for (int i = 0; i < L->n_res; ++i) {
    const MgbLossRes& r = L->res[i];
    if (r.n_mels > 128 || r.n_fft / 2 >= L->Ls) return 1;
  }
  return 0;
}

}  // namespace

int mgb_loss_init() {
  // set smem attributes eagerly (outside any stream capture)
  MgbLossRes r{};
  (void)r;
  int rc = 0;
  rc |= cudaFuncSetAttribute(k_mr_fwd<4096>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LossCfg<4096>::SMEM);
  rc |= cudaFuncSetAttribute(k_mr_bwd<4096>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LossCfg<4096>::SMEM);
  rc |= cudaFuncSetAttribute(k_mr_fwd<8192>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LossCfg<8192>::SMEM);
  rc |= cudaFuncSetAttribute(k_mr_bwd<8192>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LossCfg<8192>::SMEM);
  rc |= cudaFuncSetAttribute(k_mr_fwd<2048>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LossCfg<2048>::SMEM);
  rc |= cudaFuncSetAttribute(k_mr_bwd<2048>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LossCfg<2048>::SMEM);
  return rc ? 2 : 0;
}

extern "C" int mgb_mrstft_target(const MgbLoss* L, const float* tl, const float* tr, void* stream) {
  if (int rc = check_loss(L)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  for (int i = 0; i < L->n_res; ++i)
    if (int rc = dispatch_fwd(L->res[i], tl, tr, L->Ls, 0, st)) return rc;
  k_mr_finalize<<<4 * L->n_res, 256, 0, st>>>(*L, 0);
  MGB_CHECK_LAUNCH();
  return 0;
}

extern "C" int mgb_mrstft_forward(const MgbLoss* L, const float* yl, const float* yr, void* stream) {
  if (int rc = check_loss(L)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  for (int i = 0; i < L->n_res; ++i)
    if (int rc = dispatch_fwd(L->res[i], yl, yr, L->Ls, 1, st)) return rc;
  k_mr_finalize<<<4 * L->n_res, 256, 0, st>>>(*L, 1);
  MGB_CHECK_LAUNCH();
  k_mr_total<<<1, 32, 0, st>>>(*L);
  MGB_CHECK_LAUNCH();
  return 0;
}

extern "C" int mgb_mrstft_backward(const MgbLoss* L, const float* yl, const float* yr, float* gl, float* gr,
                                   void* stream) {
  if (int rc = check_loss(L)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  for (int i = 0; i < L->n_res; ++i)
    if (int rc = dispatch_bwd(L->res[i], L->stats + (size_t)i * 16, *L, yl, yr, L->Ls, st)) return rc;
  const int blocks = (int)((L->Ls + 255) / 256 < 2048 ? (L->Ls + 255) / 256 : 2048);
  k_mr_ola<<<blocks, 256, 0, st>>>(*L, gl, gr);
  MGB_CHECK_LAUNCH();
  return 0;
}
