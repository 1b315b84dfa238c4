// FFT-convolution levels: equalizer (e), reverb (r), multitap delay (d).
//
// Forward (per level of B nodes, all rows batched in every launch):
//   FIR synthesis -> packed complex FIR (h_l + i h_r, zero padded to N)
//   FFT(H), FFT(pack(u)) = X   (both kept for the backward)
//   Q = X_l H_l + i X_r H_r (Hermitian pairing), IFFT(Q)/N
//   epilogue: ybar = conv[off : off+L], y = drywet(ybar, u, w), gain-staging norms
// Backward:
//   prologue: dybar = w gy + gain-staging term, gu = (1-w) gy + gain-staging term, dw partials
//   G = FFT(pack(dybar) at off);  GX = G conj(H), GH = G conj(X);  IFFT both
//   gu += gx[:L];  FIR adjoint from gh[:M] -> parameter gradient rows.
// This is fft_conv and its adjoints (mg/engine.py:549-585) with
// N = next_pow2(L + M - 1) exactly as the reference chooses it.
//
// FIRs:  e  zero_phase_fir(p, 2047), same FIR on both channels, offset 1023
//           (mg/processors.py:53-58, 115-120)
//        r  STFT-domain filtered noise, 313 frames x 384, OLA, / wss, L/R from
//           mid/side, offset 0 (mg/processors.py:127-188)
//        d  20 taps x 39-sample colour FIRs at m*3000 + rint-quantised offset,
//           offset 19; custom surrogate backward (mg/processors.py:250-318)
#include "common.cuh"
#include "mgb_internal.h"
#include "tables.cuh"

namespace {

constexpr int NT = 256;
constexpr int kMaxGrid = 2048;  // per-row CTAs of the grid-stride kernels (partials slots)
constexpr double PI = 3.141592653589793238462643383279502884;

struct ConvGeom {
  int M, off, logN;
  long long N;
};

ConvGeom geom(char tag, int L) {
  ConvGeom g;
  g.M = tag == 'e' ? MGB_EQ_LEN : (tag == 'r' ? MGB_REV_LEN : MGB_DLY_FIR);
  g.off = tag == 'e' ? (MGB_EQ_LEN - 1) / 2 : (tag == 'r' ? 0 : (MGB_COLOR_LEN - 1) / 2);
  g.logN = mgb_log2_ceil((long long)L + g.M - 1);
  if (g.logN < 5) g.logN = 5;
  g.N = 1LL << g.logN;
  return g;
}

int conv_nblk(int L) {
  int n = (L + 4 * NT - 1) / (4 * NT);
  return n < 1 ? 1 : (n > 128 ? 128 : n);
}

struct ConvWs {
  float2 *Z, *H, *T, *Q, *Q2;  // Q and Q2 adjacent (batched inverse FFT in bwd)
  double* stats;               // [B][4]: nu, ny, s (= sign(diff)), spare
  double* part;                // [B][nblk][4]
  float* aux;                  // r: frames (B,2,313,384) | d: colours (B,2,20,39)
  float* aux2;                 // r: dexpo (B,2,313,193)
  int* offs;                   // d: (B,2,20) quantised delays
};

ConvWs carve(char tag, int B, int L, void* base) {
  const ConvGeom g = geom(tag, L);
  MgbArena a{(char*)base, 0};
  ConvWs w;
  const size_t BN = (size_t)B * g.N;
  w.Z = a.take<float2>(BN);
  w.H = a.take<float2>(BN);
  w.T = a.take<float2>(BN);
  w.Q = a.take<float2>(2 * BN);
  w.Q2 = w.Q ? w.Q + BN : nullptr;
  w.stats = a.take<double>((size_t)B * 4);
  w.part = a.take<double>((size_t)B * kMaxGrid * 4);
  w.aux = w.aux2 = nullptr;
  w.offs = nullptr;
  if (tag == 'r') {
    w.aux = a.take<float>((size_t)B * 2 * MGB_REV_FRAMES * MGB_REV_NFFT);
    w.aux2 = a.take<float>((size_t)B * 2 * MGB_REV_FRAMES * MGB_REV_BINS);
  } else if (tag == 'd') {
    w.aux = a.take<float>((size_t)B * 2 * MGB_DLY_TAPS * MGB_COLOR_LEN);
    w.offs = a.take<int>((size_t)B * 2 * MGB_DLY_TAPS);
  }
  return w;
}

size_t carve_size(char tag, int B, int L) {
  const ConvGeom g = geom(tag, L);
  MgbArena a{nullptr, 0};
  const size_t BN = (size_t)B * g.N;
  a.take<float2>(BN);
  a.take<float2>(BN);
  a.take<float2>(BN);
  a.take<float2>(2 * BN);
  a.take<double>((size_t)B * 4);
  a.take<double>((size_t)B * kMaxGrid * 4);
  if (tag == 'r') {
    a.take<float>((size_t)B * 2 * MGB_REV_FRAMES * MGB_REV_NFFT);
    a.take<float>((size_t)B * 2 * MGB_REV_FRAMES * MGB_REV_BINS);
  } else if (tag == 'd') {
    a.take<float>((size_t)B * 2 * MGB_DLY_TAPS * MGB_COLOR_LEN);
    a.take<int>((size_t)B * 2 * MGB_DLY_TAPS);
  }
  return a.off;
}

// ---------------------------------------------------------------------------
// EQ FIR: centred[t'] = hann_sym(2047)[t'] * irfft(exp(p), 2047)[(t'+1024) % 2047]

__global__ void __launch_bounds__(NT) k_eq_fir(const double* __restrict__ bank, const int* __restrict__ prow,
                                               float2* __restrict__ H, long long N) {
  __shared__ double X[MGB_EQ_BINS];
  __shared__ double ct[MGB_EQ_LEN];
  const int b = blockIdx.y;
  float2* h = H + (size_t)b * N;
  const long long c0 = (long long)blockIdx.x * NT;
  for (long long k = c0 + threadIdx.x; k < N; k += (long long)gridDim.x * NT)  // zero tail
    if (k >= MGB_EQ_LEN) h[k] = make_float2(0.f, 0.f);
  if (c0 >= MGB_EQ_LEN) return;
  const double* p = bank + (size_t)prow[b] * MGB_EQ_BINS;
  for (int k = threadIdx.x; k < MGB_EQ_BINS; k += NT) X[k] = exp(p[k]);
  for (int j = threadIdx.x; j < MGB_EQ_LEN; j += NT) ct[j] = cospi(2.0 * j / (double)MGB_EQ_LEN);
  __syncthreads();
  const int tp = (int)c0 + threadIdx.x;
  if (tp < MGB_EQ_LEN) {
    const int t = (tp + 1024) % MGB_EQ_LEN;
    double acc = 0.0;
    int idx = t;
    for (int k = 1; k < MGB_EQ_BINS; ++k) {
      acc += X[k] * ct[idx];
      idx += t;
      if (idx >= MGB_EQ_LEN) idx -= MGB_EQ_LEN;
    }
    const double hv = (X[0] + 2.0 * acc) / (double)MGB_EQ_LEN;
    const double win = 0.5 - 0.5 * cospi(2.0 * tp / (double)(MGB_EQ_LEN - 1));
    const float c = (float)(hv * win);
    h[tp] = make_float2(c, c);
  }
}

// d p_k = X_k * (2/n) sum_t dh[t] cos(2 pi k t / n)   (k = 0: 1/n), dh summed over channels
__global__ void __launch_bounds__(1024) k_eq_fir_bwd(const double* __restrict__ bank, const int* __restrict__ prow,
                                                     const float2* __restrict__ GH, long long N,
                                                     double* __restrict__ gbank) {
  __shared__ double dh[MGB_EQ_LEN];
  __shared__ double ct[MGB_EQ_LEN];
  const int b = blockIdx.x;
  const float2* g = GH + (size_t)b * N;
  for (int tp = threadIdx.x; tp < MGB_EQ_LEN; tp += blockDim.x) {
    const double win = 0.5 - 0.5 * cospi(2.0 * tp / (double)(MGB_EQ_LEN - 1));
    const int t = (tp + 1024) % MGB_EQ_LEN;
    dh[t] = ((double)g[tp].x + (double)g[tp].y) * win;
    ct[tp] = cospi(2.0 * tp / (double)MGB_EQ_LEN);
  }
  __syncthreads();
  const int k = threadIdx.x;
  if (k < MGB_EQ_BINS) {
    double acc = 0.0;
    int idx = 0;
    for (int t = 0; t < MGB_EQ_LEN; ++t) {
      acc += dh[t] * ct[idx];
      idx += k;
      if (idx >= MGB_EQ_LEN) idx -= MGB_EQ_LEN;
    }
    const double scale = (k == 0 ? 1.0 : 2.0) / (double)MGB_EQ_LEN;
    const double* p = bank + (size_t)prow[b] * MGB_EQ_BINS;
    gbank[(size_t)prow[b] * MGB_EQ_BINS + k] = acc * scale * exp(p[k]);
  }
}

// ---------------------------------------------------------------------------
// Reverb FIR synthesis

__global__ void __launch_bounds__(MGB_REV_NFFT) k_rev_frames(const double* __restrict__ bank,
                                                             const int* __restrict__ prow,
                                                             float* __restrict__ frames) {
  __shared__ float2 X[2][MGB_REV_BINS];
  __shared__ float2 cs[MGB_REV_NFFT];
  const int m = blockIdx.x, b = blockIdx.y;
  const double* p = bank + (size_t)prow[b] * 768;
  const int i = threadIdx.x;
  {
    double s, c;
    sincospi(2.0 * i / (double)MGB_REV_NFFT, &s, &c);
    cs[i] = make_float2((float)c, (float)s);
  }
  for (int q = threadIdx.x; q < 2 * MGB_REV_BINS; q += blockDim.x) {
    const int ch = q / MGB_REV_BINS, k = q % MGB_REV_BINS;
    const int kk = k < MGB_REV_PBINS ? k : MGB_REV_PBINS - 1;  // Nyquist repeats the last bin
    const double h0 = p[ch * 384 + kk], hd = p[ch * 384 + 192 + kk];
    const float mag = (float)exp(h0 + hd * (double)m);
    const float2 s = g_rev_spec[ch][m][k];
    X[ch][k] = make_float2(mag * s.x, mag * s.y);
  }
  __syncthreads();
  float a0 = 0.f, a1 = 0.f;
  int idx = i;
  for (int k = 1; k < MGB_REV_PBINS; ++k) {
    const float2 w = cs[idx];
    a0 = fmaf(X[0][k].x, w.x, fmaf(-X[0][k].y, w.y, a0));
    a1 = fmaf(X[1][k].x, w.x, fmaf(-X[1][k].y, w.y, a1));
    idx += i;
    if (idx >= MGB_REV_NFFT) idx -= MGB_REV_NFFT;
  }
  const float sgn = (i & 1) ? -1.f : 1.f;
  const float win = 0.5f - 0.5f * cs[i].x;
  const float inv = 1.0f / (float)MGB_REV_NFFT;
  const float f0 = (X[0][0].x + sgn * X[0][MGB_REV_PBINS].x + 2.f * a0) * inv * win;
  const float f1 = (X[1][0].x + sgn * X[1][MGB_REV_PBINS].x + 2.f * a1) * inv * win;
  frames[(((size_t)b * 2 + 0) * MGB_REV_FRAMES + m) * MGB_REV_NFFT + i] = f0;
  frames[(((size_t)b * 2 + 1) * MGB_REV_FRAMES + m) * MGB_REV_NFFT + i] = f1;
}

__global__ void __launch_bounds__(NT) k_rev_assemble(const float* __restrict__ frames, float2* __restrict__ H,
                                                     long long N) {
  const int b = blockIdx.y;
  float2* h = H + (size_t)b * N;
  const float* fm = frames + (size_t)b * 2 * MGB_REV_FRAMES * MGB_REV_NFFT;
  const float* fs = fm + (size_t)MGB_REV_FRAMES * MGB_REV_NFFT;
  for (long long t = (long long)blockIdx.x * NT + threadIdx.x; t < N; t += (long long)gridDim.x * NT) {
    if (t >= MGB_REV_LEN) { h[t] = make_float2(0.f, 0.f); continue; }
    const int P = (int)t + MGB_REV_HOP;
    const int j = P / MGB_REV_HOP;
    float vm = 0.f, vs = 0.f;
    if (j < MGB_REV_FRAMES) {
      vm += fm[(size_t)j * MGB_REV_NFFT + (P - j * MGB_REV_HOP)];
      vs += fs[(size_t)j * MGB_REV_NFFT + (P - j * MGB_REV_HOP)];
    }
    if (j >= 1) {
      vm += fm[(size_t)(j - 1) * MGB_REV_NFFT + (P - (j - 1) * MGB_REV_HOP)];
      vs += fs[(size_t)(j - 1) * MGB_REV_NFFT + (P - (j - 1) * MGB_REV_HOP)];
    }
    const float iw = g_rev_inv_wss[t];
    vm *= iw;
    vs *= iw;
    h[t] = make_float2(0.5f * (vm + vs), 0.5f * (vm - vs));
  }
}

// dexpo[c][m][k] = Re(dX_k conj(S_mk)) * M_mk, dX = irfft adjoint of the windowed frame grad
__global__ void __launch_bounds__(MGB_REV_NFFT) k_rev_bwd_frames(const double* __restrict__ bank,
                                                                 const int* __restrict__ prow,
                                                                 const float2* __restrict__ GH, long long N,
                                                                 float* __restrict__ dexpo) {
  __shared__ float fr[2][MGB_REV_NFFT];
  __shared__ float2 cs[MGB_REV_NFFT];
  const int m = blockIdx.x, b = blockIdx.y;
  const float2* g = GH + (size_t)b * N;
  const int i = threadIdx.x;
  {
    double s, c;
    sincospi(2.0 * i / (double)MGB_REV_NFFT, &s, &c);
    cs[i] = make_float2((float)c, (float)s);
  }
  {
    const int t = m * MGB_REV_HOP + i - MGB_REV_HOP;  // position in the sliced FIR
    float dm = 0.f, ds = 0.f;
    if (t >= 0 && t < MGB_REV_LEN) {
      const float2 v = g[t];
      const float iw = g_rev_inv_wss[t];
      dm = 0.5f * (v.x + v.y) * iw;
      ds = 0.5f * (v.x - v.y) * iw;
    }
    const float win = 0.5f - 0.5f * (float)cospi(2.0 * i / (double)MGB_REV_NFFT);
    fr[0][i] = dm * win;
    fr[1][i] = ds * win;
  }
  __syncthreads();
  const double* p = bank + (size_t)prow[b] * 768;
  for (int q = threadIdx.x; q < 2 * MGB_REV_BINS; q += blockDim.x) {
    const int ch = q / MGB_REV_BINS, k = q % MGB_REV_BINS;
    float re = 0.f, im = 0.f;
    int idx = 0;
    for (int t = 0; t < MGB_REV_NFFT; ++t) {
      const float2 w = cs[idx];
      re = fmaf(fr[ch][t], w.x, re);
      im = fmaf(-fr[ch][t], w.y, im);
      idx += k;
      if (idx >= MGB_REV_NFFT) idx -= MGB_REV_NFFT;
    }
    float sc = 2.f / (float)MGB_REV_NFFT;
    if (k == 0 || k == MGB_REV_PBINS) sc *= 0.5f;
    re *= sc;
    im *= sc;
    const float2 s = g_rev_spec[ch][m][k];
    const int kk = k < MGB_REV_PBINS ? k : MGB_REV_PBINS - 1;
    const float mag = (float)exp(p[ch * 384 + kk] + p[ch * 384 + 192 + kk] * (double)m);
    dexpo[(((size_t)b * 2 + ch) * MGB_REV_FRAMES + m) * MGB_REV_BINS + k] = (re * s.x + im * s.y) * mag;
  }
}

__global__ void k_rev_bwd_reduce(const float* __restrict__ dexpo, const int* __restrict__ prow,
                                 double* __restrict__ gbank) {
  __shared__ double d0[2][MGB_REV_BINS], dd[2][MGB_REV_BINS];
  const int b = blockIdx.x;
  for (int q = threadIdx.x; q < 2 * MGB_REV_BINS; q += blockDim.x) {
    const int ch = q / MGB_REV_BINS, k = q % MGB_REV_BINS;
    const float* e = dexpo + ((size_t)b * 2 + ch) * MGB_REV_FRAMES * MGB_REV_BINS + k;
    double s0 = 0.0, s1 = 0.0;
    for (int m = 0; m < MGB_REV_FRAMES; ++m) {
      const double v = e[(size_t)m * MGB_REV_BINS];
      s0 += v;
      s1 += v * m;
    }
    d0[ch][k] = s0;
    dd[ch][k] = s1;
  }
  __syncthreads();
  double* g = gbank + (size_t)prow[b] * 768;
  for (int q = threadIdx.x; q < 2 * MGB_REV_PBINS; q += blockDim.x) {
    const int ch = q / MGB_REV_PBINS, k = q % MGB_REV_PBINS;
    double a = d0[ch][k], c = dd[ch][k];
    if (k == MGB_REV_PBINS - 1) { a += d0[ch][MGB_REV_PBINS]; c += dd[ch][MGB_REV_PBINS]; }
    g[ch * 384 + k] = a;
    g[ch * 384 + 192 + k] = c;
  }
}

// ---------------------------------------------------------------------------
// Multitap delay

// colour[t'] = hann_sym(39)[t'] * irfft(exp(bins), 39)[(t'+20) % 39] and the
// quantised offset d = rint(((-angle z) mod 2pi) / 2pi * 3000) mod 3000 in fp64
__global__ void k_dly_colour(const double* __restrict__ bank, const int* __restrict__ prow,
                             float* __restrict__ colour, int* __restrict__ offs) {
  const int tap = blockIdx.x, ch = blockIdx.y, b = blockIdx.z;
  const double* p = bank + (size_t)prow[b] * 880 + ch * 440;
  const int tp = threadIdx.x;
  if (tp < MGB_COLOR_LEN) {
    const double* bins = p + 40 + tap * MGB_COLOR_BINS;
    const int t = (tp + 20) % MGB_COLOR_LEN;
    double acc = 0.0;
    for (int k = 1; k < MGB_COLOR_BINS; ++k) acc += exp(bins[k]) * cospi(2.0 * ((k * t) % MGB_COLOR_LEN) / 39.0);
    const double hv = (exp(bins[0]) + 2.0 * acc) / 39.0;
    const double win = 0.5 - 0.5 * cospi(2.0 * tp / 38.0);
    colour[(((size_t)b * 2 + ch) * MGB_DLY_TAPS + tap) * MGB_COLOR_LEN + tp] = (float)(hv * win);
  }
  if (tp == 0) {
    const double re = p[tap], im = p[20 + tap];
    const double theta = atan2(im, re);
    const double two_pi = 2.0 * PI;
    double r = fmod(-theta, two_pi);
    if (r != 0.0 && r < 0.0) r += two_pi;
    const double pos = r / two_pi * (double)MGB_DLY_WIN;
    int d = (int)rint(pos);
    d %= MGB_DLY_WIN;
    offs[((size_t)b * 2 + ch) * MGB_DLY_TAPS + tap] = d;
  }
}

__global__ void __launch_bounds__(NT) k_dly_place(const float* __restrict__ colour, const int* __restrict__ offs,
                                                  float2* __restrict__ H, long long N) {
  __shared__ float col[2][MGB_DLY_TAPS][MGB_COLOR_LEN];
  __shared__ int dd[2][MGB_DLY_TAPS];
  const int b = blockIdx.y;
  for (int i = threadIdx.x; i < 2 * MGB_DLY_TAPS * MGB_COLOR_LEN; i += NT)
    (&col[0][0][0])[i] = colour[(size_t)b * 2 * MGB_DLY_TAPS * MGB_COLOR_LEN + i];
  for (int i = threadIdx.x; i < 2 * MGB_DLY_TAPS; i += NT) (&dd[0][0])[i] = offs[(size_t)b * 2 * MGB_DLY_TAPS + i];
  __syncthreads();
  float2* h = H + (size_t)b * N;
  for (long long k = (long long)blockIdx.x * NT + threadIdx.x; k < N; k += (long long)gridDim.x * NT) {
    float v[2] = {0.f, 0.f};
    if (k < MGB_DLY_FIR) {
      const int m1 = (int)(k / MGB_DLY_WIN);
#pragma unroll
      for (int ch = 0; ch < 2; ++ch) {
        float acc = 0.f;
        for (int m = m1 - 1; m <= m1; ++m) {
          if (m < 0 || m >= MGB_DLY_TAPS) continue;
          const int j = (int)k - m * MGB_DLY_WIN - dd[ch][m];
          if (j >= 0 && j < MGB_COLOR_LEN) acc += col[ch][m][j];
        }
        v[ch] = acc;
      }
    }
    h[k] = make_float2(v[0], v[1]);
  }
}

// One CTA per (tap, channel, row): colour gradient (gather + zero-phase FIR
// adjoint) and the damped-sinusoid surrogate z-gradient
// graw = conj( (1/n) sum_k k z^{k-1} E_k ),  E_k = sum_t e_t e^{+2 pi i k t / n},
// e_t = sum_j dh[m*3000 + t + j] colour[j]   (mg/processors.py:274-300).
// E is a 3000-point DFT done as 60 x 50 (t = t1 + 50 t2, k = k2 + 60 k1).
__global__ void __launch_bounds__(NT) k_dly_bwd(const double* __restrict__ bank, const int* __restrict__ prow,
                                                const float* __restrict__ colour, const int* __restrict__ offs,
                                                const float2* __restrict__ GH, long long N,
                                                double* __restrict__ gbank) {
  extern __shared__ __align__(16) unsigned char dsm[];
  float2* A = reinterpret_cast<float2*>(dsm);                  // 3000
  float2* E = A + MGB_DLY_WIN;                                 // 3000
  float* seg = reinterpret_cast<float*>(E + MGB_DLY_WIN);      // 3040
  float* et = seg + 3040;                                      // 3000
  __shared__ float col[MGB_COLOR_LEN];
  __shared__ double dhz[MGB_COLOR_LEN];
  __shared__ float2 w60[60], w50[50];
  __shared__ double red[32];
  const int tap = blockIdx.x, ch = blockIdx.y, b = blockIdx.z;
  const float2* g = GH + (size_t)b * N;
  const int base = tap * MGB_DLY_WIN;
  for (int i = threadIdx.x; i < MGB_DLY_WIN + MGB_COLOR_LEN - 1; i += NT) {
    const float2 v = g[base + i];
    seg[i] = ch == 0 ? v.x : v.y;
  }
  if (threadIdx.x < MGB_COLOR_LEN)
    col[threadIdx.x] = colour[(((size_t)b * 2 + ch) * MGB_DLY_TAPS + tap) * MGB_COLOR_LEN + threadIdx.x];
  if (threadIdx.x < 60) {
    float s, c;
    sincospif(2.0f * threadIdx.x / 60.0f, &s, &c);
    w60[threadIdx.x] = make_float2(c, s);
  }
  if (threadIdx.x < 50) {
    float s, c;
    sincospif(2.0f * threadIdx.x / 50.0f, &s, &c);
    w50[threadIdx.x] = make_float2(c, s);
  }
  const int d = offs[((size_t)b * 2 + ch) * MGB_DLY_TAPS + tap];
  const double* p = bank + (size_t)prow[b] * 880 + ch * 440;
  double* gp = gbank + (size_t)prow[b] * 880 + ch * 440;
  __syncthreads();
  // colour gradient -> bins
  if (threadIdx.x < MGB_COLOR_LEN) {
    const int tp = threadIdx.x;
    const double win = 0.5 - 0.5 * cospi(2.0 * tp / 38.0);
    dhz[(tp + 20) % MGB_COLOR_LEN] = (double)seg[d + tp] * win;
  }
  // e_t
  for (int t = threadIdx.x; t < MGB_DLY_WIN; t += NT) {
    float acc = 0.f;
#pragma unroll
    for (int j = 0; j < MGB_COLOR_LEN; ++j) acc = fmaf(seg[t + j], col[j], acc);
    et[t] = acc;
  }
  __syncthreads();
  if (threadIdx.x < MGB_COLOR_BINS) {
    const int k = threadIdx.x;
    double acc = 0.0;
    for (int t = 0; t < MGB_COLOR_LEN; ++t) acc += dhz[t] * cospi(2.0 * ((k * t) % MGB_COLOR_LEN) / 39.0);
    const double sc = (k == 0 ? 1.0 : 2.0) / 39.0;
    gp[40 + tap * MGB_COLOR_BINS + k] = acc * sc * exp(p[40 + tap * MGB_COLOR_BINS + k]);
  }
  // step A: A[t1][k2] = w_3000^{k2 t1} * sum_{t2} e[t1 + 50 t2] w_60^{k2 t2}
  for (int o = threadIdx.x; o < MGB_DLY_WIN; o += NT) {
    const int t1 = o / 60, k2 = o % 60;
    float re = 0.f, im = 0.f;
    int idx = 0;
    for (int t2 = 0; t2 < 60; ++t2) {
      const float e = et[t1 + 50 * t2];
      re = fmaf(e, w60[idx].x, re);
      im = fmaf(e, w60[idx].y, im);
      idx += k2;
      if (idx >= 60) idx -= 60;
    }
    float s, c;
    sincospif(2.0f * (float)(k2 * t1) / 3000.0f, &s, &c);
    A[o] = make_float2(re * c - im * s, re * s + im * c);
  }
  __syncthreads();
  // step B: E[k2 + 60 k1] = sum_{t1} A[t1][k2] w_50^{k1 t1}
  for (int o = threadIdx.x; o < MGB_DLY_WIN; o += NT) {
    const int k1 = o / 60, k2 = o % 60;
    float re = 0.f, im = 0.f;
    int idx = 0;
    for (int t1 = 0; t1 < 50; ++t1) {
      const float2 a = A[t1 * 60 + k2];
      const float2 w = w50[idx];
      re += a.x * w.x - a.y * w.y;
      im += a.x * w.y + a.y * w.x;
      idx += k1;
      if (idx >= 50) idx -= 50;
    }
    E[k2 + 60 * k1] = make_float2(re, im);
  }
  __syncthreads();
  // S = (1/n) sum_{k>=1} k z^{k-1} E_k   (z projected into the unit disk)
  double zr = p[tap], zi = p[20 + tap];
  const double mag = sqrt(zr * zr + zi * zi);
  if (mag > 1.0) { zr /= mag; zi /= mag; }
  const bool zero = (zr == 0.0 && zi == 0.0);
  const double lmag = zero ? 0.0 : log(zero ? 1.0 : fmin(mag, 1.0));
  const double th = atan2(zi, zr);
  double sre = 0.0, sim = 0.0;
  for (int k = 1 + threadIdx.x; k < MGB_DLY_WIN; k += NT) {
    double pr, pi;
    if (zero) {
      pr = (k == 1) ? 1.0 : 0.0;
      pi = 0.0;
    } else {
      const double a = exp((double)(k - 1) * lmag);
      double s, c;
      sincos((double)(k - 1) * th, &s, &c);
      pr = a * c;
      pi = a * s;
    }
    const double er = E[k].x, ei = E[k].y;
    sre += (double)k * (pr * er - pi * ei);
    sim += (double)k * (pr * ei + pi * er);
  }
  sre = block_sum(sre, red);
  __syncthreads();
  sim = block_sum(sim, red);
  if (threadIdx.x == 0) {
    gp[tap] = sre / (double)MGB_DLY_WIN;
    gp[20 + tap] = -sim / (double)MGB_DLY_WIN;
  }
}

// ---------------------------------------------------------------------------
// conv epilogue / prologue with dry/wet and gain staging

__global__ void __launch_bounds__(NT) k_conv_fwd_epi(const float* const* __restrict__ u_rows,
                                                     const float2* __restrict__ Yc, long long N, int off,
                                                     const int* __restrict__ widx, const double* __restrict__ w,
                                                     float* __restrict__ y, float* __restrict__ ybar,
                                                     double* __restrict__ part, int L) {
  __shared__ double scratch[32];
  const int b = blockIdx.y;
  const float* u = u_rows[b];
  const float2* yc = Yc + (size_t)b * N + off;
  float* yo = y + (size_t)b * 2 * L;
  float* yb = ybar + (size_t)b * 2 * L;
  const double wv = w ? w[widx[b]] : 1.0;
  const float wf = (float)wv, om = (float)(1.0 - wv);
  const bool bypass = (wv == 0.0);
  double su = 0.0, sy = 0.0;
  float fu = 0.f, fy = 0.f;
  int cnt = 0;
  for (long long n = (long long)blockIdx.x * NT + threadIdx.x; n < L; n += (long long)gridDim.x * NT) {
    const float2 v = yc[n];
    const float l = u[n], r = u[L + n];
    yb[n] = v.x;
    yb[L + n] = v.y;
    if (bypass) { yo[n] = l; yo[L + n] = r; }
    else { yo[n] = wf * v.x + om * l; yo[L + n] = wf * v.y + om * r; }
    const float mu = l + r, my = v.x + v.y;
    fu = fmaf(mu, mu, fu);
    fy = fmaf(my, my, fy);
    if (++cnt == 8) { su += fu; sy += fy; fu = fy = 0.f; cnt = 0; }
  }
  su += fu;
  sy += fy;
  su = block_sum(su, scratch);
  sy = block_sum(sy, scratch);
  if (threadIdx.x == 0) {
    double* pp = part + ((size_t)b * gridDim.x + blockIdx.x) * 4;
    pp[0] = su;
    pp[1] = sy;
  }
}

// norms and gain-staging term |log(ny+eps) - log(nu+eps)|  (mg/processors.py:83-90)
__global__ void k_gs_norms(const double* __restrict__ part, int nblk, double* __restrict__ stats,
                           double* __restrict__ reg) {
  const int b = blockIdx.x;
  if (threadIdx.x) return;
  double su = 0.0, sy = 0.0;
  for (int i = 0; i < nblk; ++i) {
    su += part[((size_t)b * nblk + i) * 4];
    sy += part[((size_t)b * nblk + i) * 4 + 1];
  }
  const double nu = sqrt(su), ny = sqrt(sy);
  const double diff = log(ny + MGB_GS_EPS) - log(nu + MGB_GS_EPS);
  stats[b * 4 + 0] = nu;
  stats[b * 4 + 1] = ny;
  stats[b * 4 + 2] = (diff > 0.0) ? 1.0 : (diff < 0.0 ? -1.0 : 0.0);
  if (reg) reg[b] = fabs(diff);
}

__global__ void __launch_bounds__(NT) k_conv_bwd_pro(const float* const* __restrict__ u_rows,
                                                     const float* const* __restrict__ gy_rows,
                                                     const float* __restrict__ ybar, const int* __restrict__ widx,
                                                     const double* __restrict__ w, const double* __restrict__ greg,
                                                     const double* __restrict__ stats, float2* __restrict__ G,
                                                     long long N, int off, float* __restrict__ gu,
                                                     double* __restrict__ part, int L) {
  __shared__ double scratch[32];
  const int b = blockIdx.y;
  const float* u = u_rows[b];
  const float* gy = gy_rows[b];
  const float* yb = ybar + (size_t)b * 2 * L;
  float* go = gu + (size_t)b * 2 * L;
  float2* g = G + (size_t)b * N;
  const double wv = w ? w[widx[b]] : 1.0;
  const float wf = (float)wv, om = (float)(1.0 - wv);
  const bool bypass = (wv == 0.0);
  const double gr = greg ? *greg : 0.0;
  const double nu = stats[b * 4], ny = stats[b * 4 + 1], sg = stats[b * 4 + 2] * gr;
  const float cy = (ny > 0.0) ? (float)(sg / ((ny + MGB_GS_EPS) * ny)) : 0.f;
  const float cu = (nu > 0.0) ? (float)(-sg / ((nu + MGB_GS_EPS) * nu)) : 0.f;
  double sw = 0.0;
  float fw = 0.f;
  int cnt = 0;
  for (long long k = (long long)blockIdx.x * NT + threadIdx.x; k < N; k += (long long)gridDim.x * NT) {
    const long long n = k - off;
    if (n < 0 || n >= L) { g[k] = make_float2(0.f, 0.f); continue; }
    const float l = u[n], r = u[L + n], gl = gy[n], grr = gy[L + n];
    const float yl = yb[n], yr = yb[L + n];
    const float my = yl + yr, mu = l + r;
    float dl, dr, ul, ur;
    if (bypass) { dl = 0.f; dr = 0.f; ul = gl; ur = grr; }
    else {
      dl = wf * gl; dr = wf * grr; ul = om * gl; ur = om * grr;
      fw = fmaf(gl, yl - l, fmaf(grr, yr - r, fw));
      if (++cnt == 8) { sw += fw; fw = 0.f; cnt = 0; }
    }
    dl = fmaf(cy, my, dl);
    dr = fmaf(cy, my, dr);
    go[n] = fmaf(cu, mu, ul);
    go[L + n] = fmaf(cu, mu, ur);
    g[k] = make_float2(dl, dr);
  }
  sw += fw;
  sw = block_sum(sw, scratch);
  if (threadIdx.x == 0) part[((size_t)b * gridDim.x + blockIdx.x) * 4 + 2] = sw;
}

__global__ void __launch_bounds__(NT) k_conv_bwd_epi(const float2* __restrict__ GXc, long long N,
                                                     float* __restrict__ gu, int L) {
  const int b = blockIdx.y;
  const float2* gx = GXc + (size_t)b * N;
  float* go = gu + (size_t)b * 2 * L;
  for (long long n = (long long)blockIdx.x * NT + threadIdx.x; n < L; n += (long long)gridDim.x * NT) {
    const float2 v = gx[n];
    go[n] += v.x;
    go[L + n] += v.y;
  }
}

__global__ void k_dw_finalize(const double* __restrict__ part, int nblk, const int* __restrict__ widx,
                              const double* __restrict__ w, double* __restrict__ gw) {
  const int b = blockIdx.x;
  if (threadIdx.x) return;
  double s = 0.0;
  for (int i = 0; i < nblk; ++i) s += part[((size_t)b * nblk + i) * 4 + 2];
  const double wv = w ? w[widx[b]] : 1.0;
  if (gw) gw[widx[b]] = (wv == 0.0) ? 0.0 : s;
}

int grid_for(long long n) {
  long long g = (n + NT - 1) / NT;
  return (int)(g < 1 ? 1 : (g > kMaxGrid ? kMaxGrid : g));
}

constexpr int kDlyBwdSmem = (2 * MGB_DLY_WIN) * 8 + (3040 + MGB_DLY_WIN) * 4;

}  // namespace

int mgb_conv_init() {
  if (cudaFuncSetAttribute(k_dly_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, kDlyBwdSmem) != cudaSuccess)
    return 2;
  return 0;
}

size_t mgb_conv_workspace(char tag, int B, int L) { return carve_size(tag, B, L); }

int mgb_conv_forward(const MgbLevel* lv, cudaStream_t st) {
  const char tag = lv->tag;
  const int B = lv->B, L = lv->L;
  if (!lv->ybar) return 1;
  const ConvGeom g = geom(tag, L);
  ConvWs w = carve(tag, B, L, lv->ws);
  int rc;
  // FIR synthesis into H
  if (tag == 'e') {
    k_eq_fir<<<dim3(grid_for(g.N), B), NT, 0, st>>>(lv->bank, lv->prow, w.H, g.N);
  } else if (tag == 'r') {
    k_rev_frames<<<dim3(MGB_REV_FRAMES, B), MGB_REV_NFFT, 0, st>>>(lv->bank, lv->prow, w.aux);
    MGB_CHECK_LAUNCH();
    k_rev_assemble<<<dim3(grid_for(g.N), B), NT, 0, st>>>(w.aux, w.H, g.N);
  } else {
    k_dly_colour<<<dim3(MGB_DLY_TAPS, 2, B), 64, 0, st>>>(lv->bank, lv->prow, w.aux, w.offs);
    MGB_CHECK_LAUNCH();
    k_dly_place<<<dim3(grid_for(g.N), B), NT, 0, st>>>(w.aux, w.offs, w.H, g.N);
  }
  MGB_CHECK_LAUNCH();
  if ((rc = mgb_fft_c2c(w.H, w.H, w.T, B, g.logN, 0, 1.f, st))) return rc;
  if ((rc = mgb_pack_rows(lv->u_rows, w.Z, B, L, g.N, st))) return rc;
  if ((rc = mgb_fft_c2c(w.Z, w.Z, w.T, B, g.logN, 0, 1.f, st))) return rc;
  if ((rc = mgb_spec_pair(w.Z, w.H, w.Q, nullptr, nullptr, B, g.N, 0, st))) return rc;
  if ((rc = mgb_fft_c2c(w.Q, w.Q, w.T, B, g.logN, 1, 1.f / (float)g.N, st))) return rc;
  const int nblk = conv_nblk(L);
  k_conv_fwd_epi<<<dim3(nblk, B), NT, 0, st>>>(lv->u_rows, w.Q, g.N, g.off, lv->widx, lv->w, lv->y, lv->ybar,
                                               w.part, L);
  MGB_CHECK_LAUNCH();
  k_gs_norms<<<B, 32, 0, st>>>(w.part, nblk, w.stats, lv->reg);
  MGB_CHECK_LAUNCH();
  return 0;
}

int mgb_conv_backward(const MgbLevel* lv, cudaStream_t st) {
  const char tag = lv->tag;
  const int B = lv->B, L = lv->L;
  if (!lv->ybar) return 1;
  const ConvGeom g = geom(tag, L);
  ConvWs w = carve(tag, B, L, lv->ws);
  int rc;
  const int nblk = conv_nblk(L);
  k_conv_bwd_pro<<<dim3(grid_for(g.N), B), NT, 0, st>>>(lv->u_rows, lv->gy_rows, lv->ybar, lv->widx, lv->w,
                                                        lv->greg, w.stats, w.Q, g.N, g.off, lv->gu, w.part, L);
  MGB_CHECK_LAUNCH();
  if ((rc = mgb_fft_c2c(w.Q, w.Q, w.T, B, g.logN, 0, 1.f, st))) return rc;
  if ((rc = mgb_spec_pair(w.Q, w.H, w.Q, w.Z, w.Q2, B, g.N, 1, st))) return rc;
  if ((rc = mgb_fft_c2c(w.Q, w.Q, w.T, 2 * B, g.logN, 1, 1.f / (float)g.N, st))) return rc;
  k_conv_bwd_epi<<<dim3(nblk, B), NT, 0, st>>>(w.Q, g.N, lv->gu, L);
  MGB_CHECK_LAUNCH();
  if (tag == 'e') {
    k_eq_fir_bwd<<<B, 1024, 0, st>>>(lv->bank, lv->prow, w.Q2, g.N, lv->gbank);
  } else if (tag == 'r') {
    k_rev_bwd_frames<<<dim3(MGB_REV_FRAMES, B), MGB_REV_NFFT, 0, st>>>(lv->bank, lv->prow, w.Q2, g.N, w.aux2);
    MGB_CHECK_LAUNCH();
    k_rev_bwd_reduce<<<B, 256, 0, st>>>(w.aux2, lv->prow, lv->gbank);
  } else {
    k_dly_bwd<<<dim3(MGB_DLY_TAPS, 2, B), NT, kDlyBwdSmem, st>>>(lv->bank, lv->prow, w.aux, w.offs, w.Q2, g.N, lv->gbank);
  }
  MGB_CHECK_LAUNCH();
  k_dw_finalize<<<B, 32, 0, st>>>(w.part, grid_for(g.N), lv->widx, lv->w, lv->gw);
  MGB_CHECK_LAUNCH();
  return 0;
}
