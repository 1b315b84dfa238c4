// FIR synthesis and FIR adjoint kernels of the e / r / d levels (included by conv.cu).
#pragma once
// ---------------------------------------------------------------------------
// EQ FIR: centred[t'] = hann_sym(2047)[t'] * irfft(exp(p), 2047)[(t'+1024) % 2047]

// 32 outputs per CTA (lane), 8 warps split the 1023 cosine terms; compact (B, 2047) output
__global__ void __launch_bounds__(256) k_eq_fir(const double* __restrict__ bank, const int* __restrict__ prow,
                                                float2* __restrict__ H) {
  mgb_pdl_entry();
  __shared__ double X[MGB_EQ_BINS];
  __shared__ double part[8][33];
  const int b = blockIdx.y;
  const double* p = bank + (size_t)prow[b] * MGB_EQ_BINS;
  for (int k = threadIdx.x; k < MGB_EQ_BINS; k += 256) X[k] = exp(p[k]);
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int tp = blockIdx.x * 32 + lane;
  const int t = (tp + 1024) % MGB_EQ_LEN;
  const int k0 = 1 + w * 128, k1 = min(MGB_EQ_BINS, k0 + 128);
  // cos(2 pi k t / n) by a float64 rotation recurrence from an exactly reduced start
  // (per-lane table lookups at scattered indices were shared-memory bound)
  double acc = 0.0, cr, ci, sr, si;
  sincospi(2.0 * (double)(((long long)k0 * t) % MGB_EQ_LEN) / (double)MGB_EQ_LEN, &ci, &cr);
  sincospi(2.0 * (double)t / (double)MGB_EQ_LEN, &si, &sr);
  for (int k = k0; k < k1; ++k) {
    acc = fma(X[k], cr, acc);
    const double nr = cr * sr - ci * si;
    ci = fma(cr, si, ci * sr);
    cr = nr;
  }
  part[w][lane] = acc;
  __syncthreads();
  if (w == 0 && tp < MGB_EQ_LEN) {
    double s = 0.0;
    for (int i = 0; i < 8; ++i) s += part[i][lane];
    const double hv = (X[0] + 2.0 * s) / (double)MGB_EQ_LEN;
    const float c = (float)(hv * g_hann2047[tp]);
    H[(size_t)b * MGB_EQ_LEN + tp] = make_float2(c, c);
  }
}

// d p_k = X_k * (2/n) sum_t dh[t] cos(2 pi k t / n)   (k = 0: 1/n), dh summed over channels.
// 32 bins per CTA (lane), 8 warps split t.
__global__ void __launch_bounds__(256) k_eq_fir_bwd(const double* __restrict__ bank, const int* __restrict__ prow,
                                                    const float2* __restrict__ GH, int M,
                                                    double* __restrict__ gbank) {
  mgb_pdl_entry();
  __shared__ double dh[MGB_EQ_LEN];
  __shared__ double part[8][33];
  const int b = blockIdx.y;
  const float2* g = GH + (size_t)b * M;
  for (int tp = threadIdx.x; tp < MGB_EQ_LEN; tp += 256) {
    const float2 v = g[tp];
    dh[(tp + 1024) % MGB_EQ_LEN] = ((double)v.x + (double)v.y) * g_hann2047[tp];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int k = blockIdx.x * 32 + lane;
  const int t0 = w * 256, t1 = min(MGB_EQ_LEN, t0 + 256);
  double acc = 0.0, cr, ci, sr, si;  // rotation recurrence, as in k_eq_fir
  sincospi(2.0 * (double)(((long long)k * t0) % MGB_EQ_LEN) / (double)MGB_EQ_LEN, &ci, &cr);
  sincospi(2.0 * (double)k / (double)MGB_EQ_LEN, &si, &sr);
  for (int t = t0; t < t1; ++t) {
    acc = fma(dh[t], cr, acc);
    const double nr = cr * sr - ci * si;
    ci = fma(cr, si, ci * sr);
    cr = nr;
  }
  part[w][lane] = acc;
  __syncthreads();
  if (w == 0 && k < MGB_EQ_BINS) {
    double s = 0.0;
    for (int i = 0; i < 8; ++i) s += part[i][lane];
    const double scale = (k == 0 ? 1.0 : 2.0) / (double)MGB_EQ_LEN;
    const double* p = bank + (size_t)prow[b] * MGB_EQ_BINS;
    gbank[(size_t)prow[b] * MGB_EQ_BINS + k] = s * scale * exp(p[k]);
  }
}

// ---------------------------------------------------------------------------
// Reverb FIR synthesis

__global__ void __launch_bounds__(NT) k_rev_assemble(const float* __restrict__ frames, float2* __restrict__ H) {
  mgb_pdl_entry();
  const int b = blockIdx.y;
  const long long N = MGB_REV_LEN;
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

// d H0[c][k] = sum_m dexpo[c][m][k],  d HD[c][k] = sum_m m dexpo[c][m][k]: k_rev_bwd_frames_fft
// leaves per-CTA (8-frame) float64 partials part[b][cta][c][k][2]; this sums the
// RV_CTAS partials in a fixed order and folds the Nyquist bin into the last
// parameter bin.  One thread per (c, k).
constexpr int RV_CTAS = (MGB_REV_FRAMES + 7) / 8;
__global__ void __launch_bounds__(256) k_rev_bwd_reduce(const double* __restrict__ part,
                                                        const int* __restrict__ prow,
                                                        double* __restrict__ gbank) {
  mgb_pdl_entry();
  const int b = blockIdx.y;
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= 2 * MGB_REV_PBINS) return;
  const int ch = q / MGB_REV_PBINS, k = q % MGB_REV_PBINS;
  const double* pp = part + (size_t)b * RV_CTAS * 2 * MGB_REV_BINS * 2;
  double a0 = 0.0, a1 = 0.0;
  for (int c = 0; c < RV_CTAS; ++c) {
    const double* e = pp + ((size_t)c * 2 + ch) * MGB_REV_BINS * 2;
    a0 += e[2 * k];
    a1 += e[2 * k + 1];
    if (k == MGB_REV_PBINS - 1) {
      a0 += e[2 * MGB_REV_PBINS];
      a1 += e[2 * MGB_REV_PBINS + 1];
    }
  }
  double* g = gbank + (size_t)prow[b] * 768 + ch * 384;
  g[k] = a0;
  g[192 + k] = a1;
}

// ---------------------------------------------------------------------------
// Multitap delay

// colour[t'] = hann_sym(39)[t'] * irfft(exp(bins), 39)[(t'+20) % 39] and the
// quantised offset d = rint(((-angle z) mod 2pi) / 2pi * 3000) mod 3000 in fp64
__global__ void k_dly_colour(const double* __restrict__ bank, const int* __restrict__ prow,
                             float* __restrict__ colour, int* __restrict__ offs) {
  mgb_pdl_entry();
  const int tap = blockIdx.x, ch = blockIdx.y, b = blockIdx.z;
  const double* p = bank + (size_t)prow[b] * 880 + ch * 440;
  const int tp = threadIdx.x;
  if (tp < MGB_COLOR_LEN) {
    const double* bins = p + 40 + tap * MGB_COLOR_BINS;
    const int t = (tp + 20) % MGB_COLOR_LEN;
    double acc = 0.0;
    for (int k = 1; k < MGB_COLOR_BINS; ++k) acc += exp(bins[k]) * g_cos39[(k * t) % MGB_COLOR_LEN];
    const double hv = (exp(bins[0]) + 2.0 * acc) / 39.0;
    colour[(((size_t)b * 2 + ch) * MGB_DLY_TAPS + tap) * MGB_COLOR_LEN + tp] = (float)(hv * g_hann39[tp]);
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
                                                  float2* __restrict__ H) {
  mgb_pdl_entry();
  const long long N = MGB_DLY_FIR;
  __shared__ float col[2][MGB_DLY_TAPS][MGB_COLOR_LEN];
  __shared__ int dd[2][MGB_DLY_TAPS];
  const int b = blockIdx.y;
  {
    constexpr int CN = 2 * MGB_DLY_TAPS * MGB_COLOR_LEN, IT = (CN + NT - 1) / NT;
    float cv[IT];
#pragma unroll
    for (int k = 0; k < IT; ++k) {
      const int i = threadIdx.x + k * NT;
      cv[k] = i < CN ? __ldg(colour + (size_t)b * CN + i) : 0.f;
    }
#pragma unroll
    for (int k = 0; k < IT; ++k)
      if (threadIdx.x + k * NT < CN) (&col[0][0][0])[threadIdx.x + k * NT] = cv[k];
  }
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
// adjoint) and the damped-sinusoid surrogate z-gradient (mg/processors.py:274-300)
//   graw = conj( sum_t e_t deriv_t ),  deriv = ifft(k z^{k-1}) (length n = 3000, k = 0 term 0),
//   e_t = sum_j dh[m*3000 + t + j] colour[j].
// deriv has a closed form: with w = e^{2 pi i / n} and q = z w^t (so q^n = z^n),
//   deriv_t = (1/n) w^t f(q),  f(q) = sum_{k=1}^{n-1} k q^{k-1} = (1 - n z^{n-1} w^{-t} + (n-1) z^n) / (1 - q)^2,
// evaluated in float64 (relative error ~ 2 eps / (n |1-q|^2)); for |1-q| < 1e-6 the
// series itself is summed.  This replaces the 3000-point DFT of e_t.
__global__ void __launch_bounds__(NT) k_dly_bwd(const double* __restrict__ bank, const int* __restrict__ prow,
                                                const float* __restrict__ colour, const int* __restrict__ offs,
                                                const float2* __restrict__ GH, int N,
                                                double* __restrict__ gbank) {
  mgb_pdl_entry();
  __shared__ float seg[3040];
  __shared__ float col[MGB_COLOR_LEN];
  __shared__ double dhz[MGB_COLOR_LEN];
  __shared__ double red[32];
  const int tap = blockIdx.x, ch = blockIdx.y, b = blockIdx.z;
  const float2* g = GH + (size_t)b * N;
  const int base = tap * MGB_DLY_WIN;
  {  // all loads in flight at once (a rolled loop waits on each in turn)
    constexpr int SEGN = MGB_DLY_WIN + MGB_COLOR_LEN - 1, IT = (SEGN + NT - 1) / NT;
    float sv[IT];
#pragma unroll
    for (int k = 0; k < IT; ++k) {
      const int i = threadIdx.x + k * NT;
      sv[k] = 0.f;
      if (i < SEGN) {
        const float2 v = __ldg(g + base + i);
        sv[k] = ch == 0 ? v.x : v.y;
      }
    }
#pragma unroll
    for (int k = 0; k < IT; ++k)
      if (threadIdx.x + k * NT < SEGN) seg[threadIdx.x + k * NT] = sv[k];
  }
  if (threadIdx.x < MGB_COLOR_LEN)
    col[threadIdx.x] = colour[(((size_t)b * 2 + ch) * MGB_DLY_TAPS + tap) * MGB_COLOR_LEN + threadIdx.x];
  const int d = offs[((size_t)b * 2 + ch) * MGB_DLY_TAPS + tap];
  const double* p = bank + (size_t)prow[b] * 880 + ch * 440;
  double* gp = gbank + (size_t)prow[b] * 880 + ch * 440;
  __syncthreads();
  // colour gradient -> bins
  if (threadIdx.x < MGB_COLOR_LEN) {
    const int tp = threadIdx.x;
    dhz[(tp + 20) % MGB_COLOR_LEN] = (double)seg[d + tp] * g_hann39[tp];
  }
  __syncthreads();
  if (threadIdx.x < MGB_COLOR_BINS) {
    const int k = threadIdx.x;
    double acc = 0.0;
    for (int t = 0; t < MGB_COLOR_LEN; ++t) acc += dhz[t] * g_cos39[(k * t) % MGB_COLOR_LEN];
    const double sc = (k == 0 ? 1.0 : 2.0) / 39.0;
    gp[40 + tap * MGB_COLOR_BINS + k] = acc * sc * exp(p[40 + tap * MGB_COLOR_BINS + k]);
  }
  // z projected into the unit disk; z^n, z^{n-1} from log space (as the reference's powers)
  constexpr int n = MGB_DLY_WIN;
  double zr = p[tap], zi = p[20 + tap];
  const double mag = sqrt(zr * zr + zi * zi);
  if (mag > 1.0) { zr /= mag; zi /= mag; }
  const bool zero = (zr == 0.0 && zi == 0.0);
  const double lmag = zero ? 0.0 : log(fmin(mag, 1.0));
  const double th = atan2(zi, zr);
  double zn_r = 0.0, zn_i = 0.0, zm_r = 0.0, zm_i = 0.0;  // z^n, z^{n-1}
  if (!zero) {
    double s, c;
    const double an = exp((double)n * lmag), am = exp((double)(n - 1) * lmag);
    sincos((double)n * th, &s, &c);
    zn_r = an * c;
    zn_i = an * s;
    sincos((double)(n - 1) * th, &s, &c);
    zm_r = am * c;
    zm_i = am * s;
  }
  // this thread's contiguous run of t; w^t by a float64 recurrence from one sincospi
  constexpr int PER = (n + NT - 1) / NT;
  const int t0 = threadIdx.x * PER;
  double wr, wi, sr, si;
  sincospi(2.0 * (double)t0 / (double)n, &wi, &wr);
  sincospi(2.0 / (double)n, &si, &sr);
  double sre = 0.0, sim = 0.0;
  // e_t for this thread's run from a register window of seg (one shared-memory read
  // per sample and per colour tap instead of two per multiply-add; same summation order)
  float et[PER];
  {
    constexpr int WIN = PER + MGB_COLOR_LEN - 1, SEGN = MGB_DLY_WIN + MGB_COLOR_LEN - 1;
    float win[WIN];
#pragma unroll
    for (int i = 0; i < WIN; ++i) win[i] = (t0 + i < SEGN) ? seg[t0 + i] : 0.f;
#pragma unroll
    for (int i = 0; i < PER; ++i) et[i] = 0.f;
#pragma unroll
    for (int j = 0; j < MGB_COLOR_LEN; ++j) {
      const float c = col[j];
#pragma unroll
      for (int i = 0; i < PER; ++i) et[i] = fmaf(win[i + j], c, et[i]);
    }
  }
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int t = t0 + i;
    if (t >= n) break;
    // q = z w^t
    const double qr = zr * wr - zi * wi, qi = zr * wi + zi * wr;
    const double ar = 1.0 - qr, ai = -qi;  // 1 - q
    double fr, fi;
    if (ar * ar + ai * ai >= 1e-12) {
      // numerator 1 - n z^{n-1} conj(w^t) + (n-1) z^n
      const double nr = 1.0 - (double)n * (zm_r * wr + zm_i * wi) + (double)(n - 1) * zn_r;
      const double ni = -(double)n * (zm_i * wr - zm_r * wi) + (double)(n - 1) * zn_i;
      const double dr = ar * ar - ai * ai, di = 2.0 * ar * ai;  // (1 - q)^2
      const double iden = 1.0 / (dr * dr + di * di);
      fr = (nr * dr + ni * di) * iden;
      fi = (ni * dr - nr * di) * iden;
    } else {  // q ~ 1: Horner on the series
      fr = (double)(n - 1);
      fi = 0.0;
      for (int k = n - 2; k >= 1; --k) {
        const double tr = fr * qr - fi * qi + (double)k;
        fi = fr * qi + fi * qr;
        fr = tr;
      }
    }
    // deriv_t = w^t f / n
    constexpr double inv_n = 1.0 / (double)n;
    const double der = (wr * fr - wi * fi) * inv_n, dei = (wr * fi + wi * fr) * inv_n;
    sre += (double)et[i] * der;
    sim += (double)et[i] * dei;
    const double nw = wr * sr - wi * si;
    wi = wr * si + wi * sr;
    wr = nw;
  }
  sre = block_sum(sre, red);
  __syncthreads();
  sim = block_sum(sim, red);
  if (threadIdx.x == 0) {
    gp[tap] = sre;
    gp[20 + tap] = -sim;
  }
}

// ---------------------------------------------------------------------------
// conv epilogue / prologue with dry/wet and gain staging

