// Reverb FIR synthesis and its adjoint with 384-point FFTs (included by conv.cu).
//
// Forward (mg/processors.py:148-181): per frame m and channel c in {mid, side}
//   X_c[k] = exp(H0_c[k] + m HD_c[k]) * S_c[m][k]   (k = 0..192, bin 192 repeats param 191)
//   frame_c = irfft(X_c, 384) * periodic_hann(384)
// Both channels ride one complex inverse DFT: Z = Xh_mid + i Xh_side with Xh the
// Hermitian extension (numpy's irfft drops the imaginary part of bins 0 and
// 192), so z = IDFT(Z) = frame_mid + i frame_side.  The 384-point DFT is a
// four-step 3 x 128: a radix-3 step down the 128 columns with twiddles
// e^{+-2 pi i k2 n1 / 384}, then three 128-point shared-memory FFTs.
// Backward: the frame adjoint (the OLA slice / wss, times the window) of both
// channels is packed into one forward DFT; the irfft adjoint (rfft * 2/n,
// halved at bins 0 and 192) and the Re(g conj S) * M chain give d expo.
#pragma once

constexpr int RV_F = 8;                         // frames per CTA
constexpr int RV_NT = 256;
constexpr int RV_P = padded_len<128>();         // padded 128-point row
constexpr int RV_FRAME = 3 * RV_P;              // one frame = 3 rows
constexpr int kRevFftSmem = RV_F * RV_FRAME * 8;

// in-place 384-point DFT of RV_F frames laid out [f][n1 or k1 row][padded 128]
__device__ __forceinline__ void dft384(float2* s, bool inv) {
  const float c3 = -0.5f, s3 = inv ? 0.86602540378443864676f : -0.86602540378443864676f;
  __syncthreads();
  for (int q = threadIdx.x; q < RV_F * 128; q += RV_NT) {  // radix-3 down each column + twiddle
    const int f = q >> 7, k2 = q & 127;
    float2* col = s + f * RV_FRAME + pidx<true>(k2);
    const float2 a0 = col[0], a1 = col[RV_P], a2 = col[2 * RV_P];
    const float2 t = make_float2(a1.x + a2.x, a1.y + a2.y);
    const float2 d = make_float2(a1.x - a2.x, a1.y - a2.y);
    const float2 b0 = make_float2(a0.x + t.x, a0.y + t.y);
    const float2 m = make_float2(a0.x + c3 * t.x, a0.y + c3 * t.y);
    // b1 = m + w3 * d_perp, b2 = m - w3 * d_perp  with d_perp = i * d * s3
    const float2 b1 = make_float2(m.x - s3 * d.y, m.y + s3 * d.x);
    const float2 b2 = make_float2(m.x + s3 * d.y, m.y - s3 * d.x);
    float sn, cs;
    sincospif((inv ? 2.f : -2.f) * (float)k2 / 384.f, &sn, &cs);
    const float2 w1 = make_float2(cs, sn);
    const float2 w2 = cmul(w1, w1);
    col[0] = b0;
    col[RV_P] = cmul(b1, w1);
    col[2 * RV_P] = cmul(b2, w2);
  }
  smem_fft<float, 128, 3 * RV_F, RV_NT, RV_P, 1, false, true>(s, inv);
}

__global__ void __launch_bounds__(RV_NT) k_rev_frames_fft(const double* __restrict__ bank,
                                                           const int* __restrict__ prow,
                                                           float* __restrict__ frames) {
  mgb_pdl_entry();
  extern __shared__ __align__(16) unsigned char dsm[];
  float2* s = reinterpret_cast<float2*>(dsm);
  __shared__ float win[MGB_REV_NFFT];  // periodic Hann(384) / 384
  const int m0 = blockIdx.x * RV_F, b = blockIdx.y;
  const double* p = bank + (size_t)prow[b] * 768;
  for (int i = threadIdx.x; i < MGB_REV_NFFT; i += RV_NT)
    win[i] = (0.5f - 0.5f * cospif(2.f * (float)i / (float)MGB_REV_NFFT)) * (1.0f / (float)MGB_REV_NFFT);
  // (f, k) = divmod(q, 193) stepped without divisions
  int f = 0, k = threadIdx.x;
  while (k >= MGB_REV_PBINS + 1) k -= MGB_REV_PBINS + 1, ++f;
  for (int q = threadIdx.x; q < RV_F * (MGB_REV_PBINS + 1); q += RV_NT, k += RV_NT) {
    while (k >= MGB_REV_PBINS + 1) k -= MGB_REV_PBINS + 1, ++f;
    const int m = m0 + f;
    float2 Z0 = make_float2(0.f, 0.f), Z1 = Z0;  // Z[k], Z[384-k]
    if (m < MGB_REV_FRAMES) {
      const int kk = k < MGB_REV_PBINS ? k : MGB_REV_PBINS - 1;
      const float mm = expf((float)(p[kk] + p[192 + kk] * (double)m));
      const float ms = expf((float)(p[384 + kk] + p[576 + kk] * (double)m));
      const float2 sm = g_rev_spec[0][m][k], ss = g_rev_spec[1][m][k];
      float2 xm = make_float2(mm * sm.x, mm * sm.y), xs = make_float2(ms * ss.x, ms * ss.y);
      if (k == 0 || k == MGB_REV_PBINS) { xm.y = 0.f; xs.y = 0.f; }
      Z0 = make_float2(xm.x - xs.y, xm.y + xs.x);   // xm + i xs
      Z1 = make_float2(xm.x + xs.y, -xm.y + xs.x);  // conj(xm) + i conj(xs)
    }
    float2* fr = s + f * RV_FRAME;
    fr[(k >> 7) * RV_P + pidx<true>(k & 127)] = Z0;
    if (k != 0 && k != MGB_REV_PBINS) {
      const int k2 = MGB_REV_NFFT - k;
      fr[(k2 >> 7) * RV_P + pidx<true>(k2 & 127)] = Z1;
    }
  }
  dft384(s, true);  // (its barriers publish the window table)
  int fo = 0, i = threadIdx.x;  // (fo, i) = divmod(q, 384), stepped
  for (int q = threadIdx.x; q < RV_F * MGB_REV_NFFT; q += RV_NT, i += RV_NT) {
    while (i >= MGB_REV_NFFT) i -= MGB_REV_NFFT, ++fo;
    const int m = m0 + fo;
    if (m >= MGB_REV_FRAMES) continue;
    const float2 z = s[fo * RV_FRAME + (i % 3) * RV_P + pidx<true>(i / 3)];
    const float wv = win[i];
    frames[(((size_t)b * 2 + 0) * MGB_REV_FRAMES + m) * MGB_REV_NFFT + i] = z.x * wv;
    frames[(((size_t)b * 2 + 1) * MGB_REV_FRAMES + m) * MGB_REV_NFFT + i] = z.y * wv;
  }
}

__global__ void __launch_bounds__(RV_NT) k_rev_bwd_frames_fft(const double* __restrict__ bank,
                                                               const int* __restrict__ prow,
                                                               const float2* __restrict__ GH, int M,
                                                               double* __restrict__ dpart) {
  mgb_pdl_entry();
  extern __shared__ __align__(16) unsigned char dsm[];
  float2* s = reinterpret_cast<float2*>(dsm);
  __shared__ float hann[MGB_REV_NFFT];  // periodic Hann(384)
  const int m0 = blockIdx.x * RV_F, m0f = m0, b = blockIdx.y;
  const float2* g = GH + (size_t)b * M;
  for (int i = threadIdx.x; i < MGB_REV_NFFT; i += RV_NT)
    hann[i] = 0.5f - 0.5f * cospif(2.f * (float)i / (float)MGB_REV_NFFT);
  __syncthreads();
  int f = 0, i = threadIdx.x;  // (f, i) = divmod(q, 384), stepped
  for (int q = threadIdx.x; q < RV_F * MGB_REV_NFFT; q += RV_NT, i += RV_NT) {
    while (i >= MGB_REV_NFFT) i -= MGB_REV_NFFT, ++f;
    const int t = (m0 + f) * MGB_REV_HOP + i - MGB_REV_HOP;  // position in the sliced FIR
    float dm = 0.f, ds = 0.f;
    if (m0 + f < MGB_REV_FRAMES && t >= 0 && t < MGB_REV_LEN) {
      const float2 v = g[t];
      const float iw = g_rev_inv_wss[t] * hann[i];
      dm = 0.5f * (v.x + v.y) * iw;
      ds = 0.5f * (v.x - v.y) * iw;
    }
    s[f * RV_FRAME + (i >> 7) * RV_P + pidx<true>(i & 127)] = make_float2(dm, ds);
  }
  dft384(s, false);
  const double* p = bank + (size_t)prow[b] * 768;
  const float sc = 2.f / (float)MGB_REV_NFFT;
  // per (bin k, channel): this CTA's sums over its RV_F frames of dexpo and m * dexpo
  double* out = dpart + ((size_t)b * gridDim.x + blockIdx.x) * 2 * MGB_REV_BINS * 2;
  for (int k = threadIdx.x; k < MGB_REV_BINS; k += RV_NT) {
    const int kn = (MGB_REV_NFFT - k) % MGB_REV_NFFT;
    const int kk = k < MGB_REV_PBINS ? k : MGB_REV_PBINS - 1;
    const double h0m = p[kk], hdm = p[192 + kk], h0s = p[384 + kk], hds = p[576 + kk];
    const float scale = (k == 0 || k == MGB_REV_PBINS) ? 0.5f * sc : sc;
    double m0 = 0.0, m1 = 0.0, s0 = 0.0, s1 = 0.0;
    for (int f = 0; f < RV_F; ++f) {
      const int m = m0f + f;
      if (m >= MGB_REV_FRAMES) break;
      // output index k = k1 + 3 k2 lives at row k1, column k2
      const float2 zk = s[f * RV_FRAME + (k % 3) * RV_P + pidx<true>(k / 3)];
      const float2 zp = s[f * RV_FRAME + (kn % 3) * RV_P + pidx<true>(kn / 3)];
      // split the packed spectrum: Dm = (Zk + conj Zp)/2, Ds = (Zk - conj Zp)/(2i)
      const float2 dmx = make_float2(0.5f * (zk.x + zp.x), 0.5f * (zk.y - zp.y));
      const float2 dd = make_float2(0.5f * (zk.x - zp.x), 0.5f * (zk.y + zp.y));
      const float2 dsx = make_float2(dd.y, -dd.x);
      const float mm = expf((float)(h0m + hdm * (double)m));
      const float ms = expf((float)(h0s + hds * (double)m));
      const float2 sm = g_rev_spec[0][m][k], ss = g_rev_spec[1][m][k];
      const double vm = (double)(scale * (dmx.x * sm.x + dmx.y * sm.y) * mm);
      const double vs = (double)(scale * (dsx.x * ss.x + dsx.y * ss.y) * ms);
      m0 += vm;
      m1 += vm * (double)m;
      s0 += vs;
      s1 += vs * (double)m;
    }
    out[(0 * MGB_REV_BINS + k) * 2] = m0;
    out[(0 * MGB_REV_BINS + k) * 2 + 1] = m1;
    out[(1 * MGB_REV_BINS + k) * 2] = s0;
    out[(1 * MGB_REV_BINS + k) * 2 + 1] = s1;
  }
}
