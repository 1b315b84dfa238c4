// Equalizer level by overlap-save in shared memory (included by conv.cu).
//
// ybar[n] = sum_t h[t] x[n + 1023 - t]  (2047-tap zero-phase FIR, offset 1023,
// mg/processors.py:115-120 via mg/engine.py:549-585).  Output block
// [n0, n0 + HOP) with HOP = 8192 - 2046 needs the input window
// xw[i] = x[n0 - 1023 + i], i < 8192, and ybar[n0 + j] = (xw (*) h)[2046 + j]
// (8192-point circular convolution, no wrap).  Both channels ride one complex
// transform (h is real and shared, so Y = Z H needs no pairing).
//
// Backward per block (one CTA, two 8192-point buffers):
//   d window  dw[i] = dybar[n0 - 1023 + i] computed on the fly from
//             (gy, ybar) = w gy + gain-staging term;
//   gx[n0+j]  = (dw corr h)[j]           -> gu = (1-w) gy + gain-staging + gx, one write
//   gh part   = sum_{n in block} dybar[n] x[n + 1023 - t]
//             = IDFT( conj(FFT(dw masked to the block)) . FFT(xw) )[(1023 - t) mod 8192]
//   the per-block cross spectra are summed per node by k_eqos_gh (float64) and
//   one inverse FFT gives dh, consumed by the existing FIR adjoint k_eq_fir_bwd.
#pragma once

constexpr int EOS_N = 8192;
constexpr int EOS_OFF = (MGB_EQ_LEN - 1) / 2;        // 1023
constexpr int EOS_HOP = EOS_N - (MGB_EQ_LEN - 1);    // 6146
constexpr int EOS_NT = 512;
constexpr int EOS_P = padded_len<EOS_N>();
constexpr int kEosSmem1 = EOS_P * 8;
constexpr int kEosSmem2 = 2 * EOS_P * 8;
constexpr int EOS_PER = EOS_N / EOS_NT;              // 16 window elements per thread
constexpr int EOS_OUT = (EOS_HOP + EOS_NT - 1) / EOS_NT;  // 13 outputs per thread

int eos_nblk(int L) { return (L + EOS_HOP - 1) / EOS_HOP; }

// H = FFT_8192(h) per node, natural order
__global__ void __launch_bounds__(EOS_NT) k_eqos_hspec(const float2* __restrict__ hbuf, float2* __restrict__ Hs) {
  extern __shared__ __align__(16) unsigned char dsm[];
  float2* s = reinterpret_cast<float2*>(dsm);
  const int b = blockIdx.x;
  for (int i = threadIdx.x; i < EOS_N; i += EOS_NT)
    s[pidx<true>(i)] = make_float2(i < MGB_EQ_LEN ? hbuf[(size_t)b * MGB_EQ_LEN + i].x : 0.f, 0.f);
  smem_fft<float, EOS_N, 1, EOS_NT, EOS_P, 1, false, true>(s, false);
  for (int i = threadIdx.x; i < EOS_N; i += EOS_NT) Hs[(size_t)b * EOS_N + i] = s[pidx<true>(i)];
}

__global__ void __launch_bounds__(EOS_NT) k_eqos_fwd(const float* const* __restrict__ u_rows,
                                                     const float2* __restrict__ Hs, const int* __restrict__ widx,
                                                     const double* __restrict__ w, float* __restrict__ y,
                                                     float* __restrict__ ybar, double* __restrict__ part, int L) {
  extern __shared__ __align__(16) unsigned char dsm[];
  float2* s = reinterpret_cast<float2*>(dsm);
  __shared__ double red[32];
  const int blk = blockIdx.x, b = blockIdx.y;
  const float* u = u_rows[b];
  const long long n0 = (long long)blk * EOS_HOP, w0 = n0 - EOS_OFF;
  {
    float2 v[EOS_PER];
#pragma unroll
    for (int k = 0; k < EOS_PER; ++k) {
      const long long n = w0 + threadIdx.x + EOS_NT * k;
      v[k] = (n >= 0 && n < L) ? make_float2(__ldg(u + n), __ldg(u + L + n)) : make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int k = 0; k < EOS_PER; ++k) s[pidx<true>(threadIdx.x + EOS_NT * k)] = v[k];
  }
  smem_fft<float, EOS_N, 1, EOS_NT, EOS_P, 1, false, true>(s, false);
  const float2* H = Hs + (size_t)b * EOS_N;
  const float sc = 1.f / (float)EOS_N;
#pragma unroll 4
  for (int k = 0; k < EOS_PER; ++k) {
    const int i = threadIdx.x + EOS_NT * k;
    const float2 h = __ldg(H + i);
    const float2 z = s[pidx<true>(i)];
    s[pidx<true>(i)] = make_float2(sc * (z.x * h.x - z.y * h.y), sc * (z.x * h.y + z.y * h.x));
  }
  smem_fft<float, EOS_N, 1, EOS_NT, EOS_P, 1, false, true>(s, true);
  const double wv = w ? w[widx[b]] : 1.0;
  const float wf = (float)wv, om = (float)(1.0 - wv);
  const bool bypass = wv == 0.0;
  float* yo = y + (size_t)b * 2 * L;
  float* yb = ybar + (size_t)b * 2 * L;
  float2 uu[EOS_OUT];
#pragma unroll
  for (int k = 0; k < EOS_OUT; ++k) {
    const int j = threadIdx.x + EOS_NT * k;
    const long long n = n0 + j;
    uu[k] = (j < EOS_HOP && n < L) ? make_float2(__ldg(u + n), __ldg(u + L + n)) : make_float2(0.f, 0.f);
  }
  float su = 0.f, sy = 0.f;
#pragma unroll
  for (int k = 0; k < EOS_OUT; ++k) {
    const int j = threadIdx.x + EOS_NT * k;
    const long long n = n0 + j;
    if (j < EOS_HOP && n < L) {
      const float2 v = s[pidx<true>(EOS_N - EOS_HOP + j)];
      yb[n] = v.x;
      yb[L + n] = v.y;
      if (bypass) {
        yo[n] = uu[k].x;
        yo[L + n] = uu[k].y;
      } else {
        yo[n] = wf * v.x + om * uu[k].x;
        yo[L + n] = wf * v.y + om * uu[k].y;
      }
      const float mu = uu[k].x + uu[k].y, my = v.x + v.y;
      su = fmaf(mu, mu, su);
      sy = fmaf(my, my, sy);
    }
  }
  const double tu = block_sum((double)su, red);
  __syncthreads();
  const double ty = block_sum((double)sy, red);
  if (threadIdx.x == 0) {
    double* pp = part + ((size_t)b * kMaxParts + blk) * 4;
    pp[0] = tu;
    pp[1] = ty;
  }
}

__global__ void __launch_bounds__(EOS_NT) k_eqos_bwd(const float* const* __restrict__ u_rows,
                                                     const float* const* __restrict__ gy_rows,
                                                     const float* __restrict__ ybar, const float2* __restrict__ Hs,
                                                     const int* __restrict__ widx, const double* __restrict__ w,
                                                     const double* __restrict__ greg,
                                                     const double* __restrict__ stats, float* __restrict__ gu,
                                                     double* __restrict__ part, float2* __restrict__ pspec,
                                                     int L, int nblk) {
  extern __shared__ __align__(16) unsigned char dsm[];
  float2* A = reinterpret_cast<float2*>(dsm);  // full d window, then xw
  float2* Bm = A + EOS_P;                       // d window masked to this block
  __shared__ double red[32];
  const int blk = blockIdx.x, b = blockIdx.y;
  const float* u = u_rows[b];
  const float* gy = gy_rows[b];
  const float* yb = ybar + (size_t)b * 2 * L;
  const long long n0 = (long long)blk * EOS_HOP, w0 = n0 - EOS_OFF;
  const double wv = w ? w[widx[b]] : 1.0;
  const bool bypass = wv == 0.0;
  const float wf = bypass ? 0.f : (float)wv, om = (float)(1.0 - wv);
  const double sg = stats[b * 4 + 2] * (greg ? *greg : 0.0);
  const double nu = stats[b * 4], ny = stats[b * 4 + 1];
  const float cy = (ny > 0.0) ? (float)(sg / ((ny + MGB_GS_EPS) * ny)) : 0.f;
  const float cu = (nu > 0.0) ? (float)(-sg / ((nu + MGB_GS_EPS) * nu)) : 0.f;
  // 1. dybar window (full) and its block-masked copy
#pragma unroll 1
  for (int k0 = 0; k0 < EOS_PER; k0 += 8) {
    float4 g[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const long long n = w0 + threadIdx.x + EOS_NT * (k0 + k);
      g[k] = (n >= 0 && n < L) ? make_float4(__ldg(gy + n), __ldg(gy + L + n), __ldg(yb + n), __ldg(yb + L + n))
                               : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int i = threadIdx.x + EOS_NT * (k0 + k);
      const float my = g[k].z + g[k].w;
      const float2 d = make_float2(fmaf(cy, my, wf * g[k].x), fmaf(cy, my, wf * g[k].y));
      const long long n = w0 + i;
      A[pidx<true>(i)] = d;
      const bool inblk = i >= EOS_OFF && i < EOS_OFF + EOS_HOP && n < L;
      Bm[pidx<true>(i)] = inblk ? d : make_float2(0.f, 0.f);
    }
  }
  smem_fft<float, EOS_N, 2, EOS_NT, EOS_P, 1, false, true>(A, false);
  // 2. gx = IDFT(D conj(H)) over the block, fused with the dry/wet + gain-staging prologue
  const float2* H = Hs + (size_t)b * EOS_N;
  const float sc = 1.f / (float)EOS_N;
#pragma unroll 4
  for (int k = 0; k < EOS_PER; ++k) {
    const int i = threadIdx.x + EOS_NT * k;
    const float2 h = __ldg(H + i);
    const float2 z = A[pidx<true>(i)];
    A[pidx<true>(i)] = make_float2(sc * (z.x * h.x + z.y * h.y), sc * (z.y * h.x - z.x * h.y));
  }
  smem_fft<float, EOS_N, 1, EOS_NT, EOS_P, 1, false, true>(A, true);
  float* go = gu + (size_t)b * 2 * L;
  float fw = 0.f;
  {
    float4 gq[EOS_OUT];
    float4 uq[EOS_OUT];
#pragma unroll
    for (int k = 0; k < EOS_OUT; ++k) {
      const int j = threadIdx.x + EOS_NT * k;
      const long long n = n0 + j;
      const bool in = j < EOS_HOP && n < L;
      gq[k] = in ? make_float4(__ldg(gy + n), __ldg(gy + L + n), __ldg(yb + n), __ldg(yb + L + n))
                 : make_float4(0.f, 0.f, 0.f, 0.f);
      uq[k] = in ? make_float4(__ldg(u + n), __ldg(u + L + n), 0.f, 0.f) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int k = 0; k < EOS_OUT; ++k) {
      const int j = threadIdx.x + EOS_NT * k;
      const long long n = n0 + j;
      if (j < EOS_HOP && n < L) {
        const float2 gx = A[pidx<true>(j)];
        const float mu = uq[k].x + uq[k].y;
        const float ul = bypass ? gq[k].x : om * gq[k].x, ur = bypass ? gq[k].y : om * gq[k].y;
        go[n] = fmaf(cu, mu, ul) + gx.x;
        go[L + n] = fmaf(cu, mu, ur) + gx.y;
        if (!bypass) fw = fmaf(gq[k].x, gq[k].z - uq[k].x, fmaf(gq[k].y, gq[k].w - uq[k].y, fw));
      }
    }
  }
  const double tw = block_sum((double)fw, red);
  if (threadIdx.x == 0) part[((size_t)b * kMaxParts + blk) * 4 + 2] = tw;
  // 3. xw and the cross spectrum  sum_c conj(D'_c) XW_c  (Hermitian pairing on both)
  {
    float2 v[EOS_PER];
#pragma unroll
    for (int k = 0; k < EOS_PER; ++k) {
      const long long n = w0 + threadIdx.x + EOS_NT * k;
      v[k] = (n >= 0 && n < L) ? make_float2(__ldg(u + n), __ldg(u + L + n)) : make_float2(0.f, 0.f);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < EOS_PER; ++k) A[pidx<true>(threadIdx.x + EOS_NT * k)] = v[k];
  }
  smem_fft<float, EOS_N, 1, EOS_NT, EOS_P, 1, false, true>(A, false);
  float2* ps = pspec + ((size_t)b * nblk + blk) * (EOS_N / 2 + 1);
  for (int k = threadIdx.x; k <= EOS_N / 2; k += EOS_NT) {
    const int p = (EOS_N - k) & (EOS_N - 1);
    float2 dl, dr, xl, xr;
    fs::split_pair(Bm[pidx<true>(k)], Bm[pidx<true>(p)], dl, dr);
    fs::split_pair(A[pidx<true>(k)], A[pidx<true>(p)], xl, xr);
    const float2 c1 = cmulc(xl, dl), c2 = cmulc(xr, dr);  // X conj(D)
    ps[k] = make_float2(c1.x + c2.x, c1.y + c2.y);
  }
}

// dh[t] = (1/N) IDFT( sum_blocks P )[(1023 - t) mod N], P Hermitian (real correlation)
__global__ void __launch_bounds__(EOS_NT) k_eqos_gh(const float2* __restrict__ pspec, int nblk,
                                                    float2* __restrict__ ghbuf) {
  extern __shared__ __align__(16) unsigned char dsm[];
  float2* s = reinterpret_cast<float2*>(dsm);
  const int b = blockIdx.x;
  const float2* ps = pspec + (size_t)b * nblk * (EOS_N / 2 + 1);
  for (int k = threadIdx.x; k <= EOS_N / 2; k += EOS_NT) {
    double re = 0.0, im = 0.0;
    for (int q = 0; q < nblk; ++q) {
      const float2 v = ps[(size_t)q * (EOS_N / 2 + 1) + k];
      re += v.x;
      im += v.y;
    }
    const float2 v = make_float2((float)re, (float)im);
    s[pidx<true>(k)] = v;
    if (k != 0 && k != EOS_N / 2) s[pidx<true>(EOS_N - k)] = make_float2(v.x, -v.y);
  }
  smem_fft<float, EOS_N, 1, EOS_NT, EOS_P, 1, false, true>(s, true);
  const float sc = 1.f / (float)EOS_N;
  for (int t = threadIdx.x; t < MGB_EQ_LEN; t += EOS_NT) {
    const int sidx = (EOS_OFF - t) & (EOS_N - 1);
    ghbuf[(size_t)b * MGB_EQ_LEN + t] = make_float2(sc * s[pidx<true>(sidx)].x, 0.f);
  }
}
