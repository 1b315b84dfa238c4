// Equalizer level by overlap-save with register-resident 8192-point FFTs
// (included by conv.cu).
//
// ybar[n] = sum_t h[t] x[n + 1023 - t]  (2047-tap zero-phase FIR, offset 1023,
// mg/processors.py:115-120 via mg/engine.py:549-585).  Output block
// [n0, n0 + HOP) with HOP = 8192 - 2046 needs the input window
// xw[i] = x[n0 - 1023 + i], i < 8192, and ybar[n0 + j] = (xw (*) h)[2046 + j]
// (8192-point circular convolution, no wrap).  Both channels ride one complex
// transform (h is real and shared, so Y = Z H needs no pairing).
//
// The 8192-point transform (eos_fft / eos_ifft) runs on 256 threads holding 32
// values each: a 32-point register DFT, one exchange, 2 x 16-point register
// DFTs, one exchange, 2 x 16-point register DFTs (8192 = 32 x 16 x 16).  The
// forward leaves spectra in a fixed thread-private order (thread t, slot r),
// which is exactly the input order of the inverse, so pointwise products
// with a spectrum stored in the same order (Hs[r][t]) need no shuffling.
//
// Backward per block (one CTA):
//   D   = FFT(d window), d = dybar = w gy + gain-staging term (on the fly)
//   gx  = IDFT(D conj H)[j], j < HOP  -> gu = (1-w) gy + gain-staging + gx
//   C   = conj(D) FFT(x masked to the block)      (packed: conj(d_l + i d_r)(x_l + i x_r))
//   dh[t] = Re IDFT(sum_blocks C)[(1023 - t) mod 8192] = sum_c sum_n d_c[n] x_c[n + 1023 - t]
//   (the real part of the packed cross-correlation is the channel sum; the
//   per-block C are reduced in float64 by k_eqos_gh)
#pragma once
#include "regfft.cuh"

constexpr int EOS_N = 8192;
constexpr int EOS_OFF = (MGB_EQ_LEN - 1) / 2;        // 1023
constexpr int EOS_HOP = EOS_N - (MGB_EQ_LEN - 1);    // 6146
constexpr int EOS_NT = 256;
constexpr int EOS_S2P = 17;                          // stage-2 exchange row pitch
constexpr int EOS_SM = 32 * 16 * EOS_S2P;            // 8704 float2 >= 8192
constexpr int kEosSmem1 = EOS_SM * 8;

int eos_nblk(int L) { return (L + EOS_HOP - 1) / EOS_HOP; }
// backward blocks per CTA: about two CTAs per SM over the level (B nodes)
int eos_per(int L, int B) {
  const int n = eos_nblk(L) * B, per = (n + 2 * 148 - 1) / (2 * 148);
  return per < 1 ? 1 : per;
}
int eos_nchunk(int L, int B) { return (eos_nblk(L) + eos_per(L, B) - 1) / eos_per(L, B); }

// natural order (thread t holds x[t + 256 m]) -> spectrum in (t, r) order:
// v[s*16 + ka] = X[k1 + 32 kb + 512 ka], k1 = (t >> 4) + 16 s, kb = t & 15
__device__ __forceinline__ void eos_fft(float2 (&v)[32], float2* S) {
  const int t = threadIdx.x, lo = t & 15, kq = t >> 4;
  rf::rdft<32, false>(v);
  fs2::twiddle_run<13, 32, false>(v, 0, t);
#pragma unroll
  for (int k1 = 0; k1 < 32; ++k1) S[k1 * 256 + t] = v[k1];
  __syncthreads();
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int k1 = kq + 16 * s;
    float2 u[16];
#pragma unroll
    for (int tb = 0; tb < 16; ++tb) u[tb] = S[k1 * 256 + lo + 16 * tb];
    rf::rdft<16, false>(u);
    fs2::twiddle_run<8, 16, false>(u, 0, lo);
#pragma unroll
    for (int kb = 0; kb < 16; ++kb) v[s * 16 + kb] = u[kb];
  }
  __syncthreads();
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int k1 = kq + 16 * s;
#pragma unroll
    for (int kb = 0; kb < 16; ++kb) S[k1 * 16 * EOS_S2P + kb * EOS_S2P + lo] = v[s * 16 + kb];
  }
  __syncthreads();
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int k1 = kq + 16 * s;
    float2 u[16];
#pragma unroll
    for (int ta = 0; ta < 16; ++ta) u[ta] = S[k1 * 16 * EOS_S2P + lo * EOS_S2P + ta];
    rf::rdft<16, false>(u);
#pragma unroll
    for (int ka = 0; ka < 16; ++ka) v[s * 16 + ka] = u[ka];
  }
  __syncthreads();
}

// (t, r) spectrum order -> natural order, unnormalised inverse
__device__ __forceinline__ void eos_ifft(float2 (&v)[32], float2* S) {
  const int t = threadIdx.x, lo = t & 15, kq = t >> 4;
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int k1 = kq + 16 * s;
    float2 u[16];
#pragma unroll
    for (int ka = 0; ka < 16; ++ka) u[ka] = v[s * 16 + ka];
    rf::rdft<16, true>(u);
#pragma unroll
    for (int ta = 0; ta < 16; ++ta) S[k1 * 16 * EOS_S2P + lo * EOS_S2P + ta] = u[ta];
  }
  __syncthreads();
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int k1 = kq + 16 * s;
    float2 u[16];
#pragma unroll
    for (int kb = 0; kb < 16; ++kb) u[kb] = S[k1 * 16 * EOS_S2P + kb * EOS_S2P + lo];
    fs2::twiddle_run<8, 16, true>(u, 0, lo);
    rf::rdft<16, true>(u);
#pragma unroll
    for (int tb = 0; tb < 16; ++tb) v[s * 16 + tb] = u[tb];
  }
  __syncthreads();
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    const int k1 = kq + 16 * s;
#pragma unroll
    for (int tb = 0; tb < 16; ++tb) S[k1 * 256 + lo + 16 * tb] = v[s * 16 + tb];
  }
  __syncthreads();
#pragma unroll
  for (int k1 = 0; k1 < 32; ++k1) v[k1] = S[k1 * 256 + t];
  fs2::twiddle_run<13, 32, true>(v, 0, t);
  rf::rdft<32, true>(v);
  __syncthreads();
}

// H = FFT_8192(h) per node, (t, r) order: Hs[b][r * 256 + t]
__global__ void __launch_bounds__(EOS_NT) k_eqos_hspec(const float2* __restrict__ hbuf, float2* __restrict__ Hs) {
  mgb_pdl_entry();
  extern __shared__ __align__(16) unsigned char dsm[];
  float2* S = reinterpret_cast<float2*>(dsm);
  const int b = blockIdx.x, t = threadIdx.x;
  float2 v[32];
#pragma unroll
  for (int m = 0; m < 32; ++m) {
    const int i = t + 256 * m;
    v[m] = make_float2(i < MGB_EQ_LEN ? hbuf[(size_t)b * MGB_EQ_LEN + i].x : 0.f, 0.f);
  }
  eos_fft(v, S);
#pragma unroll
  for (int r = 0; r < 32; ++r) Hs[(size_t)b * EOS_N + r * 256 + t] = v[r];
}

__global__ void __launch_bounds__(EOS_NT, 2) k_eqos_fwd(const float* const* __restrict__ u_rows,
                                                     const float2* __restrict__ Hs, const int* __restrict__ widx,
                                                     const double* __restrict__ w, float* __restrict__ y,
                                                     float* __restrict__ ybar, double* __restrict__ part, int L) {
  mgb_pdl_entry();
  extern __shared__ __align__(16) unsigned char dsm[];
  float2* S = reinterpret_cast<float2*>(dsm);
  __shared__ double red[32];
  const int blk = blockIdx.x, b = blockIdx.y, t = threadIdx.x;
  const float* u = u_rows[b];
  const long long n0 = (long long)blk * EOS_HOP, w0 = n0 - EOS_OFF;
  float2 v[32];
#pragma unroll
  for (int m = 0; m < 32; ++m) {
    const long long n = w0 + t + 256 * m;
    v[m] = (n >= 0 && n < L) ? make_float2(__ldg(u + n), __ldg(u + L + n)) : make_float2(0.f, 0.f);
  }
  eos_fft(v, S);
  const float2* H = Hs + (size_t)b * EOS_N + t;
  const float sc = 1.f / (float)EOS_N;
#pragma unroll
  for (int r = 0; r < 32; ++r) {
    const float2 h = __ldg(H + r * 256);
    v[r] = make_float2(sc * (v[r].x * h.x - v[r].y * h.y), sc * (v[r].x * h.y + v[r].y * h.x));
  }
  eos_ifft(v, S);
  // window index i = t + 256 m holds ybar[n0 + i - 2046] for i >= 2046
  const double wv = w ? w[widx[b]] : 1.0;
  const float wf = (float)wv, om = (float)(1.0 - wv);
  const bool bypass = wv == 0.0;
  float* yo = y + (size_t)b * 2 * L;
  float* yb = ybar + (size_t)b * 2 * L;
  float su = 0.f, sy = 0.f;
#pragma unroll
  for (int m0 = 7; m0 < 32; m0 += 5) {
    float2 uu[5];
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      const int i = t + 256 * (m0 + q);
      const long long n = n0 + i - (EOS_N - EOS_HOP);
      uu[q] = (m0 + q < 32 && i >= EOS_N - EOS_HOP && n < L) ? make_float2(__ldg(u + n), __ldg(u + L + n))
                                                              : make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int q = 0; q < 5; ++q) {
      const int m = m0 + q;
      if (m >= 32) break;
      const int i = t + 256 * m;
      const long long n = n0 + i - (EOS_N - EOS_HOP);
      if (i >= EOS_N - EOS_HOP && n < L) {
        const float2 vv = v[m];
        yb[n] = vv.x;
        yb[L + n] = vv.y;
        if (bypass) {
          yo[n] = uu[q].x;
          yo[L + n] = uu[q].y;
        } else {
          yo[n] = wf * vv.x + om * uu[q].x;
          yo[L + n] = wf * vv.y + om * uu[q].y;
        }
        const float mu = uu[q].x + uu[q].y, my = vv.x + vv.y;
        su = fmaf(mu, mu, su);
        sy = fmaf(my, my, sy);
      }
    }
  }
  const double tu = block_sum((double)su, red);
  __syncthreads();
  const double ty = block_sum((double)sy, red);
  if (t == 0) {
    double* pp = part + ((size_t)b * kMaxParts + blk) * 4;
    pp[0] = tu;
    pp[1] = ty;
  }
}

__global__ void __launch_bounds__(EOS_NT, 2) k_eqos_bwd(const float* const* __restrict__ u_rows,
                                                     const float* const* __restrict__ gy_rows,
                                                     const float* __restrict__ ybar, const float2* __restrict__ Hs,
                                                     const int* __restrict__ widx, const double* __restrict__ w,
                                                     const double* __restrict__ greg,
                                                     const double* __restrict__ stats, float* __restrict__ gu,
                                                     double* __restrict__ part, float2* __restrict__ pspec,
                                                     int L, int nblk, int per, int passes) {
  mgb_pdl_entry();
  extern __shared__ __align__(16) unsigned char dsm[];
  float2* S = reinterpret_cast<float2*>(dsm);
  __shared__ double red[32];
  // a CTA handles `per` consecutive blocks of one node: its D park and its C
  // accumulator are two 8192-point slots of its own (L2-resident across the blocks),
  // and its dL/dw partial is one slot
  const int chunk = blockIdx.x, b = blockIdx.y, t = threadIdx.x;
  const float* u = u_rows[b];
  const float* gy = gy_rows[b];
  const float* yb = ybar + (size_t)b * 2 * L;
  float2* dpark = pspec + ((size_t)b * gridDim.x + chunk) * 2 * EOS_N + t;
  float2* cacc = dpark + EOS_N;
  float fw = 0.f;
  const int blk_end = min(nblk, (chunk + 1) * per);
#pragma unroll 1
  for (int blk = chunk * per; blk < blk_end; ++blk) {
  const bool first = blk == chunk * per;
  const long long n0 = (long long)blk * EOS_HOP, w0 = n0 - EOS_OFF;
  const double wv = w ? w[widx[b]] : 1.0;
  const bool bypass = wv == 0.0;
  const float wf = bypass ? 0.f : (float)wv, om = (float)(1.0 - wv);
  const double sg = stats[b * 4 + 2] * (greg ? *greg : 0.0);
  const double nu = stats[b * 4], ny = stats[b * 4 + 1];
  const float cy = (ny > 0.0) ? (float)(sg / ((ny + MGB_GS_EPS) * ny)) : 0.f;
  const float cu = (nu > 0.0) ? (float)(-sg / ((nu + MGB_GS_EPS) * nu)) : 0.f;
  float2 v[32];
  // pass 0 input: the d window (dybar)
#pragma unroll
  for (int m0 = 0; m0 < 32; m0 += 4) {
    float4 g[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const long long n = w0 + t + 256 * (m0 + q);
      g[q] = (n >= 0 && n < L) ? make_float4(__ldg(gy + n), __ldg(gy + L + n), __ldg(yb + n), __ldg(yb + L + n))
                               : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float my = g[q].z + g[q].w;
      v[m0 + q] = make_float2(fmaf(cy, my, wf * g[q].x), fmaf(cy, my, wf * g[q].y));
    }
  }
  // pass 0: D = FFT(d) (parked in the CTA's D slot), gx = IDFT(D conj H) -> gu;
  // pass 1: Xm = FFT(x masked to the block), C += conj(D) Xm in the CTA's C slot.  One
  // copy of the forward-transform code serves both passes (instruction-cache footprint).
#pragma unroll 1
  for (int pass = 0; pass < 2; ++pass) {
    eos_fft(v, S);
    if (pass == 1) {
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        const float2 c = cmulc(v[r], dpark[r * 256]);
        if (first) {
          cacc[r * 256] = c;
        } else {
          const float2 a = cacc[r * 256];
          cacc[r * 256] = make_float2(a.x + c.x, a.y + c.y);
        }
      }
      break;
    }
#pragma unroll
    for (int r = 0; r < 32; ++r) dpark[r * 256] = v[r];
    float* go = gu ? gu + (size_t)b * 2 * L : nullptr;  // null: input gradient not requested (no gx transform)
    if (go) {
      const float2* H = Hs + (size_t)b * EOS_N + t;
      const float sc = 1.f / (float)EOS_N;
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        const float2 h = __ldg(H + r * 256);
        v[r] = make_float2(sc * (v[r].x * h.x + v[r].y * h.y), sc * (v[r].y * h.x - v[r].x * h.y));
      }
      eos_ifft(v, S);
    }
#pragma unroll
    for (int m0 = 0; m0 < EOS_HOP / 256 + 1; m0 += 5) {  // window indices i < HOP: m <= 24
      float4 gq[5];
      float2 uq[5];
#pragma unroll
      for (int q = 0; q < 5; ++q) {
        const int i = t + 256 * (m0 + q);
        const long long n = n0 + i;
        const bool in = i < EOS_HOP && n < L;
        gq[q] = in ? make_float4(__ldg(gy + n), __ldg(gy + L + n), __ldg(yb + n), __ldg(yb + L + n))
                   : make_float4(0.f, 0.f, 0.f, 0.f);
        uq[q] = in ? make_float2(__ldg(u + n), __ldg(u + L + n)) : make_float2(0.f, 0.f);
      }
#pragma unroll
      for (int q = 0; q < 5; ++q) {
        const int i = t + 256 * (m0 + q);
        const long long n = n0 + i;
        if (i < EOS_HOP && n < L) {
          if (go) {
            const float2 gx = v[m0 + q];
            const float mu = uq[q].x + uq[q].y;
            const float ul = bypass ? gq[q].x : om * gq[q].x, ur = bypass ? gq[q].y : om * gq[q].y;
            go[n] = fmaf(cu, mu, ul) + gx.x;
            go[L + n] = fmaf(cu, mu, ur) + gx.y;
          }
          if (!bypass) fw = fmaf(gq[q].x, gq[q].z - uq[q].x, fmaf(gq[q].y, gq[q].w - uq[q].y, fw));
        }
      }
    }
    if (passes == 1) break;  // the FIR-gradient pass runs in phase 2 (k_eqos_bwd_c)
    // pass 1 input: x masked to the block
#pragma unroll
    for (int m = 0; m < 32; ++m) {
      const int i = t + 256 * m;
      const long long n = w0 + i;
      v[m] = (i >= EOS_OFF && i < EOS_OFF + EOS_HOP && n < L) ? make_float2(__ldg(u + n), __ldg(u + L + n))
                                                                : make_float2(0.f, 0.f);
    }
  }
  }
  const double tw = block_sum((double)fw, red);
  if (t == 0) part[((size_t)b * kMaxParts + chunk) * 4 + 2] = tw;
}

// The FIR-gradient pass of k_eqos_bwd on its own (narrow levels, one block per CTA:
// backward phase 2, off the critical path): C = conj(D) FFT(x masked to the block),
// D parked by phase 1 in the CTA's slot.
__global__ void __launch_bounds__(EOS_NT, 2) k_eqos_bwd_c(const float* const* __restrict__ u_rows,
                                                       float2* __restrict__ pspec, int L) {
  mgb_pdl_entry();
  extern __shared__ __align__(16) unsigned char dsm[];
  float2* S = reinterpret_cast<float2*>(dsm);
  const int blk = blockIdx.x, b = blockIdx.y, t = threadIdx.x;
  const float* u = u_rows[b];
  float2* dpark = pspec + ((size_t)b * gridDim.x + blk) * 2 * EOS_N + t;
  float2* cacc = dpark + EOS_N;
  const long long w0 = (long long)blk * EOS_HOP - EOS_OFF;
  float2 v[32];
#pragma unroll
  for (int m = 0; m < 32; ++m) {
    const int i = t + 256 * m;
    const long long n = w0 + i;
    v[m] = (i >= EOS_OFF && i < EOS_OFF + EOS_HOP && n < L) ? make_float2(__ldg(u + n), __ldg(u + L + n))
                                                              : make_float2(0.f, 0.f);
  }
  eos_fft(v, S);
#pragma unroll
  for (int r = 0; r < 32; ++r) cacc[r * 256] = cmulc(v[r], dpark[r * 256]);
}

// Csum[b][slot] = sum over the backward CTAs' C accumulators (float64, fixed order)
__global__ void __launch_bounds__(256) k_eqos_csum(const float2* __restrict__ pspec, int nchunk,
                                                   float2* __restrict__ csum) {
  mgb_pdl_entry();
  const int b = blockIdx.y, slot = blockIdx.x * 256 + threadIdx.x;
  const float2* ps = pspec + (size_t)b * nchunk * 2 * EOS_N + EOS_N + slot;
  double re = 0.0, im = 0.0;
#pragma unroll 8
  for (int q = 0; q < nchunk; ++q) {
    const float2 c = __ldg(ps + (size_t)q * 2 * EOS_N);
    re += c.x;
    im += c.y;
  }
  csum[(size_t)b * EOS_N + slot] = make_float2((float)re, (float)im);
}

// dh[t] = Re IDFT(Csum)[(1023 - t) mod N] / N
__global__ void __launch_bounds__(EOS_NT) k_eqos_gh(const float2* __restrict__ csum, float2* __restrict__ ghbuf) {
  mgb_pdl_entry();
  extern __shared__ __align__(16) unsigned char dsm[];
  float2* S = reinterpret_cast<float2*>(dsm);
  const int b = blockIdx.x, t = threadIdx.x;
  float2 v[32];
#pragma unroll
  for (int r = 0; r < 32; ++r) v[r] = csum[(size_t)b * EOS_N + r * 256 + t];
  eos_ifft(v, S);
  const float sc = 1.f / (float)EOS_N;
#pragma unroll
  for (int m = 0; m < 32; ++m) {
    const int i = t + 256 * m;
    const int tt = (EOS_OFF - i) & (EOS_N - 1);
    if (tt < MGB_EQ_LEN) ghbuf[(size_t)b * MGB_EQ_LEN + tt] = make_float2(sc * v[m].x, 0.f);
  }
}
