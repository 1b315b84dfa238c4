// Fused four-step FFT-convolution building blocks (sm_100a).
//
// N = N1 * N2 complex points.  A signal index is n = n1*N2 + n2, a spectral
// index k = k1 + N1*k2.  Spectra are never transposed to natural order: they
// stay in "row layout" (element (k1, k2) at k1*N2 + k2), which is all the
// pointwise products need.  One forward transform = column pass (k_colA:
// N1-point FFTs down the columns + twiddle w_N^{k1 n2}) followed by row FFTs;
// one inverse = row IFFTs + conj twiddle, then column IFFTs (k_colC).  The row
// work of a convolution's forward and inverse transforms is fused in one
// kernel (k_rowB_*), which also owns the Hermitian pairing: the partner of
// (k1, k2), i.e. spectral index N - k, is (N1 - k1, N2 - 1 - k2) for k1 > 0
// and (0, (N2 - k2) mod N2) for k1 = 0 — so a CTA that holds rows k1 and
// N1 - k1 can split the packed stereo spectrum (left + i*right) locally.
//
// Column passes take a Loader (what to transform: packed input rows, a
// compact FIR, or the backward prologue computed on the fly) and an Epilogue
// (what to do with the time-domain result: dry/wet + gain-staging partials,
// gradient accumulation, FIR-gradient extraction), so every HBM sweep carries
// useful work.
#pragma once
#include "common.cuh"

namespace fs {

template <int N1, int N2>
struct Geo {
  static constexpr int TC = (N1 >= 1024) ? 8 : 16;  // columns per column-pass CTA
  static constexpr int NTC = 256;
  static constexpr int NTR = (N2 >= 2048) ? 512 : 256;
  static constexpr int P = padded_len<N2>();        // padded row pitch in the row kernel
  static constexpr int LOG = __builtin_ctz(N1) + __builtin_ctz(N2);
  static constexpr long long N = (long long)N1 * N2;
};

__device__ __forceinline__ void split_pair(float2 zk, float2 zp, float2& a, float2& b) {
  a = make_float2(0.5f * (zk.x + zp.x), 0.5f * (zk.y - zp.y));
  const float2 d = make_float2(0.5f * (zk.x - zp.x), 0.5f * (zk.y + zp.y));
  b = make_float2(d.y, -d.x);
}

// ---------------------------------------------------------------------------
// column pass, forward direction: A[b][k1*N2 + n2] = w_N^{k1 n2} * FFT_{N1}(x[. * N2 + n2])
template <int N1, int N2, class Ld>
__global__ void __launch_bounds__(Geo<N1, N2>::NTC) k_colA(Ld ld, float2* __restrict__ A, int nz_rows) {
  constexpr int TC = Geo<N1, N2>::TC, NT = Geo<N1, N2>::NTC;
  constexpr long long N = Geo<N1, N2>::N;
  extern __shared__ __align__(16) unsigned char smraw[];
  float2* sm = reinterpret_cast<float2*>(smraw);  // [N1][TC]
  __shared__ double red[32];
  const int b = blockIdx.y;
  const int c0 = blockIdx.x * TC;
  float acc = 0.f;
  for (int i = threadIdx.x; i < TC * N1; i += NT) {
    const int c = i % TC, n1 = i / TC;
    sm[i] = (n1 < nz_rows) ? ld.load(b, (long long)n1 * N2 + c0 + c, acc) : make_float2(0.f, 0.f);
  }
  if (Ld::kAccum) {
    const double t = block_sum((double)acc, red);
    if (threadIdx.x == 0) ld.commit(b, blockIdx.x, t);
  }
  smem_fft<float, N1, TC, NT, 1, TC, true>(sm, false);
  float2* dst = A + (long long)b * N;
  for (int i = threadIdx.x; i < TC * N1; i += NT) {
    const int c = i % TC, k1 = i / TC;
    dst[(long long)k1 * N2 + c0 + c] = cmul(sm[i], fs_twiddle<Geo<N1, N2>::LOG>(k1 * (c0 + c), false));
  }
}

// column pass, inverse direction: y[b][n1*N2 + n2] = scale * IFFT_{N1}(B[. * N2 + n2]); epilogue consumes y
template <int N1, int N2, class Ep>
__global__ void __launch_bounds__(Geo<N1, N2>::NTC) k_colC(const float2* __restrict__ Bb, Ep ep, float scale,
                                                          int out_rows) {
  constexpr int TC = Geo<N1, N2>::TC, NT = Geo<N1, N2>::NTC;
  constexpr long long N = Geo<N1, N2>::N;
  extern __shared__ __align__(16) unsigned char smraw[];
  float2* sm = reinterpret_cast<float2*>(smraw);
  __shared__ double red[32];
  const int b = blockIdx.y;
  const int c0 = blockIdx.x * TC;
  const float2* src = Bb + (long long)b * N;
  for (int i = threadIdx.x; i < TC * N1; i += NT) {
    const int c = i % TC, k1 = i / TC;
    sm[i] = src[(long long)k1 * N2 + c0 + c];
  }
  smem_fft<float, N1, TC, NT, 1, TC, true>(sm, true);
  float a0 = 0.f, a1 = 0.f;
  for (int i = threadIdx.x; i < TC * out_rows; i += NT) {
    const int c = i % TC, n1 = i / TC;
    float2 v = sm[i];
    v.x *= scale;
    v.y *= scale;
    ep.store(b, (long long)n1 * N2 + c0 + c, v, a0, a1);
  }
  if (Ep::kAccum) {
    const double t0 = block_sum((double)a0, red);
    __syncthreads();
    const double t1 = block_sum((double)a1, red);
    if (threadIdx.x == 0) ep.commit(b, blockIdx.x, t0, t1);
  }
}

// ---------------------------------------------------------------------------
// row kernel, forward convolution: rows (r, N1-r) of X and H are FFT'd, stored
// (row layout) for the backward, multiplied pairwise (Q = X_l H_l + i X_r H_r),
// inverse-FFT'd along the rows, conj-twiddled and written to Bo.
template <int N1, int N2>
__global__ void __launch_bounds__(Geo<N1, N2>::NTR) k_rowB_fwd(const float2* __restrict__ Ax,
                                                              const float2* __restrict__ Ah,
                                                              float2* __restrict__ X, float2* __restrict__ H,
                                                              float2* __restrict__ Bo) {
  constexpr int NT = Geo<N1, N2>::NTR, P = Geo<N1, N2>::P;
  constexpr long long N = Geo<N1, N2>::N;
  extern __shared__ __align__(16) unsigned char smraw[];
  float2* s = reinterpret_cast<float2*>(smraw);  // 4 rows: x0, x1, h0, h1
  const int r = blockIdx.x, b = blockIdx.y;
  const int row[2] = {r, (N1 - r) % N1};
  const int nr = (row[0] == row[1]) ? 1 : 2;
  const long long base = (long long)b * N;
  for (int i = threadIdx.x; i < 2 * N2; i += NT) {
    const int q = i / N2, k = i % N2;
    const int rr = row[q < nr ? q : 0];
    s[q * P + pidx<true>(k)] = Ax[base + (long long)rr * N2 + k];
    s[(2 + q) * P + pidx<true>(k)] = Ah[base + (long long)rr * N2 + k];
  }
  smem_fft<float, N2, 4, NT, P, 1, false, true>(s, false);
  for (int i = threadIdx.x; i < nr * N2; i += NT) {
    const int q = i / N2, k = i % N2;
    X[base + (long long)row[q] * N2 + k] = s[q * P + pidx<true>(k)];
    H[base + (long long)row[q] * N2 + k] = s[(2 + q) * P + pidx<true>(k)];
  }
  constexpr int PER = (2 * N2 + NT - 1) / NT;
  float2 qv[PER];
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int i = threadIdx.x + j * NT;
    if (i < nr * N2) {
      const int q = i / N2, k = i % N2;
      int qp, kp;
      if (nr == 2) { qp = 1 - q; kp = N2 - 1 - k; }
      else { qp = 0; kp = (row[0] == 0) ? ((N2 - k) & (N2 - 1)) : (N2 - 1 - k); }
      float2 xl, xr, hl, hr;
      split_pair(s[q * P + pidx<true>(k)], s[qp * P + pidx<true>(kp)], xl, xr);
      split_pair(s[(2 + q) * P + pidx<true>(k)], s[(2 + qp) * P + pidx<true>(kp)], hl, hr);
      const float2 y1 = cmul(xl, hl), y2 = cmul(xr, hr);
      qv[j] = make_float2(y1.x - y2.y, y1.y + y2.x);
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int i = threadIdx.x + j * NT;
    if (i < nr * N2) s[(i / N2) * P + pidx<true>(i % N2)] = qv[j];
  }
  smem_fft<float, N2, 2, NT, P, 1, false, true>(s, true);
  for (int i = threadIdx.x; i < nr * N2; i += NT) {
    const int q = i / N2, n2 = i % N2;
    const float2 w = fs_twiddle<Geo<N1, N2>::LOG>(row[q] * n2, true);
    Bo[base + (long long)row[q] * N2 + n2] = cmul(s[q * P + pidx<true>(n2)], w);
  }
}

// row kernel, backward: G rows FFT'd; GX = G conj(H), GH = G conj(X) paired;
// both inverse-FFT'd along rows, conj-twiddled, written to B1 (gx) and B2 (gh).
template <int N1, int N2>
__global__ void __launch_bounds__(Geo<N1, N2>::NTR) k_rowB_bwd(const float2* __restrict__ Ag,
                                                              const float2* __restrict__ X,
                                                              const float2* __restrict__ H,
                                                              float2* __restrict__ B1, float2* __restrict__ B2) {
  constexpr int NT = Geo<N1, N2>::NTR, P = Geo<N1, N2>::P;
  constexpr long long N = Geo<N1, N2>::N;
  extern __shared__ __align__(16) unsigned char smraw[];
  float2* s = reinterpret_cast<float2*>(smraw);  // g0, g1 then gx0, gx1, gh0, gh1
  const int r = blockIdx.x, b = blockIdx.y;
  const int row[2] = {r, (N1 - r) % N1};
  const int nr = (row[0] == row[1]) ? 1 : 2;
  const long long base = (long long)b * N;
  for (int i = threadIdx.x; i < 2 * N2; i += NT) {
    const int q = i / N2, k = i % N2;
    s[q * P + pidx<true>(k)] = Ag[base + (long long)row[q < nr ? q : 0] * N2 + k];
  }
  smem_fft<float, N2, 2, NT, P, 1, false, true>(s, false);
  constexpr int PER = (2 * N2 + NT - 1) / NT;
  float2 gx[PER], gh[PER];
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int i = threadIdx.x + j * NT;
    if (i < nr * N2) {
      const int q = i / N2, k = i % N2;
      int qp, kp;
      if (nr == 2) { qp = 1 - q; kp = N2 - 1 - k; }
      else { qp = 0; kp = (row[0] == 0) ? ((N2 - k) & (N2 - 1)) : (N2 - 1 - k); }
      const long long ik = base + (long long)row[q] * N2 + k, ip = base + (long long)row[qp] * N2 + kp;
      float2 gl, gr, hl, hr, xl, xr;
      split_pair(s[q * P + pidx<true>(k)], s[qp * P + pidx<true>(kp)], gl, gr);
      split_pair(H[ik], H[ip], hl, hr);
      split_pair(X[ik], X[ip], xl, xr);
      float2 y1 = cmulc(gl, hl), y2 = cmulc(gr, hr);
      gx[j] = make_float2(y1.x - y2.y, y1.y + y2.x);
      y1 = cmulc(gl, xl);
      y2 = cmulc(gr, xr);
      gh[j] = make_float2(y1.x - y2.y, y1.y + y2.x);
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int i = threadIdx.x + j * NT;
    if (i < nr * N2) {
      s[(i / N2) * P + pidx<true>(i % N2)] = gx[j];
      s[(2 + i / N2) * P + pidx<true>(i % N2)] = gh[j];
    }
  }
  smem_fft<float, N2, 4, NT, P, 1, false, true>(s, true);
  for (int i = threadIdx.x; i < nr * N2; i += NT) {
    const int q = i / N2, n2 = i % N2;
    const float2 w = fs_twiddle<Geo<N1, N2>::LOG>(row[q] * n2, true);
    B1[base + (long long)row[q] * N2 + n2] = cmul(s[q * P + pidx<true>(n2)], w);
    B2[base + (long long)row[q] * N2 + n2] = cmul(s[(2 + q) * P + pidx<true>(n2)], w);
  }
}

template <int N1, int N2>
constexpr size_t col_smem() { return sizeof(float2) * Geo<N1, N2>::TC * N1; }
template <int N1, int N2>
constexpr size_t row_smem() { return sizeof(float2) * 4 * Geo<N1, N2>::P; }

}  // namespace fs
