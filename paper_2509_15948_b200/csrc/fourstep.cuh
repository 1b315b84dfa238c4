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
// useful work.  Loaders/epilogues are split into fetch (global loads only)
// and finish (math + stores) so a thread issues a whole batch of independent
// loads before it stalls: these passes are latency-bound otherwise.
#pragma once
#include "common.cuh"

namespace fs {

template <int N1, int N2>
struct Geo {
  static constexpr int TC = 8;                      // columns per column-pass CTA (64 B row segments)
  static constexpr int NTC = (TC * N1 / 8 >= 256) ? 256 : (TC * N1 / 8 < 32 ? 32 : TC * N1 / 8);
  static constexpr int PERC = TC * N1 / NTC;        // elements per thread in a column tile
  static constexpr int BATCHC = PERC < 8 ? PERC : 8;
  static constexpr int NTR = (N2 >= 2048) ? 512 : 256;
  static constexpr int P = padded_len<N2>();        // padded row pitch in the row kernels
  static constexpr int LOG = __builtin_ctz(N1) + __builtin_ctz(N2);
  static constexpr long long N = (long long)N1 * N2;
};

constexpr int BATCH = 8;  // independent global loads issued per thread before use

__device__ __forceinline__ void split_pair(float2 zk, float2 zp, float2& a, float2& b) {
  a = make_float2(0.5f * (zk.x + zp.x), 0.5f * (zk.y - zp.y));
  const float2 d = make_float2(0.5f * (zk.x - zp.x), 0.5f * (zk.y + zp.y));
  b = make_float2(d.y, -d.x);
}

// ---------------------------------------------------------------------------
// column pass, forward direction: A[b][k1*N2 + n2] = w_N^{k1 n2} * FFT_{N1}(x[. * N2 + n2])
template <int N1, int N2, class Ld>
__global__ void __launch_bounds__(Geo<N1, N2>::NTC, 4) k_colA(Ld ld, float2* __restrict__ A, int nz_rows) {
  mgb_pdl_entry();
  constexpr int TC = Geo<N1, N2>::TC, NT = Geo<N1, N2>::NTC;
  constexpr long long N = Geo<N1, N2>::N;
  constexpr int PER = Geo<N1, N2>::PERC, BATCH = Geo<N1, N2>::BATCHC;
  static_assert(PER % BATCH == 0, "batching");
  extern __shared__ __align__(16) unsigned char smraw[];
  float2* sm = reinterpret_cast<float2*>(smraw);  // [N1][TC]
  __shared__ double red[32];
  const int b = blockIdx.y;
  const int c0 = blockIdx.x * TC;
  const typename Ld::Ctx ctx = ld.prepare(b);
  float acc = 0.f;
#pragma unroll 1
  for (int j0 = 0; j0 < PER; j0 += BATCH) {
    typename Ld::Raw raw[BATCH];
#pragma unroll
    for (int j = 0; j < BATCH; ++j) {
      const int i = threadIdx.x + (j0 + j) * NT;
      const int c = i % TC, n1 = i / TC;
      raw[j] = ld.fetch(ctx, b, (long long)n1 * N2 + c0 + c, n1 < nz_rows);
    }
#pragma unroll
    for (int j = 0; j < BATCH; ++j) {
      const int i = threadIdx.x + (j0 + j) * NT;
      const int c = i % TC, n1 = i / TC;
      sm[i] = ld.finish(ctx, b, (long long)n1 * N2 + c0 + c, raw[j], acc);
    }
  }
  if (Ld::kAccum) {
    const double t = block_sum((double)acc, red);
    if (threadIdx.x == 0) ld.commit(b, blockIdx.x, t);
  }
  smem_fft<float, N1, TC, NT, 1, TC, true>(sm, false);
  float2* dst = A + (long long)b * N;
#pragma unroll 4
  for (int j = 0; j < PER; ++j) {
    const int i = threadIdx.x + j * NT;
    const int c = i % TC, k1 = i / TC;
    dst[(long long)k1 * N2 + c0 + c] = cmul(sm[i], fs_twiddle<Geo<N1, N2>::LOG>(k1 * (c0 + c), false));
  }
}

// column pass, inverse direction: y[b][n1*N2 + n2] = scale * IFFT_{N1}(B[. * N2 + n2]); epilogue consumes y
template <int N1, int N2, class Ep>
__global__ void __launch_bounds__(Geo<N1, N2>::NTC, 4) k_colC(const float2* __restrict__ Bb, Ep ep, float scale,
                                                             int out_rows) {
  mgb_pdl_entry();
  constexpr int TC = Geo<N1, N2>::TC, NT = Geo<N1, N2>::NTC;
  constexpr long long N = Geo<N1, N2>::N;
  constexpr int PER = Geo<N1, N2>::PERC, BATCH = Geo<N1, N2>::BATCHC;
  static_assert(PER % BATCH == 0, "batching");
  extern __shared__ __align__(16) unsigned char smraw[];
  float2* sm = reinterpret_cast<float2*>(smraw);
  __shared__ double red[32];
  const int b = blockIdx.y;
  const int c0 = blockIdx.x * TC;
  const float2* src = Bb + (long long)b * N;
#pragma unroll 1
  for (int j0 = 0; j0 < PER; j0 += BATCH) {
    float2 v[BATCH];
#pragma unroll
    for (int j = 0; j < BATCH; ++j) {
      const int i = threadIdx.x + (j0 + j) * NT;
      v[j] = src[(long long)(i / TC) * N2 + c0 + i % TC];
    }
#pragma unroll
    for (int j = 0; j < BATCH; ++j) sm[threadIdx.x + (j0 + j) * NT] = v[j];
  }
  smem_fft<float, N1, TC, NT, 1, TC, true>(sm, true);
  const typename Ep::Ctx ctx = ep.prepare(b);
  float a0 = 0.f, a1 = 0.f;
  const int nout = TC * out_rows;
#pragma unroll 1
  for (int j0 = 0; j0 < PER; j0 += BATCH) {
    if (threadIdx.x + j0 * NT >= nout) break;
    typename Ep::Raw raw[BATCH];
#pragma unroll
    for (int j = 0; j < BATCH; ++j) {
      const int i = threadIdx.x + (j0 + j) * NT;
      raw[j] = ep.fetch(ctx, b, (long long)(i / TC) * N2 + c0 + i % TC, i < nout);
    }
#pragma unroll
    for (int j = 0; j < BATCH; ++j) {
      const int i = threadIdx.x + (j0 + j) * NT;
      if (i < nout) {
        float2 y = sm[i];
        y.x *= scale;
        y.y *= scale;
        ep.finish(ctx, b, (long long)(i / TC) * N2 + c0 + i % TC, y, raw[j], a0, a1);
      }
    }
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
__global__ void __launch_bounds__(Geo<N1, N2>::NTR, 3) k_rowB_fwd(const float2* __restrict__ Ax,
                                                                 const float2* __restrict__ Ah,
                                                                 float2* __restrict__ X, float2* __restrict__ H,
                                                                 float2* __restrict__ Bo) {
  mgb_pdl_entry();
  constexpr int NT = Geo<N1, N2>::NTR, P = Geo<N1, N2>::P;
  constexpr long long N = Geo<N1, N2>::N;
  constexpr int PER = 2 * N2 / NT;
  extern __shared__ __align__(16) unsigned char smraw[];
  float2* s = reinterpret_cast<float2*>(smraw);  // 4 rows: x0, x1, h0, h1
  const int r = blockIdx.x, b = blockIdx.y;
  const int row[2] = {r, (N1 - r) % N1};
  const int nr = (row[0] == row[1]) ? 1 : 2;
  const long long base = (long long)b * N;
  {
    float2 vx[PER], vh[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int i = threadIdx.x + j * NT, q = i / N2, k = i % N2;
      const long long g = base + (long long)row[q < nr ? q : 0] * N2 + k;
      vx[j] = Ax[g];
      vh[j] = Ah[g];
    }
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int i = threadIdx.x + j * NT, q = i / N2, k = i % N2;
      s[q * P + pidx<true>(k)] = vx[j];
      s[(2 + q) * P + pidx<true>(k)] = vh[j];
    }
  }
  smem_fft<float, N2, 4, NT, P, 1, false, true>(s, false);
  float2 qv[PER];
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int i = threadIdx.x + j * NT;
    const int q = i / N2, k = i % N2;
    if (q < nr) {
      const float2 xk = s[q * P + pidx<true>(k)], hk = s[(2 + q) * P + pidx<true>(k)];
      X[base + (long long)row[q] * N2 + k] = xk;
      H[base + (long long)row[q] * N2 + k] = hk;
      int qp, kp;
      if (nr == 2) { qp = 1 - q; kp = N2 - 1 - k; }
      else { qp = 0; kp = (row[0] == 0) ? ((N2 - k) & (N2 - 1)) : (N2 - 1 - k); }
      float2 xl, xr, hl, hr;
      split_pair(xk, s[qp * P + pidx<true>(kp)], xl, xr);
      split_pair(hk, s[(2 + qp) * P + pidx<true>(kp)], hl, hr);
      const float2 y1 = cmul(xl, hl), y2 = cmul(xr, hr);
      qv[j] = make_float2(y1.x - y2.y, y1.y + y2.x);
    }
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int i = threadIdx.x + j * NT;
    if (i / N2 < nr) s[(i / N2) * P + pidx<true>(i % N2)] = qv[j];
  }
  smem_fft<float, N2, 2, NT, P, 1, false, true>(s, true);
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int i = threadIdx.x + j * NT;
    const int q = i / N2, n2 = i % N2;
    if (q < nr) {
      const float2 w = fs_twiddle<Geo<N1, N2>::LOG>(row[q] * n2, true);
      Bo[base + (long long)row[q] * N2 + n2] = cmul(s[q * P + pidx<true>(n2)], w);
    }
  }
}

// row kernel, backward: G rows FFT'd; GX = G conj(H), GH = G conj(X) paired (X and H
// rows staged in smem); both inverse-FFT'd along rows, conj-twiddled, written to
// B1 (gx) and B2 (gh).  smem rows: g0 g1 x0 x1 h0 h1 -> gx0 gx1 gh0 gh1.
template <int N1, int N2>
__global__ void __launch_bounds__(Geo<N1, N2>::NTR, 3) k_rowB_bwd(const float2* __restrict__ Ag,
                                                                 const float2* __restrict__ X,
                                                                 const float2* __restrict__ H,
                                                                 float2* __restrict__ B1, float2* __restrict__ B2) {
  mgb_pdl_entry();
  constexpr int NT = Geo<N1, N2>::NTR, P = Geo<N1, N2>::P;
  constexpr long long N = Geo<N1, N2>::N;
  constexpr int PER = 2 * N2 / NT;
  extern __shared__ __align__(16) unsigned char smraw[];
  float2* s = reinterpret_cast<float2*>(smraw);
  const int r = blockIdx.x, b = blockIdx.y;
  const int row[2] = {r, (N1 - r) % N1};
  const int nr = (row[0] == row[1]) ? 1 : 2;
  const long long base = (long long)b * N;
  {
    float2 vg[PER], vx[PER], vh[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int i = threadIdx.x + j * NT, q = i / N2, k = i % N2;
      const long long g = base + (long long)row[q < nr ? q : 0] * N2 + k;
      vg[j] = Ag[g];
      vx[j] = X[g];
      vh[j] = H[g];
    }
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int i = threadIdx.x + j * NT, q = i / N2, k = i % N2;
      s[q * P + pidx<true>(k)] = vg[j];
      s[(2 + q) * P + pidx<true>(k)] = vx[j];
      s[(4 + q) * P + pidx<true>(k)] = vh[j];
    }
  }
  smem_fft<float, N2, 2, NT, P, 1, false, true>(s, false);
  float2 gx[PER], gh[PER];
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int i = threadIdx.x + j * NT;
    const int q = i / N2, k = i % N2;
    if (q < nr) {
      int qp, kp;
      if (nr == 2) { qp = 1 - q; kp = N2 - 1 - k; }
      else { qp = 0; kp = (row[0] == 0) ? ((N2 - k) & (N2 - 1)) : (N2 - 1 - k); }
      const int ik = pidx<true>(k), ip = pidx<true>(kp);
      float2 gl, gr, hl, hr, xl, xr;
      split_pair(s[q * P + ik], s[qp * P + ip], gl, gr);
      split_pair(s[(2 + q) * P + ik], s[(2 + qp) * P + ip], xl, xr);
      split_pair(s[(4 + q) * P + ik], s[(4 + qp) * P + ip], hl, hr);
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
    if (i / N2 < nr) {
      s[(i / N2) * P + pidx<true>(i % N2)] = gx[j];
      s[(2 + i / N2) * P + pidx<true>(i % N2)] = gh[j];
    }
  }
  smem_fft<float, N2, 4, NT, P, 1, false, true>(s, true);
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    const int i = threadIdx.x + j * NT;
    const int q = i / N2, n2 = i % N2;
    if (q < nr) {
      const float2 w = fs_twiddle<Geo<N1, N2>::LOG>(row[q] * n2, true);
      const int ii = pidx<true>(n2);
      B1[base + (long long)row[q] * N2 + n2] = cmul(s[q * P + ii], w);
      B2[base + (long long)row[q] * N2 + n2] = cmul(s[(2 + q) * P + ii], w);
    }
  }
}

template <int N1, int N2>
constexpr size_t col_smem() { return sizeof(float2) * Geo<N1, N2>::TC * N1; }
template <int N1, int N2>
constexpr size_t row_smem() { return sizeof(float2) * 4 * Geo<N1, N2>::P; }
template <int N1, int N2>
constexpr size_t rowbwd_smem() { return sizeof(float2) * 6 * Geo<N1, N2>::P; }

}  // namespace fs
