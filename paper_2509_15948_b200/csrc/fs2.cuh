// Four-step FFT convolution with register-resident transforms (sm_100a).
//
// Same data flow and layouts as fourstep.cuh (N = N1 * N2, signal index
// n = n1*N2 + n2, spectra kept in "row layout" k1*N2 + k2), but every
// transform is done in registers with a single shared-memory exchange:
//
// * column pass, length N1 = P*Q (Q = min(N1, 32)): P threads per column, each
//   holding the Q samples j + P*m; a Q-point register DFT, a twiddle, ONE
//   exchange through padded shared memory, then Q/P P-point register DFTs.
//   The thread ends up holding outputs j + P*m' again, so loads and stores
//   are the same coalesced pattern (16+ consecutive columns per half-warp).
// * row pass, length N2 = 1024 = 32 x 32: one warp per row, lane j holding
//   samples j + 32 m; 32-point register DFT, twiddle, a 32x33 warp-private
//   transpose, 32-point register DFT; the lane then owns spectral bins
//   lane + 32 ka, which is also the input pattern of the inverse transform.
//
// The packed stereo spectrum (left + i*right) is split against its Hermitian
// partner (row N1 - r, column N2 - 1 - k; row 0: column -k), exchanged between
// the two warps of a row pair through shared memory (or read straight from
// global / L1 for the stored X and H spectra).  Shared-memory traffic per
// element and transform drops from 8 accesses (four radix-8/4/2 Stockham
// passes) to 2, which was the limiter of the Stockham kernels (ncu: L1/smem
// pipe 88-90 %, DRAM 18-30 %).
#pragma once
#include "common.cuh"
#include "regfft.cuh"

namespace fs2 {

constexpr int N2 = 1024;
constexpr int RP = 2;  // row pairs (4 warps) per row-kernel CTA

template <int N1>
struct G {
  static constexpr int Q = N1 < 32 ? N1 : 32;
  static constexpr int P = N1 / Q;
  static_assert(P <= Q && Q % P == 0, "N1 <= 1024");
  static constexpr int TC = P >= 16 ? 16 : 256 / P;  // columns per column-pass CTA
  static constexpr int NT = TC * P;                   // 256 (512 for N1 = 1024)
  static constexpr int PITCH = N1 + 1;                // odd: conflict-free 8-byte column accesses
  static constexpr int LOG1 = __builtin_ctz(N1);
  static constexpr int LOGN = LOG1 + 10;
  static constexpr long long N = (long long)N1 * N2;
  static constexpr int NBLK = N2 / TC;                // column CTAs per row (partial-sum slots)
  static constexpr size_t COL_SMEM = P > 1 ? (size_t)TC * PITCH * sizeof(float2) : 0;
  static constexpr int ROW_ITEMS = N1 / 2 + 1;        // row pairs (r, N1 - r), r = 0..N1/2
  static constexpr int ROW_CTAS = (ROW_ITEMS + RP - 1) / RP;
};

constexpr int TP = 33;                 // transpose pitch
constexpr int TBUF = 32 * TP;          // per-warp transpose buffer (float2)
constexpr size_t ROWF_SMEM = (size_t)2 * RP * TBUF * sizeof(float2);
constexpr size_t ROWG_SMEM = (size_t)2 * RP * (TBUF + N2) * sizeof(float2);

__device__ __forceinline__ void split_pair(float2 zk, float2 zp, float2& a, float2& b) {
  a = make_float2(0.5f * (zk.x + zp.x), 0.5f * (zk.y - zp.y));
  const float2 d = make_float2(0.5f * (zk.x - zp.x), 0.5f * (zk.y + zp.y));
  b = make_float2(d.y, -d.x);
}

// compiler fence every 8 iterations of an unrolled product loop: bounds how many
// independent spectrum loads get hoisted (register pressure vs memory parallelism)
__device__ __forceinline__ void chunk_fence(int ka) {
  if ((ka & 7) == 7) asm volatile("" ::: "memory");
}

// v[i] *= W_M^{(e0 + de*i)}, i < n, re-anchored from the table every 8 steps
template <int LOGM, int n, bool INV>
__device__ __forceinline__ void twiddle_run(float2* v, int e0, int de) {
  const float2 step = rf::wexp<LOGM>(de, INV);
#pragma unroll
  for (int i0 = 0; i0 < n; i0 += 8) {
    float2 w = rf::wexp<LOGM>(e0 + de * i0, INV);
#pragma unroll
    for (int i = i0; i < i0 + 8 && i < n; ++i) {
      if (i > 0 || e0 != 0) v[i] = cmul(v[i], w);
      w = cmul(w, step);
    }
  }
}

// column transform: thread (c, j) holds x[j + P m] (m < Q) -> X[j + P m'] (m' < Q)
template <int N1, bool INV>
__device__ __forceinline__ void col_fft(float2 (&v)[G<N1>::Q], float2* sm, int c, int j) {
  using g = G<N1>;
  constexpr int Q = g::Q, P = g::P;
  rf::rdft<Q, INV>(v);
  if constexpr (P > 1) {
    twiddle_run<g::LOG1, Q, INV>(v, 0, j);
    float2* col = sm + c * g::PITCH;
#pragma unroll
    for (int kb = 0; kb < Q; ++kb) col[j * Q + kb] = v[kb];
    __syncthreads();
#pragma unroll
    for (int t = 0; t < Q / P; ++t) {
      float2 s[P];
#pragma unroll
      for (int jj = 0; jj < P; ++jj) s[jj] = col[jj * Q + j + P * t];
      rf::rdft<P, INV>(s);
#pragma unroll
      for (int ka = 0; ka < P; ++ka) v[t + (Q / P) * ka] = s[ka];
    }
  }
}

// row transform (one warp): lane j holds x[j + 32 m] -> X[lane + 32 ka]
template <bool INV>
__device__ __forceinline__ void row_fft(float2 (&v)[32], float2* T, int lane) {
  rf::rdft<32, INV>(v);
  twiddle_run<10, 32, INV>(v, 0, lane);
#pragma unroll
  for (int kb = 0; kb < 32; ++kb) T[lane * TP + kb] = v[kb];
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = T[j * TP + lane];
  __syncwarp();
  rf::rdft<32, INV>(v);
}

// ---------------------------------------------------------------------------
// column pass, forward: A[b][k1*N2 + n2] = w_N^{k1 n2} FFT_{N1}(x[. * N2 + n2])
template <int N1, class Ld>
__global__ void __launch_bounds__(G<N1>::NT, 512 / G<N1>::NT) k_colA(Ld ld, float2* __restrict__ A, int nz_rows) {
  using g = G<N1>;
  constexpr int Q = g::Q, P = g::P, TC = g::TC, B8 = Q < 8 ? Q : 8;
  extern __shared__ __align__(16) unsigned char smraw[];
  float2* sm = reinterpret_cast<float2*>(smraw);
  __shared__ double red[32];
  const int c = threadIdx.x % TC, j = threadIdx.x / TC;
  const int b = blockIdx.y, col = blockIdx.x * TC + c;
  const typename Ld::Ctx ctx = ld.prepare(b);
  float acc = 0.f;
  float2 v[Q];
#pragma unroll
  for (int m0 = 0; m0 < Q; m0 += B8) {
    typename Ld::Raw raw[B8];
#pragma unroll
    for (int i = 0; i < B8; ++i) {
      const int n1 = j + P * (m0 + i);
      raw[i] = ld.fetch(ctx, b, (long long)n1 * N2 + col, n1 < nz_rows);
    }
#pragma unroll
    for (int i = 0; i < B8; ++i) {
      const int n1 = j + P * (m0 + i);
      v[m0 + i] = ld.finish(ctx, b, (long long)n1 * N2 + col, raw[i], acc);
    }
  }
  if (Ld::kAccum) {
    const double t = block_sum((double)acc, red);
    if (threadIdx.x == 0) ld.commit(b, blockIdx.x, t);
  }
  col_fft<N1, false>(v, sm, c, j);
  twiddle_run<g::LOGN, Q, false>(v, j * col, P * col);
  float2* dst = A + (long long)b * g::N + col;
#pragma unroll
  for (int m = 0; m < Q; ++m) dst[(long long)(j + P * m) * N2] = v[m];
}

// column pass, inverse: y[b][n1*N2 + n2] = scale * IFFT_{N1}(B[. * N2 + n2]); epilogue consumes y
template <int N1, class Ep>
__global__ void __launch_bounds__(G<N1>::NT, 512 / G<N1>::NT) k_colC(const float2* __restrict__ Bb, Ep ep, float scale,
                                                   int out_rows) {
  using g = G<N1>;
  constexpr int Q = g::Q, P = g::P, TC = g::TC, B8 = Q < 8 ? Q : 8;
  extern __shared__ __align__(16) unsigned char smraw[];
  float2* sm = reinterpret_cast<float2*>(smraw);
  __shared__ double red[32];
  const int c = threadIdx.x % TC, j = threadIdx.x / TC;
  const int b = blockIdx.y, col = blockIdx.x * TC + c;
  const float2* src = Bb + (long long)b * g::N + col;
  float2 v[Q];
#pragma unroll
  for (int m = 0; m < Q; ++m) v[m] = src[(long long)(j + P * m) * N2];
  col_fft<N1, true>(v, sm, c, j);
  const typename Ep::Ctx ctx = ep.prepare(b);
  float a0 = 0.f, a1 = 0.f;
#pragma unroll
  for (int m0 = 0; m0 < Q; m0 += B8) {
    typename Ep::Raw raw[B8];
#pragma unroll
    for (int i = 0; i < B8; ++i) {
      const int n1 = j + P * (m0 + i);
      raw[i] = ep.fetch(ctx, b, (long long)n1 * N2 + col, n1 < out_rows);
    }
#pragma unroll
    for (int i = 0; i < B8; ++i) {
      const int n1 = j + P * (m0 + i);
      if (n1 < out_rows) {
        float2 y = v[m0 + i];
        y.x *= scale;
        y.y *= scale;
        ep.finish(ctx, b, (long long)n1 * N2 + col, y, raw[i], a0, a1);
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
// row kernels: warp w of a CTA handles row pair item q = blockIdx.x*RP + w/2,
// rows (q, N1 - q); the second warp of a self-paired item (q = 0 or N1/2) idles.

struct RowMap {
  int q, row, prow, lane, wpair;
  bool active, valid;
};

template <int N1>
__device__ __forceinline__ RowMap row_map() {
  RowMap m;
  const int w = threadIdx.x >> 5;
  m.lane = threadIdx.x & 31;
  m.wpair = w & 1;
  m.q = blockIdx.x * RP + (w >> 1);
  m.valid = m.q < G<N1>::ROW_ITEMS;
  const int r0 = m.q, r1 = (N1 - m.q) % N1;
  m.row = m.wpair ? r1 : r0;
  m.prow = m.wpair ? r0 : r1;
  m.active = m.valid && !(m.wpair && r0 == r1);
  return m;
}

// Hermitian partner column of spectral column k in row `row` (partner row prow)
__device__ __forceinline__ int partner_col(int row, int k) { return row == 0 ? ((N2 - k) & (N2 - 1)) : (N2 - 1 - k); }

// prep: H[b][row][k] = FFT_{N2}(Ah[b][row][.])  (FIR spectrum, row layout)
template <int N1>
__global__ void __launch_bounds__(2 * RP * 32) k_rowH(const float2* __restrict__ Ah, float2* __restrict__ H) {
  using g = G<N1>;
  extern __shared__ __align__(16) unsigned char smraw[];
  float2* T = reinterpret_cast<float2*>(smraw) + (threadIdx.x >> 5) * TBUF;
  const RowMap rm = row_map<N1>();
  if (!rm.active) return;
  const long long base = (long long)blockIdx.y * g::N + (long long)rm.row * N2;
  float2 v[32];
#pragma unroll
  for (int m = 0; m < 32; ++m) v[m] = Ah[base + rm.lane + 32 * m];
  row_fft<false>(v, T, rm.lane);
#pragma unroll
  for (int ka = 0; ka < 32; ++ka) H[base + rm.lane + 32 * ka] = v[ka];
}

// forward convolution rows: X = FFT rows of Ax (stored for the backward);
// Y = X_l H_l + i X_r H_r (paired split); Bo = w_N^{-row n2} IFFT rows of Y
template <int N1>
__global__ void __launch_bounds__(2 * RP * 32, 3) k_rowF(const float2* __restrict__ Ax, const float2* __restrict__ H,
                                                     float2* __restrict__ X, float2* __restrict__ Bo) {
  using g = G<N1>;
  extern __shared__ __align__(16) unsigned char smraw[];
  float2* T = reinterpret_cast<float2*>(smraw) + (threadIdx.x >> 5) * TBUF;
  float2* Tp = reinterpret_cast<float2*>(smraw) + ((threadIdx.x >> 5) ^ 1) * TBUF;
  const RowMap rm = row_map<N1>();
  const bool self = rm.row == rm.prow;
  const long long bb = (long long)blockIdx.y * g::N;
  const long long base = bb + (long long)rm.row * N2, pbase = bb + (long long)rm.prow * N2;
  float2 v[32];
  if (rm.active) {
#pragma unroll
    for (int m = 0; m < 32; ++m) v[m] = Ax[base + rm.lane + 32 * m];
    row_fft<false>(v, T, rm.lane);
#pragma unroll
    for (int ka = 0; ka < 32; ++ka) {
      X[base + rm.lane + 32 * ka] = v[ka];
      T[rm.lane + 32 * ka] = v[ka];  // natural order for the partner warp
    }
  }
  __syncthreads();
  if (rm.active) {
    const float2* ps = self ? T : Tp;
#pragma unroll
    for (int ka = 0; ka < 32; ++ka) {
      const int k = rm.lane + 32 * ka, kp = partner_col(rm.row, k);
      float2 xl, xr, hl, hr;
      split_pair(v[ka], ps[kp], xl, xr);
      split_pair(__ldg(H + base + k), __ldg(H + pbase + kp), hl, hr);
      const float2 y1 = cmul(xl, hl), y2 = cmul(xr, hr);
      v[ka] = make_float2(y1.x - y2.y, y1.y + y2.x);
      chunk_fence(ka);
    }
  }
  __syncthreads();  // partner reads done before T is reused as the transpose buffer
  if (!rm.active) return;
  row_fft<true>(v, T, rm.lane);
  twiddle_run<g::LOGN, 32, true>(v, rm.row * rm.lane, rm.row * 32);
#pragma unroll
  for (int n = 0; n < 32; ++n) Bo[base + rm.lane + 32 * n] = v[n];
}

// backward rows: G = FFT rows of Ag; GX = G_l conj(H_l) + i G_r conj(H_r) -> B1,
// GH = G_l conj(X_l) + i G_r conj(X_r) -> B2, both inverse row FFT'd and conj-twiddled
template <int N1>
__global__ void __launch_bounds__(2 * RP * 32, 3) k_rowG(const float2* __restrict__ Ag, const float2* __restrict__ X,
                                                     const float2* __restrict__ H, float2* __restrict__ B1,
                                                     float2* __restrict__ B2) {
  using g = G<N1>;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int w = threadIdx.x >> 5;
  float2* T = reinterpret_cast<float2*>(smraw) + w * TBUF;
  float2* S = reinterpret_cast<float2*>(smraw) + 2 * RP * TBUF + w * N2;        // own G spectrum
  float2* Sp = reinterpret_cast<float2*>(smraw) + 2 * RP * TBUF + (w ^ 1) * N2;  // partner's
  const RowMap rm = row_map<N1>();
  const bool self = rm.row == rm.prow;
  const long long bb = (long long)blockIdx.y * g::N;
  const long long base = bb + (long long)rm.row * N2, pbase = bb + (long long)rm.prow * N2;
  float2 v[32];
  if (rm.active) {
#pragma unroll
    for (int m = 0; m < 32; ++m) v[m] = Ag[base + rm.lane + 32 * m];
    row_fft<false>(v, T, rm.lane);
#pragma unroll
    for (int ka = 0; ka < 32; ++ka) S[rm.lane + 32 * ka] = v[ka];
  }
  __syncthreads();
  if (!rm.active) return;
  const float2* ps = self ? S : Sp;
#pragma unroll
  for (int ka = 0; ka < 32; ++ka) {
    const int k = rm.lane + 32 * ka, kp = partner_col(rm.row, k);
    float2 gl, gr, hl, hr;
    split_pair(v[ka], ps[kp], gl, gr);
    split_pair(__ldg(H + base + k), __ldg(H + pbase + kp), hl, hr);
    const float2 y1 = cmulc(gl, hl), y2 = cmulc(gr, hr);
    v[ka] = make_float2(y1.x - y2.y, y1.y + y2.x);
    chunk_fence(ka);
  }
  row_fft<true>(v, T, rm.lane);
  twiddle_run<g::LOGN, 32, true>(v, rm.row * rm.lane, rm.row * 32);
#pragma unroll
  for (int n = 0; n < 32; ++n) B1[base + rm.lane + 32 * n] = v[n];
#pragma unroll
  for (int ka = 0; ka < 32; ++ka) {
    const int k = rm.lane + 32 * ka, kp = partner_col(rm.row, k);
    float2 gl, gr, xl, xr;
    split_pair(S[k], ps[kp], gl, gr);
    split_pair(__ldg(X + base + k), __ldg(X + pbase + kp), xl, xr);
    const float2 y1 = cmulc(gl, xl), y2 = cmulc(gr, xr);
    v[ka] = make_float2(y1.x - y2.y, y1.y + y2.x);
    chunk_fence(ka);
  }
  __syncwarp();
  row_fft<true>(v, T, rm.lane);
  twiddle_run<g::LOGN, 32, true>(v, rm.row * rm.lane, rm.row * 32);
#pragma unroll
  for (int n = 0; n < 32; ++n) B2[base + rm.lane + 32 * n] = v[n];
}

}  // namespace fs2
