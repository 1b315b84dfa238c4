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
constexpr int RP = 1;  // row pairs (2 warps) per row-kernel CTA

template <int N1>
struct G {
  static constexpr int Q = N1 < 32 ? N1 : 32;
  static constexpr int P = N1 / Q;
  // (the column transform below needs P <= Q, i.e. N1 <= 1024; N1 = 2048 uses fs2_col64.cuh)
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
// per-warp shared memory of the row kernels: the staged operand rows (cp.async
// prefetch), padded to TBUF where a row buffer doubles as the transpose scratch
// once its contents are in registers (no separate transpose buffer)
constexpr int ROWH_WARP = TBUF;                 // [Ah row | scratch]
constexpr int ROWF_WARP = TBUF + N2;            // [Ax row -> spectrum | scratch], [H row]
constexpr int ROWG_WARP = TBUF + N2 + TBUF;     // [Ag row -> G spectrum | scratch], [X row], [H row | scratch]
constexpr size_t ROWH_SMEM = (size_t)2 * RP * ROWH_WARP * sizeof(float2);
constexpr size_t ROWF_SMEM = (size_t)2 * RP * ROWF_WARP * sizeof(float2);
constexpr size_t ROWG_SMEM = (size_t)2 * RP * ROWG_WARP * sizeof(float2);

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }
// one warp copies a row of N2 float2 (8 KB) into shared memory, 16 B per request
__device__ __forceinline__ void row_prefetch(float2* dst, const float2* __restrict__ src, int lane) {
#pragma unroll
  for (int i = 0; i < N2 / 2 / 32; ++i) cp_async16(dst + 2 * (lane + 32 * i), src + 2 * (lane + 32 * i));
}

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
  static_assert(g::P <= g::Q && g::Q % g::P == 0, "register column transform: N1 <= 1024");
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

// The same forward transform with ONE copy of the 32-point DFT code (run twice
// in a non-unrolled loop): the row kernels run three transforms per warp and
// were instruction-cache bound with fully unrolled copies.  Inverses use
// IFFT(x) = conj(FFT(conj(x))).
__device__ __forceinline__ void row_fft_compact(float2 (&v)[32], float2* T, int lane) {
#pragma unroll 1
  for (int h = 0; h < 2; ++h) {
    rf::rdft<32, false>(v);
    if (h == 1) break;
    twiddle_run<10, 32, false>(v, 0, lane);
#pragma unroll
    for (int kb = 0; kb < 32; ++kb) T[lane * TP + kb] = v[kb];
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = T[j * TP + lane];
    __syncwarp();
  }
}

// epilogues with a prefetch(ctx, n, b) hook (kPrefetch = true)
template <class Ep, class = void>
struct ep_prefetch {
  static constexpr bool value = false;
};
template <class Ep>
struct ep_prefetch<Ep, decltype(void(Ep::kPrefetch))> {
  static constexpr bool value = Ep::kPrefetch;
};

// ---------------------------------------------------------------------------
// column pass, forward: A[b][k1*N2 + n2] = w_N^{k1 n2} FFT_{N1}(x[. * N2 + n2])
template <int N1, class Ld>
__global__ void __launch_bounds__(G<N1>::NT, 512 / G<N1>::NT) k_colA(Ld ld, float2* __restrict__ A, int nz_rows, int rev) {
  mgb_pdl_entry();
  using g = G<N1>;
  constexpr int Q = g::Q, P = g::P, TC = g::TC, B8 = Q < 8 ? Q : 8;
  extern __shared__ __align__(16) unsigned char smraw[];
  float2* sm = reinterpret_cast<float2*>(smraw);
  __shared__ double red[32];
  const int c = threadIdx.x % TC, j = threadIdx.x / TC;
  // rev: walk the nodes backwards, so the kernel starts on the nodes the previous
  // kernel touched last (still in L2)
  const int b = rev ? gridDim.y - 1 - blockIdx.y : blockIdx.y, col = blockIdx.x * TC + c;
  const typename Ld::Ctx ctx = ld.prepare(b);
  float acc = 0.f;
  float2 v[Q];
  // software-pipelined loader: batch m0 + BL is fetched before batch m0 is finished
  constexpr int BL = Ld::kBatch < B8 ? Ld::kBatch : B8;
  typename Ld::Raw raw[2][BL];
#pragma unroll
  for (int i = 0; i < BL; ++i) {
    const int n1 = j + P * i;
    raw[0][i] = ld.fetch(ctx, b, (long long)n1 * N2 + col, n1 < nz_rows);
  }
#pragma unroll
  for (int m0 = 0; m0 < Q; m0 += BL) {
    const int cur = (m0 / BL) & 1;
    if (m0 + BL < Q) {
#pragma unroll
      for (int i = 0; i < BL; ++i) {
        const int n1 = j + P * (m0 + BL + i);
        raw[cur ^ 1][i] = ld.fetch(ctx, b, (long long)n1 * N2 + col, n1 < nz_rows);
      }
    }
#pragma unroll
    for (int i = 0; i < BL; ++i) {
      const int n1 = j + P * (m0 + i);
      v[m0 + i] = ld.finish(ctx, b, (long long)n1 * N2 + col, raw[cur][i], acc);
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
                                                   int out_rows, int rev) {
  mgb_pdl_entry();
  using g = G<N1>;
  constexpr int Q = g::Q, P = g::P, TC = g::TC, B8 = Q < 8 ? Q : 8;
  extern __shared__ __align__(16) unsigned char smraw[];
  float2* sm = reinterpret_cast<float2*>(smraw);
  __shared__ double red[32];
  const int c = threadIdx.x % TC, j = threadIdx.x / TC;
  // rev: walk the nodes backwards, so the kernel starts on the nodes the previous
  // kernel touched last (still in L2)
  const int b = rev ? gridDim.y - 1 - blockIdx.y : blockIdx.y, col = blockIdx.x * TC + c;
  const float2* src = Bb + (long long)b * g::N + col;
  float2 v[Q];
#pragma unroll
  for (int m = 0; m < Q; ++m) v[m] = src[(long long)(j + P * m) * N2];
  const typename Ep::Ctx ctx = ep.prepare(b);
  typename Ep::Raw raw[2][B8];
  // first epilogue batch issued before the transform so its latency hides behind it
#pragma unroll
  for (int i = 0; i < B8; ++i) {
    const int n1 = j + P * i;
    raw[0][i] = ep.fetch(ctx, b, (long long)n1 * N2 + col, n1 < out_rows);
  }
  if constexpr (ep_prefetch<Ep>::value) {  // the later batches' inputs towards L2 meanwhile
#pragma unroll
    for (int m = B8; m < Q; ++m) {
      const int n1 = j + P * m;
      if (n1 < out_rows) ep.prefetch(ctx, (long long)n1 * N2 + col, b);
    }
  }
  col_fft<N1, true>(v, sm, c, j);
  float a0 = 0.f, a1 = 0.f;
  // software-pipelined epilogue: batch m0 + B8 is fetched before batch m0 is consumed
#pragma unroll
  for (int m0 = 0; m0 < Q; m0 += B8) {
    const int cur = (m0 / B8) & 1;
    if (m0 + B8 < Q) {
#pragma unroll
      for (int i = 0; i < B8; ++i) {
        const int n1 = j + P * (m0 + B8 + i);
        raw[cur ^ 1][i] = ep.fetch(ctx, b, (long long)n1 * N2 + col, n1 < out_rows);
      }
    }
#pragma unroll
    for (int i = 0; i < B8; ++i) {
      const int n1 = j + P * (m0 + i);
      if (n1 < out_rows) {
        float2 y = v[m0 + i];
        y.x *= scale;
        y.y *= scale;
        ep.finish(ctx, b, (long long)n1 * N2 + col, y, raw[cur][i], a0, a1);
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

// warp-private region of a row kernel with WARP float2 per warp
template <int WARP>
__device__ __forceinline__ float2* warp_region(unsigned char* smraw, int w) {
  return reinterpret_cast<float2*>(smraw) + (size_t)w * WARP;
}

// prep: H[b][row][k] = FFT_{N2}(Ah[b][row][.])  (FIR spectrum, row layout)
template <int N1>
__global__ void __launch_bounds__(2 * RP * 32) k_rowH(const float2* __restrict__ Ah, float2* __restrict__ H, int rev) {
  mgb_pdl_entry();
  using g = G<N1>;
  extern __shared__ __align__(16) unsigned char smraw[];
  const RowMap rm = row_map<N1>();
  if (!rm.active) return;
  float2* sA = warp_region<ROWH_WARP>(smraw, threadIdx.x >> 5);  // Ah row, then the transpose scratch
  const int bnode = rev ? gridDim.y - 1 - blockIdx.y : blockIdx.y;
  const long long base = (long long)bnode * g::N + (long long)rm.row * N2;
  row_prefetch(sA, Ah + base, rm.lane);
  cp_async_wait_all();
  __syncwarp();
  float2 v[32];
#pragma unroll
  for (int m = 0; m < 32; ++m) v[m] = sA[rm.lane + 32 * m];
  __syncwarp();
  row_fft<false>(v, sA, rm.lane);
#pragma unroll
  for (int ka = 0; ka < 32; ++ka) H[base + rm.lane + 32 * ka] = v[ka];
}

// forward convolution rows: X = FFT rows of Ax (stored for the backward);
// Y = X_l H_l + i X_r H_r (paired split); Bo = w_N^{-row n2} IFFT rows of Y.
// Both operand rows of the warp (Ax, H) are prefetched with cp.async; the
// partner warp's staged H row and spectrum are read from its region.  The two
// transforms share one code copy (pass loop); the duplicate warp of a
// self-paired row computes along but stores nothing.
// CONJ (the backward's input gradient): Ax = the column pass of dL/dy, X receives its row
// spectrum G (kept for k_rowP), Bo = the inverse rows of G_l conj(H_l) + i G_r conj(H_r).
template <int N1, bool CONJ = false>
__global__ void __launch_bounds__(2 * RP * 32) k_rowF(const float2* __restrict__ Ax, const float2* __restrict__ H,
                                                     float2* __restrict__ X, float2* __restrict__ Bo, int rev) {
  mgb_pdl_entry();
  using g = G<N1>;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int w = threadIdx.x >> 5;
  float2* sA = warp_region<ROWF_WARP>(smraw, w);  // Ax row, scratch, this row's spectrum, scratch
  float2* sH = sA + TBUF;                          // H row
  const RowMap rm = row_map<N1>();
  const bool self = rm.row == rm.prow;
  float2* pA = self ? sA : warp_region<ROWF_WARP>(smraw, w ^ 1);
  float2* pH = pA + TBUF;
  const int bnode = rev ? gridDim.y - 1 - blockIdx.y : blockIdx.y;
  const long long base = (long long)bnode * g::N + (long long)rm.row * N2;
  const int lane = rm.lane;
  row_prefetch(sA, Ax + base, lane);
  cp_async_commit();
  row_prefetch(sH, H + base, lane);  // not needed before the product: its latency hides behind the FFT
  cp_async_commit();
  cp_async_wait<1>();
  __syncwarp();
  float2 v[32];
#pragma unroll
  for (int m = 0; m < 32; ++m) v[m] = sA[lane + 32 * m];
  __syncwarp();  // sA becomes the transpose scratch
#pragma unroll 1
  for (int pass = 0; pass < 2; ++pass) {
    row_fft_compact(v, sA, lane);
    if (pass == 1) break;
#pragma unroll
    for (int ka = 0; ka < 32; ++ka) {
      if (rm.active) X[base + lane + 32 * ka] = v[ka];
      sA[lane + 32 * ka] = v[ka];  // natural order for the partner warp
    }
    cp_async_wait<0>();  // own H row landed (the barrier publishes it to the partner)
    __syncthreads();
#pragma unroll
    for (int ka = 0; ka < 32; ++ka) {
      const int k = lane + 32 * ka, kp = partner_col(rm.row, k);
      float2 xl, xr, hl, hr;
      split_pair(v[ka], pA[kp], xl, xr);
      split_pair(sH[k], pH[kp], hl, hr);
      const float2 y1 = CONJ ? cmulc(xl, hl) : cmul(xl, hl), y2 = CONJ ? cmulc(xr, hr) : cmul(xr, hr);
      v[ka] = make_float2(y1.x - y2.y, -(y1.y + y2.x));  // conj: inverse via the forward code
    }
    __syncthreads();  // both warps done reading the spectra before sA is scratch again
  }
  if (!rm.active) return;
#pragma unroll
  for (int n = 0; n < 32; ++n) v[n].y = -v[n].y;
  twiddle_run<g::LOGN, 32, true>(v, rm.row * lane, rm.row * 32);
#pragma unroll
  for (int n = 0; n < 32; ++n) Bo[base + lane + 32 * n] = v[n];
}

// backward rows: G = FFT rows of Ag; GX = G_l conj(H_l) + i G_r conj(H_r) -> B1,
// GH = G_l conj(X_l) + i G_r conj(X_r) -> B2, both inverse row FFT'd and conj-twiddled.
// Ag, X and H rows are prefetched with cp.async into the warp's region; the three
// transforms share one code copy (pass loop).
template <int N1>
__global__ void __launch_bounds__(2 * RP * 32) k_rowG(const float2* __restrict__ Ag, const float2* __restrict__ X,
                                                     const float2* __restrict__ H, float2* __restrict__ B1,
                                                     float2* __restrict__ B2, int rev) {
  mgb_pdl_entry();
  using g = G<N1>;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int w = threadIdx.x >> 5;
  float2* sA = warp_region<ROWG_WARP>(smraw, w);  // Ag row, scratch, then this row's G spectrum
  float2* sX = sA + TBUF;
  float2* sH = sX + N2;                            // H row, then the scratch of passes 1-2
  const RowMap rm = row_map<N1>();
  const bool self = rm.row == rm.prow;
  float2* pA = self ? sA : warp_region<ROWG_WARP>(smraw, w ^ 1);
  float2* pX = pA + TBUF;
  float2* pH = pX + N2;
  const int bnode = rev ? gridDim.y - 1 - blockIdx.y : blockIdx.y;
  const long long base = (long long)bnode * g::N + (long long)rm.row * N2;
  const int lane = rm.lane;
  row_prefetch(sA, Ag + base, lane);
  cp_async_commit();
  row_prefetch(sX, X + base, lane);  // X and H are first read after the G transform
  row_prefetch(sH, H + base, lane);
  cp_async_commit();
  cp_async_wait<1>();
  __syncwarp();
  float2 v[32];
#pragma unroll
  for (int m = 0; m < 32; ++m) v[m] = sA[lane + 32 * m];
  __syncwarp();  // sA becomes the transpose scratch of pass 0
#pragma unroll 1
  for (int pass = 0; pass < 3; ++pass) {
    row_fft_compact(v, pass == 0 ? sA : sH, lane);
    if (pass == 0) {
#pragma unroll
      for (int ka = 0; ka < 32; ++ka) sA[lane + 32 * ka] = v[ka];
      cp_async_wait<0>();  // own X and H rows landed (the barrier publishes them to the partner)
      __syncthreads();
    } else {
#pragma unroll
      for (int n = 0; n < 32; ++n) v[n].y = -v[n].y;
      twiddle_run<g::LOGN, 32, true>(v, rm.row * lane, rm.row * 32);
      float2* dst = (pass == 1 ? B1 : B2) + base + lane;
      if (rm.active) {
#pragma unroll
        for (int n = 0; n < 32; ++n) dst[32 * n] = v[n];
      }
      if (pass == 2) break;
    }
    // next transform's input: conj(G_l conj(O_l) + i G_r conj(O_r)), O = H (pass 1) or X (pass 2)
    const float2* oS = pass == 0 ? sH : sX;
    const float2* oP = pass == 0 ? pH : pX;
#pragma unroll
    for (int ka = 0; ka < 32; ++ka) {
      const int k = lane + 32 * ka, kp = partner_col(rm.row, k);
      float2 gl, gr, ol, orr;
      split_pair(sA[k], pA[kp], gl, gr);
      split_pair(oS[k], oP[kp], ol, orr);
      const float2 y1 = cmulc(gl, ol), y2 = cmulc(gr, orr);
      v[ka] = make_float2(y1.x - y2.y, -(y1.y + y2.x));
    }
    if (pass == 0) __syncthreads();  // partner done reading our H row: it is scratch from here on
  }
}


// FIR-gradient rows (backward phase 2, off the critical path): B = conj-twiddled inverse
// rows of A_l conj(O_l) + i A_r conj(O_r) for two kept row spectra (A = G from
// k_rowF<N1, true>, O = X).  B may alias A: both warps of a row pair stage their rows in
// shared memory and pass a barrier before either writes.
template <int N1>
__global__ void __launch_bounds__(2 * RP * 32) k_rowP(const float2* A, const float2* __restrict__ O, float2* B,
                                                     int rev) {
  mgb_pdl_entry();
  using g = G<N1>;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int w = threadIdx.x >> 5;
  float2* sA = warp_region<ROWF_WARP>(smraw, w);  // A row, then the transpose scratch
  float2* sO = sA + TBUF;                          // O row
  const RowMap rm = row_map<N1>();
  const bool self = rm.row == rm.prow;
  float2* pA = self ? sA : warp_region<ROWF_WARP>(smraw, w ^ 1);
  float2* pO = pA + TBUF;
  const int bnode = rev ? gridDim.y - 1 - blockIdx.y : blockIdx.y;
  const long long base = (long long)bnode * g::N + (long long)rm.row * N2;
  const int lane = rm.lane;
  row_prefetch(sA, A + base, lane);
  row_prefetch(sO, O + base, lane);
  cp_async_wait_all();
  __syncthreads();  // both warps' rows staged (and A read: B may overwrite it from here on)
  float2 v[32];
#pragma unroll
  for (int ka = 0; ka < 32; ++ka) {
    const int k = lane + 32 * ka, kp = partner_col(rm.row, k);
    float2 al, ar, ol, orr;
    split_pair(sA[k], pA[kp], al, ar);
    split_pair(sO[k], pO[kp], ol, orr);
    const float2 y1 = cmulc(al, ol), y2 = cmulc(ar, orr);
    v[ka] = make_float2(y1.x - y2.y, -(y1.y + y2.x));  // conj: inverse via the forward code
  }
  __syncthreads();  // partner done reading sA before it is scratch
  row_fft_compact(v, sA, lane);
  if (!rm.active) return;
#pragma unroll
  for (int n = 0; n < 32; ++n) v[n].y = -v[n].y;
  twiddle_run<g::LOGN, 32, true>(v, rm.row * lane, rm.row * 32);
#pragma unroll
  for (int n = 0; n < 32; ++n) B[base + lane + 32 * n] = v[n];
}

// ---------------------------------------------------------------------------
// Persistent column pass with bulk-async (TMA engine) tile staging.
//
// One CTA per SM walks the (node, column block) tiles t = blockIdx.x + k*gridDim.x.
// A tile (N1 rows x TC columns of the complex input, TC*8-byte row segments 8 KB
// apart) is copied global -> shared memory by cp.async.bulk (one 128-byte segment
// per instruction, issued by warp 0, completion counted in bytes on an mbarrier)
// into one of two stages; the next tile's copy is in flight while the CTA
// transforms the current one, so the load latency that dominated the
// one-tile-per-CTA kernels (ncu: long_scoreboard 40-60 % of stalls at 34-45 % of
// DRAM bandwidth) overlaps the math.  A stage doubles as the transform's exchange
// buffer once its tile is in registers.

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}

template <int N1>
struct GP {
  using g = G<N1>;
  static constexpr int TILES_PER_NODE = N2 / g::TC;
  static constexpr int TILE = N1 * g::TC;                       // float2 per tile
  static constexpr int STAGE = ((g::TC * g::PITCH > TILE ? g::TC * g::PITCH : TILE) + 15) / 16 * 16;
  static constexpr size_t SMEM = 2 * (size_t)STAGE * sizeof(float2);
};

// warp 0: stage tile t of Bb (rows n1 < rows) into st, completion on bar
template <int N1>
__device__ __forceinline__ void stage_tile(const float2* __restrict__ Bb, int t, int rows, float2* st,
                                           unsigned long long* bar, int lane) {
  using g = G<N1>;
  const int b = t / GP<N1>::TILES_PER_NODE, col0 = (t % GP<N1>::TILES_PER_NODE) * g::TC;
  if (lane == 0) mbar_expect_tx(bar, (unsigned)(rows * g::TC * sizeof(float2)));
  __syncwarp();
  const float2* src = Bb + (long long)b * g::N + col0;
  for (int r = lane; r < rows; r += 32) bulk_g2s(st + r * g::TC, src + (long long)r * N2, g::TC * sizeof(float2), bar);
}

template <int N1, class Ep>
__global__ void __launch_bounds__(G<N1>::NT, 1) k_colC_p(const float2* __restrict__ Bb, Ep ep, float scale, int out_rows,
                                                        int ntiles) {
  using g = G<N1>;
  using gp = GP<N1>;
  constexpr int Q = g::Q, P = g::P, TC = g::TC, B8 = Q < 8 ? Q : 8;
  extern __shared__ __align__(128) unsigned char smraw[];
  float2* stage = reinterpret_cast<float2*>(smraw);
  __shared__ __align__(8) unsigned long long bar[2];
  __shared__ double red[32];
  const int c = threadIdx.x % TC, j = threadIdx.x / TC, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  mgb_pdl_entry();
  int t = blockIdx.x;
  if (warp == 0 && t < ntiles) stage_tile<N1>(Bb, t, N1, stage, &bar[0], lane);
  for (int k = 0; t < ntiles; ++k, t += gridDim.x) {
    const int s = k & 1;
    float2* cur = stage + s * gp::STAGE;
    // the other stage was last read in iteration k-1, which ended with a barrier
    if (warp == 0 && t + (int)gridDim.x < ntiles)
      stage_tile<N1>(Bb, t + gridDim.x, N1, stage + (s ^ 1) * gp::STAGE, &bar[s ^ 1], lane);
    const int b = t / gp::TILES_PER_NODE, cb = t % gp::TILES_PER_NODE, col = cb * TC + c;
    const typename Ep::Ctx ctx = ep.prepare(b);
    typename Ep::Raw raw[2][B8];
#pragma unroll
    for (int i = 0; i < B8; ++i) {
      const int n1 = j + P * i;
      raw[0][i] = ep.fetch(ctx, b, (long long)n1 * N2 + col, n1 < out_rows);
    }
    mbar_wait(&bar[s], (k >> 1) & 1);
    float2 v[Q];
#pragma unroll
    for (int m = 0; m < Q; ++m) v[m] = cur[(j + P * m) * TC + c];
    __syncthreads();  // every thread holds its column values: the stage becomes the exchange buffer
    col_fft<N1, true>(v, cur, c, j);
    float a0 = 0.f, a1 = 0.f;
#pragma unroll
    for (int m0 = 0; m0 < Q; m0 += B8) {
      const int cr = (m0 / B8) & 1;
      if (m0 + B8 < Q) {
#pragma unroll
        for (int i = 0; i < B8; ++i) {
          const int n1 = j + P * (m0 + B8 + i);
          raw[cr ^ 1][i] = ep.fetch(ctx, b, (long long)n1 * N2 + col, n1 < out_rows);
        }
      }
#pragma unroll
      for (int i = 0; i < B8; ++i) {
        const int n1 = j + P * (m0 + i);
        if (n1 < out_rows) {
          float2 y = v[m0 + i];
          y.x *= scale;
          y.y *= scale;
          ep.finish(ctx, b, (long long)n1 * N2 + col, y, raw[cr][i], a0, a1);
        }
      }
    }
    if (Ep::kAccum) {
      const double t0 = block_sum((double)a0, red);
      __syncthreads();
      const double t1 = block_sum((double)a1, red);
      if (threadIdx.x == 0) ep.commit(b, cb, t0, t1);
    }
    // the stage's generic-proxy accesses (exchange) are ordered before the async-proxy
    // (bulk copy) writes that refill it in iteration k+1
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();  // stage s is free for the copy issued at the top of iteration k+1
  }
}

}  // namespace fs2
