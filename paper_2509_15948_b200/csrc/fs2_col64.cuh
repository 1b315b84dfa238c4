// Column passes of the register four-step for N1 = 2048 (N = 2^21).
//
// fs2.cuh's column transform needs P <= Q (N1 <= 1024).  A 2048-point column
// is split 2048 = 32 x 64 with P = 64 threads per column holding Q = 32 values;
// the 64-point second stage is 32 x 2: a 32-point register DFT over even / odd
// j in each thread of a pair (j, j ^ 1 = lanes TC apart in the same warp) and a
// radix-2 butterfly through one shuffle per value.  8 columns per CTA (512
// threads, 131 KB of exchange buffer, one CTA per SM).
//
//   input  thread (c, j) holds x[j + 64 m], m < 32
//   output thread (c, j) holds X[row(j, m)], row = (j >> 1) + 32 m + 1024 (j & 1)
//   X[kb + 32 (k' + 32 h')] = A_0[k'] + (-1)^h' W_64^k' A_1[k'],
//   A_h[k'] = sum_jj W_32^(jj k') Y[2 jj + h][kb],  Y[j][kb] = W_2048^(j kb) sum_m x[j + 64 m] W_32^(m kb)
#pragma once
#include "fs2.cuh"

namespace fs2 {

struct C64 {
  static constexpr int N1 = 2048, Q = 32, P = 64, TC = 8, NT = TC * P;  // 512 threads
  static constexpr int PITCH = N1 + 1;
  static constexpr size_t SMEM = (size_t)TC * PITCH * sizeof(float2);
  static constexpr int LOGN = 11 + 10;
  static constexpr long long N = (long long)N1 * N2;
  static constexpr int NBLK = N2 / TC;  // column CTAs per node (partial-sum slots)
  __device__ static __forceinline__ int row(int j, int m) { return (j >> 1) + 32 * m + 1024 * (j & 1); }
};

// epilogue batch of the 2048-point inverse column pass: Ep::kBatch64 if declared, else 8
template <class Ep, class = void>
struct ep_batch64 {
  static constexpr int value = 8;
};
template <class Ep>
struct ep_batch64<Ep, decltype(void(Ep::kBatch64))> {
  static constexpr int value = Ep::kBatch64;
};

template <bool INV>
__device__ __forceinline__ void col_fft64(float2 (&v)[32], float2* sm, int c, int j) {
  rf::rdft<32, INV>(v);
  twiddle_run<11, 32, INV>(v, 0, j);  // W_2048^(j kb)
  float2* col = sm + c * C64::PITCH;
#pragma unroll
  for (int kb = 0; kb < 32; ++kb) col[j * 32 + kb] = v[kb];
  __syncthreads();
  const int kb = j >> 1, h = j & 1;
#pragma unroll
  for (int jj = 0; jj < 32; ++jj) v[jj] = col[(2 * jj + h) * 32 + kb];
  rf::rdft<32, INV>(v);
  if (h) twiddle_run<6, 32, INV>(v, 0, 1);  // W_64^k' on the odd half
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const float ox = __shfl_xor_sync(0xffffffffu, v[k].x, C64::TC), oy = __shfl_xor_sync(0xffffffffu, v[k].y, C64::TC);
    v[k] = h ? make_float2(ox - v[k].x, oy - v[k].y) : make_float2(v[k].x + ox, v[k].y + oy);
  }
}

// forward column pass (as k_colA): rows j + 64 m in, rows C64::row(j, m) out
template <class Ld>
__global__ void __launch_bounds__(C64::NT, 1) k_colA64(Ld ld, float2* __restrict__ A, int nz_rows, int rev) {
  mgb_pdl_entry();
  extern __shared__ __align__(16) unsigned char smraw[];
  float2* sm = reinterpret_cast<float2*>(smraw);
  __shared__ double red[32];
  const int c = threadIdx.x % C64::TC, j = threadIdx.x / C64::TC;
  const int b = rev ? gridDim.y - 1 - blockIdx.y : blockIdx.y, col = blockIdx.x * C64::TC + c;
  const typename Ld::Ctx ctx = ld.prepare(b);
  float acc = 0.f;
  float2 v[32];
  constexpr int BL = Ld::kBatch < 8 ? Ld::kBatch : 8;
  typename Ld::Raw raw[2][BL];
#pragma unroll
  for (int i = 0; i < BL; ++i) {
    const int n1 = j + 64 * i;
    raw[0][i] = ld.fetch(ctx, b, (long long)n1 * N2 + col, n1 < nz_rows);
  }
#pragma unroll
  for (int m0 = 0; m0 < 32; m0 += BL) {
    const int cur = (m0 / BL) & 1;
    if (m0 + BL < 32) {
#pragma unroll
      for (int i = 0; i < BL; ++i) {
        const int n1 = j + 64 * (m0 + BL + i);
        raw[cur ^ 1][i] = ld.fetch(ctx, b, (long long)n1 * N2 + col, n1 < nz_rows);
      }
    }
#pragma unroll
    for (int i = 0; i < BL; ++i) {
      const int n1 = j + 64 * (m0 + i);
      v[m0 + i] = ld.finish(ctx, b, (long long)n1 * N2 + col, raw[cur][i], acc);
    }
  }
  if (Ld::kAccum) {
    const double t = block_sum((double)acc, red);
    if (threadIdx.x == 0) ld.commit(b, blockIdx.x, t);
  }
  col_fft64<false>(v, sm, c, j);
  const int r0 = C64::row(j, 0);
  twiddle_run<C64::LOGN, 32, false>(v, r0 * col, 32 * col);
  float2* dst = A + (long long)b * C64::N + col;
#pragma unroll
  for (int m = 0; m < 32; ++m) dst[(long long)(r0 + 32 * m) * N2] = v[m];
}

// inverse column pass (as k_colC): spectral rows j + 64 m in, time rows C64::row(j, m) out
template <class Ep>
__global__ void __launch_bounds__(C64::NT, 1) k_colC64(const float2* __restrict__ Bb, Ep ep, float scale, int out_rows,
                                                      int rev) {
  mgb_pdl_entry();
  extern __shared__ __align__(16) unsigned char smraw[];
  float2* sm = reinterpret_cast<float2*>(smraw);
  __shared__ double red[32];
  const int c = threadIdx.x % C64::TC, j = threadIdx.x / C64::TC;
  const int b = rev ? gridDim.y - 1 - blockIdx.y : blockIdx.y, col = blockIdx.x * C64::TC + c;
  const float2* src = Bb + (long long)b * C64::N + col;
  float2 v[32];
#pragma unroll
  for (int m = 0; m < 32; ++m) v[m] = src[(long long)(j + 64 * m) * N2];
  const typename Ep::Ctx ctx = ep.prepare(b);
  constexpr int B8 = ep_batch64<Ep>::value;  // epilogue batch (register budget at 512 threads)
  typename Ep::Raw raw[2][B8];
#pragma unroll
  for (int i = 0; i < B8; ++i) {
    const int n1 = C64::row(j, i);
    raw[0][i] = ep.fetch(ctx, b, (long long)n1 * N2 + col, n1 < out_rows);
  }
  col_fft64<true>(v, sm, c, j);
  float a0 = 0.f, a1 = 0.f;
#pragma unroll
  for (int m0 = 0; m0 < 32; m0 += B8) {
    const int cur = (m0 / B8) & 1;
    if (m0 + B8 < 32) {
#pragma unroll
      for (int i = 0; i < B8; ++i) {
        const int n1 = C64::row(j, m0 + B8 + i);
        raw[cur ^ 1][i] = ep.fetch(ctx, b, (long long)n1 * N2 + col, n1 < out_rows);
      }
    }
#pragma unroll
    for (int i = 0; i < B8; ++i) {
      const int n1 = C64::row(j, m0 + i);
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

}  // namespace fs2
