// Shared device helpers for libmixgraph_b200 (sm_100a).
//
// * complex helpers over float2 / double2
// * a twiddle table e^{-2*pi*i*j/TW_N} (fp64-accurate) in device global memory,
//   initialised once per device by mgb_init()
// * a shared-memory Stockham radix-4/2 FFT that runs a tile of independent
//   power-of-two sequences in place (all reads of a pass land in registers
//   before the barrier, then all writes).  It is the building block of the
//   four-step large FFT (fft.cu), the MRSTFT frame transforms (loss.cu) and
//   the small FIR-synthesis transforms.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define MGB_TW_LOG 14
#define MGB_TW_N (1 << MGB_TW_LOG)

extern __device__ float2 g_tw32[MGB_TW_N];
extern __device__ double2 g_tw64[MGB_TW_N];

template <typename R> struct Cplx;
template <> struct Cplx<float> { typedef float2 T; };
template <> struct Cplx<double> { typedef double2 T; };

__device__ __forceinline__ float2 cmk(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ double2 cmk(double a, double b) { return make_double2(a, b); }

template <typename V> __device__ __forceinline__ V cadd(V a, V b) { V r; r.x = a.x + b.x; r.y = a.y + b.y; return r; }
template <typename V> __device__ __forceinline__ V csub(V a, V b) { V r; r.x = a.x - b.x; r.y = a.y - b.y; return r; }
template <typename V> __device__ __forceinline__ V cmul(V a, V b) {
  V r; r.x = a.x * b.x - a.y * b.y; r.y = a.x * b.y + a.y * b.x; return r;
}
template <typename V> __device__ __forceinline__ V cmulc(V a, V b) {  // a * conj(b)
  V r; r.x = a.x * b.x + a.y * b.y; r.y = a.y * b.x - a.x * b.y; return r;
}
template <typename V> __device__ __forceinline__ V cconj(V a) { V r; r.x = a.x; r.y = -a.y; return r; }
template <typename V, typename R> __device__ __forceinline__ V cscale(V a, R s) { V r; r.x = a.x * s; r.y = a.y * s; return r; }
// multiply by -i (dir=+1 forward) or +i (inverse)
template <typename V> __device__ __forceinline__ V cmul_mi(V a) { V r; r.x = a.y; r.y = -a.x; return r; }
template <typename V> __device__ __forceinline__ V cmul_pi(V a) { V r; r.x = -a.y; r.y = a.x; return r; }

__device__ __forceinline__ float2 tw_lookup(int idx, bool inv, float) {
  float2 w = g_tw32[idx];
  if (inv) w.y = -w.y;
  return w;
}
__device__ __forceinline__ double2 tw_lookup(int idx, bool inv, double) {
  double2 w = g_tw64[idx];
  if (inv) w.y = -w.y;
  return w;
}

// e^{-+2 pi i e / n} with exact integer argument reduction (e < n <= 2^24)
__device__ __forceinline__ float2 twiddle_exact(long long e, long long n, bool inv, float) {
  float s, c;
  e %= n;
  sincospif(-2.0f * (float)e / (float)n, &s, &c);
  return make_float2(c, inv ? -s : s);
}
__device__ __forceinline__ double2 twiddle_exact(long long e, long long n, bool inv, double) {
  double s, c;
  e %= n;
  sincospi(-2.0 * (double)e / (double)n, &s, &c);
  return make_double2(c, inv ? -s : s);
}

// ---------------------------------------------------------------------------
// Shared-memory Stockham FFT over a tile of NSEQ sequences of length N (pow2).
// Element j of sequence q lives at s[q * SEQ_STRIDE + j * ELEM_STRIDE].
// SEQ_FAST: consecutive threads walk sequences (use when ELEM_STRIDE > 1 and
// sequences are adjacent in memory, i.e. column tiles).
// Unnormalised; inverse uses conjugate twiddles.  Must be called by all
// NT threads of the block; ends with a __syncthreads().
template <typename R, int N, int NSEQ, int NT, int SEQ_STRIDE, int ELEM_STRIDE, bool SEQ_FAST>
__device__ __forceinline__ void smem_fft(typename Cplx<R>::T* s, bool inv) {
  typedef typename Cplx<R>::T V;
  static_assert((N & (N - 1)) == 0 && N >= 2, "pow2");
  static_assert(N <= MGB_TW_N, "twiddle table");
  constexpr int N4 = (N >= 4) ? N / 4 : 1;
  constexpr int NB4 = NSEQ * N4;                            // radix-4 butterflies per pass
  constexpr int BPT4 = (NB4 + NT - 1) / NT;
  constexpr int NB2 = NSEQ * (N / 2);
  constexpr int BPT2 = (NB2 + NT - 1) / NT;
  const int tid = threadIdx.x;
  int Ns = 1;
  __syncthreads();
  // radix-4 passes
  if constexpr (N >= 4) for (; Ns * 4 <= N; Ns *= 4) {
    V v[BPT4][4];
#pragma unroll
    for (int i = 0; i < BPT4; ++i) {
      const int b = tid + i * NT;
      if (b < NB4) {
        int q, j;
        if (SEQ_FAST) { q = b % NSEQ; j = b / NSEQ; } else { j = b % (N / 4); q = b / (N / 4); }
        const int k = j & (Ns - 1);
        V* base = s + q * SEQ_STRIDE;
#pragma unroll
        for (int r = 0; r < 4; ++r) v[i][r] = base[(j + r * (N / 4)) * ELEM_STRIDE];
        if (Ns > 1) {
          const int step = (MGB_TW_N / (4 * Ns)) * k;
          v[i][1] = cmul(v[i][1], tw_lookup(step, inv, R()));
          v[i][2] = cmul(v[i][2], tw_lookup(2 * step, inv, R()));
          v[i][3] = cmul(v[i][3], tw_lookup(3 * step, inv, R()));
        }
        V a0 = cadd(v[i][0], v[i][2]), a1 = csub(v[i][0], v[i][2]);
        V a2 = cadd(v[i][1], v[i][3]), a3 = csub(v[i][1], v[i][3]);
        V a3r = inv ? cmul_pi(a3) : cmul_mi(a3);
        v[i][0] = cadd(a0, a2);
        v[i][2] = csub(a0, a2);
        v[i][1] = cadd(a1, a3r);
        v[i][3] = csub(a1, a3r);
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < BPT4; ++i) {
      const int b = tid + i * NT;
      if (b < NB4) {
        int q, j;
        if (SEQ_FAST) { q = b % NSEQ; j = b / NSEQ; } else { j = b % (N / 4); q = b / (N / 4); }
        const int k = j & (Ns - 1);
        const int d = (j / Ns) * (4 * Ns) + k;
        V* base = s + q * SEQ_STRIDE;
#pragma unroll
        for (int r = 0; r < 4; ++r) base[(d + r * Ns) * ELEM_STRIDE] = v[i][r];
      }
    }
    __syncthreads();
  }
  // final radix-2 pass when log2(N) is odd
  if (Ns < N) {
    V v[BPT2][2];
#pragma unroll
    for (int i = 0; i < BPT2; ++i) {
      const int b = tid + i * NT;
      if (b < NB2) {
        int q, j;
        if (SEQ_FAST) { q = b % NSEQ; j = b / NSEQ; } else { j = b % (N / 2); q = b / (N / 2); }
        const int k = j & (Ns - 1);
        V* base = s + q * SEQ_STRIDE;
        v[i][0] = base[j * ELEM_STRIDE];
        v[i][1] = base[(j + N / 2) * ELEM_STRIDE];
        if (Ns > 1) v[i][1] = cmul(v[i][1], tw_lookup((MGB_TW_N / (2 * Ns)) * k, inv, R()));
        V t0 = cadd(v[i][0], v[i][1]), t1 = csub(v[i][0], v[i][1]);
        v[i][0] = t0;
        v[i][1] = t1;
      }
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < BPT2; ++i) {
      const int b = tid + i * NT;
      if (b < NB2) {
        int q, j;
        if (SEQ_FAST) { q = b % NSEQ; j = b / NSEQ; } else { j = b % (N / 2); q = b / (N / 2); }
        const int k = j & (Ns - 1);
        const int d = (j / Ns) * (2 * Ns) + k;
        V* base = s + q * SEQ_STRIDE;
        base[d * ELEM_STRIDE] = v[i][0];
        base[(d + Ns) * ELEM_STRIDE] = v[i][1];
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// block reductions (fp64 accumulation)

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// sum over the block; result valid in thread 0. scratch: >= 32 doubles of smem
__device__ __forceinline__ double block_sum(double v, double* scratch) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) scratch[wid] = v;
  __syncthreads();
  double r = 0.0;
  if (wid == 0) {
    r = (lane < (int)((blockDim.x + 31) >> 5)) ? scratch[lane] : 0.0;
    r = warp_sum(r);
  }
  return r;
}

// logistic in float64 with scipy.special.expit's branch structure
__device__ __forceinline__ double expit64(double x) {
  if (x >= 0.0) return 1.0 / (1.0 + exp(-x));
  const double e = exp(x);
  return e / (1.0 + e);
}

__device__ __forceinline__ double softplus64(double x) {  // np.logaddexp(0, x)
  return fmax(x, 0.0) + log1p(exp(-fabs(x)));
}

#define MGB_CHECK_LAUNCH() \
  do { cudaError_t e__ = cudaGetLastError(); if (e__ != cudaSuccess) return 2; } while (0)
