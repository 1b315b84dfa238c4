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
//
// Element j of sequence q lives at s[q * SEQ_STRIDE + pidx<PAD>(j) * ELEM_STRIDE].
// PAD (unit-stride layouts only) inserts one slot every 8 elements so the
// stride-R Stockham writes and the stride-N/R reads are bank-conflict free;
// a padded sequence occupies padded_len<N>() slots.
// SEQ_FAST: consecutive threads walk sequences (column tiles, ELEM_STRIDE > 1).
// Radix-8 passes (radix-4 / radix-2 first when log2 N is not a multiple of 3);
// one twiddle-table lookup per butterfly, higher powers by multiplication.
// Unnormalised; inverse uses conjugate twiddles.  Called by all NT threads;
// starts and ends with __syncthreads().

template <bool PAD>
__device__ __forceinline__ int pidx(int j) { return PAD ? j + (j >> 3) : j; }
template <int N>
constexpr int padded_len() { return N + N / 8; }

template <typename V>
__device__ __forceinline__ void dft4(V* v, bool inv) {
  const V a0 = cadd(v[0], v[2]), a1 = csub(v[0], v[2]), a2 = cadd(v[1], v[3]), a3 = csub(v[1], v[3]);
  const V a3r = inv ? cmul_pi(a3) : cmul_mi(a3);
  v[0] = cadd(a0, a2);
  v[2] = csub(a0, a2);
  v[1] = cadd(a1, a3r);
  v[3] = csub(a1, a3r);
}

template <typename V, typename R>
__device__ __forceinline__ void dft8(V* v, bool inv) {
  V e[4] = {v[0], v[2], v[4], v[6]}, o[4] = {v[1], v[3], v[5], v[7]};
  dft4(e, inv);
  dft4(o, inv);
  const R h = (R)0.70710678118654752440;
  V t[4];
  t[0] = o[0];
  if (!inv) {
    t[1] = cmk(h * (o[1].x + o[1].y), h * (o[1].y - o[1].x));
    t[2] = cmul_mi(o[2]);
    t[3] = cmk(h * (o[3].y - o[3].x), -h * (o[3].x + o[3].y));
  } else {
    t[1] = cmk(h * (o[1].x - o[1].y), h * (o[1].x + o[1].y));
    t[2] = cmul_pi(o[2]);
    t[3] = cmk(-h * (o[3].x + o[3].y), h * (o[3].x - o[3].y));
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    v[k] = cadd(e[k], t[k]);
    v[k + 4] = csub(e[k], t[k]);
  }
}

template <typename R, int RAD, int Ns, int N, int NSEQ, int NT, int SEQ_STRIDE, int ELEM_STRIDE, bool SEQ_FAST,
          bool PAD>
__device__ __forceinline__ void stockham_pass(typename Cplx<R>::T* s, bool inv) {
  typedef typename Cplx<R>::T V;
  constexpr int M = N / RAD;
  constexpr int NB = NSEQ * M;
  constexpr int BPT = (NB + NT - 1) / NT;
  V v[BPT][RAD];
#pragma unroll
  for (int i = 0; i < BPT; ++i) {
    const int b = threadIdx.x + i * NT;
    if (b < NB) {
      int q, j;
      if (SEQ_FAST) { q = b % NSEQ; j = b / NSEQ; } else { j = b % M; q = b / M; }
      const int k = j & (Ns - 1);
      V* base = s + q * SEQ_STRIDE;
#pragma unroll
      for (int r = 0; r < RAD; ++r) v[i][r] = base[pidx<PAD>(j + r * M) * ELEM_STRIDE];
      if constexpr (Ns > 1) {
        const V w1 = tw_lookup((MGB_TW_N / (RAD * Ns)) * k, inv, R());
        v[i][1] = cmul(v[i][1], w1);
        if (RAD >= 4) {
          const V w2 = cmul(w1, w1), w3 = cmul(w2, w1);
          v[i][2] = cmul(v[i][2], w2);
          v[i][3] = cmul(v[i][3], w3);
          if (RAD == 8) {
            const V w4 = cmul(w2, w2);
            v[i][4] = cmul(v[i][4], w4);
            v[i][5] = cmul(v[i][5], cmul(w4, w1));
            v[i][6] = cmul(v[i][6], cmul(w4, w2));
            v[i][7] = cmul(v[i][7], cmul(w4, w3));
          }
        }
      }
      if (RAD == 8) dft8<V, R>(v[i], inv);
      else if (RAD == 4) dft4(v[i], inv);
      else {
        const V t0 = v[i][0];
        v[i][0] = cadd(t0, v[i][1]);
        v[i][1] = csub(t0, v[i][1]);
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < BPT; ++i) {
    const int b = threadIdx.x + i * NT;
    if (b < NB) {
      int q, j;
      if (SEQ_FAST) { q = b % NSEQ; j = b / NSEQ; } else { j = b % M; q = b / M; }
      const int k = j & (Ns - 1);
      const int d = (j / Ns) * (RAD * Ns) + k;
      V* base = s + q * SEQ_STRIDE;
#pragma unroll
      for (int r = 0; r < RAD; ++r) base[pidx<PAD>(d + r * Ns) * ELEM_STRIDE] = v[i][r];
    }
  }
  __syncthreads();
}

// radix-8 passes with compile-time strides Ns = NS, 8 NS, ... < N
template <typename R, int NS, int N, int NSEQ, int NT, int SEQ_STRIDE, int ELEM_STRIDE, bool SEQ_FAST, bool PAD>
__device__ __forceinline__ void fft_passes8(typename Cplx<R>::T* s, bool inv) {
  if constexpr (NS < N) {
    stockham_pass<R, 8, NS, N, NSEQ, NT, SEQ_STRIDE, ELEM_STRIDE, SEQ_FAST, PAD>(s, inv);
    fft_passes8<R, NS * 8, N, NSEQ, NT, SEQ_STRIDE, ELEM_STRIDE, SEQ_FAST, PAD>(s, inv);
  }
}

template <typename R, int N, int NSEQ, int NT, int SEQ_STRIDE, int ELEM_STRIDE, bool SEQ_FAST, bool PAD = false>
__device__ __forceinline__ void smem_fft(typename Cplx<R>::T* s, bool inv) {
  static_assert((N & (N - 1)) == 0 && N >= 2, "pow2");
  static_assert(N <= MGB_TW_N, "twiddle table");
  static_assert(!PAD || ELEM_STRIDE == 1, "padding is for unit-stride layouts");
  constexpr int LOG = __builtin_ctz(N);
  constexpr int REM = LOG % 3;
  __syncthreads();
  constexpr int NS0 = (REM == 1) ? 2 : (REM == 2 ? 4 : 1);
  if constexpr (REM == 1) stockham_pass<R, 2, 1, N, NSEQ, NT, SEQ_STRIDE, ELEM_STRIDE, SEQ_FAST, PAD>(s, inv);
  if constexpr (REM == 2) stockham_pass<R, 4, 1, N, NSEQ, NT, SEQ_STRIDE, ELEM_STRIDE, SEQ_FAST, PAD>(s, inv);
  fft_passes8<R, NS0, N, NSEQ, NT, SEQ_STRIDE, ELEM_STRIDE, SEQ_FAST, PAD>(s, inv);
}

// ---------------------------------------------------------------------------
// four-step twiddles w_N^e, N = 2^l (11 <= l <= 22): two-level tables
#define MGB_FS_LMIN 11
#define MGB_FS_LMAX 22
extern __device__ float2 g_fs_lo[MGB_FS_LMAX - MGB_FS_LMIN + 1][2048];
extern __device__ float2 g_fs_hi[MGB_FS_LMAX - MGB_FS_LMIN + 1][2048];

template <int LOGN>
__device__ __forceinline__ float2 fs_twiddle(int e, bool inv) {
  static_assert(LOGN >= MGB_FS_LMIN && LOGN <= MGB_FS_LMAX, "four-step size");
  const float2 a = __ldg(&g_fs_lo[LOGN - MGB_FS_LMIN][e & 2047]);  // read-only path: loads may be hoisted
  const float2 b = __ldg(&g_fs_hi[LOGN - MGB_FS_LMIN][e >> 11]);
  float2 w = cmul(a, b);
  if (inv) w.y = -w.y;
  return w;
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

// Every library kernel is launched with programmatic dependent launch (PDL):
// its launch processing may overlap the previous kernel's drain, and it starts
// with mgb_pdl_entry() = griddepcontrol.wait (returns once the previous grid's
// results are visible; a no-op without PDL), so stream-order semantics hold.
// (An early griddepcontrol.launch_dependents was measured slower: waiting
// dependent CTAs took SM slots from the primary's last wave.)
__device__ __forceinline__ void mgb_pdl_entry() {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
}

template <typename... KArgs, typename... Args>
static inline cudaError_t mgb_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                                     Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

void mgb_count_launch();  // capi.cu (atomic)

// after EVERY kernel launch: error check + the host launch counter (mgb_launch_count)
#define MGB_CHECK_LAUNCH() \
  do { mgb_count_launch(); cudaError_t e__ = cudaGetLastError(); if (e__ != cudaSuccess) return 2; } while (0)
