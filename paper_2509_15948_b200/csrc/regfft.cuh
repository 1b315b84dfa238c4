// Register-resident DFT codelets (sm_100a).
//
// rdft<N, INV>(v): in-register, natural-order-in / natural-order-out DFT of
// N = 1..32 float2 values held by ONE thread (forward e^{-2 pi i nk/N},
// inverse conjugate, unnormalised).  Built by radix composition
// N = A x B (X[kb + B ka] = sum_na W_A^{na ka} W_N^{na kb} sum_nb x[na + A nb] W_B^{nb kb})
// from exact radix-2/4/8 butterflies; every twiddle index is a compile-time
// constant after unrolling, so the trivial ones (1, -i, (1-i)/sqrt2 ...) fold
// and the rest become immediates.  These are the building blocks of the
// shared-memory-light FFT passes in fs2.cuh: a length-(P*Q) transform done as
// one Q-point register DFT, one twiddle, ONE shared-memory exchange and one
// P-point register DFT.
#pragma once
#include "common.cuh"

namespace rf {

// cos / sin (2 pi k / 32)
__device__ __forceinline__ float c32(int k) {
  constexpr float t[32] = {
      1.0f, 9.807852804e-01f, 9.238795325e-01f, 8.314696123e-01f, 7.071067812e-01f, 5.555702330e-01f,
      3.826834324e-01f, 1.950903220e-01f, 0.0f, -1.950903220e-01f, -3.826834324e-01f, -5.555702330e-01f,
      -7.071067812e-01f, -8.314696123e-01f, -9.238795325e-01f, -9.807852804e-01f, -1.0f, -9.807852804e-01f,
      -9.238795325e-01f, -8.314696123e-01f, -7.071067812e-01f, -5.555702330e-01f, -3.826834324e-01f,
      -1.950903220e-01f, 0.0f, 1.950903220e-01f, 3.826834324e-01f, 5.555702330e-01f, 7.071067812e-01f,
      8.314696123e-01f, 9.238795325e-01f, 9.807852804e-01f};
  return t[k & 31];
}
__device__ __forceinline__ float s32(int k) { return c32(k - 8); }  // sin x = cos(x - pi/2)

// x * W_N^e (forward W = e^{-2 pi i / N}; INV: conjugate), N | 32, e constant after unrolling
template <int N, bool INV>
__device__ __forceinline__ float2 tw(float2 x, int e) {
  static_assert(32 % N == 0, "twiddle table covers N | 32");
  const int k = (e % N) * (32 / N);
  if (k == 0) return x;
  if (k == 16) return make_float2(-x.x, -x.y);
  if (k == 8) return INV ? make_float2(-x.y, x.x) : make_float2(x.y, -x.x);
  if (k == 24) return INV ? make_float2(x.y, -x.x) : make_float2(-x.y, x.x);
  const float c = c32(k), s = INV ? s32(k) : -s32(k);
  return make_float2(x.x * c - x.y * s, x.x * s + x.y * c);
}

template <bool INV>
__device__ __forceinline__ void r2(float2& a, float2& b) {
  const float2 t = a;
  a = make_float2(t.x + b.x, t.y + b.y);
  b = make_float2(t.x - b.x, t.y - b.y);
}

template <int N, bool INV>
struct Dft;

template <bool INV>
struct Dft<1, INV> {
  static __device__ __forceinline__ void run(float2*) {}
};
template <bool INV>
struct Dft<2, INV> {
  static __device__ __forceinline__ void run(float2* v) { r2<INV>(v[0], v[1]); }
};
template <bool INV>
struct Dft<4, INV> {
  static __device__ __forceinline__ void run(float2* v) {
    r2<INV>(v[0], v[2]);
    r2<INV>(v[1], v[3]);
    v[3] = tw<4, INV>(v[3], 1);
    r2<INV>(v[0], v[1]);
    r2<INV>(v[2], v[3]);
    const float2 t = v[1];  // bit reversal: [0 2 1 3]
    v[1] = v[2];
    v[2] = t;
  }
};

// N = A * B composition
template <int A, int B, bool INV>
__device__ __forceinline__ void dft_ab(float2* v) {
  constexpr int N = A * B;
  float2 t[A][B];
#pragma unroll
  for (int na = 0; na < A; ++na) {
#pragma unroll
    for (int nb = 0; nb < B; ++nb) t[na][nb] = v[na + A * nb];
    Dft<B, INV>::run(t[na]);
#pragma unroll
    for (int kb = 0; kb < B; ++kb) t[na][kb] = tw<N, INV>(t[na][kb], na * kb);
  }
#pragma unroll
  for (int kb = 0; kb < B; ++kb) {
    float2 s[A];
#pragma unroll
    for (int na = 0; na < A; ++na) s[na] = t[na][kb];
    Dft<A, INV>::run(s);
#pragma unroll
    for (int ka = 0; ka < A; ++ka) v[kb + B * ka] = s[ka];
  }
}

template <bool INV>
struct Dft<8, INV> {
  static __device__ __forceinline__ void run(float2* v) { dft_ab<2, 4, INV>(v); }
};
template <bool INV>
struct Dft<16, INV> {
  static __device__ __forceinline__ void run(float2* v) { dft_ab<4, 4, INV>(v); }
};
template <bool INV>
struct Dft<32, INV> {
  static __device__ __forceinline__ void run(float2* v) { dft_ab<4, 8, INV>(v); }
};

template <int N, bool INV>
__device__ __forceinline__ void rdft(float2* v) { Dft<N, INV>::run(v); }

// W_M^e for runtime e (M = 2^logM <= 2^22) from the two-level four-step tables
template <int LOGM>
__device__ __forceinline__ float2 wexp(int e, bool inv) {
  if constexpr (LOGM < MGB_FS_LMIN) {
    return wexp<MGB_FS_LMIN>(e << (MGB_FS_LMIN - LOGM), inv);
  } else {
    return fs_twiddle<LOGM>(e & ((1 << LOGM) - 1), inv);
  }
}

}  // namespace rf
