// Hand-written batched complex FFTs for sm_100a (no cuFFT on the product path).
//
// * N <= 8192: one kernel, a tile of sequences per CTA, shared-memory
//   Stockham radix-4/2 (common.cuh: smem_fft).
// * N  > 8192: four-step, N = N1 * N2, natural order in and out:
//     column pass: per column n2, N1-point FFT down the column (stride N2),
//                  twiddle w_N^{k1 n2}, written in place of the column;
//     row pass:    per row k1, N2-point FFT along the row (contiguous),
//                  stored transposed to k1 + N1*k2 (coalesced in chunks of TR).
//   Each pass reads and writes the whole array once (2 HBM sweeps / transform;
//   at the level batch sizes used here the scratch array mostly stays in L2).
//
// The convolution helpers implement mg/engine.py:549-585 (fft_conv) for
// stereo rows: the two real channels ride one complex transform
// (z = left + i*right), and the per-channel spectra are separated with the
// Hermitian pairing X_l[k] = (Z[k] + conj Z[-k])/2, X_r[k] = (Z[k] - conj Z[-k])/2i.
#include "common.cuh"
#include "tables.cuh"
#include "mgb_internal.h"

__device__ float2 g_tw32[MGB_TW_N];
__device__ double2 g_tw64[MGB_TW_N];
__device__ float2 g_fs_lo[MGB_FS_LMAX - MGB_FS_LMIN + 1][2048];
__device__ float2 g_fs_hi[MGB_FS_LMAX - MGB_FS_LMIN + 1][2048];
// FIR-synthesis tables (float64): the symmetric Hann of n = 2047 (EQ); cos(2 pi j / n) and Hann of n = 39 (colour)
__device__ double g_hann2047[MGB_EQ_LEN];
__device__ double g_cos39[MGB_COLOR_LEN], g_hann39[MGB_COLOR_LEN];

__global__ void k_init_fir_tables() {
  mgb_pdl_entry();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < MGB_EQ_LEN) {
    g_hann2047[j] = 0.5 - 0.5 * cospi(2.0 * j / (double)(MGB_EQ_LEN - 1));
  }
  if (j < MGB_COLOR_LEN) {
    g_cos39[j] = cospi(2.0 * j / (double)MGB_COLOR_LEN);
    g_hann39[j] = 0.5 - 0.5 * cospi(2.0 * j / (double)(MGB_COLOR_LEN - 1));
  }
}

__global__ void k_init_fs_twiddles() {
  mgb_pdl_entry();
  const int l = blockIdx.y, j = blockIdx.x * blockDim.x + threadIdx.x;
  const long long N = 1LL << (l + MGB_FS_LMIN);
  if (j < 2048) {
    double s, c;
    sincospi(-2.0 * (double)j / (double)N, &s, &c);
    g_fs_lo[l][j] = make_float2((float)c, (float)s);
    const long long e = (2048LL * j) % N;
    sincospi(-2.0 * (double)e / (double)N, &s, &c);
    g_fs_hi[l][j] = make_float2((float)c, (float)s);
  }
}

__global__ void k_init_twiddles() {
  mgb_pdl_entry();
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < MGB_TW_N) {
    double s, c;
    sincospi(-2.0 * (double)j / (double)MGB_TW_N, &s, &c);
    g_tw64[j] = make_double2(c, s);
    g_tw32[j] = make_float2((float)c, (float)s);
  }
}

int mgb_init_device(cudaStream_t st) {
  mgb_launch(k_init_twiddles, dim3(MGB_TW_N / 256), dim3(256), 0, st);
  MGB_CHECK_LAUNCH();
  mgb_launch(k_init_fir_tables, dim3((MGB_EQ_LEN + 255) / 256), dim3(256), 0, st);
  MGB_CHECK_LAUNCH();
  mgb_launch(k_init_fs_twiddles, dim3(dim3(2048 / 256, MGB_FS_LMAX - MGB_FS_LMIN + 1)), dim3(256), 0, st);
  MGB_CHECK_LAUNCH();
  return 0;
}

// ---------------------------------------------------------------------------
// single-kernel small FFT: SEQ sequences of length N per CTA

template <int N, int SEQ, int NT>
__global__ void __launch_bounds__(NT) k_fft_small(const float2* __restrict__ in, float2* __restrict__ out,
                                                  int batch, bool inv, float scale) {
  mgb_pdl_entry();
  extern __shared__ __align__(16) unsigned char smraw[];
  float2* sm = reinterpret_cast<float2*>(smraw);
  const long long b0 = (long long)blockIdx.x * SEQ;
  constexpr int P = padded_len<N>();
  for (int i = threadIdx.x; i < SEQ * N; i += NT) {
    const long long b = b0 + i / N;
    sm[(i / N) * P + pidx<true>(i % N)] = (b < batch) ? in[b0 * N + i] : make_float2(0.f, 0.f);
  }
  smem_fft<float, N, SEQ, NT, P, 1, false, true>(sm, inv);
  for (int i = threadIdx.x; i < SEQ * N; i += NT) {
    const long long b = b0 + i / N;
    if (b < batch) { float2 v = sm[(i / N) * P + pidx<true>(i % N)]; v.x *= scale; v.y *= scale; out[b0 * N + i] = v; }
  }
}

// ---------------------------------------------------------------------------
// four-step passes

template <int N1, int N2, int TC, int NT>
__global__ void __launch_bounds__(NT) k_fft_col(const float2* __restrict__ in, float2* __restrict__ out, bool inv) {
  mgb_pdl_entry();
  extern __shared__ __align__(16) unsigned char smraw[];
  float2* sm = reinterpret_cast<float2*>(smraw);  // [N1][TC]
  const long long N = (long long)N1 * N2;
  const int c0 = blockIdx.x * TC;
  const float2* src = in + (long long)blockIdx.y * N;
  float2* dst = out + (long long)blockIdx.y * N;
  for (int i = threadIdx.x; i < TC * N1; i += NT) {
    const int c = i % TC, n1 = i / TC;
    sm[i] = src[(long long)n1 * N2 + c0 + c];
  }
  smem_fft<float, N1, TC, NT, 1, TC, true>(sm, inv);
  for (int i = threadIdx.x; i < TC * N1; i += NT) {
    const int c = i % TC, k1 = i / TC;
    const float2 w = twiddle_exact((long long)k1 * (c0 + c), N, inv, 0.f);
    dst[(long long)k1 * N2 + c0 + c] = cmul(sm[i], w);
  }
}

template <int N1, int N2, int TR, int NT>
__global__ void __launch_bounds__(NT) k_fft_row(const float2* __restrict__ in, float2* __restrict__ out, bool inv,
                                                float scale) {
  mgb_pdl_entry();
  extern __shared__ __align__(16) unsigned char smraw[];
  float2* sm = reinterpret_cast<float2*>(smraw);  // [TR][padded N2]
  constexpr int P = padded_len<N2>();
  const long long N = (long long)N1 * N2;
  const int r0 = blockIdx.x * TR;
  const float2* src = in + (long long)blockIdx.y * N;
  float2* dst = out + (long long)blockIdx.y * N;
  for (int i = threadIdx.x; i < TR * N2; i += NT) {
    const int n2 = i % N2, r = i / N2;
    sm[r * P + pidx<true>(n2)] = src[(long long)(r0 + r) * N2 + n2];
  }
  smem_fft<float, N2, TR, NT, P, 1, false, true>(sm, inv);
  for (int i = threadIdx.x; i < TR * N2; i += NT) {
    const int r = i % TR, k2 = i / TR;
    float2 v = sm[r * P + pidx<true>(k2)];
    v.x *= scale;
    v.y *= scale;
    dst[(long long)(r0 + r) + (long long)N1 * k2] = v;
  }
}

template <int N, int SEQ, int NT>
static int launch_small(const float2* in, float2* out, int batch, bool inv, float scale, cudaStream_t st) {
  const size_t smem = sizeof(float2) * SEQ * padded_len<N>();
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_fft_small<N, SEQ, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  mgb_launch(k_fft_small<N, SEQ, NT>, dim3((batch + SEQ - 1) / SEQ), dim3(NT), smem, st, in, out, batch, inv, scale);
  MGB_CHECK_LAUNCH();
  return 0;
}

template <int N1, int N2>
static int launch_four_step(const float2* in, float2* out, float2* tmp, int batch, bool inv, float scale,
                            cudaStream_t st) {
  constexpr int TC = (N1 >= 1024) ? 8 : 16;
  constexpr int TR = (N2 >= 4096) ? 2 : (N2 >= 2048 ? 4 : 8);
  constexpr int NT = 256;
  const size_t smc = sizeof(float2) * TC * N1;
  const size_t smr = sizeof(float2) * TR * padded_len<N2>();
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_fft_col<N1, N2, TC, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smc);
    cudaFuncSetAttribute(k_fft_row<N1, N2, TR, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smr);
    attr = true;
  }
  mgb_launch(k_fft_col<N1, N2, TC, NT>, dim3(dim3(N2 / TC, batch)), dim3(NT), smc, st, in, tmp, inv);
  MGB_CHECK_LAUNCH();
  mgb_launch(k_fft_row<N1, N2, TR, NT>, dim3(dim3(N1 / TR, batch)), dim3(NT), smr, st, tmp, out, inv, scale);
  MGB_CHECK_LAUNCH();
  return 0;
}

// out may alias in; tmp must hold batch*N complex when N > 8192.
int mgb_fft_c2c(const float2* in, float2* out, float2* tmp, int batch, int log2n, int inverse, float scale,
                cudaStream_t st) {
  const bool inv = inverse != 0;
  switch (log2n) {
    case 5: return launch_small<32, 32, 256>(in, out, batch, inv, scale, st);
    case 6: return launch_small<64, 16, 256>(in, out, batch, inv, scale, st);
    case 7: return launch_small<128, 8, 256>(in, out, batch, inv, scale, st);
    case 8: return launch_small<256, 4, 256>(in, out, batch, inv, scale, st);
    case 9: return launch_small<512, 2, 256>(in, out, batch, inv, scale, st);
    case 10: return launch_small<1024, 1, 256>(in, out, batch, inv, scale, st);
    case 11: return launch_small<2048, 1, 512>(in, out, batch, inv, scale, st);
    case 12: return launch_small<4096, 1, 512>(in, out, batch, inv, scale, st);
    case 13: return launch_small<8192, 1, 1024>(in, out, batch, inv, scale, st);
    case 14: return launch_four_step<16, 1024>(in, out, tmp, batch, inv, scale, st);
    case 15: return launch_four_step<32, 1024>(in, out, tmp, batch, inv, scale, st);
    case 16: return launch_four_step<64, 1024>(in, out, tmp, batch, inv, scale, st);
    case 17: return launch_four_step<128, 1024>(in, out, tmp, batch, inv, scale, st);
    case 18: return launch_four_step<256, 1024>(in, out, tmp, batch, inv, scale, st);
    case 19: return launch_four_step<512, 1024>(in, out, tmp, batch, inv, scale, st);
    case 20: return launch_four_step<1024, 1024>(in, out, tmp, batch, inv, scale, st);
    case 21: return launch_four_step<1024, 2048>(in, out, tmp, batch, inv, scale, st);
    case 22: return launch_four_step<1024, 4096>(in, out, tmp, batch, inv, scale, st);
    default: return 1;
  }
}

// ---------------------------------------------------------------------------
// FFT-convolution helpers (stereo rows packed as left + i*right)

// Z[b][k] = (u_l, u_r)[k] for k < L, 0 up to N
__global__ void k_pack_rows(const float* const* __restrict__ rows, float2* __restrict__ Z, int L, long long N) {
  mgb_pdl_entry();
  const int b = blockIdx.y;
  const float* u = rows[b];
  float2* z = Z + (long long)b * N;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < N; k += (long long)gridDim.x * blockDim.x)
    z[k] = (k < L) ? make_float2(u[k], u[L + k]) : make_float2(0.f, 0.f);
}

int mgb_pack_rows(const float* const* rows, float2* Z, int B, int L, long long N, cudaStream_t st) {
  const int blocks = (int)min((N + 255) / 256, (long long)1184);
  mgb_launch(k_pack_rows, dim3(dim3(blocks, B)), dim3(256), 0, st, rows, Z, L, N);
  MGB_CHECK_LAUNCH();
  return 0;
}

// Pairwise spectral products.
//  mode 0: Q = X_l H_l + i X_r H_r          (forward conv)
//  mode 1: Q = G_l conj(H_l) + i G_r conj(H_r)   (adjoint wrt x)
// A second optional output (Q2 with operand C) applies mode 1 against C:
//  Q2 = G_l conj(C_l) + i G_r conj(C_r)     (adjoint wrt h, C = X)
__device__ __forceinline__ void split_pair(float2 zk, float2 zp, float2& a, float2& b) {
  // a = (zk + conj zp)/2 ; b = (zk - conj zp)/(2i)
  a = make_float2(0.5f * (zk.x + zp.x), 0.5f * (zk.y - zp.y));
  const float2 d = make_float2(0.5f * (zk.x - zp.x), 0.5f * (zk.y + zp.y));
  b = make_float2(d.y, -d.x);
}

__global__ void k_spec_pair(const float2* __restrict__ Z, const float2* __restrict__ H, float2* __restrict__ Q,
                            const float2* __restrict__ C, float2* __restrict__ Q2, long long N, int mode) {
  mgb_pdl_entry();
  const int b = blockIdx.y;
  const long long off = (long long)b * N;
  const long long half = N / 2;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k <= half;
       k += (long long)gridDim.x * blockDim.x) {
    const long long p = (N - k) & (N - 1);
    float2 zl, zr, hl, hr;
    split_pair(Z[off + k], Z[off + p], zl, zr);
    split_pair(H[off + k], H[off + p], hl, hr);
    float2 y1, y2;
    if (mode == 0) { y1 = cmul(zl, hl); y2 = cmul(zr, hr); }
    else { y1 = cmulc(zl, hl); y2 = cmulc(zr, hr); }
    // Q[k] = y1 + i y2 ; Q[p] = conj(y1) + i conj(y2)
    Q[off + k] = make_float2(y1.x - y2.y, y1.y + y2.x);
    if (p != k) Q[off + p] = make_float2(y1.x + y2.y, -y1.y + y2.x);
    if (Q2) {
      float2 cl, cr;
      split_pair(C[off + k], C[off + p], cl, cr);
      const float2 v1 = cmulc(zl, cl), v2 = cmulc(zr, cr);
      Q2[off + k] = make_float2(v1.x - v2.y, v1.y + v2.x);
      if (p != k) Q2[off + p] = make_float2(v1.x + v2.y, -v1.y + v2.x);
    }
  }
}

int mgb_spec_pair(const float2* Z, const float2* H, float2* Q, const float2* C, float2* Q2, int B, long long N,
                  int mode, cudaStream_t st) {
  const int blocks = (int)min((N / 2 + 256) / 256, (long long)1184);
  mgb_launch(k_spec_pair, dim3(dim3(blocks, B)), dim3(256), 0, st, Z, H, Q, C, Q2, N, mode);
  MGB_CHECK_LAUNCH();
  return 0;
}
