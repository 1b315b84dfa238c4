// Elementwise levels: gain/pan (g), stereo imager (s), dry/wet weights and the
// mix/output bus sums.  Coalesced streaming kernels; dry/wet is fused into the
// processor's epilogue; all parameter reductions accumulate in float64 via
// per-CTA partials + a deterministic finalize (no atomics).
//
//  g: ybar[c] = e^{p_c} u[c]                           mg/processors.py:97-99
//  s: ybar = ((l+r) +- e^p (l-r)) / 2                   mg/processors.py:102-108
//  dry/wet: y = w ybar + (1-w) u, y = u exactly if w==0 mg/processors.py:61-73
//  bus: out[s] = sum of its fan-in rows                 mg/engine.py:439-450
#include "common.cuh"
#include "mgb_internal.h"

namespace {

constexpr int NT = 256;
constexpr int KP = 4;      // partial slots per CTA
#ifndef MGB_GS_VPT
#define MGB_GS_VPT 2
#endif
constexpr int VPT = MGB_GS_VPT;  // float4 (or scalar groups of 4) per thread per channel
constexpr int CHUNK = NT * VPT * 4;  // samples per channel per CTA

__host__ __device__ inline int simple_nblk(int L) {
  const int n = (L + CHUNK - 1) / CHUNK;
  return n < 1 ? 1 : n;
}

// Four consecutive samples n..n+3 of both channels: float4 when the rows are
// 16-byte aligned and L % 4 == 0 (VEC), else guarded scalars.
template <bool VEC>
__device__ __forceinline__ void ld4(const float* __restrict__ p, long long n, int L, float (&v)[4]) {
  if (VEC) {
    const float4 t = __ldg(reinterpret_cast<const float4*>(p + n));
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = (n + i < L) ? __ldg(p + n + i) : 0.f;
  }
}
template <bool VEC>
__device__ __forceinline__ void st4(float* __restrict__ p, long long n, int L, const float (&v)[4]) {
  if (VEC) {
    *reinterpret_cast<float4*>(p + n) = make_float4(v[0], v[1], v[2], v[3]);
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (n + i < L) p[n + i] = v[i];
  }
}

// forward: yo = w*ybar + (1-w)*u, exactly u when w == 0
template <char TAG, bool VEC>
__global__ void __launch_bounds__(NT) k_gs_fwd(const float* const* __restrict__ u_rows,
                                               const double* __restrict__ bank, const int* __restrict__ prow,
                                               const int* __restrict__ widx, const double* __restrict__ w,
                                               float* __restrict__ y, int L) {
  mgb_pdl_entry();
  const int b = blockIdx.y;
  const float* u = u_rows[b];
  float* yo = y + (size_t)b * 2 * L;
  const double wv = w ? w[widx[b]] : 1.0;
  const bool bypass = (wv == 0.0);
  float c0, c1, k = 0.f, wf = 0.f, om = 0.f;
  if (TAG == 'g') {
    const double g0 = exp(bank[(size_t)prow[b] * 2]), g1 = exp(bank[(size_t)prow[b] * 2 + 1]);
    c0 = bypass ? 1.f : (float)(wv * g0 + (1.0 - wv));
    c1 = bypass ? 1.f : (float)(wv * g1 + (1.0 - wv));
  } else {
    k = (float)exp(bank[prow[b]]);
    wf = (float)wv;
    om = (float)(1.0 - wv);
    c0 = c1 = 1.f;
  }
  const long long base = (long long)blockIdx.x * CHUNK;
  float l[VPT][4], r[VPT][4];
#pragma unroll
  for (int j = 0; j < VPT; ++j) {
    const long long n = base + 4LL * (threadIdx.x + j * NT);
    if (n < L) {
      ld4<VEC>(u, n, L, l[j]);
      ld4<VEC>(u + L, n, L, r[j]);
    }
  }
#pragma unroll
  for (int j = 0; j < VPT; ++j) {
    const long long n = base + 4LL * (threadIdx.x + j * NT);
    if (n >= L) continue;
    float ol[4], orr[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (bypass) {
        ol[i] = l[j][i];
        orr[i] = r[j][i];
      } else if (TAG == 'g') {
        ol[i] = c0 * l[j][i];
        orr[i] = c1 * r[j][i];
      } else {
        const float mid = l[j][i] + r[j][i], side = k * (l[j][i] - r[j][i]);
        const float yl = (mid + side) * 0.5f, yr = (mid - side) * 0.5f;
        ol[i] = wf * yl + om * l[j][i];
        orr[i] = wf * yr + om * r[j][i];
      }
    }
    st4<VEC>(yo, n, L, ol);
    st4<VEC>(yo + L, n, L, orr);
  }
}

// backward: gu and the two per-row reductions (g: sum gy_c u_c per channel;
// s: sum (l-r)(gl-gr) for dp and sum g.(ybar-u) for dw), float64 per CTA
template <char TAG, bool VEC>
__global__ void __launch_bounds__(NT) k_gs_bwd(const float* const* __restrict__ u_rows,
                                               const float* const* __restrict__ gy_rows,
                                               const double* __restrict__ bank, const int* __restrict__ prow,
                                               const int* __restrict__ widx, const double* __restrict__ w,
                                               float* __restrict__ gu, double* __restrict__ part, int L) {
  mgb_pdl_entry();
  __shared__ double scratch[32];
  const int b = blockIdx.y;
  const float* u = u_rows[b];
  const float* gy = gy_rows[b];
  float* go = gu ? gu + (size_t)b * 2 * L : nullptr;  // null: input gradient not requested
  const double wv = w ? w[widx[b]] : 1.0;
  const bool bypass = (wv == 0.0);
  float c0 = 1.f, c1 = 1.f, k = 0.f, wf = 0.f, om = 0.f;
  if (TAG == 'g') {
    const double g0 = exp(bank[(size_t)prow[b] * 2]), g1 = exp(bank[(size_t)prow[b] * 2 + 1]);
    c0 = (float)(wv * g0 + (1.0 - wv));
    c1 = (float)(wv * g1 + (1.0 - wv));
  } else {
    k = (float)exp(bank[prow[b]]);
    wf = (float)wv;
    om = (float)(1.0 - wv);
  }
  const long long base = (long long)blockIdx.x * CHUNK;
  float gl[VPT][4], gr[VPT][4], l[VPT][4], r[VPT][4];
#pragma unroll
  for (int j = 0; j < VPT; ++j) {
    const long long n = base + 4LL * (threadIdx.x + j * NT);
    if (n < L) {
      ld4<VEC>(gy, n, L, gl[j]);
      ld4<VEC>(gy + L, n, L, gr[j]);
      if (!bypass) {
        ld4<VEC>(u, n, L, l[j]);
        ld4<VEC>(u + L, n, L, r[j]);
      }
    }
  }
  float s0 = 0.f, s1 = 0.f;
#pragma unroll
  for (int j = 0; j < VPT; ++j) {
    const long long n = base + 4LL * (threadIdx.x + j * NT);
    if (n >= L) continue;
    float ol[4], orr[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const bool in = VEC || (n + i < L);
      if (bypass) {
        ol[i] = gl[j][i];
        orr[i] = gr[j][i];
      } else if (TAG == 'g') {
        ol[i] = c0 * gl[j][i];
        orr[i] = c1 * gr[j][i];
        if (in) {
          s0 = fmaf(gl[j][i], l[j][i], s0);
          s1 = fmaf(gr[j][i], r[j][i], s1);
        }
      } else {
        const float dl = wf * gl[j][i], dr = wf * gr[j][i];  // d ybar
        const float sm = 0.5f * (dl + dr), sd = 0.5f * k * (dl - dr);
        ol[i] = om * gl[j][i] + sm + sd;
        orr[i] = om * gr[j][i] + sm - sd;
        if (in) {
          const float mid = l[j][i] + r[j][i], side = k * (l[j][i] - r[j][i]);
          const float yl = (mid + side) * 0.5f, yr = (mid - side) * 0.5f;
          s0 = fmaf(l[j][i] - r[j][i], gl[j][i] - gr[j][i], s0);
          s1 = fmaf(gl[j][i], yl - l[j][i], fmaf(gr[j][i], yr - r[j][i], s1));
        }
      }
    }
    if (go) {
      st4<VEC>(go, n, L, ol);
      st4<VEC>(go + L, n, L, orr);
    }
  }
  const double t0 = block_sum((double)s0, scratch);
  const double t1 = block_sum((double)s1, scratch);
  if (threadIdx.x == 0) {
    double* pp = part + ((size_t)b * gridDim.x + blockIdx.x) * KP;
    pp[0] = t0;
    pp[1] = t1;
  }
}

// one CTA per row: deterministic fixed-order float64 sum of the CTA partials
__global__ void k_gs_finalize(char tag, const double* __restrict__ part, int nblk, const double* __restrict__ bank,
                              const int* __restrict__ prow, const int* __restrict__ widx,
                              const double* __restrict__ w, double* __restrict__ gbank, double* __restrict__ gw) {
  mgb_pdl_entry();
  __shared__ double red[32];
  const int b = blockIdx.x;
  double s0 = 0.0, s1 = 0.0;
  for (int i = threadIdx.x; i < nblk; i += blockDim.x) {
    s0 += part[((size_t)b * nblk + i) * KP];
    s1 += part[((size_t)b * nblk + i) * KP + 1];
  }
  s0 = block_sum(s0, red);
  __syncthreads();
  s1 = block_sum(s1, red);
  if (threadIdx.x != 0) return;
  const double wv = w ? w[widx[b]] : 1.0;
  if (tag == 'g') {
    const double g0 = exp(bank[(size_t)prow[b] * 2]), g1 = exp(bank[(size_t)prow[b] * 2 + 1]);
    gbank[(size_t)prow[b] * 2] = wv * g0 * s0;
    gbank[(size_t)prow[b] * 2 + 1] = wv * g1 * s1;
    if (gw) gw[widx[b]] = (wv == 0.0) ? 0.0 : (g0 - 1.0) * s0 + (g1 - 1.0) * s1;
  } else {
    const double k = exp(bank[prow[b]]);
    gbank[prow[b]] = wv * 0.5 * k * s0;
    if (gw) gw[widx[b]] = (wv == 0.0) ? 0.0 : s1;
  }
}

__global__ void k_weights(const double* __restrict__ raw, const double* __restrict__ mask, double* __restrict__ w,
                          int P) {
  mgb_pdl_entry();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < P) {
    double v = expit64(raw[i]);
    if (mask) v *= mask[i];
    w[i] = v;
  }
}

// out[s] = sum of rows seg_off[s]..seg_off[s+1]-1 over 2L samples, fixed order
template <bool VEC>
__global__ void __launch_bounds__(NT) k_bus_sum(const float* const* __restrict__ in_rows,
                                                const int* __restrict__ seg_off, float* __restrict__ out, int L) {
  mgb_pdl_entry();
  const int s = blockIdx.y;
  const int i0 = seg_off[s], i1 = seg_off[s + 1];
  float* o = out + (size_t)s * 2 * L;
  const int twoL = 2 * L;
  const long long base = (long long)blockIdx.x * CHUNK;
  float acc[VPT][4];
#pragma unroll
  for (int j = 0; j < VPT; ++j)
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[j][i] = 0.f;
  for (int r = i0; r < i1; ++r) {
    const float* p = in_rows[r];
#pragma unroll
    for (int j = 0; j < VPT; ++j) {
      const long long n = base + 4LL * (threadIdx.x + j * NT);
      if (n < twoL) {
        float v[4];
        ld4<VEC>(p, n, twoL, v);
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[j][i] += v[i];
      }
    }
  }
#pragma unroll
  for (int j = 0; j < VPT; ++j) {
    const long long n = base + 4LL * (threadIdx.x + j * NT);
    if (n < twoL) st4<VEC>(o, n, twoL, acc[j]);
  }
}

}  // namespace

size_t mgb_simple_workspace(char, int B, int L) { return mgb_align(sizeof(double) * KP * B * simple_nblk(L)); }

static bool rows_vec_ok(int L) { return (L & 3) == 0; }  // row starts are then 16-byte aligned

int mgb_simple_forward(const MgbLevel* lv, cudaStream_t st) {
  const dim3 grid(simple_nblk(lv->L), lv->B);
  const bool vec = rows_vec_ok(lv->L);
#define LAUNCH(T, V) mgb_launch(k_gs_fwd<T, V>, dim3(grid), dim3(NT), 0, st, lv->u_rows, lv->bank, lv->prow, lv->widx, lv->w, lv->y, lv->L)
  if (lv->tag == 'g') { if (vec) LAUNCH('g', true); else LAUNCH('g', false); }
  else { if (vec) LAUNCH('s', true); else LAUNCH('s', false); }
#undef LAUNCH
  MGB_CHECK_LAUNCH();
  return 0;
}

int mgb_simple_backward(const MgbLevel* lv, cudaStream_t st) {
  const int nblk = simple_nblk(lv->L);
  const dim3 grid(nblk, lv->B);
  const bool vec = rows_vec_ok(lv->L);
  double* part = reinterpret_cast<double*>(lv->ws);
#define LAUNCH(T, V) mgb_launch(k_gs_bwd<T, V>, dim3(grid), dim3(NT), 0, st, lv->u_rows, lv->gy_rows, lv->bank, lv->prow, lv->widx, \
                                                          lv->w, lv->gu, part, lv->L)
  if (lv->tag == 'g') { if (vec) LAUNCH('g', true); else LAUNCH('g', false); }
  else { if (vec) LAUNCH('s', true); else LAUNCH('s', false); }
#undef LAUNCH
  MGB_CHECK_LAUNCH();
  return 0;
}

// backward phase 2: per-row reductions into gbank / gw
int mgb_simple_param_grad(const MgbLevel* lv, cudaStream_t st) {
  const int nblk = simple_nblk(lv->L);
  const double* part = reinterpret_cast<const double*>(lv->ws);
  mgb_launch(k_gs_finalize, dim3(lv->B), dim3(256), 0, st, lv->tag, part, nblk, lv->bank, lv->prow, lv->widx, lv->w, lv->gbank,
             lv->gw);
  MGB_CHECK_LAUNCH();
  return 0;
}

extern "C" int mgb_weights(const double* raw, const double* mask, double* w, int P, void* stream) {
  if (P <= 0) return 0;
  mgb_launch(k_weights, dim3((P + 255) / 256), dim3(256), 0, (cudaStream_t)stream, raw, mask, w, P);
  MGB_CHECK_LAUNCH();
  return 0;
}

extern "C" int mgb_bus_sum(const float* const* in_rows, const int* seg_off, float* out, int S, int L,
                           void* stream) {
  if (S <= 0) return 0;
  const dim3 grid(simple_nblk(2 * L), S);
  if (rows_vec_ok(L)) mgb_launch(k_bus_sum<true>, dim3(grid), dim3(NT), 0, (cudaStream_t)stream, in_rows, seg_off, out, L);
  else mgb_launch(k_bus_sum<false>, dim3(grid), dim3(NT), 0, (cudaStream_t)stream, in_rows, seg_off, out, L);
  MGB_CHECK_LAUNCH();
  return 0;
}

// ---------------------------------------------------------------------------
// Segment gather (mg/optimizer.py:97-105 sample_segment, on device): row r of the
// output is src[r][song_off[row_song[r]] : + len].  One launch copies a step's
// segments of every stem channel and target channel of every song of a batch,
// reading the per-song offsets from device memory (so a captured step replays
// with new offsets).
__global__ void __launch_bounds__(256) k_gather_rows(const float* const* __restrict__ src, float* const* __restrict__ dst,
                                                     const int* __restrict__ row_song,
                                                     const long long* __restrict__ song_off, int len) {
  mgb_pdl_entry();
  const int r = blockIdx.y;
  const float* s = src[r] + song_off[row_song[r]];
  float* d = dst[r];
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += (long long)gridDim.x * blockDim.x)
    d[i] = __ldg(s + i);
}

extern "C" int mgb_gather_rows(const float* const* src, float* const* dst, const int* row_song,
                               const long long* song_off, int rows, int len, void* stream) {
  if (rows <= 0 || len <= 0) return 0;
  if (!src || !dst || !row_song || !song_off) return 1;
  int bx = (len + 255) / 256;
  if (bx > 64) bx = 64;
  mgb_launch(k_gather_rows, dim3(bx, rows), dim3(256), 0, (cudaStream_t)stream, src, dst, row_song, song_off, len);
  MGB_CHECK_LAUNCH();
  return 0;
}
