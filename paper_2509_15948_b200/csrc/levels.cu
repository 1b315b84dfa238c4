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
constexpr int KP = 4;  // partial slots per CTA

__host__ __device__ inline int simple_nblk(int L) {
  int n = (L + 4 * NT - 1) / (4 * NT);
  return n < 1 ? 1 : (n > 64 ? 64 : n);
}

__global__ void __launch_bounds__(NT) k_gs_fwd(char tag, const float* const* __restrict__ u_rows,
                                               const double* __restrict__ bank, const int* __restrict__ prow,
                                               const int* __restrict__ widx, const double* __restrict__ w,
                                               float* __restrict__ y, int L) {
  const int b = blockIdx.y;
  const float* u = u_rows[b];
  float* yo = y + (size_t)b * 2 * L;
  const double wv = w ? w[widx[b]] : 1.0;
  const long long stride = (long long)gridDim.x * NT;
  if (wv == 0.0) {  // exact bypass
    for (long long n = (long long)blockIdx.x * NT + threadIdx.x; n < L; n += stride) {
      yo[n] = u[n];
      yo[L + n] = u[L + n];
    }
    return;
  }
  if (tag == 'g') {
    const int P = 2;
    const double g0 = exp(bank[(size_t)prow[b] * P]), g1 = exp(bank[(size_t)prow[b] * P + 1]);
    const float c0 = (float)(wv * g0 + (1.0 - wv)), c1 = (float)(wv * g1 + (1.0 - wv));
    for (long long n = (long long)blockIdx.x * NT + threadIdx.x; n < L; n += stride) {
      yo[n] = c0 * u[n];
      yo[L + n] = c1 * u[L + n];
    }
  } else {
    const float k = (float)exp(bank[prow[b]]);
    const float wf = (float)wv, om = (float)(1.0 - wv);
    for (long long n = (long long)blockIdx.x * NT + threadIdx.x; n < L; n += stride) {
      const float l = u[n], r = u[L + n];
      const float mid = l + r, side = k * (l - r);
      const float yl = (mid + side) * 0.5f, yr = (mid - side) * 0.5f;
      yo[n] = wf * yl + om * l;
      yo[L + n] = wf * yr + om * r;
    }
  }
}

__global__ void __launch_bounds__(NT) k_gs_bwd(char tag, const float* const* __restrict__ u_rows,
                                               const float* const* __restrict__ gy_rows,
                                               const double* __restrict__ bank, const int* __restrict__ prow,
                                               const int* __restrict__ widx, const double* __restrict__ w,
                                               float* __restrict__ gu, double* __restrict__ part, int L) {
  __shared__ double scratch[32];
  const int b = blockIdx.y;
  const float* u = u_rows[b];
  const float* gy = gy_rows[b];
  float* go = gu + (size_t)b * 2 * L;
  const double wv = w ? w[widx[b]] : 1.0;
  const long long stride = (long long)gridDim.x * NT;
  double a0 = 0.0, a1 = 0.0;
  if (wv == 0.0) {
    for (long long n = (long long)blockIdx.x * NT + threadIdx.x; n < L; n += stride) {
      go[n] = gy[n];
      go[L + n] = gy[L + n];
    }
  } else if (tag == 'g') {
    const double g0 = exp(bank[(size_t)prow[b] * 2]), g1 = exp(bank[(size_t)prow[b] * 2 + 1]);
    const float c0 = (float)(wv * g0 + (1.0 - wv)), c1 = (float)(wv * g1 + (1.0 - wv));
    float s0 = 0.f, s1 = 0.f;
    int cnt = 0;
    for (long long n = (long long)blockIdx.x * NT + threadIdx.x; n < L; n += stride) {
      const float gl = gy[n], gr = gy[L + n];
      go[n] = c0 * gl;
      go[L + n] = c1 * gr;
      s0 = fmaf(gl, u[n], s0);
      s1 = fmaf(gr, u[L + n], s1);
      if (++cnt == 16) { a0 += s0; a1 += s1; s0 = s1 = 0.f; cnt = 0; }
    }
    a0 += s0;
    a1 += s1;
  } else {
    const float k = (float)exp(bank[prow[b]]);
    const float wf = (float)wv, om = (float)(1.0 - wv);
    float s0 = 0.f, s1 = 0.f;
    int cnt = 0;
    for (long long n = (long long)blockIdx.x * NT + threadIdx.x; n < L; n += stride) {
      const float l = u[n], r = u[L + n], gl = gy[n], gr = gy[L + n];
      const float dl = wf * gl, dr = wf * gr;           // d ybar
      const float sm = 0.5f * (dl + dr), sd = 0.5f * k * (dl - dr);
      go[n] = om * gl + sm + sd;
      go[L + n] = om * gr + sm - sd;
      const float mid = l + r, side = k * (l - r);
      const float yl = (mid + side) * 0.5f, yr = (mid - side) * 0.5f;
      s0 = fmaf(l - r, gl - gr, s0);                   // for d p
      s1 = fmaf(gl, yl - l, fmaf(gr, yr - r, s1));     // for d w
      if (++cnt == 16) { a0 += s0; a1 += s1; s0 = s1 = 0.f; cnt = 0; }
    }
    a0 += s0;
    a1 += s1;
  }
  const double t0 = block_sum(a0, scratch);
  const double t1 = block_sum(a1, scratch);
  if (threadIdx.x == 0) {
    double* pp = part + ((size_t)b * gridDim.x + blockIdx.x) * KP;
    pp[0] = t0;
    pp[1] = t1;
  }
}

__global__ void k_gs_finalize(char tag, const double* __restrict__ part, int nblk, const double* __restrict__ bank,
                              const int* __restrict__ prow, const int* __restrict__ widx,
                              const double* __restrict__ w, double* __restrict__ gbank, double* __restrict__ gw) {
  const int b = blockIdx.x;
  if (threadIdx.x != 0) return;
  double s0 = 0.0, s1 = 0.0;
  for (int i = 0; i < nblk; ++i) {
    s0 += part[((size_t)b * nblk + i) * KP];
    s1 += part[((size_t)b * nblk + i) * KP + 1];
  }
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
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < P) {
    double v = expit64(raw[i]);
    if (mask) v *= mask[i];
    w[i] = v;
  }
}

__global__ void __launch_bounds__(NT) k_bus_sum(const float* const* __restrict__ in_rows,
                                                const int* __restrict__ seg_off, float* __restrict__ out, int L) {
  const int s = blockIdx.y;
  const int i0 = seg_off[s], i1 = seg_off[s + 1];
  float* o = out + (size_t)s * 2 * L;
  const long long twoL = 2LL * L;
  for (long long n = (long long)blockIdx.x * NT + threadIdx.x; n < twoL; n += (long long)gridDim.x * NT) {
    float acc = 0.f;
    for (int i = i0; i < i1; ++i) acc += in_rows[i][n];
    o[n] = acc;
  }
}

}  // namespace

size_t mgb_simple_workspace(char, int B, int L) { return mgb_align(sizeof(double) * KP * B * simple_nblk(L)); }

int mgb_simple_forward(const MgbLevel* lv, cudaStream_t st) {
  const int nblk = simple_nblk(lv->L);
  k_gs_fwd<<<dim3(nblk, lv->B), NT, 0, st>>>(lv->tag, lv->u_rows, lv->bank, lv->prow, lv->widx, lv->w, lv->y,
                                             lv->L);
  MGB_CHECK_LAUNCH();
  return 0;
}

int mgb_simple_backward(const MgbLevel* lv, cudaStream_t st) {
  const int nblk = simple_nblk(lv->L);
  double* part = reinterpret_cast<double*>(lv->ws);
  k_gs_bwd<<<dim3(nblk, lv->B), NT, 0, st>>>(lv->tag, lv->u_rows, lv->gy_rows, lv->bank, lv->prow, lv->widx,
                                             lv->w, lv->gu, part, lv->L);
  MGB_CHECK_LAUNCH();
  k_gs_finalize<<<lv->B, 32, 0, st>>>(lv->tag, part, nblk, lv->bank, lv->prow, lv->widx, lv->w, lv->gbank,
                                      lv->gw);
  MGB_CHECK_LAUNCH();
  return 0;
}

extern "C" int mgb_weights(const double* raw, const double* mask, double* w, int P, void* stream) {
  if (P <= 0) return 0;
  k_weights<<<(P + 255) / 256, 256, 0, (cudaStream_t)stream>>>(raw, mask, w, P);
  MGB_CHECK_LAUNCH();
  return 0;
}

extern "C" int mgb_bus_sum(const float* const* in_rows, const int* seg_off, float* out, int S, int L,
                           void* stream) {
  if (S <= 0) return 0;
  const int nblk = simple_nblk(2 * L);
  k_bus_sum<<<dim3(nblk, S), NT, 0, (cudaStream_t)stream>>>(in_rows, seg_off, out, L);
  MGB_CHECK_LAUNCH();
  return 0;
}
