// Compressor (c) and noise gate (n): truncated one-pole ballistics as a
// parallel scan, quadratic-knee gain computer, fused dry/wet.
//
// Reference (mg/processors.py:195-243): g = conv(mid^2, h)[0:L] with the
// 8192-tap FIR h[k] = (1-a) a^k, a = sigmoid(a_raw) taken from log space,
// clamp g >= 0, G = log(g + 1e-8), knee branches, y = u * exp(G_y - G).
//
// Here the FIR is never materialised.  With y_iir[n] = a y_iir[n-1] + x[n]
// (zero state before the signal), the truncated filter is exactly
//     g[n] = (1-a) (y_iir[n] - a^8192 y_iir[n-8192]).
// Time is cut into chunks of C = 8192 samples (= the truncation length) so
// y_iir[n-8192] sits at the same local offset of the previous chunk: a CTA
// scans chunk j-1 and chunk j together (carries from per-chunk aggregates),
// and each thread pairs its own samples -- no cross-thread exchange.
// All scan state is float64 (fp32 recursions lose 1e-4..1e-3
// at long ballistics); signals are float32 in HBM.
//
// Backward: the adjoint of the truncated causal filter is the truncated
// anti-causal filter, i.e. the same construction on reversed time:
//     v[m] = a v[m+1] + dg[m],  w[m] = a (w[m+1] + v[m+1])   (2-state scan)
//     dx[m] = (1-a)(v[m] - a^C v[m+C]),
//     r[m]  = (1-a)(w[m] - a^C (w[m+C] + C v[m+C]))   = sum_k k h[k] dg[m+k]
//     d a_raw = (1-a) sum x r - a sum x dx     (from dh[k]/da = h[k](k(1-a) - a)).
#include "common.cuh"
#include "mgb_internal.h"
#include "tables.cuh"

namespace {

constexpr int NT = 256;
constexpr int SEG = 32;
constexpr int CH = NT * SEG;  // 8192 == MGB_ENV_LEN
static_assert(CH == MGB_ENV_LEN, "chunk = truncation length");
constexpr int NW = NT / 32;

struct DynP {
  double la, lb, a, b, aC, T, W, R, Wraw, Rraw;
};

__device__ __forceinline__ DynP load_params(const double* bank, int row) {
  const double* p = bank + (size_t)row * 4;
  DynP q;
  q.la = -softplus64(-p[0]);
  q.lb = -softplus64(p[0]);
  q.a = exp(q.la);
  q.b = exp(q.lb);
  q.aC = exp((double)CH * q.la);
  q.T = p[1];
  q.Wraw = p[2];
  q.Rraw = p[3];
  q.W = softplus64(p[2]) + 1e-3;
  q.R = softplus64(p[3]) + 1.0;
  return q;
}

__device__ __forceinline__ double mid_sq(const float* u, int L, long long n) {
  if (n < 0 || n >= L) return 0.0;
  const double m = (double)u[n] + (double)u[L + n];
  return m * m;
}

// gain-computer: returns G_y for envelope G (mg/processors.py:217-232)
__device__ __forceinline__ double knee_gy(double G, const DynP& q, bool gate) {
  const bool above = G >= q.T + q.W, below = G < q.T - q.W;
  if (gate) {
    if (above) return G;
    if (below) return q.T + q.R * (G - q.T);
    const double z = G - q.T - q.W;
    return G + (1.0 - q.R) * (z * z / (q.W * 4.0));
  }
  if (above) return q.T + (G - q.T) / q.R;
  if (below) return G;
  const double z = G - q.T + q.W;
  return G + (1.0 / q.R - 1.0) * (z * z / (q.W * 4.0));
}

// forward inclusive scan of S_t = a^SEG S_{t-1} + v_t over the block's threads;
// returns the state at the end of the PREVIOUS thread's segment (exclusive),
// excluding any chunk carry.  pw[i] = a^(SEG * 2^i), i = 0..12.
__device__ __forceinline__ double block_scan_excl(double v, const double* pw, double* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double s = v;
#pragma unroll
  for (int o = 1, i = 0; o < 32; o <<= 1, ++i) {
    const double t = __shfl_up_sync(0xffffffffu, s, o);
    if (lane >= o) s = fma(pw[i], t, s);
  }
  __syncthreads();
  if (lane == 31) sh[wid] = s;
  __syncthreads();
  if (threadIdx.x == 0) {  // exclusive over warps: carry into warp w = state at end of warp w-1
    double c = 0.0;
    for (int w = 0; w < NW; ++w) {
      const double tot = sh[w];
      sh[w] = c;
      c = fma(c, pw[5], tot);  // a^(SEG*32) = a^1024
    }
  }
  __syncthreads();
  double prev = __shfl_up_sync(0xffffffffu, s, 1);
  if (lane == 0) prev = 0.0;
  // warp carry propagated to the end of thread (lane-1): a^(SEG*lane) * carry
  const double wc = sh[wid];
  double p = 1.0;  // a^(SEG*lane)
#pragma unroll
  for (int i = 0; i < 5; ++i)
    if (lane & (1 << i)) p *= pw[i];
  return fma(wc, p, prev);
}

// chunk aggregates: agg[b][j] = sum_{n in chunk j} a^{end-n} x[n]   (no (1-a) factor)
__global__ void __launch_bounds__(NT) k_dyn_agg(const float* const* __restrict__ u_rows,
                                                const double* __restrict__ bank, const int* __restrict__ prow,
                                                double* __restrict__ agg, int L, int nch) {
  __shared__ double red[32];
  const int j = blockIdx.x, b = blockIdx.y;
  const float* u = u_rows[b];
  const DynP q = load_params(bank, prow[b]);
  const long long s0 = (long long)j * CH + threadIdx.x * SEG;
  double v = 0.0;
  for (int i = 0; i < SEG; ++i) v = fma(q.a, v, mid_sq(u, L, s0 + i));
  const double f = exp((double)SEG * (NT - 1 - threadIdx.x) * q.la);
  const double tot = block_sum(v * f, red);
  if (threadIdx.x == 0) agg[(size_t)b * nch + j] = tot;
}

__global__ void __launch_bounds__(NT) k_dyn_fwd(char tag, const float* const* __restrict__ u_rows,
                                                const double* __restrict__ bank, const int* __restrict__ prow,
                                                const int* __restrict__ widx, const double* __restrict__ w,
                                                const double* __restrict__ agg, float* __restrict__ env,
                                                float* __restrict__ y, int L, int nch) {
  __shared__ double pw[14];
  __shared__ double sh[NW];
  __shared__ double carry[2];
  const int j = blockIdx.x, b = blockIdx.y;
  const float* u = u_rows[b];
  const DynP q = load_params(bank, prow[b]);
  const bool gate = tag == 'n';
  if (threadIdx.x < 14) pw[threadIdx.x] = exp((double)SEG * (double)(1 << threadIdx.x) * q.la);
  if (threadIdx.x == 0) {
    // y_iir at the end of chunk j-2 (prev carry) and j-1 (cur carry)
    const double aC = q.aC;
    double c = 0.0, cprev = 0.0;
    for (int i = 0; i < j; ++i) {
      if (i == j - 1) cprev = c;
      c = fma(c, aC, agg[(size_t)b * nch + i]);
    }
    carry[0] = cprev;
    carry[1] = c;
  }
  __syncthreads();
  const long long base_c = (long long)j * CH + threadIdx.x * SEG;
  const long long base_p = base_c - CH;
  double xp[SEG];
  double vp = 0.0, vc = 0.0;
#pragma unroll
  for (int i = 0; i < SEG; ++i) {
    xp[i] = mid_sq(u, L, base_p + i);
    vp = fma(q.a, vp, xp[i]);
  }
#pragma unroll 4
  for (int i = 0; i < SEG; ++i) vc = fma(q.a, vc, mid_sq(u, L, base_c + i));
  const double ep = block_scan_excl(vp, pw, sh);
  const double ec = block_scan_excl(vc, pw, sh);
  // chunk carry into this thread's segment start: carry * a^(SEG*t)
  const double at = exp((double)SEG * threadIdx.x * q.la);
  double yp = fma(carry[0], at, ep);
  double yc = fma(carry[1], at, ec);
  if (j == 0) yp = 0.0;
  const double wv = w ? w[widx[b]] : 1.0;
  const float wf = (float)wv, om = (float)(1.0 - wv);
  const bool bypass = wv == 0.0;
  float* yo = y + (size_t)b * 2 * L;
  float* eo = env + (size_t)b * L;
#pragma unroll
  for (int i = 0; i < SEG; ++i) {
    yp = fma(q.a, yp, xp[i]);
    xp[i] = yp;  // reuse as y_iir[n - C]
  }
#pragma unroll 2
  for (int i = 0; i < SEG; ++i) {
    const long long n = base_c + i;
    yc = fma(q.a, yc, mid_sq(u, L, n));
    if (n >= L) continue;
    const double gc = q.b * (yc - q.aC * xp[i]);
    eo[n] = (float)gc;
    const double G = log(fmax(gc, 0.0) + MGB_ENV_EPS);
    const float gain = expf((float)(knee_gy(G, q, gate) - G));
    const float l = u[n], r = u[L + n];
    if (bypass) { yo[n] = l; yo[L + n] = r; }
    else {
      yo[n] = wf * (l * gain) + om * l;
      yo[L + n] = wf * (r * gain) + om * r;
    }
  }
}

// backward part 1: elementwise chain down to dg (grad wrt the unclamped envelope)
__global__ void __launch_bounds__(NT) k_dyn_bwd0(char tag, const float* const* __restrict__ u_rows,
                                                 const float* const* __restrict__ gy_rows,
                                                 const double* __restrict__ bank, const int* __restrict__ prow,
                                                 const int* __restrict__ widx, const double* __restrict__ w,
                                                 const float* __restrict__ env, float* __restrict__ dg,
                                                 float* __restrict__ gu, double* __restrict__ part, int L) {
  __shared__ double red[32];
  const int b = blockIdx.y;
  const float* u = u_rows[b];
  const float* gy = gy_rows[b];
  const DynP q = load_params(bank, prow[b]);
  const bool gate = tag == 'n';
  const double wv = w ? w[widx[b]] : 1.0;
  const float wf = (float)wv, om = (float)(1.0 - wv);
  const bool bypass = wv == 0.0;
  const float* eo = env + (size_t)b * L;
  float* dgo = dg + (size_t)b * L;
  float* go = gu + (size_t)b * 2 * L;
  double sT = 0.0, sW = 0.0, sR = 0.0, sw = 0.0;
  for (long long n = (long long)blockIdx.x * NT + threadIdx.x; n < L; n += (long long)gridDim.x * NT) {
    const float l = u[n], r = u[L + n], gl = gy[n], gr = gy[L + n];
    const double gc = eo[n];
    const double gcl = fmax(gc, 0.0);
    const double G = log(gcl + MGB_ENV_EPS);
    const bool above = G >= q.T + q.W, below = G < q.T - q.W;
    double Gy, dGu, dT = 0.0, dW = 0.0, dR = 0.0;
    if (gate) {
      if (above) { Gy = G; dGu = 1.0; }
      else if (below) { Gy = q.T + q.R * (G - q.T); dGu = q.R; dT = 1.0 - q.R; dR = G - q.T; }
      else {
        const double z = G - q.T - q.W, k = 1.0 - q.R;
        Gy = G + k * (z * z / (q.W * 4.0));
        dGu = 1.0 + k * z / (2.0 * q.W);
        dT = -k * z / (2.0 * q.W);
        dW = k * (-z / (2.0 * q.W) - z * z / (4.0 * q.W * q.W));
        dR = -z * z / (4.0 * q.W);
      }
    } else {
      if (above) { Gy = q.T + (G - q.T) / q.R; dGu = 1.0 / q.R; dT = 1.0 - 1.0 / q.R; dR = -(G - q.T) / (q.R * q.R); }
      else if (below) { Gy = G; dGu = 1.0; }
      else {
        const double z = G - q.T + q.W, k = 1.0 / q.R - 1.0;
        Gy = G + k * (z * z / (q.W * 4.0));
        dGu = 1.0 + k * z / (2.0 * q.W);
        dT = -k * z / (2.0 * q.W);
        dW = k * (z / (2.0 * q.W) - z * z / (4.0 * q.W * q.W));
        dR = -z * z / (4.0 * q.W * q.R * q.R);
      }
    }
    const float gain = expf((float)(Gy - G));
    float dl, dr, ul, ur;
    if (bypass) { dl = dr = 0.f; ul = gl; ur = gr; }
    else {
      dl = wf * gl; dr = wf * gr; ul = om * gl; ur = om * gr;
      sw += (double)gl * (double)(l * gain - l) + (double)gr * (double)(r * gain - r);
    }
    go[n] = fmaf(dl, gain, ul);
    go[L + n] = fmaf(dr, gain, ur);
    const double D = ((double)dl * l + (double)dr * r) * (double)gain;
    sT += D * dT;
    sW += D * dW;
    sR += D * dR;
    const double dG = D * dGu - D;
    dgo[n] = (gc > 0.0) ? (float)(dG / (gcl + MGB_ENV_EPS)) : 0.f;
  }
  sT = block_sum(sT, red);
  __syncthreads();
  sW = block_sum(sW, red);
  __syncthreads();
  sR = block_sum(sR, red);
  __syncthreads();
  sw = block_sum(sw, red);
  if (threadIdx.x == 0) {
    double* pp = part + ((size_t)b * gridDim.x + blockIdx.x) * 8;
    pp[0] = sT;
    pp[1] = sW;
    pp[2] = sR;
    pp[3] = sw;
  }
}

struct VW {
  double v, w;
};

// state X entering from the right, propagated through len zero-input steps
__device__ __forceinline__ VW prop(VW x, double alen, double len) {
  VW r;
  r.v = alen * x.v;
  r.w = alen * fma(len, x.v, x.w);
  return r;
}

// reverse aggregates: state at the chunk start from the chunk's own dg only
__global__ void __launch_bounds__(NT) k_dyn_bagg(const double* __restrict__ bank, const int* __restrict__ prow,
                                                 const float* __restrict__ dg, double* __restrict__ bagg, int L,
                                                 int nch) {
  __shared__ double red[32];
  const int j = blockIdx.x, b = blockIdx.y;
  const DynP q = load_params(bank, prow[b]);
  const float* d = dg + (size_t)b * L;
  const long long s0 = (long long)j * CH + threadIdx.x * SEG;
  VW s{0.0, 0.0};
  for (int i = SEG - 1; i >= 0; --i) {
    const long long m = s0 + i;
    const double x = (m < L) ? (double)d[m] : 0.0;
    s.w = q.a * (s.w + s.v);
    s.v = fma(q.a, s.v, x);
  }
  // propagate this segment's start state to the chunk start: through SEG*t samples
  const double len = (double)SEG * threadIdx.x;
  const VW pr = prop(s, exp(len * q.la), len);
  const double tv = block_sum(pr.v, red);
  __syncthreads();
  const double tw = block_sum(pr.w, red);
  if (threadIdx.x == 0) {
    bagg[((size_t)b * nch + j) * 2] = tv;
    bagg[((size_t)b * nch + j) * 2 + 1] = tw;
  }
}

// reverse exclusive scan over the block: state at the END of this thread's
// segment (start of the next), from segments t+1.. of the chunk only.
__device__ __forceinline__ VW block_rscan_excl(VW s, const double* pw, double* shv, double* shw) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  VW r = s;  // inclusive: segments [t, t+o) covered
#pragma unroll
  for (int o = 1, i = 0; o < 32; o <<= 1, ++i) {
    const double tv = __shfl_down_sync(0xffffffffu, r.v, o);
    const double tw = __shfl_down_sync(0xffffffffu, r.w, o);
    if (lane + o < 32) {
      const VW p = prop(VW{tv, tw}, pw[i], (double)SEG * o);
      r.v += p.v;
      r.w += p.w;
    }
  }
  __syncthreads();
  if (lane == 0) { shv[wid] = r.v; shw[wid] = r.w; }
  __syncthreads();
  if (threadIdx.x == 0) {  // state at the end of warp w from warps w+1..
    VW c{0.0, 0.0};
    for (int w = NW - 1; w >= 0; --w) {
      const VW tot{shv[w], shw[w]};
      shv[w] = c.v;
      shw[w] = c.w;
      const VW p = prop(c, pw[5], (double)SEG * 32);
      c.v = tot.v + p.v;
      c.w = tot.w + p.w;
    }
  }
  __syncthreads();
  double nv = __shfl_down_sync(0xffffffffu, r.v, 1);
  double nw = __shfl_down_sync(0xffffffffu, r.w, 1);
  if (lane == 31) { nv = 0.0; nw = 0.0; }
  // warp carry enters after lane 31: propagate through segments lane+1..31
  const int k = 31 - lane;
  double p = 1.0;
#pragma unroll
  for (int i = 0; i < 5; ++i)
    if (k & (1 << i)) p *= pw[i];
  const VW wc = prop(VW{shv[wid], shw[wid]}, p, (double)SEG * k);
  return VW{nv + wc.v, nw + wc.w};
}

__global__ void __launch_bounds__(NT) k_dyn_bwd1(const float* const* __restrict__ u_rows,
                                                 const double* __restrict__ bank, const int* __restrict__ prow,
                                                 const double* __restrict__ bagg, const float* __restrict__ dg,
                                                 float* __restrict__ gu, double* __restrict__ part, int L,
                                                 int nch) {
  __shared__ double pw[14];
  __shared__ double shv[NW], shw[NW];
  __shared__ double carry[4];
  __shared__ double red[32];
  const int j = blockIdx.x, b = blockIdx.y;
  const float* u = u_rows[b];
  const DynP q = load_params(bank, prow[b]);
  const float* d = dg + (size_t)b * L;
  if (threadIdx.x < 14) pw[threadIdx.x] = exp((double)SEG * (double)(1 << threadIdx.x) * q.la);
  if (threadIdx.x == 0) {
    // state at the start of chunk j+1 (cur carry) and j+2 (next carry)
    VW c{0.0, 0.0}, cnext{0.0, 0.0};
    for (int i = nch - 1; i > j; --i) {
      if (i == j + 1) cnext = c;
      const VW p = prop(c, q.aC, (double)CH);
      c.v = bagg[((size_t)b * nch + i) * 2] + p.v;
      c.w = bagg[((size_t)b * nch + i) * 2 + 1] + p.w;
    }
    carry[0] = c.v;
    carry[1] = c.w;
    carry[2] = cnext.v;
    carry[3] = cnext.w;
  }
  __syncthreads();
  const long long base_c = (long long)j * CH + threadIdx.x * SEG;
  const long long base_n = base_c + CH;
  // local segment aggregates (zero state after segment end)
  VW sc{0.0, 0.0}, sn{0.0, 0.0};
  for (int i = SEG - 1; i >= 0; --i) {
    const long long m = base_c + i, mn = base_n + i;
    const double xc = (m < L) ? (double)d[m] : 0.0;
    const double xn = (mn < L) ? (double)d[mn] : 0.0;
    sc.w = q.a * (sc.w + sc.v);
    sc.v = fma(q.a, sc.v, xc);
    sn.w = q.a * (sn.w + sn.v);
    sn.v = fma(q.a, sn.v, xn);
  }
  const VW ec = block_rscan_excl(sc, pw, shv, shw);
  const VW en = block_rscan_excl(sn, pw, shv, shw);
  // chunk carry enters after the last segment: propagate through segments t+1..NT-1
  const double len = (double)SEG * (NT - 1 - threadIdx.x);
  const double alen = exp(len * q.la);
  const VW cc = prop(VW{carry[0], carry[1]}, alen, len);
  const VW cn = prop(VW{carry[2], carry[3]}, alen, len);
  VW stc{ec.v + cc.v, ec.w + cc.w};
  VW stn{en.v + cn.v, en.w + cn.w};
  double nv[SEG], nw[SEG];
#pragma unroll
  for (int i = SEG - 1; i >= 0; --i) {
    const long long mn = base_n + i;
    const double xn = (mn < L) ? (double)d[mn] : 0.0;
    stn.w = q.a * (stn.w + stn.v);
    stn.v = fma(q.a, stn.v, xn);
    nv[i] = stn.v;
    nw[i] = stn.w;
  }
  double sxd = 0.0, sxr = 0.0;
  float* go = gu + (size_t)b * 2 * L;
#pragma unroll
  for (int i = SEG - 1; i >= 0; --i) {
    const long long m = base_c + i;
    const double xc = (m < L) ? (double)d[m] : 0.0;
    stc.w = q.a * (stc.w + stc.v);
    stc.v = fma(q.a, stc.v, xc);
    if (m >= L) continue;
    const double dx = q.b * (stc.v - q.aC * nv[i]);
    const double rr = q.b * (stc.w - q.aC * fma((double)CH, nv[i], nw[i]));
    const double mid = (double)u[m] + (double)u[L + m];
    const double x = mid * mid;
    sxd = fma(x, dx, sxd);
    sxr = fma(x, rr, sxr);
    const float dm = (float)(2.0 * mid * dx);
    go[m] += dm;
    go[L + m] += dm;
  }
  sxd = block_sum(sxd, red);
  __syncthreads();
  sxr = block_sum(sxr, red);
  if (threadIdx.x == 0) {
    double* pp = part + ((size_t)b * nch + j) * 8;
    pp[4] = sxd;
    pp[5] = sxr;
  }
}

__global__ void k_dyn_final(const double* __restrict__ part, int nblk0, int nch, const double* __restrict__ bank,
                            const int* __restrict__ prow, const int* __restrict__ widx, const double* __restrict__ w,
                            double* __restrict__ gbank, double* __restrict__ gw, const double* __restrict__ part1) {
  const int b = blockIdx.x;
  if (threadIdx.x) return;
  const DynP q = load_params(bank, prow[b]);
  double sT = 0, sW = 0, sR = 0, sw = 0, sxd = 0, sxr = 0;
  for (int i = 0; i < nblk0; ++i) {
    const double* pp = part + ((size_t)b * nblk0 + i) * 8;
    sT += pp[0];
    sW += pp[1];
    sR += pp[2];
    sw += pp[3];
  }
  for (int i = 0; i < nch; ++i) {
    const double* pp = part1 + ((size_t)b * nch + i) * 8;
    sxd += pp[4];
    sxr += pp[5];
  }
  double* g = gbank + (size_t)prow[b] * 4;
  g[0] = (1.0 - q.a) * sxr - q.a * sxd;
  g[1] = sT;
  g[2] = sW * expit64(q.Wraw);
  g[3] = sR * expit64(q.Rraw);
  const double wv = w ? w[widx[b]] : 1.0;
  if (gw) gw[widx[b]] = (wv == 0.0) ? 0.0 : sw;
}

int nchunks(int L) { return (L + CH - 1) / CH; }
int bwd0_grid(int L) {
  int n = (L + 4 * NT - 1) / (4 * NT);
  return n < 1 ? 1 : (n > 256 ? 256 : n);
}

struct DynWs {
  double *agg, *bagg, *part0, *part1;
  float* dg;
};

DynWs dcarve(int B, int L, void* base) {
  MgbArena a{(char*)base, 0};
  DynWs w;
  const int nch = nchunks(L);
  w.agg = a.take<double>((size_t)B * nch);
  w.bagg = a.take<double>((size_t)B * nch * 2);
  w.part0 = a.take<double>((size_t)B * bwd0_grid(L) * 8);
  w.part1 = a.take<double>((size_t)B * nch * 8);
  w.dg = a.take<float>((size_t)B * L);
  return w;
}

}  // namespace

size_t mgb_dyn_workspace(char, int B, int L) {
  MgbArena a{nullptr, 0};
  const int nch = nchunks(L);
  a.take<double>((size_t)B * nch);
  a.take<double>((size_t)B * nch * 2);
  a.take<double>((size_t)B * bwd0_grid(L) * 8);
  a.take<double>((size_t)B * nch * 8);
  a.take<float>((size_t)B * L);
  return a.off;
}

int mgb_dyn_forward(const MgbLevel* lv, cudaStream_t st) {
  if (!lv->aux) return 1;
  const int B = lv->B, L = lv->L, nch = nchunks(L);
  DynWs w = dcarve(B, L, lv->ws);
  k_dyn_agg<<<dim3(nch, B), NT, 0, st>>>(lv->u_rows, lv->bank, lv->prow, w.agg, L, nch);
  MGB_CHECK_LAUNCH();
  k_dyn_fwd<<<dim3(nch, B), NT, 0, st>>>(lv->tag, lv->u_rows, lv->bank, lv->prow, lv->widx, lv->w, w.agg,
                                         lv->aux, lv->y, L, nch);
  MGB_CHECK_LAUNCH();
  return 0;
}

int mgb_dyn_backward(const MgbLevel* lv, cudaStream_t st) {
  if (!lv->aux) return 1;
  const int B = lv->B, L = lv->L, nch = nchunks(L), g0 = bwd0_grid(L);
  DynWs w = dcarve(B, L, lv->ws);
  k_dyn_bwd0<<<dim3(g0, B), NT, 0, st>>>(lv->tag, lv->u_rows, lv->gy_rows, lv->bank, lv->prow, lv->widx, lv->w,
                                         lv->aux, w.dg, lv->gu, w.part0, L);
  MGB_CHECK_LAUNCH();
  k_dyn_bagg<<<dim3(nch, B), NT, 0, st>>>(lv->bank, lv->prow, w.dg, w.bagg, L, nch);
  MGB_CHECK_LAUNCH();
  k_dyn_bwd1<<<dim3(nch, B), NT, 0, st>>>(lv->u_rows, lv->bank, lv->prow, w.bagg, w.dg, lv->gu, w.part1, L, nch);
  MGB_CHECK_LAUNCH();
  k_dyn_final<<<B, 32, 0, st>>>(w.part0, g0, nch, lv->bank, lv->prow, lv->widx, lv->w, lv->gbank, lv->gw, w.part1);
  MGB_CHECK_LAUNCH();
  return 0;
}
