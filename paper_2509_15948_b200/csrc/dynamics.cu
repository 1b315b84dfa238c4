// Compressor (c) and noise gate (n): truncated one-pole ballistics as a
// parallel scan, quadratic-knee gain computer, fused dry/wet.
//
// Reference (mg/processors.py:195-243): g = conv(mid^2, h)[0:L] with the
// 8192-tap FIR h[k] = (1-a) a^k, a = sigmoid(a_raw) taken from log space,
// clamp g >= 0, G = log(g + 1e-8), knee branches, y = u * exp(G_y - G).
//
// The FIR is never materialised.  With y_iir[n] = a y_iir[n-1] + x[n] (zero
// state before the signal) the truncated filter is exactly
//     g[n] = (1-a) (y_iir[n] - a^8192 y_iir[n-8192]).
// Time is cut into chunks of C = 8192 samples (= the truncation length), so
// y_iir[n-8192] sits at the same local offset of the previous chunk: a CTA
// scans chunk j-1 and chunk j together (chunk carries from per-chunk
// aggregates) and every thread pairs its own samples.  Scan state is float64
// (fp32 recursions lose 1e-4..1e-3 at long ballistics);
// inputs x = mid^2, the envelope and the gain computer are float32.
//
// Forward in one scan pass: by linearity the truncated filter is the plain
// recursion driven by the differenced input x'[n] = x[n] - a^8192 x[n-8192]
// (S[n] = sum_{k<8192} a^k x[n-k] = IIR(x')[n]), so a CTA scans only its own
// chunk; x' is formed in float64 from the float32 mid^2 of this chunk and of
// the previous one (same local offset).  The gain computer runs in float32
// with MUFU exp/log (abs. error ~1e-6 in the log domain, far inside 1e-4).
//
// Backward (one kernel per level + a per-node finalize): the adjoint of the truncated causal filter is the truncated
// anti-causal filter — the same construction on reversed time with the
// 2-state recursion  v[m] = a v[m+1] + dg[m],  w[m] = a (w[m+1] + v[m+1]):
//     dx[m] = (1-a)(v[m] - a^C v[m+C])
//     r[m]  = (1-a)(w[m] - a^C (w[m+C] + C v[m+C])) = sum_k k h[k] dg[m+k]
//     d a_raw = (1-a) sum x r - a sum x dx   (dh[k]/da = h[k](k(1-a) - a)).
#include "common.cuh"
#include "mgb_internal.h"
#include "tables.cuh"

namespace {

constexpr int NT = 512;
constexpr int SEG = 16;
constexpr int CH = NT * SEG;  // 8192 == MGB_ENV_LEN
static_assert(CH == MGB_ENV_LEN, "chunk = truncation length");
constexpr int NW = NT / 32;
constexpr int NPW = 14;  // pw[i] = a^(SEG * 2^i)

struct DynP {
  double la, a, b, aC;
  float T, W, R;
  float iR, i2W, i4W;  // 1/R, 1/(2W), 1/(4W)
  double Wraw, Rraw;
};

__device__ __forceinline__ DynP load_params(const double* bank, int row) {
  const double* p = bank + (size_t)row * 4;
  DynP q;
  q.la = -softplus64(-p[0]);
  q.a = exp(q.la);
  q.b = exp(-softplus64(p[0]));
  q.aC = exp((double)CH * q.la);
  q.T = (float)p[1];
  q.Wraw = p[2];
  q.Rraw = p[3];
  q.W = (float)(softplus64(p[2]) + 1e-3);
  q.R = (float)(softplus64(p[3]) + 1.0);
  q.iR = 1.f / q.R;
  q.i2W = 1.f / (2.f * q.W);
  q.i4W = 1.f / (4.f * q.W);
  return q;
}

// per-node parameter block, computed once per forward by k_dyn_pre (forward
// phase 1, params only) so the signal kernels' CTAs do not each redo the
// float64 softplus/exp chains before issuing their loads
struct DynPre {
  DynP q;
  double pw[NPW];  // a^(SEG * 2^i)
};

__global__ void k_dyn_pre(const double* __restrict__ bank, const int* __restrict__ prow, DynPre* __restrict__ pre) {
  mgb_pdl_entry();
  const int b = blockIdx.x;
  const DynP q = load_params(bank, prow[b]);
  if (threadIdx.x == 0) pre[b].q = q;
  if (threadIdx.x < NPW) pre[b].pw[threadIdx.x] = exp((double)SEG * (double)(1 << threadIdx.x) * q.la);
}

__device__ __forceinline__ float mid_sq(const float* u, int L, long long n) {
  if (n < 0 || n >= L) return 0.f;
  const float m = __ldg(u + n) + __ldg(u + L + n);
  return m * m;
}

// a^(SEG * k) for 0 <= k < 2^NPW from the power table
__device__ __forceinline__ double powseg(const double* pw, int k) {
  double p = 1.0;
#pragma unroll
  for (int i = 0; i < 10; ++i)
    if (k & (1 << i)) p *= pw[i];
  return p;
}

// gain-computer G_y (mg/processors.py:217-232), float32
template <bool GATE>
__device__ __forceinline__ float knee_gy(float G, const DynP& q) {
  const bool above = G >= q.T + q.W, below = G < q.T - q.W;
  const float d = G - q.T;
  if (GATE) {
    const float z = d - q.W;
    const float knee = G + (1.f - q.R) * (z * z * q.i4W);
    return above ? G : (below ? fmaf(q.R, d, q.T) : knee);
  }
  const float z = d + q.W;
  const float knee = G + (q.iR - 1.f) * (z * z * q.i4W);
  return below ? G : (above ? fmaf(d, q.iR, q.T) : knee);
}

__device__ __forceinline__ float env_log(float gc) { return __logf(fmaxf(gc, 0.f) + 1e-8f); }

// Two forward exclusive scans at once: S_t = a^SEG S_{t-1} + v_t over the
// block's threads; returns the state at the end of thread t-1's segment.
__device__ __forceinline__ void scan2_excl(double& v0, double& v1, const double* pw, double* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double s0 = v0, s1 = v1;
#pragma unroll
  for (int o = 1, i = 0; o < 32; o <<= 1, ++i) {
    const double t0 = __shfl_up_sync(0xffffffffu, s0, o);
    const double t1 = __shfl_up_sync(0xffffffffu, s1, o);
    if (lane >= o) {
      s0 = fma(pw[i], t0, s0);
      s1 = fma(pw[i], t1, s1);
    }
  }
  if (lane == 31) { sh[wid] = s0; sh[NW + wid] = s1; }
  __syncthreads();
  if (threadIdx.x < 2) {  // exclusive over warps (carry into warp w)
    double c = 0.0;
    double* x = sh + threadIdx.x * NW;
    for (int w = 0; w < NW; ++w) {
      const double tot = x[w];
      x[w] = c;
      c = fma(c, pw[5], tot);  // a^(SEG*32)
    }
  }
  __syncthreads();
  double p0 = __shfl_up_sync(0xffffffffu, s0, 1), p1 = __shfl_up_sync(0xffffffffu, s1, 1);
  if (lane == 0) { p0 = 0.0; p1 = 0.0; }
  const double pl = powseg(pw, lane);
  v0 = fma(sh[wid], pl, p0);
  v1 = fma(sh[NW + wid], pl, p1);
}

// one forward exclusive scan S_t = a^SEG S_{t-1} + v_t over the block's threads
__device__ __forceinline__ void scan1_excl(double& v0, const double* pw, double* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double s0 = v0;
#pragma unroll
  for (int o = 1, i = 0; o < 32; o <<= 1, ++i) {
    const double t0 = __shfl_up_sync(0xffffffffu, s0, o);
    if (lane >= o) s0 = fma(pw[i], t0, s0);
  }
  if (lane == 31) sh[wid] = s0;
  __syncthreads();
  if (threadIdx.x == 0) {  // exclusive over warps (carry into warp w)
    double c = 0.0;
    for (int w = 0; w < NW; ++w) {
      const double tot = sh[w];
      sh[w] = c;
      c = fma(c, pw[5], tot);  // a^(SEG*32)
    }
  }
  __syncthreads();
  double p0 = __shfl_up_sync(0xffffffffu, s0, 1);
  if (lane == 0) p0 = 0.0;
  v0 = fma(sh[wid], powseg(pw, lane), p0);
}

__device__ __forceinline__ void init_pw(double* pw, const DynPre& p) {
  if (threadIdx.x < NPW) pw[threadIdx.x] = p.pw[threadIdx.x];
}

// padded segment-major staging index: thread t's sample i of a chunk
__device__ __forceinline__ int sidx(int t, int i) { return t * (SEG + 1) + i; }
__device__ __forceinline__ int sidx_n(int o) { return sidx(o / SEG, o % SEG); }
constexpr int SPAD = NT * (SEG + 1);
constexpr int kDynSmem = 2 * SPAD * 4;                 // bwd1: two float chunks
constexpr int kDynSmemF = SPAD * 8 + SPAD * 4;         // fwd: x' (double) + previous mid^2
constexpr int Q4 = CH / (4 * NT);  // float4 groups per thread per chunk

// 16-byte vector access is used when both channel rows are 16-byte aligned
__device__ __forceinline__ bool vec_ok(const void* p, int L) {
  return (L & 3) == 0 && (reinterpret_cast<uintptr_t>(p) & 15) == 0;
}

// samples n..n+3 of both channels of a (2, L) row, zeros outside [0, L)
__device__ __forceinline__ void load4(const float* u, int L, long long n, bool vec, float4& l, float4& r) {
  if (vec) {
    if (n >= 0 && n < L) {
      l = __ldg(reinterpret_cast<const float4*>(u + n));
      r = __ldg(reinterpret_cast<const float4*>(u + L + n));
    } else {
      l = r = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    return;
  }
  float a[4], c[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const bool in = n + e >= 0 && n + e < L;
    a[e] = in ? u[n + e] : 0.f;
    c[e] = in ? u[L + n + e] : 0.f;
  }
  l = make_float4(a[0], a[1], a[2], a[3]);
  r = make_float4(c[0], c[1], c[2], c[3]);
}

__device__ __forceinline__ float msq(float l, float r) {
  const float m = l + r;
  return m * m;
}

__device__ __forceinline__ void stage_msq(float* dst, float4 l, float4 r) {
  dst[0] = msq(l.x, r.x);
  dst[1] = msq(l.y, r.y);
  dst[2] = msq(l.z, r.z);
  dst[3] = msq(l.w, r.w);
}

// y rows (2 channels) and one mono row at samples n..n+3 (bounds-checked when !vec)
__device__ __forceinline__ void store4(float* yo, int L, long long n, bool vec, float4 yl, float4 yr, float* mono,
                                       float4 m) {
  if (vec) {
    if (n < L) {
      *reinterpret_cast<float4*>(yo + n) = yl;
      *reinterpret_cast<float4*>(yo + L + n) = yr;
      if (mono) *reinterpret_cast<float4*>(mono + n) = m;
    }
    return;
  }
  const float a[4] = {yl.x, yl.y, yl.z, yl.w}, c[4] = {yr.x, yr.y, yr.z, yr.w}, d[4] = {m.x, m.y, m.z, m.w};
#pragma unroll
  for (int e = 0; e < 4; ++e)
    if (n + e < L) {
      yo[n + e] = a[e];
      yo[L + n + e] = c[e];
      if (mono) mono[n + e] = d[e];
    }
}

// samples n..n+3 of a mono row, zeros outside [0, L)
__device__ __forceinline__ float4 load4m(const float* d, int L, long long n, bool vec) {
  if (vec) return (n >= 0 && n < L) ? __ldg(reinterpret_cast<const float4*>(d + n)) : make_float4(0.f, 0.f, 0.f, 0.f);
  float a[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) a[e] = (n + e >= 0 && n + e < L) ? d[n + e] : 0.f;
  return make_float4(a[0], a[1], a[2], a[3]);
}

template <bool GATE>
__global__ void __launch_bounds__(NT, 2) k_dyn_fwd(const float* const* __restrict__ u_rows,
                                                const DynPre* __restrict__ pre,
                                                const int* __restrict__ widx, const double* __restrict__ w,
                                                float* __restrict__ env, float* __restrict__ y, int L) {
  mgb_pdl_entry();
  extern __shared__ __align__(16) unsigned char dsm[];
  double* xd = reinterpret_cast<double*>(dsm);        // [SPAD] x' of this chunk (segment-major)
  float* xps = reinterpret_cast<float*>(xd + SPAD);   // [SPAD] mid^2 of the previous chunk
  __shared__ double pw[NPW];
  __shared__ double sh[2 * NW];
  __shared__ double carry;
  __shared__ double red[32];
  const int j = blockIdx.x, b = blockIdx.y;
  const float* u = u_rows[b];
  const DynP q = pre[b].q;
  init_pw(pw, pre[b]);
  const long long c0 = (long long)j * CH;
  const bool vec = vec_ok(u, L);
  {  // coalesced staging of x' = mid^2 - a^C mid_prev^2 (float64), two float4 groups at a time
#pragma unroll
    for (int k0 = 0; k0 < Q4; k0 += 2) {
      float4 pl[2], pr[2], cl[2], cr[2];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int o = 4 * (threadIdx.x + NT * (k0 + k));
        load4(u, L, c0 - CH + o, vec, pl[k], pr[k]);
        load4(u, L, c0 + o, vec, cl[k], cr[k]);
      }
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int o = 4 * (threadIdx.x + NT * (k0 + k));
        stage_msq(xps + sidx_n(o), pl[k], pr[k]);
        double* d = xd + sidx_n(o);
        d[0] = fma(-q.aC, (double)msq(pl[k].x, pr[k].x), (double)msq(cl[k].x, cr[k].x));
        d[1] = fma(-q.aC, (double)msq(pl[k].y, pr[k].y), (double)msq(cl[k].y, cr[k].y));
        d[2] = fma(-q.aC, (double)msq(pl[k].z, pr[k].z), (double)msq(cl[k].z, cr[k].z));
        d[3] = fma(-q.aC, (double)msq(pl[k].w, pr[k].w), (double)msq(cl[k].w, cr[k].w));
      }
    }
  }
  __syncthreads();
  // local aggregates: x' over this thread's segment, and mid^2 of the previous chunk's
  // segment (their weighted block sum is the state entering the chunk: the windowed
  // sum S at the end of chunk j-1 spans exactly that chunk, as C = 8192 = chunk)
  double v = 0.0, vp = 0.0;
#pragma unroll
  for (int i = 0; i < SEG; ++i) {
    v = fma(q.a, v, xd[sidx(threadIdx.x, i)]);
    vp = fma(q.a, vp, (double)xps[sidx(threadIdx.x, i)]);
  }
  const double tot = block_sum(vp * powseg(pw, NT - 1 - threadIdx.x), red);
  if (threadIdx.x == 0) carry = tot;
  scan1_excl(v, pw, sh);  // (its barriers publish `carry`)
  double yc = fma(carry, powseg(pw, threadIdx.x), v);
  // second pass: each thread overwrites its own x' slots with (envelope, gain) pairs
  float2* eg = reinterpret_cast<float2*>(dsm);
#pragma unroll
  for (int i = 0; i < SEG; ++i) {
    yc = fma(q.a, yc, xd[sidx(threadIdx.x, i)]);
    const float gc = (float)(q.b * yc);
    const float G = env_log(gc);
    eg[sidx(threadIdx.x, i)] = make_float2(gc, __expf(knee_gy<GATE>(G, q) - G));
  }
  __syncthreads();
  const double wv = w ? w[widx[b]] : 1.0;
  const float wf = (float)wv, om = (float)(1.0 - wv);
  const bool bypass = wv == 0.0;
  float* yo = y + (size_t)b * 2 * L;
  float* eo = env + (size_t)b * L;
  float4 ul[Q4], ur[Q4];
#pragma unroll
  for (int k = 0; k < Q4; ++k) load4(u, L, c0 + 4 * (threadIdx.x + NT * k), vec, ul[k], ur[k]);
#pragma unroll
  for (int k = 0; k < Q4; ++k) {  // coalesced outputs
    const int o = 4 * (threadIdx.x + NT * k);
    const long long n = c0 + o;
    const float2* p = eg + sidx_n(o);
    const float2 e0 = p[0], e1 = p[1], e2 = p[2], e3 = p[3];
    float4 yl, yr;
    const float4 g4 = make_float4(e0.y, e1.y, e2.y, e3.y);
    if (bypass) {
      yl = ul[k];
      yr = ur[k];
    } else {
      yl = make_float4(wf * (ul[k].x * g4.x) + om * ul[k].x, wf * (ul[k].y * g4.y) + om * ul[k].y,
                       wf * (ul[k].z * g4.z) + om * ul[k].z, wf * (ul[k].w * g4.w) + om * ul[k].w);
      yr = make_float4(wf * (ur[k].x * g4.x) + om * ur[k].x, wf * (ur[k].y * g4.y) + om * ur[k].y,
                       wf * (ur[k].z * g4.z) + om * ur[k].z, wf * (ur[k].w * g4.w) + om * ur[k].w);
    }
    store4(yo, L, n, vec, yl, yr, eo, make_float4(e0.x, e1.x, e2.x, e3.x));
  }
}

// Per-sample adjoint of the gain computer and dry/wet (mg/processors.py:195-243):
// given u (l, r), dL/dy (gl, gr) and the stored envelope gc, returns dL/du's
// elementwise part (ol, orr), dL/d(envelope) og, and accumulates the T/W/R/w
// partials.  The knee masks are constants of the backward (mg/engine.py:328-341).
struct DynAcc {
  float T, W, R, w;
};
// Branch-free: the three knee regions are evaluated arithmetically and selected.
template <bool GATE, bool ACC>
__device__ __forceinline__ void dyn_adjoint(float l, float r, float gl, float gr, float gc, const DynP& q,
                                            float wf, float om, bool bypass, float& ol, float& orr, float& og,
                                            DynAcc& A) {
  const float gcl = fmaxf(gc, 0.f);
  const float G = __logf(gcl + 1e-8f);
  const bool above = G >= q.T + q.W, below = G < q.T - q.W;
  const float d = G - q.T;
  float Gy, dGu, dT, dW, dR;
  if (GATE) {
    const float z = d - q.W, k = 1.f - q.R, zh = z * q.i2W, zq = z * z * q.i4W;
    Gy = G + k * zq;  // knee
    dGu = fmaf(k, zh, 1.f);
    dT = -k * zh;
    dW = k * (-zh - zq * (4.f * q.i4W));
    dR = -zq;
    Gy = above ? G : (below ? fmaf(q.R, d, q.T) : Gy);
    dGu = above ? 1.f : (below ? q.R : dGu);
    dT = above ? 0.f : (below ? 1.f - q.R : dT);
    dW = (above || below) ? 0.f : dW;
    dR = above ? 0.f : (below ? d : dR);
  } else {
    const float z = d + q.W, k = q.iR - 1.f, zh = z * q.i2W, zq = z * z * q.i4W;
    Gy = G + k * zq;  // knee
    dGu = fmaf(k, zh, 1.f);
    dT = -k * zh;
    dW = k * (zh - zq * (4.f * q.i4W));
    dR = -zq * q.iR * q.iR;
    Gy = below ? G : (above ? fmaf(d, q.iR, q.T) : Gy);
    dGu = below ? 1.f : (above ? q.iR : dGu);
    dT = below ? 0.f : (above ? 1.f - q.iR : dT);
    dW = (above || below) ? 0.f : dW;
    dR = below ? 0.f : (above ? -d * q.iR * q.iR : dR);
  }
  const float gain = __expf(Gy - G);
  float dl, dr, ul, ur;
  if (bypass) { dl = dr = 0.f; ul = gl; ur = gr; }
  else {
    dl = wf * gl; dr = wf * gr; ul = om * gl; ur = om * gr;
    if (ACC) A.w = fmaf(gl, l * gain - l, fmaf(gr, r * gain - r, A.w));
  }
  ol = fmaf(dl, gain, ul);
  orr = fmaf(dr, gain, ur);
  const float D = (dl * l + dr * r) * gain;
  if (ACC) {
    A.T = fmaf(D, dT, A.T);
    A.W = fmaf(D, dW, A.W);
    A.R = fmaf(D, dR, A.R);
  }
  const float dG = D * dGu - D;
  og = (gc > 0.f) ? __fdividef(dG, gcl + 1e-8f) : 0.f;
}

// phase A of the backward for one chunk (C = 0: this chunk, accumulate and write the
// elementwise dL/du; C = 1: the next chunk, envelope adjoint only)
template <bool GATE, int C>
__device__ __forceinline__ void dyn_phase_a(const float* u, const float* gy, const float* eo, float* go, int L,
                                            long long c0, bool vec, const DynP& q, float wf, float om, bool bypass,
                                            float* ds, DynAcc& A) {
#pragma unroll 2
  for (int k = 0; k < Q4; ++k) {
    const int o = 4 * (threadIdx.x + NT * k);
    const long long n = c0 + (long long)C * CH + o;
    float4 ul4, ur4, gl4, gr4;
    load4(u, L, n, vec, ul4, ur4);
    load4(gy, L, n, vec, gl4, gr4);
    const float4 ev4 = load4m(eo, L, n, vec);
    const float U[4] = {ul4.x, ul4.y, ul4.z, ul4.w}, V[4] = {ur4.x, ur4.y, ur4.z, ur4.w};
    const float GL[4] = {gl4.x, gl4.y, gl4.z, gl4.w}, GR[4] = {gr4.x, gr4.y, gr4.z, gr4.w};
    const float EV[4] = {ev4.x, ev4.y, ev4.z, ev4.w};
    float OL[4], OR[4];
    float* dst = ds + C * SPAD + sidx_n(o);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float og;
      // samples beyond L load as zeros and contribute nothing to the partial sums
      dyn_adjoint<GATE, C == 0>(U[e], V[e], GL[e], GR[e], EV[e], q, wf, om, bypass, OL[e], OR[e], og, A);
      dst[e] = og;
    }
    if (C == 0 && go)
      store4(go, L, n, vec, make_float4(OL[0], OL[1], OL[2], OL[3]), make_float4(OR[0], OR[1], OR[2], OR[3]),
             nullptr, make_float4(0.f, 0.f, 0.f, 0.f));
  }
}

struct VW {
  double v, w;
};

// state X entering from the right, propagated through len zero-input steps
__device__ __forceinline__ VW prop(VW x, double alen, double len) {
  return VW{alen * x.v, alen * fma(len, x.v, x.w)};
}

__device__ __forceinline__ void rstep(VW& s, double a, double x) {
  s.w = a * (s.w + s.v);
  s.v = fma(a, s.v, x);
}

// Two reverse exclusive scans at once (segments t+1.. of the chunk) of 2-state
// values: returns the state at the END of this thread's segment.
__device__ __forceinline__ void rscan2_excl(VW& a, VW& c, const double* pw, double* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  VW ra = a, rc = c;
#pragma unroll
  for (int o = 1, i = 0; o < 32; o <<= 1, ++i) {
    const double av = __shfl_down_sync(0xffffffffu, ra.v, o), aw = __shfl_down_sync(0xffffffffu, ra.w, o);
    const double cv = __shfl_down_sync(0xffffffffu, rc.v, o), cw = __shfl_down_sync(0xffffffffu, rc.w, o);
    if (lane + o < 32) {
      const double len = (double)SEG * o;
      const VW pa = prop(VW{av, aw}, pw[i], len), pc = prop(VW{cv, cw}, pw[i], len);
      ra.v += pa.v; ra.w += pa.w;
      rc.v += pc.v; rc.w += pc.w;
    }
  }
  if (lane == 0) {
    sh[wid] = ra.v; sh[NW + wid] = ra.w;
    sh[2 * NW + wid] = rc.v; sh[3 * NW + wid] = rc.w;
  }
  __syncthreads();
  if (threadIdx.x < 2) {  // state at the end of warp w from warps w+1..
    double* xv = sh + threadIdx.x * 2 * NW;
    double* xw = xv + NW;
    VW cc{0.0, 0.0};
    for (int w = NW - 1; w >= 0; --w) {
      const VW tot{xv[w], xw[w]};
      xv[w] = cc.v;
      xw[w] = cc.w;
      const VW p = prop(cc, pw[5], (double)SEG * 32);
      cc.v = tot.v + p.v;
      cc.w = tot.w + p.w;
    }
  }
  __syncthreads();
  double nav = __shfl_down_sync(0xffffffffu, ra.v, 1), naw = __shfl_down_sync(0xffffffffu, ra.w, 1);
  double ncv = __shfl_down_sync(0xffffffffu, rc.v, 1), ncw = __shfl_down_sync(0xffffffffu, rc.w, 1);
  if (lane == 31) nav = naw = ncv = ncw = 0.0;
  const int k = 31 - lane;
  const double p = powseg(pw, k);
  const VW wa = prop(VW{sh[wid], sh[NW + wid]}, p, (double)SEG * k);
  const VW wc = prop(VW{sh[2 * NW + wid], sh[3 * NW + wid]}, p, (double)SEG * k);
  a = VW{nav + wa.v, naw + wa.w};
  c = VW{ncv + wc.v, ncw + wc.w};
}

// Backward of one chunk: (A) the elementwise chain for this chunk and the next
// (dL/d envelope staged segment-major in shared memory; this chunk's elementwise
// dL/du written to gu, T/W/R/w partials), then (B) the truncated reverse scans,
// dx and r, dL/du += 2 mid dx and the x.dx / x.r partials.  The next chunk's
// envelope adjoint is recomputed instead of round-tripping dg through HBM.
template <bool GATE>
__global__ void __launch_bounds__(NT, 2) k_dyn_bwd(const float* const* __restrict__ u_rows,
                                                const float* const* __restrict__ gy_rows,
                                                const DynPre* __restrict__ pre,
                                                const int* __restrict__ widx, const double* __restrict__ w,
                                                const float* __restrict__ env, float* __restrict__ gu,
                                                double* __restrict__ part, int L, int nch) {
  mgb_pdl_entry();
  extern __shared__ __align__(16) unsigned char dsm[];
  float* ds = reinterpret_cast<float*>(dsm);  // [2][SPAD]: cur chunk, next chunk
  __shared__ double pw[NPW];
  __shared__ double sh[4 * NW];
  __shared__ double carry[2];
  __shared__ double red[32];
  const int j = blockIdx.x, b = blockIdx.y;
  const float* u = u_rows[b];
  const float* gy = gy_rows[b];
  const DynP q = pre[b].q;
  const double wv = w ? w[widx[b]] : 1.0;
  const float wf = (float)wv, om = (float)(1.0 - wv);
  const bool bypass = wv == 0.0;
  const float* eo = env + (size_t)b * L;
  float* go = gu ? gu + (size_t)b * 2 * L : nullptr;  // null: input gradient not requested
  init_pw(pw, pre[b]);
  const long long c0 = (long long)j * CH;
  const bool vec = vec_ok(u, L) && vec_ok(gy, L) && vec_ok(eo, L) && (!go || vec_ok(go, L));
  DynAcc A{0.f, 0.f, 0.f, 0.f};
  dyn_phase_a<GATE, 0>(u, gy, eo, go, L, c0, vec, q, wf, om, bypass, ds, A);
  dyn_phase_a<GATE, 1>(u, gy, eo, go, L, c0, vec, q, wf, om, bypass, ds, A);
  {
    double t0 = block_sum((double)A.T, red);
    __syncthreads();
    double t1 = block_sum((double)A.W, red);
    __syncthreads();
    double t2 = block_sum((double)A.R, red);
    __syncthreads();
    double t3 = block_sum((double)A.w, red);
    if (threadIdx.x == 0) {
      double* pp = part + ((size_t)b * nch + j) * 8;
      pp[0] = t0;
      pp[1] = t1;
      pp[2] = t2;
      pp[3] = t3;
    }
  }
  __syncthreads();
  const float* dc = ds + sidx(threadIdx.x, 0);
  const float* dn = ds + SPAD + sidx(threadIdx.x, 0);
  VW sc{0.0, 0.0}, sn{0.0, 0.0};
#pragma unroll
  for (int i = SEG - 1; i >= 0; --i) {
    rstep(sc, q.a, (double)dc[i]);
    rstep(sn, q.a, (double)dn[i]);
  }
  // The truncated windows of chunk j end inside chunk j+1, so both recursions start
  // from zero at the end of chunk j+1: the state entering `cur` is the total of
  // `next` (segment aggregates moved to the chunk start, block-summed).
  {
    const VW tn = prop(sn, powseg(pw, threadIdx.x), (double)SEG * threadIdx.x);
    const double tv = block_sum(tn.v, red);
    __syncthreads();
    const double tw = block_sum(tn.w, red);
    if (threadIdx.x == 0) {
      carry[0] = tv;
      carry[1] = tw;
    }
  }
  rscan2_excl(sc, sn, pw, sh);  // (its barriers publish `carry`)
  const double len = (double)SEG * (NT - 1 - threadIdx.x);
  const double alen = powseg(pw, NT - 1 - threadIdx.x);
  const VW cc = prop(VW{carry[0], carry[1]}, alen, len);
  VW stc{sc.v + cc.v, sc.w + cc.w};
  VW stn = sn;
  // each thread overwrites its own dg slots: cur <- dx, next <- r (read before write, same slot)
  float* dcw = ds + sidx(threadIdx.x, 0);
  float* dnw = ds + SPAD + sidx(threadIdx.x, 0);
#pragma unroll
  for (int i = SEG - 1; i >= 0; --i) {
    rstep(stc, q.a, (double)dcw[i]);
    rstep(stn, q.a, (double)dnw[i]);
    dcw[i] = (float)(q.b * (stc.v - q.aC * stn.v));
    dnw[i] = (float)(q.b * (stc.w - q.aC * fma((double)CH, stn.v, stn.w)));
  }
  __syncthreads();
  double sxd = 0.0, sxr = 0.0;
  const bool vg = vec;
#pragma unroll
  for (int k0 = 0; k0 < Q4; k0 += 2) {  // coalesced: dmid = 2 mid dx; sums for d a_raw (2 groups at a time)
  float4 ul[2], ur[2], gl[2], gr[2];
#pragma unroll
  for (int kk = 0; kk < 2; ++kk) {
    const long long m = c0 + 4 * (threadIdx.x + NT * (k0 + kk));
    load4(u, L, m, vg, ul[kk], ur[kk]);
    if (go) load4(go, L, m, vg, gl[kk], gr[kk]);
    else gl[kk] = gr[kk] = make_float4(0.f, 0.f, 0.f, 0.f);
  }
#pragma unroll
  for (int kk = 0; kk < 2; ++kk) {
    const int k = kk;
    const int o = 4 * (threadIdx.x + NT * (k0 + kk));
    const long long m = c0 + o;
    const float* dxp = ds + sidx_n(o);
    const float* rrp = ds + SPAD + sidx_n(o);
    const float lu[4] = {ul[k].x, ul[k].y, ul[k].z, ul[k].w}, ru[4] = {ur[k].x, ur[k].y, ur[k].z, ur[k].w};
    float ol[4] = {gl[k].x, gl[k].y, gl[k].z, gl[k].w}, orr[4] = {gr[k].x, gr[k].y, gr[k].z, gr[k].w};
    float fxd = 0.f, fxr = 0.f;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (m + e >= L) continue;
      const float mid = lu[e] + ru[e];
      const float x = mid * mid;
      fxd = fmaf(x, dxp[e], fxd);
      fxr = fmaf(x, rrp[e], fxr);
      const float dm = 2.f * mid * dxp[e];
      ol[e] += dm;
      orr[e] += dm;
    }
    sxd += (double)fxd;
    sxr += (double)fxr;
    if (go)
      store4(go, L, m, vg, make_float4(ol[0], ol[1], ol[2], ol[3]), make_float4(orr[0], orr[1], orr[2], orr[3]),
             nullptr, make_float4(0.f, 0.f, 0.f, 0.f));
  }
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

__global__ void k_dyn_final(const double* __restrict__ part0, int nblk0, int nch, const double* __restrict__ bank,
                            const int* __restrict__ prow, const int* __restrict__ widx, const double* __restrict__ w,
                            double* __restrict__ gbank, double* __restrict__ gw, const double* __restrict__ part1) {
  mgb_pdl_entry();
  __shared__ double red[32];
  const int b = blockIdx.x;
  double s[6] = {0, 0, 0, 0, 0, 0};
  for (int i = threadIdx.x; i < nblk0; i += blockDim.x) {
    const double* pp = part0 + ((size_t)b * nblk0 + i) * 8;
    s[0] += pp[0]; s[1] += pp[1]; s[2] += pp[2]; s[3] += pp[3];
  }
  for (int i = threadIdx.x; i < nch; i += blockDim.x) {
    const double* pp = part1 + ((size_t)b * nch + i) * 8;
    s[4] += pp[4]; s[5] += pp[5];
  }
  for (int k = 0; k < 6; ++k) {
    s[k] = block_sum(s[k], red);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const DynP q = load_params(bank, prow[b]);
    double* g = gbank + (size_t)prow[b] * 4;
    g[0] = (1.0 - q.a) * s[5] - q.a * s[4];
    g[1] = s[0];
    g[2] = s[1] * expit64(q.Wraw);
    g[3] = s[2] * expit64(q.Rraw);
    const double wv = w ? w[widx[b]] : 1.0;
    if (gw) gw[widx[b]] = (wv == 0.0) ? 0.0 : s[3];
  }
}

int nchunks(int L) { return (L + CH - 1) / CH; }
struct DynWs {
  double* part;  // [B][nch][8]: T, W, R, w partials (phase A) and x.dx, x.r (phase B) per chunk
  DynPre* pre;   // [B]
};

template <class A>
DynWs dcarve(A& a, int B, int L) {
  DynWs w;
  w.part = a.template take<double>((size_t)B * nchunks(L) * 8);
  w.pre = a.template take<DynPre>((size_t)B);
  return w;
}

}  // namespace

int mgb_dyn_init() {
  cudaFuncSetAttribute(k_dyn_fwd<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kDynSmemF);
  cudaFuncSetAttribute(k_dyn_fwd<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kDynSmemF);
  cudaFuncSetAttribute(k_dyn_bwd<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kDynSmem);
  cudaFuncSetAttribute(k_dyn_bwd<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kDynSmem);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

size_t mgb_dyn_workspace(char, int B, int L) {
  MgbArena a{nullptr, 0};
  dcarve(a, B, L);
  return a.off;
}

// forward phase 1 (params only): the per-node parameter blocks
int mgb_dyn_prepare(const MgbLevel* lv, cudaStream_t st) {
  const int B = lv->B, L = lv->L;
  MgbArena a{(char*)lv->ws, 0};
  DynWs w = dcarve(a, B, L);
  mgb_launch(k_dyn_pre, dim3(B), dim3(32), 0, st, lv->bank, lv->prow, w.pre);
  MGB_CHECK_LAUNCH();
  return 0;
}

int mgb_dyn_forward(const MgbLevel* lv, cudaStream_t st) {
  if (!lv->aux) return 1;
  const int B = lv->B, L = lv->L, nch = nchunks(L);
  MgbArena a{(char*)lv->ws, 0};
  DynWs w = dcarve(a, B, L);
  auto kern = lv->tag == 'n' ? k_dyn_fwd<true> : k_dyn_fwd<false>;
  mgb_launch(kern, dim3(dim3(nch, B)), dim3(NT), kDynSmemF, st, lv->u_rows, (const DynPre*)w.pre, lv->widx, lv->w,
             lv->aux, lv->y, L);
  MGB_CHECK_LAUNCH();
  return 0;
}

int mgb_dyn_backward(const MgbLevel* lv, cudaStream_t st) {
  if (!lv->aux) return 1;
  const int B = lv->B, L = lv->L, nch = nchunks(L);
  MgbArena a{(char*)lv->ws, 0};
  DynWs w = dcarve(a, B, L);
  auto kern = lv->tag == 'n' ? k_dyn_bwd<true> : k_dyn_bwd<false>;
  mgb_launch(kern, dim3(nch, B), dim3(NT), kDynSmem, st, lv->u_rows, lv->gy_rows, (const DynPre*)w.pre, lv->widx,
             lv->w, lv->aux, lv->gu, w.part, L, nch);
  MGB_CHECK_LAUNCH();
  return 0;
}

// backward phase 2: per-node reductions into gbank / gw
int mgb_dyn_param_grad(const MgbLevel* lv, cudaStream_t st) {
  const int B = lv->B, L = lv->L, nch = nchunks(L);
  MgbArena a{(char*)lv->ws, 0};
  DynWs w = dcarve(a, B, L);
  mgb_launch(k_dyn_final, dim3(B), dim3(256), 0, st, w.part, nch, nch, lv->bank, lv->prow, lv->widx, lv->w, lv->gbank,
             lv->gw, w.part);
  MGB_CHECK_LAUNCH();
  return 0;
}
