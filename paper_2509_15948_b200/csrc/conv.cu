// FFT-convolution levels: equalizer (e), reverb (r), multitap delay (d).
//
// fft_conv and its two adjoints (mg/engine.py:549-585), batched over the B
// nodes of a level, with N = next_pow2(L + M - 1) as the reference chooses it
// and the stereo channels packed as one complex signal (left + i*right).
//
// Forward, 4 launches after FIR synthesis (fourstep.cuh):
//   colA(H)  column pass of the compact packed FIR
//   colA(X)  column pass of the packed input rows (read straight from the
//            producer level through the row-pointer table)
//   rowB     row FFTs of X and H (both kept, row layout, for the backward),
//            paired product X_l H_l + i X_r H_r, row IFFT
//   colC     column IFFT + epilogue: ybar = conv[off:off+L], dry/wet,
//            gain-staging norm partials (mg/processors.py:61-90)
// Backward, 4 launches before the FIR adjoint:
//   colA(G)  column pass whose loader IS the backward prologue: dybar =
//            w*gy + gain-staging term, gu = (1-w)*gy + gain-staging term,
//            dw partials
//   rowB     row FFT of G, GX = G conj(H), GH = G conj(X) paired, row IFFTs
//   colC(GX) gu += gx[0:L];   colC(GH) dh = gh[0:M] (compact)
//
// FIRs:  e  zero_phase_fir(p, 2047), same FIR on both channels, offset 1023
//        r  STFT-domain filtered noise, 313 frames x 384, OLA, / wss, offset 0
//        d  20 taps x 39-tap colour FIRs at m*3000 + quantised offset, offset 19;
//           custom surrogate backward (mg/processors.py:250-318)
#include <stdlib.h>

#include "common.cuh"
#include "fourstep.cuh"
#include "fs2.cuh"
#include "fs2_col64.cuh"
#include "mgb_internal.h"
#include "tables.cuh"

namespace {

constexpr int NT = 256;
constexpr int kMaxParts = 1024;  // partial-sum slots per row
constexpr double PI = 3.141592653589793238462643383279502884;

#include "fir.cuh"
#include "rev_fft.cuh"
#include "eq_os.cuh"

int g_num_sms = 148;
// MGB_COLC_PERSISTENT=1: the persistent bulk-copy-pipelined column pass (fs2::k_colC_p) instead of
// one tile per CTA.  Measured slower (336 vs 437 steps/s), kept off for A/B runs.
bool g_colc_persistent = false;
// Narrow levels move their FIR-gradient transform to backward phase 2 (side stream, off
// the critical path): conv levels of at most g_split_rows (B x N1) rows, EQ levels of at
// most g_split_fir_b nodes with one overlap-save block per backward CTA.  Measured
// (MGB_SPLIT_ROWS / MGB_SPLIT_FIR_B): config 1 +7.7 %, config 2 +1.3 %; wide levels
// (B = 16 at N1 = 512, B = 4 at N1 = 2048) are slower split: the GPU is saturated there.
int g_split_rows = 2048;
int g_split_fir_b = 4;
bool split_fir_rows(int B, int N1) { return (long long)B * N1 <= g_split_rows; }
bool eos_split(int L, int B) { return B <= g_split_fir_b && eos_per(L, B) == 1; }

struct ConvGeom {
  int M, off, logN;
  long long N;
};

ConvGeom geom(char tag, int L) {
  ConvGeom g;
  g.M = tag == 'e' ? MGB_EQ_LEN : (tag == 'r' ? MGB_REV_LEN : MGB_DLY_FIR);
  g.off = tag == 'e' ? (MGB_EQ_LEN - 1) / 2 : (tag == 'r' ? 0 : (MGB_COLOR_LEN - 1) / 2);
  g.logN = mgb_log2_ceil((long long)L + g.M - 1);
  if (g.logN < 12) g.logN = 12;
  g.N = 1LL << g.logN;
  return g;
}

struct ConvWs {
  float2 *Ax, *Ah, *X, *H, *Bo;
  float2 *hbuf, *ghbuf;        // compact (B, M) packed FIR and FIR gradient
  double* stats;               // [B][4]: nu, ny, sign(diff), spare
  double* part;                // [B][kMaxParts][4]
  float* aux;                  // r: frames (B,2,313,384) | d: colours (B,2,20,39)
  float* aux2;                 // r: dexpo (B,2,313,193)
  int* offs;                   // d: (B,2,20) quantised delays
  float2 *Hs, *pspec, *csum;   // e (overlap-save): 8192-pt FIR spectra, per-block / summed dh cross spectra
};

template <class A>
ConvWs carve_into(A& a, char tag, int B, int L) {
  const ConvGeom g = geom(tag, L);
  ConvWs w;
  w.Hs = w.pspec = w.csum = nullptr;
  if (tag == 'e') {  // overlap-save path: no four-step buffers
    w.Ax = w.Ah = w.X = w.H = w.Bo = nullptr;
    w.hbuf = a.template take<float2>((size_t)B * g.M);
    w.ghbuf = a.template take<float2>((size_t)B * g.M);
    w.stats = a.template take<double>((size_t)B * 4);
    w.part = a.template take<double>((size_t)B * kMaxParts * 4);
    w.aux = w.aux2 = nullptr;
    w.offs = nullptr;
    w.Hs = a.template take<float2>((size_t)B * EOS_N);
    w.pspec = a.template take<float2>((size_t)B * eos_nchunk(L, B) * 2 * EOS_N);  // D park + C accumulator per CTA
    w.csum = a.template take<float2>((size_t)B * EOS_N);
    return w;
  }
  const size_t BN = (size_t)B * g.N;
  w.Ax = a.template take<float2>(BN);
  w.Ah = a.template take<float2>(BN);
  w.X = a.template take<float2>(BN);
  w.H = a.template take<float2>(BN);
  w.Bo = a.template take<float2>(BN);
  w.hbuf = a.template take<float2>((size_t)B * g.M);
  w.ghbuf = a.template take<float2>((size_t)B * g.M);
  w.stats = a.template take<double>((size_t)B * 4);
  w.part = a.template take<double>((size_t)B * kMaxParts * 4);
  w.aux = w.aux2 = nullptr;
  w.offs = nullptr;
  if (tag == 'r') {
    w.aux = a.template take<float>((size_t)B * 2 * MGB_REV_FRAMES * MGB_REV_NFFT);
    w.aux2 = a.template take<float>((size_t)B * 2 * MGB_REV_FRAMES * MGB_REV_BINS);
  } else if (tag == 'd') {
    w.aux = a.template take<float>((size_t)B * 2 * MGB_DLY_TAPS * MGB_COLOR_LEN);
    w.offs = a.template take<int>((size_t)B * 2 * MGB_DLY_TAPS);
  }
  return w;
}

// ---------------------------------------------------------------------------
// loaders (column pass inputs) and epilogues (column pass outputs)

struct NoCtx {};

__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

struct LdRows {
  static constexpr bool kAccum = false;
  static constexpr int kBatch = 8;  // loads per pipelined batch (register budget)
  typedef NoCtx Ctx;
  typedef float2 Raw;
  const float* const* rows;
  int L;
  __device__ __forceinline__ Ctx prepare(int) const { return Ctx{}; }
  __device__ __forceinline__ Raw fetch(const Ctx&, int b, long long n, bool ok) const {
    if (!ok || n >= L) return make_float2(0.f, 0.f);
    const float* u = rows[b];
    return make_float2(__ldg(u + n), __ldg(u + L + n));
  }
  __device__ __forceinline__ float2 finish(const Ctx&, int, long long, const Raw& r, float&) const { return r; }
  __device__ __forceinline__ void commit(int, int, double) const {}
};

struct LdFir {
  static constexpr bool kAccum = false;
  static constexpr int kBatch = 8;
  typedef NoCtx Ctx;
  typedef float2 Raw;
  const float2* h;
  int M;
  __device__ __forceinline__ Ctx prepare(int) const { return Ctx{}; }
  __device__ __forceinline__ Raw fetch(const Ctx&, int b, long long n, bool ok) const {
    return (ok && n < M) ? __ldg(h + (size_t)b * M + n) : make_float2(0.f, 0.f);
  }
  __device__ __forceinline__ float2 finish(const Ctx&, int, long long, const Raw& r, float&) const { return r; }
  __device__ __forceinline__ void commit(int, int, double) const {}
};

// Backward prologue (dry/wet + gain-staging adjoints) as the G loader.
struct LdBwdPro {
  static constexpr bool kAccum = true;
  static constexpr int kBatch = 4;
  struct Ctx {
    const float* u;
    const float* gy;
    const float* yb;
    float* go;
    float wf, om, cy, cu;
    bool bypass;
  };
  struct Raw {
    float l, r, gl, gr, yl, yr;
    bool in;
  };
  const float* const* u_rows;
  const float* const* gy_rows;
  const float* ybar;
  const int* widx;
  const double* w;
  const double* greg;
  const double* stats;
  float* gu;
  double* part;
  int L, off;
  __device__ __forceinline__ Ctx prepare(int b) const {
    Ctx c;
    const double wv = w ? w[widx[b]] : 1.0;
    const double sg = stats[b * 4 + 2] * (greg ? *greg : 0.0);
    const double nu = stats[b * 4], ny = stats[b * 4 + 1];
    c.cy = (ny > 0.0) ? (float)(sg / ((ny + MGB_GS_EPS) * ny)) : 0.f;
    c.cu = (nu > 0.0) ? (float)(-sg / ((nu + MGB_GS_EPS) * nu)) : 0.f;
    c.bypass = (wv == 0.0);
    c.wf = (float)wv;
    c.om = (float)(1.0 - wv);
    c.u = u_rows[b];
    c.gy = gy_rows[b];
    c.yb = ybar + (size_t)b * 2 * L;
    c.go = gu ? gu + (size_t)b * 2 * L : nullptr;  // null: input gradient not requested
    return c;
  }
  __device__ __forceinline__ Raw fetch(const Ctx& c, int, long long n, bool ok) const {
    // zero defaults (not "undefined"): otherwise the compiler seeds the predicated-off
    // destinations with earlier loaded registers, chaining each batch on the last one
    Raw r{0.f, 0.f, 0.f, 0.f, 0.f, 0.f, false};
    const long long m = n - off;
    r.in = ok && m >= 0 && m < L;
    if (r.in) {
      r.l = __ldg(c.u + m);
      r.r = __ldg(c.u + L + m);
      r.gl = __ldg(c.gy + m);
      r.gr = __ldg(c.gy + L + m);
      r.yl = __ldg(c.yb + m);
      r.yr = __ldg(c.yb + L + m);
    }
    return r;
  }
  __device__ __forceinline__ float2 finish(const Ctx& c, int, long long n, const Raw& r, float& acc) const {
    if (!r.in) return make_float2(0.f, 0.f);
    const long long m = n - off;
    const float my = r.yl + r.yr, mu = r.l + r.r;
    float dl, dr, ul, ur;
    if (c.bypass) {
      dl = dr = 0.f;
      ul = r.gl;
      ur = r.gr;
    } else {
      dl = c.wf * r.gl;
      dr = c.wf * r.gr;
      ul = c.om * r.gl;
      ur = c.om * r.gr;
      acc = fmaf(r.gl, r.yl - r.l, fmaf(r.gr, r.yr - r.r, acc));
    }
    if (c.go) {
      c.go[m] = fmaf(c.cu, mu, ul);
      c.go[L + m] = fmaf(c.cu, mu, ur);
    }
    return make_float2(fmaf(c.cy, my, dl), fmaf(c.cy, my, dr));
  }
  __device__ __forceinline__ void commit(int b, int blk, double t) const { part[((size_t)b * kMaxParts + blk) * 4 + 2] = t; }
};

struct EpFwd {
  static constexpr bool kAccum = true;
  static constexpr bool kPrefetch = true;
  struct Ctx {
    const float* u;
    float* yo;
    float* yb;
    float wf, om;
    bool bypass;
  };
  typedef float2 Raw;
  const float* const* u_rows;
  const int* widx;
  const double* w;
  float* y;
  float* ybar;
  double* part;
  int L, off;
  __device__ __forceinline__ Ctx prepare(int b) const {
    Ctx c;
    const double wv = w ? w[widx[b]] : 1.0;
    c.bypass = (wv == 0.0);
    c.wf = (float)wv;
    c.om = (float)(1.0 - wv);
    c.u = u_rows[b];
    c.yo = y + (size_t)b * 2 * L;
    c.yb = ybar + (size_t)b * 2 * L;
    return c;
  }
  __device__ __forceinline__ Raw fetch(const Ctx& c, int, long long n, bool ok) const {
    const long long m = n - off;
    if (!ok || m < 0 || m >= L) return make_float2(0.f, 0.f);
    return make_float2(__ldg(c.u + m), __ldg(c.u + L + m));
  }
  // the dry input of a later epilogue batch, requested into L2 before the transform
  // (measured: +0.9 % steps/s; the same hook on the column loaders and on EpGx was slower)
  __device__ __forceinline__ void prefetch(const Ctx& c, long long n, int) const {
    const long long m = n - off;
    if (m >= 0 && m < L) {
      prefetch_l2(c.u + m);
      prefetch_l2(c.u + L + m);
    }
  }
  __device__ __forceinline__ void finish(const Ctx& c, int, long long n, float2 v, const Raw& u, float& a0,
                                         float& a1) const {
    const long long m = n - off;
    if (m < 0 || m >= L) return;
    c.yb[m] = v.x;
    c.yb[L + m] = v.y;
    if (c.bypass) {
      c.yo[m] = u.x;
      c.yo[L + m] = u.y;
    } else {
      c.yo[m] = c.wf * v.x + c.om * u.x;
      c.yo[L + m] = c.wf * v.y + c.om * u.y;
    }
    const float mu = u.x + u.y, my = v.x + v.y;
    a0 = fmaf(mu, mu, a0);
    a1 = fmaf(my, my, a1);
  }
  __device__ __forceinline__ void commit(int b, int blk, double t0, double t1) const {
    double* pp = part + ((size_t)b * kMaxParts + blk) * 4;
    pp[0] = t0;
    pp[1] = t1;
  }
};

struct EpGx {
  static constexpr bool kAccum = false;
  static constexpr int kBatch64 = 2;  // k_colC64: a batch of 8 spilled 116 bytes, 4 spilled 32, at the 128-register cap
  typedef NoCtx Ctx;
  typedef float2 Raw;
  float* gu;
  int L;
  __device__ __forceinline__ Ctx prepare(int) const { return Ctx{}; }
  __device__ __forceinline__ Raw fetch(const Ctx&, int b, long long n, bool ok) const {
    if (!ok || n >= L) return make_float2(0.f, 0.f);
    const float* go = gu + (size_t)b * 2 * L;
    return make_float2(go[n], go[L + n]);
  }
  __device__ __forceinline__ void finish(const Ctx&, int b, long long n, float2 v, const Raw& g, float&,
                                         float&) const {
    if (n >= L) return;
    float* go = gu + (size_t)b * 2 * L;
    go[n] = g.x + v.x;
    go[L + n] = g.y + v.y;
  }
  __device__ __forceinline__ void commit(int, int, double, double) const {}
};

struct EpGh {
  static constexpr bool kAccum = false;
  typedef NoCtx Ctx;
  typedef int Raw;
  float2* gh;
  int M;
  __device__ __forceinline__ Ctx prepare(int) const { return Ctx{}; }
  __device__ __forceinline__ Raw fetch(const Ctx&, int, long long, bool) const { return 0; }
  __device__ __forceinline__ void finish(const Ctx&, int b, long long n, float2 v, const Raw&, float&,
                                         float&) const {
    if (n < M) gh[(size_t)b * M + n] = v;
  }
  __device__ __forceinline__ void commit(int, int, double, double) const {}
};

// norms and gain-staging term |log(ny+eps) - log(nu+eps)|  (mg/processors.py:83-90)
__global__ void k_gs_norms(const double* __restrict__ part, int nblk, double* __restrict__ stats,
                           double* __restrict__ reg) {
  mgb_pdl_entry();
  __shared__ double red[32];
  const int b = blockIdx.x;
  double su = 0.0, sy = 0.0;
  for (int i = threadIdx.x; i < nblk; i += blockDim.x) {
    su += part[((size_t)b * kMaxParts + i) * 4];
    sy += part[((size_t)b * kMaxParts + i) * 4 + 1];
  }
  su = block_sum(su, red);
  __syncthreads();
  sy = block_sum(sy, red);
  if (threadIdx.x == 0) {
    const double nu = sqrt(su), ny = sqrt(sy);
    const double diff = log(ny + MGB_GS_EPS) - log(nu + MGB_GS_EPS);
    stats[b * 4 + 0] = nu;
    stats[b * 4 + 1] = ny;
    stats[b * 4 + 2] = (diff > 0.0) ? 1.0 : (diff < 0.0 ? -1.0 : 0.0);
    if (reg) reg[b] = fabs(diff);
  }
}

__global__ void k_dw_finalize(const double* __restrict__ part, int nblk, const int* __restrict__ widx,
                              const double* __restrict__ w, double* __restrict__ gw) {
  mgb_pdl_entry();
  __shared__ double red[32];
  const int b = blockIdx.x;
  double s = 0.0;
  for (int i = threadIdx.x; i < nblk; i += blockDim.x) s += part[((size_t)b * kMaxParts + i) * 4 + 2];
  s = block_sum(s, red);
  if (threadIdx.x == 0 && gw) {
    const double wv = w ? w[widx[b]] : 1.0;
    gw[widx[b]] = (wv == 0.0) ? 0.0 : s;
  }
}

constexpr int kDlyBwdSmem = 0;

// ---------------------------------------------------------------------------
// per-size drivers

template <int N1, int N2>
struct Conv {
  using G = fs::Geo<N1, N2>;
  static constexpr int DW_NBLK = N2 / G::TC;  // column CTAs per node = dw partial slots
  static void attrs() {
    const int sc = (int)fs::col_smem<N1, N2>(), sr = (int)fs::row_smem<N1, N2>();
    cudaFuncSetAttribute(fs::k_colA<N1, N2, LdRows>, cudaFuncAttributeMaxDynamicSharedMemorySize, sc);
    cudaFuncSetAttribute(fs::k_colA<N1, N2, LdFir>, cudaFuncAttributeMaxDynamicSharedMemorySize, sc);
    cudaFuncSetAttribute(fs::k_colA<N1, N2, LdBwdPro>, cudaFuncAttributeMaxDynamicSharedMemorySize, sc);
    cudaFuncSetAttribute(fs::k_colC<N1, N2, EpFwd>, cudaFuncAttributeMaxDynamicSharedMemorySize, sc);
    cudaFuncSetAttribute(fs::k_colC<N1, N2, EpGx>, cudaFuncAttributeMaxDynamicSharedMemorySize, sc);
    cudaFuncSetAttribute(fs::k_colC<N1, N2, EpGh>, cudaFuncAttributeMaxDynamicSharedMemorySize, sc);
    cudaFuncSetAttribute(fs::k_rowB_fwd<N1, N2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sr);
    cudaFuncSetAttribute(fs::k_rowB_bwd<N1, N2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)fs::rowbwd_smem<N1, N2>());
  }

  static int prep(const MgbLevel* lv, const ConvWs& w, const ConvGeom& g, cudaStream_t st) {
    const dim3 gc(N2 / G::TC, lv->B);
    const int fir_rows = (int)((g.M + N2 - 1) / N2);
    mgb_launch(fs::k_colA<N1, N2, LdFir>, dim3(gc), dim3(G::NTC), fs::col_smem<N1, N2>(), st, LdFir{w.hbuf, g.M}, w.Ah,
                                                                  fir_rows < N1 ? fir_rows : N1);
    MGB_CHECK_LAUNCH();
    return 0;
  }

  static int fwd(const MgbLevel* lv, const ConvWs& w, const ConvGeom& g, cudaStream_t st) {
    const int B = lv->B, L = lv->L;
    const dim3 gc(N2 / G::TC, B), gr(N1 / 2 + 1, B);
    const size_t sc = fs::col_smem<N1, N2>(), sr = fs::row_smem<N1, N2>();
    const int x_rows = (int)((L + N2 - 1) / N2);
    mgb_launch(fs::k_colA<N1, N2, LdRows>, dim3(gc), dim3(G::NTC), sc, st, LdRows{lv->u_rows, L}, w.Ax, x_rows < N1 ? x_rows : N1);
    MGB_CHECK_LAUNCH();
    mgb_launch(fs::k_rowB_fwd<N1, N2>, dim3(gr), dim3(G::NTR), sr, st, w.Ax, w.Ah, w.X, w.H, w.Bo);
    MGB_CHECK_LAUNCH();
    EpFwd ep{lv->u_rows, lv->widx, lv->w, lv->y, lv->ybar, w.part, L, g.off};
    mgb_launch(fs::k_colC<N1, N2, EpFwd>, dim3(gc), dim3(G::NTC), sc, st, w.Bo, ep, 1.f / (float)G::N, N1);
    MGB_CHECK_LAUNCH();
    return 0;
  }

  static int bwd(const MgbLevel* lv, const ConvWs& w, const ConvGeom& g, cudaStream_t st) {
    const int B = lv->B, L = lv->L;
    const dim3 gc(N2 / G::TC, B), gr(N1 / 2 + 1, B);
    const size_t sc = fs::col_smem<N1, N2>(), sr = fs::row_smem<N1, N2>();
    LdBwdPro ld{lv->u_rows, lv->gy_rows, lv->ybar, lv->widx, lv->w, lv->greg, w.stats, lv->gu, w.part, L, g.off};
    const int g_rows = (int)((g.off + L + N2 - 1) / N2);
    mgb_launch(fs::k_colA<N1, N2, LdBwdPro>, dim3(gc), dim3(G::NTC), sc, st, ld, w.Ax, g_rows < N1 ? g_rows : N1);
    MGB_CHECK_LAUNCH();
    mgb_launch(fs::k_rowB_bwd<N1, N2>, dim3(gr), dim3(G::NTR), fs::rowbwd_smem<N1, N2>(), st, w.Ax, w.X, w.H, w.Bo, w.Ah);
    MGB_CHECK_LAUNCH();
    if (lv->gu) {
      mgb_launch(fs::k_colC<N1, N2, EpGx>, dim3(gc), dim3(G::NTC), sc, st, w.Bo, EpGx{lv->gu, L}, 1.f / (float)G::N,
                 N1);
      MGB_CHECK_LAUNCH();
    }
    return 0;
  }

  // FIR gradient dh = IFFT(G conj(X))[0:M] (backward phase 2)
  static int fir_grad(const MgbLevel* lv, const ConvWs& w, const ConvGeom& g, cudaStream_t st) {
    const dim3 gc(N2 / G::TC, lv->B);
    const int h_rows = (int)((g.M + N2 - 1) / N2);
    mgb_launch(fs::k_colC<N1, N2, EpGh>, dim3(gc), dim3(G::NTC), fs::col_smem<N1, N2>(), st, w.Ah, EpGh{w.ghbuf, g.M},
               1.f / (float)G::N, h_rows < N1 ? h_rows : N1);
    MGB_CHECK_LAUNCH();
    return 0;
  }
};

// register-FFT four-step (fs2.cuh), N = N1 x 1024 with N1 = 4..1024
template <int N1>
struct Conv2 {
  using G = fs2::G<N1>;
  static constexpr int N2 = fs2::N2;
  static constexpr bool C64 = (N1 == 2048);  // 2048-point columns: fs2_col64.cuh
  static constexpr int DW_NBLK = C64 ? fs2::C64::NBLK : G::NBLK;  // column CTAs per node = dw partial slots
  template <class Ld>
  static void colA(const Ld& ld, float2* A, int nz, int rev, int B, cudaStream_t st) {
    if constexpr (C64) {
      mgb_launch(fs2::k_colA64<Ld>, dim3(dim3(N2 / fs2::C64::TC, B)), dim3(fs2::C64::NT), fs2::C64::SMEM, st, ld, A, nz, rev);
    } else {
      mgb_launch(fs2::k_colA<N1, Ld>, dim3(dim3(N2 / G::TC, B)), dim3(G::NT), G::COL_SMEM, st, ld, A, nz, rev);
    }
  }
  template <class Ep>
  static void colC(const float2* Bb, const Ep& ep, int out_rows, int rev, int B, cudaStream_t st) {
    if constexpr (N1 == 512) {
      if (g_colc_persistent) {  // persistent, bulk-copy-pipelined column pass (fs2::k_colC_p)
        const int ntiles = B * fs2::GP<N1>::TILES_PER_NODE;
        mgb_launch(fs2::k_colC_p<N1, Ep>, dim3(ntiles < g_num_sms ? ntiles : g_num_sms), dim3(G::NT),
                   fs2::GP<N1>::SMEM, st, Bb, ep, 1.f / (float)G::N, out_rows, ntiles);
        return;
      }
    }
    if constexpr (C64) {
      mgb_launch(fs2::k_colC64<Ep>, dim3(dim3(N2 / fs2::C64::TC, B)), dim3(fs2::C64::NT), fs2::C64::SMEM, st, Bb, ep,
                 1.f / (float)G::N, out_rows, rev);
    } else {
      mgb_launch(fs2::k_colC<N1, Ep>, dim3(dim3(N2 / G::TC, B)), dim3(G::NT), G::COL_SMEM, st, Bb, ep, 1.f / (float)G::N,
                 out_rows, rev);
    }
  }
  static void attrs() {
    if constexpr (C64) {
      const int s64 = (int)fs2::C64::SMEM;
      cudaFuncSetAttribute(fs2::k_colA64<LdRows>, cudaFuncAttributeMaxDynamicSharedMemorySize, s64);
      cudaFuncSetAttribute(fs2::k_colA64<LdFir>, cudaFuncAttributeMaxDynamicSharedMemorySize, s64);
      cudaFuncSetAttribute(fs2::k_colA64<LdBwdPro>, cudaFuncAttributeMaxDynamicSharedMemorySize, s64);
      cudaFuncSetAttribute(fs2::k_colC64<EpFwd>, cudaFuncAttributeMaxDynamicSharedMemorySize, s64);
      cudaFuncSetAttribute(fs2::k_colC64<EpGx>, cudaFuncAttributeMaxDynamicSharedMemorySize, s64);
      cudaFuncSetAttribute(fs2::k_colC64<EpGh>, cudaFuncAttributeMaxDynamicSharedMemorySize, s64);
    }
    const int sc = C64 ? 0 : (int)G::COL_SMEM;
    if constexpr (!C64) if (sc > 0) {
      cudaFuncSetAttribute(fs2::k_colA<N1, LdRows>, cudaFuncAttributeMaxDynamicSharedMemorySize, sc);
      cudaFuncSetAttribute(fs2::k_colA<N1, LdFir>, cudaFuncAttributeMaxDynamicSharedMemorySize, sc);
      cudaFuncSetAttribute(fs2::k_colA<N1, LdBwdPro>, cudaFuncAttributeMaxDynamicSharedMemorySize, sc);
      cudaFuncSetAttribute(fs2::k_colC<N1, EpFwd>, cudaFuncAttributeMaxDynamicSharedMemorySize, sc);
      cudaFuncSetAttribute(fs2::k_colC<N1, EpGx>, cudaFuncAttributeMaxDynamicSharedMemorySize, sc);
      cudaFuncSetAttribute(fs2::k_colC<N1, EpGh>, cudaFuncAttributeMaxDynamicSharedMemorySize, sc);
    }
    if constexpr (N1 == 512) {
      const int sp = (int)fs2::GP<N1>::SMEM;
      cudaFuncSetAttribute(fs2::k_colC_p<N1, EpFwd>, cudaFuncAttributeMaxDynamicSharedMemorySize, sp);
      cudaFuncSetAttribute(fs2::k_colC_p<N1, EpGx>, cudaFuncAttributeMaxDynamicSharedMemorySize, sp);
      cudaFuncSetAttribute(fs2::k_colC_p<N1, EpGh>, cudaFuncAttributeMaxDynamicSharedMemorySize, sp);
    }
    cudaFuncSetAttribute(fs2::k_rowH<N1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fs2::ROWH_SMEM);
    cudaFuncSetAttribute(fs2::k_rowF<N1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fs2::ROWF_SMEM);
    cudaFuncSetAttribute(fs2::k_rowG<N1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fs2::ROWG_SMEM);
    cudaFuncSetAttribute(fs2::k_rowF<N1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fs2::ROWF_SMEM);
    cudaFuncSetAttribute(fs2::k_rowP<N1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fs2::ROWF_SMEM);
  }

  static int prep(const MgbLevel* lv, const ConvWs& w, const ConvGeom& g, cudaStream_t st) {
    const dim3 gc(N2 / G::TC, lv->B), gr(G::ROW_CTAS, lv->B);
    const int fir_rows = (int)((g.M + N2 - 1) / N2);
    colA(LdFir{w.hbuf, g.M}, w.Ah, fir_rows < N1 ? fir_rows : N1, 0, lv->B, st);
    MGB_CHECK_LAUNCH();
    mgb_launch(fs2::k_rowH<N1>, dim3(gr), dim3(2 * fs2::RP * 32), fs2::ROWH_SMEM, st, w.Ah, w.H, 1);
    MGB_CHECK_LAUNCH();
    return 0;
  }

  static int fwd(const MgbLevel* lv, const ConvWs& w, const ConvGeom& g, cudaStream_t st) {
    const int B = lv->B, L = lv->L;
    const dim3 gc(N2 / G::TC, B), gr(G::ROW_CTAS, B);
    const int x_rows = (int)((L + N2 - 1) / N2);
    colA(LdRows{lv->u_rows, L}, w.Ax, x_rows < N1 ? x_rows : N1, 0, B, st);
    MGB_CHECK_LAUNCH();
    mgb_launch(fs2::k_rowF<N1>, dim3(gr), dim3(2 * fs2::RP * 32), fs2::ROWF_SMEM, st, w.Ax, w.H, w.X, w.Bo, 1);
    MGB_CHECK_LAUNCH();
    EpFwd ep{lv->u_rows, lv->widx, lv->w, lv->y, lv->ybar, w.part, L, g.off};
    colC(w.Bo, ep, N1, 0, B, st);
    MGB_CHECK_LAUNCH();
    return 0;
  }

  static int bwd(const MgbLevel* lv, const ConvWs& w, const ConvGeom& g, cudaStream_t st) {
    const int B = lv->B, L = lv->L;
    const dim3 gc(N2 / G::TC, B), gr(G::ROW_CTAS, B);
    LdBwdPro ld{lv->u_rows, lv->gy_rows, lv->ybar, lv->widx, lv->w, lv->greg, w.stats, lv->gu, w.part, L, g.off};
    const int g_rows = (int)((g.off + L + N2 - 1) / N2);
    colA(ld, w.Ax, g_rows < N1 ? g_rows : N1, 1, B, st);
    MGB_CHECK_LAUNCH();
    if (split_fir_rows(B, N1)) {
      // narrow level (latency-bound): G = FFT(Ag) kept in Ah for the FIR gradient (phase 2,
      // k_rowP, off the critical path), Bo = IFFT(G conj H)
      mgb_launch(fs2::k_rowF<N1, true>, dim3(gr), dim3(2 * fs2::RP * 32), fs2::ROWF_SMEM, st, w.Ax, w.H, w.Ah, w.Bo, 0);
    } else {
      // wide level (the GPU is saturated): all three row transforms in one pass, Ah = the FIR rows
      mgb_launch(fs2::k_rowG<N1>, dim3(gr), dim3(2 * fs2::RP * 32), fs2::ROWG_SMEM, st, w.Ax, w.X, w.H, w.Bo, w.Ah, 0);
    }
    MGB_CHECK_LAUNCH();
    if (lv->gu) {
      colC(w.Bo, EpGx{lv->gu, L}, N1, 1, B, st);
      MGB_CHECK_LAUNCH();
    }
    return 0;
  }

  // FIR gradient dh = IFFT(G conj(X))[0:M] (backward phase 2: only the FIR adjoint reads it)
  static int fir_grad(const MgbLevel* lv, const ConvWs& w, const ConvGeom& g, cudaStream_t st) {
    if (split_fir_rows(lv->B, N1)) {  // the FIR rows from the kept G and X (see bwd)
      const dim3 gr(G::ROW_CTAS, lv->B);
      mgb_launch(fs2::k_rowP<N1>, dim3(gr), dim3(2 * fs2::RP * 32), fs2::ROWF_SMEM, st, w.Ah, w.X, w.Ah, 1);
      MGB_CHECK_LAUNCH();
    }
    const int h_rows = (int)((g.M + N2 - 1) / N2);
    colC(w.Ah, EpGh{w.ghbuf, g.M}, h_rows < N1 ? h_rows : N1, 1, lv->B, st);
    MGB_CHECK_LAUNCH();
    return 0;
  }
};

// register path for N <= 2^21 (N1 <= 2048; 2048 with the split column pass of fs2_col64.cuh),
// the shared-memory Stockham four-step above
#define MGB_CONV_SIZES(X) \
  X(12, 4) X(13, 8) X(14, 16) X(15, 32) X(16, 64) X(17, 128) X(18, 256) X(19, 512) X(20, 1024) X(21, 2048)
#define MGB_CONV_SIZES_OLD(X) X(22, 1024, 4096)

int conv_fwd_dispatch(const MgbLevel* lv, const ConvWs& w, const ConvGeom& g, cudaStream_t st) {
  switch (g.logN) {
#define X(l, a) case l: return Conv2<a>::fwd(lv, w, g, st);
    MGB_CONV_SIZES(X)
#undef X
#define X(l, a, b) case l: return Conv<a, b>::fwd(lv, w, g, st);
    MGB_CONV_SIZES_OLD(X)
#undef X
    default: return 1;
  }
}

int conv_dw_nblk(const ConvGeom& g) {
  switch (g.logN) {
#define X(l, a) case l: return Conv2<a>::DW_NBLK;
    MGB_CONV_SIZES(X)
#undef X
#define X(l, a, b) case l: return Conv<a, b>::DW_NBLK;
    MGB_CONV_SIZES_OLD(X)
#undef X
    default: return 0;
  }
}

int conv_prep_dispatch(const MgbLevel* lv, const ConvWs& w, const ConvGeom& g, cudaStream_t st) {
  switch (g.logN) {
#define X(l, a) case l: return Conv2<a>::prep(lv, w, g, st);
    MGB_CONV_SIZES(X)
#undef X
#define X(l, a, b) case l: return Conv<a, b>::prep(lv, w, g, st);
    MGB_CONV_SIZES_OLD(X)
#undef X
    default: return 1;
  }
}

int conv_firgrad_dispatch(const MgbLevel* lv, const ConvWs& w, const ConvGeom& g, cudaStream_t st) {
  switch (g.logN) {
#define X(l, a) case l: return Conv2<a>::fir_grad(lv, w, g, st);
    MGB_CONV_SIZES(X)
#undef X
#define X(l, a, b) case l: return Conv<a, b>::fir_grad(lv, w, g, st);
    MGB_CONV_SIZES_OLD(X)
#undef X
    default: return 1;
  }
}

int conv_bwd_dispatch(const MgbLevel* lv, const ConvWs& w, const ConvGeom& g, cudaStream_t st) {
  switch (g.logN) {
#define X(l, a) case l: return Conv2<a>::bwd(lv, w, g, st);
    MGB_CONV_SIZES(X)
#undef X
#define X(l, a, b) case l: return Conv<a, b>::bwd(lv, w, g, st);
    MGB_CONV_SIZES_OLD(X)
#undef X
    default: return 1;
  }
}

}  // namespace

int mgb_conv_init() {
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  const char* e = getenv("MGB_COLC_PERSISTENT");
  g_colc_persistent = e ? atoi(e) != 0 : false;
  const char* sf = getenv("MGB_SPLIT_FIR_B");
  g_split_fir_b = sf ? atoi(sf) : 4;
  const char* sr = getenv("MGB_SPLIT_ROWS");
  g_split_rows = sr ? atoi(sr) : 2048;
#define X(l, a) Conv2<a>::attrs();
  MGB_CONV_SIZES(X)
#undef X
#define X(l, a, b) Conv<a, b>::attrs();
  MGB_CONV_SIZES_OLD(X)
#undef X
  cudaFuncSetAttribute(k_eqos_hspec, cudaFuncAttributeMaxDynamicSharedMemorySize, kEosSmem1);
  cudaFuncSetAttribute(k_eqos_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, kEosSmem1);
  cudaFuncSetAttribute(k_eqos_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, kEosSmem1);
  cudaFuncSetAttribute(k_eqos_gh, cudaFuncAttributeMaxDynamicSharedMemorySize, kEosSmem1);
  cudaFuncSetAttribute(k_eqos_bwd_c, cudaFuncAttributeMaxDynamicSharedMemorySize, kEosSmem1);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

size_t mgb_conv_workspace(char tag, int B, int L) {
  MgbArena a{nullptr, 0};
  carve_into(a, tag, B, L);
  return a.off;
}

// forward phase 1: FIR synthesis (+ the FIR column pass / 8192-point spectra), params only
int mgb_conv_prepare(const MgbLevel* lv, cudaStream_t st) {
  const char tag = lv->tag;
  const int B = lv->B, L = lv->L;
  const ConvGeom g = geom(tag, L);
  if (g.logN > 22) return 1;
  MgbArena a{(char*)lv->ws, 0};
  const ConvWs w = carve_into(a, tag, B, L);
  if (tag == 'e') {
    mgb_launch(k_eq_fir, dim3(dim3((MGB_EQ_LEN + 31) / 32, B)), dim3(256), 0, st, lv->bank, lv->prow, w.hbuf);
    MGB_CHECK_LAUNCH();
    mgb_launch(k_eqos_hspec, dim3(B), dim3(EOS_NT), kEosSmem1, st, w.hbuf, w.Hs);
    MGB_CHECK_LAUNCH();
    return 0;
  }
  if (tag == 'r') {
    mgb_launch(k_rev_frames_fft, dim3(dim3((MGB_REV_FRAMES + RV_F - 1) / RV_F, B)), dim3(RV_NT), kRevFftSmem, st, lv->bank, lv->prow,
                                                                                              w.aux);
    MGB_CHECK_LAUNCH();
    mgb_launch(k_rev_assemble, dim3(dim3((MGB_REV_LEN + NT - 1) / NT, B)), dim3(NT), 0, st, w.aux, w.hbuf);
    MGB_CHECK_LAUNCH();
  } else {
    mgb_launch(k_dly_colour, dim3(dim3(MGB_DLY_TAPS, 2, B)), dim3(64), 0, st, lv->bank, lv->prow, w.aux, w.offs);
    MGB_CHECK_LAUNCH();
    mgb_launch(k_dly_place, dim3(dim3((MGB_DLY_FIR + NT - 1) / NT, B)), dim3(NT), 0, st, w.aux, w.offs, w.hbuf);
    MGB_CHECK_LAUNCH();
  }
  return conv_prep_dispatch(lv, w, g, st);
}

// forward phase 2: the signal pass
int mgb_conv_forward(const MgbLevel* lv, cudaStream_t st) {
  const char tag = lv->tag;
  const int B = lv->B, L = lv->L;
  if (!lv->ybar) return 1;
  const ConvGeom g = geom(tag, L);
  if (g.logN > 22) return 1;
  MgbArena a{(char*)lv->ws, 0};
  const ConvWs w = carve_into(a, tag, B, L);
  if (tag == 'e') {
    const int nb = eos_nblk(L);
    mgb_launch(k_eqos_fwd, dim3(dim3(nb, B)), dim3(EOS_NT), kEosSmem1, st, lv->u_rows, w.Hs, lv->widx, lv->w, lv->y, lv->ybar, w.part,
                                                       L);
    MGB_CHECK_LAUNCH();
    return 0;
  }
  return conv_fwd_dispatch(lv, w, g, st);
}

// forward phase 3: gain-staging norms and term per node (read by reg and by the backward)
int mgb_conv_norms(const MgbLevel* lv, cudaStream_t st) {
  const char tag = lv->tag;
  const int B = lv->B, L = lv->L;
  const ConvGeom g = geom(tag, L);
  MgbArena a{(char*)lv->ws, 0};
  const ConvWs w = carve_into(a, tag, B, L);
  mgb_launch(k_gs_norms, dim3(B), dim3(256), 0, st, w.part, tag == 'e' ? eos_nblk(L) : conv_dw_nblk(g), w.stats,
             lv->reg);
  MGB_CHECK_LAUNCH();
  return 0;
}

// backward phase 1: signal adjoint (gu, gw) and the FIR gradient in the workspace
int mgb_conv_backward(const MgbLevel* lv, cudaStream_t st) {
  const char tag = lv->tag;
  const int B = lv->B, L = lv->L;
  if (!lv->ybar) return 1;
  const ConvGeom g = geom(tag, L);
  MgbArena a{(char*)lv->ws, 0};
  const ConvWs w = carve_into(a, tag, B, L);
  if (tag == 'e') {
    const int nb = eos_nblk(L);
    mgb_launch(k_eqos_bwd, dim3(dim3(eos_nchunk(L, B), B)), dim3(EOS_NT), kEosSmem1, st, lv->u_rows, lv->gy_rows,
               lv->ybar, w.Hs, lv->widx, lv->w, lv->greg, w.stats, lv->gu, w.part, w.pspec, L, nb, eos_per(L, B),
               eos_split(L, B) ? 1 : 2);
    MGB_CHECK_LAUNCH();
    return 0;
  }
  return conv_bwd_dispatch(lv, w, g, st);
}

// backward phase 2: FIR adjoint into the gradient bank
int mgb_conv_param_grad(const MgbLevel* lv, cudaStream_t st) {
  const char tag = lv->tag;
  const int B = lv->B, L = lv->L;
  const ConvGeom g = geom(tag, L);
  MgbArena a{(char*)lv->ws, 0};
  const ConvWs w = carve_into(a, tag, B, L);
  // dL/dw from the backward prologue's per-CTA partials (phase 1)
  mgb_launch(k_dw_finalize, dim3(B), dim3(256), 0, st, w.part, tag == 'e' ? eos_nchunk(L, B) : conv_dw_nblk(g),
             lv->widx, lv->w, lv->gw);
  MGB_CHECK_LAUNCH();
  if (tag == 'e') {
    if (eos_split(L, B)) {  // the FIR-gradient pass phase 1 left out (narrow level)
      mgb_launch(k_eqos_bwd_c, dim3(dim3(eos_nchunk(L, B), B)), dim3(EOS_NT), kEosSmem1, st, lv->u_rows, w.pspec, L);
      MGB_CHECK_LAUNCH();
    }
    mgb_launch(k_eqos_csum, dim3(dim3(EOS_N / 256, B)), dim3(256), 0, st, w.pspec, eos_nchunk(L, B), w.csum);
    MGB_CHECK_LAUNCH();
    mgb_launch(k_eqos_gh, dim3(B), dim3(EOS_NT), kEosSmem1, st, w.csum, w.ghbuf);
    MGB_CHECK_LAUNCH();
    mgb_launch(k_eq_fir_bwd, dim3(dim3(MGB_EQ_BINS / 32, B)), dim3(256), 0, st, lv->bank, lv->prow, w.ghbuf, g.M, lv->gbank);
  } else if (tag == 'r') {
    if (int rc = conv_firgrad_dispatch(lv, w, g, st)) return rc;
    mgb_launch(k_rev_bwd_frames_fft, dim3(dim3((MGB_REV_FRAMES + RV_F - 1) / RV_F, B)), dim3(RV_NT), kRevFftSmem, st, 
        lv->bank, lv->prow, w.ghbuf, g.M, reinterpret_cast<double*>(w.aux2));
    MGB_CHECK_LAUNCH();
    mgb_launch(k_rev_bwd_reduce, dim3(dim3((2 * MGB_REV_PBINS + 255) / 256, B)), dim3(256), 0, st,
               reinterpret_cast<const double*>(w.aux2), lv->prow, lv->gbank);
  } else {
    if (int rc = conv_firgrad_dispatch(lv, w, g, st)) return rc;
    mgb_launch(k_dly_bwd, dim3(dim3(MGB_DLY_TAPS, 2, B)), dim3(NT), kDlyBwdSmem, st, lv->bank, lv->prow, w.aux, w.offs, w.ghbuf, g.M,
                                                                 lv->gbank);
  }
  MGB_CHECK_LAUNCH();
  return 0;
}
