// Optimiser step on device (mg/optimizer.py:82-137), float64 throughout:
//   1. raw dry/wet gradient: g_raw = dL/dw * mask * s(1-s) + alpha_p * s(1-s)
//      (effective_weights + sparsity_loss, mg/scheduler.py:218-222, mg/losses.py:181-183)
//   2. delay rule on the d-bank z gradients: sgn(raw) + 0.01(|z|-1) conj(z)/|z|
//   3. AdamW over the flat vector (banks + raw weights), fresh-state semantics
//      are the caller's (moments zeroed at each train() call)
//   4. unit-disk projection of every delay z
// all in one pass (k_optim_step), with the sticky non-finite guard.
// The AdamW arithmetic is written with explicit round-to-nearest ops so nvcc
// does not contract it into FMAs: it reproduces numpy's operation order.
#include "common.cuh"
#include "mgb_internal.h"

namespace {

__device__ __forceinline__ void adamw_update(double* __restrict__ p, double* __restrict__ m,
                                             double* __restrict__ v, long long i, double gi, double lr,
                                             double b1, double b2, double eps, double wd, double c1, double c2) {
  double mi = m[i], vi = v[i], pi = p[i];
  mi = __dadd_rn(mi, __dmul_rn(__dsub_rn(1.0, b1), __dsub_rn(gi, mi)));
  vi = __dadd_rn(vi, __dmul_rn(__dsub_rn(1.0, b2), __dsub_rn(__dmul_rn(gi, gi), vi)));
  const double mh = __ddiv_rn(mi, c1);
  const double den = __dadd_rn(__dsqrt_rn(__ddiv_rn(vi, c2)), eps);
  const double upd = __dadd_rn(__ddiv_rn(mh, den), __dmul_rn(wd, pi));
  pi = __dsub_rn(pi, __dmul_rn(lr, upd));
  m[i] = mi;
  v[i] = vi;
  p[i] = pi;
}

// NonFiniteLoss (mg/optimizer.py:164-171): the reference raises at the first step whose
// loss is non-finite, before any update, and the run ends there.  On the device the
// flag is sticky: once a step's loss is non-finite, that step and every later step of
// the same run leave parameters and moments untouched (the host raises after reading
// the per-step losses back, with the parameters as of the last finite step).
//
// The whole step in one pass (steps 1-4 of the header with the non-finite guard), the
// same arithmetic as the separate kernels above: a thread owns whole delay taps (the
// re/im pair of one z: rule, both AdamW updates, projection), a raw weight (its
// gradient, then AdamW), or a plain parameter.  The updated gradients are written back
// as the separate steps leave them.
__global__ void k_optim_step(double* __restrict__ p, double* __restrict__ g, double* __restrict__ m,
                             double* __restrict__ v, long long n, long long d_off, int d_rows, long long w_off,
                             int P, const double* __restrict__ gw, const double* __restrict__ mask,
                             const double* __restrict__ sc, const double* __restrict__ guard,
                             double* __restrict__ halt) {
  mgb_pdl_entry();
  const bool nonfinite = guard && !isfinite(*guard);
  // sticky flag: set by one thread; every thread decides from the flag's previous value
  // and the loss itself, so the order of that write does not matter
  const bool bad = nonfinite || (halt && *halt != 0.0);
  if (halt && nonfinite && blockIdx.x == 0 && threadIdx.x == 0) *halt = 1.0;
  const double lr = sc[0], b1 = sc[1], b2 = sc[2], eps = sc[3], wd = sc[4], c1 = sc[5], c2 = sc[6];
  const long long d_end = d_off + (long long)d_rows * 880;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    if (i >= d_off && i < d_end) {
      const int q = (int)((i - d_off) % 440);  // [20 z re | 20 z im | 400 colour bins] per channel
      if (q < 20) {
        const long long re = i, im = i + 20;
        const double zr = p[re], zi = p[im], gr = g[re], gi = g[im];
        const double mag = hypot(gr, gi);
        double sr = 0.0, si = 0.0;
        if (mag > 0.0) { sr = gr / mag; si = gi / mag; }
        const double zm = hypot(zr, zi);
        double cr = 0.0, ci = 0.0;
        if (zm > 0.0) { cr = zr / zm; ci = -zi / zm; }
        const double k = 0.01 * (zm - 1.0);
        const double nr = sr + k * cr, ni = si + k * ci;
        g[re] = nr;
        g[im] = ni;
        if (bad) continue;
        adamw_update(p, m, v, re, nr, lr, b1, b2, eps, wd, c1, c2);
        adamw_update(p, m, v, im, ni, lr, b1, b2, eps, wd, c1, c2);
        const double pr = p[re], pim = p[im];
        const double pm = __dsqrt_rn(__dadd_rn(__dmul_rn(pr, pr), __dmul_rn(pim, pim)));
        const double s = pm > 1.0 ? 1.0 / pm : 1.0;
        p[re] = pr * s;
        p[im] = pim * s;
        continue;
      }
      if (q < 40) continue;  // the im half of a tap: its re thread owns the pair
    }
    double gi;
    if (i >= w_off && i < w_off + P) {
      const int r = (int)(i - w_off);
      const double sg = expit64(p[i]);
      const double ds = sg * (1.0 - sg);
      gi = gw[r] * (mask ? mask[r] : 1.0) * ds;
      const double ap = sc[7];
      if (ap > 0.0) gi += ap * ds;
      g[i] = gi;
    } else {
      gi = g[i];
    }
    if (!bad) adamw_update(p, m, v, i, gi, lr, b1, b2, eps, wd, c1, c2);
  }
}

__global__ void k_sparsity(const double* __restrict__ raw, int P, double* __restrict__ out) {
  mgb_pdl_entry();
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < P; i += blockDim.x) s += expit64(raw[i]);
  s = block_sum(s, red);
  if (threadIdx.x == 0) *out = s;
}

// L = L_a + w_g * sum(reg) + alpha_p * sum sigma(raw)  (mg/optimizer.py:156-162), one
// signal per thread q: reg rows [reg_off[q], reg_off[q+1]), in row order
__global__ void k_loss_assembly(const double* __restrict__ la, const double* __restrict__ reg,
                                const int* __restrict__ reg_off, const int* __restrict__ reg_idx,
                                const double* __restrict__ sparsity,
                                const double* __restrict__ sc, double gain_w, int n, double* __restrict__ vals,
                                double* __restrict__ guard) {
  mgb_pdl_entry();
  const int q = threadIdx.x;
  __shared__ double tot[1024];
  if (q < n) {
    double r = 0.0;
    const int r0 = reg_off ? reg_off[q] : 0, r1 = reg_off ? reg_off[q + 1] : 0;
    for (int i = r0; i < r1; ++i) r += reg[reg_idx ? reg_idx[i] : i];
    const double ap = sc[7];
    double total = la[q] + r * gain_w;
    if (ap > 0.0) total += ap * sparsity[q];
    vals[q * 4 + 0] = total;
    vals[q * 4 + 1] = la[q];
    vals[q * 4 + 2] = r;
    vals[q * 4 + 3] = sparsity[q];
    tot[q] = total;
  }
  __syncthreads();
  if (q == 0 && guard) {
    double g = 0.0;
    for (int i = 0; i < n; ++i) g += tot[i];
    *guard = g;
  }
}

}  // namespace

extern "C" int mgb_loss_assembly(const double* la, const double* reg, const int* reg_off, const int* reg_idx,
                                 const double* sparsity, const double* step_scalars, double gain_w, int n, double* vals,
                                 double* guard, void* stream) {
  if (n <= 0 || n > 1024 || !la || !sparsity || !step_scalars || !vals) return 1;
  if (reg_off && !reg) return 1;
  mgb_launch(k_loss_assembly, dim3(1), dim3((n + 31) / 32 * 32), 0, (cudaStream_t)stream, la, reg, reg_off, reg_idx,
             sparsity, step_scalars, gain_w, n, vals, guard);
  MGB_CHECK_LAUNCH();
  return 0;
}

extern "C" int mgb_adamw_step(double* p, double* g, double* m, double* v, long long n, long long d_off, int d_rows,
                              long long w_off, int P, const double* gw, const double* mask,
                              const double* step_scalars, const double* loss_guard, double* halt,
                              void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n <= 0) return 0;
  if (halt && !loss_guard) return 1;
  const int blocks = (int)((n + 255) / 256 < 1184 ? (n + 255) / 256 : 1184);
  mgb_launch(k_optim_step, dim3(blocks), dim3(256), 0, st, p, g, m, v, n, d_off, d_rows, w_off, P, gw, mask,
             step_scalars, loss_guard, halt);
  MGB_CHECK_LAUNCH();
  return 0;
}

extern "C" int mgb_sparsity(const double* raw, int P, double* out, void* stream) {
  mgb_launch(k_sparsity, dim3(1), dim3(256), 0, (cudaStream_t)stream, raw, P, out);
  MGB_CHECK_LAUNCH();
  return 0;
}
