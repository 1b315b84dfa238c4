// extern "C" entry points of libmixgraph_b200 (see include/mixgraph_b200.h).
#include <stdio.h>

#include <atomic>

#include "common.cuh"
#include "mgb_internal.h"
#include "tables.cuh"

__device__ float2 g_rev_spec[2][MGB_REV_FRAMES][MGB_REV_BINS];
__device__ float g_rev_inv_wss[MGB_REV_LEN];

extern "C" int mgb_init(const double* reverb_spec_host, const double* reverb_wss_host, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  int rc = mgb_init_device(st);
  if (rc) return rc;
  if ((rc = mgb_conv_init())) return rc;
  if ((rc = mgb_loss_init())) return rc;
  if ((rc = mgb_dyn_init())) return rc;
  if (reverb_spec_host && reverb_wss_host) {
    static float2 spec[2][MGB_REV_FRAMES][MGB_REV_BINS];
    static float inv[MGB_REV_LEN];
    for (int c = 0; c < 2; ++c)
      for (int m = 0; m < MGB_REV_FRAMES; ++m)
        for (int k = 0; k < MGB_REV_BINS; ++k) {
          const double* z = reverb_spec_host + 2 * (((size_t)c * MGB_REV_FRAMES + m) * MGB_REV_BINS + k);
          spec[c][m][k] = make_float2((float)z[0], (float)z[1]);
        }
    for (int t = 0; t < MGB_REV_LEN; ++t) inv[t] = (float)(1.0 / reverb_wss_host[t]);
    if (cudaMemcpyToSymbolAsync(g_rev_spec, spec, sizeof(spec), 0, cudaMemcpyHostToDevice, st) != cudaSuccess)
      return 2;
    if (cudaMemcpyToSymbolAsync(g_rev_inv_wss, inv, sizeof(inv), 0, cudaMemcpyHostToDevice, st) != cudaSuccess)
      return 2;
    if (cudaStreamSynchronize(st) != cudaSuccess) return 2;
  }
  return 0;
}

extern "C" size_t mgb_level_workspace(char tag, int B, int L) {
  switch (tag) {
    case 'g':
    case 's': return mgb_simple_workspace(tag, B, L);
    case 'e':
    case 'r':
    case 'd': return mgb_conv_workspace(tag, B, L);
    case 'c':
    case 'n': return mgb_dyn_workspace(tag, B, L);
    default: return 0;
  }
}

static int check_level(const MgbLevel* lv) {
  if (!lv || lv->B <= 0 || lv->L <= 0 || !lv->u_rows || !lv->bank || !lv->prow || !lv->y) return 1;
  if (lv->ws_bytes < mgb_level_workspace(lv->tag, lv->B, lv->L)) return 1;
  return 0;
}

extern "C" int mgb_level_forward_phase(const MgbLevel* lv, int phase, void* stream) {
  if (int rc = check_level(lv)) return rc;
  if (phase < 1 || phase > 3) return 1;
  cudaStream_t st = (cudaStream_t)stream;
  switch (lv->tag) {
    case 'g':
    case 's': return phase == 2 ? mgb_simple_forward(lv, st) : 0;
    case 'e':
    case 'r':
    case 'd': return phase == 1 ? mgb_conv_prepare(lv, st) : (phase == 2 ? mgb_conv_forward(lv, st) : mgb_conv_norms(lv, st));
    case 'c':
    case 'n': return phase == 1 ? mgb_dyn_prepare(lv, st) : (phase == 2 ? mgb_dyn_forward(lv, st) : 0);
    default: return 1;
  }
}

extern "C" int mgb_level_backward_phase(const MgbLevel* lv, int phase, void* stream) {
  if (int rc = check_level(lv)) return rc;
  if (!lv->gy_rows || !lv->gbank) return 1;  // gu == NULL: the input gradient is not requested
  if (phase != 1 && phase != 2) return 1;
  cudaStream_t st = (cudaStream_t)stream;
  switch (lv->tag) {
    case 'g':
    case 's': return phase == 1 ? mgb_simple_backward(lv, st) : mgb_simple_param_grad(lv, st);
    case 'e':
    case 'r':
    case 'd': return phase == 1 ? mgb_conv_backward(lv, st) : mgb_conv_param_grad(lv, st);
    case 'c':
    case 'n': return phase == 1 ? mgb_dyn_backward(lv, st) : mgb_dyn_param_grad(lv, st);
    default: return 1;
  }
}

extern "C" int mgb_level_forward(const MgbLevel* lv, void* stream) {
  for (int ph = 1; ph <= 3; ++ph)
    if (int rc = mgb_level_forward_phase(lv, ph, stream)) return rc;
  return 0;
}

extern "C" int mgb_level_backward(const MgbLevel* lv, void* stream) {
  if (int rc = mgb_level_backward_phase(lv, 1, stream)) return rc;
  return mgb_level_backward_phase(lv, 2, stream);
}

static std::atomic<long long> g_mgb_launches{0};
void mgb_count_launch() { g_mgb_launches.fetch_add(1, std::memory_order_relaxed); }
extern "C" long long mgb_launch_count(void) { return g_mgb_launches.load(std::memory_order_relaxed); }

extern "C" void* mgb_stream_create_priority(int level);

__global__ void k_timestamp(unsigned long long* dst) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *dst = t;
}

extern "C" int mgb_timestamp(unsigned long long* dst, void* stream) {
  k_timestamp<<<1, 1, 0, (cudaStream_t)stream>>>(dst);
  return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

extern "C" int mgb_zero(void* ptr, size_t bytes, void* stream) {
  if (!bytes) return 0;
  return cudaMemsetAsync(ptr, 0, bytes, (cudaStream_t)stream) == cudaSuccess ? 0 : 2;
}

extern "C" void* mgb_stream_create(void) { return mgb_stream_create_priority(0); }

// level > 0: the device's greatest priority (the critical path of a step: its
// kernels' CTAs are scheduled first when side-stream work competes for SMs);
// level < 0: the least; 0: default.  Captured kernels keep their stream's priority.
extern "C" void* mgb_stream_create_priority(int level) {
  int least = 0, greatest = 0;
  if (cudaDeviceGetStreamPriorityRange(&least, &greatest) != cudaSuccess) return nullptr;
  const int prio = level > 0 ? greatest : (level < 0 ? least : 0);
  cudaStream_t s = nullptr;
  if (cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, prio) != cudaSuccess) return nullptr;
  return (void*)s;
}

extern "C" int mgb_stream_destroy(void* stream) {
  return cudaStreamDestroy((cudaStream_t)stream) == cudaSuccess ? 0 : 2;
}

extern "C" int mgb_fft(const void* in, void* out, void* tmp, int batch, int log2n, int inverse, float scale,
                       void* stream) {
  if (batch <= 0) return 0;
  if (log2n > 13 && !tmp) return 1;
  return mgb_fft_c2c((const float2*)in, (float2*)out, (float2*)tmp, batch, log2n, inverse, scale,
                     (cudaStream_t)stream);
}

extern "C" int mgb_abi_version(void) { return MGB_ABI_VERSION; }
