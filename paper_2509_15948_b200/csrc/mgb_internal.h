// Internal launcher declarations shared between the .cu files of libmixgraph_b200.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "../../include/mixgraph_b200.h"

int mgb_init_device(cudaStream_t st);
int mgb_fft_c2c(const float2* in, float2* out, float2* tmp, int batch, int log2n, int inverse, float scale,
                cudaStream_t st);
int mgb_pack_rows(const float* const* rows, float2* Z, int B, int L, long long N, cudaStream_t st);
int mgb_spec_pair(const float2* Z, const float2* H, float2* Q, const float2* C, float2* Q2, int B, long long N,
                  int mode, cudaStream_t st);

// level implementations (levels.cu / conv.cu / dynamics.cu)
int mgb_simple_forward(const MgbLevel* lv, cudaStream_t st);
int mgb_simple_backward(const MgbLevel* lv, cudaStream_t st);
int mgb_simple_param_grad(const MgbLevel* lv, cudaStream_t st);
size_t mgb_simple_workspace(char tag, int B, int L);
int mgb_conv_prepare(const MgbLevel* lv, cudaStream_t st);
int mgb_conv_norms(const MgbLevel* lv, cudaStream_t st);
int mgb_conv_forward(const MgbLevel* lv, cudaStream_t st);
int mgb_conv_backward(const MgbLevel* lv, cudaStream_t st);
int mgb_conv_param_grad(const MgbLevel* lv, cudaStream_t st);
size_t mgb_conv_workspace(char tag, int B, int L);
int mgb_conv_init();
int mgb_loss_init();
int mgb_dyn_init();
int mgb_dyn_prepare(const MgbLevel* lv, cudaStream_t st);
int mgb_dyn_forward(const MgbLevel* lv, cudaStream_t st);
int mgb_dyn_backward(const MgbLevel* lv, cudaStream_t st);
int mgb_dyn_param_grad(const MgbLevel* lv, cudaStream_t st);
size_t mgb_dyn_workspace(char tag, int B, int L);

// host-side launch counter (mgb_launch_count); every launch site bumps it.  Song
// searches issue from several host threads at once, so the counter is atomic.
void mgb_count_launch();

static inline int mgb_log2_ceil(long long n) {
  int l = 0;
  while ((1LL << l) < n) ++l;
  return l;
}

static inline size_t mgb_align(size_t x) { return (x + 255) & ~(size_t)255; }

// bump allocator over a caller-provided workspace
struct MgbArena {
  char* base;
  size_t off;
  template <typename T>
  T* take(size_t count) {
    T* p = reinterpret_cast<T*>(base ? base + off : nullptr);
    off += mgb_align(count * sizeof(T));
    return p;
  }
};
