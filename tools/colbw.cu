// Microbenchmark: DRAM bandwidth of the four-step column-pass access pattern.
// B nodes x (N1 = 512 rows x N2 = 1024 columns) float2; a CTA reads TC adjacent
// columns of all 512 rows (row segments of TC*8 bytes, 8 KB apart) and writes them
// back in the same pattern; compared with a contiguous copy.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o colbw tools/colbw.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N1 = 512, N2 = 1024;

template <int TC>
__global__ void __launch_bounds__(256) k_col(const float2* __restrict__ in, float2* __restrict__ out) {
  constexpr int P = 256 / TC;          // threads per column
  constexpr int Q = N1 / P;            // values per thread
  const int c = threadIdx.x % TC, j = threadIdx.x / TC;
  const int b = blockIdx.y, col = blockIdx.x * TC + c;
  const float2* src = in + (size_t)b * N1 * N2 + col;
  float2 v[Q];
#pragma unroll
  for (int m = 0; m < Q; ++m) v[m] = src[(size_t)(j + P * m) * N2];
  float2* dst = out + (size_t)b * N1 * N2 + col;
#pragma unroll
  for (int m = 0; m < Q; ++m) dst[(size_t)(j + P * m) * N2] = make_float2(v[m].x * 1.0001f, v[m].y);
}

// TMA-free bulk staging: one CTA copies a 512 x TC tile through shared memory with
// cp.async.bulk row segments (TC*8 bytes each), then stores it back coalesced
template <int TC>
__global__ void __launch_bounds__(256) k_col_bulk(const float2* __restrict__ in, float2* __restrict__ out) {
  extern __shared__ __align__(128) float2 tile[];  // N1 x TC
  __shared__ __align__(8) unsigned long long bar;
  const int b = blockIdx.y, col0 = blockIdx.x * TC;
  const unsigned sb = (unsigned)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sb));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  constexpr unsigned BYTES = N1 * TC * 8;
  if (threadIdx.x == 0)
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sb), "r"(BYTES));
  __syncthreads();
  const float2* src = in + (size_t)b * N1 * N2 + col0;
  for (int r = threadIdx.x; r < N1; r += blockDim.x) {
    const unsigned sd = (unsigned)__cvta_generic_to_shared(tile + r * TC);
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sd),
                 "l"(src + (size_t)r * N2), "r"(TC * 8), "r"(sb)
                 : "memory");
  }
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra WAIT_%=;\n}\n" ::"r"(sb)
      : "memory");
  float2* dst = out + (size_t)b * N1 * N2 + col0;
  for (int i = threadIdx.x; i < N1 * TC; i += blockDim.x) {
    const int r = i / TC, c = i % TC;
    const float2 v = tile[i];
    dst[(size_t)r * N2 + c] = make_float2(v.x * 1.0001f, v.y);
  }
}

__global__ void k_copy(const float4* __restrict__ in, float4* __restrict__ out, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    out[i] = in[i];
}

template <class F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaEventRecord(a);
  for (int i = 0; i < 10; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / 10;
}

int main() {
  const int B = 16;
  const size_t n = (size_t)B * N1 * N2;
  float2 *x, *y;
  cudaMalloc(&x, n * 8);
  cudaMalloc(&y, n * 8);
  cudaMemset(x, 0, n * 8);
  const double bytes = 2.0 * n * 8;
  float ms = timeit([&] { k_copy<<<148 * 8, 256>>>((float4*)x, (float4*)y, n / 2); });
  printf("contiguous copy          %7.1f us  %6.0f GB/s\n", ms * 1e3, bytes / ms / 1e6);
  ms = timeit([&] { k_col<16><<<dim3(N2 / 16, B), 256>>>(x, y); });
  printf("column tiles TC=16       %7.1f us  %6.0f GB/s\n", ms * 1e3, bytes / ms / 1e6);
  ms = timeit([&] { k_col<32><<<dim3(N2 / 32, B), 256>>>(x, y); });
  printf("column tiles TC=32       %7.1f us  %6.0f GB/s\n", ms * 1e3, bytes / ms / 1e6);
  ms = timeit([&] { k_col<64><<<dim3(N2 / 64, B), 256>>>(x, y); });
  printf("column tiles TC=64       %7.1f us  %6.0f GB/s\n", ms * 1e3, bytes / ms / 1e6);
  cudaFuncSetAttribute(k_col_bulk<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, N1 * 16 * 8);
  cudaFuncSetAttribute(k_col_bulk<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, N1 * 32 * 8);
  cudaFuncSetAttribute(k_col_bulk<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, N1 * 64 * 8);
  ms = timeit([&] { k_col_bulk<16><<<dim3(N2 / 16, B), 256, N1 * 16 * 8>>>(x, y); });
  printf("bulk-copy tiles TC=16    %7.1f us  %6.0f GB/s\n", ms * 1e3, bytes / ms / 1e6);
  ms = timeit([&] { k_col_bulk<32><<<dim3(N2 / 32, B), 256, N1 * 32 * 8>>>(x, y); });
  printf("bulk-copy tiles TC=32    %7.1f us  %6.0f GB/s\n", ms * 1e3, bytes / ms / 1e6);
  ms = timeit([&] { k_col_bulk<64><<<dim3(N2 / 64, B), 256, N1 * 64 * 8>>>(x, y); });
  printf("bulk-copy tiles TC=64    %7.1f us  %6.0f GB/s\n", ms * 1e3, bytes / ms / 1e6);
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
