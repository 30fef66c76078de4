// Streaming-read probe: 1-D bulk copies (TMA engine) vs plain 16-byte loads,
// one CTA per SM, to size the producer of the dense kernels.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(128, 1) bulk_kernel(const char* src, int64_t bytes, int chunk, int depth, int* sink) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) uint64_t bars[16];
  const int64_t nchunks = bytes / chunk;
  if (threadIdx.x == 0) {
    for (int i = 0; i < depth; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(bars + i)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  int j = 0;
  int acc = 0;
  for (int64_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++j) {
    const int s = j % depth;
    if (j >= depth) {  // wait for the copy issued depth iterations ago
      uint32_t ph = ((j / depth) - 1) & 1, done = 0;
      while (!done) asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(done) : "r"(su(bars + s)), "r"(ph) : "memory");
      acc += sm[s * chunk];
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(bars + s)), "r"(chunk) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(sm + s * chunk)), "l"(src + c * chunk), "r"(chunk), "r"(su(bars + s)) : "memory");
  }
  for (int k = 0; k < depth && k < j; ++k) {
    const int jj = j - 1 - k; const int s = jj % depth; uint32_t ph = (jj / depth) & 1, done = 0;
    while (!done) asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(done) : "r"(su(bars + s)), "r"(ph) : "memory");
  }
  if (acc == 12345) *sink = acc;
}

__global__ void __launch_bounds__(384, 1) ldg_kernel(const float4* src, int64_t n4, int* sink) {
  float acc = 0.f;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n4; i += 8 * stride) {
    float4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldg(src + i + u * stride);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  if (acc == 1.2345f) *sink = 1;
}

int main() {
  const int64_t bytes = 1ll << 30;
  char* src; int* sink;
  cudaMalloc(&src, bytes); cudaMemset(src, 1, bytes); cudaMalloc(&sink, 4);
  cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int chunks[] = {4096, 8192, 16384, 32768, 51200};
  for (int chunk : chunks) for (int depth : {2, 4, 8, 12}) {
    if ((int64_t)chunk * depth > 200 * 1024) continue;
    for (int it = 0; it < 2; ++it) {
      cudaEventRecord(a);
      bulk_kernel<<<148, 128, chunk * depth>>>(src, bytes, chunk, depth, sink);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (it) printf("bulk chunk=%6d depth=%2d in_flight=%7d B/SM: %.0f GB/s\n", chunk, depth, chunk * depth, bytes / ms / 1e6);
    }
  }
  for (int it = 0; it < 2; ++it) {
    cudaEventRecord(a);
    ldg_kernel<<<148, 384>>>((const float4*)src, bytes / 16, sink);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (it) printf("ldg 148x384 x8 float4: %.0f GB/s\n", bytes / ms / 1e6);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
