// tcgen05.mma throughput probe: back-to-back MMAs on one CTA, cycles per MMA
// for SS / TS tf32 at N = 64 / 128 / 256 (M = 128, K = 8 per instruction).
#include <cstdio>
#include <cstdint>
#include "../../paper_2409_14939_b200/csrc/tcgen05.cuh"
using namespace fgl::tc;

__global__ void __launch_bounds__(128, 1) probe(int N, int ts, int iters, long long* out) {
  extern __shared__ __align__(1024) char sm[];
  __shared__ uint64_t mbar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += 128) reinterpret_cast<float*>(sm)[i] = 0.f;
  if (warp == 0) tmem_alloc(&tslot, 512);
  if (threadIdx.x == 0) { mbar_init_n(smem_u32(&mbar), 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  fence_async_smem();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tm = tslot;
  if (warp == 0) {
    const uint32_t idesc = idesc_tf32(128, N, 0, 0);
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 32768);
    long long t0 = clock64();
    if (elect_one()) {
      for (int i = 0; i < iters; ++i) {
        const uint32_t o = (i & 3) * 32;
        if (ts) mma_tf32_ts(tm, tm + 256 + 8 * (i & 3), umma_desc_sw128(b + o), idesc, 1);
        else mma_tf32(tm, umma_desc_sw128(a + o), umma_desc_sw128(b + o), idesc, 1);
      }
      mma_commit(smem_u32(&mbar));
    }
    __syncwarp();
    mbar_wait(smem_u32(&mbar), 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) *out = t1 - t0;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_free(tm, 512); }
}

int main() {
  long long* d; cudaMalloc(&d, 8); long long h;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int ts = 0; ts < 2; ++ts) for (int N : {64, 128, 256}) {
    if (ts && N > 256) continue;
    for (int rep = 0; rep < 2; ++rep) {
      probe<<<1, 128, 64 * 1024>>>(N, ts, 1024, d);
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    }
    printf("%s tf32 M128 N%3d: %.1f cyc/mma (floor 128*N/256 = %d)\n", ts ? "TS" : "SS", N, h / 1024.0, 128 * N / 256);
  }
  // all SMs at once
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
