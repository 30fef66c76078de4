// Layout probe: what a CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B TMA load writes to
// shared memory (value = row * 1000 + col), to derive the physical -> logical
// map the tc_wgrad5 split pass needs.  nvcc -arch=sm_100a tma_atom32.cu -lcuda
#include <cuda.h>
#include <cstdio>
#include <vector>
#include "../../paper_2409_14939_b200/csrc/tcgen05.cuh"
using namespace fgl::tc;

__global__ void k(const __grid_constant__ CUtensorMap m, float* out) {
  __shared__ __align__(1024) float s[32 * 32];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init_n(smem_u32(&bar), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(smem_u32(&bar), 32 * 32 * 4);
    tma_load_2d(smem_u32(s), &m, 0, 0, smem_u32(&bar));
  }
  mbar_wait(smem_u32(&bar), 0);
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) out[i] = s[i];
}

int main() {
  const int R = 64, C = 40;
  std::vector<float> h(R * C);
  for (int r = 0; r < R; ++r) for (int c = 0; c < C; ++c) h[r * C + c] = r * 1000 + c;
  float *d, *o;
  cudaMalloc(&d, h.size() * 4); cudaMalloc(&o, 4096);
  cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)R};
  cuuint64_t strides[1] = {(cuuint64_t)C * 4};
  cuuint32_t box[2] = {32, 32};
  cuuint32_t es[2] = {1, 1};
  CUresult rc = cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                                      CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode rc %d\n", (int)rc);
  k<<<1, 128>>>(m, o);
  std::vector<float> out(1024);
  cudaMemcpy(out.data(), o, 4096, cudaMemcpyDeviceToHost);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  // for each physical slot: logical (row, col); check the hypothesis col = (p&7) + 8*(((p>>3) ^ (row&3)))
  int bad = 0;
  for (int pr = 0; pr < 32; ++pr)
    for (int p = 0; p < 32; ++p) {
      const int v = (int)out[pr * 32 + p], lr = v / 1000, lc = v % 1000;
      const int hyp = (p & 7) + 8 * ((p >> 3) ^ (pr & 3));
      if (lr != pr || lc != hyp) ++bad;
    }
  printf("hypothesis row-preserving, granule ^= row&3: %d mismatches\n", bad);
  for (int pr = 0; pr < 6; ++pr) {
    for (int p = 0; p < 32; p += 4) printf("%6d ", (int)out[pr * 32 + p]);
    printf("\n");
  }
  return 0;
}
