// TMA tile::gather4 semantics probe: 2-D fp32 tensor [rows][100], gather 4
// rows by index into shared memory; try box {100,1} and report the smem image.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../../paper_2409_14939_b200/csrc/tcgen05.cuh"
using namespace fgl::tc;

__global__ void g4(const __grid_constant__ CUtensorMap m, int r0, int r1, int r2, int r3, float* out, int nfl) {
  extern __shared__ __align__(128) float sm[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) { mbar_init_n(smem_u32(&bar), 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(smem_u32(&bar), nfl * 4);
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                 :: "r"(smem_u32(sm)), "l"(reinterpret_cast<uint64_t>(&m)), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(&bar)) : "memory");
  }
  mbar_wait(smem_u32(&bar), 0);
  for (int i = threadIdx.x; i < nfl; i += blockDim.x) out[i] = sm[i];
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  const int R = 1000, C = 100;
  float* h = new float[R * C];
  for (int i = 0; i < R * C; ++i) h[i] = (float)i;
  float *d, *o;
  cudaMalloc(&d, R * C * 4); cudaMalloc(&o, 4 * 128 * 4);
  cudaMemcpy(d, h, R * C * 4, cudaMemcpyHostToDevice);
  void* f; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  Enc enc = (Enc)f;
  for (int by : {1, 4}) for (int bx : {100, 64, 32}) {
    CUtensorMap m;
    cuuint64_t dims[2] = {C, R}; cuuint64_t str[1] = {C * 4};
    cuuint32_t box[2] = {(cuuint32_t)bx, (cuuint32_t)by}; cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("box {%d,%d}: encode failed %d\n", bx, by, (int)r); continue; }
    const int nfl = 4 * bx;
    cudaMemset(o, 0, 4 * 128 * 4);
    g4<<<1, 128, 4 * 128 * 4>>>(m, 7, 123, 5, 999, o, nfl);
    cudaError_t e = cudaDeviceSynchronize();
    float hb[512];
    cudaMemcpy(hb, o, nfl * 4, cudaMemcpyDeviceToHost);
    printf("box {%d,%d}: %s  first of each row slot: %.0f %.0f %.0f %.0f  (expect %d %d %d %d)\n", bx, by,
           cudaGetErrorString(e), hb[0], hb[bx], hb[2 * bx], hb[3 * bx], 7 * C, 123 * C, 5 * C, 999 * C);
    if (e != cudaSuccess) { cudaGetLastError(); break; }
  }
}
