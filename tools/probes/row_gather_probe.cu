// Ceiling probe for the layer-0 aggregation: random 400-byte feature rows
// (products table 2.45M x 100 fp32, larger than L2) read by warps with
// 16-byte lanes, R rows in flight per warp, nothing else.  Reports GB/s of
// row bytes read, for R = 1, 2, 4, 8 and rows of 100 / 128 floats.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probes/row_gather_probe tools/probes/row_gather_probe.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

template <int R>
__global__ void __launch_bounds__(256) gather_rows(const float4* __restrict__ X, int ld4, int d4,
                                                   const int* __restrict__ idx, long n, float* out) {
  const int lane = threadIdx.x & 31;
  const long nw = ((long)gridDim.x * blockDim.x) >> 5;
  float acc = 0.f;
  for (long r0 = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r0 * R < n; r0 += nw) {
    float4 v[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const long r = r0 * R + k;
      const int c = r < n ? __ldg(idx + r) : 0;
      v[k] = (lane < d4 && r < n) ? __ldg(X + (long)c * ld4 + lane) : make_float4(0, 0, 0, 0);
    }
#pragma unroll
    for (int k = 0; k < R; ++k) acc += v[k].x + v[k].y + v[k].z + v[k].w;
  }
  if (acc == 1234.5f) out[0] = acc;
}

int main() {
  const long N = 2450000;
  const long n = 2000000;
  for (int d : {100, 128}) {
    const int ld4 = (d + 3) / 4, d4 = ld4;
    float4* X;
    int* idx;
    float* out;
    cudaMalloc(&X, N * ld4 * 16);
    cudaMemset(X, 0, N * ld4 * 16);
    cudaMalloc(&idx, n * 4);
    cudaMalloc(&out, 4);
    std::vector<int> h(n);
    srand(1);
    for (long i = 0; i < n; ++i) h[i] = (int)(((long)rand() * 7919L + rand()) % N);
    cudaMemcpy(idx, h.data(), n * 4, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int R : {1, 2, 4, 8}) {
      for (int blocksPerSm : {4, 8}) {
        const int grid = 148 * blocksPerSm;
        float best = 1e9;
        for (int rep = 0; rep < 5; ++rep) {
          cudaEventRecord(e0);
          if (R == 1) gather_rows<1><<<grid, 256>>>(X, ld4, d4, idx, n, out);
          if (R == 2) gather_rows<2><<<grid, 256>>>(X, ld4, d4, idx, n, out);
          if (R == 4) gather_rows<4><<<grid, 256>>>(X, ld4, d4, idx, n, out);
          if (R == 8) gather_rows<8><<<grid, 256>>>(X, ld4, d4, idx, n, out);
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          float ms;
          cudaEventElapsedTime(&ms, e0, e1);
          if (ms < best) best = ms;
        }
        printf("d=%d R=%d ctas/sm=%d: %.1f us, %.0f GB/s of rows\n", d, R, blocksPerSm, best * 1e3,
               n * (double)d * 4 / (best * 1e-3) / 1e9);
      }
    }
    cudaFree(X);
    cudaFree(idx);
    cudaFree(out);
  }
  return 0;
}
