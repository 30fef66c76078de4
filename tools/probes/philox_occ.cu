// Philox4x64-10 throughput vs resident warps per SM and blocks in flight per
// thread (ILP), with and without a per-lane key schedule (vector vs table round
// keys).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2409_14939_b200/csrc philox_occ.cu
#include <cstdio>

#include "common.cuh"

using namespace fgl;

template <int ILP, int MODE>  // MODE 0: per-lane keys (vector adds); 1: round keys from shared memory
__global__ void probe(uint64_t k0, uint64_t k1, int iters, uint64_t* out) {
  __shared__ ulonglong2 rk[10];
  if (threadIdx.x < 10) rk[threadIdx.x] = make_ulonglong2(k0 + threadIdx.x * kPhiloxW0, k1 + threadIdx.x * kPhiloxW1);
  __syncthreads();
  uint64_t acc = 0;
  uint64_t lk0 = k0 ^ threadIdx.x, lk1 = k1;  // per-lane key: defeats the uniform datapath
  const uint64_t base = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * (uint64_t)iters * ILP;
  for (int i = 0; i < iters; ++i) {
    uint64_t w[ILP][4];
#pragma unroll
    for (int j = 0; j < ILP; ++j) {
      if (MODE == 0) philox4x64_10(base + i * ILP + j + 1, lk0, lk1, w[j][0], w[j][1], w[j][2], w[j][3]);
      else philox4x64_10_rk(base + i * ILP + j + 1, rk, w[j]);
    }
#pragma unroll
    for (int j = 0; j < ILP; ++j) acc ^= w[j][0] ^ w[j][1] ^ w[j][2] ^ w[j][3];
  }
  if (acc == 0x1234567ull) out[0] = acc;
}

template <int ILP, int MODE>
void run(int warps_per_sm, uint64_t* out) {
  const int threads = 128, ctas = 148 * warps_per_sm / 4;
  const int iters = 256 / ILP;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  probe<ILP, MODE><<<ctas, threads>>>(1, 2, iters, out);
  cudaEventRecord(a);
  probe<ILP, MODE><<<ctas, threads>>>(1, 2, iters, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double draws = 4.0 * ILP * iters * (double)ctas * threads;
  printf("ILP %d keys %s warps/SM %2d: %6.1f G draws/s\n", ILP, MODE ? "table " : "vector", warps_per_sm,
         draws / (ms * 1e-3) / 1e9);
}

int main() {
  uint64_t* out;
  cudaMalloc(&out, 8);
  for (int w : {8, 12, 16, 20, 24, 32, 48, 64}) {
    run<1, 0>(w, out);
    run<2, 0>(w, out);
    run<1, 1>(w, out);
    run<2, 1>(w, out);
  }
  return 0;
}
