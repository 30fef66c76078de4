// Host cost of cudaLaunchKernel on this box: n launches of an empty kernel,
// plus the same n kernels replayed from a captured CUDA graph.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/probes/launch_probe tools/probes/launch_probe.cu
#include <chrono>
#include <cstdio>
__global__ void empty_kernel(float* p) { if (p && threadIdx.x == 0 && blockIdx.x == 1 << 30) p[0] = 1.f; }
int main() {
  cudaStream_t s;
  cudaStreamCreate(&s);
  for (int i = 0; i < 100; ++i) empty_kernel<<<1, 32, 0, s>>>(nullptr);
  cudaStreamSynchronize(s);
  for (int rep = 0; rep < 3; ++rep) {
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < 1000; ++i) empty_kernel<<<148, 256, 0, s>>>(nullptr);
    auto t1 = std::chrono::steady_clock::now();
    cudaStreamSynchronize(s);
    auto t2 = std::chrono::steady_clock::now();
    printf("1000 launches: issue %.2f us/launch, total %.2f us/kernel\n",
           std::chrono::duration<double, std::micro>(t1 - t0).count() / 1000,
           std::chrono::duration<double, std::micro>(t2 - t0).count() / 1000);
  }
  cudaGraph_t g;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < 100; ++i) empty_kernel<<<148, 256, 0, s>>>(nullptr);
  cudaStreamEndCapture(s, &g);
  cudaGraphExec_t ge;
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < 10; ++i) cudaGraphLaunch(ge, s);
  auto t1 = std::chrono::steady_clock::now();
  cudaStreamSynchronize(s);
  auto t2 = std::chrono::steady_clock::now();
  printf("graph of 100 kernels x10: issue %.2f us/kernel, total %.2f us/kernel\n",
         std::chrono::duration<double, std::micro>(t1 - t0).count() / 1000,
         std::chrono::duration<double, std::micro>(t2 - t0).count() / 1000);
  return 0;
}
