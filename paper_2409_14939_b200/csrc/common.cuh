// Shared device utilities for the FastGL B200 hot path (sm_100a).
//
// Everything here is plain CUDA C++ compiled with
//   nvcc -gencode arch=compute_100a,code=sm_100a --fmad=false
// --fmad=false is load-bearing: the reference aggregation accumulates
// `acc = acc + w*x` with a rounded multiply and a rounded add
// (compute.py:115-148); contracting that into an FMA would change bits.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/fastgl_b200.h"

namespace fgl {

constexpr int kWarp = 32;
constexpr int kNumSMs = 148;

// Integer A/B switch from the environment (read by each call site once, into
// a function-local static).
int env_int(const char* name, int dflt);

// ------------------------------------------------------------------ errors --
void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* what);

// Process-wide count of kernels this library has launched (bench.py reports
// it as gpu_launches); every launch site is written FGL_COUNT_LAUNCH(), k<<<...>>>(...).
void count_launch();
#define FGL_COUNT_LAUNCH() ::fgl::count_launch()
// Dense layers that ran on the SIMT kernels because their shape is outside
// the tensor-core envelope (fgl_dense_fallback_count; bench.py requires 0).
void count_dense_fallback();

// ------------------------------------------------------- live kernel timing --
// Measurement hook (fgl_profile, bench.py's per-stage rooflines): while
// enabled, the dominant launches of each stage are bracketed by CUDA events
// on their own stream (event-record nodes when the stream is being captured
// into a graph), tagged with a kernel id and three shape ints.
enum ProfId : int {
  kProfSelect = 1,      // select_bal + select_hub of one hop      (a0 = hop)
  kProfSpmmGather = 2,  // layer-0 block aggregation, spmm_pipe    (a0 = rows, a1 = d)
  kProfSpmm = 3,        // fgl_spmm                                 (a0 = rows, a1 = d)
  kProfDenseFwd = 4,    // tc_gemm3 mode 0                          (a0 = M, a1 = N, a2 = K)
  kProfDgrad = 5,       // tc_gemm3 mode 1                          (a0 = M, a1 = N, a2 = K)
  kProfWgrad = 6,       // tc_wgrad3 (+ its partial reduction)      (a0 = M, a1 = K, a2 = N)
  kProfGather = 7,      // x0 row gather (Match / cache / store)    (a0 = rows, a1 = d)
  kProfTopLayer = 8,    // fused top layer (agg, logits, loss, dH)  (a0 = B, a1 = din, a2 = C)
  kProfSgd = 9,         // SGD step                                 (a0 = params)
};
struct ProfMark {
  cudaEvent_t e0 = nullptr;
  cudaStream_t st = nullptr;
  bool captured = false;
};
ProfMark prof_begin(cudaStream_t st);
void prof_end(const ProfMark& m, int id, int64_t a0, int64_t a1 = 0, int64_t a2 = 0);

#define FGL_CUDA(call)                                              \
  do {                                                              \
    cudaError_t _e = (call);                                        \
    if (_e != cudaSuccess) return ::fgl::cuda_status(_e, #call);    \
  } while (0)

#define FGL_LAUNCH_CHECK(what)                                      \
  do {                                                              \
    cudaError_t _e = cudaGetLastError();                            \
    if (_e != cudaSuccess) return ::fgl::cuda_status(_e, what);     \
  } while (0)

// ------------------------------------------------------------------ philox --
// Random123 Philox4x64-10 as used by numpy's np.random.Philox.  Draw j of a
// generator with key (k0,k1) is word (j & 3) of philox(counter=(j>>2)+1, 0, 0, 0);
// Generator.random() keeps the top 53 bits (word >> 11).  See oracle/philox.py.
constexpr uint64_t kPhiloxM0 = 0xD2E7470EE14C6C93ull;
constexpr uint64_t kPhiloxM1 = 0xCA5A826395121157ull;
constexpr uint64_t kPhiloxW0 = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kPhiloxW1 = 0xBB67AE8584CAA73Bull;

__device__ __forceinline__ void philox4x64_10(uint64_t ctr, uint64_t k0, uint64_t k1,
                                              uint64_t& o0, uint64_t& o1, uint64_t& o2,
                                              uint64_t& o3) {
  uint64_t c0 = ctr, c1 = 0, c2 = 0, c3 = 0;
  // keep the 20 round keys from being hoisted out of callers' loops (they
  // would pin 40 registers); the per-round key add is 2 integer ops
  asm volatile("" : "+l"(k0), "+l"(k1));
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t hi0 = __umul64hi(kPhiloxM0, c0);
    const uint64_t lo0 = kPhiloxM0 * c0;
    const uint64_t hi1 = __umul64hi(kPhiloxM1, c2);
    const uint64_t lo1 = kPhiloxM1 * c2;
    c0 = hi1 ^ c1 ^ k0;
    c1 = lo1;
    c2 = hi0 ^ c3 ^ k1;
    c3 = lo0;
    k0 += kPhiloxW0;
    k1 += kPhiloxW1;
  }
  o0 = c0; o1 = c1; o2 = c2; o3 = c3;
}

// two independent Philox4x64-10 blocks, rounds interleaved (4 multiply chains)
__device__ __forceinline__ void philox4x64_10_x2(uint64_t ctrA, uint64_t kA0, uint64_t kA1, uint64_t ctrB,
                                                 uint64_t kB0, uint64_t kB1, uint64_t (&oA)[4],
                                                 uint64_t (&oB)[4]) {
  uint64_t a0 = ctrA, a1 = 0, a2 = 0, a3 = 0;
  uint64_t b0 = ctrB, b1 = 0, b2 = 0, b3 = 0;
  asm volatile("" : "+l"(kA0), "+l"(kA1), "+l"(kB0), "+l"(kB1));
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t ahi0 = __umul64hi(kPhiloxM0, a0), alo0 = kPhiloxM0 * a0;
    const uint64_t ahi1 = __umul64hi(kPhiloxM1, a2), alo1 = kPhiloxM1 * a2;
    const uint64_t bhi0 = __umul64hi(kPhiloxM0, b0), blo0 = kPhiloxM0 * b0;
    const uint64_t bhi1 = __umul64hi(kPhiloxM1, b2), blo1 = kPhiloxM1 * b2;
    a0 = ahi1 ^ a1 ^ kA0; a1 = alo1; a2 = ahi0 ^ a3 ^ kA1; a3 = alo0;
    b0 = bhi1 ^ b1 ^ kB0; b1 = blo1; b2 = bhi0 ^ b3 ^ kB1; b3 = blo0;
    kA0 += kPhiloxW0; kA1 += kPhiloxW1;
    kB0 += kPhiloxW0; kB1 += kPhiloxW1;
  }
  oA[0] = a0; oA[1] = a1; oA[2] = a2; oA[3] = a3;
  oB[0] = b0; oB[1] = b1; oB[2] = b2; oB[3] = b3;
}

// --------------------------------------------------------------- warp/block --
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ int warp_id() { return threadIdx.x >> 5; }

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane_id() >= o) v += n;
  }
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide exclusive scan; returns the exclusive prefix for this thread and
// the block total in *total.  `smem` needs blockDim.x/32 + 1 entries.
template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T* smem, T* total) {
  const int lane = lane_id(), wid = warp_id(), nw = blockDim.x >> 5;
  T inc = warp_incl_scan(v);
  if (lane == 31) smem[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    T s = lane < nw ? smem[lane] : T(0);
    T si = warp_incl_scan(s);
    if (lane < nw) smem[lane] = si - s;
    if (lane == nw - 1) smem[32] = si;
  }
  __syncthreads();
  T res = inc - v + smem[wid];
  *total = smem[32];
  __syncthreads();
  return res;
}

template <typename T>
__device__ __forceinline__ T block_sum(T v, T* smem) {
  const int lane = lane_id(), wid = warp_id(), nw = blockDim.x >> 5;
  v = warp_sum(v);
  if (lane == 0) smem[wid] = v;
  __syncthreads();
  T r = 0;
  if (wid == 0) {
    r = lane < nw ? smem[lane] : T(0);
    r = warp_sum(r);
    if (lane == 0) smem[32] = r;
  }
  __syncthreads();
  r = smem[32];
  __syncthreads();
  return r;
}

__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Fixed grid for device-count-driven ("persistent") kernels: 2 CTAs per SM.
constexpr int kPersistentCTAs = 2 * kNumSMs;

// tcgen05 3xTF32 GEMM (tc_gemm3.cu).  mode 0: C = act(A W + bias), W [K, N];
// mode 1: C = (A * (mask > 0)) W^T, W [N, K].  ldw = W's row stride (default
// the row length: N in mode 0, K in mode 1), so callers can pass column / K
// slices of a wider W; accum adds into C (K slices).  Returns false if the shape is
// outside the kernel's envelope (the caller then runs the SIMT kernel and
// counts it with count_dense_fallback); *err receives an FGL status otherwise.
bool tc_gemm(int mode, const float* A, int64_t lda, const float* mask, int64_t ldm, const float* W,
             const float* bias, float* C, int64_t ldc, int64_t M, int N, int K, int relu,
             cudaStream_t st, int* err);
bool tc_gemm3(int mode, const float* A, int64_t lda, const float* mask, int64_t ldm, const float* W,
              const float* bias, float* C, int64_t ldc, int64_t M, int N, int K, int relu,
              cudaStream_t st, int* err, int accum = 0, int64_t ldw = -1);
// tcgen05 3xTF32 weight gradient partials: part[c][K+1][N] (row K = db).
// nks > 1: the K features in nks slices of kslice in ONE launch (chunks CTAs
// per slice); slice s's partials at part + s * chunks * (kslice + 1) * N,
// each [c][K_s + 1][N] with K_s = min(kslice, K - s kslice).
bool tc_wgrad3(const float* H, int64_t ldh, const float* dZ, int64_t ldz, const float* mask, int64_t ldm,
               int64_t M, int K, int N, float* part, int chunks, cudaStream_t st, int* err, int nks = 1,
               int kslice = 0);

}  // namespace fgl
