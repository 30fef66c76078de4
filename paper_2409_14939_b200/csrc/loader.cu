// Match-Reorder feature loader (sm_100a).
//
//  * fgl_match_counts -- |U_i ∩ U_j| for every pair of batches of a sampled
//    window from their node bitmaps (AND + popcount, one pass over the
//    window's bitmaps).  The host turns the counts into the match-degree
//    matrix M_ij = |U_i ∩ U_j| / min(|U_i|, |U_j|) of schedule.py:68-89 and
//    runs the greedy chain of schedule.py:92-113 on it.
//  * fgl_gather_rows  -- builds a batch's input feature block x0 (rows in
//    local-ID order, trainer.py:315).  With a previous batch resident in HBM
//    (Match), rows the previous batch already holds are copied device-to-
//    device from its block and only the delta rows are read from the feature
//    store, which may be pinned host memory (zero-copy over the host link) or
//    HBM.  Rows are moved with 16-byte vector loads, one warp per row.  The
//    count of rows read from the store is accumulated for the IO accounting
//    of memsim.simulate_epoch_io (memsim.py:129-186).
#include <algorithm>

#include "common.cuh"

namespace fgl {
namespace {

constexpr int kMaxMatchBatches = 16;

template <int NB>
__global__ void match_counts_kernel(const uint32_t* __restrict__ bm, int64_t words, int nb,
                                    unsigned long long* __restrict__ out) {
  constexpr int NP = NB * (NB - 1) / 2;
  uint32_t cnt[NP];
#pragma unroll
  for (int p = 0; p < NP; ++p) cnt[p] = 0;
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < words;
       w += (int64_t)gridDim.x * blockDim.x) {
    uint32_t v[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i) v[i] = i < nb ? __ldg(bm + i * words + w) : 0u;
    int p = 0;
#pragma unroll
    for (int i = 0; i < NB; ++i)
#pragma unroll
      for (int j = i + 1; j < NB; ++j) cnt[p++] += __popc(v[i] & v[j]);
  }
  __shared__ unsigned long long sm[NP];
  for (int p = threadIdx.x; p < NP; p += blockDim.x) sm[p] = 0;
  __syncthreads();
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    const uint32_t s = warp_sum(cnt[p]);
    if ((threadIdx.x & 31) == 0 && s) atomicAdd(sm + p, (unsigned long long)s);
  }
  __syncthreads();
  for (int p = threadIdx.x; p < NP; p += blockDim.x)
    if (sm[p]) atomicAdd(out + p, sm[p]);
}

__device__ __forceinline__ bool bm_test(const uint32_t* bm, int32_t g) {
  return (__ldg(bm + (g >> 5)) >> (g & 31)) & 1u;
}

// one warp per output row; 16-byte vectors when every row is 16-byte aligned
template <bool VEC>
__global__ void gather_rows_kernel(const float* __restrict__ feats, int64_t ldf, int d,
                                   const int32_t* __restrict__ ids, int64_t n,
                                   const uint32_t* __restrict__ prev_bm,
                                   const int32_t* __restrict__ prev_prefix, int64_t prev_base,
                                   const float* __restrict__ prev_x, int64_t ldp,
                                   float* __restrict__ out, int64_t ldo,
                                   unsigned long long* __restrict__ loaded) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  uint32_t my_loaded = 0;
  for (int64_t r = warp; r < n; r += nwarps) {
    const int32_t g = ids[r];
    const float* src;
    if (prev_bm && bm_test(prev_bm, g)) {
      const int64_t wi = g >> 5;
      const int64_t pr = prev_prefix[wi] + __popc(prev_bm[wi] & ((1u << (g & 31)) - 1u)) - prev_base;
      src = prev_x + pr * ldp;
    } else {
      src = feats + (int64_t)g * ldf;
      ++my_loaded;
    }
    float* dst = out + r * ldo;
    if (VEC) {
      const float4* s4 = reinterpret_cast<const float4*>(src);
      float4* d4 = reinterpret_cast<float4*>(dst);
      for (int c = lane; c < (d >> 2); c += 32) d4[c] = s4[c];
      for (int c = (d & ~3) + lane; c < d; c += 32) dst[c] = src[c];
    } else {
      for (int c = lane; c < d; c += 32) dst[c] = src[c];
    }
  }
  if (loaded && lane == 0 && my_loaded) atomicAdd(loaded, (unsigned long long)my_loaded);
}

}  // namespace
}  // namespace fgl

using namespace fgl;

extern "C" {

int fgl_match_counts(const uint32_t* bitmaps, int64_t words, int32_t nb, uint64_t* out_pairs,
                     void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (!bitmaps || !out_pairs || words < 1 || nb < 2 || nb > kMaxMatchBatches) {
    set_error("fgl_match_counts: bad arguments (2 <= nb <= %d)", kMaxMatchBatches);
    return FGL_E_INVALID;
  }
  constexpr int NP = kMaxMatchBatches * (kMaxMatchBatches - 1) / 2;
  FGL_CUDA(cudaMemsetAsync(out_pairs, 0, 8 * (size_t)NP, st));
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(words, 256), 2 * kNumSMs));
  auto* o = reinterpret_cast<unsigned long long*>(out_pairs);
  // pair (i < j) lands at i*16 - i*(i+1)/2 + (j-i-1) of a 16 x 16 triangle
  FGL_COUNT_LAUNCH(), match_counts_kernel<kMaxMatchBatches><<<grid, 256, 0, st>>>(bitmaps, words, nb, o);
  FGL_LAUNCH_CHECK("match_counts_kernel");
  return FGL_OK;
}

int fgl_gather_rows(const float* feats, int64_t ldf, int32_t d, const int32_t* ids, int64_t n,
                    const uint32_t* prev_bitmap, const int32_t* prev_prefix, int64_t prev_base,
                    const float* prev_x, int64_t ldp, float* out, int64_t ldo, uint64_t* loaded,
                    void* stream) {
  if (n < 0 || d < 1 || ldf < d || ldo < d || !feats || !out || (n > 0 && !ids) ||
      (prev_bitmap && (!prev_prefix || !prev_x || ldp < d))) {
    set_error("fgl_gather_rows: bad arguments");
    return FGL_E_INVALID;
  }
  if (n == 0) return FGL_OK;
  const bool vec = ((ldf | ldo | (prev_bitmap ? ldp : 0)) % 4 == 0) &&
                   !((reinterpret_cast<uintptr_t>(feats) | reinterpret_cast<uintptr_t>(out) |
                      reinterpret_cast<uintptr_t>(prev_x)) & 15);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 8), 148 * 16));
  auto* ld = reinterpret_cast<unsigned long long*>(loaded);
  if (vec)
    FGL_COUNT_LAUNCH(), gather_rows_kernel<true><<<grid, 256, 0, (cudaStream_t)stream>>>(
        feats, ldf, d, ids, n, prev_bitmap, prev_prefix, prev_base, prev_x, ldp, out, ldo, ld);
  else
    FGL_COUNT_LAUNCH(), gather_rows_kernel<false><<<grid, 256, 0, (cudaStream_t)stream>>>(
        feats, ldf, d, ids, n, prev_bitmap, prev_prefix, prev_base, prev_x, ldp, out, ldo, ld);
  FGL_LAUNCH_CHECK("gather_rows_kernel");
  return FGL_OK;
}

}  // extern "C"
