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
//  * fgl_gather_rows_cached -- the same with a static HBM feature cache
//    (memsim.py:110-126 static-degree policy made real): a row the previous
//    batch does not hold is read from the cache table when its node has a
//    cache slot, else from the store; cache hits are counted separately
//    (bytes_served_by_cache of simulate_epoch_io).
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

// Row gather: each warp copies R = 4 rows per iteration (lane = 16-byte
// chunk), so every lane keeps 4 independent loads in flight.  The source of a
// row is the previous batch's block when its bitmap holds the ID (Match), else
// the feature store (HBM or mapped pinned host memory).
template <bool VEC>
__global__ void __launch_bounds__(256) gather_rows_kernel(
    const float* __restrict__ feats, int64_t ldf, int d, const int32_t* __restrict__ ids, int64_t n,
    const uint32_t* __restrict__ prev_bm, const int32_t* __restrict__ prev_prefix, int64_t prev_base,
    const float* __restrict__ prev_x, int64_t ldp, const int32_t* __restrict__ prev_row_map,
    const int32_t* __restrict__ cache_slot, const float* __restrict__ cache_x, int64_t ldc,
    float* __restrict__ out, int64_t ldo, unsigned long long* __restrict__ loaded,
    unsigned long long* __restrict__ hits) {
  constexpr int R = 4;
  const int lane = threadIdx.x & 31;
  const int w = VEC ? (d + 3) >> 2 : d;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  uint32_t my_loaded = 0, my_hits = 0;
  for (int64_t r0 = warp * R; r0 < n; r0 += nwarps * R) {
    // lanes 0..R-1 resolve the R rows' sources, then broadcast
    const float* mine = nullptr;
    if (lane < R && r0 + lane < n) {
      const int32_t g = ids[r0 + lane];
      mine = feats + (int64_t)g * ldf;
      bool store = true;
      if (prev_bm) {
        const uint32_t word = __ldg(prev_bm + (g >> 5));
        if ((word >> (g & 31)) & 1u) {
          int64_t pr = __ldg(prev_prefix + (g >> 5)) + __popc(word & ((1u << (g & 31)) - 1u)) - prev_base;
          if (prev_row_map) pr = __ldg(prev_row_map + pr + prev_base) - prev_base;  // depth-major rows
          mine = prev_x + pr * ldp;
          store = false;
        }
      }
      if (store && cache_slot) {  // static HBM cache (memsim.py:110-186): after Match
        const int32_t cs = __ldg(cache_slot + g);
        if (cs >= 0) {
          mine = cache_x + (int64_t)cs * ldc;
          store = false;
          ++my_hits;
        }
      }
      my_loaded += store ? 1u : 0u;
    }
    const float* src[R];
#pragma unroll
    for (int q = 0; q < R; ++q)
      src[q] = reinterpret_cast<const float*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(mine), q));
    for (int c = lane; c < w; c += 32) {
      if (VEC) {
        float4 v[R];
#pragma unroll
        for (int q = 0; q < R; ++q)
          if (r0 + q < n) v[q] = reinterpret_cast<const float4*>(src[q])[c];
#pragma unroll
        for (int q = 0; q < R; ++q) {
          if (r0 + q >= n) continue;
          float* drow = out + (r0 + q) * ldo;
          const int c0 = 4 * c;
          if (c0 + 3 < d) {
            *reinterpret_cast<float4*>(drow + c0) = v[q];
          } else {  // ragged tail when d is not a multiple of 4
            const float t[4] = {v[q].x, v[q].y, v[q].z, v[q].w};
            for (int k = 0; c0 + k < d; ++k) drow[c0 + k] = t[k];
          }
        }
      } else {
        float v[R];
#pragma unroll
        for (int q = 0; q < R; ++q)
          if (r0 + q < n) v[q] = src[q][c];
#pragma unroll
        for (int q = 0; q < R; ++q)
          if (r0 + q < n) out[(r0 + q) * ldo + c] = v[q];
      }
    }
  }
  if (loaded) {
    my_loaded = warp_sum(my_loaded);
    if (lane == 0 && my_loaded) atomicAdd(loaded, (unsigned long long)my_loaded);
  }
  if (hits) {
    my_hits = warp_sum(my_hits);
    if (lane == 0 && my_hits) atomicAdd(hits, (unsigned long long)my_hits);
  }
}

__device__ __forceinline__ int find_set(const int64_t* off, int n, int64_t i) {
  int lo = 0, hi = n;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (off[mid] <= i) lo = mid; else hi = mid;
  }
  return lo;
}

__global__ void mark_bitmaps_kernel(const int32_t* __restrict__ ids, const int64_t* __restrict__ off,
                                    int nsets, int64_t total, int64_t words, uint32_t* __restrict__ bm) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t g = ids[i];
    const int s = find_set(off, nsets, i);
    atomicOr(bm + s * words + (g >> 5), 1u << (g & 31));
  }
}

__global__ void bitmap_test_kernel(const int32_t* __restrict__ ids, int64_t n,
                                   const uint32_t* __restrict__ bm, int8_t* __restrict__ hit) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t g = ids[i];
    hit[i] = (int8_t)((bm[g >> 5] >> (g & 31)) & 1u);
  }
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

int fgl_mark_bitmaps(const int32_t* ids, const int64_t* offsets, int32_t nsets, int64_t total,
                     int64_t words, uint32_t* bitmaps, void* stream) {
  if (nsets < 1 || total < 0 || words < 1 || !bitmaps || (total > 0 && (!ids || !offsets))) {
    set_error("fgl_mark_bitmaps: bad arguments");
    return FGL_E_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  FGL_CUDA(cudaMemsetAsync(bitmaps, 0, 4 * words * (size_t)nsets, st));
  if (total == 0) return FGL_OK;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(total, 256), 148 * 16));
  FGL_COUNT_LAUNCH(), mark_bitmaps_kernel<<<grid, 256, 0, st>>>(ids, offsets, nsets, total, words, bitmaps);
  FGL_LAUNCH_CHECK("mark_bitmaps_kernel");
  return FGL_OK;
}

int fgl_bitmap_test(const int32_t* ids, int64_t n, const uint32_t* bitmap, int8_t* hit, void* stream) {
  if (n < 0 || (n > 0 && (!ids || !bitmap || !hit))) {
    set_error("fgl_bitmap_test: bad arguments");
    return FGL_E_INVALID;
  }
  if (n == 0) return FGL_OK;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), 148 * 16));
  FGL_COUNT_LAUNCH(), bitmap_test_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(ids, n, bitmap, hit);
  FGL_LAUNCH_CHECK("bitmap_test_kernel");
  return FGL_OK;
}

int fgl_gather_rows_cached(const float* feats, int64_t ldf, int32_t d, const int32_t* ids, int64_t n,
                           const uint32_t* prev_bitmap, const int32_t* prev_prefix, int64_t prev_base,
                           const float* prev_x, int64_t ldp, const int32_t* prev_row_map,
                           const int32_t* cache_slot, const float* cache_x, int64_t ldc, float* out, int64_t ldo,
                           uint64_t* loaded, uint64_t* hits, void* stream) {
  if (n < 0 || d < 1 || ldf < d || ldo < d || !feats || !out || (n > 0 && !ids) ||
      (prev_bitmap && (!prev_prefix || !prev_x || ldp < d)) || (cache_slot && (!cache_x || ldc < d))) {
    set_error("fgl_gather_rows: bad arguments");
    return FGL_E_INVALID;
  }
  if (n == 0) return FGL_OK;
  const bool vec = ((ldf | ldo | (prev_bitmap ? ldp : 0) | (cache_slot ? ldc : 0)) % 4 == 0) &&
                   !((reinterpret_cast<uintptr_t>(feats) | reinterpret_cast<uintptr_t>(out) |
                      reinterpret_cast<uintptr_t>(prev_x) | reinterpret_cast<uintptr_t>(cache_x)) & 15);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 8 * 4), 148 * 16));
  auto* ld = reinterpret_cast<unsigned long long*>(loaded);
  auto* ht = reinterpret_cast<unsigned long long*>(hits);
  const ProfMark pm = prof_begin((cudaStream_t)stream);
  if (vec)
    FGL_COUNT_LAUNCH(), gather_rows_kernel<true><<<grid, 256, 0, (cudaStream_t)stream>>>(
        feats, ldf, d, ids, n, prev_bitmap, prev_prefix, prev_base, prev_x, ldp, prev_row_map, cache_slot, cache_x,
        ldc, out, ldo, ld, ht);
  else
    FGL_COUNT_LAUNCH(), gather_rows_kernel<false><<<grid, 256, 0, (cudaStream_t)stream>>>(
        feats, ldf, d, ids, n, prev_bitmap, prev_prefix, prev_base, prev_x, ldp, prev_row_map, cache_slot, cache_x,
        ldc, out, ldo, ld, ht);
  prof_end(pm, kProfGather, n, d);
  FGL_LAUNCH_CHECK("gather_rows_kernel");
  return FGL_OK;
}

int fgl_gather_rows(const float* feats, int64_t ldf, int32_t d, const int32_t* ids, int64_t n,
                    const uint32_t* prev_bitmap, const int32_t* prev_prefix, int64_t prev_base,
                    const float* prev_x, int64_t ldp, float* out, int64_t ldo, uint64_t* loaded,
                    void* stream) {
  return fgl_gather_rows_cached(feats, ldf, d, ids, n, prev_bitmap, prev_prefix, prev_base, prev_x, ldp, nullptr,
                                nullptr, nullptr, 0, out, ldo, loaded, nullptr, stream);
}

// Page-lock (and map) a host feature table the caller allocated -- e.g. a
// shared-memory table every rank of a node maps -- so the loader reads it
// zero-copy; *dev_ptr receives the device address of its first byte.
int fgl_host_register(void* host, int64_t bytes, void** dev_ptr) {
  if (!host || bytes <= 0 || !dev_ptr) {
    set_error("fgl_host_register: bad arguments");
    return FGL_E_INVALID;
  }
  FGL_CUDA(cudaHostRegister(host, (size_t)bytes, cudaHostRegisterMapped | cudaHostRegisterPortable));
  void* d = nullptr;
  cudaError_t e = cudaHostGetDevicePointer(&d, host, 0);
  if (e != cudaSuccess) {
    cudaHostUnregister(host);
    return cuda_status(e, "cudaHostGetDevicePointer");
  }
  *dev_ptr = d;
  return FGL_OK;
}

int fgl_host_unregister(void* host) {
  FGL_CUDA(cudaHostUnregister(host));
  return FGL_OK;
}

}  // extern "C"
