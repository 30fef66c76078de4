// Depth-major window rows for the all-rows layouts (GIN / GraphSAGE), sm_100a.
//
// The reference computes every layer of GIN over all num_local rows
// (trainer.py:182-195).  Layer i only needs the rows of R_i = the nodes first
// reached within H-1-i hops (the targets of hop H-1-i and, through the root
// term, of every later hop), and R_{L-1} ⊆ ... ⊆ R_0 ⊆ unique.  Ordering each
// batch's unique rows by (depth, node id) -- depth = first hop whose frontier
// holds the node (seeds 0, last-hop-only sources H) -- makes every R_i a
// PREFIX of the batch's block, so layer i simply runs on the first |R_i| rows
// (layer 0 on products: ~130K of ~615K rows).  Row values are unchanged
// (row-independent math, same CSR edge order); only the row numbering moves.
//
// fgl_depth_relayout rewrites, on the device and without a host sync, a
// sampled window (fgl_sample_window outputs + workspace) into that order:
// unique_nodes, tgt_row / src_row, seed_rows, plus row_map[old row] = new row
// (for the Match loader, whose bitmaps speak old ranks) and the per-batch
// depth counts depth_cnt[b * (H + 1) + h].
#include <algorithm>

#include "common.cuh"

namespace fgl {
namespace {

constexpr int LT = 256;

__device__ __forceinline__ int seg_of(const int64_t* off, int n, int64_t i) {
  int lo = 0, hi = n;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(off + mid) <= i) lo = mid; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ int32_t rank_in(const uint32_t* __restrict__ bm, const int32_t* __restrict__ wprefix,
                                           int64_t base_word, int32_t g) {
  const int64_t w = base_word + (g >> 5);
  return (int32_t)(wprefix[w] + __popc(bm[w] & ((1u << (g & 31)) - 1u)));
}

__global__ void depth_init_kernel(int8_t* depth, const int64_t* uoff, int nb, int H) {
  const int64_t U = uoff[nb];
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < U; u += (int64_t)gridDim.x * blockDim.x)
    depth[u] = (int8_t)H;
}

__global__ void depth_mark_kernel(const int32_t* __restrict__ front, const int64_t* __restrict__ fo, int nb,
                                  const uint32_t* __restrict__ bm_all, const int32_t* __restrict__ wprefix,
                                  int64_t words, int h, int8_t* depth) {
  const int64_t F = fo[nb];
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < F; j += (int64_t)gridDim.x * blockDim.x) {
    const int b = seg_of(fo, nb, j);
    depth[rank_in(bm_all, wprefix, (int64_t)b * words, front[j])] = (int8_t)h;
  }
}

// per (batch, depth) counts: block-local histogram, then global atomics
__global__ void depth_count_kernel(const int8_t* __restrict__ depth, const int64_t* __restrict__ uoff, int nb,
                                   int H, unsigned long long* cnt) {
  __shared__ unsigned int sh[64 * 9];
  const int K = nb * (H + 1);
  for (int k = threadIdx.x; k < K; k += blockDim.x) sh[k] = 0;
  __syncthreads();
  const int64_t U = uoff[nb];
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < U; u += (int64_t)gridDim.x * blockDim.x) {
    const int b = seg_of(uoff, nb, u);
    atomicAdd(sh + b * (H + 1) + depth[u], 1u);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < K; k += blockDim.x)
    if (sh[k]) atomicAdd(cnt + k, (unsigned long long)sh[k]);
}

// rows of depth h: count per chunk
__global__ void depth_chunk_kernel(const int8_t* __restrict__ depth, const int64_t* __restrict__ uoff, int nb,
                                   int h, int64_t* part) {
  __shared__ int64_t sm[33];
  const int64_t U = uoff[nb];
  const int64_t chunk = ceil_div(U, gridDim.x);
  const int64_t i0 = blockIdx.x * chunk, i1 = min(U, i0 + chunk);
  int64_t c = 0;
  for (int64_t u = i0 + threadIdx.x; u < i1; u += blockDim.x) c += depth[u] == h ? 1 : 0;
  c = block_sum(c, sm);
  if (threadIdx.x == 0) part[blockIdx.x] = c;
}

__global__ void depth_part_scan_kernel(int64_t* part, int n) {
  __shared__ int64_t sm[33];
  int64_t carry = 0;
  for (int base = 0; base < n; base += blockDim.x) {
    const int i = base + threadIdx.x;
    int64_t v = i < n ? part[i] : 0, tot;
    const int64_t ex = block_excl_scan(v, sm, &tot);
    if (i < n) part[i] = carry + ex;
    carry += tot;
  }
}

// All depths in one pass (instead of one count / scan / apply pass per depth).
// Per-chunk counts of every depth: part[d * (G + 1) + blk].
__global__ void depth_chunk_all_kernel(const int8_t* __restrict__ depth, const int64_t* __restrict__ uoff, int nb,
                                       int D, int64_t* part) {
  __shared__ unsigned int sc[8];
  if (threadIdx.x < 8) sc[threadIdx.x] = 0;
  __syncthreads();
  const int64_t U = uoff[nb];
  const int64_t chunk = ceil_div(U, gridDim.x);
  const int64_t i0 = blockIdx.x * chunk, i1 = min(U, i0 + chunk);
  unsigned int c[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int64_t u = i0 + threadIdx.x; u < i1; u += blockDim.x) {
    const int d = depth[u];
#pragma unroll
    for (int k = 0; k < 8; ++k) c[k] += (d == k) ? 1u : 0u;
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    unsigned int v = c[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(sc + k, v);
  }
  __syncthreads();
  if (threadIdx.x < D) part[(int64_t)threadIdx.x * (gridDim.x + 1) + blockIdx.x] = sc[threadIdx.x];
}

// block d: exclusive scan of depth d's chunk counts
__global__ void depth_part_scan_all_kernel(int64_t* part, int n) {
  __shared__ int64_t sm[33];
  int64_t* q = part + (int64_t)blockIdx.x * (n + 1);
  int64_t carry = 0;
  for (int base = 0; base < n; base += blockDim.x) {
    const int i = base + threadIdx.x;
    int64_t v = i < n ? q[i] : 0, tot;
    const int64_t ex = block_excl_scan(v, sm, &tot);
    if (i < n) q[i] = carry + ex;
    carry += tot;
  }
}

// new row of every row, all depths at once: warp ballots give each row its
// rank among same-depth rows of the tile; u0[b] + rows of smaller depth in
// batch b + (same-depth rows of batch b before it)
__global__ void __launch_bounds__(256) depth_apply_all_kernel(const int8_t* __restrict__ depth,
                                                              const int64_t* __restrict__ uoff, int nb, int D,
                                                              const int64_t* __restrict__ part,
                                                              const unsigned long long* __restrict__ cnt,
                                                              int32_t* __restrict__ row_map) {
  __shared__ int64_t sbase[64 * 9], sbefore[64 * 9];
  __shared__ int64_t srun[8], tot[8];
  __shared__ int wcnt[8][8], wex[8][8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int k = tid; k < nb * D; k += blockDim.x) {
    const int b = k / D, d = k - b * D;
    int64_t base = 0, before = 0;
    for (int hh = 0; hh < d; ++hh) base += (int64_t)cnt[b * D + hh];
    for (int bb = 0; bb < b; ++bb) before += (int64_t)cnt[bb * D + d];
    sbase[k] = uoff[b] + base;
    sbefore[k] = before;
  }
  if (tid < D) srun[tid] = part[(int64_t)tid * (gridDim.x + 1) + blockIdx.x];
  __syncthreads();
  const int64_t U = uoff[nb];
  const int64_t chunk = ceil_div(U, gridDim.x);
  const int64_t i0 = blockIdx.x * chunk, i1 = min(U, i0 + chunk);
  const unsigned lt_mask = (1u << lane) - 1u;
  for (int64_t t0 = i0; t0 < i1; t0 += blockDim.x) {
    const int64_t u = t0 + tid;
    const int dd = u < i1 ? (int)depth[u] : -1;
    int mypre = 0;
    for (int d = 0; d < D; ++d) {
      const unsigned m = __ballot_sync(0xffffffffu, dd == d);
      if (lane == 0) wcnt[warp][d] = __popc(m);
      if (dd == d) mypre = __popc(m & lt_mask);
    }
    __syncthreads();
    if (tid < D) {
      int acc = 0;
      for (int w = 0; w < 8; ++w) {
        wex[w][tid] = acc;
        acc += wcnt[w][tid];
      }
      tot[tid] = acc;
    }
    __syncthreads();
    if (dd >= 0) {
      const int b = seg_of(uoff, nb, u);
      const int64_t ex = srun[dd] + wex[warp][dd] + mypre;
      row_map[u] = (int32_t)(sbase[b * D + dd] + ex - sbefore[b * D + dd]);
    }
    __syncthreads();
    if (tid < D) srun[tid] += tot[tid];
    __syncthreads();
  }
}

// new row of every depth-h row: u0[b] + (depth-h rows of batch b before it,
// = global depth-h rank minus the depth-h rows of earlier batches) + the rows
// of smaller depth in batch b
__global__ void depth_apply_kernel(const int8_t* __restrict__ depth, const int64_t* __restrict__ uoff, int nb,
                                   int H, int h, const int64_t* __restrict__ part,
                                   const unsigned long long* __restrict__ cnt, int32_t* __restrict__ row_map) {
  __shared__ int64_t sm[33];
  __shared__ int64_t sbase[64], sbefore[64];
  if (threadIdx.x < nb) {
    const int b = threadIdx.x;
    int64_t base = 0, before = 0;
    for (int hh = 0; hh < h; ++hh) base += (int64_t)cnt[b * (H + 1) + hh];
    for (int bb = 0; bb < b; ++bb) before += (int64_t)cnt[bb * (H + 1) + h];
    sbase[b] = uoff[b] + base;
    sbefore[b] = before;
  }
  __syncthreads();
  const int64_t U = uoff[nb];
  const int64_t chunk = ceil_div(U, gridDim.x);
  const int64_t i0 = blockIdx.x * chunk, i1 = min(U, i0 + chunk);
  int64_t run = part[blockIdx.x];
  for (int64_t t0 = i0; t0 < i1; t0 += blockDim.x) {
    const int64_t u = t0 + threadIdx.x;
    const int64_t f = (u < i1 && depth[u] == h) ? 1 : 0;
    int64_t tot;
    const int64_t ex = run + block_excl_scan(f, sm, &tot);
    if (f) {
      const int b = seg_of(uoff, nb, u);
      row_map[u] = (int32_t)(sbase[b] + ex - sbefore[b]);
    }
    run += tot;
  }
}

__global__ void remap_kernel(int32_t* __restrict__ a, const int64_t* __restrict__ n_ptr, int64_t n_fixed,
                             const int32_t* __restrict__ row_map) {
  const int64_t n = n_ptr ? *n_ptr : n_fixed;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] = row_map[a[i]];
}

__global__ void permute_unique_kernel(const int32_t* __restrict__ uniq, const int64_t* __restrict__ uoff, int nb,
                                      const int32_t* __restrict__ row_map, int32_t* __restrict__ out) {
  const int64_t U = uoff[nb];
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < U; u += (int64_t)gridDim.x * blockDim.x)
    out[row_map[u]] = uniq[u];
}

__global__ void copy_i32_kernel(const int32_t* __restrict__ src, const int64_t* __restrict__ n_ptr, int nb,
                                int32_t* __restrict__ dst) {
  const int64_t n = n_ptr[nb];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

// Y[r][c] += X[r][c] (one rounded add: the root term of the GIN / SAGE
// backward, dx = aggregate_T(dh) + dh, trainer.py:226-228) for r < nrows
__global__ void add_rows_kernel(float* __restrict__ Y, int64_t ldy, const float* __restrict__ X, int64_t ldx,
                                int64_t nrows, int d) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nrows * d;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / d;
    const int c = (int)(i - r * d);
    Y[r * ldy + c] = __fadd_rn(Y[r * ldy + c], X[r * ldx + c]);
  }
}

}  // namespace
}  // namespace fgl

using namespace fgl;

extern "C" {

int64_t fgl_depth_relayout_ws_bytes(int64_t unique_cap) {
  const int64_t u = std::max<int64_t>(unique_cap, 1);
  return (u + 255) / 256 * 256 + 4 * u + 8 * 8 * (kPersistentCTAs + 1) + 256;  // part: up to 8 depths x (G + 1)
}

int fgl_depth_relayout(const int64_t* counts, int32_t H, int32_t nb, const int32_t* frontier,
                       int64_t frontier_stride, const uint32_t* bm_all, const int32_t* wprefix, int64_t words,
                       int32_t* unique_nodes, int64_t unique_cap, int32_t* tgt_row, int32_t* src_row,
                       int32_t* seed_rows, int64_t num_seeds, int32_t* row_map, int64_t* depth_cnt, void* ws,
                       int64_t ws_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (!counts || H < 1 || H > FGL_MAX_HOPS || nb < 1 || nb > 64 || !frontier || !bm_all || !wprefix ||
      !unique_nodes || !row_map || !depth_cnt || !ws) {
    set_error("fgl_depth_relayout: bad arguments");
    return FGL_E_INVALID;
  }
  if (nb * (H + 1) > 64 * 9) {
    set_error("fgl_depth_relayout: too many (batch, depth) classes");
    return FGL_E_UNSUPPORTED;
  }
  if (ws_bytes < fgl_depth_relayout_ws_bytes(unique_cap)) {
    set_error("fgl_depth_relayout: workspace too small");
    return FGL_E_CAPACITY;
  }
  const int64_t* uoff = counts + FGL_CNT_UNIQ(H, nb);
  char* p = static_cast<char*>(ws);
  // layout: depth int8 [cap], tmp unique int32 [cap], part int64 [2G+2]
  const int64_t cap = std::max<int64_t>(unique_cap, 1);
  int8_t* depth = reinterpret_cast<int8_t*>(p);
  int32_t* tmp = reinterpret_cast<int32_t*>(p + (cap + 255) / 256 * 256);
  int64_t* part = reinterpret_cast<int64_t*>(p + (cap + 255) / 256 * 256 + 4 * cap);
  const int G = kPersistentCTAs;
  const int TG = 4 * G;
  auto* cnt = reinterpret_cast<unsigned long long*>(depth_cnt);
  FGL_CUDA(cudaMemsetAsync(depth_cnt, 0, sizeof(int64_t) * nb * (H + 1), st));
  FGL_COUNT_LAUNCH(), depth_init_kernel<<<TG, LT, 0, st>>>(depth, uoff, nb, H);
  for (int h = H - 1; h >= 0; --h) {
    const int64_t* fo = counts + FGL_CNT_FRONT(H, nb) + (int64_t)h * (nb + 1);
    FGL_COUNT_LAUNCH(), depth_mark_kernel<<<TG, LT, 0, st>>>(frontier + h * frontier_stride, fo, nb, bm_all,
                                                            wprefix, words, h, depth);
  }
  FGL_COUNT_LAUNCH(), depth_count_kernel<<<TG, LT, 0, st>>>(depth, uoff, nb, H, cnt);
  if (H + 1 <= 8 && LT == 256) {
    // all depths in one count / scan / apply pass
    FGL_COUNT_LAUNCH(), depth_chunk_all_kernel<<<G, LT, 0, st>>>(depth, uoff, nb, H + 1, part);
    FGL_COUNT_LAUNCH(), depth_part_scan_all_kernel<<<H + 1, 1024, 0, st>>>(part, G);
    FGL_COUNT_LAUNCH(), depth_apply_all_kernel<<<G, LT, 0, st>>>(depth, uoff, nb, H + 1, part, cnt, row_map);
  } else {
    for (int h = 0; h <= H; ++h) {
      FGL_COUNT_LAUNCH(), depth_chunk_kernel<<<G, LT, 0, st>>>(depth, uoff, nb, h, part);
      FGL_COUNT_LAUNCH(), depth_part_scan_kernel<<<1, 1024, 0, st>>>(part, G);
      FGL_COUNT_LAUNCH(), depth_apply_kernel<<<G, LT, 0, st>>>(depth, uoff, nb, H, h, part, cnt, row_map);
    }
  }
  FGL_COUNT_LAUNCH(), permute_unique_kernel<<<TG, LT, 0, st>>>(unique_nodes, uoff, nb, row_map, tmp);
  FGL_COUNT_LAUNCH(), copy_i32_kernel<<<TG, LT, 0, st>>>(tmp, uoff, nb, unique_nodes);
  const int64_t* eoff_end = counts + (int64_t)H * nb;  // total edges of the window
  if (tgt_row) FGL_COUNT_LAUNCH(), remap_kernel<<<TG, LT, 0, st>>>(tgt_row, eoff_end, 0, row_map);
  if (src_row) FGL_COUNT_LAUNCH(), remap_kernel<<<TG, LT, 0, st>>>(src_row, eoff_end, 0, row_map);
  if (seed_rows && num_seeds > 0) FGL_COUNT_LAUNCH(), remap_kernel<<<TG, LT, 0, st>>>(seed_rows, nullptr, num_seeds, row_map);
  FGL_LAUNCH_CHECK("depth_relayout");
  return FGL_OK;
}

int fgl_add_rows(float* Y, int64_t ldy, const float* X, int64_t ldx, int64_t nrows, int32_t d, void* stream) {
  if (nrows < 0 || d < 1 || !Y || !X || ldy < d || ldx < d) {
    set_error("fgl_add_rows: bad arguments");
    return FGL_E_INVALID;
  }
  if (nrows == 0) return FGL_OK;
  FGL_COUNT_LAUNCH(), add_rows_kernel<<<(int)std::min<int64_t>(ceil_div(nrows * d, LT), 148 * 16), LT, 0,
                                         (cudaStream_t)stream>>>(Y, ldy, X, ldx, nrows, d);
  FGL_LAUNCH_CHECK("add_rows_kernel");
  return FGL_OK;
}

}  // extern "C"
