// Per-layer CSR packing for the sampled block graph (sm_100a).
//
// Replaces, on device, trainer._prepare_batch's per-hop work
// (trainer.py:165-179): _layer_edge_weights (trainer.py:156-162),
// compute.edges_to_csr (compute.py:219-230) and compute.csr_transpose
// (compute.py:233-239).
//
// * forward CSR: sampled targets are already grouped in ascending row order
//   (frontier order), so the reference's stable argsort is the identity and
//   indptr comes from one "sorted keys -> offsets" pass;
// * transpose: a STABLE counting sort by source row -- histogram, exclusive
//   scan, atomic scatter of edge indices, then a segmented sort of each row's
//   edge indices (rows are short: thread-level sorting networks; long rows:
//   warp / CTA bitonic sorts in shared memory; huge rows: CTA bitonic in
//   global memory).  Stability makes the backward aggregation bit-exact.
// * GCN weights 1/sqrt(indeg_t * outdeg_s) in fp64, rounded once to f32.
#include <algorithm>

#include "common.cuh"

namespace fgl {
namespace {

constexpr int kThreads = 256;
constexpr int kWarpSortMax = 1024;    // rows sorted by one warp in smem
constexpr int kBlockSortMax = 32768;  // rows sorted by one CTA in smem (128 KB)

inline int64_t al(int64_t x) { return (x + 255) / 256 * 256; }

struct GroupWs {
  int32_t* counts;   // [num_keys]
  int32_t* cursor;   // [num_keys]
  int64_t* part;     // [kScanCTAs + 1]
  int32_t* lists;    // [3 * num_keys]: medium, large, huge row lists
  int32_t* nlist;    // [4]
  int64_t bytes;
};

// the count scans: one 2048-key tile per CTA up to 8 CTAs per SM (GIN / SAGE
// index every hop over the window's ~5M rows: 296 CTAs walking 8 serial
// tiles each took 28 us per scan)
constexpr int kScanCTAs = 8 * kNumSMs;

GroupWs group_ws(void* base, int64_t num_keys) {
  char* p = static_cast<char*>(base);
  GroupWs w;
  int64_t o = 0;
  w.counts = reinterpret_cast<int32_t*>(p + o); o = al(o + 4 * num_keys);
  w.cursor = reinterpret_cast<int32_t*>(p + o); o = al(o + 4 * num_keys);
  w.part = reinterpret_cast<int64_t*>(p + o); o = al(o + 8 * (kScanCTAs + 1));
  w.lists = reinterpret_cast<int32_t*>(p + o); o = al(o + 4 * 3 * num_keys);
  w.nlist = reinterpret_cast<int32_t*>(p + o); o = al(o + 4 * 4);
  w.bytes = o;
  return w;
}

// ------------------------------------------------------------------ kernels --
__global__ void offsets_from_sorted_kernel(const int32_t* __restrict__ rows, int64_t nnz,
                                           int64_t num_rows, int64_t base, int64_t* __restrict__ indptr) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e <= nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t prev = e > 0 ? rows[e - 1] : -1;
    const int64_t cur = e < nnz ? rows[e] : num_rows;
    for (int64_t r = prev + 1; r <= cur; ++r) indptr[r] = base + e;
  }
}

// row-parallel variant for sparse targets (long runs of rows without edges,
// e.g. the depth-major rows of the GIN / SAGE layout): lower_bound per row
__global__ void offsets_bsearch_kernel(const int32_t* __restrict__ rows, int64_t nnz, int64_t num_rows,
                                       int64_t base, int64_t* __restrict__ indptr) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r <= num_rows;
       r += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = nnz;  // first e with rows[e] >= r
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (__ldg(rows + mid) < r) lo = mid + 1; else hi = mid;
    }
    indptr[r] = base + lo;
  }
}

__global__ void histogram_kernel(const int32_t* __restrict__ keys, int64_t n, int32_t* counts) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(counts + keys[e], 1);
}

__global__ void chunk_sum_kernel(const int32_t* __restrict__ v, int64_t n, int64_t* part) {
  __shared__ int64_t sm[33];
  const int64_t chunk = ceil_div(n, gridDim.x);
  const int64_t i0 = blockIdx.x * chunk, i1 = min(n, i0 + chunk);
  int64_t s = 0;
  for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) s += v[i];
  s = block_sum(s, sm);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void part_scan_kernel(int64_t* part, int n) {
  __shared__ int64_t sm[33];
  int64_t carry = 0;
  for (int b = 0; b < n; b += blockDim.x) {
    const int i = b + threadIdx.x;
    int64_t v = i < n ? part[i] : 0, tot;
    const int64_t ex = block_excl_scan(v, sm, &tot);
    if (i < n) part[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) part[n] = carry;
}

// indptr[i] = base + exclusive prefix of v; indptr[n] = base + total
__global__ void chunk_scan_kernel(const int32_t* __restrict__ v, int64_t n, const int64_t* part,
                                  int64_t base, int64_t* __restrict__ out) {
  __shared__ int64_t sm[33];
  const int64_t chunk = ceil_div(n, gridDim.x);
  const int64_t i0 = blockIdx.x * chunk, i1 = min(n, i0 + chunk);
  int64_t run = base + part[blockIdx.x];
  constexpr int IT = 8;  // items per thread per tile (thread-blocked)
  for (int64_t t0 = i0; t0 < i1; t0 += (int64_t)blockDim.x * IT) {
    const int64_t first = t0 + (int64_t)threadIdx.x * IT;
    int64_t x[IT], local = 0;
#pragma unroll
    for (int q = 0; q < IT; ++q) {
      x[q] = first + q < i1 ? v[first + q] : 0;
      const int64_t t = x[q];
      x[q] = local;  // exclusive within the thread
      local += t;
    }
    int64_t tot;
    const int64_t ex = run + block_excl_scan(local, sm, &tot);
#pragma unroll
    for (int q = 0; q < IT; ++q)
      if (first + q < i1) out[first + q] = ex + x[q];
    run += tot;
  }
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) out[n] = base + part[gridDim.x];
}

__global__ void scatter_kernel(const int32_t* __restrict__ keys, int64_t n,
                               const int64_t* __restrict__ indptr, int64_t base,
                               int32_t* cursor, int32_t* __restrict__ perm) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t k = keys[e];
    const int64_t pos = indptr[k] - base + atomicAdd(cursor + k, 1);
    perm[pos] = (int32_t)e;
  }
}

__device__ __forceinline__ void cex(int32_t& a, int32_t& b) {
  const int32_t lo = min(a, b), hi = max(a, b);
  a = lo; b = hi;
}

template <int N>
__device__ __forceinline__ void reg_sort(int32_t* g, int len) {
  int32_t v[N];
#pragma unroll
  for (int i = 0; i < N; ++i) v[i] = i < len ? g[i] : INT32_MAX;
#pragma unroll
  for (int r = 0; r < N; ++r) {
#pragma unroll
    for (int i = r & 1; i + 1 < N; i += 2) cex(v[i], v[i + 1]);
  }
#pragma unroll
  for (int i = 0; i < N; ++i)
    if (i < len) g[i] = v[i];
}

// Rows of length <= 16 are sorted in registers; longer rows are queued.
__global__ void seg_sort_small_kernel(const int64_t* __restrict__ indptr, int64_t num_keys,
                                      int64_t base, int32_t* __restrict__ perm, int32_t* lists,
                                      int32_t* nlist) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < num_keys;
       k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = indptr[k] - base;
    const int64_t len = indptr[k + 1] - base - s;
    if (len <= 1) continue;
    int32_t* g = perm + s;
    if (len == 2) {
      int32_t a = g[0], b = g[1];
      if (a > b) { g[0] = b; g[1] = a; }
    } else if (len <= 4) {
      reg_sort<4>(g, (int)len);
    } else if (len <= 8) {
      reg_sort<8>(g, (int)len);
    } else if (len <= 16) {
      reg_sort<16>(g, (int)len);
    } else {
      const int cls = len <= kWarpSortMax ? 0 : (len <= kBlockSortMax ? 1 : 2);
      const int slot = atomicAdd(nlist + cls, 1);
      lists[cls * num_keys + slot] = (int32_t)k;
    }
  }
}

// Ascending bitonic sort of n values with virtual +inf padding to the next
// power of two: every comparator is (lo < hi) -> min at lo, so comparators
// whose hi index falls in the padding are no-ops and are skipped.
struct WarpSync { __device__ void operator()() const { __syncwarp(); } };
struct BlockSync { __device__ void operator()() const { __syncthreads(); } };

template <typename Sync>
__device__ __forceinline__ void bitonic_asc(int32_t* v, int n, int tid, int nthr, Sync sync) {
  int P = 1;
  while (P < n) P <<= 1;
  const int half = P >> 1;
  for (int size = 2; size <= P; size <<= 1) {
    const int hs = size >> 1;
    for (int t = tid; t < half; t += nthr) {
      const int blk = t / hs, off = t % hs;
      const int lo = blk * size + off, hi = blk * size + size - 1 - off;
      if (hi < n) cex(v[lo], v[hi]);
    }
    sync();
    for (int stride = size >> 2; stride > 0; stride >>= 1) {
      for (int t = tid; t < half; t += nthr) {
        const int lo = (t / stride) * 2 * stride + (t % stride), hi = lo + stride;
        if (hi < n) cex(v[lo], v[hi]);
      }
      sync();
    }
  }
}

__global__ void seg_sort_warp_kernel(const int64_t* __restrict__ indptr, int64_t base,
                                     int32_t* __restrict__ perm, const int32_t* __restrict__ list,
                                     const int32_t* nlist) {
  extern __shared__ int32_t smem[];
  const int wid = warp_id(), lane = lane_id();
  int32_t* buf = smem + wid * kWarpSortMax;
  const int n_rows = nlist[0];
  const int wpb = blockDim.x >> 5;
  for (int r = blockIdx.x * wpb + wid; r < n_rows; r += gridDim.x * wpb) {
    const int64_t k = list[r];
    const int64_t s = indptr[k] - base;
    const int len = (int)(indptr[k + 1] - base - s);
    for (int i = lane; i < len; i += 32) buf[i] = perm[s + i];
    __syncwarp();
    bitonic_asc(buf, len, lane, 32, WarpSync{});
    for (int i = lane; i < len; i += 32) perm[s + i] = buf[i];
    __syncwarp();
  }
}

__global__ void seg_sort_block_kernel(const int64_t* __restrict__ indptr, int64_t base,
                                      int32_t* __restrict__ perm, const int32_t* __restrict__ list,
                                      const int32_t* nlist, int global_mem) {
  extern __shared__ int32_t smem[];
  const int n_rows = nlist[0];
  for (int r = blockIdx.x; r < n_rows; r += gridDim.x) {
    const int64_t k = list[r];
    const int64_t s = indptr[k] - base;
    const int len = (int)(indptr[k + 1] - base - s);
    int32_t* buf = global_mem ? perm + s : smem;
    if (!global_mem) {
      for (int i = threadIdx.x; i < len; i += blockDim.x) buf[i] = perm[s + i];
      __syncthreads();
    }
    bitonic_asc(buf, len, threadIdx.x, blockDim.x, BlockSync{});
    if (!global_mem) {
      for (int i = threadIdx.x; i < len; i += blockDim.x) perm[s + i] = buf[i];
    }
    __syncthreads();
  }
}

// GCN weight of each edge + the transposed edge arrays in stable source order
__device__ __forceinline__ float gcn_weight(int64_t indeg, int64_t outdeg) {
  const double prod = (double)(indeg * outdeg);
  return __double2float_rn(__ddiv_rn(1.0, __dsqrt_rn(prod)));
}

__global__ void layer_weights_kernel(const int32_t* __restrict__ lt, const int32_t* __restrict__ ls,
                                     int64_t nnz, const int64_t* __restrict__ indptr,
                                     const int32_t* __restrict__ outdeg, int gcn,
                                     float* __restrict__ w) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (gcn == 0) { w[e] = 1.0f; continue; }  // GIN
    const int32_t t = lt[e];
    const int64_t indeg = indptr[t + 1] - indptr[t];
    if (gcn == 2) {  // SAGE mean: f32(1 / indeg) from fp64
      w[e] = __double2float_rn(__ddiv_rn(1.0, (double)indeg));
      continue;
    }
    w[e] = gcn_weight(indeg, outdeg[ls[e]]);
  }
}

__global__ void gather_i32_f32_kernel(const int32_t* __restrict__ perm, int64_t n,
                                      const int32_t* __restrict__ a, const float* __restrict__ b,
                                      int32_t* __restrict__ ao, float* __restrict__ bo) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int32_t e = perm[p];
    if (ao) ao[p] = a[e];
    if (bo) bo[p] = b[e];
  }
}

int grid_for(int64_t n, int per = kThreads) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, per), 148 * 16));
}

int stable_group_impl(const int32_t* keys, int64_t nnz, int64_t num_keys, int64_t base,
                      int64_t* indptr, int32_t* perm, int32_t* counts_out, void* ws,
                      int64_t ws_bytes, cudaStream_t st) {
  GroupWs w = group_ws(ws, num_keys);
  if (w.bytes > ws_bytes) {
    set_error("stable_group workspace too small (%lld < %lld)", (long long)ws_bytes, (long long)w.bytes);
    return FGL_E_CAPACITY;
  }
  int32_t* counts = counts_out ? counts_out : w.counts;
  FGL_CUDA(cudaMemsetAsync(counts, 0, 4 * num_keys, st));
  FGL_CUDA(cudaMemsetAsync(w.cursor, 0, 4 * num_keys, st));
  FGL_CUDA(cudaMemsetAsync(w.nlist, 0, 16, st));
  if (nnz > 0) FGL_COUNT_LAUNCH(), histogram_kernel<<<grid_for(nnz), kThreads, 0, st>>>(keys, nnz, counts);
  const int G = (int)std::max<int64_t>(1, std::min<int64_t>(kScanCTAs, ceil_div(num_keys, 2048)));
  FGL_COUNT_LAUNCH(), chunk_sum_kernel<<<G, kThreads, 0, st>>>(counts, num_keys, w.part);
  FGL_COUNT_LAUNCH(), part_scan_kernel<<<1, 1024, 0, st>>>(w.part, G);
  FGL_COUNT_LAUNCH(), chunk_scan_kernel<<<G, kThreads, 0, st>>>(counts, num_keys, w.part, base, indptr);
  if (nnz > 0) {
    FGL_COUNT_LAUNCH(), scatter_kernel<<<grid_for(nnz), kThreads, 0, st>>>(keys, nnz, indptr, base, w.cursor, perm);
    FGL_COUNT_LAUNCH(), seg_sort_small_kernel<<<grid_for(num_keys), kThreads, 0, st>>>(indptr, num_keys, base, perm,
                                                                    w.lists, w.nlist);
    FGL_COUNT_LAUNCH(), seg_sort_warp_kernel<<<4 * kNumSMs, 128, 4 * kWarpSortMax * 4, st>>>(indptr, base, perm,
                                                                         w.lists, w.nlist);
    static bool attr = false;
    if (!attr) {
      FGL_CUDA(cudaFuncSetAttribute(seg_sort_block_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * kBlockSortMax));
      attr = true;
    }
    FGL_COUNT_LAUNCH(), seg_sort_block_kernel<<<kNumSMs, 1024, 4 * kBlockSortMax, st>>>(
        indptr, base, perm, w.lists + num_keys, w.nlist + 1, 0);
    FGL_COUNT_LAUNCH(), seg_sort_block_kernel<<<kNumSMs, 1024, 0, st>>>(indptr, base, perm, w.lists + 2 * num_keys,
                                                    w.nlist + 2, 1);
  }
  FGL_LAUNCH_CHECK("stable_group");
  return FGL_OK;
}

}  // namespace
}  // namespace fgl

using namespace fgl;

extern "C" {

int64_t fgl_stable_group_ws_bytes(int64_t num_keys) {
  return group_ws(nullptr, std::max<int64_t>(num_keys, 1)).bytes;
}

int fgl_csr_offsets_sorted(const int32_t* rows, int64_t nnz, int64_t num_rows, int64_t base,
                           int64_t* indptr, void* stream) {
  if (nnz < 0 || num_rows < 0 || !indptr || (nnz > 0 && !rows)) {
    set_error("fgl_csr_offsets_sorted: bad arguments");
    return FGL_E_INVALID;
  }
  FGL_COUNT_LAUNCH(), offsets_from_sorted_kernel<<<grid_for(nnz + 1), kThreads, 0, (cudaStream_t)stream>>>(
      rows, nnz, num_rows, base, indptr);
  FGL_LAUNCH_CHECK("offsets_from_sorted_kernel");
  return FGL_OK;
}

int fgl_stable_group(const int32_t* keys, int64_t nnz, int64_t num_keys, int64_t* indptr,
                     int32_t* perm, int32_t* counts_out, void* ws, int64_t ws_bytes, void* stream) {
  if (nnz < 0 || num_keys < 1 || nnz >= (1ll << 31) || !indptr || (nnz > 0 && (!keys || !perm))) {
    set_error("fgl_stable_group: bad arguments");
    return FGL_E_INVALID;
  }
  return stable_group_impl(keys, nnz, num_keys, 0, indptr, perm, counts_out, ws, ws_bytes,
                           (cudaStream_t)stream);
}

int fgl_gather_i32_f32(const int32_t* perm, int64_t n, const int32_t* a, const float* b,
                       int32_t* a_out, float* b_out, void* stream) {
  if (n < 0 || (n > 0 && !perm)) {
    set_error("fgl_gather_i32_f32: bad arguments");
    return FGL_E_INVALID;
  }
  if (n == 0) return FGL_OK;
  FGL_COUNT_LAUNCH(), gather_i32_f32_kernel<<<grid_for(n), kThreads, 0, (cudaStream_t)stream>>>(perm, n, a, b, a_out, b_out);
  FGL_LAUNCH_CHECK("gather_i32_f32_kernel");
  return FGL_OK;
}

int64_t fgl_prepare_layer_ws_bytes(int64_t nnz, int64_t num_rows, int64_t num_cols) {
  (void)num_rows;
  return al(4 * std::max<int64_t>(nnz, 1)) + al(4 * std::max<int64_t>(num_cols, 1)) +
         fgl_stable_group_ws_bytes(num_cols);
}

static int prepare_layer_impl(const int32_t* lt, const int32_t* ls, int64_t nnz, int64_t num_rows,
                              int64_t num_cols, int32_t arch_gcn, int64_t* indptr, float* w,
                              int64_t* t_indptr, int32_t* t_col, float* t_w, void* ws, int64_t ws_bytes,
                              void* stream_, bool sparse_rows);

int fgl_prepare_layer(const int32_t* lt, const int32_t* ls, int64_t nnz, int64_t num_rows,
                      int64_t num_cols, int32_t arch_gcn, int64_t* indptr, float* w,
                      int64_t* t_indptr, int32_t* t_col, float* t_w, void* ws, int64_t ws_bytes,
                      void* stream_) {
  return prepare_layer_impl(lt, ls, nnz, num_rows, num_cols, arch_gcn, indptr, w, t_indptr, t_col, t_w, ws,
                            ws_bytes, stream_, false);
}

static int prepare_layer_impl(const int32_t* lt, const int32_t* ls, int64_t nnz, int64_t num_rows,
                              int64_t num_cols, int32_t arch_gcn, int64_t* indptr, float* w,
                              int64_t* t_indptr, int32_t* t_col, float* t_w, void* ws, int64_t ws_bytes,
                              void* stream_, bool sparse_rows) {
  cudaStream_t st = (cudaStream_t)stream_;
  // t_indptr == t_col == t_w == NULL: no transpose (model layer 0 -- the input
  // features need no gradient); only the source degrees for the weights
  const bool transpose = t_indptr != nullptr;
  if (nnz < 0 || num_rows < 1 || num_cols < 1 || nnz >= (1ll << 31) || !indptr || !w ||
      (nnz > 0 && (!lt || !ls)) || (transpose && nnz > 0 && (!t_col || !t_w)) ||
      (!transpose && (t_col || t_w))) {
    set_error("fgl_prepare_layer: bad arguments");
    return FGL_E_INVALID;
  }
  if (ws_bytes < fgl_prepare_layer_ws_bytes(nnz, num_rows, num_cols)) {
    set_error("fgl_prepare_layer: workspace too small");
    return FGL_E_CAPACITY;
  }
  char* p = static_cast<char*>(ws);
  int32_t* perm = reinterpret_cast<int32_t*>(p);
  int32_t* outdeg = reinterpret_cast<int32_t*>(p + al(4 * std::max<int64_t>(nnz, 1)));
  void* gws = p + al(4 * std::max<int64_t>(nnz, 1)) + al(4 * std::max<int64_t>(num_cols, 1));
  if (sparse_rows) {
    // grouped path: the stable grouping by target already wrote these
    // offsets (its exclusive scan of the per-row counts) -- nothing to do
  } else
    FGL_COUNT_LAUNCH(), offsets_from_sorted_kernel<<<grid_for(nnz + 1), kThreads, 0, st>>>(lt, nnz, num_rows, 0, indptr);
  if (transpose) {
    int rc = stable_group_impl(ls, nnz, num_cols, 0, t_indptr, perm, outdeg, gws,
                               fgl_stable_group_ws_bytes(num_cols), st);
    if (rc) return rc;
  } else {
    FGL_CUDA(cudaMemsetAsync(outdeg, 0, 4 * num_cols, st));
    if (nnz > 0) FGL_COUNT_LAUNCH(), histogram_kernel<<<grid_for(nnz), kThreads, 0, st>>>(ls, nnz, outdeg);
  }
  if (nnz > 0) {
    FGL_COUNT_LAUNCH(), layer_weights_kernel<<<grid_for(nnz), kThreads, 0, st>>>(lt, ls, nnz, indptr, outdeg, arch_gcn, w);
    if (transpose)
      FGL_COUNT_LAUNCH(), gather_i32_f32_kernel<<<grid_for(nnz), kThreads, 0, st>>>(perm, nnz, lt, w, t_col, t_w);
  }
  FGL_LAUNCH_CHECK("prepare_layer");
  return FGL_OK;
}

int64_t fgl_prepare_layer_grouped_ws_bytes(int64_t nnz, int64_t num_rows, int64_t num_cols) {
  const int64_t n = std::max<int64_t>(nnz, 1);
  return 2 * al(4 * n) + std::max(fgl_stable_group_ws_bytes(num_rows), fgl_prepare_layer_ws_bytes(nnz, num_rows, num_cols));
}

// fgl_prepare_layer for targets that are grouped but NOT ascending (the
// depth-major rows of fgl_depth_relayout): a stable grouping by target first
// (compute.edges_to_csr's stable argsort, compute.py:219-230), then the
// sorted-target path; col_out receives the forward CSR's column array.
int fgl_prepare_layer_grouped(const int32_t* lt, const int32_t* ls, int64_t nnz, int64_t num_rows,
                              int64_t num_cols, int32_t arch, int64_t* indptr, int32_t* col_out, float* w,
                              int64_t* t_indptr, int32_t* t_col, float* t_w, void* ws, int64_t ws_bytes,
                              void* stream_) {
  cudaStream_t st = (cudaStream_t)stream_;
  if (nnz < 0 || num_rows < 1 || num_cols < 1 || nnz >= (1ll << 31) || !indptr || !w ||
      (nnz > 0 && (!lt || !ls || !col_out)) || (t_indptr && nnz > 0 && (!t_col || !t_w)) ||
      (!t_indptr && (t_col || t_w))) {
    set_error("fgl_prepare_layer_grouped: bad arguments");
    return FGL_E_INVALID;
  }
  if (ws_bytes < fgl_prepare_layer_grouped_ws_bytes(nnz, num_rows, num_cols)) {
    set_error("fgl_prepare_layer_grouped: workspace too small");
    return FGL_E_CAPACITY;
  }
  char* p = static_cast<char*>(ws);
  const int64_t n = std::max<int64_t>(nnz, 1);
  int32_t* perm = reinterpret_cast<int32_t*>(p);
  int32_t* lt_s = reinterpret_cast<int32_t*>(p + al(4 * n));
  void* rest = p + 2 * al(4 * n);
  const int64_t rest_bytes = ws_bytes - 2 * al(4 * n);
  int rc = stable_group_impl(lt, nnz, num_rows, 0, indptr, perm, nullptr, rest, rest_bytes, st);
  if (rc) return rc;
  if (nnz > 0) {
    FGL_COUNT_LAUNCH(), gather_i32_f32_kernel<<<grid_for(nnz), kThreads, 0, st>>>(perm, nnz, lt, nullptr, lt_s, nullptr);
    FGL_COUNT_LAUNCH(), gather_i32_f32_kernel<<<grid_for(nnz), kThreads, 0, st>>>(perm, nnz, ls, nullptr, col_out, nullptr);
  }
  return prepare_layer_impl(lt_s, col_out, nnz, num_rows, num_cols, arch, indptr, w, t_indptr, t_col, t_w, rest,
                            rest_bytes, stream_, true);
}

}  // extern "C"
