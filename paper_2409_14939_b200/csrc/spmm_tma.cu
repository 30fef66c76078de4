// Memory-aware SpMM with neighbour feature rows staged in shared memory by TMA
// gathers (sm_100a `cp.async.bulk.tensor.2d ... tile::gather4`).
//
// Same contract and arithmetic as compute.cu's fgl_spmm (compute.py:115-185:
// h_u = sum_e w_e x_{idx_e}, fp32 product then fp32 add per edge in CSR
// order, empty rows exactly 0) for SHORT rows (<= max_row_len edges, the
// sampled block graph: rows hold at most `fanout` edges).  A CTA walks blocks
// of 16 target rows: one producer warp reads the block's row offsets and
// column indices and issues one gather4 per 4 edges (4 feature rows of d fp32
// each -> shared memory, completion on an mbarrier), three blocks ahead of the
// consumers; 4 consumer warps (4 rows each, lanes over 16-byte chunks)
// accumulate from shared memory in CSR order and store the output rows.  The
// TMA engine keeps ~100 KB of random feature rows in flight per SM without
// tying up registers or warps, which is what the register-staged kernel was
// short of (it was latency bound on dependent index -> row loads).
#include <algorithm>
#include <cstring>

#include "common.cuh"
#include "tcgen05.cuh"

namespace fgl {
namespace {
using namespace tc;


struct StArgs {
  const int64_t* indptr;
  const int32_t* col;
  int64_t col_base;
  const float* w;
  const float* X;
  int64_t ldx;
  int64_t nrows;
  float* Y;
  int64_t ldy;
  int d, row_bytes, g_stride, max_len, buf_bytes;  // g_stride: 4 rows rounded to 128 B
};

// ST_ROWS target rows per block, ST_BUFS blocks in flight per CTA, ST_CONS
// consumer warps (ST_ROWS / ST_CONS rows each)
template <int ST_ROWS, int ST_BUFS, int ST_CONS>
__global__ void __launch_bounds__(32 * (1 + ST_CONS)) spmm_tma_kernel(const __grid_constant__ CUtensorMap tmX, StArgs a) {
  extern __shared__ __align__(128) char smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  char* bufs = smem;
  int64_t* meta = reinterpret_cast<int64_t*>(smem + ST_BUFS * a.buf_bytes);  // [ST_BUFS][ST_ROWS + 1]
  uint64_t* bars = reinterpret_cast<uint64_t*>(meta + ST_BUFS * (ST_ROWS + 2));
  auto bar = [&](int i) { return smem_u32(bars + i); };
  const int FULL = 0, EMPTY = ST_BUFS;
  if (threadIdx.x == 0) {
    for (int i = 0; i < ST_BUFS; ++i) {
      mbar_init_n(bar(FULL + i), 1);
      mbar_init_n(bar(EMPTY + i), ST_CONS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t nblocks = ceil_div(a.nrows, ST_ROWS);
  const int d4 = (a.d + 3) >> 2;
  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) tma_prefetch_desc(&tmX);
    int k = 0;
    for (int64_t bi = blockIdx.x; bi < nblocks; bi += gridDim.x, ++k) {
      const int s = k % ST_BUFS;
      const uint32_t ph = (uint32_t)(k / ST_BUFS) & 1u;
      mbar_wait(bar(EMPTY + s), ph ^ 1u);
      const int64_t r0 = bi * ST_ROWS;
      const int rows = (int)(a.nrows - r0 < ST_ROWS ? a.nrows - r0 : ST_ROWS);
      int64_t* ip = meta + s * (ST_ROWS + 2);
      if (lane <= rows) ip[lane] = a.indptr[r0 + lane];
      __syncwarp();
      const int64_t eb = ip[0], ee = ip[rows];
      const int ne = (int)(ee - eb);
      // a block longer than the staging buffer (rows above max_row_len) is
      // not staged: the consumers read it from global memory (same order)
      const int ng = ((ne + 3) >> 2) * a.g_stride <= a.buf_bytes ? (ne + 3) >> 2 : 0;
      if (lane == 0) {
        if (ng == 0 && ne > 0) ip[ST_ROWS + 1] = 1;  // direct-read flag
        else ip[ST_ROWS + 1] = 0;
        mbar_arrive_expect_tx(bar(FULL + s), (uint32_t)(ng * 4 * a.row_bytes));
      }
      __syncwarp();
      const int32_t first = ne > 0 ? (int32_t)(a.col[eb] - a.col_base) : 0;
      const uint32_t dst0 = smem_u32(bufs + s * a.buf_bytes);
      for (int g = lane; g < ng; g += 32) {
        int32_t r[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int e = 4 * g + t;
          r[t] = e < ne ? (int32_t)(a.col[eb + e] - a.col_base) : first;  // pad: a valid row
        }
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst0 + (uint32_t)(g * a.g_stride)),
            "l"(reinterpret_cast<uint64_t>(&tmX)), "r"(0), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]),
            "r"(bar(FULL + s))
            : "memory");
      }
    }
  } else {
    // ----------------------------------------------------------- consumers
    const int cw = warp - 1;
    int k = 0;
    for (int64_t bi = blockIdx.x; bi < nblocks; bi += gridDim.x, ++k) {
      const int s = k % ST_BUFS;
      mbar_wait(bar(FULL + s), (uint32_t)(k / ST_BUFS) & 1u);
      const int64_t r0 = bi * ST_ROWS;
      const int rows = (int)(a.nrows - r0 < ST_ROWS ? a.nrows - r0 : ST_ROWS);
      const int64_t* ip = meta + s * (ST_ROWS + 2);
      const int64_t eb = ip[0];
      const char* buf = bufs + s * a.buf_bytes;
      const bool direct = ip[ST_ROWS + 1] != 0;
      for (int rr = cw * (ST_ROWS / ST_CONS); rr < (cw + 1) * (ST_ROWS / ST_CONS) && rr < rows; ++rr) {
        const int64_t e0 = ip[rr], e1 = ip[rr + 1];
        for (int c0 = 0; c0 < d4; c0 += 32) {
          const int ch = c0 + lane;
          float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
          for (int64_t e = e0; e < e1; ++e) {
            const float we = __ldg(a.w + e);
            if (ch < d4) {
              const float4 x =
                  direct ? __ldg(reinterpret_cast<const float4*>(a.X + (int64_t)(a.col[e] - a.col_base) * a.ldx) + ch)
                         : lds128(smem_u32(buf + ((e - eb) >> 2) * a.g_stride + ((e - eb) & 3) * a.row_bytes) + 16u * ch);
              acc.x = __fadd_rn(acc.x, __fmul_rn(we, x.x));
              acc.y = __fadd_rn(acc.y, __fmul_rn(we, x.y));
              acc.z = __fadd_rn(acc.z, __fmul_rn(we, x.z));
              acc.w = __fadd_rn(acc.w, __fmul_rn(we, x.w));
            }
          }
          if (ch < d4) reinterpret_cast<float4*>(a.Y + (r0 + rr) * a.ldy)[ch] = acc;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(bar(EMPTY + s));
    }
  }
}

// ------------------------------------------------ software-pipelined rows --
// One warp per row, lane = 16-byte feature chunk (d <= 128).  Three-stage
// pipeline over the warp's rows so that one row costs about one memory
// latency instead of four: while row i's (<= 8) neighbour rows are being
// gathered, row i+1's column / weight lists and row i+2's offsets are already
// in flight.  Accumulation is in CSR order with a rounded multiply then a
// rounded add (bit-identical to fgl_spmm); rows longer than SP_MAXE take a
// plain in-order loop.
__device__ __forceinline__ float4 fmadd4(float4 acc, float w, float4 x) {
  acc.x = __fadd_rn(acc.x, __fmul_rn(w, x.x));
  acc.y = __fadd_rn(acc.y, __fmul_rn(w, x.y));
  acc.z = __fadd_rn(acc.z, __fmul_rn(w, x.z));
  acc.w = __fadd_rn(acc.w, __fmul_rn(w, x.w));
  return acc;
}

constexpr int SP_MAXE = 8;

__global__ void __launch_bounds__(256) spmm_pipe_kernel(const int64_t* __restrict__ indptr,
                                                        const int32_t* __restrict__ col,
                                                        const float* __restrict__ w, int64_t nrows, int64_t col_base,
                                                        const float* __restrict__ X, int64_t ldx,
                                                        float* __restrict__ Y, int64_t ldy, int d4) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (r >= nrows) return;
  auto ip_pair = [&](int64_t row, int64_t& b, int64_t& e) {
    int64_t v = 0;
    if (row < nrows && lane < 2) v = indptr[row + lane];
    b = __shfl_sync(0xffffffffu, v, 0);
    e = __shfl_sync(0xffffffffu, v, 1);
  };
  auto lists = [&](int64_t b, int64_t e, int32_t& cl, float& wl) {
    const int n = (int)(e - b);
    cl = 0;
    wl = 0.f;
    if (lane < n && lane < SP_MAXE) {
      cl = (int32_t)(col[b + lane] - col_base);
      wl = w[b + lane];
    }
  };
  int64_t b0, e0, b1, e1;
  ip_pair(r, b0, e0);
  ip_pair(r + nw, b1, e1);
  int32_t cl0;
  float wl0;
  lists(b0, e0, cl0, wl0);
  while (r < nrows) {
    const int n = (int)(e0 - b0);
    // stage 1: gather row r's neighbour feature rows
    float4 x[SP_MAXE];
#pragma unroll
    for (int u = 0; u < SP_MAXE; ++u) {
      const int32_t c = __shfl_sync(0xffffffffu, cl0, u);
      x[u] = (u < n && lane < d4) ? __ldg(reinterpret_cast<const float4*>(X + (int64_t)c * ldx) + lane)
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    // stage 2 / 3: next row's lists, the row after that's offsets
    int32_t cl1;
    float wl1;
    lists(b1, e1, cl1, wl1);
    int64_t b2, e2;
    ip_pair(r + 2 * nw, b2, e2);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (n <= SP_MAXE) {
#pragma unroll
      for (int u = 0; u < SP_MAXE; ++u) {
        const float wk = __shfl_sync(0xffffffffu, wl0, u);
        if (u < n) acc = fmadd4(acc, wk, x[u]);
      }
    } else {
      for (int64_t e = b0; e < e0; ++e) {
        const int32_t c = (int32_t)(col[e] - col_base);
        const float wk = w[e];
        if (lane < d4) acc = fmadd4(acc, wk, __ldg(reinterpret_cast<const float4*>(X + (int64_t)c * ldx) + lane));
      }
    }
    if (lane < d4) reinterpret_cast<float4*>(Y + r * ldy)[lane] = acc;
    r += nw;
    b0 = b1; e0 = e1; cl0 = cl1; wl0 = wl1;
    b1 = b2; e1 = e2;
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<EncodeTiledFn>(f);
    return (EncodeTiledFn) nullptr;
  }();
  return fn;
}

template <int ROWS, int BUFS, int CONS>
int launch_gather(const CUtensorMap& m, StArgs a, cudaStream_t st) {
  const int max_edges = (ROWS * std::max(a.max_len, 1) + 3) / 4 * 4;
  a.buf_bytes = max_edges / 4 * a.g_stride;
  const int smem = 128 + BUFS * a.buf_bytes + 8 * BUFS * (ROWS + 2) + 8 * 2 * BUFS;
  if (smem > 227 * 1024) {
    set_error("fgl_spmm_gather: staging buffers exceed shared memory");
    return FGL_E_UNSUPPORTED;
  }
  auto kern = spmm_tma_kernel<ROWS, BUFS, CONS>;
  static int attr_set = 0;
  if (smem > attr_set) {
    FGL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_set = smem;
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * (1 + CONS), smem) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  const int64_t nblocks = ceil_div(a.nrows, ROWS);
  const int grid = (int)std::min<int64_t>(nblocks, (int64_t)per_sm * kNumSMs);
  FGL_COUNT_LAUNCH(), kern<<<grid, 32 * (1 + CONS), smem, st>>>(m, a);
  FGL_LAUNCH_CHECK("spmm_tma_kernel");
  return FGL_OK;
}

}  // namespace
}  // namespace fgl

using namespace fgl;

extern "C" {

int fgl_spmm_gather(const int64_t* indptr, const int32_t* col, const float* w, int64_t num_rows, int64_t col_base,
                    const float* X, int64_t ldx, int64_t x_rows, float* Y, int64_t ldy, int32_t d,
                    int32_t max_row_len, void* stream) {
  if ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(Y)) & 15) {
    set_error("fgl_spmm_gather: feature pointers must be 16-byte aligned");
    return FGL_E_INVALID;
  }
  if (num_rows < 0 || d < 1 || d > 256 || ldx > 256 || !indptr || !Y || !X || ldy < d || ldx < d || (ldx % 4) || (ldy % 4) ||
      max_row_len < 0 || x_rows < 1) {
    set_error("fgl_spmm_gather: bad arguments");
    return FGL_E_INVALID;
  }
  if (max_row_len > 16) {
    set_error("fgl_spmm_gather: rows longer than 16 edges use fgl_spmm");
    return FGL_E_UNSUPPORTED;
  }
  if (num_rows == 0) return FGL_OK;
  static const int use_tma = getenv("FGL_GATHER_TMA") ? atoi(getenv("FGL_GATHER_TMA")) : 0;
  if (!use_tma && d <= 128) {
    static int per_sm = 0;
    if (!per_sm && (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, spmm_pipe_kernel, 256, 0) != cudaSuccess ||
                    per_sm < 1))
      per_sm = 2;
    // rows per warp: 0 = persistent grid (one wave); > 0 = finite CTAs that
    // retire, so a concurrent high-priority stream gets SM slots sooner
    static const int rpw = getenv("FGL_PIPE_RPW") ? atoi(getenv("FGL_PIPE_RPW")) : 8;
    const int64_t cap = rpw > 0 ? ceil_div(num_rows, 8LL * rpw) : (int64_t)kNumSMs * per_sm;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(num_rows, 8), cap));
    FGL_COUNT_LAUNCH(), spmm_pipe_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(indptr, col, w, num_rows, col_base, X,
                                                                                ldx, Y, ldy, (d + 3) / 4);
    FGL_LAUNCH_CHECK("spmm_pipe_kernel");
    return FGL_OK;
  }
  EncodeTiledFn fn = encode_fn();
  if (!fn) {
    set_error("fgl_spmm_gather: cuTensorMapEncodeTiled unavailable");
    return FGL_E_CUDA;
  }
  // encoding a map costs a few microseconds of host time; the trainer calls
  // this with the same feature table every batch, so keep the last few maps
  struct MapCache { const float* X; int64_t ldx, rows; CUtensorMap m; };
  static thread_local MapCache cache[4];
  static thread_local int cache_next = 0;
  const CUtensorMap* mp = nullptr;
  for (auto& c : cache)
    if (c.X == X && c.ldx == ldx && c.rows == x_rows) mp = &c.m;
  if (!mp) {
    MapCache& c = cache[cache_next];
    cache_next = (cache_next + 1) % 4;
    std::memset(&c, 0, sizeof(c));
    cuuint64_t dims[2] = {(cuuint64_t)ldx, (cuuint64_t)x_rows};
    cuuint64_t strides[1] = {(cuuint64_t)ldx * 4};
    cuuint32_t box[2] = {(cuuint32_t)ldx, 1};
    cuuint32_t es[2] = {1, 1};
    if (ldx > 256 || fn(&c.m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(X), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      c.X = nullptr;
      set_error("fgl_spmm_gather: tensor map encode failed (ld %lld)", (long long)ldx);
      return FGL_E_UNSUPPORTED;
    }
    c.X = X; c.ldx = ldx; c.rows = x_rows;
    mp = &c.m;
  }
  StArgs a;
  a.indptr = indptr; a.col = col; a.col_base = col_base; a.w = w; a.X = X; a.ldx = ldx; a.nrows = num_rows;
  a.Y = Y; a.ldy = ldy; a.d = d;
  a.row_bytes = (int)(ldx * 4);
  a.max_len = max_row_len;
  a.g_stride = (4 * a.row_bytes + 127) / 128 * 128;  // gather4 destinations are 128-byte aligned
  const int rc = launch_gather<16, 3, 4>(*mp, a, (cudaStream_t)stream);
  if (rc) return rc;
  return FGL_OK;
}

}  // extern "C"
