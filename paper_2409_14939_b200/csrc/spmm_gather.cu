// Layer-0 aggregation over the sampled block graph (fgl_spmm_gather).
//
// Same contract and arithmetic as compute.cu's fgl_spmm (compute.py:115-185:
// h_u = sum_e w_e x_{idx_e}, fp32 product then fp32 add per edge in CSR
// order, empty rows exactly 0) for SHORT rows (<= max_row_len <= 16 edges:
// rows of the block graph hold at most `fanout` edges) gathered straight
// from the HBM feature table.  The kernel software-pipelines the dependent
// index -> row loads of a warp's rows so every lane keeps several 16-byte
// row loads in flight.  Inputs wider than 128 floats
// take fgl_spmm (same results).
#include <algorithm>

#include "common.cuh"

namespace fgl {
namespace {

// ------------------------------------------------ software-pipelined rows --
// One warp per row, lane = 16-byte feature chunk (d <= 128).  Three-stage
// pipeline over the warp's rows so that one row costs about one memory
// latency instead of four: while row i's (<= 8) neighbour rows are being
// gathered, row i+1's column / weight lists and row i+2's offsets are already
// in flight.  Accumulation is in CSR order with a rounded multiply then a
// rounded add (bit-identical to fgl_spmm); rows longer than MAXE take a
// plain in-order loop.
__device__ __forceinline__ float4 fmadd4(float4 acc, float w, float4 x) {
  acc.x = __fadd_rn(acc.x, __fmul_rn(w, x.x));
  acc.y = __fadd_rn(acc.y, __fmul_rn(w, x.y));
  acc.z = __fadd_rn(acc.z, __fmul_rn(w, x.z));
  acc.w = __fadd_rn(acc.w, __fmul_rn(w, x.w));
  return acc;
}

// MAXE = the rows' edge bound (the hop's fanout, rounded up): the gathered
// rows live in MAXE float4 registers, so a small bound leaves registers for
// more resident warps -- more random row reads in flight per SM.
template <int MAXE, int MINB>
__global__ void __launch_bounds__(256, MINB) spmm_pipe_kernel(const int64_t* __restrict__ indptr,
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
    if (lane < n && lane < MAXE) {
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
    float4 x[MAXE];
#pragma unroll
    for (int u = 0; u < MAXE; ++u) {
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
    if (n <= MAXE) {
#pragma unroll
      for (int u = 0; u < MAXE; ++u) {
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
  if (d <= 128) {
    static const int minb = getenv("FGL_PIPE_MINB") ? atoi(getenv("FGL_PIPE_MINB")) : 4;
    auto kern = max_row_len <= 4 ? (minb >= 5 ? spmm_pipe_kernel<4, 5> : spmm_pipe_kernel<4, 4>)
              : max_row_len <= 6 ? (minb >= 5 ? spmm_pipe_kernel<6, 5> : spmm_pipe_kernel<6, 4>)
              : max_row_len <= 8 ? spmm_pipe_kernel<8, 4>
              : max_row_len <= 12 ? spmm_pipe_kernel<12, 2> : spmm_pipe_kernel<16, 2>;
    // rows per warp: 0 = persistent grid (one wave); > 0 = finite CTAs that
    // retire, so a concurrent high-priority stream gets SM slots sooner
    static const int rpw = getenv("FGL_PIPE_RPW") ? atoi(getenv("FGL_PIPE_RPW")) : 8;
    int per_sm = 0;
    if (rpw <= 0 && (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0) != cudaSuccess ||
                     per_sm < 1))
      per_sm = 2;
    const int64_t cap = rpw > 0 ? ceil_div(num_rows, 8LL * rpw) : (int64_t)kNumSMs * per_sm;
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(num_rows, 8), cap));
    const ProfMark pm = prof_begin((cudaStream_t)stream);
    FGL_COUNT_LAUNCH(), kern<<<grid, 256, 0, (cudaStream_t)stream>>>(indptr, col, w, num_rows, col_base, X, ldx, Y,
                                                                    ldy, (d + 3) / 4);
    prof_end(pm, kProfSpmmGather, num_rows, d);
    FGL_LAUNCH_CHECK("spmm_pipe_kernel");
    return FGL_OK;
  }
  return fgl_spmm(indptr, col, w, num_rows, col_base, X, ldx, nullptr, ldx, Y, ldy, d, stream);
}

}  // extern "C"
