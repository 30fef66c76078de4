// Model compute of one mini-batch on the sampled block graph (sm_100a).
//
//  * fgl_spmm      -- Memory-Aware CSR aggregation, compute.py:115-195: one
//                     row per lane group, neighbour (col, w) lists staged in
//                     registers and broadcast with warp shuffles, 16-byte
//                     feature loads, fp32 accumulation in CSR order with a
//                     rounded multiply then a rounded add (no FMA) -- bit-
//                     identical to the reference; backward = the same kernel
//                     on the stable transpose (compute.py:188-195).
//  * fgl_dense_fwd -- act(h @ W + b) (compute.py:198-216), fused bias + ReLU.
//  * fgl_dense_bwd -- dz = dx * (x_out > 0), dW = h^T dz (deterministic
//                     split-K), db = sum dz, dh = dz W^T (trainer.py:212-228).
//  * fgl_softmax_xent -- fp64 softmax cross entropy over the seed rows
//                     (trainer.py:198-209) writing dlogits/B as f32.
//  * fgl_sgd       -- w -= f32(lr) * g (trainer.py:321-323).
#include <algorithm>

#include "common.cuh"

namespace fgl {
namespace {

// --------------------------------------------------------------- spmm -----
__device__ __forceinline__ float4 fmadd4(float4 acc, float w, float4 x) {
  acc.x = __fadd_rn(acc.x, __fmul_rn(w, x.x));
  acc.y = __fadd_rn(acc.y, __fmul_rn(w, x.y));
  acc.z = __fadd_rn(acc.z, __fmul_rn(w, x.z));
  acc.w = __fadd_rn(acc.w, __fmul_rn(w, x.w));
  return acc;
}

template <int L, int CPL, int U = 4>
__global__ void __launch_bounds__(256) spmm_kernel(
    const int64_t* __restrict__ indptr, const int32_t* __restrict__ col,
    const float* __restrict__ w, int64_t nrows, int64_t col_base, const float* __restrict__ X,
    int64_t ldx, const float* __restrict__ self_x, int64_t ld_self, float* __restrict__ Y,
    int64_t ldy, int d4) {
  constexpr int G = 32 / L;  // rows per warp
  const int lane = threadIdx.x & 31;
  const int grp = lane / L, g = lane % L;
  const unsigned gmask = (L == 32) ? 0xffffffffu : (((1u << L) - 1u) << (grp * L));
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t rbase = warp * G; rbase < nrows; rbase += nwarps * G) {
    const int64_t r = rbase + grp;
    const bool live = r < nrows;
    const int64_t e0 = live ? indptr[r] : 0, e1 = live ? indptr[r + 1] : 0;
    float4 acc[CPL];
#pragma unroll
    for (int q = 0; q < CPL; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t e = e0; e < e1; e += L) {
      const int64_t me = e + g;
      const int32_t cl = me < e1 ? (int32_t)(col[me] - col_base) : 0;
      const float wl = me < e1 ? w[me] : 0.f;
      const int n = (int)(e1 - e < L ? e1 - e : L);
      int k = 0;
      for (; k + U <= n; k += U) {  // U neighbour rows in flight
        int32_t c[U];
        float wk[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          c[u] = __shfl_sync(gmask, cl, k + u, L);
          wk[u] = __shfl_sync(gmask, wl, k + u, L);
        }
        float4 x[U][CPL];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const float4* xr = reinterpret_cast<const float4*>(X + (int64_t)c[u] * ldx);
#pragma unroll
          for (int q = 0; q < CPL; ++q) {
            const int ch = g + q * L;
            x[u][q] = ch < d4 ? __ldg(xr + ch) : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int q = 0; q < CPL; ++q) acc[q] = fmadd4(acc[q], wk[u], x[u][q]);
      }
      for (; k < n; ++k) {
        const int32_t c = __shfl_sync(gmask, cl, k, L);
        const float wk = __shfl_sync(gmask, wl, k, L);
        const float4* xr = reinterpret_cast<const float4*>(X + (int64_t)c * ldx);
#pragma unroll
        for (int q = 0; q < CPL; ++q) {
          const int ch = g + q * L;
          if (ch < d4) acc[q] = fmadd4(acc[q], wk, __ldg(xr + ch));
        }
      }
    }
    if (live) {
      float4* yr = reinterpret_cast<float4*>(Y + r * ldy);
#pragma unroll
      for (int q = 0; q < CPL; ++q) {
        const int ch = g + q * L;
        if (ch < d4) {
          float4 v = acc[q];
          if (self_x) {  // GIN: h = aggregate + x, one rounded add (trainer.py:189-190)
            const float4 s = reinterpret_cast<const float4*>(self_x + r * ld_self)[ch];
            v.x = __fadd_rn(v.x, s.x); v.y = __fadd_rn(v.y, s.y);
            v.z = __fadd_rn(v.z, s.z); v.w = __fadd_rn(v.w, s.w);
          }
          yr[ch] = v;
        }
      }
    }
  }
}

// Rows of <= 32 float4 chunks (d <= 128): W threads per row (16 for d <= 64,
// 32 above), lane = 16-byte chunk; the row's (col, w) pairs are loaded once
// per W edges and broadcast by shuffles; neighbour rows are gathered G at a
// time (G loads in flight per lane, then G multiply-adds in CSR order:
// bit-identical to spmm_kernel).  At most 32 registers, so 64 warps per SM
// keep their random row reads in flight -- what a bare random-row read needs
// to approach its ceiling (tools/probes/row_gather_probe.cu: 5.6 TB/s for
// 400-byte rows at 64 warps / SM, 4.6 TB/s at 32).  Serves the layer-0
// aggregation (fgl_spmm_gather: rows of <= fanout edges from the HBM feature
// table), the upper layers and the transposed (~1-edge rows) backward
// aggregations.
// xids (fgl_spmm_ids): source row c reads X row xids[c] and the root term of
// output row r is X row xids[self_base + r] (GIN / SAGE layer 0 straight from
// the HBM feature table, no x0 block); the arithmetic is unchanged.
template <int G, int W>
__global__ void __launch_bounds__(256, 8) spmm_lean_kernel(
    const int64_t* __restrict__ indptr, const int32_t* __restrict__ col, const float* __restrict__ w,
    int64_t nrows, int64_t col_base, const float* __restrict__ X, int64_t ldx, const float* __restrict__ self_x,
    int64_t ld_self, float* __restrict__ Y, int64_t ldy, int d4, const int32_t* __restrict__ xids = nullptr,
    int64_t self_base = 0) {
  const int lane = threadIdx.x & (W - 1);
  const unsigned mask = W == 32 ? 0xffffffffu : (0xffffu << (threadIdx.x & 16));
  const int64_t ng = ((int64_t)gridDim.x * blockDim.x) / W;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / W; r < nrows; r += ng) {
    int64_t v = 0;
    if (lane < 2) v = indptr[r + lane];
    const int64_t b = __shfl_sync(mask, v, 0, W);
    const int n = (int)(__shfl_sync(mask, v, 1, W) - b);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int u0 = 0; u0 < n; u0 += W) {
      const int m = n - u0 < W ? n - u0 : W;
      int32_t cl = 0;
      float wl = 0.f;
      if (lane < m) {
        cl = (int32_t)(col[b + u0 + lane] - col_base);
        if (xids) cl = __ldg(xids + cl);
        wl = w[b + u0 + lane];
      }
      for (int u = 0; u < m; u += G) {
        float4 x[G];
#pragma unroll
        for (int k = 0; k < G; ++k) {
          const int32_t c = __shfl_sync(mask, cl, (u + k) & (W - 1), W);
          x[k] = (u + k < m && lane < d4) ? __ldg(reinterpret_cast<const float4*>(X + (int64_t)c * ldx) + lane)
                                          : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int k = 0; k < G; ++k) {
          const float wk = __shfl_sync(mask, wl, (u + k) & (W - 1), W);
          if (u + k < m) acc = fmadd4(acc, wk, x[k]);
        }
      }
    }
    if (lane < d4) {
      if (self_x) {  // GIN / SAGE root term: h = aggregate + x, one rounded add (trainer.py:189-190)
        const int64_t sr = xids ? (int64_t)__ldg(xids + self_base + r) : r;
        const float4 sx = reinterpret_cast<const float4*>(self_x + sr * ld_self)[lane];
        acc.x = __fadd_rn(acc.x, sx.x); acc.y = __fadd_rn(acc.y, sx.y);
        acc.z = __fadd_rn(acc.z, sx.z); acc.w = __fadd_rn(acc.w, sx.w);
      }
      reinterpret_cast<float4*>(Y + r * ldy)[lane] = acc;
    }
  }
}

void launch_spmm_lean(const int64_t* indptr, const int32_t* col, const float* w, int64_t nrows, int64_t col_base,
                      const float* X, int64_t ldx, const float* self_x, int64_t ld_self, float* Y, int64_t ldy,
                      int d4, cudaStream_t st, int64_t max_ctas = (int64_t)kNumSMs * 8,
                      const int32_t* xids = nullptr, int64_t self_base = 0) {
  const int per_cta = d4 <= 16 ? 16 : 8;  // rows per 256-thread CTA
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(nrows, per_cta), max_ctas));
  if (d4 <= 16)
    FGL_COUNT_LAUNCH(), spmm_lean_kernel<2, 16><<<grid, 256, 0, st>>>(indptr, col, w, nrows, col_base, X, ldx, self_x,
                                                                     ld_self, Y, ldy, d4, xids, self_base);
  else
    FGL_COUNT_LAUNCH(), spmm_lean_kernel<2, 32><<<grid, 256, 0, st>>>(indptr, col, w, nrows, col_base, X, ldx, self_x,
                                                                     ld_self, Y, ldy, d4, xids, self_base);
}

template <int L, int CPL, int U = 4>
void launch_spmm(const int64_t* indptr, const int32_t* col, const float* w, int64_t nrows,
                 int64_t col_base, const float* X, int64_t ldx, const float* self_x,
                 int64_t ld_self, float* Y, int64_t ldy, int d4, cudaStream_t st) {
  constexpr int G = 32 / L;
  const int64_t warps = ceil_div(nrows, G);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(warps, 8), 148 * 16));
  FGL_COUNT_LAUNCH(), spmm_kernel<L, CPL, U><<<grid, 256, 0, st>>>(indptr, col, w, nrows, col_base, X, ldx, self_x,
                                            ld_self, Y, ldy, d4);
}

// --------------------------------------------------------------- dense ----
// C[M, N] = A[M, K] @ B + bias  (B is [K, N] row-major, or B^T stored as [N, K]
// when b_trans); optional ReLU.  64x64 output tile per CTA, 256 threads with
// 4x4 register micro-tiles, K staged through shared memory in chunks of 32.
constexpr int BM = 64, BN = 64, BK = 32;

__global__ void __launch_bounds__(256) gemm_kernel(
    const float* __restrict__ A, int64_t lda, const float* __restrict__ B, int64_t ldb, int b_trans,
    const float* __restrict__ bias, float* __restrict__ C, int64_t ldc, int64_t M, int N, int K,
    int relu, const float* __restrict__ amask, int64_t ldm) {
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  const int64_t m0 = blockIdx.x * (int64_t)BM;
  const int n0 = blockIdx.y * BN;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += BK) {
    // A tile: 64 rows x 32 k, stored k-major in smem
    for (int i = tid; i < BM * BK; i += 256) {
      const int r = i / BK, k = i % BK;
      const int64_t gr = m0 + r;
      float v = 0.f;
      if (gr < M && k0 + k < K) {
        v = A[gr * lda + k0 + k];
        if (amask && !(amask[gr * ldm + k0 + k] > 0.f)) v = 0.f;  // relu mask of dz
      }
      As[k][r] = v;
    }
    for (int i = tid; i < BK * BN; i += 256) {
      const int k = i / BN, n = i % BN;
      float v = 0.f;
      if (k0 + k < K && n0 + n < N) v = b_trans ? B[(int64_t)(n0 + n) * ldb + k0 + k] : B[(int64_t)(k0 + k) * ldb + n0 + n];
      Bs[k][n] = v;
    }
    __syncthreads();
#pragma unroll 8
    for (int k = 0; k < BK; ++k) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[k][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[k][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = __fmaf_rn(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t r = m0 + ty * 4 + i;
    if (r >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = n0 + tx * 4 + j;
      if (c >= N) continue;
      float v = acc[i][j];
      if (bias) v = __fadd_rn(v, bias[c]);
      if (relu) v = v > 0.f ? v : 0.f;
      C[r * ldc + c] = v;
    }
  }
}

// Partial [dW; db] = [H | 1]^T dZ over a fixed row chunk per CTA (the bias
// gradient is the extra "ones" column of H, k == K).  Output tile 128 (k) x
// 64 (n) per CTA; 256 threads each own an 8 x 4 register micro tile; rows are
// streamed through shared memory 32 at a time with 16-byte loads.
constexpr int WK = 128, WN = 64, WR = 32;

__global__ void __launch_bounds__(256) wgrad_partial_kernel(
    const float* __restrict__ A, int64_t lda, const float* __restrict__ dZ, int64_t ldz,
    const float* __restrict__ zmask, int64_t ldm, int64_t M, int K, int N, int64_t rows_per_cta,
    float* __restrict__ part, int vec) {
  __shared__ __align__(16) float As[WR][WK];
  __shared__ __align__(16) float Zs[WR][WN];
  const int tid = threadIdx.x;
  const int tn = tid % 16, tk = tid / 16;  // n = tn*4..+3, k = tk*8..+7
  const int k0 = blockIdx.y * WK, n0 = blockIdx.z * WN;
  const int KE = K + 1;  // + ones column -> db
  const int64_t r_begin = blockIdx.x * rows_per_cta;
  const int64_t r_end = min(M, r_begin + rows_per_cta);
  float acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  for (int64_t r0 = r_begin; r0 < r_end; r0 += WR) {
    // A tile: 32 rows x 128 k (4 float4 per thread)
    for (int i = tid; i < WR * (WK / 4); i += 256) {
      const int rr = i / (WK / 4), kq = (i % (WK / 4)) * 4;
      const int64_t r = r0 + rr;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (r < r_end) {
        const int k = k0 + kq;
        if (vec && k + 3 < K) {
          v = *reinterpret_cast<const float4*>(A + r * lda + k);
        } else {
          float t[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) t[q] = (k + q < K) ? A[r * lda + k + q] : (k + q == K ? 1.f : 0.f);
          v = make_float4(t[0], t[1], t[2], t[3]);
        }
      }
      *reinterpret_cast<float4*>(&As[rr][kq]) = v;
    }
    // dZ tile: 32 rows x 64 n, ReLU-masked by the layer output
    for (int i = tid; i < WR * (WN / 4); i += 256) {
      const int rr = i / (WN / 4), nq = (i % (WN / 4)) * 4;
      const int64_t r = r0 + rr;
      float t[4] = {0.f, 0.f, 0.f, 0.f};
      if (r < r_end) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int n = n0 + nq + q;
          if (n < N) {
            float v = dZ[r * ldz + n];
            if (zmask && !(zmask[r * ldm + n] > 0.f)) v = 0.f;
            t[q] = v;
          }
        }
      }
      *reinterpret_cast<float4*>(&Zs[rr][nq]) = make_float4(t[0], t[1], t[2], t[3]);
    }
    __syncthreads();
#pragma unroll 4
    for (int rr = 0; rr < WR; ++rr) {
      const float4 a0 = *reinterpret_cast<const float4*>(&As[rr][tk * 8]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[rr][tk * 8 + 4]);
      const float4 z = *reinterpret_cast<const float4*>(&Zs[rr][tn * 4]);
      const float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      const float zz[4] = {z.x, z.y, z.z, z.w};
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = __fmaf_rn(a[i], zz[j], acc[i][j]);
    }
    __syncthreads();
  }
  float* pw = part + (int64_t)blockIdx.x * KE * N;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int k = k0 + tk * 8 + i;
    if (k >= KE) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tn * 4 + j;
      if (n < N) pw[(int64_t)k * N + n] = acc[i][j];
    }
  }
}

// Sum partials over chunks in a fixed order (deterministic): each CTA owns 32
// outputs; 8 thread groups sum interleaved chunks, then a fixed-order combine.
// dW / db from per-CTA partials, summed in a fixed order (deterministic).
// kp1 == 0: partial element i is output i (dW row-major, then db); kp1 = K+1:
// partials are stored feature-major ([N][K+1], coalesced tensor-core
// epilogue), element j = n*(K+1) + k is output k*N + n (k == K: db[n]).
// kp1 > 0 (tensor-core partials, feature-major [N][kp1]): element (nn, k) ->
// out[k * ldo + col0 + nn] for k < kp1 - 1 (dW rows), out2[col0 + nn] for the
// last (db).  kp1 == 0 (SIMT partials): element i -> out[i] / out2[i - split].
__global__ void reduce_partials_kernel(const float* __restrict__ part, int chunks, int64_t n,
                                       float* __restrict__ out, int64_t split, float* __restrict__ out2, int kp1,
                                       int64_t ldo = 0, int64_t col0 = 0) {
  __shared__ float sm[8][33];
  const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const int64_t i = blockIdx.x * 32 + lane;
  float s = 0.f;
  if (i < n) {
    const float* q = part + i;
    int c = grp;
    for (; c + 24 < chunks; c += 32) {  // four independent loads in flight
      const float a = q[(int64_t)c * n], b = q[(int64_t)(c + 8) * n], d = q[(int64_t)(c + 16) * n],
                  e = q[(int64_t)(c + 24) * n];
      s = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(s, a), b), d), e);
    }
    for (; c < chunks; c += 8) s = __fadd_rn(s, q[(int64_t)c * n]);
  }
  sm[grp][lane] = s;
  __syncthreads();
  if (grp == 0 && i < n) {
    float t = sm[0][lane];
#pragma unroll
    for (int g = 1; g < 8; ++g) t = __fadd_rn(t, sm[g][lane]);
    if (kp1 > 0) {
      const int64_t nn = i / kp1, k = i - nn * kp1;
      if (k < kp1 - 1) out[k * ldo + col0 + nn] = t;
      else out2[col0 + nn] = t;
    } else {
      if (i < split) out[i] = t; else out2[i - split] = t;
    }
  }
}

// --------------------------------------------------------------- loss -----
__global__ void softmax_xent_kernel(const float* __restrict__ logits, int64_t ldl,
                                    const int32_t* __restrict__ rows, int64_t row_base,
                                    const int32_t* __restrict__ seed_ids,
                                    const int64_t* __restrict__ labels, int64_t B, int C,
                                    float* __restrict__ dlog, int64_t ldd,
                                    double* __restrict__ loss_part) {
  // one warp per seed row; fp64 throughout (trainer.py:198-209)
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double lsum = 0.0;
  for (int64_t i = warp; i < B; i += nwarps) {
    const int64_t r = rows[i] - row_base;
    const float* z = logits + r * ldl;
    double mx = -INFINITY;
    for (int c = lane; c < C; c += 32) mx = fmax(mx, (double)z[c]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    double se = 0.0;
    for (int c = lane; c < C; c += 32) se += exp((double)z[c] - mx);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
    const int64_t y = labels[seed_ids ? (int64_t)seed_ids[i] : i];
    for (int c = lane; c < C; c += 32) {
      const double p = exp((double)z[c] - mx) / se;
      const double g = (c == y ? p - 1.0 : p) / (double)B;
      dlog[r * ldd + c] = (float)g;
      if (c == y) lsum += -log(p + 1e-30);
    }
  }
  lsum = warp_sum(lsum);
  if (lane == 0) loss_part[warp] = lsum;
}

__global__ void sum_doubles_kernel(const double* __restrict__ v, int n, double* out) {
  __shared__ double sm[33];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += v[i];
  s = block_sum(s, sm);
  if (threadIdx.x == 0) *out = s;
}

__global__ void sgd_kernel(float* __restrict__ p, const float* __restrict__ g, int64_t n, float lr) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = __fsub_rn(p[i], __fmul_rn(lr, g[i]));
}

__global__ void fill_rows_kernel(float* __restrict__ Y, int64_t ldy, int64_t nrows, int d,
                                 const float* __restrict__ rowval, int relu) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nrows * d;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / d;
    const int c = (int)(i % d);
    float v = rowval ? rowval[c] : 0.f;
    if (relu) v = v > 0.f ? v : 0.f;
    Y[r * ldy + c] = v;
  }
}

// Top model layer in one launch (compact GCN: the layer's rows are exactly
// the batch's seeds): logits Y = H W + b, fp64 softmax cross entropy
// (trainer.py:198-209) with dY = (p - onehot)/B, dH = dY W^T, and per-CTA
// partials of dW = H^T dY, db = sum dY and of the loss (reduced off the
// critical chain).  Replaces the dense forward, the softmax, the loss sum
// and the dgrad launches of the top layer.  8 seeds per CTA, din <= 64, C <= CW
// (64: products / Reddit; 192: papers' 172 classes); fp32 FMA in a fixed order
// (within 1e-5), fp64 loss.  W, W^T and the logits live in dynamic shared
// memory ((128 CW + 8 CW) floats).
constexpr int TOP_ROWS = 8;  // one warp per seed row in the softmax; 128 CTAs for a 1024-seed batch

template <int CW>
__global__ void __launch_bounds__(256) top_layer_kernel(
    const float* __restrict__ H, int64_t ldh, const int32_t* __restrict__ rows, int64_t row_base,
    const int32_t* __restrict__ seed_ids, const int64_t* __restrict__ labels, int64_t B, int din, int C,
    const float* __restrict__ W, const float* __restrict__ b, float* __restrict__ dH, int64_t lddh,
    float* __restrict__ part, double* __restrict__ loss_part, const int64_t* __restrict__ agg_indptr,
    const int32_t* __restrict__ agg_col, const float* __restrict__ agg_w, int64_t agg_col_base) {
  extern __shared__ __align__(16) float top_dyn[];
  float (*Ws)[CW] = reinterpret_cast<float (*)[CW]>(top_dyn);                 // [64][CW]: [k][c]
  float (*WsT)[64] = reinterpret_cast<float (*)[64]>(top_dyn + 64 * CW);      // [CW][64]: [c][k]
  float (*Ys)[CW] = reinterpret_cast<float (*)[CW]>(top_dyn + 128 * CW);      // [TOP_ROWS][CW]
  __shared__ __align__(16) float Hs[TOP_ROWS][68];
  __shared__ double lsum[TOP_ROWS];
  constexpr int NWV = 64 * CW / 256;  // staged weight elements per thread
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int64_t i0 = (int64_t)blockIdx.x * TOP_ROWS;
  const int nr = (int)(B - i0 < TOP_ROWS ? B - i0 : TOP_ROWS);
  // every global load of the staging is issued before the first shared
  // store (one memory latency, not one per element)
  float wv[NWV];
#pragma unroll
  for (int u = 0; u < NWV; ++u) {
    const int i = t + 256 * u, k = i / CW, c = i % CW;
    wv[u] = (k < din && c < C) ? __ldg(W + (int64_t)k * C + c) : 0.f;
  }
  if (agg_indptr) {
    // H = A X for this CTA's rows, gathered here (one warp per row, float4
    // lanes, CSR order with a rounded multiply then a rounded add: the
    // arithmetic of fgl_spmm, bit-identical); H never leaves the chip
    const int rw = warp, ln = lane & 15, d4 = (din + 3) >> 2;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    if (rw < nr) {
      const int64_t r = rows[i0 + rw] - row_base;
      const int64_t e0 = agg_indptr[r], e1 = agg_indptr[r + 1];
      for (int64_t e = e0; e < e1; e += 4) {
        const int n = (int)(e1 - e < 4 ? e1 - e : 4);
        int32_t cc[4];
        float ww[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          cc[u] = u < n ? (int32_t)(__ldg(agg_col + e + u) - agg_col_base) : 0;
          ww[u] = u < n ? __ldg(agg_w + e + u) : 0.f;
        }
        float4 x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
          x[u] = (u < n && lane < 16 && ln < d4)
                     ? __ldg(reinterpret_cast<const float4*>(H + (int64_t)cc[u] * ldh) + ln)
                     : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (u < n) acc = fmadd4(acc, ww[u], x[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < NWV; ++u) {
      const int i = t + 256 * u, k = i / CW, c = i % CW;
      Ws[k][c] = wv[u];
      WsT[c][k] = wv[u];
    }
    for (int k = lane; k < 68; k += 32) Hs[rw][k] = (rw < nr && k == din) ? 1.f : 0.f;
    __syncwarp();
    if (lane < 16 && ln < d4 && rw < nr) {
      Hs[rw][4 * ln] = acc.x;
      if (4 * ln + 1 < din) Hs[rw][4 * ln + 1] = acc.y;
      if (4 * ln + 2 < din) Hs[rw][4 * ln + 2] = acc.z;
      if (4 * ln + 3 < din) Hs[rw][4 * ln + 3] = acc.w;
    }
  } else {
    float hv3[3];
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      const int i = t + 256 * u, r = i / 68, k = i - r * 68;
      float v = 0.f;
      if (i < TOP_ROWS * 68 && r < nr) {
        if (k < din) v = __ldg(H + (int64_t)(rows[i0 + r] - row_base) * ldh + k);
        else if (k == din) v = 1.f;
      }
      hv3[u] = v;
    }
#pragma unroll
    for (int u = 0; u < NWV; ++u) {
      const int i = t + 256 * u, k = i / CW, c = i % CW;
      Ws[k][c] = wv[u];
      WsT[c][k] = wv[u];
    }
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      const int i = t + 256 * u;
      if (i < TOP_ROWS * 68) Hs[i / 68][i % 68] = hv3[u];
    }
  }
  __syncthreads();
  const int rr = warp;  // every phase: warp = seed row of the CTA
  // logits: lane -> columns 64 j + 2 lane, 64 j + 2 lane + 1
#pragma unroll
  for (int j = 0; j < CW / 64; ++j) {
    const int c0 = 64 * j + 2 * lane;
    float a0 = 0.f, a1 = 0.f;
    for (int k = 0; k < din; ++k) {
      const float h = Hs[rr][k];
      const float2 w = *reinterpret_cast<const float2*>(&Ws[k][c0]);
      a0 = __fmaf_rn(h, w.x, a0);
      a1 = __fmaf_rn(h, w.y, a1);
    }
    Ys[rr][c0] = c0 < C ? (b ? __fadd_rn(a0, b[c0]) : a0) : 0.f;
    Ys[rr][c0 + 1] = c0 + 1 < C ? (b ? __fadd_rn(a1, b[c0 + 1]) : a1) : 0.f;
  }
  __syncwarp();
  // softmax cross entropy of the warp's row (fp64); Ys <- dY
  {
    double l = 0.0;
    if (rr < nr) {
      double mx = -INFINITY;
      for (int c = lane; c < C; c += 32) mx = fmax(mx, (double)Ys[rr][c]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      double ex[CW / 32];
      double se = 0.0;
#pragma unroll
      for (int u = 0; u < CW / 32; ++u) {
        ex[u] = 0.0;
        const int c = lane + 32 * u;
        if (c < C) { ex[u] = exp((double)Ys[rr][c] - mx); se += ex[u]; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
      const int64_t y = labels[seed_ids ? (int64_t)seed_ids[i0 + rr] : i0 + rr];
      __syncwarp();
#pragma unroll
      for (int u = 0; u < CW / 32; ++u) {
        const int c = lane + 32 * u;
        if (c < C) {
          const double pc = ex[u] / se;
          if (c == y) l += -log(pc + 1e-30);
          Ys[rr][c] = (float)((c == y ? pc - 1.0 : pc) / (double)B);
        }
      }
      l = warp_sum(l);
    } else {
      for (int c = lane; c < CW; c += 32) Ys[rr][c] = 0.f;
    }
    if (lane == 0) lsum[rr] = l;
  }
  __syncwarp();
  // dH = dY W^T: lane -> input features 2 lane, 2 lane + 1
  if (rr < nr) {
    const int k0 = 2 * lane;
    float a0 = 0.f, a1 = 0.f;
    for (int c = 0; c < C; ++c) {
      const float g = Ys[rr][c];
      const float2 w = *reinterpret_cast<const float2*>(&WsT[c][k0]);
      a0 = __fmaf_rn(g, w.x, a0);
      a1 = __fmaf_rn(g, w.y, a1);
    }
    float* out = dH + (int64_t)(rows[i0 + rr] - row_base) * lddh;
    if (k0 < din) out[k0] = a0;
    if (k0 + 1 < din) out[k0 + 1] = a1;
  }
  __syncthreads();
  // dW / db partials [(din + 1) x C] (row din = db): thread = 4 k x 4 c block
  {
    float* pp = part + (int64_t)blockIdx.x * (din + 1) * C;
    const int kb = (din + 1 + 3) >> 2, cb = (C + 3) >> 2;
    for (int blk = t; blk < kb * cb; blk += 256) {
      const int k0 = (blk / cb) * 4, c0 = (blk % cb) * 4;
      float a[4][4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) a[u][v] = 0.f;
      for (int r = 0; r < nr; ++r) {
        const float4 h = *reinterpret_cast<const float4*>(&Hs[r][k0]);
        const float4 g = *reinterpret_cast<const float4*>(&Ys[r][c0]);
        const float hv[4] = {h.x, h.y, h.z, h.w}, gv[4] = {g.x, g.y, g.z, g.w};
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int v = 0; v < 4; ++v) a[u][v] = __fmaf_rn(hv[u], gv[v], a[u][v]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v)
          if (k0 + u <= din && c0 + v < C) pp[(int64_t)(k0 + u) * C + c0 + v] = a[u][v];
    }
  }
  if (t == 0) {
    double l = 0.0;
    for (int r = 0; r < TOP_ROWS; ++r) l += lsum[r];
    loss_part[blockIdx.x] = l;
  }
}

// partials -> dW / db and the batch loss (fp64).  A CTA owns 32 outputs; its
// 8 warps sum interleaved chunks (c = warp mod 8, two independent chains
// each), combined in a fixed order: deterministic, and 8x fewer dependent L2
// round trips per thread than one thread per output (12 -> ~3 us)
__global__ void top_reduce_kernel(const float* __restrict__ part, int chunks, int64_t outs, float* __restrict__ dW,
                                  int64_t split, float* __restrict__ db, const double* __restrict__ loss_part,
                                  double* __restrict__ loss_sum) {
  __shared__ float sm[8][33];
  const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
  const int64_t i = blockIdx.x * 32 + lane;
  float s = 0.f;
  if (i < outs) {
    float s1 = 0.f;
    int c = grp;
    for (; c + 8 < chunks; c += 16) {
      s = __fadd_rn(s, part[(int64_t)c * outs + i]);
      s1 = __fadd_rn(s1, part[(int64_t)(c + 8) * outs + i]);
    }
    if (c < chunks) s = __fadd_rn(s, part[(int64_t)c * outs + i]);
    s = __fadd_rn(s, s1);
  }
  sm[grp][lane] = s;
  __syncthreads();
  if (grp == 0 && i < outs) {
    float t = sm[0][lane];
#pragma unroll
    for (int g = 1; g < 8; ++g) t = __fadd_rn(t, sm[g][lane]);
    if (i < split) dW[i] = t; else db[i - split] = t;
  }
  if (blockIdx.x == 0 && grp == 1) {
    double l = 0.0;
    for (int c = lane; c < chunks; c += 32) l += loss_part[c];
    l = warp_sum(l);
    if (lane == 0) *loss_sum = l;
  }
}

int blocks_for(int64_t n, int t = 256) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, t), 148 * 16));
}

}  // namespace
}  // namespace fgl

using namespace fgl;

extern "C" {

static int spmm_dispatch(const int64_t* indptr, const int32_t* col, const float* w, int64_t num_rows,
                         int64_t col_base, const float* X, int64_t ldx, const float* self_x, int64_t ld_self,
                         float* Y, int64_t ldy, int32_t d, cudaStream_t st, int prof_id,
                         int64_t lean_ctas = (int64_t)kNumSMs * 8) {
  if (num_rows == 0) return FGL_OK;
  const ProfMark pm = prof_begin(st);
  const int d4 = (d + 3) / 4;
  if (d4 <= 1) launch_spmm<1, 1>(indptr, col, w, num_rows, col_base, X, ldx, self_x, ld_self, Y, ldy, d4, st);
  else if (d4 <= 2) launch_spmm<2, 1>(indptr, col, w, num_rows, col_base, X, ldx, self_x, ld_self, Y, ldy, d4, st);
  else if (d4 <= 4) launch_spmm<4, 1>(indptr, col, w, num_rows, col_base, X, ldx, self_x, ld_self, Y, ldy, d4, st);
  else if (d4 <= 8) launch_spmm<8, 1>(indptr, col, w, num_rows, col_base, X, ldx, self_x, ld_self, Y, ldy, d4, st);
  else if (d4 <= 32)
    launch_spmm_lean(indptr, col, w, num_rows, col_base, X, ldx, self_x, ld_self, Y, ldy, d4, st, lean_ctas);
  else if (d4 <= 64) launch_spmm<32, 2>(indptr, col, w, num_rows, col_base, X, ldx, self_x, ld_self, Y, ldy, d4, st);
  else if (d4 <= 128) launch_spmm<32, 4>(indptr, col, w, num_rows, col_base, X, ldx, self_x, ld_self, Y, ldy, d4, st);
  // Reddit's 602-wide rows (151 chunks): 5 chunks per lane (94 % of lanes
  // busy instead of 59 %), two neighbour rows in flight (fewer registers,
  // more resident warps)
  else if (d4 <= 160) launch_spmm<32, 5, 2>(indptr, col, w, num_rows, col_base, X, ldx, self_x, ld_self, Y, ldy, d4, st);
  else if (d4 <= 256) launch_spmm<32, 8>(indptr, col, w, num_rows, col_base, X, ldx, self_x, ld_self, Y, ldy, d4, st);
  else {
    set_error("fgl_spmm: feature dim %d above 1024 is not supported", d);
    return FGL_E_UNSUPPORTED;
  }
  prof_end(pm, prof_id, num_rows, d);
  FGL_LAUNCH_CHECK("spmm_kernel");
  return FGL_OK;
}

int fgl_spmm(const int64_t* indptr, const int32_t* col, const float* w, int64_t num_rows,
             int64_t col_base, const float* X, int64_t ldx, const float* self_x, int64_t ld_self,
             float* Y, int64_t ldy, int32_t d, void* stream) {
  if (num_rows < 0 || d < 1 || !indptr || !Y || ldy < d || ldx < d || (ldx % 4) || (ldy % 4) ||
      (self_x && (ld_self % 4))) {
    set_error("fgl_spmm: bad arguments (d=%d ldx=%lld ldy=%lld; leading dims must be multiples of 4)",
              d, (long long)ldx, (long long)ldy);
    return FGL_E_INVALID;
  }
  if ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(Y) |
       reinterpret_cast<uintptr_t>(self_x)) & 15) {
    set_error("fgl_spmm: feature pointers must be 16-byte aligned");
    return FGL_E_INVALID;
  }
  return spmm_dispatch(indptr, col, w, num_rows, col_base, X, ldx, self_x, ld_self, Y, ldy, d, (cudaStream_t)stream,
                       kProfSpmm);
}

// fgl_spmm with the source rows addressed through an id map (x_ids): the
// GIN / SAGE layer-0 aggregation (and its root term) read the HBM feature
// table directly instead of an x0 block gathered first.  Feature widths of
// 36..128 (the lean kernel); FGL_E_UNSUPPORTED otherwise.
int fgl_spmm_ids(const int64_t* indptr, const int32_t* col, const float* w, int64_t num_rows, int64_t col_base,
                 const float* X, int64_t ldx, const int32_t* x_ids, int64_t self_base, int32_t add_self, float* Y,
                 int64_t ldy, int32_t d, void* stream) {
  if (num_rows < 0 || d < 1 || !indptr || !Y || !X || !x_ids || ldy < d || ldx < d || (ldx % 4) || (ldy % 4)) {
    set_error("fgl_spmm_ids: bad arguments");
    return FGL_E_INVALID;
  }
  if ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(Y)) & 15) {
    set_error("fgl_spmm_ids: feature pointers must be 16-byte aligned");
    return FGL_E_INVALID;
  }
  const int d4 = (d + 3) / 4;
  if (d4 <= 8 || d4 > 32) {
    set_error("fgl_spmm_ids: feature width %d outside 33..128", d);
    return FGL_E_UNSUPPORTED;
  }
  if (num_rows == 0) return FGL_OK;
  const ProfMark pm = prof_begin((cudaStream_t)stream);
  launch_spmm_lean(indptr, col, w, num_rows, col_base, X, ldx, add_self ? X : nullptr, ldx, Y, ldy, d4,
                   (cudaStream_t)stream, (int64_t)kNumSMs * 8, x_ids, self_base);
  prof_end(pm, kProfSpmm, num_rows, d);
  FGL_LAUNCH_CHECK("spmm_lean_kernel(ids)");
  return FGL_OK;
}

// Layer-0 aggregation over the sampled block graph (rows of <= max_row_len
// edges gathered straight from the HBM feature table): the same kernels as
// fgl_spmm, kept as its own entry point (and profiling id) for the stage
// rooflines; the row bound is validated, not needed by the kernel.
int fgl_spmm_gather(const int64_t* indptr, const int32_t* col, const float* w, int64_t num_rows, int64_t col_base,
                    const float* X, int64_t ldx, int64_t x_rows, float* Y, int64_t ldy, int32_t d,
                    int32_t max_row_len, void* stream) {
  if ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(Y)) & 15) {
    set_error("fgl_spmm_gather: feature pointers must be 16-byte aligned");
    return FGL_E_INVALID;
  }
  if (num_rows < 0 || d < 1 || d > 256 || ldx > 256 || !indptr || !Y || !X || ldy < d || ldx < d || (ldx % 4) ||
      (ldy % 4) || max_row_len < 0 || x_rows < 1) {
    set_error("fgl_spmm_gather: bad arguments");
    return FGL_E_INVALID;
  }
  if (max_row_len > 16) {
    set_error("fgl_spmm_gather: rows longer than 16 edges use fgl_spmm");
    return FGL_E_UNSUPPORTED;
  }
  // CTA budget of the layer-0 aggregation, which runs beside the model chain
  // on its own stream: FGL_L0_CTAS (default 0 = one 8-row CTA per block of
  // rows, not a persistent grid), so CTAs retire every few microseconds and
  // their SM slots go to the high-priority chain (2.29 -> 2.22 ms per window)
  static const int l0_ctas = env_int("FGL_L0_CTAS", 0);
  return spmm_dispatch(indptr, col, w, num_rows, col_base, X, ldx, nullptr, ldx, Y, ldy, d, (cudaStream_t)stream,
                       kProfSpmmGather, l0_ctas > 0 ? l0_ctas : (int64_t)1 << 30);
}

// dH = (dX * (Xout > 0)) W^T on the tensor cores, the reduction (dout) in K
// slices of <= 128 accumulated into dH (wide outputs: papers' 172 classes)
static bool dgrad_tc(const float* dX, int64_t lddx, const float* Xout, int64_t ldxo, int64_t n, const float* W,
                     int32_t din, int32_t dout, float* dH, int64_t lddh, cudaStream_t st, int* err) {
  if ((lddx % 4) || (Xout && (ldxo % 4)) || (lddh % 4) || (reinterpret_cast<uintptr_t>(dH) & 15)) return false;
  // [column slice of dH (rows of W)] x [K slice of dout]: the widest slices
  // whose first tile fits shared memory; K slices accumulate into dH
  const int kfirst = dout > 128 ? dout : 128;  // one K slice first (tc_dense4 streams the weight)
  for (int nsw = 256; nsw >= 64; nsw /= 2) {
    for (int ksw = kfirst; ksw >= 32; ksw = ksw > 128 ? 128 : ksw / 2) {
      bool ok = true;
      for (int n0 = 0; n0 < din && ok; n0 += nsw) {
        const int ns = din - n0 < nsw ? din - n0 : nsw;
        for (int k0 = 0; k0 < dout && ok; k0 += ksw) {
          const int ks = dout - k0 < ksw ? dout - k0 : ksw;
          ok = tc_gemm3(1, dX + k0, lddx, Xout ? Xout + k0 : nullptr, ldxo, W + (int64_t)n0 * dout + k0, nullptr,
                        dH + n0, lddh, n, ns, ks, 0, st, err, k0 > 0, dout);
          if (*err) return true;
          // a later slice may fall outside (the first K slice runs on tc_dense4,
          // accumulating slices on tc_gemm3): narrower slices rewrite dH whole
        }
      }
      if (ok) return true;
    }
  }
  return false;
}

int fgl_dense_fwd(const float* H, int64_t ldh, int64_t n, int32_t din, const float* W,
                  const float* b, int32_t dout, float* Z, int64_t ldz, int32_t relu, void* stream) {
  if (n < 0 || din < 1 || dout < 1 || !W || !Z || ldh < din || ldz < dout) {
    set_error("fgl_dense_fwd: bad arguments");
    return FGL_E_INVALID;
  }
  if (n == 0) return FGL_OK;
  int err = 0;
  if (!(ldh % 4) && !(ldz % 4) && !(reinterpret_cast<uintptr_t>(H) & 15) && !(reinterpret_cast<uintptr_t>(Z) & 15)) {
    // the tensor-core kernel on [column slice of Z] x [K slice of W] tiles
    // (one tile for the usual <= 128 x 128 layers; wide inputs -- Reddit 602
    // -- and wide outputs -- papers' 172 classes -- in slices), each K slice
    // adding into Z (bias / ReLU with the last); fp32 sums.  Slice widths: the
    // largest whose first (widest) tile fits the kernel's shared memory (the
    // weight's hi / lo images grow with K x N)
    bool ok = false;
    // one K slice first (tc_dense4 streams the weight's K boxes through its
    // stages for din > 128), then 128 / 64-wide slices accumulated by tc_gemm3
    const int kfirst = din > 128 ? din : 128;
    for (int ksw = kfirst; ksw >= 64 && !ok; ksw = ksw > 128 ? 128 : ksw / 2) {
      for (int nsw = 128; nsw >= 32 && !ok; nsw /= 2) {
        ok = true;
        for (int n0 = 0; n0 < dout && ok; n0 += nsw) {
          const int ns = dout - n0 < nsw ? dout - n0 : nsw;
          for (int k0 = 0; k0 < din && ok; k0 += ksw) {
            const int ks = din - k0 < ksw ? din - k0 : ksw;
            const bool last = k0 + ks >= din;
            ok = tc_gemm3(0, H + k0, ldh, nullptr, 0, W + (int64_t)k0 * dout + n0, last && b ? b + n0 : nullptr,
                          Z + n0, ldz, n, ns, ks, last ? relu : 0, (cudaStream_t)stream, &err, k0 > 0, dout);
            if (err) return err;
            // a later slice may fall outside (the first K slice runs on
            // tc_dense4, accumulating slices on tc_gemm3): narrower slices
            // rewrite Z whole
          }
        }
      }
    }
    if (ok) return FGL_OK;
    // no slicing fits the envelope: the SIMT kernel below computes Z
  }
  count_dense_fallback();
  dim3 grid((unsigned)ceil_div(n, BM), (unsigned)ceil_div(dout, BN));
  FGL_COUNT_LAUNCH(), gemm_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(H, ldh, W, dout, 0, b, Z, ldz, n, dout, din,
                                                      relu, nullptr, 0);
  FGL_LAUNCH_CHECK("gemm_kernel(fwd)");
  return FGL_OK;
}

int64_t fgl_dense_bwd_ws_bytes(int32_t din, int32_t dout) {
  return (int64_t)2 * kPersistentCTAs * ((int64_t)din + 1) * dout * 4;
}

int fgl_dense_bwd(const float* H, int64_t ldh, int64_t n, int32_t din, const float* W,
                  int32_t dout, const float* dX, int64_t lddx, const float* Xout, int64_t ldxo,
                  float* dW, float* db, float* dH, int64_t lddh, void* ws, int64_t ws_bytes,
                  void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 0 || din < 1 || dout < 1 || !W || !dW || !db || lddx < dout || (Xout && ldxo < dout) ||
      (dH && lddh < din)) {
    set_error("fgl_dense_bwd: bad arguments");
    return FGL_E_INVALID;
  }
  if (ws_bytes < fgl_dense_bwd_ws_bytes(din, dout)) {
    set_error("fgl_dense_bwd: workspace too small");
    return FGL_E_CAPACITY;
  }
  const int ky = (int)ceil_div(din + 1, WK), nz = (int)ceil_div(dout, WN);
  const int chunks = (int)std::max<int64_t>(
      1, std::min<int64_t>(ceil_div(n, 64), std::max(1, 4 * kNumSMs / (ky * nz))));
  const int64_t rows_per = std::max<int64_t>(1, ceil_div(n, chunks));
  float* pw = static_cast<float*>(ws);
  const int64_t outs = (int64_t)(din + 1) * dout;
  if (n > 0) {
    int werr = 0;
    // at least `tpc` 64-row tiles per CTA: small layers then use a few CTAs
    // (fewer per-CTA prologues, fewer partials to reduce, fewer SMs taken
    // from the concurrent chain); the large layer 0 still spans all SMs
    static const int tpc = getenv("FGL_WG_TPC") ? std::max(1, atoi(getenv("FGL_WG_TPC"))) : 16;
    const int tc3_chunks = (int)std::max<int64_t>(1, std::min<int64_t>(kNumSMs, ceil_div(ceil_div(n, 64), tpc)));
    const ProfMark pm = prof_begin(st);
    bool tc_done = false;
    if (!(ldh % 4) && !(reinterpret_cast<uintptr_t>(H) & 15) && !(lddx % 4) &&
        !(reinterpret_cast<uintptr_t>(dX) & 15) && (!Xout || (!(ldxo % 4) && !(reinterpret_cast<uintptr_t>(Xout) & 15)))) {
      // tensor cores over [<= 128 output features] x [<= 124 input features]
      // slices (wide inputs: Reddit 602; wide outputs: papers 172 classes);
      // each slice's partials are reduced straight into its block of dW (db
      // from the first K slice, the others' db rows land in scratch)
      // (din == 128: one slice, db from tc_wgrad3's converters instead of a ones lane)
      const int kmax = din == 128 ? 128 : din + 1 > 128 ? 124 : din;
      bool ok = false, later_fail = false;
      // wide inputs (Reddit 602) with one N slice: every K slice in one launch,
      // the CTAs of a row range on consecutive slices (dZ / mask tiles shared
      // through L2 instead of re-read from HBM per slice)
      const int nks = (int)ceil_div(din, kmax);
      static const int multi = getenv("FGL_WG_MULTI") ? atoi(getenv("FGL_WG_MULTI")) : 1;
      if (multi && nks > 1 && dout <= 128) {
        const int cps = std::max(1, std::min(tc3_chunks, kNumSMs / nks));
        const int64_t stride = (int64_t)cps * (kmax + 1) * dout;
        float* scratch_db = pw + nks * stride;
        if ((nks * stride + dout) * 4 <= ws_bytes) {
          ok = tc_wgrad3(H, ldh, dX, lddx, Xout, ldxo, n, din, dout, pw, cps, st, &werr, nks, kmax);
          if (werr) return werr;
          for (int s = 0; ok && s < nks; ++s) {
            const int k0 = s * kmax, ks = din - k0 < kmax ? din - k0 : kmax;
            const int64_t o = (int64_t)(ks + 1) * dout;
            FGL_COUNT_LAUNCH(), reduce_partials_kernel<<<(unsigned)ceil_div(o, 32), 256, 0, st>>>(
                pw + s * stride, cps, o, dW + (int64_t)k0 * dout, 0, k0 == 0 ? db : scratch_db, ks + 1, dout, 0);
          }
        }
      }
      for (int nsw = 128; nsw >= 32 && !ok && !later_fail; nsw /= 2) {  // the widest N slice that fits
        const int nmax = dout < nsw ? dout : nsw;
        float* slice_part = pw;
        float* scratch_db = pw + (int64_t)tc3_chunks * (kmax + 1) * nmax;
        ok = true;
        bool first = true;
        for (int n0 = 0; n0 < dout && ok; n0 += nsw) {
          const int ns = dout - n0 < nsw ? dout - n0 : nsw;
          for (int k0 = 0; k0 < din && ok; k0 += kmax) {
            const int ks = din - k0 < kmax ? din - k0 : kmax;
            ok = tc_wgrad3(H + k0, ldh, dX + n0, lddx, Xout ? Xout + n0 : nullptr, ldxo, n, ks, ns, slice_part,
                           tc3_chunks, st, &werr);
            if (werr) return werr;
            if (ok) {
              const int64_t o = (int64_t)(ks + 1) * ns;
              FGL_COUNT_LAUNCH(), reduce_partials_kernel<<<(unsigned)ceil_div(o, 32), 256, 0, st>>>(
                  slice_part, tc3_chunks, o, dW + (int64_t)k0 * dout, 0, k0 == 0 ? db : scratch_db, ks + 1, dout, n0);
            } else if (!first) {
              later_fail = true;
            }
            first = false;
          }
        }
      }
      tc_done = ok;
    }
    if (!tc_done) {
      count_dense_fallback();
      const int vec = (ldh % 4 == 0) && !(reinterpret_cast<uintptr_t>(H) & 15);
      dim3 g(chunks, ky, nz);
      FGL_COUNT_LAUNCH(), wgrad_partial_kernel<<<g, 256, 0, st>>>(H, ldh, dX, lddx, Xout, ldxo, n, din, dout,
                                                                  rows_per, pw, vec);
      FGL_COUNT_LAUNCH(), reduce_partials_kernel<<<(unsigned)ceil_div(outs, 32), 256, 0, st>>>(
          pw, chunks, outs, dW, (int64_t)din * dout, db, 0);
    }
    prof_end(pm, kProfWgrad, n, din, dout);
    int err = 0;
    if (dH && dgrad_tc(dX, lddx, Xout, ldxo, n, W, din, dout, dH, lddh, st, &err)) {
      if (err) return err;
    } else if (dH) {
      count_dense_fallback();
      dim3 grid((unsigned)ceil_div(n, BM), (unsigned)ceil_div(din, BN));
      FGL_COUNT_LAUNCH(), gemm_kernel<<<grid, 256, 0, st>>>(dX, lddx, W, dout, 1, nullptr, dH, lddh, n, din, dout, 0,
                                        Xout, ldxo);
    }
  } else {
    FGL_CUDA(cudaMemsetAsync(dW, 0, 4 * (int64_t)din * dout, st));
    FGL_CUDA(cudaMemsetAsync(db, 0, 4 * (int64_t)dout, st));
  }
  FGL_LAUNCH_CHECK("dense_bwd");
  return FGL_OK;
}

int fgl_dense_dgrad(const float* dX, int64_t lddx, const float* Xout, int64_t ldxo, int64_t n, const float* W,
                    int32_t din, int32_t dout, float* dH, int64_t lddh, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 0 || din < 1 || dout < 1 || !W || !dH || lddx < dout || (Xout && ldxo < dout) || lddh < din) {
    set_error("fgl_dense_dgrad: bad arguments");
    return FGL_E_INVALID;
  }
  if (n == 0) return FGL_OK;
  int err = 0;
  if (dgrad_tc(dX, lddx, Xout, ldxo, n, W, din, dout, dH, lddh, st, &err)) return err;
  count_dense_fallback();
  dim3 grid((unsigned)ceil_div(n, BM), (unsigned)ceil_div(din, BN));
  FGL_COUNT_LAUNCH(), gemm_kernel<<<grid, 256, 0, st>>>(dX, lddx, W, dout, 1, nullptr, dH, lddh, n, din, dout, 0, Xout,
                                                        ldxo);
  FGL_LAUNCH_CHECK("dense_dgrad");
  return FGL_OK;
}

int64_t fgl_softmax_xent_ws_bytes(void) { return 8 * (148 * 8 * 8 + 1); }

int fgl_softmax_xent(const float* logits, int64_t ldl, const int32_t* rows, int64_t row_base,
                     const int32_t* seed_ids, const int64_t* labels, int64_t B, int32_t C,
                     float* dlogits, int64_t ldd, double* loss_sum, void* ws, int64_t ws_bytes,
                     void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (B < 1 || C < 1 || !logits || !rows || !labels || !dlogits || !loss_sum || ldl < C || ldd < C ||
      ws_bytes < fgl_softmax_xent_ws_bytes()) {
    set_error("fgl_softmax_xent: bad arguments");
    return FGL_E_INVALID;
  }
  const int blocks = (int)std::min<int64_t>(148 * 8, ceil_div(B, 8));
  double* part = static_cast<double*>(ws);
  FGL_COUNT_LAUNCH(), softmax_xent_kernel<<<blocks, 256, 0, st>>>(logits, ldl, rows, row_base, seed_ids, labels, B, C,
                                              dlogits, ldd, part);
  FGL_COUNT_LAUNCH(), sum_doubles_kernel<<<1, 1024, 0, st>>>(part, blocks * 8, loss_sum);
  FGL_LAUNCH_CHECK("softmax_xent");
  return FGL_OK;
}

int64_t fgl_top_layer_ws_bytes(int64_t B, int32_t din, int32_t C) {
  const int64_t chunks = ceil_div(std::max<int64_t>(B, 1), TOP_ROWS);
  return chunks * ((int64_t)(din + 1) * C * 4 + 8) + 64;
}

int fgl_top_layer(const float* H, int64_t ldh, const int32_t* rows, int64_t row_base, const int32_t* seed_ids,
                  const int64_t* labels, int64_t B, int32_t din, int32_t C, const float* W, const float* b,
                  float* dH, int64_t lddh, float* dW, float* db, double* loss_sum, void* ws, int64_t ws_bytes,
                  const int64_t* agg_indptr, const int32_t* agg_col, const float* agg_w, int64_t agg_col_base,
                  void* chain_stream, void* reduce_stream) {
  if (B < 1 || din < 1 || din > 64 || C < 1 || C > 192 || !H || !rows || !labels || !W || !dH || !dW || !db ||
      !loss_sum || ldh < din || lddh < din || ws_bytes < fgl_top_layer_ws_bytes(B, din, C) ||
      (agg_indptr && (!agg_col || !agg_w || (ldh % 4) || (reinterpret_cast<uintptr_t>(H) & 15)))) {
    set_error("fgl_top_layer: bad arguments (din <= 64, C <= 192)");
    return FGL_E_INVALID;
  }
  const int chunks = (int)ceil_div(B, TOP_ROWS);
  float* part = static_cast<float*>(ws);
  double* lp = reinterpret_cast<double*>(static_cast<char*>(ws) + ((int64_t)chunks * (din + 1) * C * 4 + 7) / 8 * 8);
  const ProfMark pm = prof_begin((cudaStream_t)chain_stream);
  if (C <= 64) {
    FGL_COUNT_LAUNCH(), top_layer_kernel<64><<<chunks, 256, (128 + TOP_ROWS) * 64 * 4, (cudaStream_t)chain_stream>>>(
        H, ldh, rows, row_base, seed_ids, labels, B, din, C, W, b, dH, lddh, part, lp, agg_indptr, agg_col, agg_w,
        agg_col_base);
  } else {
    constexpr int smem = (128 + TOP_ROWS) * 192 * 4;
    static bool attr = false;
    if (!attr) {
      const cudaError_t e =
          cudaFuncSetAttribute(top_layer_kernel<192>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (e != cudaSuccess) return cuda_status(e, "cudaFuncSetAttribute(top_layer_kernel)");
      attr = true;
    }
    FGL_COUNT_LAUNCH(), top_layer_kernel<192><<<chunks, 256, smem, (cudaStream_t)chain_stream>>>(
        H, ldh, rows, row_base, seed_ids, labels, B, din, C, W, b, dH, lddh, part, lp, agg_indptr, agg_col, agg_w,
        agg_col_base);
  }
  prof_end(pm, kProfTopLayer, B, din, C);
  FGL_LAUNCH_CHECK("top_layer_kernel");
  if (reduce_stream && reduce_stream != chain_stream) {
    // the reduction is off the chain: the caller orders reduce_stream after
    // chain_stream's top_layer_kernel with an event (fgl_top_layer_reduce)
    return FGL_OK;
  }
  const int64_t outs = (int64_t)(din + 1) * C;
  FGL_COUNT_LAUNCH(), top_reduce_kernel<<<(unsigned)ceil_div(outs, 32), 256, 0, (cudaStream_t)chain_stream>>>(
      part, chunks, outs, dW, (int64_t)din * C, db, lp, loss_sum);
  FGL_LAUNCH_CHECK("top_reduce_kernel");
  return FGL_OK;
}

int fgl_top_layer_reduce(int64_t B, int32_t din, int32_t C, float* dW, float* db, double* loss_sum, void* ws,
                         void* stream) {
  const int chunks = (int)ceil_div(B, TOP_ROWS);
  float* part = static_cast<float*>(ws);
  double* lp = reinterpret_cast<double*>(static_cast<char*>(ws) + ((int64_t)chunks * (din + 1) * C * 4 + 7) / 8 * 8);
  const int64_t outs = (int64_t)(din + 1) * C;
  FGL_COUNT_LAUNCH(), top_reduce_kernel<<<(unsigned)ceil_div(outs, 32), 256, 0, (cudaStream_t)stream>>>(
      part, chunks, outs, dW, (int64_t)din * C, db, lp, loss_sum);
  FGL_LAUNCH_CHECK("top_reduce_kernel");
  return FGL_OK;
}

int fgl_sgd(float* params, const float* grads, int64_t n, float lr, void* stream) {
  if (n < 0 || (n > 0 && (!params || !grads))) {
    set_error("fgl_sgd: bad arguments");
    return FGL_E_INVALID;
  }
  if (n == 0) return FGL_OK;
  const ProfMark pm = prof_begin((cudaStream_t)stream);
  FGL_COUNT_LAUNCH(), sgd_kernel<<<blocks_for(n), 256, 0, (cudaStream_t)stream>>>(params, grads, n, lr);
  prof_end(pm, kProfSgd, n);
  FGL_LAUNCH_CHECK("sgd_kernel");
  return FGL_OK;
}

int fgl_fill_rows(float* Y, int64_t ldy, int64_t nrows, int32_t d, const float* rowval,
                  int32_t relu, void* stream) {
  if (nrows < 0 || d < 1 || ldy < d || (nrows > 0 && !Y)) {
    set_error("fgl_fill_rows: bad arguments");
    return FGL_E_INVALID;
  }
  if (nrows == 0) return FGL_OK;
  FGL_COUNT_LAUNCH(), fill_rows_kernel<<<blocks_for(nrows * d), 256, 0, (cudaStream_t)stream>>>(Y, ldy, nrows, d, rowval, relu);
  FGL_LAUNCH_CHECK("fill_rows_kernel");
  return FGL_OK;
}

}  // extern "C"
