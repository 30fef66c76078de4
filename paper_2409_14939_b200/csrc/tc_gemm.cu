// Tensor-core (tcgen05, 5th-gen) dense layer GEMMs with 3xTF32 (sm_100a).
//
// The dense per-layer transform of the reference (compute.dense_update,
// compute.py:198-216) and the dH = dZ W^T / dW = h^T dZ of trainer._backward
// (trainer.py:212-228) in fp32 accuracy on the tensor cores: every fp32
// operand x is split x = hi + lo with hi = tf32(x) (round to nearest, low 13
// bits zero) and lo = x - hi; A B ~= A_lo B_hi + A_hi B_lo + A_hi B_hi is
// accumulated in fp32 in tensor memory (relative error ~1e-6, inside the
// 1e-5 bar of the north star).
//
// Data movement (one CTA of 8 warps per SM, persistent over tiles):
//  * operand tiles are copied global -> shared with 16-byte cp.async straight
//    into the UMMA canonical K-major no-swizzle layout (8 rows x 16 B core
//    matrices; the weight gradient stages rows and transposes in shared
//    memory); zero fill handles ragged rows / columns;
//  * a split pass rewrites each raw chunk in place as its tf32 hi part and
//    writes the lo part to a second buffer (conflict-free, chunk = thread);
//  * one elected thread issues the 3*K/8 tcgen05.mma.kind::tf32 (M=128,
//    N<=256) and commits to an mbarrier; the copies of the next tile are
//    already in flight while the MMAs and the epilogue of this one run;
//  * the epilogue drains TMEM with tcgen05.ld.32x32b.x16 (warp w reads lane
//    quarter w%4, column half w/4), adds the bias, applies ReLU, stores rows.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "tcgen05.cuh"

namespace fgl {
namespace {
using namespace tc;

constexpr int TC_M = 128;
constexpr int TC_THREADS = 256;
constexpr int TC_MAX_SMEM = 220 * 1024;

// ------------------------------------------------------------- fwd / dgrad --
struct TcArgs {
  const float* A;      // [M, K] row-major (lda), 16-byte aligned rows
  int64_t lda;
  const float* mask;   // dgrad: ReLU mask (layer output) with A's shape, or null
  int64_t ldm;
  const float* W;      // layer weight [din, dout] row-major
  const float* bias;   // fwd: [N] or null
  float* C;            // [M, N] row-major (ldc)
  int64_t ldc;
  int64_t M;
  int N, K, N_pad, K_pad, relu, tmem_cols, stages;
};

// issue the cp.async copies of one 128-row tile of A (and of the mask)
template <int MODE>
__device__ __forceinline__ void issue_tile(const TcArgs& p, int64_t m0, char* raw, char* mraw, int KC) {
  for (int idx = threadIdx.x; idx < TC_M * KC; idx += TC_THREADS) {
    // thread order = (row within 8-group, chunk, 8-group): 8 consecutive threads
    // fill one 128-byte core matrix (conflict-free) from 8 rows
    const int rl = idx & 7, rest = idx >> 3;
    const int kc = rest % KC, rg = rest / KC;
    const int r = rg * 8 + rl, k = 4 * kc;
    const int64_t row = m0 + r;
    const int valid = (row < p.M && k < p.K) ? (int)min(4, p.K - k) : 0;
    const uint32_t off = (uint32_t)(rg * (KC * 128) + kc * 128 + rl * 16);
    const float* src = valid ? p.A + row * p.lda + k : p.A;
    cp_async16(smem_u32(raw + off), src, valid * 4);
    if (MODE == 1 && p.mask) {
      const float* msrc = valid ? p.mask + row * p.ldm + k : p.mask;
      cp_async16(smem_u32(mraw + off), msrc, valid * 4);
    }
  }
}

template <int MODE>  // 0: C = act(A W + b), W [K, N];  1: C = (A * (mask > 0)) W^T, W [N, K]
__global__ void __launch_bounds__(TC_THREADS, 1) tc_gemm_kernel(TcArgs p) {
  extern __shared__ __align__(1024) char smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int KC = p.K_pad / 4;
  const int a_bytes = TC_M * p.K_pad * 4, b_bytes = p.N_pad * p.K_pad * 4;
  char* sB_hi = smem;
  char* sB_lo = sB_hi + b_bytes;
  char* sA_lo = sB_lo + b_bytes;
  char* sA_raw[2] = {sA_lo + a_bytes, sA_lo + 2 * a_bytes};
  const bool use_mask = MODE == 1 && p.mask;
  char* sM_raw[2] = {sA_lo + (1 + p.stages) * a_bytes, sA_lo + (2 + p.stages) * a_bytes};
  char* tail = sA_lo + (1 + p.stages + (use_mask ? p.stages : 0)) * a_bytes;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(tail);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mbar + 1);
  float* sbias = reinterpret_cast<float*>(tail + 16);
  const bool out_vec = (p.ldc % 4 == 0) && !(reinterpret_cast<uintptr_t>(p.C) & 15);

  const int64_t tiles = ceil_div(p.M, TC_M);
  int64_t t = blockIdx.x;
  if (t < tiles) issue_tile<MODE>(p, t * TC_M, sA_raw[0], sM_raw[0], KC);
  cp_async_commit();
  for (int c = tid; c < p.N_pad; c += TC_THREADS) sbias[c] = (MODE == 0 && p.bias && c < p.N) ? p.bias[c] : 0.f;
  if (warp == 0) tmem_alloc(tmem_slot, p.tmem_cols);
  if (tid == 0) {
    mbar_init(smem_u32(mbar));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  // weight operand B[n][k], split once per CTA
  for (int idx = tid; idx < p.N_pad * p.K_pad; idx += TC_THREADS) {
    const int n = idx / p.K_pad, k = idx % p.K_pad;
    float v = 0.f;
    if (n < p.N && k < p.K) v = MODE == 0 ? p.W[(int64_t)k * p.N + n] : p.W[(int64_t)n * p.K + k];
    const float h = tf32_hi(v);
    const uint32_t off = kmaj_off(n, k, KC) + (k & 3) * 4;
    *reinterpret_cast<float*>(sB_hi + off) = h;
    *reinterpret_cast<float*>(sB_lo + off) = __fsub_rn(v, h);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;
  const uint32_t bar = smem_u32(mbar);
  const uint32_t idesc = idesc_tf32(TC_M, p.N_pad, 0, 0);
  const uint32_t sbo = KC * 128;
  uint32_t phase = 0;
  for (int j = 0; t < tiles; t += gridDim.x, ++j) {
    const int buf = p.stages == 2 ? (j & 1) : 0;
    const int64_t m0 = t * TC_M;
    const int64_t tn = t + gridDim.x;
    if (p.stages == 2 && tn < tiles) {  // next tile's copies overlap this tile's work
      issue_tile<MODE>(p, tn * TC_M, sA_raw[buf ^ 1], sM_raw[buf ^ 1], KC);
      cp_async_commit();
      cp_async_wait_1();
    } else {
      cp_async_wait_all();
    }
    __syncthreads();
    // split pass (chunk = thread, smem order)
    char* raw = sA_raw[buf];
    for (int idx = tid; idx < TC_M * KC; idx += TC_THREADS) {
      const uint32_t off = (uint32_t)idx * 16u;
      float4 x = *reinterpret_cast<const float4*>(raw + off);
      if (use_mask) {
        const float4 m = *reinterpret_cast<const float4*>(sM_raw[buf] + off);
        if (!(m.x > 0.f)) x.x = 0.f;
        if (!(m.y > 0.f)) x.y = 0.f;
        if (!(m.z > 0.f)) x.z = 0.f;
        if (!(m.w > 0.f)) x.w = 0.f;
      }
      split_chunk(raw, sA_lo, off, x);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t a_hi = smem_u32(raw), a_lo = smem_u32(sA_lo);
      const uint32_t b_hi = smem_u32(sB_hi), b_lo = smem_u32(sB_lo);
      const int steps = p.K_pad / 8;
      for (int s = 0; s < steps; ++s) {  // small terms first
        mma_tf32(tmem, umma_desc(a_lo + s * 256, 128, sbo), umma_desc(b_hi + s * 256, 128, sbo), idesc, s > 0);
        mma_tf32(tmem, umma_desc(a_hi + s * 256, 128, sbo), umma_desc(b_lo + s * 256, 128, sbo), idesc, 1);
      }
      for (int s = 0; s < steps; ++s)
        mma_tf32(tmem, umma_desc(a_hi + s * 256, 128, sbo), umma_desc(b_hi + s * 256, 128, sbo), idesc, 1);
      mma_commit(bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1;
    if (p.stages == 1 && tn < tiles) {  // single buffer: next copies start once the MMAs are done
      issue_tile<MODE>(p, tn * TC_M, sA_raw[0], sM_raw[0], KC);
      cp_async_commit();
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    // epilogue: warp w drains TMEM lane quarter w%4 (rows), column half w/4
    const int quarter = warp & 3, half = warp >> 2;
    const int64_t row = m0 + quarter * 32 + lane;
    const int chunks = p.N_pad / 16;
    const int c_begin = half == 0 ? 0 : ((chunks + 1) / 2) * 16;
    const int c_end = half == 0 ? ((chunks + 1) / 2) * 16 : p.N_pad;
    for (int c0 = c_begin; c0 < c_end; c0 += 16) {
      uint32_t v[16];
      tmem_ld16(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)c0, v);
      if (row < p.M) {
        float* out = p.C + row * p.ldc;
        float x[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) {
          float y = __uint_as_float(v[q]);
          if (MODE == 0 && p.bias) y = __fadd_rn(y, sbias[c0 + q]);
          if (p.relu) y = y > 0.f ? y : 0.f;
          x[q] = y;
        }
        // 16-byte stores inside the row's leading dimension, scalar tail
#pragma unroll
        for (int q = 0; q < 16; q += 4) {
          const int col = c0 + q;
          if (col + 3 < p.ldc && col < p.N && out_vec) {
            *reinterpret_cast<float4*>(out + col) = make_float4(x[q], x[q + 1], x[q + 2], x[q + 3]);
          } else {
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (col + u < p.N) out[col + u] = x[q + u];
          }
        }
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();  // TMEM drained and sA_lo / the raw buffer free before reuse
  }
  cp_async_wait_all();
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    tmem_free(tmem, p.tmem_cols);
  }
}

int64_t tc_gemm_smem(int mode, bool has_mask, int N_pad, int K_pad, int stages) {
  const int64_t a = (int64_t)TC_M * K_pad * 4, b = (int64_t)N_pad * K_pad * 4;
  return 2 * b + a * (1 + stages + ((mode == 1 && has_mask) ? stages : 0)) + 64 + 4 * N_pad;
}

// ---------------------------------------------------------------- wgrad --
// Partial [dW; db] of a row chunk: D[m][n] = sum_r A'[m][r] B'[n][r] with
// A'[m][r] = H[r][m] (m < K), 1 (m == K: the bias row) and B'[n][r] =
// dZ[r][n] * (Xout[r][n] > 0).  Rows r are the MMA K dimension (K-major
// operands).  Each stage of 32 rows is cp.async-copied row-major into a
// double-buffered staging area; the split pass transposes 4 rows x 1 column
// into each 16-byte K-major chunk (conflict-free shared loads), splits it
// into tf32 hi/lo, and the MMAs of the stage run while the next stage lands.
constexpr int WG_KS = 32;
constexpr int WG_KC = WG_KS / 4;  // 16-byte chunks per operand row

struct WgArgs {
  const float* H; int64_t ldh;
  const float* dZ; int64_t ldz;
  const float* mask; int64_t ldm;
  float* part;          // [chunks][K+1][N]
  int64_t M;            // rows
  int64_t rows_per_cta;
  int K, N, N_pad, tmem_cols;
};

__device__ __forceinline__ void wg_issue(const WgArgs& p, int64_t rs, int64_t r_end, char* hs, char* zs,
                                         char* ms) {
  constexpr int H4 = TC_M / 4;  // staging row of H: 128 floats
  const int Z4 = p.N_pad / 4;
  for (int idx = threadIdx.x; idx < WG_KS * H4; idx += TC_THREADS) {
    const int kk = idx / H4, c = idx % H4;
    const int64_t r = rs + kk;
    const int m = 4 * c;
    const int valid = (r < r_end && m < p.K) ? (int)min(4, p.K - m) : 0;
    cp_async16(smem_u32(hs + (kk * H4 + c) * 16), valid ? p.H + r * p.ldh + m : p.H, valid * 4);
  }
  for (int idx = threadIdx.x; idx < WG_KS * Z4; idx += TC_THREADS) {
    const int kk = idx / Z4, c = idx % Z4;
    const int64_t r = rs + kk;
    const int n = 4 * c;
    const int valid = (r < r_end && n < p.N) ? (int)min(4, p.N - n) : 0;
    const int off = (kk * Z4 + c) * 16;
    cp_async16(smem_u32(zs + off), valid ? p.dZ + r * p.ldz + n : p.dZ, valid * 4);
    if (p.mask) cp_async16(smem_u32(ms + off), valid ? p.mask + r * p.ldm + n : p.mask, valid * 4);
  }
}

__global__ void __launch_bounds__(TC_THREADS, 1) tc_wgrad_kernel(WgArgs p) {
  extern __shared__ __align__(1024) char smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int hs_bytes = WG_KS * TC_M * 4, zs_bytes = WG_KS * p.N_pad * 4;
  const int a_bytes = TC_M * WG_KS * 4, b_bytes = p.N_pad * WG_KS * 4;
  char* hs[2] = {smem, smem + hs_bytes};
  char* zs[2] = {smem + 2 * hs_bytes, smem + 2 * hs_bytes + zs_bytes};
  char* ms[2] = {smem + 2 * hs_bytes + 2 * zs_bytes, smem + 2 * hs_bytes + 3 * zs_bytes};
  char* a_hi = smem + 2 * hs_bytes + 4 * zs_bytes;
  char* a_lo = a_hi + a_bytes;
  char* b_hi = a_lo + a_bytes;
  char* b_lo = b_hi + b_bytes;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(b_lo + b_bytes);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mbar + 1);

  const int64_t r_begin = blockIdx.x * p.rows_per_cta;
  const int64_t r_end = min(p.M, r_begin + p.rows_per_cta);
  const int stages = r_end > r_begin ? (int)ceil_div(r_end - r_begin, WG_KS) : 0;
  if (stages > 0) wg_issue(p, r_begin, r_end, hs[0], zs[0], ms[0]);
  cp_async_commit();
  if (warp == 0) tmem_alloc(tmem_slot, p.tmem_cols);
  if (tid == 0) {
    mbar_init(smem_u32(mbar));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;
  const uint32_t bar = smem_u32(mbar);
  const uint32_t idesc = idesc_tf32(TC_M, p.N_pad, 0, 0);
  const int Z4 = p.N_pad / 4;
  uint32_t phase = 0;
  for (int s = 0; s < stages; ++s) {
    const int buf = s & 1;
    const int64_t rs = r_begin + (int64_t)s * WG_KS;
    if (s + 1 < stages) {
      wg_issue(p, rs + WG_KS, r_end, hs[buf ^ 1], zs[buf ^ 1], ms[buf ^ 1]);
      cp_async_commit();
      cp_async_wait_1();
    } else {
      cp_async_wait_all();
    }
    __syncthreads();
    if (s > 0) {  // the operand buffers are free once the previous stage's MMAs are done
      mbar_wait(bar, phase);
      phase ^= 1;
    }
    // A' chunk (m, 4 rows): column m of 4 staged H rows (+ the ones row m == K)
    const float* H_s = reinterpret_cast<const float*>(hs[buf]);
    for (int idx = tid; idx < TC_M * WG_KC; idx += TC_THREADS) {
      const int m = idx % TC_M, kq = idx / TC_M;
      float e[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int kk = 4 * kq + q;
        e[q] = m == p.K ? (rs + kk < r_end ? 1.f : 0.f) : H_s[kk * TC_M + m];
      }
      split_chunk_to(a_hi, a_lo, kmaj_off(m, 4 * kq, WG_KC), make_float4(e[0], e[1], e[2], e[3]));
    }
    const float* Z_s = reinterpret_cast<const float*>(zs[buf]);
    const float* M_s = reinterpret_cast<const float*>(ms[buf]);
    for (int idx = tid; idx < p.N_pad * WG_KC; idx += TC_THREADS) {
      const int n = idx % p.N_pad, kq = idx / p.N_pad;
      float e[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int kk = 4 * kq + q;
        float x = Z_s[kk * 4 * Z4 + n];
        if (p.mask && !(M_s[kk * 4 * Z4 + n] > 0.f)) x = 0.f;
        e[q] = x;
      }
      split_chunk_to(b_hi, b_lo, kmaj_off(n, 4 * kq, WG_KC), make_float4(e[0], e[1], e[2], e[3]));
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t ah = smem_u32(a_hi), al = smem_u32(a_lo), bh = smem_u32(b_hi), bl = smem_u32(b_lo);
      const uint32_t sbo = WG_KC * 128;
#pragma unroll
      for (int k = 0; k < WG_KS / 8; ++k) {
        mma_tf32(tmem, umma_desc(al + k * 256, 128, sbo), umma_desc(bh + k * 256, 128, sbo), idesc, (s > 0 || k > 0));
        mma_tf32(tmem, umma_desc(ah + k * 256, 128, sbo), umma_desc(bl + k * 256, 128, sbo), idesc, 1);
        mma_tf32(tmem, umma_desc(ah + k * 256, 128, sbo), umma_desc(bh + k * 256, 128, sbo), idesc, 1);
      }
      mma_commit(bar);
    }
  }
  if (stages > 0) {
    mbar_wait(bar, phase);
    phase ^= 1;
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int quarter = warp & 3, half = warp >> 2;
  const int m = quarter * 32 + lane;
  const int chunks = p.N_pad / 16;
  const int c_begin = half == 0 ? 0 : ((chunks + 1) / 2) * 16;
  const int c_end = half == 0 ? ((chunks + 1) / 2) * 16 : p.N_pad;
  float* out = p.part + (int64_t)blockIdx.x * (p.K + 1) * p.N;
  for (int c0 = c_begin; c0 < c_end; c0 += 16) {
    uint32_t v[16];
    tmem_ld16(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)c0, v);
    if (m <= p.K) {
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int n = c0 + q;
        if (n < p.N) out[(int64_t)m * p.N + n] = stages ? __uint_as_float(v[q]) : 0.f;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    tmem_free(tmem, p.tmem_cols);
  }
}

int64_t tc_wgrad_smem(int N_pad) {
  const int64_t hs = (int64_t)WG_KS * TC_M * 4, zs = (int64_t)WG_KS * N_pad * 4;
  return 2 * hs + 4 * zs + 2 * hs + 2 * zs + 64;
}

bool dense_tc_disabled() {
  static const int disabled = [] {
    const char* v = getenv("FGL_DENSE");
    return (v && v[0] == 's') ? 1 : 0;  // FGL_DENSE=simt forces the SIMT kernels
  }();
  return disabled != 0;
}

inline bool aligned16(const void* p) { return !(reinterpret_cast<uintptr_t>(p) & 15); }

}  // namespace

bool tc_gemm(int mode, const float* A, int64_t lda, const float* mask, int64_t ldm, const float* W,
             const float* bias, float* C, int64_t ldc, int64_t M, int N, int K, int relu,
             cudaStream_t st, int* err) {
  *err = 0;
  if (tc_gemm3(mode, A, lda, mask, ldm, W, bias, C, ldc, M, N, K, relu, st, err)) return true;
  if (dense_tc_disabled() || M < 1 || N < 1 || K < 1) return false;
  if ((lda % 4) || !aligned16(A) || (mask && ((ldm % 4) || !aligned16(mask)))) return false;
  const int N_pad = (N + 15) / 16 * 16;
  const int K_pad = (K + 7) / 8 * 8;
  if (N_pad > 256 || K_pad > 256) return false;
  const bool has_mask = mode == 1 && mask;
  int stages = 2;
  if (tc_gemm_smem(mode, has_mask, N_pad, K_pad, 2) > TC_MAX_SMEM) stages = 1;
  const int64_t smem = tc_gemm_smem(mode, has_mask, N_pad, K_pad, stages);
  if (smem > TC_MAX_SMEM) return false;
  int cols = 32;
  while (cols < N_pad) cols <<= 1;
  TcArgs p{A, lda, mask, ldm, W, bias, C, ldc, M, N, K, N_pad, K_pad, relu, cols, stages};
  static bool attr_set[2] = {false, false};
  cudaError_t e;
  if (!attr_set[mode]) {
    e = mode == 0 ? cudaFuncSetAttribute(tc_gemm_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_MAX_SMEM)
                  : cudaFuncSetAttribute(tc_gemm_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_MAX_SMEM);
    if (e != cudaSuccess) { *err = cuda_status(e, "cudaFuncSetAttribute(tc_gemm)"); return true; }
    attr_set[mode] = true;
  }
  const int64_t tiles = ceil_div(M, TC_M);
  const int grid = (int)std::min<int64_t>(tiles, kNumSMs);
  if (mode == 0) FGL_COUNT_LAUNCH(), tc_gemm_kernel<0><<<grid, TC_THREADS, smem, st>>>(p);
  else FGL_COUNT_LAUNCH(), tc_gemm_kernel<1><<<grid, TC_THREADS, smem, st>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) *err = cuda_status(e, "tc_gemm_kernel");
  return true;
}

bool tc_wgrad(const float* H, int64_t ldh, const float* dZ, int64_t ldz, const float* mask, int64_t ldm,
              int64_t M, int K, int N, float* part, int chunks, cudaStream_t st, int* err) {
  *err = 0;
  if (dense_tc_disabled() || M < 1 || K + 1 > TC_M || N < 1) return false;
  if ((ldh % 4) || (ldz % 4) || !aligned16(H) || !aligned16(dZ) || (mask && ((ldm % 4) || !aligned16(mask))))
    return false;
  const int N_pad = (N + 15) / 16 * 16;
  if (N_pad > 256) return false;
  const int64_t smem = tc_wgrad_smem(N_pad);
  if (smem > TC_MAX_SMEM) return false;
  int cols = 32;
  while (cols < N_pad) cols <<= 1;
  static bool attr = false;
  cudaError_t e;
  if (!attr) {
    e = cudaFuncSetAttribute(tc_wgrad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_MAX_SMEM);
    if (e != cudaSuccess) { *err = cuda_status(e, "cudaFuncSetAttribute(tc_wgrad)"); return true; }
    attr = true;
  }
  WgArgs p{H, ldh, dZ, ldz, mask, ldm, part, M, ceil_div(M, chunks), K, N, N_pad, cols};
  FGL_COUNT_LAUNCH(), tc_wgrad_kernel<<<chunks, TC_THREADS, smem, st>>>(p);
  e = cudaGetLastError();
  if (e != cudaSuccess) *err = cuda_status(e, "tc_wgrad_kernel");
  return true;
}

}  // namespace fgl
