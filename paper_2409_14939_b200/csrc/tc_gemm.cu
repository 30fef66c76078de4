// Tensor-core (tcgen05, 5th-gen) dense layer GEMMs with 3xTF32 (sm_100a).
//
// The dense per-layer transform of the reference (compute.dense_update,
// compute.py:198-216, and the dH = dZ W^T of trainer._backward,
// trainer.py:219-221) in fp32 accuracy on the tensor cores: every fp32
// operand x is split x = hi + lo with hi = tf32(x) (round to nearest) and
// lo = x - hi, and  A B ~= A_lo B_hi + A_hi B_lo + A_hi B_hi  is accumulated
// in fp32 in tensor memory (relative error ~1e-6, inside the 1e-5 bar).
//
// Structure (one CTA of 4 warps per SM, persistent over 128-row tiles):
//  * B (the layer weight, <= 256 x 128) is split and staged in shared memory
//    once per CTA in the UMMA K-major canonical layout (no swizzle: 8x16-byte
//    core matrices, LBO = 128 B between the two K halves of an MMA, SBO =
//    KC*128 B between 8-row groups);
//  * each tile's A rows are loaded with 16-byte loads, split hi/lo and stored
//    in the same layout (plus the ReLU mask of dZ for the dgrad variant);
//  * one elected thread issues 3*K/8 tcgen05.mma.kind::tf32 (M=128, N<=256)
//    into a TMEM accumulator and commits to an mbarrier;
//  * the 4 warps drain their 32 TMEM lanes with tcgen05.ld.32x32b.x16, add
//    the bias, apply ReLU and store the rows.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace fgl {
namespace {

constexpr int TC_M = 128;
constexpr int TC_THREADS = 256;
constexpr int TC_LOADS = 8;  // 16-byte A loads in flight per thread
constexpr int TC_MAX_SMEM = 200 * 1024;

struct TcArgs {
  const float* A;      // [M, K] row-major (lda)
  int64_t lda;
  const float* mask;   // dgrad: ReLU mask (layer output), same shape as A, or null
  int64_t ldm;
  const float* W;      // layer weight [din, dout] row-major
  const float* bias;   // fwd: [N] or null
  float* C;            // [M, N] row-major (ldc)
  int64_t ldc;
  int64_t M;
  int N, K, N_pad, K_pad, relu, tmem_cols;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// UMMA shared-memory matrix descriptor, K-major, SWIZZLE_NONE (sm100 version 1)
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

// instruction descriptor: D f32, A/B tf32, both K-major, M x N
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// byte offset of the 16-byte chunk holding (row r, k..k+3) in the canonical layout
__device__ __forceinline__ uint32_t kmaj_off(int r, int k, int KC) {
  return (uint32_t)((r >> 3) * (KC * 128) + (k >> 2) * 128 + (r & 7) * 16 + (k & 3) * 4);
}

__device__ __forceinline__ void split_tf32(float x, float& hi, float& lo) {
  uint32_t h;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(x));
  hi = __uint_as_float(h);
  lo = __fsub_rn(x, hi);
}

__device__ __forceinline__ void store_split4(char* hi_base, char* lo_base, uint32_t off, float4 v) {
  float4 h, l;
  split_tf32(v.x, h.x, l.x);
  split_tf32(v.y, h.y, l.y);
  split_tf32(v.z, h.z, l.z);
  split_tf32(v.w, h.w, l.w);
  *reinterpret_cast<float4*>(hi_base + off) = h;
  *reinterpret_cast<float4*>(lo_base + off) = l;
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n"
      :
      : "r"(d_tmem), "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(bar), "r"(phase)
        : "memory");
  }
}

template <int MODE>  // 0: C = act(A W + b);  1: C = (A * (mask > 0)) W^T
__global__ void __launch_bounds__(TC_THREADS, 1) tc_gemm_kernel(TcArgs p) {
  extern __shared__ __align__(1024) char smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int KC = p.K_pad / 4;
  char* sA_hi = smem;
  char* sA_lo = sA_hi + TC_M * p.K_pad * 4;
  char* sB_hi = sA_lo + TC_M * p.K_pad * 4;
  char* sB_lo = sB_hi + p.N_pad * p.K_pad * 4;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(sB_lo + p.N_pad * p.K_pad * 4);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mbar + 1);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(p.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mbar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  // weight operand B[n][k], split once per CTA
  for (int idx = tid; idx < p.N_pad * p.K_pad; idx += TC_THREADS) {
    const int n = idx / p.K_pad, k = idx % p.K_pad;
    float v = 0.f;
    if (n < p.N && k < p.K) v = MODE == 0 ? p.W[(int64_t)k * p.N + n] : p.W[(int64_t)n * p.K + k];
    float h, l;
    split_tf32(v, h, l);
    const uint32_t off = kmaj_off(n, k, KC);
    *reinterpret_cast<float*>(sB_hi + off) = h;
    *reinterpret_cast<float*>(sB_lo + off) = l;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;
  const uint32_t bar = smem_u32(mbar);
  const uint32_t idesc = idesc_tf32(TC_M, p.N_pad);
  const bool vec = (p.lda % 4 == 0) && !(reinterpret_cast<uintptr_t>(p.A) & 15) &&
                   (MODE == 0 || ((p.ldm % 4 == 0) && !(reinterpret_cast<uintptr_t>(p.mask) & 15)));
  uint32_t phase = 0;
  const int64_t tiles = ceil_div(p.M, TC_M);
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int64_t m0 = t * TC_M;
    // ---- A tile -> shared (hi / lo): TC_LOADS independent 16-byte loads per
    // thread are issued before any of them is split and stored ----
    for (int base = 0; base < TC_M * KC; base += TC_THREADS * TC_LOADS) {
      float4 v[TC_LOADS], mk[TC_LOADS];
#pragma unroll
      for (int u = 0; u < TC_LOADS; ++u) {
        const int idx = base + u * TC_THREADS + tid;
        const int r = idx / KC, k = 4 * (idx % KC);
        const int64_t row = m0 + r;
        v[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        mk[u] = make_float4(1.f, 1.f, 1.f, 1.f);
        if (idx < TC_M * KC && row < p.M && k < p.K) {
          const float* src = p.A + row * p.lda + k;
          if (vec && k + 3 < p.K) {
            v[u] = __ldg(reinterpret_cast<const float4*>(src));
            if (MODE == 1 && p.mask) mk[u] = __ldg(reinterpret_cast<const float4*>(p.mask + row * p.ldm + k));
          } else {
            float e[4], g[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              e[q] = (k + q < p.K) ? src[q] : 0.f;
              g[q] = (MODE == 1 && p.mask && k + q < p.K) ? p.mask[row * p.ldm + k + q] : 1.f;
            }
            v[u] = make_float4(e[0], e[1], e[2], e[3]);
            mk[u] = make_float4(g[0], g[1], g[2], g[3]);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < TC_LOADS; ++u) {
        const int idx = base + u * TC_THREADS + tid;
        if (idx >= TC_M * KC) continue;
        float4 x = v[u];
        if (MODE == 1) {
          if (!(mk[u].x > 0.f)) x.x = 0.f;
          if (!(mk[u].y > 0.f)) x.y = 0.f;
          if (!(mk[u].z > 0.f)) x.z = 0.f;
          if (!(mk[u].w > 0.f)) x.w = 0.f;
        }
        store_split4(sA_hi, sA_lo, kmaj_off(idx / KC, 4 * (idx % KC), KC), x);
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    // ---- MMA issue (one thread) ----
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t a_hi = smem_u32(sA_hi), a_lo = smem_u32(sA_lo);
      const uint32_t b_hi = smem_u32(sB_hi), b_lo = smem_u32(sB_lo);
      const uint32_t sbo = KC * 128;
      const int steps = p.K_pad / 8;
      uint32_t acc = 0;
      for (int s = 0; s < steps; ++s) {  // small terms first
        mma_tf32(tmem, umma_desc(a_lo + s * 256, 128, sbo), umma_desc(b_hi + s * 256, 128, sbo), idesc, acc);
        acc = 1;
        mma_tf32(tmem, umma_desc(a_hi + s * 256, 128, sbo), umma_desc(b_lo + s * 256, 128, sbo), idesc, 1);
      }
      for (int s = 0; s < steps; ++s)
        mma_tf32(tmem, umma_desc(a_hi + s * 256, 128, sbo), umma_desc(b_hi + s * 256, 128, sbo), idesc, 1);
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
                   : "memory");
    }
    mbar_wait(bar, phase);
    phase ^= 1;
    asm volatile("tcgen05.fence::after_thread_sync;");
    // ---- epilogue: TMEM lanes 32w.. -> rows ----
    // warp w drains TMEM lane quarter w%4 (rows) and column half w/4
    const int quarter = warp & 3, half = warp >> 2;
    const int64_t row = m0 + quarter * 32 + lane;
    const int chunks = p.N_pad / 16;
    const int c_begin = half == 0 ? 0 : ((chunks + 1) / 2) * 16;
    const int c_end = half == 0 ? ((chunks + 1) / 2) * 16 : p.N_pad;
    for (int c0 = c_begin; c0 < c_end; c0 += 16) {
      uint32_t v[16];
      const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)c0;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (row < p.M) {
        float* out = p.C + row * p.ldc;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int col = c0 + j;
          if (col < p.N) {
            float x = __uint_as_float(v[j]);
            if (MODE == 0 && p.bias) x = __fadd_rn(x, p.bias[col]);
            if (p.relu) x = x > 0.f ? x : 0.f;
            out[col] = x;
          }
        }
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();  // TMEM drained and shared A free before the next tile
  }
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(p.tmem_cols));
  }
}

// ---------------------------------------------------------------- wgrad --
// Partial [dW; db] of a row chunk: D[m][n] = sum_r A'[m][r] B'[n][r] with
// A'[m][r] = H[r][m] (m < K), 1 (m == K: the bias row), B'[n][r] = dZ[r][n] *
// (Xout[r][n] > 0).  The row dimension is the MMA K dimension, consumed in
// stages of 32 rows through a 2-deep shared-memory ring (the loads of stage
// s+1 overlap the MMAs of stage s); partials of all CTAs are summed by
// reduce_partials_kernel in a fixed order (deterministic).
constexpr int WG_KS = 32;  // rows per stage (MMA K)

struct WgArgs {
  const float* H; int64_t ldh;
  const float* dZ; int64_t ldz;
  const float* mask; int64_t ldm;
  float* part;          // [chunks][K+1][N]
  int64_t M;            // rows
  int64_t rows_per_cta;
  int K, N, N_pad, tmem_cols;
};

__global__ void __launch_bounds__(TC_THREADS, 1) tc_wgrad_kernel(WgArgs p) {
  extern __shared__ __align__(1024) char smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int KC = WG_KS / 4;
  const int a_bytes = TC_M * WG_KS * 4, b_bytes = p.N_pad * WG_KS * 4;
  const int stage_bytes = 2 * a_bytes + 2 * b_bytes;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + 2 * stage_bytes);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mbar + 2);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(p.tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mbar)), "r"(1));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mbar + 1)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;
  const uint32_t idesc = idesc_tf32(TC_M, p.N_pad);
  const int64_t r_begin = blockIdx.x * p.rows_per_cta;
  const int64_t r_end = min(p.M, r_begin + p.rows_per_cta);
  const int stages = r_end > r_begin ? (int)ceil_div(r_end - r_begin, WG_KS) : 0;
  uint32_t phase[2] = {0, 0};
  for (int s = 0; s < stages; ++s) {
    const int buf = s & 1;
    char* a_hi = smem + buf * stage_bytes;
    char* a_lo = a_hi + a_bytes;
    char* b_hi = a_lo + a_bytes;
    char* b_lo = b_hi + b_bytes;
    if (s >= 2) {  // MMAs of stage s-2 must be done with this buffer
      mbar_wait(smem_u32(mbar + buf), phase[buf]);
      phase[buf] ^= 1;
    }
    const int64_t rs = r_begin + (int64_t)s * WG_KS;
    // A'[m][r]: item = (m, kq) gathers rows rs+4kq..+3 of column m
    for (int it = tid; it < TC_M * KC; it += TC_THREADS) {
      const int m = it % TC_M, kq = it / TC_M;
      float e[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t r = rs + 4 * kq + q;
        float x = 0.f;
        if (r < r_end) x = m < p.K ? p.H[r * p.ldh + m] : (m == p.K ? 1.f : 0.f);
        e[q] = x;
      }
      store_split4(a_hi, a_lo, kmaj_off(m, 4 * kq, KC), make_float4(e[0], e[1], e[2], e[3]));
    }
    for (int it = tid; it < p.N_pad * KC; it += TC_THREADS) {
      const int n = it % p.N_pad, kq = it / p.N_pad;
      float e[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t r = rs + 4 * kq + q;
        float x = 0.f;
        if (r < r_end && n < p.N) {
          x = p.dZ[r * p.ldz + n];
          if (p.mask && !(p.mask[r * p.ldm + n] > 0.f)) x = 0.f;
        }
        e[q] = x;
      }
      store_split4(b_hi, b_lo, kmaj_off(n, 4 * kq, KC), make_float4(e[0], e[1], e[2], e[3]));
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t ah = smem_u32(a_hi), al = smem_u32(a_lo), bh = smem_u32(b_hi), bl = smem_u32(b_lo);
      const uint32_t sbo = KC * 128;
#pragma unroll
      for (int k = 0; k < WG_KS / 8; ++k) {
        mma_tf32(tmem, umma_desc(al + k * 256, 128, sbo), umma_desc(bh + k * 256, 128, sbo), idesc,
                 (s > 0 || k > 0) ? 1u : 0u);
        mma_tf32(tmem, umma_desc(ah + k * 256, 128, sbo), umma_desc(bl + k * 256, 128, sbo), idesc, 1u);
        mma_tf32(tmem, umma_desc(ah + k * 256, 128, sbo), umma_desc(bh + k * 256, 128, sbo), idesc, 1u);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                       smem_u32(mbar + buf))
                   : "memory");
    }
  }
  // drain: wait for the last (up to two) outstanding commits
  for (int s = stages >= 2 ? stages - 2 : 0; s < stages; ++s) {
    const int buf = s & 1;
    mbar_wait(smem_u32(mbar + buf), phase[buf]);
    phase[buf] ^= 1;
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
    const uint32_t taddr = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (m <= p.K) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int n = c0 + j;
        if (n < p.N) out[(int64_t)m * p.N + n] = stages ? __uint_as_float(v[j]) : 0.f;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(p.tmem_cols));
  }
}

inline int64_t tc_smem_bytes(int N_pad, int K_pad) {
  return 4ll * K_pad * (2 * TC_M + 2 * N_pad) + 64;
}

}  // namespace

// Host-side dispatch; returns false when the shape is outside the kernel's
// envelope (caller falls back to the SIMT kernels).
bool tc_gemm(int mode, const float* A, int64_t lda, const float* mask, int64_t ldm, const float* W,
             const float* bias, float* C, int64_t ldc, int64_t M, int N, int K, int relu,
             cudaStream_t st, int* err) {
  *err = 0;
  static const int disabled = [] {
    const char* v = getenv("FGL_DENSE");
    return (v && v[0] == 's') ? 1 : 0;  // FGL_DENSE=simt forces the SIMT kernels
  }();
  if (disabled || M < 1 || N < 1 || K < 1) return false;
  const int N_pad = (N + 15) / 16 * 16;
  const int K_pad = (K + 7) / 8 * 8;
  if (N_pad > 256 || K_pad > 256) return false;
  const int64_t smem = tc_smem_bytes(N_pad, K_pad);
  if (smem > TC_MAX_SMEM) return false;
  int cols = 32;
  while (cols < N_pad) cols <<= 1;
  TcArgs p{A, lda, mask, ldm, W, bias, C, ldc, M, N, K, N_pad, K_pad, relu, cols};
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

// [dW; db] partials over `chunks` row chunks into part[chunks][K+1][N];
// false when the shape is outside the kernel's envelope.
bool tc_wgrad(const float* H, int64_t ldh, const float* dZ, int64_t ldz, const float* mask, int64_t ldm,
              int64_t M, int K, int N, float* part, int chunks, cudaStream_t st, int* err) {
  *err = 0;
  static const int disabled = [] {
    const char* v = getenv("FGL_DENSE");
    return (v && v[0] == 's') ? 1 : 0;
  }();
  if (disabled || M < 1 || K + 1 > TC_M || N < 1) return false;
  const int N_pad = (N + 15) / 16 * 16;
  if (N_pad > 256) return false;
  const int64_t smem = 2ll * (2 * TC_M * WG_KS * 4 + 2 * N_pad * WG_KS * 4) + 64;
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
