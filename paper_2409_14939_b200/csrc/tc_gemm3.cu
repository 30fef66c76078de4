// Warp-specialised bulk-copy + tcgen05 3xTF32 dense layer GEMM (sm_100a).
//
// Same contract as tc_gemm.cu's tc_gemm_kernel (compute.dense_update,
// compute.py:198-216, and dH = (dZ * relu'(z)) W^T of trainer._backward,
// trainer.py:212-228), organised so that the HBM stream of activation rows
// never waits on the math and shared memory is not the bottleneck:
//
//   warp 0      producer: one 1-D bulk copy (TMA engine) per 128-row tile of
//               A -- the rows are contiguous, so a tile is a single request --
//               (and of the ReLU mask for dgrad) into a ring of R raw slots;
//   warps 4-7   converters, thread = row = TMEM lane: read the row from shared
//               memory (conflict-free 16-byte loads for ld = 4 mod 8 floats),
//               mask, split x = hi + lo (hi = tf32(x)), and tcgen05.st both
//               halves into a TMEM A buffer (double-buffered when it fits);
//   warp 1      MMA issuer (one thread): per 8-wide K step three
//               tcgen05.mma.kind::tf32 with A from TMEM and the split weight
//               from shared memory (lo*hi, hi*lo, hi*hi) -> fp32 accumulator;
//   warps 8-11  epilogue: tcgen05.ld the accumulator, bias, ReLU, stores.
//
// Because A never sits in shared memory in MMA layout, shared-memory traffic
// per tile is just the raw rows in and out once plus the weight reads.
// The weight (K <= 128 here, N <= 256) is split once per CTA into hi/lo
// copies in the K-major no-swizzle canonical layout.  One persistent CTA/SM.
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "tcgen05.cuh"

namespace fgl {
namespace {
using namespace tc;

constexpr int G3_THREADS = 512;      // 16 warps, see the role map at the top
constexpr int G3_M = 128;
constexpr int G3_KCH = 32;           // K columns per TMEM A chunk (hi 32 + lo 32 TMEM columns)
constexpr int G3_MAX_SMEM = 227 * 1024;
constexpr int G3_MAX_SLOTS = 4;
constexpr int G3_CONV_THREADS = 256; // warps 4-11
constexpr int G3_EPI_THREADS = 128;  // warps 12-15

struct G3Args {
  const float* A;      // [M, K] row-major (lda)
  const float* mask;   // dgrad: [M, K] (ldm) ReLU mask, or null
  const float* W;      // mode 0: [K, N] row-major; mode 1: [N, K] row-major
  const float* bias;   // mode 0 only, [N] or null
  float* C;
  int64_t lda, ldm, ldc;
  int64_t M;
  int N, K, N_pad, K_pad, R, NC, relu, has_mask, tmem_cols, a_slot_bytes, m_slot_bytes, dbg;
  int stage_off, stage_pitch, w_vec;  // coalesced-epilogue staging tile (byte offset in smem, pitch in floats), or -1
  int accum;  // C += (earlier K slices already in C)
  int a_tma;  // A (and mask) tiles by TMA tensor copies of a column slice (rows of a_lds floats in smem)
  int a_lds;  // smem row stride of an A tile, floats (= lda for whole-row bulk copies)
  int m_lds;  // smem row stride of a mask tile, floats (= ldm for whole-row bulk copies)
  int64_t ldw;  // W row stride, floats
};

// debug timeline (FGL_G3DBG & 8): per CTA, globaltimer stamps of each role's
// progress; read back with fgl_debug_g3_trace
constexpr int G3_TR = 72;
__device__ int64_t g3_trace[148 * G3_TR];
__device__ __forceinline__ int64_t gtime() {
  int64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define G3T(slot) do { if ((p.dbg & 8) && blockIdx.x < 148 && (slot) < G3_TR) g3_trace[blockIdx.x * G3_TR + (slot)] = gtime(); } while (0)

__device__ __forceinline__ uint32_t sw128_off(int row, int kk) {
  // byte offset of element (row, kk) (kk < 32) inside a K-major SWIZZLE_128B box
  return (uint32_t)((row >> 3) * 1024 + (row & 7) * 128 + ((((kk >> 2) ^ (row & 7))) << 4) + (kk & 3) * 4);
}

__device__ __forceinline__ float tf32_rna_finite(float x) {
  // round-to-nearest(-away) to tf32 for finite x: 2 integer ops (cvt.rna.tf32
  // adds an inf/nan guard that activations never need)
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xffffe000u);
}

// the weight operand B[n][k] split into tf32 hi / lo K-major SWIZZLE_128B
// boxes of 32 K columns, by `nt` threads (t0 = 0..nt-1); 4x4 blocks over
// [N_pad x K_pad] (padding included: no zeroing pass), four 16-byte W loads,
// a register transpose for mode 0 (B = W^T), eight 16-byte shared stores
template <int MODE, bool SRC_SMEM = false>
__device__ __forceinline__ void split_weight_image(const float* __restrict__ W, int64_t ldw, int K, int N, int K_pad,
                                                   int N_pad, bool vec, char* sB_hi, char* sB_lo, int t0, int nt) {
  const int b_box = N_pad * 128;
  const int K4 = K_pad >> 2, N4 = N_pad >> 2, nblk = K4 * N4;
  const int rl = MODE == 0 ? N : K;  // W row length
  const int wr = MODE == 0 ? K : N;  // W rows
  auto wload = [&](int r, int c) {   // W[r][c..c+3], zero outside
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (r < wr && c < rl) {
      const float* src = W + (int64_t)r * ldw + c;
      if (SRC_SMEM) v = *reinterpret_cast<const float4*>(src);  // TMA-staged box: zero-filled past the edge
      else if (vec && c + 3 < rl) v = __ldg(reinterpret_cast<const float4*>(src));
      else {
        v.x = __ldg(src);
        if (c + 1 < rl) v.y = __ldg(src + 1);
        if (c + 2 < rl) v.z = __ldg(src + 2);
        if (c + 3 < rl) v.w = __ldg(src + 3);
      }
    }
    return v;
  };
  constexpr int PER = 2;
  for (int b0 = t0; b0 < nblk; b0 += PER * nt) {
    float4 w[PER][4];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int b = b0 + u * nt;
      const int k4 = b % K4, n4 = b / K4;
#pragma unroll
      for (int i = 0; i < 4; ++i)
        w[u][i] = b < nblk ? (MODE == 0 ? wload(4 * k4 + i, 4 * n4) : wload(4 * n4 + i, 4 * k4))
                           : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int b = b0 + u * nt;
      if (b >= nblk) break;
      const int k4 = b % K4, n4 = b / K4;
      float4 r4[4];  // r4[jn] = B[4 n4 + jn][4 k4 .. 4 k4 + 3]
      if (MODE == 0) {
        r4[0] = make_float4(w[u][0].x, w[u][1].x, w[u][2].x, w[u][3].x);
        r4[1] = make_float4(w[u][0].y, w[u][1].y, w[u][2].y, w[u][3].y);
        r4[2] = make_float4(w[u][0].z, w[u][1].z, w[u][2].z, w[u][3].z);
        r4[3] = make_float4(w[u][0].w, w[u][1].w, w[u][2].w, w[u][3].w);
      } else {
#pragma unroll
        for (int jn = 0; jn < 4; ++jn) r4[jn] = w[u][jn];
      }
#pragma unroll
      for (int jn = 0; jn < 4; ++jn) {
        const int n = 4 * n4 + jn, k = 4 * k4;
        float4 h4, l4;
        h4.x = tf32_hi(r4[jn].x); l4.x = __fsub_rn(r4[jn].x, h4.x);
        h4.y = tf32_hi(r4[jn].y); l4.y = __fsub_rn(r4[jn].y, h4.y);
        h4.z = tf32_hi(r4[jn].z); l4.z = __fsub_rn(r4[jn].z, h4.z);
        h4.w = tf32_hi(r4[jn].w); l4.w = __fsub_rn(r4[jn].w, h4.w);
        const uint32_t off = (uint32_t)((k >> 5) * b_box) + sw128_off(n, k & 31);
        sts128(smem_u32(sB_hi) + off, h4);
        sts128(smem_u32(sB_lo) + off, l4);
      }
    }
  }
}

template <int MODE>
__global__ void __launch_bounds__(G3_THREADS, 1) tc_gemm3_kernel(const __grid_constant__ CUtensorMap tmC,
                                                                 const __grid_constant__ CUtensorMap tmA,
                                                                 const __grid_constant__ CUtensorMap tmM, G3Args p) {
  extern __shared__ __align__(1024) char smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int R = p.R, NC = p.NC, N_pad = p.N_pad, K_pad = p.K_pad;
  const int nch = (p.K + G3_KCH - 1) / G3_KCH;  // K chunks per tile
  const int b_box = N_pad * 128, KB = (K_pad + 31) / 32;
  const int b_bytes = KB * b_box;
  char* sB_hi = smem;
  char* sB_lo = sB_hi + b_bytes;
  char* slots = sB_lo + b_bytes;
  const int slot_bytes = p.a_slot_bytes + p.m_slot_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(slots + R * slot_bytes);
  // full[R] empty[R] cfull[8] cempty[8] tfull[2] tempty[2] bready cacc
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * R + 22);
  float* sbias = reinterpret_cast<float*>(tmem_slot + 4);
  auto bar = [&](int i) { return smem_u32(bars + i); };
  const int FULL = 0, EMPTY = R, CFULL = 2 * R, CEMPTY = 2 * R + 8, TFULL = 2 * R + 16, TEMPTY = 2 * R + 18,
            BREADY = 2 * R + 20, CACC = 2 * R + 21;

  if (tid == 0) {
    G3T(0);
    for (int s = 0; s < R; ++s) {
      mbar_init_n(bar(FULL + s), 1);
      mbar_init_n(bar(EMPTY + s), G3_CONV_THREADS);
    }
    for (int c = 0; c < 8; ++c) {
      mbar_init_n(bar(CFULL + c), G3_CONV_THREADS / 2);
      mbar_init_n(bar(CEMPTY + c), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init_n(bar(TFULL + a), 1);
      mbar_init_n(bar(TEMPTY + a), G3_EPI_THREADS);
    }
    mbar_init_n(bar(BREADY), 1);
    mbar_init_n(bar(CACC), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();  // barriers initialised
  const int64_t tiles = ceil_div(p.M, G3_M);
  if (warp == 0) {
    // --------------------------------------------------------- producer --
    if (lane == 0) {
      int j = 0;
      for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++j) {
        const int s = j % R;
        mbar_wait(bar(EMPTY + s), ((uint32_t)(j / R) & 1u) ^ 1u);
        G3T(2 + 9 * j);
        const int64_t r0 = t * G3_M;
        const int rows = (int)(p.M - r0 < G3_M ? p.M - r0 : G3_M);
        const uint32_t abytes = p.a_tma ? (uint32_t)(G3_M * p.a_lds * 4) : (uint32_t)(rows * p.lda * 4);
        const uint32_t mbytes = !p.has_mask ? 0u : p.a_tma ? (uint32_t)(G3_M * p.m_lds * 4) : (uint32_t)(rows * p.ldm * 4);
        char* slot = slots + s * slot_bytes;
        mbar_arrive_expect_tx(bar(FULL + s), abytes + mbytes);
        if (p.a_tma) tma_load_2d(smem_u32(slot), &tmA, 0, (int)r0, bar(FULL + s));  // OOB rows / cols: zeros
        else bulk_load(smem_u32(slot), p.A + r0 * p.lda, abytes, bar(FULL + s));
        if (p.has_mask) {
          if (p.a_tma) tma_load_2d(smem_u32(slot + p.a_slot_bytes), &tmM, 0, (int)r0, bar(FULL + s));
          else bulk_load(smem_u32(slot + p.a_slot_bytes), p.mask + r0 * p.ldm, mbytes, bar(FULL + s));
        }
      }
    }
    return;
  }
  // TMEM allocation (warp 1), published to warps 1-15
  if (warp == 1) tmem_alloc(tmem_slot, p.tmem_cols);
  tc_fence_before();
  asm volatile("bar.sync 1, %0;" ::"r"(G3_THREADS - 32) : "memory");
  tc_fence_after();
  if (warp == 2 || warp == 3 || warp >= 12) {
    // weight operand B[n][k] split into tf32 hi / lo, K-major SWIZZLE_128B
    // boxes of 32 K columns (conflict-free tensor-core reads), by warps 2-3
    // and the epilogue warps 12-15 while the producer streams A and the
    // converters already convert it; the MMA issuer waits on BREADY.  Work
    // item = 4x4 block (n 4n4.., k 4k4..) over [N_pad x K_pad] (covers every
    // element the MMA reads, padding included, so no zeroing pass): four
    // 16-byte W loads, a register transpose (mode 0: B = W^T), eight 16-byte
    // shared stores; consecutive threads take consecutive k4 (conflict-free).
    const int nt = 192, t0 = warp < 4 ? tid - 64 : tid - 384 + 64;
    split_weight_image<MODE>(p.W, p.ldw, p.K, p.N, K_pad, N_pad, p.w_vec, sB_hi, sB_lo, t0, nt);
    fence_async_smem();
    asm volatile("bar.sync 3, %0;" ::"r"(nt) : "memory");
    if (t0 == 0) {
      G3T(1);
      mbar_arrive(bar(BREADY));
    }
  }
  const uint32_t tmem = *tmem_slot;
  // TMEM columns: accumulators [0, 2 N_pad), A chunk c: hi at 2 N_pad + 64 c, lo at +32
  auto acc_col = [&](int a) { return tmem + (uint32_t)(a * N_pad); };
  auto ch_hi = [&](int c) { return tmem + (uint32_t)(2 * N_pad + 2 * G3_KCH * c); };

  if (warp == 1) {
    // -------------------------------------------------------- MMA issuer --
    // the whole warp runs the (warp-uniform) loop so descriptors live in
    // uniform registers; one elected lane issues each tcgen05 instruction
    const uint32_t idesc = idesc_tf32(G3_M, N_pad, 0, 0);
    const uint32_t bh = smem_u32(sB_hi), bl = smem_u32(sB_lo);
    mbar_wait(bar(BREADY), 0);  // weight images split
    tc_fence_after();
    int j = 0, cc = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++j) {
      const int a = j & 1;
      mbar_wait(bar(TEMPTY + a), ((uint32_t)(j >> 1) & 1u) ^ 1u);
      tc_fence_after();
      if (lane == 0) G3T(5 + 9 * j);
      for (int c = 0; c < nch; ++c, ++cc) {
        const int cs = cc % NC;
        mbar_wait(bar(CFULL + cs), (uint32_t)(cc / NC) & 1u);
        if (j == 1 && c < 4 && lane == 0) G3T(65 + c);
        tc_fence_after();
        const int kst = min(G3_KCH, K_pad - c * G3_KCH) / 8;
        const uint32_t ahi = ch_hi(cs), alo = ahi + G3_KCH;
        const uint32_t bo0 = (uint32_t)(c * b_box);  // chunk c = SW128 box c of B
        if (elect_one()) {
          for (int st = 0; st < ((p.dbg & 2) ? 0 : kst); ++st) {
            const uint32_t bo = bo0 + (uint32_t)(st * 32);
            const uint64_t dbh = umma_desc_sw128(bh + bo), dbl = umma_desc_sw128(bl + bo);
            const uint32_t acc = (c | st) != 0;
            if (!(p.dbg & 32)) {
              mma_tf32_ts(acc_col(a), alo + 8 * st, dbh, idesc, acc);
              mma_tf32_ts(acc_col(a), ahi + 8 * st, dbl, idesc, 1);
            }
            mma_tf32_ts(acc_col(a), ahi + 8 * st, dbh, idesc, (p.dbg & 32) ? acc : 1u);
          }
          mma_commit(bar(CEMPTY + cs));
        }
        __syncwarp();
      }
      if (elect_one()) mma_commit(bar(TFULL + a));
      __syncwarp();
    }
  } else if (warp >= 4 && warp < 12) {
    // -------------------------------------------------------- converters --
    // two groups of 4 warps (thread = row = TMEM lane) take alternate 32-column
    // chunks, so one group's TMEM-store latency overlaps the other's loads
    const int quarter = warp & 3, grp = (warp - 4) >> 2, row = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    int j = 0, cc = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++j) {
      const int s = j % R;
      mbar_wait(bar(FULL + s), (uint32_t)(j / R) & 1u);
      if (row == 0 && grp == 0) G3T(3 + 9 * j);
      const uint32_t xr = smem_u32(slots + s * slot_bytes) + (uint32_t)(row * p.a_lds * 4);
      const uint32_t mr = smem_u32(slots + s * slot_bytes + p.a_slot_bytes) + (uint32_t)(row * p.m_lds * 4);
      for (int c = 0; c < nch; ++c, ++cc) {
        if ((cc & 1) != grp) continue;
        const int cs = cc % NC;
        uint32_t hv[32], lv[32];
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int k0 = c * G3_KCH + 16 * hh;
          // four 16-byte loads in flight before any conversion
          float4 x[4], m[4];
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const int k = k0 + 4 * h;
            x[h] = k < p.K ? lds128(xr + 4 * k) : make_float4(0.f, 0.f, 0.f, 0.f);
            if (MODE == 1 && p.has_mask) m[h] = k < p.K ? lds128(mr + 4 * k) : make_float4(0.f, 0.f, 0.f, 0.f);
          }
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const int k = k0 + 4 * h;
            float xs[4] = {x[h].x, x[h].y, x[h].z, x[h].w};
            if (MODE == 1 && p.has_mask) {
              const float ms[4] = {m[h].x, m[h].y, m[h].z, m[h].w};
#pragma unroll
              for (int q = 0; q < 4; ++q)
                if (!(ms[q] > 0.f)) xs[q] = 0.f;
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              if (k + q >= p.K) xs[q] = 0.f;  // columns K..K_pad-1 are zero (row padding may hold anything)
              const float hi = tf32_rna_finite(xs[q]);
              hv[16 * hh + 4 * h + q] = __float_as_uint(hi);
              lv[16 * hh + 4 * h + q] = __float_as_uint(__fsub_rn(xs[q], hi));
            }
          }
        }
        mbar_wait(bar(CEMPTY + cs), ((uint32_t)(cc / NC) & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t hi_t = ch_hi(cs) + lane_off;
        if (!(p.dbg & 1)) {
          tmem_st32(hi_t, hv);
          tmem_st32(hi_t + G3_KCH, lv);
          tmem_st_wait();
        }
        tc_fence_before();
        mbar_arrive(bar(CFULL + cs));
      }
      if (row == 0 && grp == 0) G3T(4 + 9 * j);
      mbar_arrive(bar(EMPTY + s));  // raw slot consumed
    }
  } else if (warp >= 12) {
    // ---------------------------------------------------------- epilogue --
    // TMEM -> registers (thread = row) -> bias / ReLU -> shared staging tile
    // in the SWIZZLE_128B box layout (conflict-free: a row's 16-byte chunks
    // are XOR-permuted by row & 7) -> TMA tensor stores, one per 32 columns
    const int quarter = warp & 3, et = tid - (G3_THREADS - G3_EPI_THREADS);
    const bool tma_out = p.stage_off >= 0;
    const uint32_t stg_u = tma_out ? smem_u32(smem + p.stage_off) : 0u;
    for (int c = et; c < N_pad; c += G3_EPI_THREADS) sbias[c] = (MODE == 0 && p.bias && c < p.N) ? p.bias[c] : 0.f;
    asm volatile("bar.sync 2, 128;" ::: "memory");
    int j = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++j) {
      const int a = j & 1;
      mbar_wait(bar(TFULL + a), (uint32_t)(j >> 1) & 1u);
      tc_fence_after();
      if (et == 0) G3T(6 + 9 * j);
      const int r_loc = quarter * 32 + lane;
      const int64_t row = t * G3_M + r_loc;
      float* out = p.C + row * p.ldc;
      if (tma_out && j > 0) {
        // the previous tile's TMA stores must have finished reading staging
        if (et == 0) bulk_wait_read0();
        asm volatile("bar.sync 2, 128;" ::: "memory");
      }
      const bool acc_stage = p.accum && tma_out;
      if (acc_stage) {
        // K split: the earlier slices' sum arrives in the staging boxes by TMA
        // (same SW128 layout the stores use: conflict-free, coalesced)
        if (et == 0) {
          const int nbox = (N_pad + 31) / 32;
          mbar_arrive_expect_tx(bar(CACC), (uint32_t)(nbox * G3_M * 128));
          for (int b = 0; b < nbox; ++b)
            tma_load_2d(stg_u + (uint32_t)(b * G3_M * 128), &tmC, 32 * b, (int)(t * G3_M), bar(CACC));
        }
        mbar_wait(bar(CACC), (uint32_t)j & 1u);
      }
      for (int c0 = 0; c0 < N_pad; c0 += 32) {
        uint32_t v[32];
        if (p.dbg & 4) { for (int q = 0; q < 32; ++q) v[q] = 0; } else {
        tmem_ld16_nowait(acc_col(a) + ((uint32_t)(quarter * 32) << 16) + (uint32_t)c0, v);
        if (c0 + 16 < N_pad)
          tmem_ld16_nowait(acc_col(a) + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(c0 + 16), v + 16);
        tmem_ld_wait(); }
        const int ncol = c0 + 16 < N_pad ? 32 : 16;
        for (int h = 0; h < ncol; h += 16) {
          float x[16];
          float prev[16];
          if (acc_stage) {
            const uint32_t box = stg_u + (uint32_t)((c0 >> 5) * (G3_M * 128)) + (uint32_t)(r_loc * 128);
#pragma unroll
            for (int q = 0; q < 16; q += 4) {
              const int cc = (h + q) >> 2;
              const float4 pv = lds128(box + (uint32_t)(((cc ^ (r_loc & 7)) & 7) << 4));
              prev[q] = pv.x; prev[q + 1] = pv.y; prev[q + 2] = pv.z; prev[q + 3] = pv.w;
            }
          } else if (p.accum) {  // K split without staging: row-contiguous loads
#pragma unroll
            for (int q = 0; q < 16; ++q)
              prev[q] = (row < p.M && c0 + h + q < p.N) ? out[c0 + h + q] : 0.f;
          }
#pragma unroll
          for (int q = 0; q < 16; ++q) {
            float y = __uint_as_float(v[h + q]);
            if (p.accum) y = __fadd_rn(prev[q], y);
            if (MODE == 0 && p.bias) y = __fadd_rn(y, sbias[c0 + h + q]);
            if (p.relu) y = y > 0.f ? y : 0.f;
            x[q] = y;
          }
          if (tma_out) {
            // box (c0 / 32): 128 rows x 128 B; chunk cc of row r at (cc ^ (r & 7))
            const uint32_t box = stg_u + (uint32_t)((c0 >> 5) * (G3_M * 128)) + (uint32_t)(r_loc * 128);
#pragma unroll
            for (int q = 0; q < 16; q += 4) {
              const int cc = (h + q) >> 2;
              sts128(box + (uint32_t)(((cc ^ (r_loc & 7)) & 7) << 4), make_float4(x[q], x[q + 1], x[q + 2], x[q + 3]));
            }
          } else if (row < p.M) {
            if (((reinterpret_cast<uintptr_t>(p.C) | (uintptr_t)(p.ldc * 4)) & 15) == 0) {
#pragma unroll
              for (int q = 0; q < 16; q += 4) {
                const int col = c0 + h + q;
                if (col + 3 < p.N) *reinterpret_cast<float4*>(out + col) = make_float4(x[q], x[q + 1], x[q + 2], x[q + 3]);
                else
                  for (int u = 0; u < 4; ++u)
                    if (col + u < p.N) out[col + u] = x[q + u];
              }
            } else {
#pragma unroll
              for (int q = 0; q < 16; ++q)
                if (c0 + h + q < p.N) out[c0 + h + q] = x[q];
            }
          }
        }
      }
      if (et == 0) G3T(8 + 9 * j);
      tc_fence_before();
      mbar_arrive(bar(TEMPTY + a));  // accumulator drained: tile j+2's MMAs may start
      if (tma_out) {
        fence_async_smem();
        asm volatile("bar.sync 2, 128;" ::: "memory");
        if (et == 0) {
          for (int c0 = 0; c0 < N_pad; c0 += 32)
            tma_store_2d(&tmC, stg_u + (uint32_t)((c0 >> 5) * (G3_M * 128)), c0, (int)(t * G3_M));
          bulk_commit();
        }
      }
      if (et == 0) G3T(7 + 9 * j);
    }
    if (tma_out && et == 0) bulk_wait0();
  }
  // warps 1-15 (warp 0 returned after issuing its copies)
  tc_fence_before();
  asm volatile("bar.sync 1, %0;" ::"r"(G3_THREADS - 32) : "memory");
  if (warp == 1) {
    tc_fence_after();
    tmem_free(tmem, p.tmem_cols);
  }
  if (tid == 32) G3T(G3_TR - 1);
}

// ------------------------------------------------------------------ wgrad --
// Weight-gradient partials on the tensor cores: D[m][n] = sum_r A'[m][r] B'[n][r]
// with A'[m][r] = H[r][m] (m < K), 1 (m == K: the db row), B'[n][r] =
// dZ[r][n] * (mask[r][n] > 0).  The reduction dimension r (rows) is the MMA
// K dimension, so both operands need a transpose, done by the converters on
// their way into the MMA operands:
//   warp 0      producer: bulk copies of 64-row tiles of H, dZ, mask;
//   warps 4-11  converters: per 32-row chunk, thread = feature m = TMEM lane:
//               16 rows of column m (conflict-free 4-byte shared loads) ->
//               tf32 hi/lo -> tcgen05.st into the A chunk ring; and the dZ
//               columns -> hi/lo K-major SWIZZLE_128B boxes in shared memory;
//   warp 1      MMA: 4 K steps x 3 tcgen05.mma per chunk into ONE accumulator
//               that lives for the CTA's whole row range;
//   warps 12-15 epilogue: the CTA's [K+1][N] partial -> global (summed by
//               reduce_partials_kernel, deterministic order).
constexpr int WG3_MT = 64;   // rows per bulk-copied tile
constexpr int WG3_NC = 3;    // A / B chunk ring depth (32 rows each; 3 leaves room for 3 raw slots)
constexpr int WG3_R_MAX = 4; // raw tile slots (as many as fit)

struct Wg3Args {
  const float* H; const float* dZ; const float* mask;
  int64_t ldh, ldz, ldm;
  float* part;         // [gridDim.x][N][K+1] (feature-major)
  int64_t M;
  int K, N, N_pad, tmem_cols, h_bytes, z_bytes, m_bytes, dbg;
  int R, NC;  // raw tile slots, A/B chunk ring depth
  int nacc;   // TMEM accumulators (tiles round-robin over them)
  int h_tma;  // H tiles by TMA tensor copies of a column slice (rows of h_lds floats in smem)
  int h_lds;  // smem row stride of an H tile, floats (= ldh for whole-row bulk copies)
  int z_tma;  // dZ (and mask) tiles by TMA tensor copies of a column slice (N slices)
  int z_lds, m_lds;  // smem row strides of the dZ / mask tiles, floats
  int db_conv;  // K == 128 (no TMEM lane left for the ones row): db from the B' converters' column sums
  int nks;      // K slices in this launch (CTA b: slice b % nks, row range b / nks), 1 = a single slice
  int kslice;   // slice width (nks > 1): slice s covers features [s kslice, min(K, (s+1) kslice))
  int64_t part_stride;  // floats between the slices' partial regions
};

template <bool DBC>  // DBC: db from the converters (p.db_conv, K == 128); a separate
                    // instantiation keeps the common path's registers / code unchanged
__global__ void __launch_bounds__(G3_THREADS, 1) tc_wgrad3_kernel(const __grid_constant__ CUtensorMap tmH,
                                                                  const __grid_constant__ CUtensorMap tmZ,
                                                                  const __grid_constant__ CUtensorMap tmM, Wg3Args p) {
  extern __shared__ __align__(1024) char smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int N_pad = p.N_pad;
  const int b_box = N_pad * 128;  // one SW128 box: N_pad rows x 32 K (rows r) fp32
  char* sB = smem;                                  // [NC][hi, lo] boxes
  char* slots = sB + p.NC * 2 * b_box;
  const int slot_bytes = p.h_bytes + p.z_bytes + p.m_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(slots + p.R * slot_bytes);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * p.R + 2 * p.NC + 1);
  float* dbsm = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(tmem_slot + 4) + 15) &
                                          ~uintptr_t(15));  // db_conv: [3 groups][8 row quads][N_pad]
  auto bar = [&](int i) { return smem_u32(bars + i); };
  const int FULL = 0, EMPTY = p.R, CFULL = 2 * p.R, CEMPTY = 2 * p.R + p.NC, TFULL = 2 * p.R + 2 * p.NC;
  if (tid == 0) {
    for (int s = 0; s < p.R; ++s) { mbar_init_n(bar(FULL + s), 1); mbar_init_n(bar(EMPTY + s), G3_CONV_THREADS); }
    for (int c = 0; c < p.NC; ++c) { mbar_init_n(bar(CFULL + c), G3_CONV_THREADS / 2); mbar_init_n(bar(CEMPTY + c), 1); }
    mbar_init_n(bar(TFULL), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) G3T(0);
  const int64_t tiles = ceil_div(p.M, WG3_MT);
  // multi-slice launch: CTAs rc * nks .. rc * nks + nks - 1 take the same row
  // tiles for consecutive K slices, so a dZ / mask tile read from HBM by one
  // is an L2 hit for the others
  const int ksl = (int)(blockIdx.x % p.nks), rc = (int)(blockIdx.x / p.nks), G = (int)(gridDim.x / p.nks);
  const int K = p.nks > 1 ? min(p.kslice, p.K - ksl * p.kslice) : p.K;  // this CTA's features
  if (warp == 0) {
    if (lane == 0) {
      int j = 0;
      for (int64_t t = rc; t < tiles; t += G, ++j) {
        const int s = j % p.R;
        mbar_wait(bar(EMPTY + s), ((uint32_t)(j / p.R) & 1u) ^ 1u);
        if (j < 8) G3T(58 + j);
        const int64_t r0 = t * WG3_MT;
        const int rows = (int)(p.M - r0 < WG3_MT ? p.M - r0 : WG3_MT);
        const uint32_t hb = p.h_tma ? (uint32_t)(WG3_MT * p.h_lds * 4) : (uint32_t)(rows * p.ldh * 4);
        const uint32_t zb = p.z_tma ? (uint32_t)(WG3_MT * p.z_lds * 4) : (uint32_t)(rows * p.ldz * 4);
        const uint32_t mb = !p.mask ? 0u : p.z_tma ? (uint32_t)(WG3_MT * p.m_lds * 4) : (uint32_t)(rows * p.ldm * 4);
        char* slot = slots + s * slot_bytes;
        mbar_arrive_expect_tx(bar(FULL + s), hb + zb + mb);
        if (p.h_tma) tma_load_2d(smem_u32(slot), &tmH, ksl * p.kslice, (int)r0, bar(FULL + s));  // OOB: zeros
        else bulk_load(smem_u32(slot), p.H + r0 * p.ldh, hb, bar(FULL + s));
        if (p.z_tma) {
          tma_load_2d(smem_u32(slot + p.h_bytes), &tmZ, 0, (int)r0, bar(FULL + s));
          if (p.mask) tma_load_2d(smem_u32(slot + p.h_bytes + p.z_bytes), &tmM, 0, (int)r0, bar(FULL + s));
        } else {
          bulk_load(smem_u32(slot + p.h_bytes), p.dZ + r0 * p.ldz, zb, bar(FULL + s));
          if (p.mask) bulk_load(smem_u32(slot + p.h_bytes + p.z_bytes), p.mask + r0 * p.ldm, mb, bar(FULL + s));
        }
      }
    }
    return;
  }
  if (warp == 1) tmem_alloc(tmem_slot, p.tmem_cols);
  tc_fence_before();
  asm volatile("bar.sync 1, %0;" ::"r"(G3_THREADS - 32) : "memory");
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TMEM: NACC accumulators [0, NACC N_pad) (tile j accumulates into j % NACC:
  // the tensor core's fp32 accumulation loses accuracy over long chains, the
  // epilogue sums the accumulators with IEEE adds), then the A chunk ring
  auto ch_hi = [&](int c) { return tmem + (uint32_t)(p.nacc * N_pad + 64 * c); };
  const int my_tiles = (int)(tiles > rc ? (tiles - 1 - rc) / G + 1 : 0);

  if (warp == 1) {
    const uint32_t idesc = idesc_tf32(G3_M, N_pad, 0, 0);
    const uint32_t sb = smem_u32(sB);
    int cc = 0;
    for (int j = 0; j < ((p.dbg & 16) ? 0 : my_tiles); ++j) {
      const uint32_t acc_t = tmem + (uint32_t)((j % p.nacc) * N_pad);
      for (int c = 0; c < WG3_MT / 32; ++c, ++cc) {
        const int cs = cc % p.NC;
        mbar_wait(bar(CFULL + cs), (uint32_t)(cc / p.NC) & 1u);
        if (cc < 8 && lane == 0) G3T(50 + cc);
        tc_fence_after();
        const uint32_t ahi = ch_hi(cs), alo = ahi + 32;
        const uint32_t bh = sb + (uint32_t)(cs * 2 * b_box), bl = bh + (uint32_t)b_box;
        if (elect_one()) {
#pragma unroll
          for (int st = 0; st < ((p.dbg & 2) ? 0 : 4); ++st) {
            const uint64_t dbh = umma_desc_sw128(bh + st * 32), dbl = umma_desc_sw128(bl + st * 32);
            const uint32_t first = (j < p.nacc && c == 0 && st == 0) ? 0u : 1u;  // overwrite on a fresh accumulator
            mma_tf32_ts(acc_t, alo + 8 * st, dbh, idesc, first);
            mma_tf32_ts(acc_t, ahi + 8 * st, dbl, idesc, 1);
            mma_tf32_ts(acc_t, ahi + 8 * st, dbh, idesc, 1);
          }
          mma_commit(bar(CEMPTY + cs));
        }
        __syncwarp();
      }
    }
    if (my_tiles > 0 && elect_one()) mma_commit(bar(TFULL));
    __syncwarp();
  } else if (warp >= 4) {
    // three groups of 4 warps (4-7, 8-11, 12-15) take every third 32-row
    // chunk, so one group's TMEM-store / fence latency overlaps the others'
    // shared-memory work; warps 12-15 then also run the epilogue
    const int grp = (warp - 4) >> 2;
    const int ct = tid - 128 - 128 * grp;  // 0..127 within the group
    const int quarter = warp & 3;
    const int m = quarter * 32 + lane;     // A' row = TMEM lane
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    // db_conv: this thread's B' items (fixed across chunks) summed over the
    // rows of its group's chunks, in chunk order (deterministic)
    float4 dbs[DBC ? 4 : 1];
#pragma unroll
    for (int u = 0; u < (DBC ? 4 : 1); ++u) dbs[u] = make_float4(0.f, 0.f, 0.f, 0.f);
    int kk = 0;
    for (int cc = grp; cc < 2 * my_tiles; cc += 3, ++kk) {
      const int j = cc >> 1, c = cc & 1;
      const int s = j % p.R;
      const int64_t t = rc + (int64_t)j * G;
      const int rows = (int)(p.M - t * WG3_MT < WG3_MT ? p.M - t * WG3_MT : WG3_MT);
      mbar_wait(bar(FULL + s), (uint32_t)(j / p.R) & 1u);
      const bool trc = ct == 0 && grp == 0 && kk < 8;
      if (trc) G3T(2 + 6 * kk);
      const uint32_t hs = smem_u32(slots + s * slot_bytes);
      const uint32_t zs = hs + (uint32_t)p.h_bytes, ms = zs + (uint32_t)p.z_bytes;
      {
        const int cs = cc % p.NC;
        // A': column m of rows r = 32c + [0, 32) (conflict-free: consecutive
        // lanes read consecutive features of one row)
        // branch-free: all 32 loads issue back to back (rows past the tile
        // end read stale in-bounds slot data and are zeroed after)
        uint32_t hv[32], lv[32];
        {
          const int nrow = rows - 32 * c;
          const uint32_t a0 = hs + (uint32_t)((32 * c * p.h_lds + (m < K ? m : 0)) * 4);
          const uint32_t rs = (uint32_t)(p.h_lds * 4);
          float xs[32];
#pragma unroll
          for (int q = 0; q < 32; ++q) xs[q] = lds32(a0 + (uint32_t)q * rs);
          const float one = m == K ? 1.f : 0.f;
#pragma unroll
          for (int q = 0; q < 32; ++q) {
            const float x = q < nrow ? (m < K ? xs[q] : one) : 0.f;
            const float hi = tf32_rna_finite(x);
            hv[q] = __float_as_uint(hi);
            lv[q] = __float_as_uint(__fsub_rn(x, hi));
          }
        }
        if (trc) G3T(3 + 6 * kk);
        mbar_wait(bar(CEMPTY + cs), ((uint32_t)(cc / p.NC) & 1u) ^ 1u);
        if (trc) G3T(4 + 6 * kk);
        tc_fence_after();
        const uint32_t hi_t = ch_hi(cs) + lane_off;
        tmem_st32(hi_t, hv);
        tmem_st32(hi_t + 32, lv);
        // B': 4x4 blocks (rows 4rq..4rq+3 of the chunk x features 4n4..4n4+3):
        // four 16-byte row loads, a register transpose, four 16-byte stores
        // into the SW128 box (row n, K = r).  Item -> (n4, rq) is chosen so
        // that each 8-lane phase hits 8 distinct bank groups on both sides:
        // loads by n4 mod 8, stores by rq ^ (n & 7).
        const uint32_t bh = smem_u32(sB) + (uint32_t)(cs * 2 * b_box);
        const int n4s = N_pad >> 2;
        const int items = ((n4s + 7) >> 3) * 64;
        auto b_item = [&](int t, float4& db_acc) {
          const int ph = t & 7, hi_ = t >> 3;
          const int n4 = ph + 8 * (hi_ >> 3);
          const int rq = (((ph >> 1) + (hi_ & 3)) & 3) + 4 * ((hi_ >> 2) & 1);
          if (n4 >= n4s) return;
          const int rb = 32 * c + 4 * rq;
          float4 e[4];
          if (rb + 4 <= rows && 4 * n4 + 4 <= p.N && p.mask) {
            // interior block (the common case): no row / feature predicates
            float4 mk[4];
            const uint32_t za = zs + (uint32_t)((rb * p.z_lds + 4 * n4) * 4), zr = (uint32_t)(p.z_lds * 4);
            const uint32_t ma = ms + (uint32_t)((rb * p.m_lds + 4 * n4) * 4), mr = (uint32_t)(p.m_lds * 4);
#pragma unroll
            for (int i = 0; i < 4; ++i) e[i] = lds128(za + (uint32_t)i * zr);
#pragma unroll
            for (int i = 0; i < 4; ++i) mk[i] = lds128(ma + (uint32_t)i * mr);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              e[i].x = mk[i].x > 0.f ? e[i].x : 0.f;
              e[i].y = mk[i].y > 0.f ? e[i].y : 0.f;
              e[i].z = mk[i].z > 0.f ? e[i].z : 0.f;
              e[i].w = mk[i].w > 0.f ? e[i].w : 0.f;
            }
          } else {
            const int nn = 4 * n4 < p.N ? 4 * n4 : 0;
            float4 mk[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) e[i] = lds128(zs + (uint32_t)(((rb + i) * p.z_lds + nn) * 4));
            if (p.mask) {
#pragma unroll
              for (int i = 0; i < 4; ++i) mk[i] = lds128(ms + (uint32_t)(((rb + i) * p.m_lds + nn) * 4));
            } else {
#pragma unroll
              for (int i = 0; i < 4; ++i) mk[i] = make_float4(1.f, 1.f, 1.f, 1.f);
            }
            // keep feature f < N of row r < rows with a positive mask
            const int nv = 4 * n4 < p.N ? min(p.N - 4 * n4, 4) : 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const bool rv = rb + i < rows;
              e[i].x = (rv && nv > 0 && mk[i].x > 0.f) ? e[i].x : 0.f;
              e[i].y = (rv && nv > 1 && mk[i].y > 0.f) ? e[i].y : 0.f;
              e[i].z = (rv && nv > 2 && mk[i].z > 0.f) ? e[i].z : 0.f;
              e[i].w = (rv && nv > 3 && mk[i].w > 0.f) ? e[i].w : 0.f;
            }
          }
          if (DBC) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              db_acc.x = __fadd_rn(db_acc.x, e[i].x);
              db_acc.y = __fadd_rn(db_acc.y, e[i].y);
              db_acc.z = __fadd_rn(db_acc.z, e[i].z);
              db_acc.w = __fadd_rn(db_acc.w, e[i].w);
            }
          }
          const float4 col[4] = {make_float4(e[0].x, e[1].x, e[2].x, e[3].x), make_float4(e[0].y, e[1].y, e[2].y, e[3].y),
                                 make_float4(e[0].z, e[1].z, e[2].z, e[3].z), make_float4(e[0].w, e[1].w, e[2].w, e[3].w)};
#pragma unroll
          for (int jn = 0; jn < 4; ++jn) {
            float4 h4, l4;
            h4.x = tf32_rna_finite(col[jn].x); l4.x = __fsub_rn(col[jn].x, h4.x);
            h4.y = tf32_rna_finite(col[jn].y); l4.y = __fsub_rn(col[jn].y, h4.y);
            h4.z = tf32_rna_finite(col[jn].z); l4.z = __fsub_rn(col[jn].z, h4.z);
            h4.w = tf32_rna_finite(col[jn].w); l4.w = __fsub_rn(col[jn].w, h4.w);
            const uint32_t off = sw128_off(4 * n4 + jn, 4 * rq);
            sts128(bh + off, h4);
            sts128(bh + (uint32_t)b_box + off, l4);
          }
        };
        const int lim = (p.dbg & 4) ? 0 : items;
        if constexpr (DBC) {  // static item slots: the db accumulators stay in registers
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (ct + u * (G3_CONV_THREADS / 2) < lim) b_item(ct + u * (G3_CONV_THREADS / 2), dbs[u]);
        } else {
          for (int t = ct; t < lim; t += G3_CONV_THREADS / 2) b_item(t, dbs[0]);
        }
        if (trc) G3T(5 + 6 * kk);
        tmem_st_wait();
        fence_async_smem();
        tc_fence_before();
        mbar_arrive(bar(CFULL + cs));
        if (trc) G3T(6 + 6 * kk);
      }
      mbar_arrive(bar(EMPTY + s));
      if (trc) G3T(7 + 6 * kk);
    }
    if (DBC) {
      const int n4s = N_pad >> 2, items = ((n4s + 7) >> 3) * 64;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int t = ct + u * (G3_CONV_THREADS / 2);
        if (t >= items) break;
        const int ph = t & 7, hi_ = t >> 3;
        const int n4 = ph + 8 * (hi_ >> 3);
        const int rq = (((ph >> 1) + (hi_ & 3)) & 3) + 4 * ((hi_ >> 2) & 1);
        if (n4 < n4s) *reinterpret_cast<float4*>(dbsm + (grp * 8 + rq) * N_pad + 4 * n4) = dbs[DBC ? u : 0];
      }
      asm volatile("bar.sync 5, %0;" ::"r"(G3_THREADS - 128) : "memory");  // the 12 converter warps
    }
  }
  if (warp >= 12) {
    const int quarter = warp & 3;
    const int m = quarter * 32 + lane;
    float* out = p.part + ksl * p.part_stride + (int64_t)rc * (K + 1) * p.N;
    if (my_tiles > 0) {
      mbar_wait(bar(TFULL), 0);
      tc_fence_after();
    }
    if (tid == 384) G3T(70);
    const int used = my_tiles < p.nacc ? my_tiles : p.nacc;
    for (int c0 = 0; c0 < N_pad; c0 += 16) {
      float sum[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) sum[q] = 0.f;
      for (int a = 0; a < used; ++a) {  // fixed order: deterministic
        uint32_t v[16];
        tmem_ld16(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(a * N_pad + c0), v);
#pragma unroll
        for (int q = 0; q < 16; ++q) sum[q] = a == 0 ? __uint_as_float(v[q]) : __fadd_rn(sum[q], __uint_as_float(v[q]));
      }
      if (m <= K) {  // feature-major partials: a warp stores 32 consecutive floats per column
#pragma unroll
        for (int q = 0; q < 16; ++q)
          if (c0 + q < p.N) out[(int64_t)(c0 + q) * (K + 1) + m] = sum[q];
      }
    }
    if (DBC) {  // row K (db): the converters' sums, groups then row quads in a fixed order
      for (int c = tid - 384; c < p.N; c += 128) {
        float v = 0.f;
        for (int g = 0; g < 24; ++g) v = __fadd_rn(v, dbsm[g * N_pad + c]);
        out[(int64_t)c * (K + 1) + K] = v;
      }
    }
    if (tid == 384) G3T(71);
  }
  tc_fence_before();
  asm volatile("bar.sync 1, %0;" ::"r"(G3_THREADS - 32) : "memory");
  if (warp == 1) {
    tc_fence_after();
    tmem_free(tmem, p.tmem_cols);
  }
}

// ------------------------------------------------------------ tc_dense4 --
// Forward / dgrad GEMM for the usual layer shapes (K <= 128, N <= 128, one
// tile), organised around the TMA engine and shared-memory operands:
//
//   warp 0      producer: one 2-D TMA tensor copy per [128 rows x 32 K]
//               SWIZZLE_128B box of A (and of the ReLU mask for dgrad) into a
//               ring of S box stages -- the box layout IS the K-major
//               SWIZZLE_128B operand layout the tensor core reads, so A is
//               never re-laid-out;
//   warps 4-7   splitters, thread = row: read the row's 32 floats of a box
//               (conflict-free: the swizzle spreads 8 rows over the banks),
//               mask, write hi = tf32(x) back in place and lo = x - hi to the
//               box's TMEM slot (tcgen05.st, lane = row);
//   warp 1      MMA issuer: per 8-wide K step lo*W_hi (A from TMEM), hi*W_lo,
//               hi*W_hi (A from shared memory) into a double-buffered fp32
//               accumulator; one commit per box frees its stage;
//   warps 8-11  epilogue: tcgen05.ld, bias, ReLU, SW128 staging boxes, TMA
//               tensor stores;
//   warps 2-3   (K > 128 only, "streamed weight") the weight image would not
//               fit beside the stages (Reddit's 602 inputs: 304 KB), so each
//               stage also carries the raw [32 K x N] weight box, TMA-loaded
//               from L2 with the A box, which warps 2-3 split into the stage's
//               own hi / lo boxes while the splitters split A.  One pass over
//               A instead of K slices that re-read and re-accumulate the
//               output (Reddit layer 0: 208 -> 175 us).  The accumulation
//               chain in TMEM is then K long instead of 128 (results within
//               1e-5, not bit-identical to the sliced path).
//
// Against tc_gemm3 (whole-row bulk copies converted into a TMEM A ring by
// thread-per-row converters): a stage is 16 KB instead of a 51 KB tile, so
// 8 stages (128 KB of loads in flight per SM) fit beside the weight images,
// and the tensor core reads the hi part straight from the landed box.  Same
// rounding and the same MMA order as tc_gemm3 (bit-identical results).
constexpr int T4_THREADS = 384;  // 12 warps, roles above (warps 2-3 split the weight)
constexpr int T4_M = 128;
constexpr int T4_BOX = T4_M * 128;  // one [128 rows x 32 fp32] SW128 box
constexpr int T4_MAX_STAGES = 12;

struct T4Args {
  const float* W;      // mode 0: [K, N] row-major; mode 1: [N, K] row-major (row stride ldw)
  const float* bias;   // mode 0 only, [N] or null
  int64_t M, ldw;
  int N, K, N_pad, K_pad, S, relu, has_mask, tmem_cols, w_vec, stage_off, dbg;
  int stream_w;  // K > 128: each stage carries its K box of the weight, no image
  int w_raw;     // stream_w: bytes of the TMA-staged raw weight box (1024-aligned slot)
  int w_ld;      // stream_w: row length of the raw box in floats
};

template <int MODE>
__global__ void __launch_bounds__(T4_THREADS, 1) tc_dense4_kernel(const __grid_constant__ CUtensorMap tmA,
                                                                  const __grid_constant__ CUtensorMap tmM,
                                                                  const __grid_constant__ CUtensorMap tmC,
                                                                  const __grid_constant__ CUtensorMap tmW, T4Args p) {
  extern __shared__ __align__(1024) char smem_raw[];
  char* smem = reinterpret_cast<char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int S = p.S, N_pad = p.N_pad;
  const int KB = (p.K + 31) / 32;  // A boxes per tile (= weight image boxes)
  const int b_box = N_pad * 128;
  const int img_boxes = p.stream_w ? 0 : KB;
  char* sB_hi = smem;
  char* sB_lo = sB_hi + img_boxes * b_box;
  char* stages = sB_lo + img_boxes * b_box;  // S x {A box, mask box[, W hi box, W lo box, raw W box]}
  const int stage_bytes = T4_BOX * (1 + p.has_mask) + (p.stream_w ? 2 * b_box + ((p.w_raw + 1023) & ~1023) : 0);
  auto stage_w = [&](int s) { return stages + s * stage_bytes + T4_BOX * (1 + p.has_mask); };
  const uint32_t tx_bytes = (uint32_t)(T4_BOX * (1 + p.has_mask)) + (p.stream_w ? (uint32_t)p.w_raw : 0u);
  char* stg = smem + p.stage_off;     // epilogue staging: ceil(N_pad / 32) boxes
  uint64_t* bars = reinterpret_cast<uint64_t*>(stg + ((N_pad + 31) / 32) * T4_BOX);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 3 * S + 5);
  float* sbias = reinterpret_cast<float*>(tmem_slot + 4);
  auto bar = [&](int i) { return smem_u32(bars + i); };
  const int FULL = 0, SPLIT = S, EMPTY = 2 * S, TFULL = 3 * S, TEMPTY = 3 * S + 2, BREADY = 3 * S + 4;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init_n(bar(FULL + s), 1);
      mbar_init_n(bar(SPLIT + s), 128 + (p.stream_w ? 64 : 0));  // + the weight-box producers
      mbar_init_n(bar(EMPTY + s), 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init_n(bar(TFULL + a), 1);
      mbar_init_n(bar(TEMPTY + a), 128);
    }
    mbar_init_n(bar(BREADY), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t tiles = ceil_div(p.M, T4_M);
  if (warp == 0) {
    // ---------------------------------------------------------- producer --
    if (lane == 0) {
      tma_prefetch_desc(&tmA);
      if (p.has_mask) tma_prefetch_desc(&tmM);
      if (p.w_raw) tma_prefetch_desc(&tmW);
      int g = 0;
      for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        for (int b = 0; b < KB; ++b, ++g) {
          const int s = g % S;
          mbar_wait(bar(EMPTY + s), ((uint32_t)(g / S) & 1u) ^ 1u);
          const uint32_t dst = smem_u32(stages + s * stage_bytes);
          mbar_arrive_expect_tx(bar(FULL + s), tx_bytes);
          tma_load_2d(dst, &tmA, 32 * b, (int)(t * T4_M), bar(FULL + s));  // OOB rows / columns: zeros
          if (p.has_mask) tma_load_2d(dst + T4_BOX, &tmM, 32 * b, (int)(t * T4_M), bar(FULL + s));
          if (p.w_raw)  // raw weight box b (L2-resident): rows 32b.. (mode 0) / columns 32b.. (mode 1)
            tma_load_2d(smem_u32(stage_w(s) + 2 * b_box), &tmW, MODE == 0 ? 0 : 32 * b, MODE == 0 ? 32 * b : 0,
                        bar(FULL + s));
        }
      }
    }
    return;
  }
  if (warp == 1) tmem_alloc(tmem_slot, p.tmem_cols);
  // the weight image, by every non-producer warp but the MMA issuer (the
  // first boxes are still in flight), then bias -> shared
  if (warp >= 2) {
    if (!p.stream_w)
      split_weight_image<MODE>(p.W, p.ldw, p.K, p.N, p.K_pad, N_pad, p.w_vec, sB_hi, sB_lo, tid - 64, T4_THREADS - 64);
    for (int c = tid - 64; c < N_pad; c += T4_THREADS - 64)
      sbias[c] = (MODE == 0 && p.bias && c < p.N) ? p.bias[c] : 0.f;
    fence_async_smem();
    asm volatile("bar.sync 3, %0;" ::"r"(T4_THREADS - 64) : "memory");
    if (tid == 64) mbar_arrive(bar(BREADY));
  }
  tc_fence_before();
  asm volatile("bar.sync 1, %0;" ::"r"(T4_THREADS - 32) : "memory");
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TMEM columns: accumulators [0, 2 N_pad), box s's lo part at 2 N_pad + 32 s
  auto lo_col = [&](int s) { return tmem + (uint32_t)(2 * N_pad + 32 * s); };

  if (warp == 1) {
    // -------------------------------------------------------- MMA issuer --
    const uint32_t idesc = idesc_tf32(T4_M, N_pad, 0, 0);
    const uint32_t bh = smem_u32(sB_hi), bl = smem_u32(sB_lo);
    mbar_wait(bar(BREADY), 0);
    tc_fence_after();
    int j = 0, g = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++j) {
      const int a = j & 1;
      const uint32_t acc = tmem + (uint32_t)(a * N_pad);
      mbar_wait(bar(TEMPTY + a), ((uint32_t)(j >> 1) & 1u) ^ 1u);
      tc_fence_after();
      for (int b = 0; b < KB; ++b, ++g) {
        const int s = g % S;
        mbar_wait(bar(SPLIT + s), (uint32_t)(g / S) & 1u);
        tc_fence_after();
        const int kst = min(32, p.K_pad - 32 * b) / 8;
        const uint32_t ahi = smem_u32(stages + s * stage_bytes), alo = lo_col(s);
        // weight box of this K slice: the stage's own copy, or box b of the image
        const uint32_t wbh = p.stream_w ? smem_u32(stage_w(s)) : bh + (uint32_t)(b * b_box);
        const uint32_t wbl = p.stream_w ? wbh + (uint32_t)b_box : bl + (uint32_t)(b * b_box);
        if (elect_one()) {
          for (int st = 0; st < ((p.dbg & 2) ? 0 : kst); ++st) {
            const uint32_t bo = (uint32_t)(st * 32);
            const uint64_t dbh = umma_desc_sw128(wbh + bo), dbl = umma_desc_sw128(wbl + bo);
            const uint64_t dah = umma_desc_sw128(ahi + (uint32_t)(st * 32));
            mma_tf32_ts(acc, alo + 8 * st, dbh, idesc, (b | st) != 0);
            mma_tf32(acc, dah, dbl, idesc, 1);
            mma_tf32(acc, dah, dbh, idesc, 1);
          }
          mma_commit(bar(EMPTY + s));  // stage (and its TMEM lo slot) free once these MMAs complete
        }
        __syncwarp();
      }
      if (elect_one()) mma_commit(bar(TFULL + a));
      __syncwarp();
    }
  } else if (warp >= 2 && warp < 4 && p.stream_w) {
    // ------------------------------------------------ weight-box producers --
    // (K > 128) warps 2-3 split each stage's TMA-staged raw 32-wide K box of
    // the weight into the stage's hi / lo boxes, beside the splitters
    int g = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
      for (int b = 0; b < KB; ++b, ++g) {
        const int s = g % S;
        mbar_wait(bar(FULL + s), (uint32_t)(g / S) & 1u);
        const int kl = min(32, p.K - 32 * b), kpl = min(32, p.K_pad - 32 * b);
        char* swh = stage_w(s);
        if (p.w_raw)
          split_weight_image<MODE, true>(reinterpret_cast<const float*>(swh + 2 * b_box), p.w_ld, kl, p.N, kpl,
                                         N_pad, true, swh, swh + b_box, tid - 64, 64);
        else  // weight rows not 16-byte aligned (no TMA): straight from L2
          split_weight_image<MODE>(MODE == 0 ? p.W + (int64_t)(32 * b) * p.ldw : p.W + 32 * b, p.ldw, kl, p.N, kpl,
                                   N_pad, p.w_vec, swh, swh + b_box, tid - 64, 64);
        fence_async_smem();
        mbar_arrive(bar(SPLIT + s));
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // --------------------------------------------------------- splitters --
    const int r = (warp & 3) * 32 + lane;  // row = TMEM lane
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    int g = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
      for (int b = 0; b < KB; ++b, ++g) {
        const int s = g % S;
        mbar_wait(bar(FULL + s), (uint32_t)(g / S) & 1u);
        const uint32_t xr = smem_u32(stages + s * stage_bytes) + (uint32_t)(r * 128);
        uint32_t lv[32];
#pragma unroll
        for (int h = 0; h < ((p.dbg & 1) ? 0 : 2); ++h) {
          float4 x[4], m[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int c = 4 * h + q;  // 16-byte chunk c (k = 4c..4c+3) sits at chunk c ^ (r & 7)
            x[q] = lds128(xr + (uint32_t)((c ^ (r & 7)) << 4));
            if (MODE == 1 && p.has_mask) m[q] = lds128(xr + T4_BOX + (uint32_t)((c ^ (r & 7)) << 4));
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int c = 4 * h + q;
            float xs[4] = {x[q].x, x[q].y, x[q].z, x[q].w};
            if (MODE == 1 && p.has_mask) {
              const float ms[4] = {m[q].x, m[q].y, m[q].z, m[q].w};
#pragma unroll
              for (int u = 0; u < 4; ++u)
                if (!(ms[u] > 0.f)) xs[u] = 0.f;
            }
            float hs[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              hs[u] = tf32_rna_finite(xs[u]);
              lv[4 * c + u] = __float_as_uint(__fsub_rn(xs[u], hs[u]));
            }
            sts128(xr + (uint32_t)((c ^ (r & 7)) << 4), make_float4(hs[0], hs[1], hs[2], hs[3]));
          }
        }
        if (!(p.dbg & 1)) {
          tmem_st32(lo_col(s) + lane_off, lv);
        }
        if (!(p.dbg & 1)) tmem_st_wait();
        fence_async_smem();  // hi / weight stores -> visible to the tensor core (async proxy)
        tc_fence_before();
        mbar_arrive(bar(SPLIT + s));
      }
    }
  } else if (warp >= 8) {
    // ---------------------------------------------------------- epilogue --
    const int quarter = warp & 3, et = tid - 256, r_loc = quarter * 32 + lane;
    const uint32_t stg_u = smem_u32(stg);
    int j = 0;
    for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x, ++j) {
      const int a = j & 1;
      mbar_wait(bar(TFULL + a), (uint32_t)(j >> 1) & 1u);
      tc_fence_after();
      if (j > 0) {  // the previous tile's TMA stores must have finished reading staging
        if (et == 0) bulk_wait_read0();
        asm volatile("bar.sync 2, 128;" ::: "memory");
      }
      for (int c0 = 0; c0 < N_pad; c0 += 32) {
        uint32_t v[32];
        const uint32_t ta = tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(a * N_pad + c0);
        tmem_ld16_nowait(ta, v);
        if (c0 + 16 < N_pad) tmem_ld16_nowait(ta + 16, v + 16);
        tmem_ld_wait();
        const int ncol = c0 + 16 < N_pad ? 32 : 16;
        const uint32_t box = stg_u + (uint32_t)((c0 >> 5) * T4_BOX) + (uint32_t)(r_loc * 128);
#pragma unroll
        for (int h = 0; h < 32; h += 4) {
          if (h >= ncol) break;
          float x[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            float y = __uint_as_float(v[h + q]);
            if (MODE == 0 && p.bias) y = __fadd_rn(y, sbias[c0 + h + q]);
            if (p.relu) y = y > 0.f ? y : 0.f;
            x[q] = y;
          }
          sts128(box + (uint32_t)((((h >> 2) ^ (r_loc & 7)) & 7) << 4), make_float4(x[0], x[1], x[2], x[3]));
        }
      }
      tc_fence_before();
      mbar_arrive(bar(TEMPTY + a));  // accumulator drained: tile j+2's MMAs may start
      fence_async_smem();
      asm volatile("bar.sync 2, 128;" ::: "memory");
      if (et == 0) {
        for (int c0 = 0; c0 < N_pad; c0 += 32)
          tma_store_2d(&tmC, stg_u + (uint32_t)((c0 >> 5) * T4_BOX), c0, (int)(t * T4_M));
        bulk_commit();
      }
    }
    if (et == 0) bulk_wait0();
  }
  // warps 1-11 (warp 0 returned after issuing its copies)
  tc_fence_before();
  asm volatile("bar.sync 1, %0;" ::"r"(T4_THREADS - 32) : "memory");
  if (warp == 1) {
    tc_fence_after();
    tmem_free(tmem, p.tmem_cols);
  }
}


// ------------------------------------------------------------ host side --
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

// fp32 [rows, cols] row-major (ld floats) in 128-row x 32-column SWIZZLE_128B boxes
bool make_map_sw128(CUtensorMap* m, const float* base, int64_t rows, int cols, int64_t ld) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {32, (cuuint32_t)G3_M};
  cuuint32_t es[2] = {1, 1};
  static const int promo = getenv("FGL_A_L2PROMO") ? atoi(getenv("FGL_A_L2PROMO")) : 0;
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, (CUtensorMapL2promotion)promo,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// fp32 [rows, cols] row-major (ld floats) in boxes of [box_rows x box_cols]
// (box_cols = cols rounded up to 4; columns past `cols` and rows past `rows`
// read as zeros): a column slice of a wider matrix, rows packed in smem
bool make_map_cols(CUtensorMap* m, const float* base, int64_t rows, int cols, int64_t ld, int box_cols, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int64_t g3_fixed(int N_pad, int K_pad, int R, int64_t a_slot, int64_t m_slot) {
  return 1024 + 2 * (int64_t)N_pad * ((K_pad + 31) / 32) * 128 + R * (a_slot + m_slot) + 8 * (2 * R + 22) + 16 + 4 * N_pad;
}
int64_t g3_stage_bytes(int N_pad) { return (int64_t)G3_M * ((N_pad + 31) / 32) * 128; }  // SW128 boxes
int64_t g3_smem(int N_pad, int K_pad, int R, int64_t a_slot, int64_t m_slot) {
  return g3_fixed(N_pad, K_pad, R, a_slot, m_slot) + 1024 + g3_stage_bytes(N_pad);
}

std::atomic<int> g_dense_ctas{kNumSMs};
int dense_cta_budget() { return g_dense_ctas.load(std::memory_order_relaxed); }

bool tc3_disabled() {
  static const int v = [] {
    const char* e = getenv("FGL_DENSE");
    return (e && (e[0] == 's' || e[0] == 'v')) ? 1 : 0;  // simt / v2 force the older kernels
  }();
  return v != 0;
}

// tensor maps are host microseconds to encode and the trainer reuses the same
// buffers every batch: keep the last few per thread
bool cached_map_sw128(CUtensorMap* out, const float* base, int64_t rows, int cols, int64_t ld) {
  struct Entry { const float* base; int64_t rows, ld; int cols; CUtensorMap m; };
  static thread_local Entry cache[16];
  static thread_local int next = 0;
  for (auto& c : cache)
    if (c.base == base && c.rows == rows && c.cols == cols && c.ld == ld) { *out = c.m; return true; }
  if (!make_map_sw128(out, base, rows, cols, ld)) return false;
  Entry& c = cache[next];
  next = (next + 1) % 16;
  c.base = base; c.rows = rows; c.cols = cols; c.ld = ld; c.m = *out;
  return true;
}

bool tc4_disabled() {
  static const int v = getenv("FGL_TC4") ? atoi(getenv("FGL_TC4")) == 0 : 0;
  return v != 0;
}


// tc_dense4_kernel for one [M x N] output with N <= 128, K <= FGL_TC4_KMAX
// (default 1024; K > 128 streams the weight per stage) and no K-slice
// accumulation; false outside that envelope (tc_gemm3 then runs the tile)
bool tc_dense4(int mode, const float* A, int64_t lda, const float* mask, int64_t ldm, const float* W,
               const float* bias, float* C, int64_t ldc, int64_t M, int N, int K, int relu, int64_t ldw,
               cudaStream_t st, int* err) {
  *err = 0;
  static const int kmax_stream = getenv("FGL_TC4_KMAX") ? atoi(getenv("FGL_TC4_KMAX")) : 1024;
  if (tc4_disabled() || M < 1 || K < 1 || K > std::max(128, kmax_stream) || N < 1 || N > 128) return false;
  // K > 128: the weight image would not fit beside the stages -- each stage
  // carries its own 32-wide K box of the weight instead (split per tile from L2)
  const int stream_w = K > 128 ? 1 : 0;
  const int has_mask = (mode == 1 && mask) ? 1 : 0;
  if ((lda % 4) || (ldc % 4) || (reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(C) & 15))
    return false;
  if (has_mask && ((ldm % 4) || (reinterpret_cast<uintptr_t>(mask) & 15))) return false;
  const int N_pad = (N + 15) / 16 * 16, K_pad = (K + 7) / 8 * 8, KB = (K + 31) / 32;
  // raw weight box of a K slice: mode 0 rows [32 x ceil4(N)], mode 1 [N x 32]
  const int w_ld = mode == 0 ? (N + 3) / 4 * 4 : 32;
  const bool w_tma = stream_w && !(ldw % 4) && !(reinterpret_cast<uintptr_t>(W) & 15);
  const int w_raw = w_tma ? ((mode == 0 ? 32 * w_ld : N * 32) * 4 + 1023) / 1024 * 1024 : 0;
  const int64_t stage_bytes = (int64_t)T4_BOX * (1 + has_mask) + (stream_w ? 2 * (int64_t)N_pad * 128 + w_raw : 0);
  const int img_boxes = stream_w ? 0 : KB;
  const int nob = (N_pad + 31) / 32;
  auto fixed = [&](int S) {
    return 1024 + 2 * (int64_t)img_boxes * N_pad * 128 + (int64_t)S * stage_bytes + (int64_t)nob * T4_BOX +
           8 * (3 * S + 5) + 16 + 4 * N_pad;
  };
  static const int env_s = getenv("FGL_TC4_STAGES") ? atoi(getenv("FGL_TC4_STAGES")) : 0;
  int S = std::min(env_s > 0 ? env_s : T4_MAX_STAGES, (512 - 2 * N_pad) / 32);
  while (S >= 2 && fixed(S) > G3_MAX_SMEM) --S;
  if (S < 2) return false;
  int cols = 32;
  while (cols < 2 * N_pad + 32 * S) cols <<= 1;
  if (cols > 512) return false;
  CUtensorMap mA, mM, mC, mW;
  std::memset(&mM, 0, sizeof(mM));
  std::memset(&mW, 0, sizeof(mW));
  if (w_tma && !(mode == 0 ? make_map_cols(&mW, W, K, N, ldw, w_ld, 32) : make_map_cols(&mW, W, N, K, ldw, 32, N)))
    return false;
  if (!cached_map_sw128(&mA, A, M, K, lda) || !cached_map_sw128(&mC, C, M, N, ldc) ||
      (has_mask && !cached_map_sw128(&mM, mask, M, K, ldm)))
    return false;
  static bool attr[2] = {false, false};
  if (!attr[mode]) {
    const cudaError_t e =
        mode == 0 ? cudaFuncSetAttribute(tc_dense4_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, G3_MAX_SMEM)
                  : cudaFuncSetAttribute(tc_dense4_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, G3_MAX_SMEM);
    if (e != cudaSuccess) { *err = cuda_status(e, "cudaFuncSetAttribute(tc_dense4)"); return true; }
    attr[mode] = true;
  }
  static const int dbg = getenv("FGL_G3DBG") ? atoi(getenv("FGL_G3DBG")) : 0;
  const int stage_off = (int)(2 * (int64_t)img_boxes * N_pad * 128 + (int64_t)S * stage_bytes);
  T4Args p{W, bias, M, ldw, N, K, N_pad, K_pad, S, relu, has_mask, cols,
           !(reinterpret_cast<uintptr_t>(W) & 15) && ((mode == 0 ? N : K) % 4 == 0) && (ldw % 4 == 0), stage_off, dbg,
           stream_w, w_tma ? (mode == 0 ? 32 * w_ld : N * 32) * 4 : 0, w_ld};
  const int grid = (int)std::min<int64_t>(ceil_div(M, T4_M), dense_cta_budget());
  const int64_t smem = fixed(S);
  const ProfMark pm = prof_begin(st);
  if (mode == 0) FGL_COUNT_LAUNCH(), tc_dense4_kernel<0><<<grid, T4_THREADS, smem, st>>>(mA, mM, mC, mW, p);
  else FGL_COUNT_LAUNCH(), tc_dense4_kernel<1><<<grid, T4_THREADS, smem, st>>>(mA, mM, mC, mW, p);
  prof_end(pm, mode == 0 ? kProfDenseFwd : kProfDgrad, M, N, K);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) *err = cuda_status(e, "tc_dense4_kernel");
  return true;
}

}  // namespace

// Returns false if the shape is outside this kernel's envelope (caller falls
// back); *err receives an FGL status otherwise.
bool tc_gemm3(int mode, const float* A, int64_t lda, const float* mask, int64_t ldm, const float* W,
              const float* bias, float* C, int64_t ldc, int64_t M, int N, int K, int relu, cudaStream_t st,
              int* err, int accum, int64_t ldw) {
  *err = 0;
  if (ldw < 0) ldw = mode == 0 ? N : K;
  if (!accum && !tc3_disabled() && ldw >= (mode == 0 ? N : K) &&
      tc_dense4(mode, A, lda, mask, ldm, W, bias, C, ldc, M, N, K, relu, ldw, st, err))
    return true;
  if (tc3_disabled() || M < 1 || N < 1 || K < 1 || K > 128 || lda < K || ldw < (mode == 0 ? N : K)) return false;
  if ((lda % 4) || (reinterpret_cast<uintptr_t>(A) & 15)) return false;
  const int has_mask = (mode == 1 && mask) ? 1 : 0;
  if (has_mask && ((ldm % 4) || ldm < K || (reinterpret_cast<uintptr_t>(mask) & 15))) return false;
  const int N_pad = (N + 15) / 16 * 16;
  const int K_pad = (K + 7) / 8 * 8;
  if (N_pad > 256) return false;
  // TMEM: two accumulators + a ring of NC A chunks (64 columns each)
  const int NC = std::min(8, (512 - 2 * N_pad) / (2 * G3_KCH));
  if (NC < 2) return false;
  // a column slice of A (a K slice, or rows wider than 256 floats that
  // whole-row bulk copies could not stage): 2-D TMA tensor copies of [128
  // rows x K_box] tiles of A (and of the mask) instead
  const int K4 = (K + 3) / 4 * 4;
  const int a_tma = (lda > 256 || lda > K4 || (has_mask && (ldm > 256 || ldm > K4))) ? 1 : 0;
  const int a_lds = a_tma ? K4 : (int)lda;
  const int m_lds = a_tma ? K4 : (int)ldm;
  const int64_t a_slot = (int64_t)G3_M * a_lds * 4, m_slot = has_mask ? (int64_t)G3_M * m_lds * 4 : 0;
  static const int dbg = getenv("FGL_G3DBG") ? atoi(getenv("FGL_G3DBG")) : 0;
  static const int rmax = getenv("FGL_G3SLOTS") ? atoi(getenv("FGL_G3SLOTS")) : G3_MAX_SLOTS;
  // stage mode: 1 (default) = stage the epilogue for TMA tensor stores; 0 =
  // trade the staging tile for a third raw slot and direct row stores
  // (measured slower: 28.3 vs 26.6 us at the products layer-0 shape)
  static const int stage_pref = getenv("FGL_G3STAGE") ? atoi(getenv("FGL_G3STAGE")) : 1;
  int R = 0;
  for (int r = G3_MAX_SLOTS; r >= 2; --r)
    if (g3_smem(N_pad, K_pad, r, a_slot, m_slot) <= G3_MAX_SMEM) { R = r; break; }
  bool stage = true;
  if (stage_pref == 0 && R < 3 && rmax >= 3 &&
      g3_fixed(N_pad, K_pad, 3, a_slot, m_slot) <= G3_MAX_SMEM) {
    R = 3;
    stage = false;
  }
  if (R == 0) {  // no room for the staging tile (wide N with a mask): direct row stores
    for (int r = 3; r >= 2 && R == 0; --r)
      if (g3_fixed(N_pad, K_pad, r, a_slot, m_slot) <= G3_MAX_SMEM) R = r;
    stage = false;
  }
  if (R == 0) return false;
  if (R > rmax) R = rmax;
  const int cols = 512;
  // output through TMA tensor stores (SW128 boxes of 128 rows x 32 columns)
  // tensor-map encodes cost host microseconds per call; the trainer reuses
  // the same output buffers every batch, so keep the last few maps
  struct MapCache { const float* C; int64_t M, ldc; int N; CUtensorMap m; };
  static thread_local MapCache cache[8];
  static thread_local int cache_next = 0;
  CUtensorMap mC;
  std::memset(&mC, 0, sizeof(mC));
  bool coal = false;
  if (stage && (ldc % 4 == 0) && !(reinterpret_cast<uintptr_t>(C) & 15)) {
    for (auto& c : cache)
      if (c.C == C && c.M == M && c.N == N && c.ldc == ldc) { mC = c.m; coal = true; break; }
    if (!coal && make_map_sw128(&mC, C, M, N, ldc)) {
      MapCache& c = cache[cache_next];
      cache_next = (cache_next + 1) % 8;
      c.C = C; c.M = M; c.N = N; c.ldc = ldc; c.m = mC;
      coal = true;
    }
  }
  const int64_t stage_off = (g3_fixed(N_pad, K_pad, R, a_slot, m_slot) - 1024 + 1023) / 1024 * 1024;
  G3Args p{A, mask, W, bias, C, lda, ldm, ldc, M, N, K, N_pad, K_pad, R, NC, relu, has_mask, cols,
           (int)a_slot, (int)m_slot, dbg, coal ? (int)stage_off : -1, 0,
           !(reinterpret_cast<uintptr_t>(W) & 15) && ((mode == 0 ? N : K) % 4 == 0) && (ldw % 4 == 0), accum, a_tma,
           a_lds, m_lds, ldw};
  const int64_t smem = coal ? g3_smem(N_pad, K_pad, R, a_slot, m_slot) : g3_fixed(N_pad, K_pad, R, a_slot, m_slot);
  static bool attr[2] = {false, false};
  cudaError_t e;
  if (!attr[mode]) {
    e = mode == 0 ? cudaFuncSetAttribute(tc_gemm3_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, G3_MAX_SMEM)
                  : cudaFuncSetAttribute(tc_gemm3_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, G3_MAX_SMEM);
    if (e != cudaSuccess) { *err = cuda_status(e, "cudaFuncSetAttribute(tc_gemm3)"); return true; }
    attr[mode] = true;
  }
  const int64_t tiles = ceil_div(M, G3_M);
  // persistent CTAs (one per SM by smem), at most fgl_set_dense_ctas' budget
  const int grid = (int)std::min<int64_t>(tiles, dense_cta_budget());
  CUtensorMap mA, mM;
  std::memset(&mA, 0, sizeof(mA));
  std::memset(&mM, 0, sizeof(mM));
  if (a_tma && (!make_map_cols(&mA, A, M, K, lda, a_lds, G3_M) ||
                (has_mask && !make_map_cols(&mM, mask, M, K, ldm, m_lds, G3_M))))
    return false;
  const ProfMark pm = prof_begin(st);
  if (mode == 0) FGL_COUNT_LAUNCH(), tc_gemm3_kernel<0><<<grid, G3_THREADS, smem, st>>>(mC, mA, mM, p);
  else FGL_COUNT_LAUNCH(), tc_gemm3_kernel<1><<<grid, G3_THREADS, smem, st>>>(mC, mA, mM, p);
  prof_end(pm, mode == 0 ? kProfDenseFwd : kProfDgrad, M, N, K);
  e = cudaGetLastError();
  if (e != cudaSuccess) *err = cuda_status(e, "tc_gemm3_kernel");
  return true;
}

bool tc_gemm(int mode, const float* A, int64_t lda, const float* mask, int64_t ldm, const float* W,
             const float* bias, float* C, int64_t ldc, int64_t M, int N, int K, int relu, cudaStream_t st,
             int* err) {
  return tc_gemm3(mode, A, lda, mask, ldm, W, bias, C, ldc, M, N, K, relu, st, err, 0);
}

// Weight-gradient partials part[c][K+1][N] (row K = db) over `chunks` CTAs;
// returns false outside the envelope (K <= 128, N <= 256, 16-byte rows; at
// K = 128 the db row comes from the converters instead of a TMEM ones lane).
bool tc_wgrad3(const float* H, int64_t ldh, const float* dZ, int64_t ldz, const float* mask, int64_t ldm,
               int64_t M, int K, int N, float* part, int chunks, cudaStream_t st, int* err, int nks, int kslice) {
  *err = 0;
  if (nks < 1 || (nks > 1 && (kslice < 1 || kslice + 1 > G3_M || (int64_t)(nks - 1) * kslice >= K))) return false;
  const int Kw = nks > 1 ? kslice : K;  // widest slice of this launch
  if (tc3_disabled() || M < 1 || K < 1 || Kw > G3_M || N < 1 || N > 256) return false;
  const int db_conv = Kw == G3_M ? 1 : 0;
  if ((ldh % 4) || (ldz % 4) || (reinterpret_cast<uintptr_t>(H) & 15) || (reinterpret_cast<uintptr_t>(dZ) & 15))
    return false;
  if (mask && ((ldm % 4) || (reinterpret_cast<uintptr_t>(mask) & 15))) return false;
  const int N_pad = (N + 15) / 16 * 16;
  // a column slice of a wide H (ldh > 256 floats): 2-D TMA tensor copies of
  // [64 rows x K_box] tiles instead of whole-row bulk copies
  const int h_tma = (ldh > 256 || nks > 1) ? 1 : 0;
  const int h_lds = h_tma ? (Kw + 3) / 4 * 4 : (int)ldh;
  // a column slice of dZ / mask (an N slice of a wider layer, or rows wider
  // than 256 floats): TMA tensor copies of [64 rows x N_box] tiles
  const int N4 = (N + 3) / 4 * 4;
  const int z_tma = (ldz > 256 || ldz > N4 || (mask && (ldm > 256 || ldm > N4))) ? 1 : 0;
  const int z_lds = z_tma ? N4 : (int)ldz, m_lds = z_tma ? N4 : (int)ldm;
  const int hb = WG3_MT * h_lds * 4, zb = WG3_MT * z_lds * 4, mb = mask ? WG3_MT * m_lds * 4 : 0;
  // deepest raw-tile ring that fits next to the chunk ring: the kernel is a
  // stream over H / dZ / mask, so bytes in flight per SM set its speed
  static const int env_r = getenv("FGL_WG3_R") ? atoi(getenv("FGL_WG3_R")) : 0;
  static const int env_nc = getenv("FGL_WG3_NC") ? atoi(getenv("FGL_WG3_NC")) : 0;
  const int NC = env_nc > 0 ? env_nc : WG3_NC;
  auto smem_of = [&](int R) {
    return 1024 + (int64_t)NC * 2 * N_pad * 128 + (int64_t)R * (hb + zb + mb) + 8 * (2 * R + 2 * NC + 1) + 16 +
           (db_conv ? 16 + 24 * 4 * (int64_t)N_pad : 0);
  };
  int R = env_r > 0 ? env_r : WG3_R_MAX;
  while (R > 2 && smem_of(R) > G3_MAX_SMEM) --R;
  const int64_t smem = smem_of(R);
  if (smem > G3_MAX_SMEM) return false;
  static const int env_acc = getenv("FGL_WG3_ACC") ? atoi(getenv("FGL_WG3_ACC")) : 4;
  const int nacc = std::max(1, std::min(env_acc, (512 - 64 * NC) / N_pad));
  int cols = 32;
  while (cols < nacc * N_pad + 64 * NC) cols <<= 1;
  if (cols > 512) return false;
  static bool attr = false;
  cudaError_t e;
  if (!attr) {
    e = cudaFuncSetAttribute(tc_wgrad3_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, G3_MAX_SMEM);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(tc_wgrad3_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, G3_MAX_SMEM);
    if (e != cudaSuccess) { *err = cuda_status(e, "cudaFuncSetAttribute(tc_wgrad3)"); return true; }
    attr = true;
  }
  static const int dbg = getenv("FGL_G3DBG") ? atoi(getenv("FGL_G3DBG")) : 0;
  Wg3Args p{H, dZ, mask, ldh, ldz, ldm, part, M, K, N, N_pad, cols, hb, zb, mb, dbg, R, NC, nacc, h_tma, h_lds,
            z_tma, z_lds, m_lds, db_conv, nks, kslice, (int64_t)chunks * (Kw + 1) * N};
  CUtensorMap mH, mZ, mM;
  std::memset(&mH, 0, sizeof(mH));
  std::memset(&mZ, 0, sizeof(mZ));
  std::memset(&mM, 0, sizeof(mM));
  if (h_tma && !make_map_cols(&mH, H, M, K, ldh, h_lds, WG3_MT)) return false;  // all K columns: slices by offset
  if (z_tma && (!make_map_cols(&mZ, dZ, M, N, ldz, z_lds, WG3_MT) ||
                (mask && !make_map_cols(&mM, mask, M, N, ldm, m_lds, WG3_MT))))
    return false;
  if (db_conv) FGL_COUNT_LAUNCH(), tc_wgrad3_kernel<true><<<chunks * nks, G3_THREADS, smem, st>>>(mH, mZ, mM, p);
  else FGL_COUNT_LAUNCH(), tc_wgrad3_kernel<false><<<chunks * nks, G3_THREADS, smem, st>>>(mH, mZ, mM, p);
  e = cudaGetLastError();
  if (e != cudaSuccess) *err = cuda_status(e, "tc_wgrad3_kernel");
  return true;
}

}  // namespace fgl

extern "C" int fgl_set_dense_ctas(int32_t ctas) {
  if (ctas < 0) return FGL_E_INVALID;
  fgl::g_dense_ctas.store(ctas == 0 ? fgl::kNumSMs : std::min(ctas, fgl::kNumSMs), std::memory_order_relaxed);
  return FGL_OK;
}

extern "C" int fgl_debug_g3_trace(int64_t* host, int64_t n) {
  return cudaMemcpyFromSymbol(host, fgl::g3_trace, sizeof(int64_t) * (n < 148 * fgl::G3_TR ? n : 148 * fgl::G3_TR)) == cudaSuccess ? 0 : -1;
}
