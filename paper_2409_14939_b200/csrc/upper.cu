// Fused training step of the UPPER model layers (1 .. L-1) of a compact GCN
// batch in one persistent kernel (sm_100a).
//
// Layers 1 .. L-1 of the sampled block graph are small (products, batch 1024:
// ~15K and ~1K rows) and their dozen kernels per batch -- aggregation, dense,
// loss, dense backward, transposed aggregation, partial reductions -- were
// each latency bound (~10 us apiece for microseconds of work).  Here every
// phase of trainer._forward / _softmax_xent / _backward (trainer.py:182-228)
// for those layers is a grid-stride loop of one persistent kernel, separated
// by a device-wide barrier (all CTAs co-resident by construction: the grid is
// sized from the occupancy calculator):
//
//   for i = 1 .. L-1:   H_i = A_i X_i          (CSR order, __fmul_rn/__fadd_rn:
//                                               bit-identical to fgl_spmm)
//                       Y_i = act(H_i W_i + b_i)   (fp32 FMA)
//   loss:               fp64 softmax cross entropy over the seed rows,
//                       dY_{L-1} = (p - onehot) / B     (softmax_xent_kernel)
//   for i = L-1 .. 1:   dZ = dY_i * relu'(Y_i);  dW_i, db_i partials per CTA;
//                       dH_i = dZ W_i^T;  dY_{i-1} = A_i^T dH_i  (stable
//                       transpose order, bit-identical to fgl_spmm)
//   reduce:             dW_i, db_i = sum of the per-CTA partials in CTA order
//                       (deterministic), loss = sum of per-warp partials.
//
// dY_0 (the gradient of layer 0's output) is left for the layer-0 backward
// (tcgen05 wgrad), which stays a separate kernel.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace fgl {
namespace {

constexpr int UP_THREADS = 256;
constexpr int UP_WG_ROWS = 32;  // rows staged per wgrad tile

struct Barrier {
  unsigned int count;
  unsigned int gen;
};

__device__ __forceinline__ void grid_barrier(Barrier* b, unsigned int nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned int* vgen = &b->gen;
    const unsigned int g = *vgen;
    __threadfence();
    if (atomicAdd(&b->count, 1u) == nblocks - 1) {
      b->count = 0;
      __threadfence();
      atomicAdd(&b->gen, 1u);
    } else {
      while (*vgen == g) __nanosleep(64);
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ float4 fma4_rn(float4 acc, float w, float4 x) {
  acc.x = __fadd_rn(acc.x, __fmul_rn(w, x.x));
  acc.y = __fadd_rn(acc.y, __fmul_rn(w, x.y));
  acc.z = __fadd_rn(acc.z, __fmul_rn(w, x.z));
  acc.w = __fadd_rn(acc.w, __fmul_rn(w, x.w));
  return acc;
}

// Y[r] = sum_e w_e X[col_e - base] in CSR order; identical arithmetic to
// compute.cu's spmm_kernel.  A warp works on 4 rows at once (8 lanes per row,
// each lane up to 4 16-byte chunks of the row, d <= 128), and the feature
// loads of 4 edges per row are issued together: 4 independent index -> edge
// -> feature chains per warp instead of one.
__device__ void agg_phase(const int64_t* __restrict__ indptr, const int32_t* __restrict__ col, int64_t base,
                          const float* __restrict__ w, int64_t nrows, const float* __restrict__ X, int64_t ldx,
                          float* __restrict__ Y, int64_t ldy, int d) {
  constexpr int G = 8, RPW = 4, EB = 4, CPL = 4;
  const int lane = threadIdx.x & 31, grp = lane / G, g = lane % G;
  const unsigned gmask = 0xFFu << (grp * G);
  const int d4 = (d + 3) >> 2;  // <= 32
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t rb = warp * RPW; rb < nrows; rb += nwarps * RPW) {
    const int64_t r = rb + grp;
    const bool live = r < nrows;
    const int64_t e0 = live ? indptr[r] : 0, e1 = live ? indptr[r + 1] : 0;
    float4 acc[CPL];
#pragma unroll
    for (int q = 0; q < CPL; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t e = e0; e < e1; e += G) {
      const int64_t me = e + g;
      const int32_t cl = me < e1 ? (int32_t)(col[me] - base) : 0;
      const float wl = me < e1 ? w[me] : 0.f;
      const int n = (int)(e1 - e < G ? e1 - e : G);
      for (int k0 = 0; k0 < n; k0 += EB) {
        float4 xv[EB][CPL];
        float wk[EB];
#pragma unroll
        for (int u = 0; u < EB; ++u) {
          const int k = k0 + u;
          const int32_t c = __shfl_sync(gmask, cl, k < n ? k : 0, G);
          wk[u] = __shfl_sync(gmask, wl, k < n ? k : 0, G);
          const float4* xr = reinterpret_cast<const float4*>(X + (int64_t)c * ldx);
#pragma unroll
          for (int q = 0; q < CPL; ++q) {
            const int ch = g + G * q;
            xv[u][q] = (k < n && ch < d4) ? __ldg(xr + ch) : make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
#pragma unroll
        for (int u = 0; u < EB; ++u)
          if (k0 + u < n) {
#pragma unroll
            for (int q = 0; q < CPL; ++q) acc[q] = fma4_rn(acc[q], wk[u], xv[u][q]);
          }
      }
    }
    if (live) {
#pragma unroll
      for (int q = 0; q < CPL; ++q) {
        const int ch = g + G * q;
        if (ch < d4) reinterpret_cast<float4*>(Y + r * ldy)[ch] = acc[q];
      }
    }
  }
}

// out[r][o] = act(sum_k A[r][k] * Wm[k][o] + bias[o]), Wm = W (K x N row-major)
// or W^T (trans_w: W is N x K); optional mask A[r][k] * (M[r][k] > 0).
// One warp per row: the row is loaded once (lane holds A[r][lane + 32 j]),
// broadcast by shuffles; lane owns outputs o = lane + 32 j; Wm in shared memory.
constexpr int UP_MAXK = 128, UP_MAXN = 192;
__device__ void dense_phase(const float* __restrict__ A, int64_t lda, const float* __restrict__ M, int64_t ldm,
                            int64_t n, int K, int N, const float* __restrict__ W, int trans_w,
                            const float* __restrict__ bias, int relu, float* __restrict__ out, int64_t ldo,
                            float* Ws) {
  // stage Wm: 16 independent loads per thread in flight, then the stores
  for (int base = threadIdx.x; base < K * N; base += 16 * blockDim.x) {
    float v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int i = base + u * blockDim.x;
      v[u] = 0.f;
      if (i < K * N) {
        const int k = i / N, o = i - (i / N) * N;
        v[u] = trans_w ? __ldg(W + (int64_t)o * K + k) : __ldg(W + i);
      }
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int i = base + u * blockDim.x;
      if (i < K * N) Ws[i] = v[u];
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  auto load_row = [&](int64_t r, float (&av)[UP_MAXK / 32]) {
#pragma unroll
    for (int j = 0; j < UP_MAXK / 32; ++j) {
      const int k = lane + 32 * j;
      float v = 0.f;
      if (r < n && k < K) {
        v = A[r * lda + k];
        if (M && !(M[r * ldm + k] > 0.f)) v = 0.f;
      }
      av[j] = v;
    }
  };
  float nxt[UP_MAXK / 32];
  load_row(warp, nxt);
  for (int64_t r = warp; r < n; r += nwarps) {
    float av[UP_MAXK / 32];
#pragma unroll
    for (int j = 0; j < UP_MAXK / 32; ++j) av[j] = nxt[j];
    load_row(r + nwarps, nxt);  // next row's loads overlap this row's math
    float acc[UP_MAXN / 32];
#pragma unroll
    for (int j = 0; j < UP_MAXN / 32; ++j) acc[j] = 0.f;
#pragma unroll
    for (int j = 0; j < UP_MAXK / 32; ++j) {
      if (32 * j >= K) break;
      const int kn = K - 32 * j < 32 ? K - 32 * j : 32;
      for (int t = 0; t < kn; ++t) {
        const float a = __shfl_sync(0xffffffffu, av[j], t);
        const float* wr = Ws + (32 * j + t) * N + lane;
#pragma unroll
        for (int q = 0; q < UP_MAXN / 32; ++q)
          if (lane + 32 * q < N) acc[q] = __fmaf_rn(a, wr[32 * q], acc[q]);
      }
    }
    float* orow = out + r * ldo;
#pragma unroll
    for (int q = 0; q < UP_MAXN / 32; ++q) {
      const int o = lane + 32 * q;
      if (o >= N) break;
      float y = acc[q];
      if (bias) y = __fadd_rn(y, bias[o]);
      if (relu) y = y > 0.f ? y : 0.f;
      orow[o] = y;
    }
  }
  __syncthreads();
}

// per-CTA partial [dW; db] over a contiguous row chunk:
// part[blk][k][o] = sum_r H[r][k] dZ[r][o] (k < K), part[blk][K][o] = sum_r dZ[r][o]
__device__ void wgrad_phase(const float* __restrict__ H, int64_t ldh, const float* __restrict__ dY, int64_t ldd,
                            const float* __restrict__ Y, int64_t ldy, int use_mask, int64_t n, int K, int N,
                            float* __restrict__ part, float* smem) {
  float* Hs = smem;                      // [UP_WG_ROWS][K]
  float* Zs = smem + UP_WG_ROWS * K;     // [UP_WG_ROWS][N]
  const int pairs = (K + 1) * N;
  const int per = (pairs + blockDim.x - 1) / blockDim.x;  // <= 64 for K, N <= 128 ... bounded below
  float acc[24];
#pragma unroll
  for (int q = 0; q < 24; ++q) acc[q] = 0.f;
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = blockIdx.x * chunk, r1 = (r0 + chunk < n ? r0 + chunk : n);
  for (int64_t t0 = r0; t0 < r1; t0 += UP_WG_ROWS) {
    const int rows = (int)(r1 - t0 < UP_WG_ROWS ? r1 - t0 : UP_WG_ROWS);
    {  // stage the tile: all loads of a thread in flight together
      float hv[16], zv[16], mv[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int i = threadIdx.x + u * blockDim.x;
        hv[u] = 0.f; zv[u] = 0.f; mv[u] = 1.f;
        if (i < UP_WG_ROWS * K) {
          const int rr = i / K, k = i - (i / K) * K;
          if (rr < rows) hv[u] = H[(t0 + rr) * ldh + k];
        }
        if (i < UP_WG_ROWS * N) {
          const int rr = i / N, o = i - (i / N) * N;
          if (rr < rows) {
            zv[u] = dY[(t0 + rr) * ldd + o];
            if (use_mask) mv[u] = Y[(t0 + rr) * ldy + o];
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int i = threadIdx.x + u * blockDim.x;
        if (i < UP_WG_ROWS * K) Hs[i] = hv[u];
        if (i < UP_WG_ROWS * N) Zs[i] = (mv[u] > 0.f) ? zv[u] : 0.f;
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 24; ++q) {
      if (q >= per) break;
      const int p = threadIdx.x + q * blockDim.x;
      if (p >= pairs) break;
      const int k = p / N, o = p % N;
      float s = acc[q];
      for (int rr = 0; rr < rows; ++rr) {
        const float h = k < K ? Hs[rr * K + k] : 1.f;
        s = __fmaf_rn(h, Zs[rr * N + o], s);
      }
      acc[q] = s;
    }
    __syncthreads();
  }
  float* out = part + (int64_t)blockIdx.x * pairs;
#pragma unroll
  for (int q = 0; q < 24; ++q) {
    if (q >= per) break;
    const int p = threadIdx.x + q * blockDim.x;
    if (p < pairs) out[p] = acc[q];
  }
}

__device__ int64_t up_trace[64];
__device__ __forceinline__ void up_mark(int i, int on) {
  if (on && blockIdx.x == 0 && threadIdx.x == 0 && i < 64) {
    int64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    up_trace[i] = t;
  }
}

struct UpperDev {
  int dbg;
  fgl_upper_args a;
  float* part[3];       // per layer [gridDim][(din+1)*dout]
  double* loss_part;    // [gridDim * warps]
  Barrier* bar;
};

__global__ void __launch_bounds__(UP_THREADS) upper_kernel(const __grid_constant__ UpperDev u) {
  extern __shared__ __align__(16) float smem[];
  const fgl_upper_args& a = u.a;
  const unsigned nb = gridDim.x;
  const int L1 = a.num_upper;  // layers 1 .. L1
  int tk = 1;
  up_mark(0, u.dbg);
  // ---------------------------------------------------------------- forward
  for (int i = 0; i < L1; ++i) {
    const fgl_upper_layer& l = a.layer[i];
    const float* X = i == 0 ? a.X1 : a.layer[i - 1].Y;
    const int64_t ldx = i == 0 ? a.ldx1 : a.layer[i - 1].ldy;
    agg_phase(l.indptr, l.col, l.col_base, l.w, l.rows, X, ldx, l.H, l.ldh, l.din);
    grid_barrier(u.bar, nb); up_mark(tk++, u.dbg);
    dense_phase(l.H, l.ldh, nullptr, 0, l.rows, l.din, l.dout, l.W, 0, l.b, i < L1 - 1 ? 1 : 0, l.Y, l.ldy, smem);
    grid_barrier(u.bar, nb); up_mark(tk++, u.dbg);
  }
  // ------------------------------------------------------------------ loss
  {
    const fgl_upper_layer& l = a.layer[L1 - 1];
    const int lane = threadIdx.x & 31;
    const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int C = a.num_classes;
    const int64_t B = a.num_seeds;
    double lsum = 0.0;
    for (int64_t i = warp; i < B; i += nwarps) {
      const int64_t r = a.seed_rows[i] - a.seed_row_base;
      const float* z = l.Y + r * l.ldy;
      double mx = -INFINITY;
      for (int c = lane; c < C; c += 32) mx = fmax(mx, (double)z[c]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      double se = 0.0;
      for (int c = lane; c < C; c += 32) se += exp((double)z[c] - mx);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
      const int64_t y = a.labels[a.seed_ids ? (int64_t)a.seed_ids[i] : i];
      for (int c = lane; c < C; c += 32) {
        const double p = exp((double)z[c] - mx) / se;
        const double g = (c == y ? p - 1.0 : p) / (double)B;
        l.dY[r * l.ldy + c] = (float)g;
        if (c == y) lsum += -log(p + 1e-30);
      }
    }
    lsum = warp_sum(lsum);
    if (lane == 0) u.loss_part[warp] = lsum;
  }
  grid_barrier(u.bar, nb); up_mark(tk++, u.dbg);
  // -------------------------------------------------------------- backward
  for (int i = L1 - 1; i >= 0; --i) {
    const fgl_upper_layer& l = a.layer[i];
    const int use_mask = i < L1 - 1 ? 1 : 0;
    wgrad_phase(l.H, l.ldh, l.dY, l.ldy, l.Y, l.ldy, use_mask, l.rows, l.din, l.dout, u.part[i], smem);
    __syncthreads();
    // dH = (dY * relu'(Y)) W^T  ->  [rows][din]
    dense_phase(l.dY, l.ldy, use_mask ? l.Y : nullptr, l.ldy, l.rows, l.dout, l.din, l.W, 1, nullptr, 0, l.dH,
                l.ldh, smem);
    grid_barrier(u.bar, nb); up_mark(tk++, u.dbg);
    if (i == 0 && !a.dX1) continue;  // layer 1 -> layer 0 rows: caller runs fgl_spmm (wide gather)
    float* dXout = i == 0 ? a.dX1 : a.layer[i - 1].dY;
    const int64_t lddx = i == 0 ? a.ldx1 : a.layer[i - 1].ldy;
    agg_phase(l.t_indptr, l.t_col, l.t_base, l.t_w, l.prev_rows, l.dH, l.ldh, dXout, lddx, l.din);
    grid_barrier(u.bar, nb); up_mark(tk++, u.dbg);
  }
  // ------------------------------------------- deterministic reductions
  for (int i = 0; i < L1; ++i) {
    const fgl_upper_layer& l = a.layer[i];
    const int pairs = (l.din + 1) * l.dout;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < pairs;
         p += (int64_t)gridDim.x * blockDim.x) {
      float s = 0.f;
      for (unsigned b0 = 0; b0 < nb; b0 += 8) {  // 8 loads in flight, adds in CTA order
        float v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = b0 + q < nb ? u.part[i][(int64_t)(b0 + q) * pairs + p] : 0.f;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (b0 + q < nb) s = __fadd_rn(s, v[q]);
      }
      const int k = (int)(p / l.dout), o = (int)(p % l.dout);
      if (k < l.din) l.dW[(int64_t)k * l.dout + o] = s;
      else l.db[o] = s;
    }
  }
  up_mark(tk++, u.dbg);
  if (blockIdx.x == 0) {
    __shared__ double sm[33];
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    double s = 0.0;
    for (int64_t i = threadIdx.x; i < nw; i += blockDim.x) s += u.loss_part[i];
    s = block_sum(s, sm);
    if (threadIdx.x == 0) *a.loss_sum = s;
  }
}

int up_smem_bytes(const fgl_upper_args* a) {
  int64_t m = 0;
  for (int i = 0; i < a->num_upper; ++i) {
    const auto& l = a->layer[i];
    m = std::max<int64_t>(m, (int64_t)l.din * l.dout);
    m = std::max<int64_t>(m, (int64_t)UP_WG_ROWS * (l.din + l.dout));
  }
  return (int)(4 * m);
}

int up_grid(int smem) {
  static int cached_smem = -1, cached = 0;
  if (smem != cached_smem) {
    cudaFuncSetAttribute(upper_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, std::max(smem, 48 * 1024));
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, upper_kernel, UP_THREADS, smem) != cudaSuccess ||
        per_sm < 1)
      per_sm = 1;
    cached = std::min(per_sm, 2) * kNumSMs;
    cached_smem = smem;
  }
  return cached;
}

}  // namespace
}  // namespace fgl

using namespace fgl;

extern "C" {

int64_t fgl_upper_ws_bytes(const fgl_upper_args* a) {
  if (!a || a->num_upper < 1 || a->num_upper > 3) return 0;
  const int64_t G = 2 * kNumSMs;
  int64_t b = 256;  // barrier
  for (int i = 0; i < a->num_upper; ++i) b += (4 * G * (int64_t)(a->layer[i].din + 1) * a->layer[i].dout + 255) / 256 * 256;
  b += 8 * G * (UP_THREADS / 32);
  return b;
}

int fgl_upper_layers(const fgl_upper_args* a, void* ws, int64_t ws_bytes, void* stream) {
  if (!a || !ws || a->num_upper < 1 || a->num_upper > 3 || a->num_seeds < 1 || a->num_classes < 1 ||
      !a->X1 || !a->seed_rows || !a->labels || !a->loss_sum) {
    set_error("fgl_upper_layers: bad arguments");
    return FGL_E_INVALID;
  }
  for (int i = 0; i < a->num_upper; ++i) {
    const auto& l = a->layer[i];
    if (l.din < 1 || l.dout < 1 || l.din > 128 || l.dout > 192 || (int64_t)(l.din + 1) * l.dout > 24 * UP_THREADS ||
        (l.ldh % 4) || (l.ldy % 4) || l.ldh < l.din || l.ldy < l.dout) {
      set_error("fgl_upper_layers: layer %d shape %dx%d outside the fused kernel", i + 1, l.din, l.dout);
      return FGL_E_UNSUPPORTED;
    }
  }
  if (ws_bytes < fgl_upper_ws_bytes(a)) {
    set_error("fgl_upper_layers: workspace too small");
    return FGL_E_CAPACITY;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int smem = up_smem_bytes(a);
  const int grid = up_grid(smem);
  UpperDev u;
  static const int dbg = getenv("FGL_UPDBG") ? 1 : 0;
  u.dbg = dbg;
  u.a = *a;
  char* p = static_cast<char*>(ws);
  u.bar = reinterpret_cast<Barrier*>(p);
  p += 256;
  for (int i = 0; i < 3; ++i) u.part[i] = nullptr;
  for (int i = 0; i < a->num_upper; ++i) {
    u.part[i] = reinterpret_cast<float*>(p);
    p += (4 * (int64_t)2 * kNumSMs * (a->layer[i].din + 1) * a->layer[i].dout + 255) / 256 * 256;
  }
  u.loss_part = reinterpret_cast<double*>(p);
  FGL_CUDA(cudaMemsetAsync(u.bar, 0, sizeof(Barrier), st));
  FGL_COUNT_LAUNCH(), upper_kernel<<<grid, UP_THREADS, smem, st>>>(u);
  FGL_LAUNCH_CHECK("upper_kernel");
  return FGL_OK;
}

int fgl_debug_upper_trace(int64_t* host) {
  return cudaMemcpyFromSymbol(host, up_trace, sizeof(int64_t) * 64) == cudaSuccess ? 0 : -1;
}

}  // extern "C"
