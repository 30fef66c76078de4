// Fused-Map k-hop window sampler (sm_100a).
//
// Replaces, per batch, sampler.sample_khop (sampler.py:120-139) and -- on the
// trainer path -- idmap.build + translate_batch (idmap.py:198-233, :294-303).
// A whole window of nb batches is sampled by one launch sequence with no host
// synchronisation: sizes live on the device, kernels are launched on fixed
// persistent grids and read their trip counts from device memory.
//
// Data layout in HBM:
//  * per batch two node bitmaps of W = ceil(N/32) words: `front` (sources of
//    the hop being sampled -> next frontier) and `all` (seeds + every sampled
//    source = unique_nodes).  A bitmap is a direct-addressed hash set with an
//    identity hash: insertion is one atomicOr, dedup is free, and compaction
//    in word order yields the SORTED unique list the reference's np.unique
//    produces (sampler.py:129,135,138) -- so the frontier order (which fixes
//    the Philox stream positions) and the local IDs (rank in unique_nodes,
//    trainer.py:167) come out without any sort.
//  * rank(g) = prefix[word(g)] + popc(word & below(g)): O(1) global->local.
//
// Per hop: (1) degree scan over the concatenated frontier (exclusive scans of
// deg and min(deg,f)) -> candidate stream positions and output offsets;
// (2) select: one warp per frontier node draws one Philox4x64-10 block per
// lane per iteration (4 candidates), keeps a warp-distributed sorted list of
// the f smallest (key53, slot) pairs, emits them in key order and marks the
// sources in `front`; (3) compaction of `front` -> next frontier (cleared as
// it is read, OR-ed into `all`).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace fgl {
namespace {

constexpr int kScanThreads = 256;
// CTAs of the sampler's scan / compaction / degree passes (4 per SM: their
// phases are latency bound, so more resident warps, not fewer, set the pace)
constexpr int kSampCTAs = 4 * kNumSMs;
constexpr int kDegTile = 1024;  // frontier entries per tile of the single-pass degree scan
// bitmap passes over large windows (papers100M shape: 27.8M words) take one
// CTA per ~4K words instead of kSampCTAs, so the whole pass's loads are in
// flight at once rather than ~12 serial tiles per CTA
constexpr int kBmMaxCTAs = 16384;
inline int bm_grid(int64_t nwords) {
  // one tile per CTA: 4096 words (16-word runs) for large bitmaps, 1024
  // words (4-word runs) otherwise -- a 1040-word chunk cost a second block
  // scan for 16 words (products: 613K words over 592 CTAs)
  const int64_t per = ceil_div(nwords, kSampCTAs) >= 4096 ? 4096 : 1024;
  return (int)std::max<int64_t>(kSampCTAs, std::min<int64_t>(kBmMaxCTAs, ceil_div(nwords, per)));
}
constexpr int kMaxFanout = 256;

struct SampleWs {
  uint32_t* bm_front;  // [nb*W]
  uint32_t* bm_all;    // [nb*W]
  int32_t* wprefix;    // [nb*W] exclusive popcount prefix of bm_all (global)
  uint2* wrank;        // [nb*W] {prefix, bm_all word} interleaved: a rank costs one sector
  uint64_t* lb;        // [2 * (fcap / kDegTile + 2)] degree-scan look-back status words (degrees, selections)
  int32_t* lbflag;     // [4] degree-scan tile counter
  int32_t* posmap;     // [ucap] window row -> index in a hop's frontier list
  int32_t* fb;         // [fcap] batch of each frontier entry
  int64_t* scan_deg;   // [fcap]
  int64_t* scan_sel;   // [fcap]
  int64_t* part;       // [2*kBmMaxCTAs + 2]
  int64_t* pos;        // [nb]   running Philox position per batch
  int64_t* hop_pos;    // [nb]   position at the start of the current hop
  int64_t* scal;       // [8]
  int32_t* hub_list;   // [fcap] hub frontier entries of the current hop
};

enum Scal { kF = 0, kCandTot = 1, kSelTot = 2, kEdgeBase = 3, kHopEdgeBase = 4, kUniqTot = 5, kTileCtr = 6,
            kHubCnt = 7, kHubBig = 8 };
// hubs above this degree are queued at the front of the hub list and taken
// first by select_hub_kernel (longest first: they no longer start in a late
// wave and set the kernel's tail)
constexpr int64_t kGiantHub = 6144;

inline int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

struct WsLayout {
  int64_t words, fcap, bytes;
  int64_t off_front_bm, off_all_bm, off_wprefix, off_wrank, off_lb, off_lbflag, off_posmap, off_fb, off_sdeg, off_ssel, off_part,
      off_pos, off_hoppos, off_scal, off_hub;
};

WsLayout ws_layout(int64_t num_nodes, int32_t nb, int64_t fcap, int64_t ucap) {
  WsLayout L;
  L.words = align_up(ceil_div(num_nodes, 32), 4);
  L.fcap = std::max<int64_t>(fcap, 1);
  int64_t o = 0;
  auto take = [&](int64_t bytes) { int64_t r = o; o = align_up(o + bytes, 256); return r; };
  L.off_front_bm = take(4 * L.words * nb);
  L.off_all_bm = take(4 * L.words * nb);
  L.off_wprefix = take(4 * L.words * nb);
  L.off_wrank = take(8 * L.words * nb);
  L.off_lbflag = take(16);
  L.off_lb = take(8 * 2 * (L.fcap / kDegTile + 2));  // right after the counter: one memset clears both
  L.off_posmap = take(4 * std::max<int64_t>(ucap, 1));
  L.off_fb = take(4 * L.fcap);
  L.off_sdeg = take(8 * L.fcap);
  L.off_ssel = take(8 * L.fcap);
  L.off_part = take(8 * (2 * kBmMaxCTAs + 2));
  L.off_pos = take(8 * nb);
  L.off_hoppos = take(8 * nb);
  L.off_scal = take(8 * 16);
  L.off_hub = take(4 * L.fcap);
  L.bytes = o;
  return L;
}

SampleWs carve(void* base, const WsLayout& L) {
  char* p = static_cast<char*>(base);
  SampleWs w;
  w.bm_front = reinterpret_cast<uint32_t*>(p + L.off_front_bm);
  w.bm_all = reinterpret_cast<uint32_t*>(p + L.off_all_bm);
  w.wprefix = reinterpret_cast<int32_t*>(p + L.off_wprefix);
  w.wrank = reinterpret_cast<uint2*>(p + L.off_wrank);
  w.lb = reinterpret_cast<uint64_t*>(p + L.off_lb);
  w.lbflag = reinterpret_cast<int32_t*>(p + L.off_lbflag);
  w.posmap = reinterpret_cast<int32_t*>(p + L.off_posmap);
  w.fb = reinterpret_cast<int32_t*>(p + L.off_fb);
  w.scan_deg = reinterpret_cast<int64_t*>(p + L.off_sdeg);
  w.scan_sel = reinterpret_cast<int64_t*>(p + L.off_ssel);
  w.part = reinterpret_cast<int64_t*>(p + L.off_part);
  w.pos = reinterpret_cast<int64_t*>(p + L.off_pos);
  w.hop_pos = reinterpret_cast<int64_t*>(p + L.off_hoppos);
  w.scal = reinterpret_cast<int64_t*>(p + L.off_scal);
  w.hub_list = reinterpret_cast<int32_t*>(p + L.off_hub);
  return w;
}

__device__ __forceinline__ int find_segment(const int64_t* off, int n, int64_t i) {
  // largest s with off[s] <= i (off non-decreasing, n+1 entries); n <= 64 so
  // a branch-light binary search over cached loads is enough
  int lo = 0, hi = n;  // invariant off[lo] <= i < off[hi]
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (__ldg(off + mid) <= i) lo = mid; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ void set_status(int64_t* status, int64_t code) {
  atomicCAS(reinterpret_cast<unsigned long long*>(status), 0ull, (unsigned long long)code);
}

// ---------------------------------------------------------------- seeds ----
__global__ void mark_seeds_kernel(const int32_t* __restrict__ seeds, const int64_t* __restrict__ seed_off,
                                  int32_t nb, int64_t total, int64_t num_nodes, int64_t words,
                                  uint32_t* __restrict__ bm, int64_t* status) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t s = seeds[i];
    if (s < 0 || s >= num_nodes) { set_status(status, FGL_E_INVALID); continue; }
    const int b = find_segment(seed_off, nb, i);
    atomicOr(bm + b * words + (s >> 5), 1u << (s & 31));
  }
}

// ------------------------------------------------------------ bitmap scan --
// chunked over nwords words by kPersistentCTAs CTAs
// a CTA's share of a bitmap pass: a multiple of 16 words, so every thread's
// 16-word run starts 64-byte aligned (bm_count / bm_compact must agree)
__device__ __forceinline__ int64_t bm_chunk(int64_t nwords, int grid) {
  return (ceil_div(nwords, grid) + 15) & ~(int64_t)15;
}
// words per thread per tile: 16 (four 16-byte loads) for large bitmaps, where
// the serial block scans per CTA bound the pass (papers100M shape: 27.8M
// words per pass, 766 -> 597 us of compaction per window); 4 for small ones
// (products: 613K words per pass -- more threads per tile keep it latency-short)
inline int bm_it(int64_t nwords, int grid) { return ceil_div(nwords, grid) >= 4096 ? 16 : 4; }

// 16 consecutive words from w (64-byte aligned run), zeros past w1
__device__ __forceinline__ void bm_load16(const uint32_t* __restrict__ bm, int64_t w, int64_t w1, uint32_t (&v)[16]) {
  if (w + 16 <= w1) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint4 x = __ldg(reinterpret_cast<const uint4*>(bm + w) + k);
      v[4 * k] = x.x; v[4 * k + 1] = x.y; v[4 * k + 2] = x.z; v[4 * k + 3] = x.w;
    }
  } else {
#pragma unroll
    for (int q = 0; q < 16; ++q) v[q] = w + q < w1 ? bm[w + q] : 0u;
  }
}

__global__ void bm_count_kernel(const uint32_t* __restrict__ bm, int64_t nwords, int64_t* part) {
  __shared__ int64_t sm[33];
  const int64_t chunk = bm_chunk(nwords, gridDim.x);
  const int64_t w0 = min(nwords, blockIdx.x * chunk), w1 = min(nwords, w0 + chunk);
  int64_t c = 0;
  if (chunk >= 16 * (int64_t)blockDim.x) {
    for (int64_t w = w0 + 16 * (int64_t)threadIdx.x; w < w1; w += 16 * (int64_t)blockDim.x) {
      uint32_t v[16];
      bm_load16(bm, w, w1, v);
#pragma unroll
      for (int q = 0; q < 16; ++q) c += __popc(v[q]);
    }
  } else {
    for (int64_t w = w0 + threadIdx.x; w < w1; w += blockDim.x) c += __popc(bm[w]);
  }
  c = block_sum(c, sm);
  if (threadIdx.x == 0) part[blockIdx.x] = c;
}

// exclusive scan of n partials in place (one CTA); total -> *total (and
// optionally also to *total2)
__global__ void scan_partials_kernel(int64_t* part, int n, int64_t* total, int64_t* total2) {
  __shared__ int64_t sm[33];
  int64_t carry = 0;
  for (int base = 0; base < n; base += blockDim.x) {
    const int i = base + threadIdx.x;
    int64_t v = i < n ? part[i] : 0, tot;
    int64_t ex = block_excl_scan(v, sm, &tot);
    if (i < n) part[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) {
    *total = carry;
    if (total2) *total2 = carry;
  }
}

// Emit set bits of a batch-major bitmap in word order.  Optionally writes the
// node IDs + batch of each bit, the per-batch start offsets, the per-word
// global exclusive prefix, ORs the words into `or_into`, and clears them.
template <int IT>
__global__ void bm_compact_kernel(uint32_t* __restrict__ bm, int64_t nwords, int64_t words,
                                  const int64_t* __restrict__ part, int32_t* __restrict__ ids,
                                  int32_t* __restrict__ batch_of, int64_t* __restrict__ batch_off,
                                  int32_t* __restrict__ wprefix, uint32_t* __restrict__ or_into,
                                  int clear, int64_t cap, int64_t* status, uint2* __restrict__ wrank) {
  __shared__ int64_t sm[33];
  // a tile's node IDs are staged in shared memory and written out coalesced
  // (dense windows -- products unique sets, ~25 % of bits -- had each thread
  // write its own run: 32 scattered sectors per store instruction)
  constexpr int kStageIds = 6144;
  __shared__ int32_t sids[kStageIds];
  const int64_t chunk = bm_chunk(nwords, gridDim.x);
  const int64_t w0 = min(nwords, blockIdx.x * chunk), w1 = min(nwords, w0 + chunk);
  int64_t base = part[blockIdx.x];
  for (int64_t t0 = w0; t0 < w1; t0 += (int64_t)blockDim.x * IT) {
    const int64_t wf = t0 + (int64_t)threadIdx.x * IT;
    uint32_t v[IT];
    if (IT == 16) {
      bm_load16(bm, wf, w1, reinterpret_cast<uint32_t(&)[16]>(v));
    } else {
#pragma unroll
      for (int q = 0; q < IT; ++q) v[q] = wf + q < w1 ? bm[wf + q] : 0u;
    }
    int64_t local = 0;
#pragma unroll
    for (int q = 0; q < IT; ++q) local += __popc(v[q]);
    int64_t tot;
    int64_t ex = base + block_excl_scan<int64_t>(local, sm, &tot);
    const int64_t tile_base = base;
    const bool staged = ids && !batch_of && tot <= kStageIds && tile_base + tot <= cap;
    int64_t b = wf / words, bstart = b * words;  // batch of word wf (one division per run)
    // the per-word prefix: 16-byte vector stores of a full run (one store
    // instruction per 4 words instead of 4: the store path bound this pass)
    const bool vec_prefix = wprefix && wf + IT <= w1 && (IT % 4) == 0;
    if (vec_prefix) {
      int32_t pre[IT];
      int64_t e = ex;
#pragma unroll
      for (int q = 0; q < IT; ++q) { pre[q] = (int32_t)e; e += __popc(v[q]); }
#pragma unroll
      for (int q = 0; q < IT; q += 4)
        *reinterpret_cast<int4*>(wprefix + wf + q) = make_int4(pre[q], pre[q + 1], pre[q + 2], pre[q + 3]);
      if (wrank) {
#pragma unroll
        for (int q = 0; q < IT; q += 2)
          *reinterpret_cast<uint4*>(wrank + wf + q) = make_uint4((uint32_t)pre[q], v[q], (uint32_t)pre[q + 1], v[q + 1]);
      }
    }
    // all-zero runs (most of a sparse window bitmap) need no per-word pass
    // unless a batch starts inside them or the prefix is stored per word
    const bool has_start = batch_off && (wf == bstart || bstart + words < wf + IT);
    const bool skip = local == 0 && !has_start && !(wprefix && !vec_prefix);
#pragma unroll
    for (int q = 0; q < (skip ? 0 : IT); ++q) {
      const int64_t w = wf + q;
      if (w >= w1) break;
      if (w == bstart + words) { ++b; bstart += words; }
      if (batch_off && w == bstart) batch_off[b] = ex;
      if (wprefix && !vec_prefix) {
        wprefix[w] = (int32_t)ex;
        if (wrank) wrank[w] = make_uint2((uint32_t)ex, v[q]);
      }
      if (v[q]) {
        if (or_into) or_into[w] |= v[q];
        if (clear) bm[w] = 0u;
        if (ids) {
          if (ex + __popc(v[q]) > cap) {
            set_status(status, FGL_E_CAPACITY);
          } else {
            const int32_t node0 = (int32_t)((w - bstart) << 5);
            uint32_t m = v[q];
            int64_t o = ex;
            while (m) {
              const int bit = __ffs(m) - 1;
              m &= m - 1;
              if (staged) sids[o - tile_base] = node0 + bit;
              else ids[o] = node0 + bit;
              if (batch_of) batch_of[o] = (int32_t)b;
              ++o;
            }
          }
        }
      }
      ex += __popc(v[q]);
    }
    if (ids && !batch_of && tot <= kStageIds && tile_base + tot <= cap) {  // block-uniform
      __syncthreads();
      for (int64_t k = threadIdx.x; k < tot; k += blockDim.x) ids[tile_base + k] = sids[k];
      __syncthreads();
    }
    base += tot;
  }
}

void launch_bm_compact(int G, cudaStream_t st, uint32_t* bm, int64_t nwords, int64_t words, const int64_t* part,
                       int32_t* ids, int32_t* batch_of, int64_t* batch_off, int32_t* wprefix, uint32_t* or_into,
                       int clear, int64_t cap, int64_t* status, uint2* wrank = nullptr) {
  if (bm_it(nwords, G) == 16)
    FGL_COUNT_LAUNCH(), bm_compact_kernel<16><<<G, kScanThreads, 0, st>>>(bm, nwords, words, part, ids, batch_of,
                                                                          batch_off, wprefix, or_into, clear, cap,
                                                                          status, wrank);
  else
    FGL_COUNT_LAUNCH(), bm_compact_kernel<4><<<G, kScanThreads, 0, st>>>(bm, nwords, words, part, ids, batch_of,
                                                                         batch_off, wprefix, or_into, clear, cap,
                                                                         status, wrank);
}

// ------------------------------------------------------------ degree scan --
__device__ __forceinline__ void node_deg_sel(const int64_t* __restrict__ off, int32_t u, int fan,
                                             int64_t& d, int64_t& s) {
  d = __ldg(off + u + 1) - __ldg(off + u);
  s = d < fan ? d : fan;
}

// Single-pass degree scan of one hop's frontier (decoupled look-back): per
// entry the draw offset (exclusive scan of degrees) and the output offset
// (exclusive scan of min(degree, fanout)), plus both totals -- one launch
// instead of deg_up + two partial scans + deg_down.  Tiles are claimed in
// launch order through a counter, so a tile only waits on tiles already
// running.  Each tile publishes a status word per sum, flag in bits 62-63
// (1 = its aggregate, 2 = its inclusive prefix) -- one 64-bit store, so no
// fence orders a flag against its value -- and warp 0 looks back 32 tiles
// per step.
__device__ __forceinline__ uint64_t ld_status(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_status(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// exclusive prefix of tile `tile` from the status words of the tiles before it
__device__ __forceinline__ int64_t lookback_prefix(const uint64_t* st, int64_t tile, int lane) {
  constexpr uint64_t kVal = (1ull << 62) - 1;
  int64_t run = 0;
  int64_t p0 = tile - 1;
  for (;;) {
    const int64_t p = p0 - lane;
    const uint64_t v = p >= 0 ? ld_status(st + p) : (2ull << 62);  // before tile 0: inclusive 0
    const unsigned flag = (unsigned)(v >> 62);
    const unsigned incl = __ballot_sync(0xffffffffu, flag == 2);
    const unsigned zero = __ballot_sync(0xffffffffu, flag == 0);
    const int fi = incl ? __ffs(incl) - 1 : 32;  // nearest tile with its inclusive prefix
    const unsigned need = fi == 32 ? 0xffffffffu : ((2u << fi) - 1u);
    if (zero & need) continue;  // a tile up to it has not published yet: re-read
    int64_t x = lane <= fi ? (int64_t)(v & kVal) : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    run += x;
    if (fi < 32) return run;
    p0 -= 32;
  }
}

__global__ void __launch_bounds__(kScanThreads) deg_scan_kernel(const int64_t* __restrict__ off,
                                                                const int32_t* __restrict__ front, int64_t* scal,
                                                                int fan, int64_t* __restrict__ scan_deg,
                                                                int64_t* __restrict__ scan_sel, uint64_t* st_d,
                                                                uint64_t* st_s, int32_t* ctr) {
  __shared__ int64_t sm[33];
  __shared__ int64_t pre[2];
  __shared__ int tile_s;
  const int64_t F = scal[kF];
  const int64_t ntiles = ceil_div(F, kDegTile);
  if (threadIdx.x == 0) tile_s = atomicAdd(ctr, 1);
  __syncthreads();
  const int64_t tile = tile_s;
  if (tile >= ntiles) {
    if (tile == 0 && threadIdx.x == 0) { scal[kCandTot] = 0; scal[kSelTot] = 0; }  // empty frontier
    return;
  }
  constexpr int IT = kDegTile / kScanThreads;
  const int64_t first = tile * kDegTile + (int64_t)threadIdx.x * IT;
  int64_t d[IT], s[IT], ld = 0, ls = 0;
#pragma unroll
  for (int q = 0; q < IT; ++q) {
    d[q] = 0;
    s[q] = 0;
    if (first + q < F) node_deg_sel(off, front[first + q], fan, d[q], s[q]);
  }
#pragma unroll
  for (int q = 0; q < IT; ++q) {  // exclusive within the thread
    const int64_t x = d[q], y = s[q];
    d[q] = ld; s[q] = ls;
    ld += x; ls += y;
  }
  int64_t td, ts;
  const int64_t ed = block_excl_scan(ld, sm, &td);
  const int64_t es = block_excl_scan(ls, sm, &ts);
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    if (lane == 0 && tile > 0) {  // aggregates first: later tiles need not wait for this look-back
      st_status(st_d + tile, (1ull << 62) | (uint64_t)td);
      st_status(st_s + tile, (1ull << 62) | (uint64_t)ts);
    }
    const int64_t pd = tile > 0 ? lookback_prefix(st_d, tile, lane) : 0;
    const int64_t ps = tile > 0 ? lookback_prefix(st_s, tile, lane) : 0;
    if (lane == 0) {
      st_status(st_d + tile, (2ull << 62) | (uint64_t)(pd + td));
      st_status(st_s + tile, (2ull << 62) | (uint64_t)(ps + ts));
      pre[0] = pd;
      pre[1] = ps;
      if (tile == ntiles - 1) {  // the hop's totals
        scal[kCandTot] = pd + td;
        scal[kSelTot] = ps + ts;
      }
    }
  }
  __syncthreads();
  const int64_t bd = pre[0] + ed, bs = pre[1] + es;
#pragma unroll
  for (int q = 0; q < IT; ++q) {
    if (first + q < F) {
      scan_deg[first + q] = bd + d[q];
      scan_sel[first + q] = bs + s[q];
    }
  }
}

// per-batch bookkeeping of one hop (one thread per batch)
__global__ void hop_book_kernel(SampleWs w, const int64_t* __restrict__ fr_off, int32_t nb,
                                int hop, int64_t* __restrict__ counts, int H, int64_t edge_cap) {
  const int64_t F = w.scal[kF];
  if (threadIdx.x == 0) {
    w.scal[kHopEdgeBase] = w.scal[kEdgeBase];
    w.scal[kTileCtr] = 0;  // dynamic tile counter of this hop's select kernel
    w.scal[kHubCnt] = 0;   // hub nodes deferred to select_hub_kernel
    w.scal[kHubBig] = 0;   // of them the giant ones (front of the list)
  }
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    const int64_t f0 = fr_off[b], f1 = fr_off[b + 1];
    const int64_t c0 = f0 < F ? w.scan_deg[f0] : w.scal[kCandTot];
    const int64_t c1 = f1 < F ? w.scan_deg[f1] : w.scal[kCandTot];
    const int64_t s0 = f0 < F ? w.scan_sel[f0] : w.scal[kSelTot];
    w.hop_pos[b] = w.pos[b] - c0;  // so that pos = hop_pos[b] + scan_deg[i]
    w.pos[b] += c1 - c0;
    counts[FGL_CNT_DRAWS(H, nb) + b] += c1 - c0;
    counts[hop * nb + b] = w.scal[kEdgeBase] + s0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    w.scal[kEdgeBase] += w.scal[kSelTot];
    counts[(hop + 1) * nb] = w.scal[kEdgeBase];
    if (w.scal[kEdgeBase] > edge_cap) {  // caller's edge buffer too small: emit nothing
      set_status(counts + FGL_CNT_STATUS(H, nb), FGL_E_CAPACITY);
      w.scal[kF] = 0;
    }
  }
}

// --------------------------------------------------------------- select ----
__device__ __forceinline__ bool key_less(uint64_t ak, uint32_t aj, uint64_t bk, uint32_t bj) {
  return ak < bk || (ak == bk && aj < bj);
}

// Warp-distributed sorted list of up to 32*K (key, slot) pairs; entry
// r = k*32 + lane lives in lane `lane`, register k.
template <int K>
struct TopList {
  uint64_t key[K];
  uint32_t slot[K];

  __device__ __forceinline__ void init() {
#pragma unroll
    for (int k = 0; k < K; ++k) { key[k] = ~0ull; slot[k] = 0xffffffffu; }
  }
  __device__ __forceinline__ void entry(int r, uint64_t& k_out, uint32_t& s_out) const {
    const int kk = r >> 5, ln = r & 31;
    uint64_t kv = 0; uint32_t sv = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const uint64_t a = __shfl_sync(0xffffffffu, key[k], ln);
      const uint32_t b = __shfl_sync(0xffffffffu, slot[k], ln);
      if (k == kk) { kv = a; sv = b; }
    }
    k_out = kv; s_out = sv;
  }
  // insert (ck, cs) keeping the first `f` entries sorted; warp-uniform call
  __device__ __forceinline__ void insert(uint64_t ck, uint32_t cs, int f) {
    int pos = 0;
#pragma unroll
    for (int k = 0; k < K; ++k)
      pos += __popc(__ballot_sync(0xffffffffu, key_less(key[k], slot[k], ck, cs)));
    if (pos >= f) return;
    const int lane = lane_id();
    uint64_t up_k[K]; uint32_t up_s[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      up_k[k] = __shfl_up_sync(0xffffffffu, key[k], 1);
      up_s[k] = __shfl_up_sync(0xffffffffu, slot[k], 1);
    }
    uint64_t carry_k[K]; uint32_t carry_s[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      carry_k[k] = __shfl_sync(0xffffffffu, key[k], 31);
      carry_s[k] = __shfl_sync(0xffffffffu, slot[k], 31);
    }
#pragma unroll
    for (int k = K - 1; k >= 0; --k) {
      const int r = k * 32 + lane;
      uint64_t pk = up_k[k]; uint32_t ps = up_s[k];
      if (lane == 0) {
        if (k > 0) { pk = carry_k[k - 1]; ps = carry_s[k - 1]; }
      }
      if (r == pos) { key[k] = ck; slot[k] = cs; }
      else if (r > pos) { key[k] = pk; slot[k] = ps; }
    }
  }
};

struct SelectArgs {
  const int64_t* off;
  const int32_t* col;
  const float* ew;
  const int32_t* front;
  const int32_t* fb;
  const int64_t* scan_deg;
  const int64_t* scan_sel;
  const int64_t* fr_off;
  const int64_t* hop_pos;
  const uint64_t* keys;
  const int64_t* scal;
  uint32_t* bm_front;
  int64_t words;
  int32_t* tgt;
  int32_t* src;
  float* wgt;
  int32_t* tgt_front;
  int fan;
  unsigned long long* tile_ctr;  // dynamic tile scheduling (select_bal2_kernel)
  unsigned long long* hub_cnt;   // hub nodes (d > kBalHub) deferred to select_hub_kernel
  int32_t* hub_list;             // their frontier indices: giants from the front, the rest from the back
  unsigned long long* hub_big_cnt = nullptr;
  int64_t hub_cap = 0;
};

template <int K>
__global__ void __launch_bounds__(256) select_kernel(SelectArgs a) {
  const int lane = lane_id();
  const int64_t F = a.scal[kF];
  const int64_t ebase = a.scal[kHopEdgeBase];
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int fan = a.fan;
  for (int64_t i = gw; i < F; i += nwarps) {
    const int32_t u = a.front[i];
    const int64_t e0 = __ldg(a.off + u);
    const int64_t d = __ldg(a.off + u + 1) - e0;
    if (d == 0) continue;
    const int b = a.fb[i];
    const uint64_t k0 = a.keys[2 * b], k1 = a.keys[2 * b + 1];
    const int64_t p0 = a.hop_pos[b] + a.scan_deg[i];
    const int64_t p1 = p0 + d;  // exclusive
    const int64_t blk0 = p0 >> 2, blk_last = (p1 - 1) >> 2;
    TopList<K> list;
    list.init();
    uint64_t thr_k = ~0ull; uint32_t thr_s = 0xffffffffu;  // entry f-1 (inf until full)
    for (int64_t bb = blk0; bb <= blk_last; bb += 32) {
      const int64_t blk = bb + lane;
      uint64_t w[4] = {~0ull, ~0ull, ~0ull, ~0ull};
      const bool valid = blk <= blk_last;
      if (valid) philox4x64_10((uint64_t)blk + 1, k0, k1, w[0], w[1], w[2], w[3]);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t p = 4 * blk + q;
        const bool in = valid && p >= p0 && p < p1;
        const uint64_t key = w[q] >> 11;
        const uint32_t slot = (uint32_t)(p - p0);
        unsigned m = __ballot_sync(0xffffffffu, in && key_less(key, slot, thr_k, thr_s));
        while (m) {
          const int srcl = __ffs(m) - 1;
          m &= m - 1;
          const uint64_t ck = __shfl_sync(0xffffffffu, key, srcl);
          const uint32_t cs = __shfl_sync(0xffffffffu, slot, srcl);
          if (key_less(ck, cs, thr_k, thr_s)) {
            list.insert(ck, cs, fan);
            list.entry(fan - 1, thr_k, thr_s);
          }
        }
      }
    }
    // emit min(d, fan) entries in ascending key order
    const int64_t nsel = d < fan ? d : fan;
    const int64_t obase = ebase + a.scan_sel[i];
    uint32_t* bm = a.bm_front + (int64_t)b * a.words;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int r = k * 32 + lane;
      if (r < nsel) {
        const int64_t e = e0 + list.slot[k];
        const int32_t s = __ldg(a.col + e);
        a.tgt[obase + r] = u;
        a.src[obase + r] = s;
        if (a.tgt_front) a.tgt_front[obase + r] = (int32_t)i;
        a.wgt[obase + r] = a.ew ? __ldg(a.ew + e) : 1.0f;
        atomicOr(bm + (s >> 5), 1u << (s & 31));
      }
    }
  }
}

// Threshold-collect select (fanouts <= kTauMaxFan).  The f smallest of d
// uniform keys lie below ~(f + 4 sqrt f + 4)/d with overwhelming probability,
// so one pass draws every candidate's key, keeps only those below that
// threshold in a per-warp shared-memory buffer (warp-aggregated appends), and
// ranks the few survivors by counting: rank = #{collected (key,slot) < own}.
// Exact for any threshold that keeps at least min(d,f) candidates; if too few
// survive the threshold is raised 4x and the node is redrawn, and a buffer
// overflow falls back to the streaming top-list path.  No serial insertion
// chain, so the kernel is Philox-throughput bound rather than latency bound.
constexpr int kTauCap = 256;
constexpr int kTauMaxFan = 128;
constexpr uint64_t kKeyOne = 1ull << 53;

template <int K>
__device__ __noinline__ void stream_select_node(const SelectArgs& a, int64_t i, int32_t u,
                                                   int64_t e0, int64_t d, int b, int64_t p0,
                                                   int64_t obase) {
  const int lane = lane_id();
  const int fan = a.fan;
  const uint64_t k0 = a.keys[2 * b], k1 = a.keys[2 * b + 1];
  const int64_t p1 = p0 + d;
  const int64_t blk0 = p0 >> 2, blk_last = (p1 - 1) >> 2;
  TopList<K> list;
  list.init();
  uint64_t thr_k = ~0ull;
  uint32_t thr_s = 0xffffffffu;
  for (int64_t bb = blk0; bb <= blk_last; bb += 32) {
    const int64_t blk = bb + lane;
    uint64_t w[4] = {~0ull, ~0ull, ~0ull, ~0ull};
    const bool valid = blk <= blk_last;
    if (valid) philox4x64_10((uint64_t)blk + 1, k0, k1, w[0], w[1], w[2], w[3]);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t p = 4 * blk + q;
      const bool in = valid && p >= p0 && p < p1;
      const uint64_t key = w[q] >> 11;
      const uint32_t slot = (uint32_t)(p - p0);
      unsigned m = __ballot_sync(0xffffffffu, in && key_less(key, slot, thr_k, thr_s));
      while (m) {
        const int srcl = __ffs(m) - 1;
        m &= m - 1;
        const uint64_t ck = __shfl_sync(0xffffffffu, key, srcl);
        const uint32_t cs = __shfl_sync(0xffffffffu, slot, srcl);
        if (key_less(ck, cs, thr_k, thr_s)) {
          list.insert(ck, cs, fan);
          list.entry(fan - 1, thr_k, thr_s);
        }
      }
    }
  }
  const int64_t nsel = d < fan ? d : fan;
  uint32_t* bm = a.bm_front + (int64_t)b * a.words;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int r = k * 32 + lane;
    if (r < nsel) {
      const int64_t e = e0 + list.slot[k];
      const int32_t s = __ldg(a.col + e);
      a.tgt[obase + r] = u;
      a.src[obase + r] = s;
      a.wgt[obase + r] = a.ew ? __ldg(a.ew + e) : 1.0f;
      if (a.tgt_front) a.tgt_front[obase + r] = (int32_t)i;
      atomicOr(bm + (s >> 5), 1u << (s & 31));
    }
  }
}

// Warp path of the threshold-collect select for one node (all 32 lanes).
// PACKED (d <= 2048): a candidate is the single 64-bit word key53 << 11 | slot,
// whose unsigned order is exactly the (key, slot) order, so collecting and
// ranking move and compare one word.  Otherwise keys and slots are kept apart.
template <bool PACKED>
__device__ __noinline__ void tau_select_node(const SelectArgs& a, uint64_t* wk, uint32_t* wsl,
                                                int64_t i, int32_t u, int64_t e0, int64_t d, int b,
                                                int64_t p0, int64_t obase, double expect) {
  const int lane = lane_id();
  const unsigned lt_mask = (1u << lane) - 1u;
  const int fan = a.fan;
  const uint64_t k0 = a.keys[2 * b], k1 = a.keys[2 * b + 1];
  const int64_t p1 = p0 + d;
  const int64_t blk0 = p0 >> 2, blk_last = (p1 - 1) >> 2;
  const int64_t want = d < fan ? d : fan;
  // threshold on key53: expect/d of the unit interval (any value keeping
  // >= want survivors gives the exact answer; it only sets the work)
  uint64_t tau = (double)d <= expect ? kKeyOne
                                     : (uint64_t)(expect * (double)kKeyOne * (double)__frcp_rn((float)d));
  int m = 0;
  for (;;) {
    m = 0;
    for (int64_t bb = blk0; bb <= blk_last; bb += 32) {
      const int64_t blk = bb + lane;
      const bool valid = blk <= blk_last;
      uint64_t w[4] = {~0ull, ~0ull, ~0ull, ~0ull};
      if (valid) philox4x64_10((uint64_t)blk + 1, k0, k1, w[0], w[1], w[2], w[3]);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t p = 4 * blk + q;
        const uint64_t key = w[q] >> 11;
        const bool take = valid && p >= p0 && p < p1 && key < tau;
        const unsigned bal = __ballot_sync(0xffffffffu, take);
        if (take) {
          const int pos = m + __popc(bal & lt_mask);
          if (pos < kTauCap) {
            if (PACKED) {
              wk[pos] = (key << 11) | (uint64_t)(p - p0);
            } else {
              wk[pos] = key;
              wsl[pos] = (uint32_t)(p - p0);
            }
          }
        }
        m += __popc(bal);
      }
    }
    if (m >= want || tau >= kKeyOne) break;
    tau = tau > kKeyOne / 4 ? kKeyOne : tau * 4;  // too few survivors: widen and redraw
  }
  __syncwarp();
  if (m > kTauCap) {  // pathological overflow: exact streaming fallback
    if (fan <= 32) stream_select_node<1>(a, i, u, e0, d, b, p0, obase);
    else if (fan <= 64) stream_select_node<2>(a, i, u, e0, d, b, p0, obase);
    else stream_select_node<4>(a, i, u, e0, d, b, p0, obase);
    return;
  }
  uint32_t* bm = a.bm_front + (int64_t)b * a.words;
  for (int c = lane; c < m; c += 32) {
    const uint64_t ck = wk[c];
    uint32_t cs;
    int rank = 0;
    if (PACKED) {
      cs = (uint32_t)(ck & 0x7FFu);
#pragma unroll 8
      for (int j = 0; j < m; ++j) rank += wk[j] < ck ? 1 : 0;
    } else {
      cs = wsl[c];
#pragma unroll 4
      for (int j = 0; j < m; ++j) rank += key_less(wk[j], wsl[j], ck, cs) ? 1 : 0;
    }
    if (rank < want) {
      const int64_t e = e0 + cs;
      const int32_t s = __ldg(a.col + e);
      const int64_t o = obase + rank;
      a.tgt[o] = u;
      a.src[o] = s;
      a.wgt[o] = a.ew ? __ldg(a.ew + e) : 1.0f;
      if (a.tgt_front) a.tgt_front[o] = (int32_t)i;
      atomicOr(bm + (s >> 5), 1u << (s & 31));
    }
  }
  __syncwarp();
}

// Lane path: nodes of degree <= kLaneDeg are sampled by ONE lane each, 32
// nodes per warp in lock step: the lane draws its node's <= 9 Philox blocks,
// keeps the packed candidates (key53 << 11 | slot) below the node's threshold
// in its own column of the warp's shared buffer, then picks the f smallest by
// repeated minimum search.  Per node this costs a few hundred lane
// instructions instead of a full warp iteration.
constexpr int kLaneDeg = 64;
constexpr int kLaneCap = 32;                       // survivors per lane
constexpr int kWarpBufWords = kLaneCap * 32;       // u64 words per warp (8 KB)

// returns false (nothing emitted) if more than kLaneCap candidates survive;
// the caller then redoes the node on the warp path
__device__ __noinline__ bool lane_select(const SelectArgs& a, uint64_t* colbuf, int64_t i, int32_t u,
                                         int64_t e0, int d, int b, int64_t p0, int64_t obase,
                                         double expect, int max_blocks) {
  const uint64_t k0 = a.keys[2 * b], k1 = a.keys[2 * b + 1];
  const int64_t blk0 = p0 >> 2;
  const int off0 = (int)(p0 & 3);
  const int nblk = (off0 + d + 3) >> 2;  // <= 17
  const int want = d < a.fan ? d : a.fan;
  uint64_t tau = (double)d <= expect ? kKeyOne
                                     : (uint64_t)(expect * (double)kKeyOne * (double)__frcp_rn((float)d));
  int m = 0;
  for (;;) {
    m = 0;
    for (int t = 0; t < max_blocks; ++t) {
      if (t < nblk) {
        uint64_t w[4];
        philox4x64_10((uint64_t)(blk0 + t) + 1, k0, k1, w[0], w[1], w[2], w[3]);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int j = 4 * t + q - off0;  // slot
          const uint64_t key = w[q] >> 11;
          if (j >= 0 && j < d && key < tau) {
            if (m < kLaneCap) colbuf[32 * m] = (key << 11) | (uint64_t)j;
            ++m;
          }
        }
      }
    }
    if (m > kLaneCap) return false;
    if (m >= want || tau >= kKeyOne) break;
    tau = tau > kKeyOne / 4 ? kKeyOne : tau * 4;
  }
  uint32_t* bm = a.bm_front + (int64_t)b * a.words;
  uint64_t prev = 0;
  for (int r = 0; r < want; ++r) {
    uint64_t best = ~0ull;
    for (int c = 0; c < m; ++c) {
      const uint64_t x = colbuf[32 * c];
      if ((r == 0 || x > prev) && x < best) best = x;
    }
    prev = best;
    const int64_t e = e0 + (int64_t)(best & 0x7FFu);
    const int32_t s = __ldg(a.col + e);
    const int64_t o = obase + r;
    a.tgt[o] = u;
    a.src[o] = s;
    a.wgt[o] = a.ew ? __ldg(a.ew + e) : 1.0f;
    if (a.tgt_front) a.tgt_front[o] = (int32_t)i;
    atomicOr(bm + (s >> 5), 1u << (s & 31));
  }
  return true;
}

// Each warp takes a tile of up to 32 consecutive frontier entries: the lanes
// load the nodes' parameters in parallel (one latency round for all of them),
// nodes of degree <= kLaneDeg are finished lane-parallel, the rest go through
// the warp path one by one with their parameters broadcast by shuffles.
__global__ void __launch_bounds__(256, 2) select_tau_kernel(SelectArgs a) {
  extern __shared__ __align__(16) uint64_t sbuf[];
  const int lane = lane_id(), wib = warp_id();
  uint64_t* wbuf = sbuf + (int64_t)wib * kWarpBufWords;  // lane path: [slot][lane]
  uint64_t* wk = wbuf;                                      // warp path aliases it
  uint32_t* wsl = reinterpret_cast<uint32_t*>(wbuf + kTauCap);
  const int64_t F = a.scal[kF];
  const int64_t ebase = a.scal[kHopEdgeBase];
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const double expect = a.fan + 3.0 * sqrt((double)a.fan) + 3.0;
  // tile of T consecutive nodes per warp: 32 for large frontiers, fewer when
  // the frontier is small so that every warp of the grid gets work
  const int64_t per_warp = ceil_div(F, nwarps);
  const int T = per_warp >= 32 ? 32 : (per_warp < 1 ? 1 : (int)per_warp);
  const bool lane_ok = a.fan <= kLaneCap;
  for (int64_t t0 = gw * T; t0 < F; t0 += nwarps * T) {
    const int64_t i = t0 + lane;
    int32_t u = 0;
    int64_t e0 = 0, d = 0, p0 = 0, obase = 0;
    int b = 0;
    if (lane < T && i < F) {
      u = a.front[i];
      b = a.fb[i];
      const int64_t sd = a.scan_deg[i], ss = a.scan_sel[i];
      e0 = __ldg(a.off + u);
      d = __ldg(a.off + u + 1) - e0;
      p0 = a.hop_pos[b] + sd;
      obase = ebase + ss;
    }
    // the lane path pays off only when enough lanes of the tile use it
    const bool eligible = lane_ok && d > 0 && d <= kLaneDeg;
    const unsigned elig_mask = __ballot_sync(0xffffffffu, eligible);  // every lane votes
    bool mine = eligible && __popc(elig_mask) >= 8;
    const int nblk = mine ? (int)(((p0 & 3) + d + 3) >> 2) : 0;
    const int max_blocks = __reduce_max_sync(0xffffffffu, (unsigned)nblk);
    if (max_blocks > 0) {
      if (mine) mine = lane_select(a, wbuf + lane, i, u, e0, (int)d, b, p0, obase, expect, max_blocks);
      __syncwarp();
    }
    unsigned big = __ballot_sync(0xffffffffu, d > 0 && !mine);
    while (big) {
      const int src = __ffs(big) - 1;
      big &= big - 1;
      const int64_t ii = t0 + src;
      const int32_t uu = __shfl_sync(0xffffffffu, u, src);
      const int64_t ee = __shfl_sync(0xffffffffu, e0, src);
      const int64_t dd = __shfl_sync(0xffffffffu, d, src);
      const int bb = __shfl_sync(0xffffffffu, b, src);
      const int64_t pp = __shfl_sync(0xffffffffu, p0, src);
      const int64_t oo = __shfl_sync(0xffffffffu, obase, src);
      if (dd <= 2048) tau_select_node<true>(a, wk, wsl, ii, uu, ee, dd, bb, pp, oo, expect);
      else tau_select_node<false>(a, wk, wsl, ii, uu, ee, dd, bb, pp, oo, expect);
    }
  }
}

constexpr int kSelectSmem = 8 * kWarpBufWords * 8;  // 64 KB per 256-thread CTA

// Balanced threshold-collect select (fanouts <= kTauMaxFan), the default.
// Each warp takes a tile of 32 consecutive frontier entries and spreads the
// Philox blocks of ALL its nodes evenly over its 32 lanes (lane g handles
// blocks g, g+32, ... of the tile's concatenated block list), so no lane sits
// idle while a neighbour draws a long node -- the per-node lane / warp paths
// of select_tau_kernel left ~45% of the lanes idle on power-law degrees.
// A drawn candidate survives if its key is below its node's threshold tau
// (the f smallest of d uniform keys lie below ~(f + 3 sqrt f + 3)/d); the
// survivor (key53 << 11 | slot) is appended to its node's segment of a
// per-warp shared buffer (shared-memory atomic on the node's count).  Then
// every survivor is ranked against its node's other survivors by counting,
// and rank < min(d, f) is emitted at output position obase + rank: ascending
// (key, slot) order, exactly np.lexsort's.  Nodes with d > kBalHub (slot does
// not fit 11 bits), whose survivors overflow their segment, or with fewer
// than min(d, f) survivors are redone exactly by the warp path
// (tau_select_node: widened threshold / streaming fallback).
constexpr int kBalHub = 2048;

inline int bal_cap(int fan) {
  const double ex = fan + 3.0 * std::sqrt((double)fan) + 3.0;
  return (int)std::ceil(ex + 3.5 * std::sqrt(ex) + 2.0);
}

__device__ __forceinline__ int bal_find(const int32_t* arr, int g) {
  // largest n in [0, 32) with arr[n] <= g (arr non-decreasing, arr[0] = 0)
  int n = 0;
#pragma unroll
  for (int step = 16; step >= 1; step >>= 1)
    if (arr[n + step < 32 ? n + step : 31] <= g && n + step < 32) n += step;
  return n;
}

// ------------------------------------------------------------ select v2 --
// Balanced select (tile of 32 frontier entries per warp,
// survivors below the node's threshold tau, the min(d, f) smallest (key,
// slot) pairs emitted in order), with the per-draw overhead cut down:
//  * each lane draws a CONTIGUOUS run of the tile's Philox blocks, so the
//    block -> node mapping is one search per lane and the node's parameters
//    stay in registers while the run stays inside the node;
//  * the threshold test runs on the raw Philox word (key < tau <=> w <=
//    (tau << 11) - 1) and a block's survivors take ONE shared atomic;
//  * survivors are 32-bit words ck << 11 | slot with ck = key >> sh, sh
//    chosen per node so that ck < 2^21: the selection compares 32-bit words
//    and the buffers are half the size (more resident warps).  Two survivors
//    of a node with equal ck but different keys could be ordered by slot
//    instead of key; the selection checks the selected words and the first
//    unselected one for equal ck (probability ~1e-5 per node) and sends such
//    a node to the exact warp path.
constexpr int kSel2Warps = 4;

struct Sel2Tab {
  int64_t p0[32], e0[32], obase[32];
  uint64_t twi[32], k0[32], k1[32];
  int32_t d[32], dt[32], seg[32], cnt[32], bs[33], u[32], b[32], sh[32];
};

inline int sel2_buf_words(int fan) {  // u32 words: survivors (32 caps) | queue (32 * fan); >= tau-path scratch
  const int surv = 32 * bal_cap(fan);
  return std::max(surv, (kTauCap * 12 + 3) / 4) + 32 * fan;
}
inline int sel2_smem(int fan) {
  return kSel2Warps * (((sel2_buf_words(fan) * 4 + 15) / 16) * 16 + (int)sizeof(Sel2Tab));
}

__global__ void __launch_bounds__(kSel2Warps * 32, 8) select_bal2_kernel(const __grid_constant__ SelectArgs a,
                                                                        int capn, int buf_words) {
  extern __shared__ __align__(16) uint64_t sbuf2[];
  const int lane = lane_id(), wib = warp_id();
  const int wbytes = ((buf_words * 4 + 15) / 16) * 16;
  char* wbase = reinterpret_cast<char*>(sbuf2) + (int64_t)wib * (wbytes + sizeof(Sel2Tab));
  uint32_t* sv = reinterpret_cast<uint32_t*>(wbase);
  Sel2Tab& T = *reinterpret_cast<Sel2Tab*>(wbase + wbytes);
  const int64_t F = a.scal[kF];
  const int64_t ebase = a.scal[kHopEdgeBase];
  const int fan = a.fan;
  const double expect = fan + 3.0 * sqrt((double)fan) + 3.0;
  uint32_t* bm_base = a.bm_front;
  const int64_t ntiles = ceil_div(F, 32);
  const int surv_cap = 32 * capn;  // survivor words; the emission queue follows
  // first tile = the warp's global index (no atomic: with small frontiers
  // thousands of warps would otherwise serialise on the counter just to find
  // no work), later tiles from the dynamic counter past the static ones
  const int64_t nwarps = (int64_t)gridDim.x * kSel2Warps;
  unsigned long long tix = (unsigned long long)(blockIdx.x * (int64_t)kSel2Warps + wib);
  for (;;) {
    if ((int64_t)tix >= ntiles) break;
    const int64_t t0 = (int64_t)tix * 32;
    int TB;
    {  // tile setup: node parameters -> the warp's table (registers freed for the draw loop)
      const int64_t i = t0 + lane;
      int32_t u = 0, b = 0;
      int64_t e0 = 0, d = 0, p0 = 0, obase = 0;
      if (i < F) {
        u = a.front[i];
        b = a.fb[i];
        e0 = __ldg(a.off + u);
        d = __ldg(a.off + u + 1) - e0;
        p0 = a.hop_pos[b] + a.scan_deg[i];
        obase = ebase + a.scan_sel[i];
      }
      const bool elig = d > 0 && d <= kBalHub;
      const int cap = elig ? (int)(d < capn ? d : capn) : 0;
      const int seg = warp_incl_scan(cap) - cap;
      const int nblk = elig ? (int)(((p0 + d - 1) >> 2) - (p0 >> 2) + 1) : 0;
      const int bsum = warp_incl_scan(nblk);
      TB = __shfl_sync(0xffffffffu, bsum, 31);
      const uint64_t tau = (double)d <= expect ? kKeyOne
                                               : (uint64_t)(expect * (double)kKeyOne * (double)__frcp_rn((float)d));
      const int sh = max(0, (64 - __clzll((long long)(tau - 1))) - 21);
      T.p0[lane] = p0; T.e0[lane] = e0; T.obase[lane] = obase;
      T.twi[lane] = (tau << 11) - 1ull;  // tau = 2^53 wraps to all-ones: every draw survives
      T.k0[lane] = __ldg(a.keys + 2 * b); T.k1[lane] = __ldg(a.keys + 2 * b + 1);
      T.d[lane] = (int32_t)(elig ? d : 0); T.dt[lane] = (int32_t)d; T.seg[lane] = seg; T.cnt[lane] = 0;
      T.bs[lane] = bsum - nblk; T.u[lane] = u; T.b[lane] = b; T.sh[lane] = sh;
      if (lane == 31) T.bs[32] = TB;
    }
    __syncwarp();
    // ---- Philox over a contiguous run of the tile's blocks per lane
    {
      const int per = TB >> 5, rem = TB & 31;
      int g = lane * per + min(lane, rem);
      const int gend = g + per + (lane < rem ? 1 : 0);
      if (g < gend) {
        int n = bal_find(T.bs, g);
        int nb_end = T.bs[n + 1];
        int64_t kb = (T.p0[n] >> 2) - T.bs[n];
        int32_t s_off = (int32_t)(4 * ((T.p0[n] >> 2) - T.bs[n]) - T.p0[n]);  // slot of word 0 of block g: 4g + s_off
        // survivor word = (key >> (sh + 11)) << 11 | slot: one funnel shift of
        // the raw word by sh and a mask (no IMAD on the Philox-bound pipe);
        // the node's segment as a 32-bit shared address
        const uint32_t sv_u = (uint32_t)__cvta_generic_to_shared(sv);
        int nd = T.d[n], nsh = T.sh[n], ncap = nd < capn ? nd : capn;
        uint32_t sbase = sv_u + 4u * (uint32_t)T.seg[n];
        uint64_t twi = T.twi[n], k0 = T.k0[n], k1 = T.k1[n];
        for (; g < gend; ++g) {
          if (g >= nb_end) {  // next node with blocks (zero-block nodes share a start)
            do { ++n; nb_end = T.bs[n + 1]; } while (g >= nb_end);
            kb = (T.p0[n] >> 2) - T.bs[n];
            s_off = (int32_t)(4 * kb - T.p0[n]);
            nd = T.d[n]; nsh = T.sh[n]; ncap = nd < capn ? nd : capn;
            sbase = sv_u + 4u * (uint32_t)T.seg[n];
            twi = T.twi[n]; k0 = T.k0[n]; k1 = T.k1[n];
          }
          uint64_t w[4];
          philox4x64_10((uint64_t)(kb + g) + 1, k0, k1, w[0], w[1], w[2], w[3]);
          const int s0 = 4 * g + s_off;
          bool tk[4];
          int nt = 0;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            tk[q] = (unsigned)(s0 + q) < (unsigned)nd && w[q] <= twi;
            nt += tk[q] ? 1 : 0;
          }
          if (nt) {
            int c = atomicAdd(&T.cnt[n], nt);
#pragma unroll
            for (int q = 0; q < 4; ++q) {  // predicated stores, no per-survivor branches
              const uint32_t word = ((uint32_t)(w[q] >> nsh) & 0xFFFFF800u) | (uint32_t)(s0 + q);
              if (tk[q] && c < ncap)
                asm volatile("st.shared.u32 [%0], %1;" ::"r"(sbase + 4u * (uint32_t)c), "r"(word) : "memory");
              c += tk[q] ? 1 : 0;
            }
          }
        }
      }
    }
    __syncwarp();
    const int64_t i = t0 + lane;
    const int64_t d = T.dt[lane];
    const bool elig = d > 0 && d <= kBalHub;
    const int cap = elig ? (int)(d < capn ? d : capn) : 0;
    const int seg = T.seg[lane];
    const int want = (int)(d < fan ? d : fan);
    const int cnt = T.cnt[lane];
    const bool hub = d > kBalHub && a.hub_list;
    if (hub) {
      if (d > kGiantHub) a.hub_list[atomicAdd(a.hub_big_cnt, 1ull)] = (int32_t)i;
      else a.hub_list[a.hub_cap - 1 - (int64_t)atomicAdd(a.hub_cnt, 1ull)] = (int32_t)i;
    }
    bool fb = d > 0 && !hub && (!elig || cnt > cap || cnt < want);
    uint32_t* q = sv + surv_cap;  // emission queue after the survivors
    const int nsel = (!fb && !hub && d > 0) ? want : 0;
    const int qbase = warp_incl_scan(nsel) - nsel;
    const int nq = __shfl_sync(0xffffffffu, qbase + nsel, 31);
    if (nsel) {
      // ---- selection, lane = node: want passes of a minimum search over the
      // node's 32-bit survivor words, then the tie check
      const uint32_t* sg = sv + seg;
      uint32_t prev = 0;
      bool tie = false;
      for (int r = 0; r < nsel; ++r) {
        uint32_t best = 0xffffffffu;
        for (int jj = 0; jj < cnt; ++jj) {
          const uint32_t x = sg[jj];
          if ((r == 0 || x > prev) && x < best) best = x;
        }
        tie |= r > 0 && (best >> 11) == (prev >> 11);
        prev = best;
        q[qbase + r] = ((uint32_t)lane << 24) | ((uint32_t)r << 11) | (best & 0x7FFu);
      }
      if (cnt > nsel) {  // first unselected survivor vs the last selected one
        uint32_t nxt = 0xffffffffu;
        for (int jj = 0; jj < cnt; ++jj) {
          const uint32_t x = sg[jj];
          if (x > prev && x < nxt) nxt = x;
        }
        tie |= (nxt >> 11) == (prev >> 11);
      }
      if (tie) {  // equal compressed keys: redo this node exactly
        fb = true;
        for (int r = 0; r < nsel; ++r) q[qbase + r] = 0xffffffffu;
      }
    }
    __syncwarp();
    for (int k0 = 0; k0 < nq; k0 += 128) {
      uint32_t it[4];
      int32_t sidx[4];
      float wv[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {  // four independent gathers in flight per lane
        const int k = k0 + 32 * r + lane;
        it[r] = k < nq ? q[k] : 0xffffffffu;
        if (it[r] != 0xffffffffu) {
          const int n = (int)(it[r] >> 24);
          const int64_t ee = T.e0[n] + (int64_t)(it[r] & 0x7FFu);
          sidx[r] = __ldg(a.col + ee);
          wv[r] = a.ew ? __ldg(a.ew + ee) : 1.0f;
        }
      }
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        if (it[r] == 0xffffffffu) continue;
        const int n = (int)(it[r] >> 24);
        const int64_t o = T.obase[n] + (int64_t)((it[r] >> 11) & 0x1FFFu);
        a.tgt[o] = T.u[n];
        a.src[o] = sidx[r];
        a.wgt[o] = wv[r];
        if (a.tgt_front) a.tgt_front[o] = (int32_t)(t0 + n);
        atomicOr(bm_base + (int64_t)T.b[n] * a.words + (sidx[r] >> 5), 1u << (sidx[r] & 31));
      }
    }
    __syncwarp();
    // ---- exact warp path for overflow / too few survivors / compressed-key ties
    unsigned big = __ballot_sync(0xffffffffu, fb);
    uint64_t* wk = reinterpret_cast<uint64_t*>(sv);
    uint32_t* wsl = reinterpret_cast<uint32_t*>(wk + kTauCap);
    while (big) {
      const int src = __ffs(big) - 1;
      big &= big - 1;
      const int64_t ii = t0 + src;
      const int32_t uu = T.u[src];
      const int64_t ee = T.e0[src];
      const int64_t dd = T.dt[src];
      const int bb = T.b[src];
      const int64_t pp = T.p0[src];
      const int64_t oo = T.obase[src];
      if (dd <= 2048) tau_select_node<true>(a, wk, wsl, ii, uu, ee, dd, bb, pp, oo, expect);
      else tau_select_node<false>(a, wk, wsl, ii, uu, ee, dd, bb, pp, oo, expect);
    }
    __syncwarp();
    if (nwarps >= ntiles) break;  // every tile was handed out statically
    unsigned long long nx = 0;
    if (lane == 0) nx = atomicAdd(a.tile_ctr, 1ull);
    tix = (unsigned long long)nwarps + __shfl_sync(0xffffffffu, nx, 0);
  }
}

// Hub nodes (d > kBalHub) of a hop, one CTA each (select_bal2_kernel queues
// them): all 512 threads draw the hub's Philox blocks, survivors below the
// threshold go to shared memory, and the want smallest (key, slot) pairs are
// ranked by counting -- a 19K-degree hub takes one CTA a few microseconds
// instead of one warp ~100 us at the end of the select launch.  Overflow or
// too few survivors: the exact warp path (tau_select_node) of warp 0.
constexpr int kHubThreads = 256;
constexpr int kHubCap = 2048;

__global__ void __launch_bounds__(kHubThreads, 3) select_hub_kernel(const __grid_constant__ SelectArgs a) {
  __shared__ uint64_t skey[kHubCap];
  __shared__ uint32_t sslot[kHubCap];
  __shared__ int scnt;
  const int tid = threadIdx.x;
  const int64_t nbig = (int64_t)*a.hub_big_cnt;
  const int64_t nh = nbig + (int64_t)*a.hub_cnt;
  const int64_t ebase = a.scal[kHopEdgeBase];
  const int fan = a.fan;
  // hubs take a wider threshold: survivors ~ f + 6 sqrt(f) + 12 cost a CTA
  // nothing extra to rank, while too few send the hub to ONE warp's exact
  // path (4.8K Philox blocks for a 19K-degree hub): 98 -> 51 us / window
  const double expect = fan + 6.0 * sqrt((double)fan) + 12.0;
  for (int64_t h = blockIdx.x; h < nh; h += gridDim.x) {
    const int64_t i = h < nbig ? a.hub_list[h] : a.hub_list[a.hub_cap - 1 - (h - nbig)];
    const int32_t u = a.front[i];
    const int b = a.fb[i];
    const int64_t e0 = __ldg(a.off + u);
    const int64_t d = __ldg(a.off + u + 1) - e0;
    const int64_t p0 = a.hop_pos[b] + a.scan_deg[i];
    const int64_t obase = ebase + a.scan_sel[i];
    const uint64_t k0 = a.keys[2 * b], k1 = a.keys[2 * b + 1];
    const int want = (int)(d < fan ? d : fan);
    const uint64_t tau = (uint64_t)(expect * (double)kKeyOne * (double)__frcp_rn((float)d));
    if (tid == 0) scnt = 0;
    __syncthreads();
    const int64_t blk0 = p0 >> 2, blk_last = (p0 + d - 1) >> 2;
    for (int64_t blk = blk0 + tid; blk <= blk_last; blk += kHubThreads) {
      uint64_t w[4];
      philox4x64_10((uint64_t)blk + 1, k0, k1, w[0], w[1], w[2], w[3]);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t slot = 4 * blk + q - p0;
        const uint64_t key = w[q] >> 11;
        if (slot >= 0 && slot < d && key < tau) {
          const int c = atomicAdd(&scnt, 1);
          if (c < kHubCap) { skey[c] = key; sslot[c] = (uint32_t)slot; }
        }
      }
    }
    __syncthreads();
    const int cnt = scnt;
    if (cnt >= want && cnt <= kHubCap) {
      uint32_t* bm = a.bm_front + (int64_t)b * a.words;
      for (int c = tid; c < cnt; c += kHubThreads) {
        const uint64_t ck = skey[c];
        const uint32_t cs = sslot[c];
        int rank = 0;
        for (int j = 0; j < cnt; ++j) rank += key_less(skey[j], sslot[j], ck, cs) ? 1 : 0;
        if (rank < want) {
          const int64_t e = e0 + cs;
          const int32_t sidx = __ldg(a.col + e);
          const int64_t o = obase + rank;
          a.tgt[o] = u;
          a.src[o] = sidx;
          a.wgt[o] = a.ew ? __ldg(a.ew + e) : 1.0f;
          if (a.tgt_front) a.tgt_front[o] = (int32_t)i;
          atomicOr(bm + (sidx >> 5), 1u << (sidx & 31));
        }
      }
    } else if (tid < 32) {  // exact warp path (widened threshold / streaming fallback)
      tau_select_node<false>(a, skey, sslot, i, u, e0, d, b, p0, obase, expect);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------ translate ----
__device__ __forceinline__ int32_t bm_rank(const uint2* __restrict__ wrank, int64_t base_word, int32_t g) {
  const uint2 pw = __ldg(wrank + base_word + (g >> 5));  // {prefix, word}: one 8-byte load, one sector
  return (int32_t)(pw.x + __popc(pw.y & ((1u << (g & 31)) - 1u)));
}

// posmap[row(frontier[j])] = j for every entry j of one hop's frontier list
__global__ void posmap_kernel(const int32_t* __restrict__ front, const int64_t* __restrict__ fo,
                              int32_t nb, const uint2* __restrict__ wrank, int64_t words,
                              int32_t* __restrict__ posmap) {
  // batch = blockIdx.y: the segment is known, no per-entry search
  const int b = blockIdx.y;
  const int64_t j1 = fo[b + 1];
  for (int64_t j = fo[b] + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < j1;
       j += (int64_t)gridDim.x * blockDim.x)
    posmap[bm_rank(wrank, (int64_t)b * words, front[j])] = (int32_t)j;
}

// window rows of hop h's edges (+ frontier index of the source in hop h+1's
// list through posmap, or the source row itself for the last hop)
__global__ void translate_kernel(const int32_t* __restrict__ tgt, const int32_t* __restrict__ src,
                                 const int64_t* __restrict__ eoff, int32_t nb,
                                 const uint2* __restrict__ wrank, int64_t words,
                                 const int32_t* __restrict__ posmap, int32_t* __restrict__ lt,
                                 int32_t* __restrict__ ls, int32_t* __restrict__ sf) {
  // batch = blockIdx.y (edges are hop-major / batch-minor): no per-edge search
  const int b = blockIdx.y;
  const int64_t e1 = eoff[b + 1], bw = (int64_t)b * words;
  for (int64_t e = eoff[b] + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < e1;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t rs = bm_rank(wrank, bw, src[e]);
    if (lt) lt[e] = bm_rank(wrank, bw, tgt[e]);
    if (ls) ls[e] = rs;
    if (sf) sf[e] = posmap ? posmap[rs] : rs;
  }
}

__global__ void translate_seeds_kernel(const int32_t* __restrict__ seeds,
                                       const int64_t* __restrict__ seed_off, int32_t nb,
                                       int64_t total, const uint2* __restrict__ wrank, int64_t words,
                                       const int32_t* __restrict__ posmap,
                                       int32_t* __restrict__ rows, int32_t* __restrict__ fidx) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int b = find_segment(seed_off, nb, i);
    const int32_t r = bm_rank(wrank, (int64_t)b * words, seeds[i]);
    if (rows) rows[i] = r;
    if (fidx) fidx[i] = posmap[r];
  }
}

// ----------------------------------------------------------- random walk --
// sampler.sample_random_walk (sampler.py:142-186): one uniform walk of
// `length` steps per seed, one Philox stream for the batch.  At each step the
// walkers still alive whose node has out-degree > 0, in seed order, consume
// consecutive draws u (random() doubles = word >> 11 scaled by 2^-53) and step
// to col[off[v] + floor(u * deg)] (an IEEE double multiply then truncation,
// exactly numpy's (rng.random(n) * deg).astype(int64)); sinks stop their walk
// without a draw.  Edges are emitted step-major, seed order within a step.
// One CTA per batch: the per-step ranks of the stepping walkers come from a
// block-wide scan, so the whole walk is a single launch with no host sync;
// every visited node is marked in a bitmap whose compaction is the sorted
// unique_nodes.
constexpr int kWalkThreads = 1024;

__global__ void __launch_bounds__(kWalkThreads) walk_kernel(const int64_t* __restrict__ off,
                                                            const int32_t* __restrict__ col,
                                                            const float* __restrict__ ew,
                                                            const int32_t* __restrict__ seeds, int64_t n,
                                                            int length, uint64_t k0, uint64_t k1,
                                                            int64_t num_nodes, int32_t* __restrict__ cur,
                                                            int32_t* __restrict__ tgt, int32_t* __restrict__ src,
                                                            float* __restrict__ wgt,
                                                            int64_t* __restrict__ step_off,
                                                            uint32_t* __restrict__ bm, int64_t* status) {
  __shared__ int64_t sm[33];
  const int tid = threadIdx.x;
  for (int64_t i = tid; i < n; i += blockDim.x) {
    const int32_t sd = seeds[i];
    if (sd < 0 || sd >= num_nodes) { set_status(status, FGL_E_INVALID); cur[i] = -1; continue; }
    cur[i] = sd;
    atomicOr(bm + (sd >> 5), 1u << (sd & 31));
  }
  __syncthreads();
  if (tid == 0) step_off[0] = 0;
  int64_t pos = 0;  // Philox stream position = edges emitted so far
  for (int step = 0; step < length; ++step) {
    int64_t running = 0;
    for (int64_t c0 = 0; c0 < n; c0 += blockDim.x) {
      const int64_t i = c0 + tid;
      const int32_t u = i < n ? cur[i] : -1;
      int64_t e0 = 0, d = 0;
      if (u >= 0) {
        e0 = __ldg(off + u);
        d = __ldg(off + u + 1) - e0;
        if (d == 0) cur[i] = -1;  // sink: the walk stops, no draw
      }
      const int64_t flag = (u >= 0 && d > 0) ? 1 : 0;
      int64_t tot;
      const int64_t rank = running + block_excl_scan<int64_t>(flag, sm, &tot);
      if (flag) {
        const int64_t p = pos + rank;
        uint64_t w[4];
        philox4x64_10((uint64_t)(p >> 2) + 1, k0, k1, w[0], w[1], w[2], w[3]);
        const uint64_t word = w[p & 3];
        const double r = (double)(word >> 11) * 0x1.0p-53;
        const int64_t pick = (int64_t)__dmul_rn(r, (double)d);
        const int64_t e = e0 + pick;
        const int32_t nxt = __ldg(col + e);
        tgt[p] = u;
        src[p] = nxt;
        wgt[p] = ew ? __ldg(ew + e) : 1.0f;
        cur[i] = nxt;
        atomicOr(bm + (nxt >> 5), 1u << (nxt & 31));
      }
      running += tot;
    }
    pos += running;
    if (tid == 0) step_off[step + 1] = pos;
    __syncthreads();
  }
}

int select_grid(int K) {
  static int cache[9] = {0};
  if (cache[K]) return cache[K];
  int per_sm = 0;
  cudaError_t e = cudaSuccess;
  switch (K) {
    case 1: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, select_kernel<1>, 256, 0); break;
    case 2: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, select_kernel<2>, 256, 0); break;
    case 4: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, select_kernel<4>, 256, 0); break;
    case 0:
      e = cudaFuncSetAttribute(select_tau_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSelectSmem);
      if (e == cudaSuccess)
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, select_tau_kernel, 256, kSelectSmem);
      break;
    default: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, select_kernel<8>, 256, 0); break;
  }
  if (e != cudaSuccess || per_sm < 1) per_sm = 2;
  cache[K] = per_sm * kNumSMs;
  return cache[K];
}

}  // namespace
}  // namespace fgl

using namespace fgl;

extern "C" {

int fgl_sample_bounds(int64_t num_nodes, const int64_t* batch_sizes, int32_t nb,
                      const int32_t* fanouts, int32_t H, int64_t* out) {
  if (num_nodes < 1 || nb < 1 || H < 1 || H > FGL_MAX_HOPS || !batch_sizes || !fanouts || !out) {
    set_error("fgl_sample_bounds: bad arguments");
    return FGL_E_INVALID;
  }
  int64_t edges = 0, uniq = 0;
  std::vector<int64_t> hop_front(H + 1, 0);
  for (int b = 0; b < nb; ++b) {
    int64_t f = std::min<int64_t>(batch_sizes[b], num_nodes);
    int64_t u = batch_sizes[b];
    hop_front[0] += f;
    for (int h = 0; h < H; ++h) {
      const int64_t e = f * (int64_t)fanouts[h];
      edges += e;
      u += e;
      f = std::min<int64_t>(num_nodes, e);
      hop_front[h + 1] += f;
    }
    uniq += std::min<int64_t>(num_nodes, u);
  }
  const int64_t fcap = *std::max_element(hop_front.begin(), hop_front.end());
  out[0] = std::max<int64_t>(edges, 1);
  out[1] = std::max<int64_t>(fcap, 1);
  out[2] = std::max<int64_t>(uniq, 1);
  out[3] = ws_layout(num_nodes, nb, out[1], out[2]).bytes;
  out[4] = FGL_CNT_LEN(H, nb);
  return FGL_OK;
}

int fgl_sample_ws_bitmaps(int64_t num_nodes, int32_t nb, int64_t frontier_stride,
                          int64_t unique_cap, int64_t* out) {
  if (num_nodes < 1 || nb < 1 || !out) {
    set_error("fgl_sample_ws_bitmaps: bad arguments");
    return FGL_E_INVALID;
  }
  const WsLayout L = ws_layout(num_nodes, nb, frontier_stride, unique_cap);
  out[0] = L.off_all_bm;
  out[1] = L.off_wprefix;
  out[2] = L.words;
  return FGL_OK;
}

int fgl_sample_window(const fgl_graph* g, const int32_t* seeds, const int64_t* seed_off,
                      int64_t total_seeds, int32_t nb, const uint64_t* keys,
                      const int32_t* fanouts, int32_t H, const fgl_sample_out* o, void* ws,
                      int64_t ws_bytes, void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (!g || !seeds || !seed_off || !keys || !fanouts || !o || !o->tgt || !o->src || !o->wgt ||
      !o->unique_nodes || !o->frontier || !o->counts || !ws || nb < 1 || H < 1 ||
      H > FGL_MAX_HOPS || total_seeds < 1 || o->frontier_stride < 1) {
    set_error("fgl_sample_window: bad arguments");
    return FGL_E_INVALID;
  }
  if (g->num_nodes < 1 || g->num_nodes >= (1ll << 31) || (int64_t)nb * g->num_nodes >= (1ll << 31)) {
    set_error("fgl_sample_window: num_nodes * num_batches must stay below 2^31");
    return FGL_E_UNSUPPORTED;
  }
  for (int h = 0; h < H; ++h) {
    if (fanouts[h] < 1) { set_error("every fanout must be >= 1"); return FGL_E_INVALID; }
    if (fanouts[h] > kMaxFanout) {
      set_error("fanout %d exceeds the supported maximum %d", fanouts[h], kMaxFanout);
      return FGL_E_UNSUPPORTED;
    }
  }
  const WsLayout Lw = ws_layout(g->num_nodes, nb, o->frontier_stride, o->unique_cap);
  if (Lw.bytes > ws_bytes) {
    set_error("sample workspace too small (%lld < %lld bytes)", (long long)ws_bytes,
              (long long)Lw.bytes);
    return FGL_E_CAPACITY;
  }
  SampleWs w = carve(ws, Lw);
  const int64_t words = Lw.words;
  const int64_t nwords = words * nb;
  const int64_t fcap = o->frontier_stride;
  const int G = kSampCTAs;
  const int Gb = bm_grid(nwords);
  int64_t* counts = o->counts;
  int64_t* status = counts + FGL_CNT_STATUS(H, nb);
  int64_t* uniq_off = counts + FGL_CNT_UNIQ(H, nb);
  auto fr_off = [&](int h) { return counts + FGL_CNT_FRONT(H, nb) + (int64_t)h * (nb + 1); };

  FGL_CUDA(cudaMemsetAsync(counts, 0, sizeof(int64_t) * FGL_CNT_LEN(H, nb), stream));
  FGL_CUDA(cudaMemsetAsync(w.bm_front, 0, 4 * nwords, stream));
  FGL_CUDA(cudaMemsetAsync(w.bm_all, 0, 4 * nwords, stream));
  FGL_CUDA(cudaMemsetAsync(w.pos, 0, 8 * nb, stream));
  FGL_CUDA(cudaMemsetAsync(w.scal, 0, 8 * 8, stream));

  // frontier 0 = sorted unique seeds per batch
  FGL_COUNT_LAUNCH(), mark_seeds_kernel<<<(int)std::min<int64_t>(ceil_div(total_seeds, 256), 4 * G), 256, 0, stream>>>(
      seeds, seed_off, nb, total_seeds, g->num_nodes, words, w.bm_front, status);
  FGL_LAUNCH_CHECK("mark_seeds_kernel");
  // compaction of `front` into hop h's frontier list (h == H: no list, only OR into `all`)
  auto compact_front = [&](int h) -> int {
    const bool write = h < H;
    FGL_COUNT_LAUNCH(), bm_count_kernel<<<Gb, kScanThreads, 0, stream>>>(w.bm_front, nwords, w.part);
    FGL_COUNT_LAUNCH(), scan_partials_kernel<<<1, 1024, 0, stream>>>(w.part, Gb, w.scal + kF, write ? fr_off(h) + nb : nullptr);
    launch_bm_compact(Gb, stream, w.bm_front, nwords, words, w.part, write ? o->frontier + h * fcap : nullptr,
                      write ? w.fb : nullptr, write ? fr_off(h) : nullptr, nullptr, w.bm_all, 1, fcap, status);
    FGL_LAUNCH_CHECK("frontier compaction");
    return FGL_OK;
  };
  int rc = compact_front(0);
  if (rc) return rc;

  // upper bound of each hop's frontier (all batches): sizes the degree-scan grid
  int64_t f_ub = std::min<int64_t>(total_seeds, fcap);
  for (int h = 0; h < H; ++h) {
    const int fan = fanouts[h];
    const int32_t* front = o->frontier + h * fcap;
    {  // draw / output offsets of the hop's frontier: one single-pass scan
      const int64_t tiles_max = fcap / kDegTile + 1;
      const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(tiles_max, ceil_div(f_ub, kDegTile)));
      // counter and status words are adjacent in the workspace: one memset
      const int64_t tiles = std::min<int64_t>(tiles_max + 1, ceil_div(f_ub, kDegTile) + 1);
      FGL_CUDA(cudaMemsetAsync(w.lbflag, 0, reinterpret_cast<char*>(w.lb + 2 * tiles) -
                                                reinterpret_cast<char*>(w.lbflag), stream));
      FGL_COUNT_LAUNCH(), deg_scan_kernel<<<(int)grid, kScanThreads, 0, stream>>>(
          g->row_offsets, front, w.scal, fan, w.scan_deg, w.scan_sel, w.lb, w.lb + tiles, w.lbflag);
    }
    FGL_COUNT_LAUNCH(), hop_book_kernel<<<1, 64, 0, stream>>>(w, fr_off(h), nb, h, counts, H, o->edge_cap);
    FGL_LAUNCH_CHECK("degree scan");
    SelectArgs a{g->row_offsets, g->col_indices, g->edge_weights, front, w.fb,
                 w.scan_deg, w.scan_sel, fr_off(h), w.hop_pos, keys, w.scal,
                 w.bm_front, words, o->tgt, o->src, o->wgt, o->tgt_front, fan,
                 reinterpret_cast<unsigned long long*>(w.scal + kTileCtr),
                 reinterpret_cast<unsigned long long*>(w.scal + kHubCnt), w.hub_list};
    a.hub_big_cnt = reinterpret_cast<unsigned long long*>(w.scal + kHubBig);
    a.hub_cap = fcap;
    // the last hop's sources need no frontier list: the selection ORs them
    // straight into the `all` bitmaps (no count / compact / clear pass over
    // the window bitmaps: ~150 us per window at the papers100M shape)
    const bool last_direct = h + 1 == H;
    if (last_direct) a.bm_front = w.bm_all;
    // FGL_SELECT=stream forces the streaming top-list kernel (A/B parity tests)
    static const bool force_stream = [] {
      const char* v = getenv("FGL_SELECT");
      return v && v[0] == 's';
    }();
    static const bool force_tau = [] {
      const char* v = getenv("FGL_SELECT");
      return v && v[0] == 't';
    }();
    if (fan <= kTauMaxFan && sel2_smem(fan) <= 200 * 1024 && !force_stream && !force_tau) {
      const ProfMark pm = prof_begin(stream);  // bench.py: the two launches are the hop's selection
      const int s2 = sel2_smem(fan);
      // grid per fanout: the survivor buffers (and so the CTAs per SM) depend on it
      static int s2_attr = 0;
      static int s2_grid_of[kTauMaxFan + 1] = {0};
      if (s2 > s2_attr) {
        FGL_CUDA(cudaFuncSetAttribute(select_bal2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, s2));
        s2_attr = s2;
      }
      if (!s2_grid_of[fan]) {
        int per_sm = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, select_bal2_kernel, kSel2Warps * 32, s2) !=
                cudaSuccess || per_sm < 1)
          per_sm = 2;
        static const int sel_sms = env_int("FGL_SEL_SMS", kNumSMs);
        s2_grid_of[fan] = per_sm * std::max(1, std::min(sel_sms, kNumSMs));
      }
      FGL_COUNT_LAUNCH(), select_bal2_kernel<<<s2_grid_of[fan], kSel2Warps * 32, s2, stream>>>(
          a, bal_cap(fan), sel2_buf_words(fan));
      static const int hub_ctas = env_int("FGL_HUB_CTAS", 6 * kNumSMs);
      FGL_COUNT_LAUNCH(), select_hub_kernel<<<std::max(1, hub_ctas), kHubThreads, 0, stream>>>(a);
      prof_end(pm, kProfSelect, h);
    } else if (fan <= kTauMaxFan && !force_stream)
      FGL_COUNT_LAUNCH(), select_tau_kernel<<<select_grid(0), 256, kSelectSmem, stream>>>(a);
    else if (fan <= 32) FGL_COUNT_LAUNCH(), select_kernel<1><<<select_grid(1), 256, 0, stream>>>(a);
    else if (fan <= 64) FGL_COUNT_LAUNCH(), select_kernel<2><<<select_grid(2), 256, 0, stream>>>(a);
    else if (fan <= 128) FGL_COUNT_LAUNCH(), select_kernel<4><<<select_grid(4), 256, 0, stream>>>(a);
    else FGL_COUNT_LAUNCH(), select_kernel<8><<<select_grid(8), 256, 0, stream>>>(a);
    FGL_LAUNCH_CHECK("select_kernel");
    f_ub = std::min<int64_t>(std::min<int64_t>(f_ub * fan, (int64_t)nb * g->num_nodes), fcap);
    if (!last_direct) {
      rc = compact_front(h + 1);
      if (rc) return rc;
    }
  }

  // unique nodes = compaction of the `all` bitmaps; keeps per-word prefixes for ranks
  FGL_COUNT_LAUNCH(), bm_count_kernel<<<Gb, kScanThreads, 0, stream>>>(w.bm_all, nwords, w.part);
  FGL_COUNT_LAUNCH(), scan_partials_kernel<<<1, 1024, 0, stream>>>(w.part, Gb, w.scal + kUniqTot, uniq_off + nb);
  launch_bm_compact(Gb, stream, w.bm_all, nwords, words, w.part, o->unique_nodes, nullptr, uniq_off, w.wprefix,
                    nullptr, 0, o->unique_cap, status, w.wrank);
  FGL_LAUNCH_CHECK("unique compaction");

  // translation: window rows, and frontier indices through per-hop position maps
  const bool want_rows = o->tgt_row || o->src_row || o->src_front;
  const int TG = 4 * kPersistentCTAs;
  const int TGb = std::max(1, TG / nb);  // CTAs per batch of the 2-D (x, batch) translation grids
  for (int h = 0; h <= H; ++h) {
    const bool has_list = h < H && (o->src_front || (h == 0 && o->seed_front));
    if (has_list) {
      FGL_COUNT_LAUNCH(), posmap_kernel<<<dim3(TGb, nb), 256, 0, stream>>>(o->frontier + h * fcap, fr_off(h), nb,
                                                                       w.wrank, words, w.posmap);
    }
    if (h == 0 && (o->seed_rows || o->seed_front)) {
      FGL_COUNT_LAUNCH(), translate_seeds_kernel<<<(int)std::min<int64_t>(ceil_div(total_seeds, 256), TG), 256, 0,
                               stream>>>(seeds, seed_off, nb, total_seeds, w.wrank,
                                         words, w.posmap, o->seed_rows, o->seed_front);
    }
    if (h >= 1 && want_rows) {  // hop h-1 sources live in hop h's frontier
      FGL_COUNT_LAUNCH(), translate_kernel<<<dim3(TGb, nb), 256, 0, stream>>>(
          o->tgt, o->src, counts + (h - 1) * nb, nb, w.wrank, words, h < H ? w.posmap : nullptr,
          o->tgt_row, o->src_row, o->src_front);
    }
    FGL_LAUNCH_CHECK("translate");
  }
  return FGL_OK;
}


int64_t fgl_walk_ws_bytes(int64_t num_nodes, int64_t num_seeds) {
  const int64_t words = align_up(ceil_div(num_nodes, 32), 4);
  return align_up(4 * words, 256) + align_up(4 * std::max<int64_t>(num_seeds, 1), 256) +
         align_up(8 * (2 * kPersistentCTAs + 2), 256) + 256;
}

int fgl_sample_walk(const fgl_graph* g, const int32_t* seeds, int64_t num_seeds, int32_t length, uint64_t key0,
                    uint64_t key1, int32_t* tgt, int32_t* src, float* wgt, int64_t edge_cap, int64_t* step_off,
                    int32_t* unique_nodes, int64_t unique_cap, int64_t* counts, void* ws, int64_t ws_bytes,
                    void* stream_) {
  cudaStream_t stream = (cudaStream_t)stream_;
  if (!g || !seeds || num_seeds < 1 || length < 1 || !tgt || !src || !wgt || !step_off || !unique_nodes ||
      !counts || !ws) {
    set_error("fgl_sample_walk: bad arguments");
    return FGL_E_INVALID;
  }
  if (edge_cap < num_seeds * (int64_t)length) {
    set_error("fgl_sample_walk: edge buffer below num_seeds * length");
    return FGL_E_CAPACITY;
  }
  if (ws_bytes < fgl_walk_ws_bytes(g->num_nodes, num_seeds)) {
    set_error("fgl_sample_walk: workspace too small");
    return FGL_E_CAPACITY;
  }
  const int64_t words = align_up(ceil_div(g->num_nodes, 32), 4);
  char* p = static_cast<char*>(ws);
  uint32_t* bm = reinterpret_cast<uint32_t*>(p);
  p += align_up(4 * words, 256);
  int32_t* cur = reinterpret_cast<int32_t*>(p);
  p += align_up(4 * std::max<int64_t>(num_seeds, 1), 256);
  int64_t* part = reinterpret_cast<int64_t*>(p);
  p += align_up(8 * (2 * kPersistentCTAs + 2), 256);
  int64_t* scal = reinterpret_cast<int64_t*>(p);
  // counts: [0] unique total, [1] status
  FGL_CUDA(cudaMemsetAsync(counts, 0, 2 * sizeof(int64_t), stream));
  FGL_CUDA(cudaMemsetAsync(bm, 0, 4 * words, stream));
  FGL_COUNT_LAUNCH(), walk_kernel<<<1, kWalkThreads, 0, stream>>>(
      g->row_offsets, g->col_indices, g->edge_weights, seeds, num_seeds, length, key0, key1, g->num_nodes, cur,
      tgt, src, wgt, step_off, bm, counts + 1);
  FGL_LAUNCH_CHECK("walk_kernel");
  const int G = kPersistentCTAs;
  FGL_COUNT_LAUNCH(), bm_count_kernel<<<G, kScanThreads, 0, stream>>>(bm, words, part);
  FGL_COUNT_LAUNCH(), scan_partials_kernel<<<1, 1024, 0, stream>>>(part, G, scal, counts);
  launch_bm_compact(G, stream, bm, words, words, part, unique_nodes, nullptr, nullptr, nullptr, nullptr, 0, unique_cap,
                    counts + 1);
  FGL_LAUNCH_CHECK("walk unique compaction");
  return FGL_OK;
}

}  // extern "C"
