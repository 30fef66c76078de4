// Fused-Map global->local ID table on the GPU (sm_100a).
//
// Replaces idmap.build / lookup_many (idmap.py:88-117, :154-172, :198-233,
// :269-286) for arbitrary uint64 IDs with the reference's exact table state:
// open addressing, linear probing, Fibonacci hash (gid*0x9E3779B97F4A7C15)>>shift
// or gid % capacity, SENTINEL = all ones, and the single-worker result --
// local IDs in first-seen order and the slot layout of sequential insertion.
//
// The reference's concurrent build races workers on a CAS + fetch_add, which
// yields a different (race-ordered) bijection on every run.  Here the build is
// deterministic and still fully parallel:
//   A. every occurrence CAS-inserts its key into a scratch table and
//      atomicMin's its index into the slot's first-seen index;
//   B. an occurrence is "first" iff its index is that minimum; an exclusive
//      scan of the first-flags gives local IDs in first-seen order;
//   C. the distinct keys are inserted into the final table by PRIORITY linear
//      probing: a slot holds the smallest local ID that reached it
//      (atomicMin), a displaced larger ID keeps probing from the next slot.
//      A key with local ID j ends in the first slot from its hash not held by
//      a smaller ID -- exactly where sequential first-seen insertion puts it.
#include <algorithm>

#include "common.cuh"

namespace fgl {
namespace {

constexpr uint64_t kSent = ~0ull;
constexpr uint32_t kNone = 0xffffffffu;

__device__ __forceinline__ uint64_t home_slot(uint64_t gid, uint64_t cap, int shift, int mod_hash) {
  return mod_hash ? gid % cap : (gid * 0x9E3779B97F4A7C15ull) >> shift;
}

__device__ __forceinline__ void set_code(int64_t* status, int64_t code) {
  atomicCAS(reinterpret_cast<unsigned long long*>(status), 0ull, (unsigned long long)code);
}

// A: scratch insert + first-seen index per distinct key
__global__ void first_seen_kernel(const uint64_t* __restrict__ ids, int64_t n, uint64_t cap, int shift,
                                  int mod_hash, unsigned long long* __restrict__ skeys,
                                  uint32_t* __restrict__ sfirst, int64_t* status) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t g = ids[i];
    uint64_t s = home_slot(g, cap, shift, mod_hash);
    uint64_t probes = 0;
    for (;;) {
      const unsigned long long prev = atomicCAS(skeys + s, kSent, (unsigned long long)g);
      if (prev == kSent || prev == g) {
        atomicMin(sfirst + s, (uint32_t)i);
        break;
      }
      if (++probes >= cap) { set_code(status, FGL_E_CAPACITY); break; }
      if (++s == cap) s = 0;
    }
  }
}

__device__ __forceinline__ int64_t find_slot(const unsigned long long* keys, uint64_t g, uint64_t cap,
                                             int shift, int mod_hash) {
  uint64_t s = home_slot(g, cap, shift, mod_hash);
  for (uint64_t probes = 0; probes < cap; ++probes) {
    const unsigned long long k = keys[s];
    if (k == g) return (int64_t)s;
    if (k == kSent) return -1;
    if (++s == cap) s = 0;
  }
  return -1;
}

// B: first-occurrence flags
__global__ void first_flag_kernel(const uint64_t* __restrict__ ids, int64_t n, uint64_t cap, int shift,
                                  int mod_hash, const unsigned long long* __restrict__ skeys,
                                  const uint32_t* __restrict__ sfirst, int32_t* __restrict__ flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = find_slot(skeys, ids[i], cap, shift, mod_hash);
    flag[i] = (s >= 0 && sfirst[s] == (uint32_t)i) ? 1 : 0;
  }
}

__global__ void chunk_sum32_kernel(const int32_t* __restrict__ v, int64_t n, int64_t* part) {
  __shared__ int64_t sm[33];
  const int64_t chunk = ceil_div(n, gridDim.x);
  const int64_t i0 = blockIdx.x * chunk, i1 = min(n, i0 + chunk);
  int64_t s = 0;
  for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) s += v[i];
  s = block_sum(s, sm);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void scan_part_kernel(int64_t* part, int n, int64_t* total) {
  __shared__ int64_t sm[33];
  int64_t carry = 0;
  for (int b = 0; b < n; b += blockDim.x) {
    const int i = b + threadIdx.x;
    int64_t v = i < n ? part[i] : 0, tot;
    const int64_t ex = block_excl_scan(v, sm, &tot);
    if (i < n) part[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0) *total = carry;
}

// local ID of each first occurrence; distinct keys in first-seen order
__global__ void assign_kernel(const uint64_t* __restrict__ ids, const int32_t* __restrict__ flag,
                              int64_t n, const int64_t* __restrict__ part,
                              uint64_t* __restrict__ dkeys) {
  __shared__ int64_t sm[33];
  const int64_t chunk = ceil_div(n, gridDim.x);
  const int64_t i0 = blockIdx.x * chunk, i1 = min(n, i0 + chunk);
  int64_t run = part[blockIdx.x];
  for (int64_t t0 = i0; t0 < i1; t0 += blockDim.x) {
    const int64_t i = t0 + threadIdx.x;
    const int64_t f = i < i1 ? flag[i] : 0;
    int64_t tot;
    const int64_t ex = block_excl_scan(f, sm, &tot);
    if (f) dkeys[run + ex] = ids[i];
    run += tot;
  }
}

// C: priority linear probing of the distinct keys (priority = local ID)
__global__ void priority_insert_kernel(const uint64_t* __restrict__ dkeys, const int64_t* __restrict__ nd_ptr,
                                       uint64_t cap, int shift, int mod_hash,
                                       uint32_t* __restrict__ prio, int64_t* status) {
  const int64_t nd = *nd_ptr;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nd;
       j += (int64_t)gridDim.x * blockDim.x) {
    uint32_t cur = (uint32_t)j;
    uint64_t s = home_slot(dkeys[j], cap, shift, mod_hash);
    uint64_t steps = 0;
    for (;;) {
      const uint32_t old = atomicMin(prio + s, cur);
      if (old == kNone) break;           // claimed an empty slot
      if (old > cur) cur = old;          // displaced a later key: carry it on
      if (++steps >= 4 * cap + 64) { set_code(status, FGL_E_CAPACITY); break; }  // table full
      if (++s == cap) s = 0;
    }
  }
}

__global__ void materialize_kernel(const uint32_t* __restrict__ prio, uint64_t cap,
                                   const uint64_t* __restrict__ dkeys, uint64_t* __restrict__ keys,
                                   uint64_t* __restrict__ values) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < (int64_t)cap;
       s += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t p = prio[s];
    keys[s] = p == kNone ? kSent : dkeys[p];
    values[s] = p == kNone ? 0ull : (uint64_t)p;
  }
}

__global__ void lookup_kernel(const unsigned long long* __restrict__ keys, const uint64_t* __restrict__ values,
                              uint64_t cap, int shift, int mod_hash, const uint64_t* __restrict__ ids,
                              int64_t n, uint64_t* __restrict__ out, unsigned long long* first_miss) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = find_slot(keys, ids[i], cap, shift, mod_hash);
    if (s >= 0) {
      out[i] = values[s];
    } else {
      out[i] = kSent;  // SENTINEL miss marker (idmap.py:167)
      if (first_miss) atomicMin(first_miss, (unsigned long long)i);
    }
  }
}

int grid_of(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), 148 * 16)); }
inline int64_t al(int64_t x) { return (x + 255) / 256 * 256; }

}  // namespace
}  // namespace fgl

using namespace fgl;

extern "C" {

int64_t fgl_idmap_ws_bytes(int64_t n, int64_t capacity) {
  return al(8 * capacity) + al(4 * capacity) + al(4 * std::max<int64_t>(n, 1)) +
         al(8 * std::max<int64_t>(n, 1)) + al(4 * capacity) + al(8 * (kPersistentCTAs + 2));
}

int fgl_idmap_build(const uint64_t* ids, int64_t n, int32_t mod_hash, int64_t capacity,
                    int32_t shift, uint64_t* keys, uint64_t* values, int64_t* status2,
                    void* ws, int64_t ws_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 1 || capacity < 1 || !ids || !keys || !values || !status2 || shift < 0 || shift > 63 ||
      n >= (1ll << 31) || capacity >= (1ll << 32)) {
    set_error("fgl_idmap_build: bad arguments");
    return FGL_E_INVALID;
  }
  if (ws_bytes < fgl_idmap_ws_bytes(n, capacity)) {
    set_error("fgl_idmap_build: workspace too small");
    return FGL_E_CAPACITY;
  }
  char* p = static_cast<char*>(ws);
  auto* skeys = reinterpret_cast<unsigned long long*>(p); p += al(8 * capacity);
  auto* sfirst = reinterpret_cast<uint32_t*>(p); p += al(4 * capacity);
  auto* flag = reinterpret_cast<int32_t*>(p); p += al(4 * n);
  auto* dkeys = reinterpret_cast<uint64_t*>(p); p += al(8 * n);
  auto* prio = reinterpret_cast<uint32_t*>(p); p += al(4 * capacity);
  auto* part = reinterpret_cast<int64_t*>(p);
  // status2[0] = status, status2[1] = number of distinct keys
  FGL_CUDA(cudaMemsetAsync(status2, 0, 16, st));
  FGL_CUDA(cudaMemsetAsync(skeys, 0xff, 8 * capacity, st));
  FGL_CUDA(cudaMemsetAsync(sfirst, 0xff, 4 * capacity, st));
  FGL_CUDA(cudaMemsetAsync(prio, 0xff, 4 * capacity, st));
  const uint64_t cap = (uint64_t)capacity;
  FGL_COUNT_LAUNCH(), first_seen_kernel<<<grid_of(n), 256, 0, st>>>(ids, n, cap, shift, mod_hash, skeys, sfirst, status2);
  FGL_COUNT_LAUNCH(), first_flag_kernel<<<grid_of(n), 256, 0, st>>>(ids, n, cap, shift, mod_hash, skeys, sfirst, flag);
  const int G = (int)std::max<int64_t>(1, std::min<int64_t>(kPersistentCTAs, ceil_div(n, 1024)));
  FGL_COUNT_LAUNCH(), chunk_sum32_kernel<<<G, 256, 0, st>>>(flag, n, part);
  FGL_COUNT_LAUNCH(), scan_part_kernel<<<1, 1024, 0, st>>>(part, G, status2 + 1);
  FGL_COUNT_LAUNCH(), assign_kernel<<<G, 256, 0, st>>>(ids, flag, n, part, dkeys);
  FGL_COUNT_LAUNCH(), priority_insert_kernel<<<grid_of(n), 256, 0, st>>>(dkeys, status2 + 1, cap, shift, mod_hash, prio, status2);
  FGL_COUNT_LAUNCH(), materialize_kernel<<<grid_of(capacity), 256, 0, st>>>(prio, cap, dkeys, keys, values);
  FGL_LAUNCH_CHECK("idmap_build");
  return FGL_OK;
}

int fgl_idmap_lookup(const uint64_t* keys, const uint64_t* values, int64_t capacity, int32_t mod_hash,
                     int32_t shift, const uint64_t* ids, int64_t n, uint64_t* out, int64_t* first_miss,
                     void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (n < 0 || capacity < 1 || !keys || !values || (n > 0 && (!ids || !out)) || shift < 0 || shift > 63) {
    set_error("fgl_idmap_lookup: bad arguments");
    return FGL_E_INVALID;
  }
  if (first_miss) FGL_CUDA(cudaMemsetAsync(first_miss, 0x7f, 8, st));  // "no miss" = 0x7f7f...
  if (n == 0) return FGL_OK;
  FGL_COUNT_LAUNCH(), lookup_kernel<<<grid_of(n), 256, 0, st>>>(
      reinterpret_cast<const unsigned long long*>(keys), values, (uint64_t)capacity, shift, mod_hash,
      ids, n, out, reinterpret_cast<unsigned long long*>(first_miss));
  FGL_LAUNCH_CHECK("idmap_lookup");
  return FGL_OK;
}

}  // extern "C"
