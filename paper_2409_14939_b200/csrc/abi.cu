// C-ABI plumbing: error strings, version, device check, Philox known-answer
// and ALU-roofline probe kernels.
#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

namespace fgl {

static thread_local std::string g_last_error;
static std::atomic<long long> g_launches{0};

static std::atomic<long long> g_dense_fallbacks{0};

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return (v && *v) ? atoi(v) : dflt;
}

namespace {
struct ProfRec {
  int id;
  int64_t a[3];
  cudaEvent_t e0, e1;
};
std::atomic<bool> g_prof{false};
std::mutex g_prof_mu;
std::vector<ProfRec> g_prof_rec;
}  // namespace

// Inside a stream capture the events become external event-record nodes of
// the graph (cudaEventRecordExternal): they record -- with timestamps -- each
// time the executable graph replays, so the kernels are timed live in the
// pipeline that is actually measured.
static cudaError_t prof_record(cudaEvent_t e, cudaStream_t st, bool captured) {
  return captured ? cudaEventRecordWithFlags(e, st, cudaEventRecordExternal) : cudaEventRecord(e, st);
}

ProfMark prof_begin(cudaStream_t st) {
  ProfMark m;
  if (!g_prof.load(std::memory_order_relaxed)) return m;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs == cudaStreamCaptureStatusInvalidated) return m;
  if (cudaEventCreate(&m.e0) != cudaSuccess) return ProfMark{};
  m.captured = cs == cudaStreamCaptureStatusActive;
  if (prof_record(m.e0, st, m.captured) != cudaSuccess) {
    cudaGetLastError();
    cudaEventDestroy(m.e0);
    return ProfMark{};
  }
  m.st = st;
  return m;
}

void prof_end(const ProfMark& m, int id, int64_t a0, int64_t a1, int64_t a2) {
  if (!m.e0) return;
  cudaEvent_t e1 = nullptr;
  if (cudaEventCreate(&e1) != cudaSuccess) {
    cudaEventDestroy(m.e0);
    return;
  }
  if (prof_record(e1, m.st, m.captured) != cudaSuccess) {
    cudaGetLastError();
    cudaEventDestroy(e1);
    cudaEventDestroy(m.e0);
    return;
  }
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof_rec.push_back(ProfRec{id, {a0, a1, a2}, m.e0, e1});
}
void count_dense_fallback() { g_dense_fallbacks.fetch_add(1, std::memory_order_relaxed); }

void set_error(const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

int cuda_status(cudaError_t e, const char* what) {
  set_error("CUDA error in %s: %s", what, cudaGetErrorString(e));
  return FGL_E_CUDA;
}

__global__ void philox_words_kernel(uint64_t k0, uint64_t k1, int64_t start, int64_t count,
                                    uint64_t* out) {
  const int64_t first_blk = start >> 2;
  const int64_t last_blk = (start + count - 1) >> 2;
  for (int64_t b = first_blk + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b <= last_blk;
       b += (int64_t)gridDim.x * blockDim.x) {
    uint64_t w[4];
    philox4x64_10((uint64_t)b + 1, k0, k1, w[0], w[1], w[2], w[3]);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t p = 4 * b + q;
      if (p >= start && p < start + count) out[p - start] = w[q];
    }
  }
}

// ALU roofline probe: every thread draws a contiguous run of Philox blocks
// under its own key (as the select kernels do: lanes work on different nodes /
// batches, so the key schedule is per lane) and folds the words with xor so
// nothing is dead code.  Full occupancy (64 warps / SM); tools/probes/
// philox_occ.cu shows the rate saturates from ~16 warps / SM up.
__global__ void __launch_bounds__(256) philox_bench_kernel(uint64_t k0, uint64_t k1, int iters, uint64_t* out) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const uint64_t lk0 = k0 ^ (uint64_t)threadIdx.x, base = (uint64_t)tid * (uint64_t)iters;
  uint64_t acc = 0;
  for (int i = 0; i < iters; ++i) {
    uint64_t w0, w1, w2, w3;
    philox4x64_10(base + i + 1, lk0, k1, w0, w1, w2, w3);
    acc ^= w0 ^ w1 ^ w2 ^ w3;
  }
  out[tid] = acc;
}

}  // namespace fgl

extern "C" {

const char* fgl_last_error(void) { return fgl::g_last_error.c_str(); }

int fgl_version(void) { return 100; }

int64_t fgl_launch_count(void) { return fgl::g_launches.load(std::memory_order_relaxed); }
int64_t fgl_dense_fallback_count(void) { return fgl::g_dense_fallbacks.load(std::memory_order_relaxed); }

int fgl_profile(int32_t enable) {
  fgl::g_prof.store(enable != 0);
  return FGL_OK;
}

int fgl_profile_read(int64_t cap, int32_t* ids, int64_t* args3, double* ms, int64_t* count) {
  std::lock_guard<std::mutex> lk(fgl::g_prof_mu);
  int64_t k = 0;
  for (auto& r : fgl::g_prof_rec) {
    float t = 0.f;
    // a record whose capture was aborted (the work then ran eagerly) never
    // executed: skip it
    if (cudaEventSynchronize(r.e1) != cudaSuccess || cudaEventElapsedTime(&t, r.e0, r.e1) != cudaSuccess) {
      cudaGetLastError();
      cudaEventDestroy(r.e0);
      cudaEventDestroy(r.e1);
      continue;
    }
    if (k < cap) {
      if (ids) ids[k] = r.id;
      if (args3)
        for (int i = 0; i < 3; ++i) args3[3 * k + i] = r.a[i];
      if (ms) ms[k] = t;
    }
    ++k;
    cudaEventDestroy(r.e0);
    cudaEventDestroy(r.e1);
  }
  if (count) *count = k;
  fgl::g_prof_rec.clear();
  return FGL_OK;
}

int fgl_device_check(int device) {
  cudaDeviceProp p;
  cudaError_t e = cudaGetDeviceProperties(&p, device);
  if (e != cudaSuccess) return fgl::cuda_status(e, "cudaGetDeviceProperties");
  if (p.major != 10) {
    fgl::set_error("libfastgl_b200 is built for sm_100a; device %d is sm_%d%d", device, p.major,
                   p.minor);
    return FGL_E_UNSUPPORTED;
  }
  return FGL_OK;
}

int fgl_philox_words(uint64_t k0, uint64_t k1, int64_t start, int64_t count, uint64_t* out,
                     void* stream) {
  if (start < 0 || count < 0 || (count > 0 && out == nullptr)) {
    fgl::set_error("fgl_philox_words: bad arguments");
    return FGL_E_INVALID;
  }
  if (count == 0) return FGL_OK;
  const int64_t blocks = ((start + count - 1) >> 2) - (start >> 2) + 1;
  const int threads = 256;
  const int grid = (int)std::min<int64_t>(fgl::ceil_div(blocks, threads), 148 * 32);
  FGL_COUNT_LAUNCH(), fgl::philox_words_kernel<<<grid, threads, 0, (cudaStream_t)stream>>>(k0, k1, start, count, out);
  FGL_LAUNCH_CHECK("philox_words_kernel");
  return FGL_OK;
}

int fgl_philox_bench(uint64_t k0, uint64_t k1, int64_t blocks, uint64_t* out, void* stream) {
  if (blocks < 1 || !out) return FGL_E_INVALID;
  // 148 x 8 CTAs of 256 threads; blocks rounded down to a multiple of the threads
  const int64_t threads = (int64_t)148 * 8 * 256;
  const int iters = (int)std::max<int64_t>(1, blocks / threads);
  FGL_COUNT_LAUNCH(), fgl::philox_bench_kernel<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(k0, k1, iters, out);
  FGL_LAUNCH_CHECK("philox_bench_kernel");
  return FGL_OK;
}

}  // extern "C"
