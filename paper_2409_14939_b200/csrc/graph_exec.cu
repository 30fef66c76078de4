// CUDA-graph replay of the per-batch model chain.
//
// A mini-batch's weight-dependent chain (forward, loss, backward with the
// side-stream weight gradients, SGD) is ~30 dependent launches of small,
// latency-bound kernels.  Launched one by one each costs ~3-4 us of host issue
// time and a launch gap on the device; replayed from a CUDA graph the gap is
// ~0.6 us (tools/probes/launch_probe.cu).  The chain's shape is the same for
// every batch -- only sizes and pointers change -- so the trainer captures each
// batch on its stream (fgl_capture_begin), and fgl_capture_end_launch folds the
// new capture into one executable graph per caller-owned handle (fgl_exec) with cudaGraphExecUpdate
// (parameters and grid sizes change, the topology does not), instantiating only
// when the update is refused (first use, or a batch that took a different
// kernel path).  Any failure aborts the capture; the caller then runs the
// batch eagerly, so the results never depend on whether a graph was used.
#include <atomic>

#include "common.cuh"

namespace fgl {
namespace {
std::atomic<int64_t> g_stats[3];  // launches, updates, instantiations (process-wide counters)
}  // namespace
}  // namespace fgl

// One executable graph, owned by the caller (a Pipeline keeps one per
// sequence it replays: batch chain, prepare, sampler, window chain), so two
// pipelines -- or two devices -- never update each other's executables.
struct fgl_exec {
  cudaGraphExec_t exec = nullptr;
  int device = -1;
};

using namespace fgl;

extern "C" {

int fgl_exec_create(fgl_exec** out) {
  if (!out) return FGL_E_INVALID;
  fgl_exec* h = new fgl_exec();
  FGL_CUDA(cudaGetDevice(&h->device));
  *out = h;
  return FGL_OK;
}

int fgl_exec_destroy(fgl_exec* h) {
  if (!h) return FGL_OK;
  if (h->exec) cudaGraphExecDestroy(h->exec);
  delete h;
  return FGL_OK;
}

int fgl_capture_begin(void* stream) {
  FGL_CUDA(cudaStreamBeginCapture((cudaStream_t)stream, cudaStreamCaptureModeThreadLocal));
  return FGL_OK;
}

int fgl_capture_abort(void* stream) {
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture((cudaStream_t)stream, &g);
  if (g) cudaGraphDestroy(g);
  cudaGetLastError();  // clear a sticky capture-invalidation error
  (void)e;
  return FGL_OK;
}

int fgl_capture_end_launch(fgl_exec* h, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (!h) {
    fgl_capture_abort(stream);
    set_error("fgl_capture_end_launch: null executable handle");
    return FGL_E_INVALID;
  }
  int dev = -1;
  FGL_CUDA(cudaGetDevice(&dev));
  if (dev != h->device) {
    fgl_capture_abort(stream);
    set_error("fgl_capture_end_launch: handle of device %d used on device %d", h->device, dev);
    return FGL_E_INVALID;
  }
  cudaGraph_t g = nullptr;
  FGL_CUDA(cudaStreamEndCapture(st, &g));
  bool ok = false;
  if (h->exec) {
    cudaGraphExecUpdateResultInfo info;
    if (cudaGraphExecUpdate(h->exec, g, &info) == cudaSuccess) {
      ok = true;
      ++g_stats[1];
    } else {
      cudaGetLastError();
      cudaGraphExecDestroy(h->exec);
      h->exec = nullptr;
    }
  }
  if (!ok) {
    cudaError_t e = cudaGraphInstantiate(&h->exec, g, 0);
    if (e != cudaSuccess) {
      cudaGraphDestroy(g);
      h->exec = nullptr;
      return cuda_status(e, "cudaGraphInstantiate");
    }
    ++g_stats[2];
  }
  cudaGraphDestroy(g);
  FGL_CUDA(cudaGraphLaunch(h->exec, st));
  ++g_stats[0];
  return FGL_OK;
}

// Cross-graph ordering: events recorded / waited on with the External flags
// become event-record / event-wait nodes when the stream is being captured
// (a plain record/wait outside a capture otherwise), so one graph (the
// window's batch chain) can wait on a point inside another (the prepare
// graph's per-batch layer-0 aggregation) instead of on its end.
int fgl_event_create(void** out) {
  if (!out) return FGL_E_INVALID;
  cudaEvent_t e = nullptr;
  FGL_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  *out = e;
  return FGL_OK;
}

int fgl_event_destroy(void* ev) {
  if (ev) cudaEventDestroy((cudaEvent_t)ev);
  return FGL_OK;
}

static bool capturing(cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  return cudaStreamIsCapturing(st, &cs) == cudaSuccess && cs == cudaStreamCaptureStatusActive;
}

int fgl_event_record_ext(void* ev, void* stream) {
  if (!ev) return FGL_E_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  if (capturing(st)) FGL_CUDA(cudaEventRecordWithFlags((cudaEvent_t)ev, st, cudaEventRecordExternal));
  else FGL_CUDA(cudaEventRecord((cudaEvent_t)ev, st));
  return FGL_OK;
}

int fgl_stream_wait_ext(void* stream, void* ev) {
  if (!ev) return FGL_E_INVALID;
  cudaStream_t st = (cudaStream_t)stream;
  FGL_CUDA(cudaStreamWaitEvent(st, (cudaEvent_t)ev, capturing(st) ? cudaEventWaitExternal : 0));
  return FGL_OK;
}

int fgl_capture_stats(int64_t* out3) {
  if (!out3) return FGL_E_INVALID;
  for (int i = 0; i < 3; ++i) out3[i] = g_stats[i].load();
  return FGL_OK;
}

}  // extern "C"
