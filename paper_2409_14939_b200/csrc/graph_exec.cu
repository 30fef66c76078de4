// CUDA-graph replay of the per-batch model chain.
//
// A mini-batch's weight-dependent chain (forward, loss, backward with the
// side-stream weight gradients, SGD) is ~30 dependent launches of small,
// latency-bound kernels.  Launched one by one each costs ~3-4 us of host issue
// time and a launch gap on the device; replayed from a CUDA graph the gap is
// ~0.6 us (tools/probes/launch_probe.cu).  The chain's shape is the same for
// every batch -- only sizes and pointers change -- so the trainer captures each
// batch on its stream (fgl_capture_begin), and fgl_capture_end_launch folds the
// new capture into one executable graph per slot with cudaGraphExecUpdate
// (parameters and grid sizes change, the topology does not), instantiating only
// when the update is refused (first use, or a batch that took a different
// kernel path).  Any failure aborts the capture; the caller then runs the
// batch eagerly, so the results never depend on whether a graph was used.
#include "common.cuh"

namespace fgl {
namespace {
constexpr int kSlots = 4;
cudaGraphExec_t g_exec[kSlots] = {nullptr, nullptr, nullptr, nullptr};
int64_t g_stats[3] = {0, 0, 0};  // launches, updates, instantiations
}  // namespace
}  // namespace fgl

using namespace fgl;

extern "C" {

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

int fgl_capture_end_launch(int32_t slot, void* stream) {
  if (slot < 0 || slot >= kSlots) {
    set_error("fgl_capture_end_launch: slot %d out of range", slot);
    return FGL_E_INVALID;
  }
  cudaStream_t st = (cudaStream_t)stream;
  cudaGraph_t g = nullptr;
  FGL_CUDA(cudaStreamEndCapture(st, &g));
  bool ok = false;
  if (g_exec[slot]) {
    cudaGraphExecUpdateResultInfo info;
    if (cudaGraphExecUpdate(g_exec[slot], g, &info) == cudaSuccess) {
      ok = true;
      ++g_stats[1];
    } else {
      cudaGetLastError();
      cudaGraphExecDestroy(g_exec[slot]);
      g_exec[slot] = nullptr;
    }
  }
  if (!ok) {
    cudaError_t e = cudaGraphInstantiate(&g_exec[slot], g, 0);
    if (e != cudaSuccess) {
      cudaGraphDestroy(g);
      g_exec[slot] = nullptr;
      return cuda_status(e, "cudaGraphInstantiate");
    }
    ++g_stats[2];
  }
  cudaGraphDestroy(g);
  FGL_CUDA(cudaGraphLaunch(g_exec[slot], st));
  ++g_stats[0];
  return FGL_OK;
}

int fgl_capture_stats(int64_t* out3) {
  if (!out3) return FGL_E_INVALID;
  for (int i = 0; i < 3; ++i) out3[i] = g_stats[i];
  return FGL_OK;
}

}  // extern "C"
