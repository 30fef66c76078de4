/*
 * fastgl_b200.h -- C ABI of libfastgl_b200.so, the B200 (sm_100a) hot path of
 * FastGL mini-batch GNN training (arXiv 2409.14939), built behind the
 * function-level operator API of the reference package `minigl` 0.1.0.
 *
 * Conventions:
 *  - Caller-owned DEVICE buffers are passed as raw pointers (e.g. a torch
 *    tensor's data_ptr()); host arrays are marked (host).
 *  - Every call is asynchronous on `stream` (a cudaStream_t passed as void*)
 *    and never synchronises the host, unless documented otherwise.
 *  - Return value: FGL_OK (0) or a negative FGL_E_* code; a message is kept
 *    per thread in fgl_last_error().  The Python layer maps the codes to the
 *    reference's exception types (errors.py:1-35).
 *  - Node IDs on device are int32 (N < 2^31); CSR offsets are int64.
 *  - No global mutable state; calls on distinct streams/buffers are
 *    independent and thread-safe.
 */
#ifndef FASTGL_B200_H
#define FASTGL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FGL_OK 0
#define FGL_E_INVALID (-1)     /* minigl ValidationError */
#define FGL_E_CAPACITY (-2)    /* minigl CapacityError (table full / buffer too small) */
#define FGL_E_NOTFOUND (-3)    /* minigl NotFoundError */
#define FGL_E_CONFIG (-4)      /* minigl ConfigError */
#define FGL_E_CUDA (-5)        /* CUDA runtime error */
#define FGL_E_UNSUPPORTED (-6) /* configuration outside what the kernels implement */

#define FGL_MAX_HOPS 8

/* ------------------------------------------------------------------ misc -- */
const char* fgl_last_error(void);
int fgl_version(void);
/* Device properties the build was compiled for; returns FGL_E_CUDA without a GPU. */
int fgl_device_check(int device);

/* --------------------------------------------------------------- graph ---- */
/* Device-resident CSR.  Replaces the host arrays of minigl.graph.Graph
 * (graph.py:25-87): row_offsets (u64 -> int64), col_indices (u64 -> int32),
 * optional edge_weights (f32).  Plain struct of device pointers. */
typedef struct fgl_graph {
  int64_t num_nodes;
  int64_t num_edges;
  const int64_t* row_offsets;  /* device, num_nodes + 1 */
  const int32_t* col_indices;  /* device, num_edges */
  const float* edge_weights;   /* device, num_edges, or NULL for unit weights */
} fgl_graph;

/* ------------------------------------------------------------- sampler ---- */
/* Worst-case sizes for a window of `num_batches` batches with the given seed
 * counts (host) and fanouts (host): out[0] = edge capacity (all hops, all
 * batches), out[1] = concatenated frontier capacity of one hop, out[2] =
 * unique-node capacity, out[3] = workspace bytes, out[4] = counts length. */
int fgl_sample_bounds(int64_t num_nodes, const int64_t* batch_sizes, int32_t num_batches,
                      const int32_t* fanouts, int32_t num_hops, int64_t* out);

/*
 * Fused-Map k-hop sampling of a window of batches + global->local remap.
 * Replaces sampler.sample_khop (sampler.py:120-139) per batch b, with
 * batch b's Philox key keys[2b], keys[2b+1] (= Philox(derive_seed(seed,13,j))
 * key, trainer.py:304) -- bit-exact with the reference; and idmap.build /
 * translate_batch (idmap.py:198-233, :294-303) on the trainer path, where the
 * local ID of a node is its rank in the batch's sorted unique_nodes.
 *
 *  seeds       device int32, all batches concatenated
 *  seed_off    device int64[num_batches+1]
 *  keys        device uint64[2*num_batches]
 *  fanouts     host int32[num_hops]; fanouts[0] expands the seeds; 1..256
 *  tgt/src/wgt device outputs, capacity edge_cap: hop-major, batch-minor
 *  local_tgt/local_src  optional (NULL) device int32 local IDs of tgt/src
 *  unique_nodes device int32, capacity unique_cap, batch-major, each sorted
 *  seed_locals optional (NULL) device int32 local IDs of the seeds
 *  counts      device int64[counts_len] (see FGL_CNT_* below)
 *  ws          device workspace of fgl_sample_bounds()[3] bytes
 * Per-batch node bitmaps stay valid in `ws` after the call (used by
 * fgl_match_counts / fgl_gather_delta) until the next call on the same ws.
 */
int fgl_sample_window(const fgl_graph* g, const int32_t* seeds, const int64_t* seed_off,
                      int64_t total_seeds, int32_t num_batches, const uint64_t* keys,
                      const int32_t* fanouts, int32_t num_hops,
                      int32_t* tgt, int32_t* src, float* wgt, int64_t edge_cap,
                      int32_t* local_tgt, int32_t* local_src,
                      int32_t* unique_nodes, int64_t unique_cap, int32_t* seed_locals,
                      int64_t* counts, void* ws, int64_t ws_bytes, void* stream);

/* counts layout for H hops, nb batches:
 *   [0, H*nb]              edge offsets: hop h batch b spans
 *                          [counts[h*nb+b], counts[h*nb+b+1])
 *   [U0, U0+nb]            unique offsets, U0 = H*nb+1
 *   [D0, D0+nb)            Philox draws (candidates) per batch, D0 = U0+nb+1
 *   [F0, F0+H*nb)          frontier size per (hop, batch), F0 = D0+nb
 *   [S0]                   status (0 ok), S0 = F0+H*nb                        */
#define FGL_CNT_UNIQ(H, nb) ((H) * (nb) + 1)
#define FGL_CNT_DRAWS(H, nb) (FGL_CNT_UNIQ(H, nb) + (nb) + 1)
#define FGL_CNT_FRONT(H, nb) (FGL_CNT_DRAWS(H, nb) + (nb))
#define FGL_CNT_STATUS(H, nb) (FGL_CNT_FRONT(H, nb) + (H) * (nb))
#define FGL_CNT_LEN(H, nb) (FGL_CNT_STATUS(H, nb) + 1)

/* Philox4x64-10 stream words at absolute positions [start, start+count) for
 * key (k0,k1), as uint64 (>>11 gives the key Generator.random() uses).
 * Known-answer and microbenchmark entry (oracle/philox.py). */
int fgl_philox_words(uint64_t k0, uint64_t k1, int64_t start, int64_t count, uint64_t* out,
                     void* stream);
/* Draws `count` Philox blocks and reduces them to one word (ALU roofline probe). */
int fgl_philox_bench(uint64_t k0, uint64_t k1, int64_t blocks, uint64_t* out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FASTGL_B200_H */
