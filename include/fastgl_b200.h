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
 *  - Caller-owned state only (graph handles, executable graphs, work
 *    buffers), with these process-wide exceptions: the dense kernels' SM
 *    budget (fgl_set_dense_ctas), a launch counter and
 *    CUDA-graph counters (atomics), the per-thread last error, per-thread
 *    caches of TMA tensor maps keyed by buffer address, one-time kernel
 *    attribute settings (max dynamic shared memory), the profiling switch
 *    and its event record (fgl_profile), and A/B switches read once from
 *    the environment.  Calls on distinct streams/buffers are independent.
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
/* Number of CUDA kernels this library has launched in this process. */
int64_t fgl_launch_count(void);
/* Dense layer calls (fgl_dense_fwd / _bwd / _dgrad) whose shape fell outside
 * the tcgen05 kernels' envelope and ran on the SIMT fallback kernels. */
int64_t fgl_dense_fallback_count(void);
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
 * batches), out[1] = frontier stride (capacity of one hop's concatenated
 * frontier), out[2] = unique-node capacity, out[3] = workspace bytes,
 * out[4] = counts length. */
int fgl_sample_bounds(int64_t num_nodes, const int64_t* batch_sizes, int32_t num_batches,
                      const int32_t* fanouts, int32_t num_hops, int64_t* out);

/* Output buffers of fgl_sample_window (all DEVICE, caller-owned).  Edge arrays
 * are hop-major, batch-minor.  Optional pointers may be NULL. */
typedef struct fgl_sample_out {
  int32_t* tgt;          /* global target IDs (= the frontier node expanded) */
  int32_t* src;          /* global source IDs (the sampled neighbour) */
  float* wgt;            /* graph edge weight, or 1.0 */
  int64_t edge_cap;
  int32_t* tgt_row;      /* optional: window row of tgt = uniq_off[b] + rank in
                            batch b's sorted unique_nodes (trainer local ID) */
  int32_t* src_row;      /* optional: window row of src */
  int32_t* tgt_front;    /* optional: index of tgt in hop h's frontier list */
  int32_t* src_front;    /* optional: index of src in hop h+1's frontier list;
                            for the last hop: window row of src */
  int32_t* unique_nodes; /* batch-major, each batch sorted ascending */
  int64_t unique_cap;
  int32_t* frontier;     /* frontier lists: hop h at frontier + h*frontier_stride,
                            batch-major, each sorted (required if tgt_front or
                            src_front is requested) */
  int64_t frontier_stride;
  int32_t* seed_rows;    /* optional: window rows of the seeds */
  int32_t* seed_front;   /* optional: index of each seed in hop 0's frontier */
  int64_t* counts;       /* int64[counts_len], layout FGL_CNT_* below */
} fgl_sample_out;

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
 *  ws          device workspace of fgl_sample_bounds()[3] bytes
 * Per-batch node bitmaps stay valid in `ws` after the call (used by
 * fgl_match_counts) until the next call on the same ws.
 */
int fgl_sample_window(const fgl_graph* g, const int32_t* seeds, const int64_t* seed_off,
                      int64_t total_seeds, int32_t num_batches, const uint64_t* keys,
                      const int32_t* fanouts, int32_t num_hops, const fgl_sample_out* out,
                      void* ws, int64_t ws_bytes, void* stream);

/* counts layout for H hops, nb batches:
 *   [0, H*nb]            edge offsets: hop h batch b spans [c[h*nb+b], c[h*nb+b+1])
 *   [FO, FO+H*(nb+1))    frontier offsets, relative to hop h's list:
 *                        hop h batch b spans [c[FO+h*(nb+1)+b], c[FO+h*(nb+1)+b+1])
 *   [U0, U0+nb]          unique offsets (window rows)
 *   [D0, D0+nb)          Philox draws (candidates) per batch
 *   [S0]                 status (0 ok)                                          */
#define FGL_CNT_FRONT(H, nb) ((H) * (nb) + 1)
#define FGL_CNT_UNIQ(H, nb) (FGL_CNT_FRONT(H, nb) + (H) * ((nb) + 1))
#define FGL_CNT_DRAWS(H, nb) (FGL_CNT_UNIQ(H, nb) + (nb) + 1)
#define FGL_CNT_STATUS(H, nb) (FGL_CNT_DRAWS(H, nb) + (nb))
#define FGL_CNT_LEN(H, nb) (FGL_CNT_STATUS(H, nb) + 1)

/* Philox4x64-10 stream words at absolute positions [start, start+count) for
 * key (k0,k1), as uint64 (>>11 gives the key Generator.random() uses).
 * Known-answer and microbenchmark entry (oracle/philox.py). */
int fgl_philox_words(uint64_t k0, uint64_t k1, int64_t start, int64_t count, uint64_t* out,
                     void* stream);
/* ALU roofline probe: 148*8*256 threads each draw floor(blocks / 303104)
 * consecutive Philox blocks under a per-thread key and store one folded word
 * (out[303104]). */
int fgl_philox_bench(uint64_t k0, uint64_t k1, int64_t blocks, uint64_t* out, void* stream);
/* Random-walk sampler, drop-in for sampler.sample_random_walk
 * (sampler.py:142-186), bit-exact against the reference's Philox(seed) stream
 * (key0, key1 = SeedSequence(seed).generate_state(2)).  One walk of `length`
 * steps per seed; sinks stop early.  Edges (tgt, src, wgt) are step-major,
 * seed order within a step; step_off[0..length] are the step offsets
 * (step_off[length] = edges).  unique_nodes = sorted unique of seeds and
 * every visited node; counts[0] = its size, counts[1] = status (0 or an
 * FGL_E_* code written by the device).  Asynchronous on `stream`.
 * Replaces sampler.py:142-186 (the reference's pure-numpy walk). */
int64_t fgl_walk_ws_bytes(int64_t num_nodes, int64_t num_seeds);
int fgl_sample_walk(const fgl_graph* g, const int32_t* seeds, int64_t num_seeds, int32_t length, uint64_t key0,
                    uint64_t key1, int32_t* tgt, int32_t* src, float* wgt, int64_t edge_cap, int64_t* step_off,
                    int32_t* unique_nodes, int64_t unique_cap, int64_t* counts, void* ws, int64_t ws_bytes,
                    void* stream);

/* Measurement hook (bench.py per-stage rooflines): while enabled, the
 * dominant launch of every stage -- select (id 1, a = {hop}), layer-0 block
 * aggregation (2, {rows, d}), fgl_spmm (3, {rows, d}), dense forward (4,
 * {M, N, K}), dgrad (5, {M, N, K}), weight gradient (6, {M, K, N}), x0
 * gather (7, {rows, d}) -- is bracketed by CUDA events on its own stream;
 * inside a stream capture they become external event-record nodes, timed on
 * every replay of the graph.
 * fgl_profile_read synchronises on them and writes up to `cap` records
 * (ids, args3[3*k..], device ms) in issue order plus the record count, then
 * clears the record. */
int fgl_profile(int32_t enable);
int fgl_profile_read(int64_t cap, int32_t* ids, int64_t* args3, double* ms, int64_t* count);

/* ------------------------------------------------------------- prepare ---- */
/* indptr[r] = base + (first e with rows[e] >= r), r in [0, num_rows]; `rows`
 * non-decreasing.  The forward CSR of a sampled hop (targets arrive grouped in
 * ascending order, so compute.edges_to_csr's stable argsort is the identity,
 * compute.py:219-230). */
int fgl_csr_offsets_sorted(const int32_t* rows, int64_t nnz, int64_t num_rows, int64_t base,
                           int64_t* indptr, void* stream);

/* Stable counting sort of `keys` (values in [0, num_keys)): indptr[num_keys+1]
 * and perm[nnz] = element indices grouped by key, ascending index within a
 * key (np.argsort(kind="stable"), compute.py:224).  counts_out optional
 * (int32[num_keys] histogram).  ws: fgl_stable_group_ws_bytes(num_keys). */
int64_t fgl_stable_group_ws_bytes(int64_t num_keys);
int fgl_stable_group(const int32_t* keys, int64_t nnz, int64_t num_keys, int64_t* indptr,
                     int32_t* perm, int32_t* counts_out, void* ws, int64_t ws_bytes, void* stream);
/* a_out[p] = a[perm[p]], b_out[p] = b[perm[p]] (either pair may be NULL). */
int fgl_gather_i32_f32(const int32_t* perm, int64_t n, const int32_t* a, const float* b,
                       int32_t* a_out, float* b_out, void* stream);

/* One model layer's block CSR (trainer._prepare_batch, trainer.py:165-179):
 * lt (non-decreasing, in [0,num_rows)) / ls (in [0,num_cols)) are the hop's
 * edge endpoints in the layer's row / column index spaces.  Outputs:
 * indptr[num_rows+1], w[nnz] (arch_gcn == 1: GCN 1/sqrt(indeg*outdeg) in fp64
 * -> f32, trainer.py:156-162; 0: GIN 1.0; 2: SAGE mean 1/indeg in fp64 -> f32,
 * the GraphSAGE extension of SURVEY 8(c)), and the stable transpose
 * t_indptr[num_cols+1], t_col[nnz] (= lt), t_w[nnz] (compute.py:233-239).
 * t_indptr = t_col = t_w = NULL skips the transpose (model layer 0: the input
 * features need no gradient, so the backward never aggregates through it). */
int64_t fgl_prepare_layer_ws_bytes(int64_t nnz, int64_t num_rows, int64_t num_cols);
int fgl_prepare_layer(const int32_t* lt, const int32_t* ls, int64_t nnz, int64_t num_rows,
                      int64_t num_cols, int32_t arch_gcn, int64_t* indptr, float* w,
                      int64_t* t_indptr, int32_t* t_col, float* t_w, void* ws, int64_t ws_bytes,
                      void* stream);

/* --------------------------------------------------- depth layout ---- */
/* Depth-major window rows for the all-rows layouts (GIN / GraphSAGE,
 * trainer.py:182-195): rewrites a window sampled by fgl_sample_window (its
 * counts vector, frontier lists, and the `all` bitmap + word prefix of its
 * workspace, offsets from fgl_sample_ws_bitmaps) so that each batch's unique
 * rows are ordered by (depth, node id), depth = first hop whose frontier
 * holds the node (seeds 0, last-hop-only sources H).  Every R_i (rows model
 * layer i needs) is then a prefix of the batch's block.  Rewrites
 * unique_nodes, tgt_row / src_row (either may be NULL), seed_rows; writes
 * row_map[old window row] = new row and depth_cnt[b * (H + 1) + h] (int64).
 * No host synchronisation. */
int64_t fgl_depth_relayout_ws_bytes(int64_t unique_cap);
int fgl_depth_relayout(const int64_t* counts, int32_t H, int32_t nb, const int32_t* frontier,
                       int64_t frontier_stride, const uint32_t* bm_all, const int32_t* wprefix, int64_t words,
                       int32_t* unique_nodes, int64_t unique_cap, int32_t* tgt_row, int32_t* src_row,
                       int32_t* seed_rows, int64_t num_seeds, int32_t* row_map, int64_t* depth_cnt, void* ws,
                       int64_t ws_bytes, void* stream);
/* Y[r] += X[r] for r < nrows (one rounded add per element). */
int fgl_add_rows(float* Y, int64_t ldy, const float* X, int64_t ldx, int64_t nrows, int32_t d, void* stream);

/* ------------------------------------------------------- fused layers ---- */
/* fgl_prepare_layer for targets grouped but not ascending (depth-major rows
 * of fgl_depth_relayout): stable grouping by target (compute.py:219-230)
 * first; col_out receives the forward CSR's columns. */
int64_t fgl_prepare_layer_grouped_ws_bytes(int64_t nnz, int64_t num_rows, int64_t num_cols);
int fgl_prepare_layer_grouped(const int32_t* lt, const int32_t* ls, int64_t nnz, int64_t num_rows,
                              int64_t num_cols, int32_t arch, int64_t* indptr, int32_t* col_out, float* w,
                              int64_t* t_indptr, int32_t* t_col, float* t_w, void* ws, int64_t ws_bytes,
                              void* stream);

/* ------------------------------------------------------------- compute ---- */
/* Memory-Aware CSR aggregation (compute.py:115-195):
 * Y[r] = sum_{e in [indptr[r], indptr[r+1])} w[e] * X[col[e] - col_base]
 * (+ self_x[r] when self_x != NULL, the GIN self term), fp32, CSR order, no
 * FMA -- bit-identical to the reference.  Leading dims multiples of 4,
 * feature pointers 16-byte aligned, d <= 1024. */
int fgl_spmm(const int64_t* indptr, const int32_t* col, const float* w, int64_t num_rows,
             int64_t col_base, const float* X, int64_t ldx, const float* self_x, int64_t ld_self,
             float* Y, int64_t ldy, int32_t d, void* stream);

/* fgl_spmm with the source rows addressed through an id map: row c of X is
 * X + x_ids[c] * ldx (c = col[e] - col_base) and, with add_self, output row r
 * adds the root term X[x_ids[self_base + r]] -- the GIN / GraphSAGE layer-0
 * aggregation straight from the HBM feature table (replaces x0 =
 * feats[unique_nodes], trainer.py:315, followed by compute.aggregate_forward,
 * compute.py:115-185, + the root term of trainer.py:189-190).  d in 33..128. */
int fgl_spmm_ids(const int64_t* indptr, const int32_t* col, const float* w, int64_t num_rows, int64_t col_base,
                 const float* X, int64_t ldx, const int32_t* x_ids, int64_t self_base, int32_t add_self, float* Y,
                 int64_t ldy, int32_t d, void* stream);

/* The layer-0 aggregation of the trainer: fgl_spmm over the sampled block
 * graph (rows of <= max_row_len <= 16 edges, the last hop's fanout) gathering
 * straight from the HBM feature table X [x_rows, ldx], ldx <= 256.  No self
 * term.  Same kernels and results as fgl_spmm (compute.py:115-185); its own
 * entry point so the stage profile (fgl_profile id 2) can tell it apart. */
int fgl_spmm_gather(const int64_t* indptr, const int32_t* col, const float* w, int64_t num_rows,
                    int64_t col_base, const float* X, int64_t ldx, int64_t x_rows, float* Y, int64_t ldy,
                    int32_t d, int32_t max_row_len, void* stream);

/* SM budget of the tensor-core dense kernels (process-wide; 0 = every SM,
 * the default).  Their CTAs are persistent, one per SM; the pipelined
 * trainer runs them beside three other streams and caps them at half the SMs
 * so the sampling / aggregation kernels keep SMs (Pipeline(dense_ctas=74):
 * 2.21 -> 2.17 ms per products window, a standalone layer-0 forward takes
 * 29 -> 48 us). */
int fgl_set_dense_ctas(int32_t ctas);

/* Z = act(H @ W + b), W row-major [din, dout] (compute.py:198-216). */
int fgl_dense_fwd(const float* H, int64_t ldh, int64_t n, int32_t din, const float* W,
                  const float* b, int32_t dout, float* Z, int64_t ldz, int32_t relu, void* stream);

/* dZ = dX * (Xout > 0) (Xout NULL: no mask), dW = H^T dZ, db = colsum(dZ),
 * dH = dZ W^T (dH may be NULL) -- trainer.py:212-228.  Deterministic. */
int64_t fgl_dense_bwd_ws_bytes(int32_t din, int32_t dout);
int fgl_dense_bwd(const float* H, int64_t ldh, int64_t n, int32_t din, const float* W,
                  int32_t dout, const float* dX, int64_t lddx, const float* Xout, int64_t ldxo,
                  float* dW, float* db, float* dH, int64_t lddh, void* ws, int64_t ws_bytes,
                  void* stream);

/* fp64 softmax cross entropy over the B seed rows of logits (trainer.py:198-209):
 * row r_i = rows[i] - row_base, label y_i = labels[seed_ids[i]] (or labels[i]
 * when seed_ids is NULL); dlogits[r_i] = (softmax - onehot(y_i)) / B as f32;
 * *loss_sum = sum_i -log(p_i + 1e-30) (device double; mean = loss_sum / B). */
/* dH = (dX * (Xout > 0)) W^T alone (the dgrad half of fgl_dense_bwd,
 * trainer.py:212-228), so the trainer can run a layer's weight gradient on a
 * second stream while the backward chain continues. */
int fgl_dense_dgrad(const float* dX, int64_t lddx, const float* Xout, int64_t ldxo, int64_t n, const float* W,
                    int32_t din, int32_t dout, float* dH, int64_t lddh, void* stream);

/* CUDA-graph replay of a per-batch chain: begin a
 * thread-local capture on `stream`; end it and launch it through a
 * caller-owned executable-graph handle (cudaGraphExecUpdate when the topology
 * matches, else a fresh instantiation); or abort it (the caller then runs the
 * work eagerly).  A handle belongs to the device current at fgl_exec_create
 * and is rejected on any other.  fgl_capture_stats: process-wide {graph
 * launches, updates, instantiations}. */
typedef struct fgl_exec fgl_exec;
int fgl_exec_create(fgl_exec** out);
int fgl_exec_destroy(fgl_exec* h);
int fgl_capture_begin(void* stream);
int fgl_capture_end_launch(fgl_exec* h, void* stream);
int fgl_capture_abort(void* stream);
int fgl_capture_stats(int64_t* out3);

/* Events that order work across captured graphs: recorded / waited on with
 * cudaEventRecordExternal / cudaEventWaitExternal, so inside a capture they
 * become event-record / event-wait nodes (the window's chain graph waits for
 * each batch's layer-0 aggregation inside the prepare graph, not for its
 * end); outside a capture they are a plain record / wait. */
int fgl_event_create(void** out);
int fgl_event_destroy(void* ev);
int fgl_event_record_ext(void* ev, void* stream);
int fgl_stream_wait_ext(void* stream, void* ev);

int64_t fgl_softmax_xent_ws_bytes(void);
int fgl_softmax_xent(const float* logits, int64_t ldl, const int32_t* rows, int64_t row_base,
                     const int32_t* seed_ids, const int64_t* labels, int64_t B, int32_t C,
                     float* dlogits, int64_t ldd, double* loss_sum, void* ws, int64_t ws_bytes,
                     void* stream);

/* Top model layer of the compact GCN batch in one launch (its rows are the
 * seeds): logits = H W + b, fp64 softmax cross entropy (trainer.py:198-209),
 * dH = dY W^T, and per-CTA partials of dW, db and the loss; din <= 64, C <= 192.
 * agg_indptr != NULL: H is not read but gathered in-kernel as A X with
 * X = H (ldh), the layer's CSR (agg_indptr over the same rows, agg_col -
 * agg_col_base, agg_w), fgl_spmm arithmetic (bit-identical).
 * With reduce_stream == NULL (or == chain_stream) the partials are reduced
 * right after on chain_stream; otherwise the caller orders
 * fgl_top_layer_reduce on reduce_stream after the chain stream (off the
 * critical path). */
int64_t fgl_top_layer_ws_bytes(int64_t B, int32_t din, int32_t C);
int fgl_top_layer(const float* H, int64_t ldh, const int32_t* rows, int64_t row_base, const int32_t* seed_ids,
                  const int64_t* labels, int64_t B, int32_t din, int32_t C, const float* W, const float* b,
                  float* dH, int64_t lddh, float* dW, float* db, double* loss_sum, void* ws, int64_t ws_bytes,
                  const int64_t* agg_indptr, const int32_t* agg_col, const float* agg_w, int64_t agg_col_base,
                  void* chain_stream, void* reduce_stream);
int fgl_top_layer_reduce(int64_t B, int32_t din, int32_t C, float* dW, float* db, double* loss_sum, void* ws,
                         void* stream);

/* params -= f32(lr) * grads, separately rounded (trainer.py:321-323). */
int fgl_sgd(float* params, const float* grads, int64_t n, float lr, void* stream);

/* Y[r, :d] = act(rowval) (rowval NULL: zeros) for r < nrows. */
int fgl_fill_rows(float* Y, int64_t ldy, int64_t nrows, int32_t d, const float* rowval,
                  int32_t relu, void* stream);

/* --------------------------------------------------------------- idmap ---- */
/* Fused-Map ID table (idmap.py:88-117, :175-233) for arbitrary uint64 IDs:
 * keys/values uint64[capacity] receive the reference's single-worker state --
 * SENTINEL (all ones) in empty slots, local IDs in first-seen order, the slot
 * layout of sequential linear probing from hash(gid) = gid % capacity
 * (mod_hash) or (gid * 0x9E3779B97F4A7C15) >> shift.  Deterministic.
 * status2 (device int64[2]): [0] = status (FGL_E_CAPACITY when the table is
 * full), [1] = number of distinct IDs.  ws: fgl_idmap_ws_bytes(n, capacity). */
int64_t fgl_idmap_ws_bytes(int64_t n, int64_t capacity);
int fgl_idmap_build(const uint64_t* ids, int64_t n, int32_t mod_hash, int64_t capacity,
                    int32_t shift, uint64_t* keys, uint64_t* values, int64_t* status2,
                    void* ws, int64_t ws_bytes, void* stream);
/* out[i] = local ID of ids[i], or SENTINEL on a miss (idmap.py:154-172);
 * *first_miss (device, optional) = smallest missing index, or 0x7f7f7f7f7f7f7f7f. */
int fgl_idmap_lookup(const uint64_t* keys, const uint64_t* values, int64_t capacity,
                     int32_t mod_hash, int32_t shift, const uint64_t* ids, int64_t n,
                     uint64_t* out, int64_t* first_miss, void* stream);

/* -------------------------------------------------------------- loader ---- */
/* Where fgl_sample_window leaves the per-batch unique-node bitmaps in its
 * workspace: out[0] = byte offset of the bitmaps (batch b at word b*words),
 * out[1] = byte offset of the int32 per-word exclusive popcount prefixes
 * (window rows), out[2] = words per batch. */
int fgl_sample_ws_bitmaps(int64_t num_nodes, int32_t num_batches, int64_t frontier_stride,
                          int64_t unique_cap, int64_t* out);

/* |U_i ∩ U_j| for all pairs of a window's batches (2 <= nb <= 16) from their
 * bitmaps: out_pairs uint64[120], pair (i<j) at i*16 - i*(i+1)/2 + (j-i-1).
 * The match degree of schedule.py:68-89 is count / min(|U_i|, |U_j|). */
int fgl_match_counts(const uint32_t* bitmaps, int64_t words, int32_t num_batches,
                     uint64_t* out_pairs, void* stream);

/* Node bitmaps of nsets ID sets (set s = ids[offsets[s]..offsets[s+1]), IDs in
 * [0, 32*words)): bitmaps uint32[nsets*words], cleared then marked. */
int fgl_mark_bitmaps(const int32_t* ids, const int64_t* offsets, int32_t nsets, int64_t total,
                     int64_t words, uint32_t* bitmaps, void* stream);
/* hit[i] = 1 if ids[i] is set in bitmap (schedule.compute_transition overlap test). */
int fgl_bitmap_test(const int32_t* ids, int64_t n, const uint32_t* bitmap, int8_t* hit, void* stream);

/* x0 rows of one batch (trainer.py:315): out[r] = feats[ids[r]] (feats may be
 * device memory or mapped pinned host memory), except that rows whose ID is
 * set in prev_bitmap (the previously executed batch, Match reuse) are copied
 * from prev_x[rank] where rank = prev_prefix[word] + popc(...) - prev_base.
 * *loaded (device uint64, accumulated) counts rows read from feats. */
int fgl_gather_rows(const float* feats, int64_t ldf, int32_t d, const int32_t* ids, int64_t n,
                    const uint32_t* prev_bitmap, const int32_t* prev_prefix, int64_t prev_base,
                    const float* prev_x, int64_t ldp, float* out, int64_t ldo, uint64_t* loaded,
                    void* stream);
/* fgl_gather_rows with a static HBM feature cache (memsim.py:110-186,
 * static-degree policy): after the Match test, a node with cache_slot[g] >= 0
 * is copied from cache_x[cache_slot[g] * ldc] (HBM) instead of the store;
 * `hits` (optional) accumulates those rows, `loaded` the rows read from the
 * store. cache_slot has one int32 per graph node (-1 = not cached).
 * prev_row_map (optional): the previous batch's rows are in depth-major order
 * (fgl_depth_relayout); its bitmap rank r maps to row prev_row_map[r]. */
int fgl_gather_rows_cached(const float* feats, int64_t ldf, int32_t d, const int32_t* ids, int64_t n,
                           const uint32_t* prev_bitmap, const int32_t* prev_prefix, int64_t prev_base,
                           const float* prev_x, int64_t ldp, const int32_t* prev_row_map,
                           const int32_t* cache_slot, const float* cache_x, int64_t ldc, float* out, int64_t ldo,
                           uint64_t* loaded, uint64_t* hits, void* stream);

/* Page-lock and map a caller-allocated host feature table (e.g. one shared
 * by every rank of a node); *dev_ptr = its device address for
 * the loader.  Synchronous.  fgl_host_unregister undoes it. */
int fgl_host_register(void* host, int64_t bytes, void** dev_ptr);
int fgl_host_unregister(void* host);

#ifdef __cplusplus
}
#endif
#endif /* FASTGL_B200_H */
