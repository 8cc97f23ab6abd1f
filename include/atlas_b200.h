/*
 * atlas_b200.h — C-ABI of the B200 broadcast layer engine (libatlas_b200.so).
 *
 * Plain pointers and sizes only; no torch or C++ types cross this line.
 * Each entry point replaces one reference interface of the `oocgnn`
 * package (paths relative to /root/reference/pkg/src):
 *
 *   atlas_graph_create      TopologySource + in-degrees as one layer sees
 *                           them (oocgnn/chunks.py:51-78,
 *                           oocgnn/storage.py:205-250); builds the
 *                           destination-major (CSC) view on the device
 *   atlas_layer_create      init_layer (oocgnn/orchestrator.py:93-145):
 *                           pending counters, state table, hot-slot budget,
 *                           eviction policy, sub_batch / evict_batch
 *   atlas_chunk_submit      process_chunk (oocgnn/orchestrator.py:216-299)
 *                           for one caller-supplied source chunk
 *   atlas_chunk_graduated   the sink hand-off of process_chunk
 *                           (oocgnn/orchestrator.py:148-150): ids + rows of
 *                           every vertex that graduated in the last chunk
 *   atlas_layer_run_resident  one whole layer over a resident input with the
 *                           reference chunk plan (oocgnn/runtime.py:114-220
 *                           minus the disk stages): scatter-aggregate +
 *                           pending counters + min-pending control plane
 *   atlas_transform         MatmulBackend.apply + activation
 *                           (oocgnn/compute.py:25-97)
 *   atlas_layer_finish      finalize_layer (oocgnn/orchestrator.py:302-323)
 *
 * Status codes map 1:1 onto the reference's exception classes
 * (oocgnn/errors.py:8-78); the Python shim raises them.
 * Threading: one handle per GPU, single owner.
 */
#ifndef ATLAS_B200_H
#define ATLAS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ATLAS_ABI_VERSION 1

#if defined(__GNUC__)
#define ATLAS_API __attribute__((visibility("default")))
#else
#define ATLAS_API
#endif

enum {
  ATLAS_OK = 0,
  ATLAS_ECONFIG = -1,      /* ConfigError */
  ATLAS_ECONSISTENCY = -2, /* ConsistencyError */
  ATLAS_ESTATE = -3,       /* StateTransitionError */
  ATLAS_EBUDGET = -4,      /* BudgetError */
  ATLAS_EINCOMPLETE = -5,  /* IncompleteLayerError */
  ATLAS_ECOVERAGE = -6,    /* CoverageError */
  ATLAS_EFORMAT = -7,      /* FormatError */
  ATLAS_EDEVICE = -8,      /* CUDA/NCCL failure (DeviceError) */
  ATLAS_EINVARIANT = -9,   /* InvariantError */
  ATLAS_EMAGIC = -10,      /* BadMagicError (a FormatError) */
  ATLAS_ETRUNCATED = -11,  /* TruncatedFileError (a FormatError) */
  ATLAS_EVERSION = -12     /* VersionMismatchError (a FormatError) */
};

/* ModelKind (oocgnn/storage.py:498) + GAT, which the reference lacks
 * (semantics in oracle/gat.py / SURVEY.md A.5) */
enum { ATLAS_GCN = 0, ATLAS_SAGE = 1, ATLAS_GIN = 2, ATLAS_GAT = 3 };
enum { ATLAS_F32 = 0, ATLAS_F16 = 1, ATLAS_BF16 = 2 };         /* row dtype */
enum { ATLAS_MINPEND = 0, ATLAS_LRU = 1, ATLAS_RND = 2 };      /* policy */
enum { ATLAS_BACKEND_STABLE = 0, ATLAS_BACKEND_TCGEN05 = 1 };  /* transform */
enum { ATLAS_LOG_VICTIMS = 0, ATLAS_LOG_RELOADS = 1, ATLAS_LOG_GRADUATED = 2 };

typedef struct atlas_graph atlas_graph;
typedef struct atlas_layer atlas_layer;

typedef struct {
  int64_t num_vertices;  /* V of the whole graph */
  int64_t dst_lo;        /* destination range owned by this handle: */
  int64_t dst_hi;        /*   partition_ranges(V, G)[rank] */
  int32_t model;         /* ATLAS_GCN / ATLAS_SAGE / ATLAS_GIN */
  float gin_epsilon;
  int64_t embed_dim;     /* width of streamed rows */
  int64_t agg_dim;       /* aggregation record width (2*embed for SAGE) */
  int64_t slot_count;    /* hot slots of this GPU (MemoryBudget.slot_count) */
  int64_t evict_batch;   /* 0 -> max(1, slot_count / 100) */
  int32_t policy;        /* ATLAS_MINPEND / ATLAS_LRU / ATLAS_RND */
  int32_t record_log;    /* keep victim / reload / graduation logs */
  uint64_t rnd_state[4]; /* numpy PCG64 (state_hi, state_lo, inc_hi, inc_lo) */
  int32_t device;
  int32_t force_exact;   /* 1: never take the parallel eviction-free path */
} atlas_layer_desc;

typedef struct {
  int64_t messages;
  int64_t evictions;
  int64_t reloads;
  int64_t unique_reloads;
  int64_t admissions;
  int64_t graduations;
  int64_t hot_peak;
  int64_t hot_slot_count;
  int64_t chunks;          /* chunks seen */
  int64_t span_count;      /* vertices with a first step */
  int64_t span_sum;        /* exact sum of (last - first) over them */
  int64_t span_q_lo;       /* order statistics at floor / floor+1 of */
  int64_t span_q_hi;       /*   (span_count - 1) * 0.99 (np.percentile) */
  int64_t incomplete;      /* vertices not COMPLETED */
  int64_t first_incomplete[16];
  int64_t cold_bytes_read;
  int64_t cold_bytes_written;
  int32_t fast_path;       /* 1: control plane proved eviction-free */
  int32_t pad_;
} atlas_layer_metrics;

ATLAS_API const char* atlas_last_error(void);
ATLAS_API int atlas_abi_version(void);

/* ---- topology ------------------------------------------------------- */
ATLAS_API int atlas_graph_create(int32_t device, int64_t num_vertices,
                       int64_t num_edges, const int64_t* offsets_host,
                       const uint32_t* neighbors_host,
                       const uint32_t* in_degrees_host, int64_t dst_lo,
                       int64_t dst_hi, void* stream, atlas_graph** out);
/* re-upload a (new) CSR for the same destination range into the existing
 * device buffers and rebuild the CSC view; no allocation when the graph
 * has the same or a smaller size */
ATLAS_API int atlas_graph_update(atlas_graph* g, int64_t num_vertices,
                                 int64_t num_edges,
                                 const int64_t* offsets_host,
                                 const uint32_t* neighbors_host,
                                 const uint32_t* in_degrees_host,
                                 void* stream);
ATLAS_API void atlas_graph_destroy(atlas_graph* g);
/* device pointers of the CSC view (csc_ptr int64[nloc+1], csc_src u32) */
ATLAS_API int atlas_graph_csc(const atlas_graph* g, const int64_t** csc_ptr,
                    const uint32_t** csc_src, int64_t* num_local_edges);

/* ---- one layer ------------------------------------------------------ */
ATLAS_API int atlas_layer_create(const atlas_layer_desc* desc,
                       const uint32_t* in_degrees_host, void* stream,
                       atlas_layer** out);
ATLAS_API void atlas_layer_destroy(atlas_layer* layer);
/* re-arm a layer for a new pass with the same descriptor (init_layer
 * again) without reallocating its device memory */
ATLAS_API int atlas_layer_reset(atlas_layer* layer, void* stream);

/* atlas_layer_reset after a topology refresh (atlas_graph_update): the
 * layer takes its in-degrees from the graph's device copy (no host trip),
 * then re-arms like init_layer */
ATLAS_API int atlas_layer_bind_graph(atlas_layer* layer,
                                     const atlas_graph* graph, void* stream);

/* process_chunk: rows (n x embed_dim, dtype) and the chunk CSR slice are
 * HOST pointers (pinned or pageable); the library stages them to HBM. */
ATLAS_API int atlas_chunk_submit(atlas_layer* layer, int64_t start, int64_t end,
                       const void* rows_host, int32_t dtype,
                       const int64_t* local_offsets_host,
                       const int64_t* neighbors_host, int64_t num_edges,
                       void* stream);
/* graduations of the last submitted chunk, in reference order.
 * ids/rows/batch_len may be NULL to query counts only. */
ATLAS_API int atlas_chunk_graduated(atlas_layer* layer, int64_t* ids, float* rows,
                          int64_t cap, int64_t* count, int64_t* batch_len,
                          int64_t batch_cap, int64_t* num_batches);

/* whole layer over a resident input x (device pointer, V rows of
 * embed_dim, leading dimension ldx) with the reference chunk plan of
 * chunk_rows rows per chunk. Aggregation records land in the layer's
 * device accumulator (atlas_layer_accumulator). input_flag (device int,
 * may be NULL) is the extremes flag atlas_transform wrote for x; NULL makes
 * the layer scan x itself. */
ATLAS_API int atlas_layer_run_resident(atlas_layer* layer, const atlas_graph* graph,
                             const void* x_dev, int32_t dtype, int64_t ldx,
                             int64_t chunk_rows, const int32_t* input_flag,
                             void* stream);
/* same layer pass with the device records bounded: destinations
 * [v0, v0 + block_rows) aggregate into a block_rows x agg_dim record buffer
 * and are transformed (backend ATLAS_BACKEND_*, W n x agg_dim, bias n,
 * activation relu) into rows v0.. of y before the next block reuses the
 * buffer -- the reference's "graduated batches are transformed and leave
 * the hot store" (oocgnn/compute.py:125-205, memstore.py:479-494), so the
 * hot budget, not the graph, bounds record memory. Records and outputs are
 * bit-identical to atlas_layer_run_resident + atlas_transform. out_flag
 * (device int, may be NULL) receives the output's extremes flag. */
ATLAS_API int atlas_layer_run_blocked(atlas_layer* layer,
                                      const atlas_graph* graph,
                                      const void* x_dev, int32_t dtype,
                                      int64_t ldx, int64_t chunk_rows,
                                      const int32_t* input_flag,
                                      int32_t backend, const float* w,
                                      const float* bias, int64_t n,
                                      int32_t relu, void* y, int32_t y_dtype,
                                      int64_t ldy, int32_t* out_flag,
                                      int64_t block_rows, void* stream);
/* bytes of device record storage the layer holds (its accumulator) */
ATLAS_API int atlas_layer_record_bytes(const atlas_layer* layer,
                                       int64_t* bytes);
/* same layer pass, but the input stays in (pinned) HOST memory: it is
 * streamed to HBM in tiles of tile_rows rows, double-buffered on a side
 * copy stream, and every tile is aggregated as soon as it lands (SURVEY.md
 * kernel K1 + K3). Records are bit-identical to the resident pass. */
ATLAS_API int atlas_layer_run_streamed(atlas_layer* layer,
                                       const atlas_graph* graph,
                                       const void* x_host, int32_t dtype,
                                       int64_t ldx, int64_t tile_rows,
                                       int64_t chunk_rows, void* stream);
/* whole-layer pass over a DEVICE input that arrives in pieces: rows
 * [bounds[t], bounds[t+1]) of x (ldx elements per row) become valid when
 * the CUDA event ready[t] completes (NULL entries: already valid). Pieces
 * tile [0, V) in ascending order -- the multi-GPU exchange (SURVEY.md §8e:
 * each source piece broadcast by its owner, rank order) -- and each is
 * aggregated as soon as it lands, so the exchange overlaps the
 * aggregation. Records are bit-identical to atlas_layer_run_resident. */
ATLAS_API int atlas_layer_run_pieces(atlas_layer* layer,
                                     const atlas_graph* graph, const void* x,
                                     int32_t dtype, int64_t ldx,
                                     const int64_t* bounds, int32_t npieces,
                                     void* const* ready, int64_t chunk_rows,
                                     void* stream);
/* transform-first layer pass (tcgen05 backend, out_dim < aggregated
 * width): z = h . W_z^T was computed by atlas_transform_typed for every
 * source (V rows, ldz); the pass runs the layer's control plane on the
 * reference chunk plan (chunk_rows rows, as for the layer's own input) and
 * aggregates the first d columns of z with data_model's rule (ATLAS_GCN =
 * mean, for GCN and SAGE; ATLAS_GIN = sum + (1+eps) self), then writes
 * y[v] = act(agg + self_rows[v] + b)[:n] (self_rows: SAGE's h_v . W2^T for
 * the range's destinations, row v = local destination v; NULL otherwise).
 * By linearity this is the reference layer up to
 * floating-point order; no f32 records are kept. out_flag (may be NULL)
 * receives y's extremes flag. With y_host (pinned, ldy_host elements per
 * row) the output also goes to the host in host_slices destination slices,
 * each copied while the next one aggregates; the stream covers the copies. */
ATLAS_API int atlas_layer_run_fused(atlas_layer* layer,
                                    const atlas_graph* graph,
                                    const float* z_dev, int64_t ldz,
                                    int32_t data_model, int64_t d,
                                    int64_t chunk_rows,
                                    const int32_t* input_flag,
                                    const float* bias_dev,
                                    const float* self_rows_dev,
                                    int64_t ld_self, int64_t n,
                                    int32_t relu, void* y_dev,
                                    int32_t y_dtype, int64_t ldy,
                                    int32_t* out_flag, void* y_host,
                                    int64_t ldy_host, int32_t host_slices,
                                    void* stream);
ATLAS_API int atlas_layer_accumulator(atlas_layer* layer, float** acc_dev,
                            int64_t* ld);

/* y = act(x . W^T + b); x (rows x k, f32, ldx), W (n x k, f32), b (n).
 * extremes_flag (device int, may be NULL) is set to 1 iff some output is
 * non-finite or a nonzero below 2^-100 (then the next layer's exact
 * division takes its IEEE path); it spares that layer a scan of y. */
ATLAS_API int atlas_transform(int32_t backend, const float* x_dev, int64_t rows,
                    int64_t k, int64_t ldx, const float* w_dev,
                    const float* b_dev, int64_t n, int32_t relu, void* y_dev,
                    int32_t y_dtype, int64_t ldy, int32_t* extremes_flag,
                    void* stream);

/* atlas_transform with an f16/bf16 (or f32) input; 2-byte inputs need the
 * tcgen05 backend (they are exact in tf32, so 2 MMAs per k-step). GAT's
 * pass A (z = x . W_ext^T) uses it. */
ATLAS_API int atlas_transform_typed(int32_t backend, const void* x_dev,
                                    int32_t x_dtype, int64_t rows, int64_t k,
                                    int64_t ldx, const float* w_dev,
                                    const float* b_dev, int64_t n,
                                    int32_t relu, void* y_dev, int32_t y_dtype,
                                    int64_t ldy, int32_t* extremes_flag,
                                    void* stream);

/* GAT pass A with the attention score er fused into the epilogue:
 * y[:, 0:n] = x . W^T + b as atlas_transform_typed (tcgen05 backend,
 * register-split f32/bf16 or f16 kernels only, n <= 128), and
 * y[r, er_col + h] = sum_{c in head h} y[r, c] * er_w[c] for h < heads,
 * head h = columns [h*head_stride, (h+1)*head_stride), head_stride a
 * multiple of 16, heads <= 8. er_w (n, device) holds a_r[h] at head h's
 * columns (zero padding). It replaces the a_r^T W_h rows of W_ext, which
 * took n past 128 (128 + el + er = 136 for 4 x 32 heads) and so off the
 * fast kernels; pass B (gat_ring) recomputes el per edge and never reads
 * it. Returns ATLAS_ECONFIG when the shape needs another kernel. */
ATLAS_API int atlas_transform_er(int32_t backend, const void* x_dev,
                                 int32_t x_dtype, int64_t rows, int64_t k,
                                 int64_t ldx, const float* w_dev,
                                 const float* b_dev, int64_t n, void* y_dev,
                                 int32_t y_dtype, int64_t ldy,
                                 const float* er_w_dev, int32_t er_col,
                                 int32_t heads, int32_t head_stride,
                                 void* stream);

/* GAT layer pass B over a resident z_ext (device, V rows of ldz elements:
 * [z: head h at columns h*head_stride .. +head_dim | el (heads) at el_col |
 *  er (heads) at er_col]; head_stride = head_dim rounded up to 16 bytes):
 * the control plane of a layer created with model ATLAS_GAT (GCN rules:
 * pending = in-degree) on the reference chunk plan of chunk_rows rows, and
 * the edge-softmax aggregation of the range with bias, head concat (+ReLU)
 * or head mean fused, written to y (nloc x ldy). attn_l_dev (may be NULL):
 * a_l laid out like the z columns (heads x head_stride, zero pads); given
 * it, f32 z of <= 128 columns is aggregated moving only the z part of each source row, el_u = a_l . z_u
 * recomputed per edge (4 DRAM lines per edge instead of 5-6 when the z
 * rows start on 128-byte lines). No reference counterpart
 * (SPEC.md:8); oracle/gat.py defines the result. */
ATLAS_API int atlas_layer_run_gat(atlas_layer* layer, const atlas_graph* graph,
                                  const void* z_dev, int32_t z_dtype,
                                  int64_t ldz, int32_t heads,
                                  int32_t head_dim, int32_t head_stride,
                                  int32_t el_col, int32_t er_col,
                                  const float* bias_dev,
                                  int32_t mean_heads, int32_t relu,
                                  float negative_slope, void* y_dev,
                                  int32_t y_dtype, int64_t ldy,
                                  const float* attn_l_dev,
                                  int64_t chunk_rows, void* stream);

ATLAS_API int atlas_layer_finish(atlas_layer* layer, atlas_layer_metrics* out);
/* per-chunk reload and touched counters (for mean_reload_pct) */
ATLAS_API int atlas_layer_chunk_stats(atlas_layer* layer, int64_t* reloads,
                            int64_t* touched, int64_t cap, int64_t* count);
/* flattened log [len, v0, v1, ..., len, ...]; victims within an event are
 * ordered like PendingBucketHeap.pop_min (key, then arrival) */
ATLAS_API int atlas_layer_log(atlas_layer* layer, int32_t which, int64_t* out,
                    int64_t cap, int64_t* count);

/* copies of the per-vertex control state of the layer's range
 * (pending u32, lifecycle u8 0..3, first/last step int64); NULL skips */
ATLAS_API int atlas_layer_state(atlas_layer* layer, uint32_t* pending, uint8_t* state,
                      int64_t* first_step, int64_t* last_step);

/* device time (CUDA events on the launching stream) of the last
 * atlas_layer_run_resident: [0] scatter-aggregate kernel, [1] control
 * plane (walk + optional exact replay), in milliseconds */
ATLAS_API int atlas_layer_timing(atlas_layer* layer, float* ms, int32_t n);

/* greedy reordering (oocgnn/reorder.py:30-88): scores, the bit-exact
 * old->new permutation and the relabelled CSR (rows ascending), all on the
 * device; host in / host out. scores may be NULL. */
ATLAS_API int atlas_reorder(int32_t device, int64_t num_vertices,
                            int64_t num_edges, const int64_t* offsets,
                            const uint32_t* neighbors,
                            const uint32_t* in_degrees, int64_t* old_to_new,
                            int64_t* new_offsets, uint32_t* new_neighbors,
                            uint32_t* new_in_degrees, double* scores,
                            void* stream);

/* ---- layer-directory spill I/O (host only) -- */
/* read the ASPL spill files of a layer directory (oocgnn/storage.py:
 * 257-357; the reference reads them through SpillSet, oocgnn/chunks.py:
 * 103-201) into a dense row-major host buffer (num_vertices x dim, pinned
 * for the K1 streamer), files in parallel on `threads` host threads (0 =
 * all cores). Every id must arrive exactly once (ATLAS_ECOVERAGE
 * otherwise; delivery_out, may be NULL, receives the per-id counts like
 * the reference's delivery counters, oocgnn/chunks.py:145-147). */
ATLAS_API int atlas_spill_read(const char* const* paths, int32_t n_files,
                               int32_t dtype, int64_t dim,
                               int64_t num_vertices, void* rows_out,
                               uint16_t* delivery_out, int32_t threads,
                               int64_t* bytes_read);
/* the same layer directory read straight into DEVICE memory rows_dev
 * (num_vertices x dim, dense): every run of consecutive ids is one
 * GPUDirect Storage transfer (cuFileRead, storage -> HBM) when the cuFile
 * driver opens, else it streams through per-thread pinned bounce buffers
 * on the copy engines; *used_gds (may be NULL) says which. Same
 * validation, coverage and byte accounting as atlas_spill_read.
 * rows_dev == NULL validates the directory only (no device work). */
ATLAS_API int atlas_spill_read_device(const char* const* paths,
                                      int32_t n_files, int32_t dtype,
                                      int64_t dim, int64_t num_vertices,
                                      void* rows_dev, uint16_t* delivery_out,
                                      int32_t threads, int64_t* bytes_read,
                                      int32_t* used_gds);
/* "cuFile" or "bounce: <why GDS is unavailable>" */
ATLAS_API const char* atlas_gds_status(void);
/* write rows [id_lo, id_hi) of a dense host matrix (ld elements per row,
 * row 0 = id_lo) as one partition directory's spill files spill_0..k of
 * spill_rows rows each plus its manifest -- the bytes
 * oocgnn/storage.py:write_matrix_as_layer / writer.py produce */
ATLAS_API int atlas_spill_write(const char* part_dir, const void* rows,
                                int32_t dtype, int64_t dim, int64_t ld,
                                int64_t id_lo, int64_t id_hi,
                                int64_t spill_rows, int32_t threads,
                                int64_t* bytes_written);

/* Writes one output partition as the reference's writer lays it out
 * (oocgnn/writer.py:40-115: partition buffers filled in graduation order,
 * each flush sorted by id): spill f holds ids[spill_start[f] ..
 * spill_start[f+1]) (ascending), rows gathered from the dense matrix
 * `rows` (row of id v at v * ld elements), plus the manifest. */
ATLAS_API int atlas_spill_write_runs(const char* part_dir, const void* rows,
                                     int32_t dtype, int64_t dim, int64_t ld,
                                     const int64_t* ids,
                                     const int64_t* spill_start,
                                     int64_t nspills, int32_t threads,
                                     int64_t* bytes_written);

/* Gather-pattern replay (ablation criterion 11): rows a destination-major
 * gather engine loads in one layer through an LRU cache of cache_rows rows
 * fetched in block_rows blocks (0 cache rows: every touch loads). Replaces
 * oocgnn/bench.py:282-305 simulate_gather_rows; exact LRU via reuse
 * distances. Host-only. */
ATLAS_API int atlas_gather_replay(int64_t num_vertices, int64_t num_edges,
                                  const int64_t* offsets,
                                  const uint32_t* neighbors,
                                  int64_t cache_rows, int64_t block_rows,
                                  int64_t* rows_loaded);

/* number of kernels this library launched since load (evidence counter) */
ATLAS_API int64_t atlas_kernel_launches(void);

#ifdef __cplusplus
}
#endif
#endif /* ATLAS_B200_H */
