// Handle layouts and launcher declarations shared by the .cu files.
#pragma once

#include <utility>
#include <vector>

#include "common.cuh"

namespace atlas {
struct SweepWs;
void free_sweep_ws(SweepWs* w);
}  // namespace atlas

struct atlas_graph {
  int device = 0;
  int64_t V = 0;        // whole-graph vertices
  int64_t E = 0;        // whole-graph edges
  int64_t lo = 0, hi = 0;
  int64_t nloc = 0;     // hi - lo
  int64_t eloc = 0;     // edges with dst in [lo, hi)
  atlas::DevBuf<int64_t> offsets;   // CSR offsets of the whole graph (V+1)
  atlas::DevBuf<int64_t> csc_ptr;   // nloc + 1
  atlas::DevBuf<uint32_t> csc_src;  // eloc, source id (global), ascending per dst
  atlas::DevBuf<uint32_t> csc_eid;  // eloc, CSR edge index of the entry
  atlas::DevBuf<uint32_t> indeg;    // nloc
  mutable atlas::DevBuf<int> scan_flag;  // input needs the guarded division
  mutable atlas::DevBuf<unsigned long long> work;  // ring kernel scheduler
  mutable const int32_t* known_flag = nullptr;  // producer-supplied flag
  // (R * 4 + model) -> largest chunk pass; cleared by atlas_graph_update
  mutable std::vector<std::pair<int64_t, int64_t>> maxpass_cache;
  std::vector<int64_t> offsets_host;  // host copy of the CSR offsets
  // CSC build workspaces (kept for atlas_graph_update)
  atlas::DevBuf<uint32_t> ws_nbrs, ws_src, ws_keys, ws_vals, ws_keys_out,
      ws_sel;
  atlas::DevBuf<int64_t> ws_nsel;
  atlas::DevBuf<uint8_t> ws_tmp;
  // deferred consistency check of the last CSC build (in-degrees vs
  // adjacency): the device total lands in chk, verified by verify_graph
  mutable atlas::PinnedBuf<int64_t> chk;
  mutable cudaEvent_t chk_ev = nullptr;
  mutable bool chk_pending = false;
  int64_t chk_expect = 0;
  // exact-replay workspaces (control.cu / sweep.cu), sized by the graph and
  // shared by its layers: replays run one at a time, host-synchronously
  mutable atlas::SweepWs* sweep_ws = nullptr;
  uint64_t generation = 0;  // bumped by every (re)load of the topology
  ~atlas_graph() {
    if (chk_ev) cudaEventDestroy(chk_ev);
    atlas::free_sweep_ws(sweep_ws);
  }
};

namespace atlas {

// Exact single-CTA control engine state (control.cu). Plain device arrays.
struct EngineState {
  // per local vertex
  uint32_t* pending;
  uint8_t* state;
  uint32_t* seq;
  int32_t* slot_of;
  uint8_t* unique_reloaded;
  // hot set
  int32_t* hot_list;   // slot -> local vertex or -1
  uint64_t* slot_key;  // slot -> its vertex's eviction key, or ~0 if free
  int32_t* free_stack; // LIFO of free slots
  // scratch (size >= slot_count + 1024)
  int32_t* scratch_a;
  int32_t* scratch_b;
  // RND policy
  int32_t* rnd_members;
  int32_t* rnd_pos;
  // logs (record_log): victims as (vertex, key) pairs, others as vertices
  int64_t* log_victims;  // pairs
  int64_t* log_reloads;
  int64_t* log_grad;
  int64_t log_cap;
  // current-chunk graduation list (operator path)
  int32_t* chunk_grad;
  int64_t* chunk_grad_batches;
  // scalars live in EngineScalars (device memory)
};

struct EngineScalars {
  int64_t free_top;
  int64_t hot_pop;
  uint64_t seq_ctr;
  int64_t messages, evictions, reloads, admissions, graduations, hot_peak;
  int64_t log_victims_n, log_reloads_n, log_grad_n;
  int64_t chunk_grad_n, chunk_grad_batches_n;
  int64_t chunk_index;  // chunks processed so far
  uint64_t rng_state_hi, rng_state_lo, rng_inc_hi, rng_inc_lo;
  int32_t rng_has32;
  uint32_t rng_u32;
  int64_t rnd_n;
  int32_t err;          // ATLAS_* code
  int64_t err_info[4];
};

// Victim selection is a grid job: CTA 0 (the state machine) posts a scan
// of the hot list and helper CTAs of the same cooperative launch share it.
struct GridSync {
  unsigned job;   // posted job count (CTA 0)
  unsigned done;  // helper completions, cumulative
  int32_t type, byte;
  uint64_t prefix, mask;
  uint64_t anybits;
  uint32_t hist[256];
  int32_t nv;
  // sub-batch jobs over pass elements [lo, lo + n) (engine.cu pass_slice)
  int32_t pkind;
  const void* pptr;  // runs (EDGEPASS) or vertex list (PREPASS)
  int64_t pfirst;    // SELFPASS first vertex
  int64_t lo, n;
  int64_t base;      // admit / release: free-stack top; deliver: seq base
  int64_t base2;     // release: chunk_grad fill
  int32_t flag;      // admit: reload
  const int32_t* list;
  int32_t* out;
  int64_t slice;     // elements per CTA slice of an ordered compaction
  unsigned long long sum[2];
  int64_t cnt[64][2];  // per-CTA counts (<= 64 CTAs)
};

struct EngineConfig {
  int64_t lo, hi, nloc;
  int64_t slot_count, evict_batch, sub_batch;
  int32_t model, policy, record_log;
};

// Workspaces of the sweep replay (sweep.cu), grow-only across layers.
struct SweepWs {
  DevBuf<uint32_t> zr, tmp_u32, el_v, el_cnt, el_sub,
      sv, se, ent_sub, ent_next, boff, head, fresh, grad, cold, cold_out,
      victims, flags;
  DevBuf<uint8_t> cub_tmp, coop, flags8;
  DevBuf<unsigned long long> cs, P, lastP, count, pk, svk, sk64;
  DevBuf<int64_t> eoff, soff, chunk64, out;
  // run materialisation (control.cu exact_replay)
  DevBuf<uint64_t> at_pos, runs;
  DevBuf<int64_t> nsel, d_off, d_bounds;
  DevBuf<uint8_t> sel_tmp;
  // the static schedule (element stream, heap lists, per sub-batch fresh /
  // graduating counts) depends only on the topology, the chunk plan, the
  // model, the sub-batch size and the policy: layers with the same key
  // (e.g. layers 2 and 3 of a [1024,128,128,..] model) reuse it
  bool valid = false;
  uint64_t key_gen = 0;
  int64_t key_R = 0, key_sb = 0;
  int key_model = -1, key_policy = -1;
  int64_t NE = 0, S = 0, nchunks = 0, nb = 0;
  int32_t b0 = 0;
  bool lru = false;
  unsigned long long total_msgs = 0;
  std::vector<int64_t> h_soff, h_touched;
};

inline SweepWs& sweep_ws_of(const atlas_graph* g) {
  if (!g->sweep_ws) g->sweep_ws = new SweepWs();
  return *g->sweep_ws;
}

}  // namespace atlas

struct atlas_layer {
  atlas_layer_desc desc{};
  int64_t nloc = 0;
  int64_t sub_batch = 1, evict_batch = 1;
  cudaStream_t stream = nullptr;  // default launch stream for internal work
  atlas::DevBuf<uint32_t> indeg;  // local in-degrees
  // data plane
  atlas::DevBuf<float> acc;       // nloc x agg_dim
  atlas::DevBuf<uint8_t> touched; // first-touch flags (chunk path)
  // control plane
  atlas::DevBuf<uint32_t> pending;
  atlas::DevBuf<uint8_t> state;
  atlas::DevBuf<uint32_t> seq;
  atlas::DevBuf<int32_t> slot_of;
  atlas::DevBuf<uint8_t> unique_reloaded;
  atlas::DevBuf<int32_t> hot_list, free_stack, scratch_a, scratch_b;
  atlas::DevBuf<uint64_t> slot_key;
  atlas::DevBuf<int32_t> rnd_members, rnd_pos;
  atlas::DevBuf<int64_t> log_victims, log_reloads, log_grad;
  atlas::DevBuf<int32_t> chunk_grad;
  atlas::DevBuf<int64_t> chunk_grad_batches;
  atlas::DevBuf<atlas::EngineScalars> scalars;
  atlas::DevBuf<atlas::GridSync> grid_sync;
  atlas::DevBuf<int64_t> first_pos, last_pos;  // spans (per local vertex)
  std::vector<int64_t> chunk_reloads, chunk_touched;
  bool engine_initialized = false;
  bool fast_path = false;
  // sweep replay (sweep.cu) results: exact integers without per-vertex state
  bool sweep_path = false;
  int64_t sw_messages = 0, sw_evictions = 0, sw_reloads = 0, sw_hot_peak = 0,
          sw_unique = 0, sw_admissions = 0;
  bool gat = false;  // GAT layer: GCN control plane, fused GAT data plane
  bool spans_host_done = false;
  int64_t chunks_seen = 0;
  int64_t stream_step = 0;  // global stream position counter (operator path)
  // staging for the operator path
  atlas::DevBuf<uint8_t> tile;          // chunk rows on device
  atlas::DevBuf<int64_t> ch_offsets;    // n+1
  atlas::DevBuf<int64_t> ch_nbrs;       // m
  atlas::DevBuf<uint8_t> sort_tmp;
  atlas::DevBuf<uint32_t> keys_a, keys_b, vals_a, vals_b;
  atlas::DevBuf<uint64_t> runs;
  atlas::DevBuf<int64_t> run_beg;
  atlas::DevBuf<uint32_t> run_dst, ent_src;
  atlas::DevBuf<int64_t> misc64;
  atlas::DevBuf<float> grad_rows;
  // per-chunk workspaces of the operator path, grow-only across chunks
  atlas::DevBuf<uint32_t> op_srcrow;
  atlas::DevBuf<int64_t> op_counts, op_nsel, op_dv;
  atlas::DevBuf<uint64_t> op_at_first, op_ordered;
  // stream the last atlas_chunk_submit queued on: read-backs of the
  // chunk's results (graduated ids/rows, logs) synchronise on it
  cudaStream_t submit_stream = nullptr;
  atlas::PinnedBuf<int64_t> pin64;
  atlas::PinnedBuf<atlas::EngineScalars> pin_scalars;
  // fast-path metrics
  int64_t span_count = 0, span_sum = 0, span_q_lo = 0, span_q_hi = 0;
  int64_t fp_hot_peak = 0;
  int64_t fp_messages = 0;
  float timing_ms[2] = {0.f, 0.f};
  // whole-layer passes: the control plane runs on its own stream next to
  // the data plane; tev = data begin/end (launch stream), control
  // begin/end (ctl_stream). Times and a deferred verdict are read lazily.
  cudaStream_t ctl_stream = nullptr;
  cudaEvent_t tev[4] = {nullptr, nullptr, nullptr, nullptr};
  bool timing_pending = false;
  bool ctl_deferred = false;
  bool ctl_queued = false;  // control plane queued ahead of the data plane
  const atlas_graph* ctl_graph = nullptr;
  int64_t ctl_R = 0;
  atlas::PinnedBuf<unsigned long long> pin_hist;
  // reusable workspaces (kept across resets so repeated layers allocate once)
  atlas::DevBuf<unsigned long long> ctl_hist;
  atlas::DevBuf<int64_t> span_buf, span_sorted;
  atlas::DevBuf<unsigned long long> span_acc;
  atlas::DevBuf<uint8_t> span_tmp;
  // spans reduced on the control stream (whole-layer passes)
  atlas::DevBuf<int64_t> span_dev;
  atlas::PinnedBuf<int64_t> span_pin;
  cudaEvent_t span_ev = nullptr;
  bool spans_queued = false;
  // chunk streamer (host -> HBM double buffer)
  atlas::DevBuf<uint8_t> stream_tile[2];
  atlas::DevBuf<int64_t> cursor;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_ready[2] = {nullptr, nullptr};
  cudaEvent_t ev_free[2] = {nullptr, nullptr};
  bool tile_used[2] = {false, false};  // ev_free[b] was recorded
  // whole-input streaming: one ready event per in-flight tile
  cudaEvent_t tile_ev[atlas::kTileEvents] = {};
  ~atlas_layer() {
    if (copy_stream) cudaStreamDestroy(copy_stream);
    if (ctl_stream) cudaStreamDestroy(ctl_stream);
    for (auto& e : tev)
      if (e) cudaEventDestroy(e);
    for (auto& e : tile_ev)
      if (e) cudaEventDestroy(e);
    if (span_ev) cudaEventDestroy(span_ev);
    for (int i = 0; i < 2; i++) {
      if (ev_ready[i]) cudaEventDestroy(ev_ready[i]);
      if (ev_free[i]) cudaEventDestroy(ev_free[i]);
    }
  }
};

namespace atlas {

// graph.cu
void build_csc(atlas_graph* g, DevBuf<uint32_t>& nbrs_dev,
               const uint32_t* indeg_host, cudaStream_t s);
// raise the deferred in-degree/adjacency mismatch of the last build, if any
void verify_graph(const atlas_graph* g);

// aggregate.cu
void launch_agg_resident(const atlas_graph* g, const void* x, int dtype,
                         int64_t ldx, int model, float gin_epsilon, int d,
                         float* acc, int64_t ldacc, const int32_t* input_flag,
                         cudaStream_t s);
void launch_agg_resident_range(const atlas_graph* g, const void* x, int dtype,
                               int64_t ldx, int model, float gin_epsilon,
                               int d, float* acc, int64_t ldacc, int64_t v0,
                               int64_t v1, cudaStream_t s);
void launch_agg_resident_epi(const atlas_graph* g, const float* z,
                             int64_t ldz, int data_model, float gin_epsilon,
                             int d, const int32_t* input_flag, void* y,
                             int y_dtype, int64_t ldy, const float* bias,
                             const float* self_rows, int64_t ld_self, int n,
                             int relu, int32_t* out_flag, int64_t v_begin,
                             int64_t v_end, cudaStream_t s);
void launch_agg_runs(const void* tile, int dtype, int64_t ldx,
                     int64_t tile_lo, const uint32_t* run_dst,
                     const int64_t* run_beg, int64_t nruns,
                     const uint32_t* ent_src, const uint32_t* indeg,
                     int model, float gin_epsilon, int d, float* acc,
                     int64_t ldacc, uint8_t* touched, cudaStream_t s);
// last tile of a whole-input stream: the remaining edge suffixes on the
// cp.async ring (GCN, f32 rows <= 512 B); false if the shape does not fit
bool launch_agg_suffix(const void* tile, int dtype, int64_t ldx,
                       int64_t tile_lo, int64_t tile_hi,
                       const atlas_graph* g, int model, float gin_epsilon,
                       int d, float* acc, int64_t ldacc, int64_t* cursor,
                       uint8_t* touched, cudaStream_t s);
void launch_agg_tile(const void* tile, int dtype, int64_t ldx, int64_t tile_lo,
                     int64_t tile_hi, const atlas_graph* g, int model,
                     float gin_epsilon, int d, float* acc, int64_t ldacc,
                     int64_t* cursor, uint8_t* touched, cudaStream_t s);
void launch_sage_self(const void* tile, int dtype, int64_t ldx,
                      int64_t row0, int64_t nrows, int d, float* acc_rows,
                      int64_t ldacc, cudaStream_t s);
void launch_gather_rows(const float* acc, int64_t ldacc, const int32_t* ids,
                        int64_t n, int64_t width, float* out, cudaStream_t s);

// gat.cu
void launch_gat_aggregate(const atlas_graph* g, const void* z, int z_dtype,
                          int64_t ldz, int heads, int head_dim,
                          int head_stride, int el_col, int er_col,
                          const float* bias, int mean_heads, int relu,
                          float slope, void* y, int y_dtype, int64_t ldy,
                          const float* attn_l, cudaStream_t s);

// transform.cu
void launch_transform_stable(const float* x, int64_t rows, int64_t k,
                             int64_t ldx, const float* w, const float* b,
                             int64_t n, int relu, void* y, int y_dtype,
                             int64_t ldy, int32_t* flag, cudaStream_t s);
bool launch_transform_tc(const void* x, int x_dtype, int64_t rows, int64_t k,
                         int64_t ldx, const float* w, const float* b,
                         int64_t n, int relu, void* y, int y_dtype,
                         int64_t ldy, int32_t* flag, cudaStream_t s);
// pending er request for the next launch_transform_tc on this host thread
// (atlas_transform_er); w = nullptr clears it
void set_transform_er(const float* w, int col, int heads, int hs);

// control.cu
void engine_init(atlas_layer* L, cudaStream_t s);
void engine_run_chunks(atlas_layer* L, const uint64_t* runs,
                       const int64_t* run_off, const int64_t* chunk_bounds,
                       int64_t nchunks, const int64_t* host_run_off,
                       cudaStream_t s);
bool control_is_async(atlas_layer* L, const atlas_graph* g, int64_t R);
void resident_control(atlas_layer* L, const atlas_graph* g,
                      int64_t chunk_rows, cudaStream_t s);
void settle_control(atlas_layer* L);
void chunk_spans(atlas_layer* L, int64_t start, int64_t end,
                 const int64_t* offsets_dev, const int64_t* nbrs_dev,
                 int64_t m, cudaStream_t s);
void finish_spans(atlas_layer* L, cudaStream_t s);
void check_engine_error(atlas_layer* L, cudaStream_t s);

// sweep.cu
bool sweep_enabled();
bool sweep_try_cached(atlas_layer* L, const atlas_graph* g, int64_t R,
                      cudaStream_t s);
bool sweep_replay(atlas_layer* L, const atlas_graph* g, int64_t R,
                  const uint64_t* runs, const int64_t* run_off_dev,
                  const std::vector<int64_t>& run_off, cudaStream_t s);

// reorder.cu
void reorder_graph(int64_t V, int64_t E, const int64_t* off_h,
                   const uint32_t* nbrs_h, const uint32_t* indeg_h,
                   int64_t* old_to_new_h, int64_t* new_off_h,
                   uint32_t* new_nbrs_h, uint32_t* new_indeg_h,
                   double* scores_h, cudaStream_t s);

// launch accounting
void count_launch(int n = 1);

}  // namespace atlas
