// C-ABI edge of libatlas_b200.so (include/atlas_b200.h).
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "internal.cuh"

namespace atlas {

static thread_local std::string g_last_error;
static std::atomic<int64_t> g_launches{0};

void set_error(const std::string& msg) { g_last_error = msg; }
void count_launch(int n) { g_launches += n; }

EngineScalars read_scalars(atlas_layer* L, cudaStream_t s);
void submit_chunk(atlas_layer* L, int64_t start, int64_t end,
                  const void* rows_host, int dtype, const int64_t* off_host,
                  const int64_t* nbrs_host, int64_t m, cudaStream_t s);

template <typename F>
static int guarded(F f) {
  try {
    f();
    return ATLAS_OK;
  } catch (const Error& e) {
    set_error(e.msg);
    return e.code;
  } catch (const std::exception& e) {
    set_error(std::string("internal: ") + e.what());
    return ATLAS_EINVARIANT;
  }
}

static void use_device(int dev) { ATLAS_CUDA(cudaSetDevice(dev)); }

// upload a CSR (host) into the graph's buffers and rebuild its CSC view
static void load_graph(atlas_graph* g, int64_t V, int64_t E,
                       const int64_t* offsets_host,
                       const uint32_t* neighbors_host,
                       const uint32_t* in_degrees_host, cudaStream_t s) {
  verify_graph(g);  // a pending check of the previous contents
  g->maxpass_cache.clear();
  g->generation++;
  g->V = V;
  g->E = E;
  g->offsets_host.assign(offsets_host, offsets_host + V + 1);
  g->offsets.reserve(V + 1);
  ATLAS_CUDA(cudaMemcpyAsync(g->offsets.ptr, offsets_host,
                             (V + 1) * sizeof(int64_t),
                             cudaMemcpyHostToDevice, s));
  g->ws_nbrs.reserve(E > 0 ? E : 1);
  if (E > 0)
    ATLAS_CUDA(cudaMemcpyAsync(g->ws_nbrs.ptr, neighbors_host,
                               E * sizeof(uint32_t), cudaMemcpyHostToDevice,
                               s));
  build_csc(g, g->ws_nbrs, in_degrees_host, s);
}

// control stream + timing events of whole-layer passes (created once)
static void ensure_ctl(atlas_layer* L) {
  if (L->ctl_stream) return;
  ATLAS_CUDA(cudaStreamCreateWithFlags(&L->ctl_stream, cudaStreamNonBlocking));
  for (auto& e : L->tev) ATLAS_CUDA(cudaEventCreate(&e));
}

// take any deferred control verdict and the pending pass timings
// read_timing=false (a new pass is starting): an unread timing of the
// previous pass is dropped without waiting for the device, so queueing
// pass after pass never stalls the host on the data plane
static void settle(atlas_layer* L, bool read_timing = false) {
  settle_control(L);
  if (L->timing_pending && !read_timing) {
    L->timing_pending = false;
    L->timing_ms[0] = L->timing_ms[1] = 0.f;
  }
  if (L->timing_pending) {
    L->timing_pending = false;
    ATLAS_CUDA(cudaEventSynchronize(L->tev[1]));
    ATLAS_CUDA(cudaEventSynchronize(L->tev[3]));
    ATLAS_CUDA(cudaEventElapsedTime(&L->timing_ms[0], L->tev[0], L->tev[1]));
    ATLAS_CUDA(cudaEventElapsedTime(&L->timing_ms[1], L->tev[2], L->tev[3]));
  }
}

// The control plane of a whole-layer pass runs on the control stream,
// ordered after everything queued on the launch stream s before
// control_begin. It is queued (control_queue) only after the data plane:
// queueing it may wait on the host for a refreshed graph's chunk
// statistics, and the data plane (tile copies, aggregation) must already
// be in flight by then.
static void control_begin(atlas_layer* L, cudaStream_t s) {
  ensure_ctl(L);
  ATLAS_CUDA(cudaEventRecord(L->tev[0], s));
  ATLAS_CUDA(cudaStreamWaitEvent(L->ctl_stream, L->tev[0], 0));
  ATLAS_CUDA(cudaEventRecord(L->tev[2], L->ctl_stream));
}

// queue the control plane and make s wait for it
static void control_queue(atlas_layer* L, const atlas_graph* g,
                          int64_t chunk_rows, cudaStream_t s) {
  if (!L->ctl_queued) {
    resident_control(L, g, chunk_rows, L->ctl_stream);
    ATLAS_CUDA(cudaEventRecord(L->tev[3], L->ctl_stream));
  }
  L->ctl_queued = false;
  ATLAS_CUDA(cudaStreamWaitEvent(s, L->tev[3], 0));
}

// ATLAS_CTL_FIRST=1: queue the control plane BEFORE the data plane of a
// resident pass, so its short kernels take SMs ahead of the persistent
// aggregation grid instead of waiting for its CTAs to retire (the
// per-layer tail of control_ms over agg_ms). Only when queueing cannot
// block the host: the pass's chunk-statistics bound is cached and no exact
// replay is forced.
static void control_early(atlas_layer* L, const atlas_graph* g,
                          int64_t chunk_rows) {
  static const bool on = [] {
    const char* e = std::getenv("ATLAS_CTL_FIRST");
    return e && e[0] == '1';
  }();
  if (!on || !control_is_async(L, g, chunk_rows)) return;
  resident_control(L, g, chunk_rows, L->ctl_stream);
  ATLAS_CUDA(cudaEventRecord(L->tev[3], L->ctl_stream));
  L->ctl_queued = true;
}

// side copy stream and its events (created once per layer)
static void ensure_copy_stream(atlas_layer* L) {
  if (L->copy_stream) return;
  ATLAS_CUDA(cudaStreamCreateWithFlags(&L->copy_stream, cudaStreamNonBlocking));
  for (int i = 0; i < 2; i++) {
    ATLAS_CUDA(cudaEventCreateWithFlags(&L->ev_ready[i],
                                        cudaEventDisableTiming));
    ATLAS_CUDA(cudaEventCreateWithFlags(&L->ev_free[i],
                                        cudaEventDisableTiming));
  }
}

// inputs up to this many bytes land whole in HBM during a streamed pass;
// ATLAS_STREAM_WHOLE_MAX_BYTES overrides the 8 GiB default (tests set 0 to
// exercise the two-buffer tile path)
static size_t stream_whole_max() {
  static const size_t v = [] {
    const char* e = std::getenv("ATLAS_STREAM_WHOLE_MAX_BYTES");
    return e ? (size_t)std::strtoull(e, nullptr, 10) : (size_t(8) << 30);
  }();
  return v;
}

static void ensure_tile_events(atlas_layer* L) {
  for (auto& e : L->tile_ev)
    if (!e) ATLAS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
}

// the layer's f32 aggregation records (nloc x agg_dim), allocated lazily
static void ensure_records(atlas_layer* L, int64_t rows = -1) {
  if (rows < 0) rows = L->nloc;
  const size_t want = (size_t)std::max<int64_t>(rows, 1) * L->desc.agg_dim;
  if (L->acc.count < want) L->acc.alloc(want);
}

}  // namespace atlas

using namespace atlas;

extern "C" {

const char* atlas_last_error(void) { return g_last_error.c_str(); }
int atlas_abi_version(void) { return ATLAS_ABI_VERSION; }
int64_t atlas_kernel_launches(void) { return g_launches.load(); }

int atlas_graph_create(int32_t device, int64_t V, int64_t E,
                       const int64_t* offsets_host,
                       const uint32_t* neighbors_host,
                       const uint32_t* in_degrees_host, int64_t lo,
                       int64_t hi, void* stream, atlas_graph** out) {
  return guarded([&] {
    ATLAS_NVTX("atlas_graph_create");
    if (!out || V < 0 || E < 0 || lo < 0 || hi < lo || hi > V)
      fail(ATLAS_ECONFIG, "bad graph arguments");
    if (V >= (int64_t)0x7FFFFFFF || E >= (int64_t)0xFFFFFFFF)
      fail(ATLAS_ECONFIG, "graph exceeds 32-bit vertex/edge ids per rank");
    use_device(device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    auto g = new atlas_graph();
    try {
      g->device = device;
      g->lo = lo;
      g->hi = hi;
      g->nloc = hi - lo;
      load_graph(g, V, E, offsets_host, neighbors_host, in_degrees_host, s);
      verify_graph(g);  // creation reports a bad graph immediately
    } catch (...) {
      delete g;
      throw;
    }
    *out = g;
  });
}

int atlas_graph_update(atlas_graph* g, int64_t V, int64_t E,
                       const int64_t* offsets_host,
                       const uint32_t* neighbors_host,
                       const uint32_t* in_degrees_host, void* stream) {
  return guarded([&] {
    ATLAS_NVTX("atlas_graph_update");
    if (!g || V < 0 || E < 0 || g->hi > V)
      fail(ATLAS_ECONFIG, "bad graph arguments");
    if (V >= (int64_t)0x7FFFFFFF || E >= (int64_t)0xFFFFFFFF)
      fail(ATLAS_ECONFIG, "graph exceeds 32-bit vertex/edge ids per rank");
    use_device(g->device);
    load_graph(g, V, E, offsets_host, neighbors_host, in_degrees_host,
               static_cast<cudaStream_t>(stream));
  });
}

void atlas_graph_destroy(atlas_graph* g) { delete g; }

int atlas_graph_csc(const atlas_graph* g, const int64_t** csc_ptr,
                    const uint32_t** csc_src, int64_t* n) {
  return guarded([&] {
    if (!g) fail(ATLAS_ECONFIG, "null graph");
    if (csc_ptr) *csc_ptr = g->csc_ptr.ptr;
    if (csc_src) *csc_src = g->csc_src.ptr;
    if (n) *n = g->eloc;
  });
}

int atlas_layer_create(const atlas_layer_desc* desc,
                       const uint32_t* in_degrees_host, void* stream,
                       atlas_layer** out) {
  return guarded([&] {
    ATLAS_NVTX("atlas_layer_create");
    if (!desc || !out) fail(ATLAS_ECONFIG, "null argument");
    const atlas_layer_desc& D = *desc;
    if (D.slot_count < 1) fail(ATLAS_ECONFIG, "hot_slots must be >= 1");
    if (D.dst_lo < 0 || D.dst_hi < D.dst_lo || D.dst_hi > D.num_vertices)
      fail(ATLAS_ECONFIG, "bad destination range");
    if (D.model < ATLAS_GCN || D.model > ATLAS_GAT)
      fail(ATLAS_ECONFIG, "unknown model kind");
    if (D.policy < ATLAS_MINPEND || D.policy > ATLAS_RND)
      fail(ATLAS_ECONFIG, "unknown eviction policy");
    const int64_t want = D.model == ATLAS_SAGE ? 2 * D.embed_dim : D.embed_dim;
    if (D.embed_dim < 1 || D.agg_dim != want)
      fail(ATLAS_ECONFIG, "agg_dim must be embed_dim (2x for SAGE)");
    use_device(D.device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    auto L = new atlas_layer();
    try {
      L->desc = D;
      // GAT's control plane is GCN's (pending = in-degree, zero-degree
      // pre-graduation); its data plane writes outputs
      // directly, so it keeps no f32 records
      L->gat = D.model == ATLAS_GAT;
      if (L->gat) L->desc.model = ATLAS_GCN;
      L->nloc = D.dst_hi - D.dst_lo;
      L->sub_batch = std::max<int64_t>(1, D.slot_count / 2);
      L->evict_batch =
          D.evict_batch > 0 ? D.evict_batch
                            : std::max<int64_t>(1, D.slot_count / 100);
      const int64_t nn = std::max<int64_t>(L->nloc, 1);
      L->indeg.alloc(nn);
      if (L->nloc > 0)
        ATLAS_CUDA(cudaMemcpyAsync(L->indeg.ptr, in_degrees_host + D.dst_lo,
                                   L->nloc * sizeof(uint32_t),
                                   cudaMemcpyHostToDevice, s));
      // f32 records are allocated on first use: the GAT and
      // transform-first passes write layer outputs directly
      L->acc.alloc(1);
      L->touched.alloc(nn);
      ATLAS_CUDA(cudaMemsetAsync(L->touched.ptr, 0, nn, s));
      engine_init(L, s);
    } catch (...) {
      delete L;
      throw;
    }
    *out = L;
  });
}

void atlas_layer_destroy(atlas_layer* L) { delete L; }

int atlas_layer_reset(atlas_layer* L, void* stream) {
  return guarded([&] {
    if (!L) fail(ATLAS_ECONFIG, "null layer");
    use_device(L->desc.device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    settle(L);
    const int64_t nn = std::max<int64_t>(L->nloc, 1);
    ATLAS_CUDA(cudaMemsetAsync(L->touched.ptr, 0, nn, s));
    L->chunk_reloads.clear();
    L->chunk_touched.clear();
    L->fast_path = false;
    L->sweep_path = false;
    L->chunks_seen = 0;
    L->stream_step = 0;
    L->timing_ms[0] = L->timing_ms[1] = 0.f;
    engine_init(L, s);
  });
}

int atlas_layer_bind_graph(atlas_layer* L, const atlas_graph* g,
                           void* stream) {
  return guarded([&] {
    if (!L || !g) fail(ATLAS_ECONFIG, "null argument");
    const atlas_layer_desc& D = L->desc;
    if (g->V != D.num_vertices || g->lo != D.dst_lo || g->hi != D.dst_hi)
      fail(ATLAS_ECONFIG, "graph and layer disagree on the vertex range");
    use_device(D.device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    settle(L);
    if (L->nloc > 0)
      ATLAS_CUDA(cudaMemcpyAsync(L->indeg.ptr, g->indeg.ptr,
                                 L->nloc * sizeof(uint32_t),
                                 cudaMemcpyDeviceToDevice, s));
    const int64_t nn = std::max<int64_t>(L->nloc, 1);
    ATLAS_CUDA(cudaMemsetAsync(L->touched.ptr, 0, nn, s));
    L->chunk_reloads.clear();
    L->chunk_touched.clear();
    L->fast_path = false;
    L->sweep_path = false;
    L->chunks_seen = 0;
    L->stream_step = 0;
    L->timing_ms[0] = L->timing_ms[1] = 0.f;
    engine_init(L, s);
  });
}

int atlas_chunk_submit(atlas_layer* L, int64_t start, int64_t end,
                       const void* rows_host, int32_t dtype,
                       const int64_t* off, const int64_t* nbrs, int64_t m,
                       void* stream) {
  return guarded([&] {
    ATLAS_NVTX("atlas_chunk_submit");
    if (!L) fail(ATLAS_ECONFIG, "null layer");
    if (L->gat) fail(ATLAS_ECONFIG, "GAT layers run through atlas_layer_run_gat");
    use_device(L->desc.device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    ensure_records(L);
    if (L->chunks_seen == 0) {
      // records start at zero; later chunks resume via touched flags
      ATLAS_CUDA(cudaMemsetAsync(L->acc.ptr, 0, L->acc.bytes(), s));
    }
    L->submit_stream = s;
    submit_chunk(L, start, end, rows_host, dtype, off, nbrs, m, s);
  });
}

int atlas_chunk_graduated(atlas_layer* L, int64_t* ids, float* rows,
                          int64_t cap, int64_t* count, int64_t* batch_len,
                          int64_t batch_cap, int64_t* num_batches) {
  return guarded([&] {
    ATLAS_NVTX("atlas_chunk_graduated");
    if (!L) fail(ATLAS_ECONFIG, "null layer");
    use_device(L->desc.device);
    // the chunk's work was queued on the caller's stream (often a
    // non-blocking torch stream): wait for it there, then read back on it
    cudaStream_t s = L->submit_stream;
    ATLAS_CUDA(cudaStreamSynchronize(s));
    EngineScalars sc = read_scalars(L, s);
    const int64_t n = sc.chunk_grad_n, nb = sc.chunk_grad_batches_n;
    if (count) *count = n;
    if (num_batches) *num_batches = nb;
    if (!ids && !rows && !batch_len) return;
    if (cap < n || (batch_len && batch_cap < nb))
      fail(ATLAS_ECONFIG, "graduation buffers too small");
    std::vector<int32_t> loc(n);
    if (n > 0)
      ATLAS_CUDA(cudaMemcpy(loc.data(), L->chunk_grad.ptr, n * sizeof(int32_t),
                            cudaMemcpyDeviceToHost));
    if (ids)
      for (int64_t i = 0; i < n; i++) ids[i] = loc[i] + L->desc.dst_lo;
    if (batch_len && nb > 0)
      ATLAS_CUDA(cudaMemcpy(batch_len, L->chunk_grad_batches.ptr,
                            nb * sizeof(int64_t), cudaMemcpyDeviceToHost));
    if (rows && n > 0) {
      const int64_t w = L->desc.agg_dim;
      L->grad_rows.reserve(n * w);
      launch_gather_rows(L->acc.ptr, w, L->chunk_grad.ptr, n, w,
                         L->grad_rows.ptr, s);
      ATLAS_CUDA(cudaMemcpyAsync(rows, L->grad_rows.ptr,
                                 n * w * sizeof(float),
                                 cudaMemcpyDeviceToHost, s));
      ATLAS_CUDA(cudaStreamSynchronize(s));
    }
  });
}

int atlas_layer_run_resident(atlas_layer* L, const atlas_graph* g,
                             const void* x, int32_t dtype, int64_t ldx,
                             int64_t chunk_rows, const int32_t* input_flag,
                             void* stream) {
  return guarded([&] {
    ATLAS_NVTX("atlas_layer_run_resident");
    if (!L || !g) fail(ATLAS_ECONFIG, "null argument");
    const atlas_layer_desc& D = L->desc;
    if (g->V != D.num_vertices || g->lo != D.dst_lo || g->hi != D.dst_hi)
      fail(ATLAS_ECONFIG, "graph and layer disagree on the vertex range");
    if (chunk_rows < 1) fail(ATLAS_ECONFIG, "chunk_rows must be >= 1");
    if (L->chunks_seen) fail(ATLAS_ECONFIG, "layer already consumed input");
    if (L->gat) fail(ATLAS_ECONFIG, "GAT layers run through atlas_layer_run_gat");
    ensure_records(L);
    use_device(D.device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    settle(L);
    // control plane on its own stream beside the scatter-aggregate; s
    // waits for it at the end
    control_begin(L, s);
    control_early(L, g, chunk_rows);
    if (L->nloc > 0)
      launch_agg_resident(g, x, dtype, ldx, D.model, D.gin_epsilon,
                          (int)D.embed_dim, L->acc.ptr, D.agg_dim,
                          input_flag, s);
    ATLAS_CUDA(cudaEventRecord(L->tev[1], s));
    control_queue(L, g, chunk_rows, s);
    L->timing_pending = true;
  });
}

int atlas_layer_run_blocked(atlas_layer* L, const atlas_graph* g,
                            const void* x, int32_t dtype, int64_t ldx,
                            int64_t chunk_rows, const int32_t* input_flag,
                            int32_t backend, const float* w, const float* b,
                            int64_t n, int32_t relu, void* y, int32_t y_dtype,
                            int64_t ldy, int32_t* out_flag, int64_t block_rows,
                            void* stream) {
  return guarded([&] {
    ATLAS_NVTX("atlas_layer_run_blocked");
    if (!L || !g || !w || !b || !y) fail(ATLAS_ECONFIG, "null argument");
    const atlas_layer_desc& D = L->desc;
    if (g->V != D.num_vertices || g->lo != D.dst_lo || g->hi != D.dst_hi)
      fail(ATLAS_ECONFIG, "graph and layer disagree on the vertex range");
    if (chunk_rows < 1) fail(ATLAS_ECONFIG, "chunk_rows must be >= 1");
    if (block_rows < 1) fail(ATLAS_ECONFIG, "block_rows must be >= 1");
    if (L->chunks_seen) fail(ATLAS_ECONFIG, "layer already consumed input");
    if (L->gat) fail(ATLAS_ECONFIG, "GAT layers run through atlas_layer_run_gat");
    if (n < 1 || ldy < n) fail(ATLAS_ECONFIG, "bad output width");
    if (backend != ATLAS_BACKEND_STABLE && backend != ATLAS_BACKEND_TCGEN05)
      fail(ATLAS_ECONFIG, "unknown transform backend");
    use_device(D.device);
    const int64_t rows = std::min<int64_t>(block_rows, std::max<int64_t>(L->nloc, 1));
    ensure_records(L, rows);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    settle(L);
    control_begin(L, s);
    if (out_flag) ATLAS_CUDA(cudaMemsetAsync(out_flag, 0, sizeof(int32_t), s));
    // the input's extremes flag: the producer's, or one scan on the first
    // block that every later block reuses
    g->known_flag = input_flag;
    const int64_t k = D.agg_dim;
    const size_t yes = y_dtype == ATLAS_F32 ? 4 : 2;
    for (int64_t v0 = 0; v0 < L->nloc; v0 += rows) {
      const int64_t v1 = std::min(L->nloc, v0 + rows);
      launch_agg_resident_range(g, x, dtype, ldx, D.model, D.gin_epsilon,
                                (int)D.embed_dim, L->acc.ptr, k, v0, v1, s);
      if (!g->known_flag) g->known_flag = g->scan_flag.ptr;
      void* yb = static_cast<uint8_t*>(y) + (size_t)v0 * ldy * yes;
      if (backend == ATLAS_BACKEND_STABLE)
        launch_transform_stable(L->acc.ptr, v1 - v0, k, k, w, b, n, relu, yb,
                                y_dtype, ldy, out_flag, s);
      else if (!launch_transform_tc(L->acc.ptr, ATLAS_F32, v1 - v0, k, k, w,
                                    b, n, relu, yb, y_dtype, ldy, out_flag,
                                    s))
        fail(ATLAS_ECONFIG, "tcgen05 backend does not support this shape");
    }
    ATLAS_CUDA(cudaEventRecord(L->tev[1], s));
    control_queue(L, g, chunk_rows, s);
    L->timing_pending = true;
  });
}

int atlas_layer_record_bytes(const atlas_layer* L, int64_t* bytes) {
  return guarded([&] {
    if (!L || !bytes) fail(ATLAS_ECONFIG, "null argument");
    *bytes = (int64_t)L->acc.bytes();
  });
}

int atlas_layer_run_gat(atlas_layer* L, const atlas_graph* g, const void* z,
                        int32_t z_dtype, int64_t ldz, int32_t heads,
                        int32_t head_dim, int32_t head_stride,
                        int32_t el_col, int32_t er_col,
                        const float* bias, int32_t mean_heads, int32_t relu,
                        float negative_slope, void* y, int32_t y_dtype,
                        int64_t ldy, const float* attn_l,
                        int64_t chunk_rows, void* stream) {
  return guarded([&] {
    ATLAS_NVTX("atlas_layer_run_gat");
    if (!L || !g || !z || !bias || !y) fail(ATLAS_ECONFIG, "null argument");
    if (!L->gat) fail(ATLAS_ECONFIG, "layer was not created as GAT");
    const atlas_layer_desc& D = L->desc;
    if (g->V != D.num_vertices || g->lo != D.dst_lo || g->hi != D.dst_hi)
      fail(ATLAS_ECONFIG, "graph and layer disagree on the vertex range");
    if (chunk_rows < 1) fail(ATLAS_ECONFIG, "chunk_rows must be >= 1");
    if (L->chunks_seen) fail(ATLAS_ECONFIG, "layer already consumed input");
    use_device(D.device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    settle(L);
    control_begin(L, s);
    launch_gat_aggregate(g, z, z_dtype, ldz, heads, head_dim, head_stride,
                         el_col, er_col, bias, mean_heads, relu,
                         negative_slope, y, y_dtype, ldy, attn_l, s);
    ATLAS_CUDA(cudaEventRecord(L->tev[1], s));
    control_queue(L, g, chunk_rows, s);
    L->timing_pending = true;
  });
}

int atlas_layer_run_fused(atlas_layer* L, const atlas_graph* g,
                          const float* z, int64_t ldz, int32_t data_model,
                          int64_t d, int64_t chunk_rows,
                          const int32_t* input_flag, const float* bias,
                          const float* self_rows, int64_t ld_self, int64_t n,
                          int32_t relu, void* y, int32_t y_dtype, int64_t ldy,
                          int32_t* out_flag, void* y_host, int64_t ldy_host,
                          int32_t host_slices, void* stream) {
  return guarded([&] {
    ATLAS_NVTX("atlas_layer_run_fused");
    if (!L || !g || !z || !bias || !y) fail(ATLAS_ECONFIG, "null argument");
    if (L->gat) fail(ATLAS_ECONFIG, "GAT layers run through atlas_layer_run_gat");
    const atlas_layer_desc& D = L->desc;
    if (g->V != D.num_vertices || g->lo != D.dst_lo || g->hi != D.dst_hi)
      fail(ATLAS_ECONFIG, "graph and layer disagree on the vertex range");
    if (chunk_rows < 1) fail(ATLAS_ECONFIG, "chunk_rows must be >= 1");
    if (L->chunks_seen) fail(ATLAS_ECONFIG, "layer already consumed input");
    if (n < 1 || n > d || ldy < n) fail(ATLAS_ECONFIG, "bad output width");
    if (data_model != ATLAS_GCN && data_model != ATLAS_GIN)
      fail(ATLAS_ECONFIG, "fused data plane is a mean (GCN/SAGE) or a sum "
                          "(GIN)");
    if ((D.model == ATLAS_SAGE) != (self_rows != nullptr))
      fail(ATLAS_ECONFIG, "SAGE needs its self rows (and only SAGE)");
    use_device(D.device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    settle(L);
    control_begin(L, s);
    control_early(L, g, chunk_rows);
    if (out_flag) ATLAS_CUDA(cudaMemsetAsync(out_flag, 0, sizeof(int32_t), s));
    if (!y_host) {
      launch_agg_resident_epi(g, z, ldz, data_model, D.gin_epsilon, (int)d,
                              input_flag, y, y_dtype, ldy, bias, self_rows,
                              ld_self, (int)n, relu, out_flag, 0, L->nloc, s);
    } else {
      // the output goes to the host slice by slice: the D2H of slice i
      // (copy stream) overlaps the aggregation of slice i+1 (stream s)
      if (ldy_host < n) fail(ATLAS_ECONFIG, "host output too narrow");
      ensure_copy_stream(L);
      const size_t es = y_dtype == ATLAS_F32 ? 4 : 2;
      const int64_t k = std::max<int32_t>(1, host_slices);
      const int64_t step = ceil_div(std::max<int64_t>(L->nloc, 1), k);
      for (int64_t a = 0; a < L->nloc; a += step) {
        const int64_t b = std::min(L->nloc, a + step);
        launch_agg_resident_epi(g, z, ldz, data_model, D.gin_epsilon, (int)d,
                                input_flag, y, y_dtype, ldy, bias, self_rows,
                                ld_self, (int)n, relu, out_flag, a, b, s);
        ATLAS_CUDA(cudaEventRecord(L->ev_ready[0], s));
        ATLAS_CUDA(cudaStreamWaitEvent(L->copy_stream, L->ev_ready[0], 0));
        uint8_t* dst = static_cast<uint8_t*>(y_host) + a * ldy_host * es;
        const uint8_t* src = static_cast<const uint8_t*>(y) + a * ldy * es;
        if (ldy == n && ldy_host == n)  // dense rows: one linear DMA
          ATLAS_CUDA(cudaMemcpyAsync(dst, src, (b - a) * n * es,
                                     cudaMemcpyDeviceToHost, L->copy_stream));
        else
          ATLAS_CUDA(cudaMemcpy2DAsync(dst, ldy_host * es, src, ldy * es,
                                       n * es, b - a, cudaMemcpyDeviceToHost,
                                       L->copy_stream));
      }
      ATLAS_CUDA(cudaEventRecord(L->ev_ready[1], L->copy_stream));
      ATLAS_CUDA(cudaStreamWaitEvent(s, L->ev_ready[1], 0));
    }
    ATLAS_CUDA(cudaEventRecord(L->tev[1], s));
    control_queue(L, g, chunk_rows, s);
    L->timing_pending = true;
  });
}

int atlas_layer_run_streamed(atlas_layer* L, const atlas_graph* g,
                             const void* x_host, int32_t dtype, int64_t ldx,
                             int64_t tile_rows, int64_t chunk_rows,
                             void* stream) {
  return guarded([&] {
    ATLAS_NVTX("atlas_layer_run_streamed");
    if (!L || !g || !x_host) fail(ATLAS_ECONFIG, "null argument");
    const atlas_layer_desc& D = L->desc;
    if (g->V != D.num_vertices || g->lo != D.dst_lo || g->hi != D.dst_hi)
      fail(ATLAS_ECONFIG, "graph and layer disagree on the vertex range");
    if (chunk_rows < 1 || tile_rows < 1 || ldx < D.embed_dim)
      fail(ATLAS_ECONFIG, "bad tile / chunk rows");
    if (L->chunks_seen) fail(ATLAS_ECONFIG, "layer already consumed input");
    if (L->gat) fail(ATLAS_ECONFIG, "GAT layers run through atlas_layer_run_gat");
    ensure_records(L);
    use_device(D.device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t item = dtype == ATLAS_F32 ? 4 : 2;
    const int64_t V = D.num_vertices;
    tile_rows = std::min<int64_t>(tile_rows, std::max<int64_t>(V, 1));
    for (auto& b : L->stream_tile) b.reserve(tile_rows * ldx * item);
    ensure_copy_stream(L);
    const int64_t nn = std::max<int64_t>(L->nloc, 1);
    L->cursor.reserve(nn);
    if (L->nloc > 0)
      ATLAS_CUDA(cudaMemcpyAsync(L->cursor.ptr, g->csc_ptr.ptr,
                                 L->nloc * sizeof(int64_t),
                                 cudaMemcpyDeviceToDevice, s));
    ATLAS_CUDA(cudaMemsetAsync(L->touched.ptr, 0, nn, s));
    settle(L);
    // the copy stream starts at once (it overlaps whatever s is still
    // doing, e.g. a topology refresh); a tile buffer is only refilled after
    // the kernel that last read it, in this pass or the previous one.
    // An input of up to 8 GB lands whole in HBM (each tile at its own
    // rows), so the copy stream never waits for a buffer and every copy is
    // queued before any kernel; larger inputs cycle through two buffers.
    const size_t row_b = (size_t)ldx * item;
    const bool whole = (size_t)V * row_b <= stream_whole_max();
    if (whole) L->stream_tile[0].reserve((size_t)V * row_b);
    // Tile boundaries (uniform: a tapered tail measured slower, every
    // extra tile re-reads and re-writes the whole accumulator)
    std::vector<int64_t> bnd{0};
    for (int64_t r = 0; r < V;) bnd.push_back(r = std::min(V, r + tile_rows));
    const int64_t ntiles = (int64_t)bnd.size() - 1;
    auto tile_ptr = [&](int64_t t) -> uint8_t* {
      return whole ? L->stream_tile[0].ptr + (size_t)bnd[t] * row_b
                   : L->stream_tile[t & 1].ptr;
    };
    auto copy_tile = [&](int64_t t) {
      const int b = (int)(t & 1);
      const int64_t r0 = bnd[t], r1 = bnd[t + 1];
      if (whole ? (t == 0 && L->tile_used[0]) : (t >= 2 || L->tile_used[b]))
        ATLAS_CUDA(cudaStreamWaitEvent(L->copy_stream,
                                       L->ev_free[whole ? 0 : b], 0));
      // whole rows (pitch included) are one contiguous block: a single DMA
      ATLAS_CUDA(cudaMemcpyAsync(
          tile_ptr(t), static_cast<const uint8_t*>(x_host) + r0 * row_b,
          (r1 - r0) * row_b, cudaMemcpyHostToDevice, L->copy_stream));
      ATLAS_CUDA(cudaEventRecord(whole ? L->tile_ev[t % kTileEvents]
                                       : L->ev_ready[b],
                                 L->copy_stream));
    };
    if (whole) ensure_tile_events(L);
    const int64_t ahead = whole ? std::min<int64_t>(kTileEvents, ntiles)
                                : std::min<int64_t>(2, ntiles);
    for (int64_t t = 0; t < ahead; t++) copy_tile(t);
    control_begin(L, s);  // tev[0] after the resets
    for (int64_t t = 0; t < ntiles; t++) {
      const int b = (int)(t & 1);
      const int64_t r0 = bnd[t], r1 = bnd[t + 1];
      if (t >= ahead) copy_tile(t);
      ATLAS_CUDA(cudaStreamWaitEvent(
          s, whole ? L->tile_ev[t % kTileEvents] : L->ev_ready[b], 0));
      const bool suffix =
          L->nloc > 0 &&
          launch_agg_suffix(tile_ptr(t), dtype, ldx, r0, r1, g, D.model,
                            D.gin_epsilon, (int)D.embed_dim, L->acc.ptr,
                            D.agg_dim, L->cursor.ptr, L->touched.ptr, s);
      if (L->nloc > 0 && !suffix)
        launch_agg_tile(tile_ptr(t), dtype, ldx, r0, r1, g, D.model,
                        D.gin_epsilon, (int)D.embed_dim, L->acc.ptr,
                        D.agg_dim, L->cursor.ptr, L->touched.ptr, s);
      if (!whole) {
        ATLAS_CUDA(cudaEventRecord(L->ev_free[b], s));
        L->tile_used[b] = true;
      }
    }
    if (whole) {
      ATLAS_CUDA(cudaEventRecord(L->ev_free[0], s));
      L->tile_used[0] = true;
    }
    ATLAS_CUDA(cudaEventRecord(L->tev[1], s));
    control_queue(L, g, chunk_rows, s);
    L->timing_pending = true;
  });
}

int atlas_layer_run_pieces(atlas_layer* L, const atlas_graph* g,
                           const void* x, int32_t dtype, int64_t ldx,
                           const int64_t* bounds, int32_t npieces,
                           void* const* ready, int64_t chunk_rows,
                           void* stream) {
  return guarded([&] {
    ATLAS_NVTX("atlas_layer_run_pieces");
    if (!L || !g || !x || !bounds || npieces < 1)
      fail(ATLAS_ECONFIG, "null argument");
    const atlas_layer_desc& D = L->desc;
    if (g->V != D.num_vertices || g->lo != D.dst_lo || g->hi != D.dst_hi)
      fail(ATLAS_ECONFIG, "graph and layer disagree on the vertex range");
    if (chunk_rows < 1 || ldx < D.embed_dim)
      fail(ATLAS_ECONFIG, "bad pitch / chunk rows");
    if (L->chunks_seen) fail(ATLAS_ECONFIG, "layer already consumed input");
    if (L->gat) fail(ATLAS_ECONFIG, "GAT layers run through atlas_layer_run_gat");
    if (bounds[0] != 0 || bounds[npieces] != D.num_vertices)
      fail(ATLAS_ECONFIG, "pieces must tile [0, V)");
    for (int32_t t = 0; t < npieces; t++)
      if (bounds[t + 1] < bounds[t])
        fail(ATLAS_ECONFIG, "piece bounds must ascend");
    ensure_records(L);
    use_device(D.device);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t row_b = (size_t)ldx * (dtype == ATLAS_F32 ? 4 : 2);
    const int64_t nn = std::max<int64_t>(L->nloc, 1);
    L->cursor.reserve(nn);
    if (L->nloc > 0)
      ATLAS_CUDA(cudaMemcpyAsync(L->cursor.ptr, g->csc_ptr.ptr,
                                 L->nloc * sizeof(int64_t),
                                 cudaMemcpyDeviceToDevice, s));
    ATLAS_CUDA(cudaMemsetAsync(L->touched.ptr, 0, nn, s));
    settle(L);
    control_begin(L, s);
    // pieces arrive in ascending source order (the owners' broadcasts);
    // each is folded into the records as soon as its event fires, resuming
    // every destination's ascending source list from its cursor, so the
    // records are the resident pass's bits whatever the piece boundaries
    const uint8_t* base = static_cast<const uint8_t*>(x);
    for (int32_t t = 0; t < npieces; t++) {
      const int64_t r0 = bounds[t], r1 = bounds[t + 1];
      if (ready && ready[t])
        ATLAS_CUDA(cudaStreamWaitEvent(s, static_cast<cudaEvent_t>(ready[t]),
                                       0));
      if (r1 == r0 || L->nloc == 0) continue;
      const uint8_t* tile = base + (size_t)r0 * row_b;
      const bool suffix = launch_agg_suffix(
          tile, dtype, ldx, r0, r1, g, D.model, D.gin_epsilon,
          (int)D.embed_dim, L->acc.ptr, D.agg_dim, L->cursor.ptr,
          L->touched.ptr, s);
      if (!suffix)
        launch_agg_tile(tile, dtype, ldx, r0, r1, g, D.model, D.gin_epsilon,
                        (int)D.embed_dim, L->acc.ptr, D.agg_dim,
                        L->cursor.ptr, L->touched.ptr, s);
    }
    ATLAS_CUDA(cudaEventRecord(L->tev[1], s));
    control_queue(L, g, chunk_rows, s);
    L->timing_pending = true;
  });
}

int atlas_reorder(int32_t device, int64_t V, int64_t E, const int64_t* off,
                  const uint32_t* nbrs, const uint32_t* indeg,
                  int64_t* old_to_new, int64_t* new_off, uint32_t* new_nbrs,
                  uint32_t* new_indeg, double* scores, void* stream) {
  return guarded([&] {
    ATLAS_NVTX("atlas_reorder");
    if (V < 0 || E < 0 || !off || !old_to_new || !new_off)
      fail(ATLAS_ECONFIG, "bad reorder arguments");
    if (V >= (int64_t)0x7FFFFFFF || E >= (int64_t)0x7FFFFFFF)
      fail(ATLAS_ECONFIG, "graph exceeds 32-bit ids");
    use_device(device);
    reorder_graph(V, E, off, nbrs, indeg, old_to_new, new_off, new_nbrs,
                  new_indeg, scores, static_cast<cudaStream_t>(stream));
  });
}

int atlas_layer_timing(atlas_layer* L, float* ms, int32_t n) {
  return guarded([&] {
    if (!L || !ms) fail(ATLAS_ECONFIG, "null argument");
    use_device(L->desc.device);
    settle(L, true);
    for (int i = 0; i < n && i < 2; i++) ms[i] = L->timing_ms[i];
  });
}

int atlas_layer_accumulator(atlas_layer* L, float** acc, int64_t* ld) {
  return guarded([&] {
    if (!L) fail(ATLAS_ECONFIG, "null layer");
    if (!L->gat) ensure_records(L);
    if (acc) *acc = L->acc.ptr;
    if (ld) *ld = L->desc.agg_dim;
  });
}

int atlas_transform(int32_t backend, const float* x, int64_t rows, int64_t k,
                    int64_t ldx, const float* w, const float* b, int64_t n,
                    int32_t relu, void* y, int32_t y_dtype, int64_t ldy,
                    int32_t* flag, void* stream) {
  return guarded([&] {
    ATLAS_NVTX("atlas_transform");
    if (rows < 0 || k < 1 || n < 1 || ldx < k || ldy < n)
      fail(ATLAS_ECONFIG, "bad transform shape");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (flag) ATLAS_CUDA(cudaMemsetAsync(flag, 0, sizeof(int32_t), s));
    if (backend == ATLAS_BACKEND_STABLE) {
      launch_transform_stable(x, rows, k, ldx, w, b, n, relu, y, y_dtype, ldy,
                              flag, s);
    } else if (backend == ATLAS_BACKEND_TCGEN05) {
      // rows the TMA cannot address (pitch not a multiple of 16 B, e.g. a
      // 6-wide record) or N > 256 run on the SIMT kernel, which is exact
      if (!launch_transform_tc(x, ATLAS_F32, rows, k, ldx, w, b, n, relu, y,
                               y_dtype, ldy, flag, s))
        launch_transform_stable(x, rows, k, ldx, w, b, n, relu, y, y_dtype,
                                ldy, flag, s);
    } else {
      fail(ATLAS_ECONFIG, "unknown transform backend");
    }
  });
}

int atlas_transform_typed(int32_t backend, const void* x, int32_t x_dtype,
                          int64_t rows, int64_t k, int64_t ldx,
                          const float* w, const float* b, int64_t n,
                          int32_t relu, void* y, int32_t y_dtype, int64_t ldy,
                          int32_t* flag, void* stream) {
  return guarded([&] {
    ATLAS_NVTX("atlas_transform_typed");
    if (x_dtype == ATLAS_F32) {
      const int rc = atlas_transform(backend, static_cast<const float*>(x),
                                     rows, k, ldx, w, b, n, relu, y, y_dtype,
                                     ldy, flag, stream);
      if (rc != ATLAS_OK) fail(rc, g_last_error);
      return;
    }
    if (rows < 0 || k < 1 || n < 1 || ldx < k || ldy < n)
      fail(ATLAS_ECONFIG, "bad transform shape");
    if (backend != ATLAS_BACKEND_TCGEN05)
      fail(ATLAS_ECONFIG, "f16/bf16 inputs need the tcgen05 backend");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (flag) ATLAS_CUDA(cudaMemsetAsync(flag, 0, sizeof(int32_t), s));
    if (!launch_transform_tc(x, x_dtype, rows, k, ldx, w, b, n, relu, y,
                             y_dtype, ldy, flag, s))
      fail(ATLAS_ECONFIG, "tcgen05 backend does not support this shape");
  });
}

int atlas_transform_er(int32_t backend, const void* x, int32_t x_dtype,
                       int64_t rows, int64_t k, int64_t ldx, const float* w,
                       const float* b, int64_t n, void* y, int32_t y_dtype,
                       int64_t ldy, const float* er_w, int32_t er_col,
                       int32_t heads, int32_t head_stride, void* stream) {
  return guarded([&] {
    ATLAS_NVTX("atlas_transform_er");
    if (rows < 0 || k < 1 || n < 1 || n > 128 || ldx < k || !er_w ||
        heads < 1 || heads > 8 || head_stride < 16 || head_stride % 16 != 0 ||
        (int64_t)heads * head_stride != (n + 15) / 16 * 16 || er_col < n ||
        ldy < er_col + heads)
      fail(ATLAS_ECONFIG, "bad transform_er shape");
    if (backend != ATLAS_BACKEND_TCGEN05)
      fail(ATLAS_ECONFIG, "transform_er needs the tcgen05 backend");
    struct Clear {
      ~Clear() { set_transform_er(nullptr, 0, 0, 0); }
    } clear;
    set_transform_er(er_w, er_col, heads, head_stride);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (!launch_transform_tc(x, x_dtype, rows, k, ldx, w, b, n, 0, y, y_dtype,
                             ldy, nullptr, s))
      fail(ATLAS_ECONFIG, "no register-split kernel takes this shape");
  });
}

int atlas_layer_finish(atlas_layer* L, atlas_layer_metrics* m) {
  return guarded([&] {
    ATLAS_NVTX("atlas_layer_finish");
    if (!L || !m) fail(ATLAS_ECONFIG, "null argument");
    use_device(L->desc.device);
    cudaStream_t s = nullptr;
    settle(L, true);
    verify_graph(L->ctl_graph);
    ATLAS_CUDA(cudaDeviceSynchronize());
    std::memset(m, 0, sizeof(*m));
    finish_spans(L, s);
    m->span_count = L->span_count;
    m->span_sum = L->span_sum;
    m->span_q_lo = L->span_q_lo;
    m->span_q_hi = L->span_q_hi;
    m->hot_slot_count = L->desc.slot_count;
    m->chunks = L->chunks_seen;
    const int64_t w = L->desc.agg_dim * 4;
    if (L->fast_path) {
      m->fast_path = 1;
      m->messages = L->fp_messages;
      m->admissions = L->nloc;
      m->graduations = L->nloc;
      m->hot_peak = L->fp_hot_peak;
      return;
    }
    if (L->sweep_path) {
      m->messages = L->sw_messages;
      m->evictions = L->sw_evictions;
      m->reloads = L->sw_reloads;
      m->admissions = L->sw_admissions;
      m->graduations = L->nloc;
      m->hot_peak = L->sw_hot_peak;
      m->cold_bytes_written = L->sw_evictions * w;
      m->cold_bytes_read = L->sw_reloads * w;
      m->unique_reloads = L->sw_unique;
      return;
    }
    EngineScalars sc = read_scalars(L, s);
    m->messages = sc.messages;
    m->evictions = sc.evictions;
    m->reloads = sc.reloads;
    m->admissions = sc.admissions;
    m->graduations = sc.graduations;
    m->hot_peak = sc.hot_peak;
    m->cold_bytes_written = sc.evictions * w;
    m->cold_bytes_read = sc.reloads * w;
    // unique reloads and incomplete vertices
    const int64_t n = L->nloc;
    std::vector<uint8_t> ur(n), st(n);
    if (n > 0) {
      ATLAS_CUDA(cudaMemcpy(ur.data(), L->unique_reloaded.ptr, n,
                            cudaMemcpyDeviceToHost));
      ATLAS_CUDA(cudaMemcpy(st.data(), L->state.ptr, n,
                            cudaMemcpyDeviceToHost));
    }
    int64_t uniq = 0, inc = 0;
    for (int64_t i = 0; i < n; i++) {
      uniq += ur[i] != 0;
      if (st[i] != 3) {
        if (inc < 16) m->first_incomplete[inc] = i + L->desc.dst_lo;
        inc++;
      }
    }
    m->unique_reloads = uniq;
    m->incomplete = inc;
  });
}

int atlas_layer_state(atlas_layer* L, uint32_t* pending, uint8_t* state,
                      int64_t* first_step, int64_t* last_step) {
  return guarded([&] {
    if (!L) fail(ATLAS_ECONFIG, "null layer");
    use_device(L->desc.device);
    settle(L, true);
    ATLAS_CUDA(cudaDeviceSynchronize());
    const int64_t n = L->nloc;
    if (n == 0) return;
    if ((L->fast_path || L->sweep_path) && (pending || state)) {
      // the eviction-free replay never materialises per-vertex state:
      // every vertex ran to COMPLETED with zero pending
      if (pending) std::memset(pending, 0, n * sizeof(uint32_t));
      if (state) std::memset(state, 3, n);
    } else {
      if (pending)
        ATLAS_CUDA(cudaMemcpy(pending, L->pending.ptr, n * sizeof(uint32_t),
                              cudaMemcpyDeviceToHost));
      if (state)
        ATLAS_CUDA(cudaMemcpy(state, L->state.ptr, n, cudaMemcpyDeviceToHost));
    }
    if (first_step)
      ATLAS_CUDA(cudaMemcpy(first_step, L->first_pos.ptr, n * sizeof(int64_t),
                            cudaMemcpyDeviceToHost));
    if (last_step)
      ATLAS_CUDA(cudaMemcpy(last_step, L->last_pos.ptr, n * sizeof(int64_t),
                            cudaMemcpyDeviceToHost));
  });
}

int atlas_layer_chunk_stats(atlas_layer* L, int64_t* reloads, int64_t* touched,
                            int64_t cap, int64_t* count) {
  return guarded([&] {
    if (!L) fail(ATLAS_ECONFIG, "null layer");
    use_device(L->desc.device);
    settle(L, true);
    const int64_t n = (int64_t)L->chunk_reloads.size();
    if (count) *count = n;
    if (!reloads && !touched) return;
    if (cap < n) fail(ATLAS_ECONFIG, "chunk stats buffer too small");
    for (int64_t i = 0; i < n; i++) {
      if (reloads) reloads[i] = L->chunk_reloads[i];
      if (touched) touched[i] = L->chunk_touched[i];
    }
  });
}

int atlas_layer_log(atlas_layer* L, int32_t which, int64_t* out, int64_t cap,
                    int64_t* count) {
  return guarded([&] {
    ATLAS_NVTX("atlas_layer_log");
    if (!L) fail(ATLAS_ECONFIG, "null layer");
    if (!L->desc.record_log) fail(ATLAS_ECONFIG, "layer was not logging");
    use_device(L->desc.device);
    settle(L, true);
    ATLAS_CUDA(cudaStreamSynchronize(L->submit_stream));
    EngineScalars sc = read_scalars(L, L->submit_stream);
    DevBuf<int64_t>* buf;
    int64_t used;
    if (which == ATLAS_LOG_VICTIMS) {
      buf = &L->log_victims;
      used = sc.log_victims_n;
    } else if (which == ATLAS_LOG_RELOADS) {
      buf = &L->log_reloads;
      used = sc.log_reloads_n;
    } else {
      buf = &L->log_grad;
      used = sc.log_grad_n;
    }
    if (used > (int64_t)buf->count) fail(ATLAS_EINVARIANT, "log overflowed");
    std::vector<int64_t> raw(used);
    if (used > 0)
      ATLAS_CUDA(cudaMemcpy(raw.data(), buf->ptr, used * sizeof(int64_t),
                            cudaMemcpyDeviceToHost));
    std::vector<int64_t> flat;
    flat.reserve(used);
    const int64_t lo = L->desc.dst_lo;
    if (which == ATLAS_LOG_VICTIMS) {
      // [-k, (v, key) x k] -> [k, v...] ordered like pop_min (key order);
      // RandomPolicy victims keep their draw order
      size_t i = 0;
      while (i < raw.size()) {
        const int64_t k = -raw[i++];
        std::vector<std::pair<uint64_t, int64_t>> ev;
        for (int64_t j = 0; j < k; j++, i += 2)
          ev.push_back({(uint64_t)raw[i + 1], raw[i]});
        if (L->desc.policy != ATLAS_RND) std::sort(ev.begin(), ev.end());
        flat.push_back(k);
        for (auto& e : ev) flat.push_back(e.second + lo);
      }
    } else {
      size_t i = 0;
      while (i < raw.size()) {
        const int64_t k = raw[i++];
        flat.push_back(k);
        for (int64_t j = 0; j < k; j++) flat.push_back(raw[i++] + lo);
      }
    }
    if (count) *count = (int64_t)flat.size();
    if (out) {
      if (cap < (int64_t)flat.size()) fail(ATLAS_ECONFIG, "log buffer small");
      std::copy(flat.begin(), flat.end(), out);
    }
  });
}

}  // extern "C"
