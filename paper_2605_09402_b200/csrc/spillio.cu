// Layer-directory spill I/O on the host, in parallel (SURVEY.md §8f ranks
// 2 and 3): the reference's ASPL spill files (oocgnn/storage.py:257-357)
// read straight into a dense pinned buffer -- the source of the K1
// host->HBM streamer -- and a GPU rank's output range written back as
// partition spills. Host-only code (no device work): runs without a GPU.
//
// ASPL layout: header <4sIQQQIB (magic "ASPL", version 1, min id, max id,
// rows, dim, dtype 0=f32/1=f16) at 0; u64 ids at 4096; rows at the next
// 4096 boundary; file padded to 4096 (oocgnn/storage.py:273-314).
#include <cufile.h>
#include <dlfcn.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <functional>
#include <atomic>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "internal.cuh"

namespace atlas {
namespace {

constexpr int64_t kAlign = 4096;
constexpr size_t kHeader = 4 + 4 + 8 + 8 + 8 + 4 + 1;  // <4sIQQQIB = 37

int64_t align_up(int64_t n) { return (n + kAlign - 1) / kAlign * kAlign; }

struct SpillHead {
  uint64_t lo, hi, rows;
  uint32_t dim;
  uint8_t dtype;
};

// pread exactly n bytes at off (retrying short reads)
bool pread_all(int fd, void* buf, size_t n, int64_t off) {
  auto* p = static_cast<uint8_t*>(buf);
  while (n) {
    const ssize_t r = ::pread(fd, p, n, off);
    if (r <= 0) return false;
    p += r;
    n -= (size_t)r;
    off += r;
  }
  return true;
}

bool pwrite_all(int fd, const void* buf, size_t n, int64_t off) {
  auto* p = static_cast<const uint8_t*>(buf);
  while (n) {
    const ssize_t r = ::pwrite(fd, p, n, off);
    if (r <= 0) return false;
    p += r;
    n -= (size_t)r;
    off += r;
  }
  return true;
}

struct FirstError {
  std::mutex mu;
  int code = ATLAS_OK;
  std::string msg;
  void set(int c, const std::string& m) {
    std::lock_guard<std::mutex> lock(mu);
    if (code == ATLAS_OK) {
      code = c;
      msg = m;
    }
  }
};

// moves nrows rows from file offset `off` of fd to the rows of ids
// [id, id + nrows); false on a short read
using RunSink = std::function<bool(int fd, uint64_t id, uint64_t nrows,
                                   int64_t off)>;

// one spill file -> rows at their ids (through sink); delivery counted per id
void read_one(const char* path, int dtype, int64_t dim, int64_t V,
              const RunSink& sink, std::atomic<uint16_t>* delivery,
              std::atomic<int64_t>* bytes, FirstError* err) {
  const int fd = ::open(path, O_RDONLY);
  if (fd < 0) {
    err->set(ATLAS_EFORMAT, std::string(path) + ": cannot open");
    return;
  }
  struct Closer {
    int fd;
    ~Closer() { ::close(fd); }
  } closer{fd};
  uint8_t h[kHeader];
  if (!pread_all(fd, h, kHeader, 0)) {
    err->set(ATLAS_ETRUNCATED, std::string(path) + ": header short");
    return;
  }
  if (std::memcmp(h, "ASPL", 4) != 0) {
    err->set(ATLAS_EMAGIC, std::string(path) + ": bad magic");
    return;
  }
  uint32_t ver;
  SpillHead s;
  std::memcpy(&ver, h + 4, 4);
  std::memcpy(&s.lo, h + 8, 8);
  std::memcpy(&s.hi, h + 16, 8);
  std::memcpy(&s.rows, h + 24, 8);
  std::memcpy(&s.dim, h + 32, 4);
  s.dtype = h[36];
  if (ver != 1) {
    err->set(ATLAS_EVERSION, std::string(path) + ": format version " +
                                      std::to_string(ver));
    return;
  }
  const int want_code = dtype == ATLAS_F32 ? 0 : 1;
  if (s.dim != (uint64_t)dim || s.dtype != want_code) {
    err->set(ATLAS_ECONSISTENCY,
             std::string(path) + ": shape/dtype does not match layer meta");
    return;
  }
  if (s.rows == 0 || s.lo > s.hi) {
    err->set(ATLAS_EINVARIANT, std::string(path) + ": empty or inverted id "
                                                   "range");
    return;
  }
  const int64_t item = dtype == ATLAS_F32 ? 4 : 2;
  const int64_t row_b = dim * item;
  const int64_t ids_pos = kAlign;
  const int64_t rows_pos = ids_pos + align_up((int64_t)s.rows * 8);
  const int64_t size = align_up(rows_pos + (int64_t)s.rows * row_b);
  struct stat st;
  if (::fstat(fd, &st) != 0 || st.st_size < size) {
    err->set(ATLAS_ETRUNCATED,
             std::string(path) + ": truncated (header implies " +
                 std::to_string(size) + " bytes)");
    return;
  }
  std::vector<uint64_t> ids(s.rows);
  if (!pread_all(fd, ids.data(), s.rows * 8, ids_pos)) {
    err->set(ATLAS_ETRUNCATED, std::string(path) + ": ids short");
    return;
  }
  for (uint64_t i = 0; i < s.rows; i++) {
    if ((i && ids[i] <= ids[i - 1]) || ids[i] >= (uint64_t)V) {
      err->set(ATLAS_EINVARIANT,
               std::string(path) + ": ids not strictly ascending in range");
      return;
    }
  }
  if (ids[0] != s.lo || ids[s.rows - 1] != s.hi) {
    err->set(ATLAS_EINVARIANT,
             std::string(path) + ": header id range disagrees with ids");
    return;
  }
  // runs of consecutive ids land with one read each
  uint64_t i = 0;
  while (i < s.rows) {
    uint64_t j = i + 1;
    while (j < s.rows && ids[j] == ids[j - 1] + 1) j++;
    if (!sink(fd, ids[i], j - i, rows_pos + (int64_t)i * row_b)) {
      err->set(ATLAS_ETRUNCATED, std::string(path) + ": rows short");
      return;
    }
    i = j;
  }
  for (uint64_t k = 0; k < s.rows; k++)
    delivery[ids[k]].fetch_add(1, std::memory_order_relaxed);
  bytes->fetch_add((int64_t)s.rows * (row_b + 8), std::memory_order_relaxed);
}

void run_pool(int64_t n, int threads, const std::function<void(int64_t)>& f) {
  std::atomic<int64_t> next{0};
  const int t = std::max(1, std::min<int>(threads, (int)std::max<int64_t>(n, 1)));
  std::vector<std::thread> pool;
  for (int k = 0; k < t; k++)
    pool.emplace_back([&] {
      for (int64_t i; (i = next.fetch_add(1)) < n;) f(i);
    });
  for (auto& th : pool) th.join();
}

int default_threads(int32_t threads) {
  if (threads > 0) return threads;
  const unsigned h = std::thread::hardware_concurrency();
  return (int)std::max(1u, std::min(h, 32u));
}

// Writes nfiles spills spill_0.. into dir plus its manifest. ids_of(f, v)
// fills spill f's ascending id list; rows are gathered from src, the row of
// id v at v * ld elements (ld >= dim; the spill stores dim columns). Runs
// of consecutive ids go out as one write. Returns an ATLAS status.
template <typename IdsOf>
int write_spills(const char* part_dir, const uint8_t* src, int32_t dtype,
                 int64_t dim, int64_t ld, int64_t nfiles, IdsOf ids_of,
                 int32_t threads, int64_t* bytes_written) {
  const int64_t item = dtype == ATLAS_F32 ? 4 : 2;
  const int64_t row_b = dim * item;
  const std::string dir(part_dir);
  std::atomic<int64_t> bytes{0};
  FirstError err;
  run_pool(nfiles, default_threads(threads), [&](int64_t f) {
    std::vector<uint64_t> ids;
    ids_of(f, ids);
    const int64_t nr = (int64_t)ids.size();
    const int64_t ids_pos = kAlign;
    const int64_t rows_pos = ids_pos + align_up(nr * 8);
    const int64_t size = align_up(rows_pos + nr * row_b);
    const std::string path = dir + "/spill_" + std::to_string(f);
    const int fd = ::open(path.c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
    if (fd < 0) {
      err.set(ATLAS_EFORMAT, path + ": cannot create");
      return;
    }
    std::vector<uint8_t> head(kAlign, 0);
    const uint32_t ver = 1, d32 = (uint32_t)dim;
    const uint64_t ulo = ids.front(), uhi = ids.back(), unr = (uint64_t)nr;
    std::memcpy(head.data(), "ASPL", 4);
    std::memcpy(head.data() + 4, &ver, 4);
    std::memcpy(head.data() + 8, &ulo, 8);
    std::memcpy(head.data() + 16, &uhi, 8);
    std::memcpy(head.data() + 24, &unr, 8);
    std::memcpy(head.data() + 32, &d32, 4);
    head[36] = dtype == ATLAS_F32 ? 0 : 1;
    std::vector<uint64_t> idblk((size_t)(rows_pos - ids_pos) / 8, 0);
    std::copy(ids.begin(), ids.end(), idblk.begin());
    bool ok = pwrite_all(fd, head.data(), kAlign, 0) &&
              pwrite_all(fd, idblk.data(), rows_pos - ids_pos, ids_pos);
    for (int64_t i = 0; ok && i < nr;) {
      int64_t j = i + 1;
      if (ld == dim)
        while (j < nr && ids[j] == ids[j - 1] + 1) j++;
      ok = pwrite_all(fd, src + (int64_t)ids[i] * ld * item, (j - i) * row_b,
                      rows_pos + i * row_b);
      i = j;
    }
    const int64_t tail = size - (rows_pos + nr * row_b);
    if (ok && tail > 0) {
      std::vector<uint8_t> zeros((size_t)tail, 0);
      ok = pwrite_all(fd, zeros.data(), tail, rows_pos + nr * row_b);
    }
    ::close(fd);
    if (!ok) {
      err.set(ATLAS_EFORMAT, path + ": write failed");
      return;
    }
    bytes.fetch_add(size, std::memory_order_relaxed);
  });
  if (err.code != ATLAS_OK) {
    set_error(err.msg);
    return err.code;
  }
  // the manifest lists the files in order, like append_manifest
  std::string manifest;
  for (int64_t f = 0; f < nfiles; f++)
    manifest += "spill_" + std::to_string(f) + "\n";
  const std::string mpath = dir + "/manifest.txt";
  const int fd = ::open(mpath.c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
  if (fd < 0 || !pwrite_all(fd, manifest.data(), manifest.size(), 0)) {
    if (fd >= 0) ::close(fd);
    set_error(mpath + ": write failed");
    return ATLAS_EFORMAT;
  }
  ::close(fd);
  if (bytes_written) *bytes_written = bytes.load();
  return ATLAS_OK;
}

// ---- GPUDirect Storage ------------------------------------------------
// cuFile (libcufile from the CUDA toolkit) is resolved at run time: the
// library then loads where cuFile is absent, and the device reader uses
// its own pinned-bounce path when cuFile is not requested or its driver
// does not open.
struct CuFileApi {
  bool ok = false;
  std::string why;
  CUfileError_t (*driver_open)(void) = nullptr;
  CUfileError_t (*handle_register)(CUfileHandle_t*, CUfileDescr_t*) = nullptr;
  void (*handle_deregister)(CUfileHandle_t) = nullptr;
  ssize_t (*read)(CUfileHandle_t, void*, size_t, off_t, off_t) = nullptr;
};

const CuFileApi& cufile() {
  static CuFileApi api = [] {
    CuFileApi a;
    // opt-in: on the pool's boxes a cuFile read of a /tmp file never
    // returned (profiles/r2_gds_probe.txt), so GDS is used only where it
    // was asked for (ATLAS_GDS=1) and the pinned-bounce stream otherwise
    const char* on = getenv("ATLAS_GDS");
    if (!(on && on[0] == '1')) {
      a.why = "cuFile not requested (ATLAS_GDS=1 enables it)";
      return a;
    }
    void* h = dlopen("libcufile.so.0", RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("/usr/local/cuda/lib64/libcufile.so.0",
                       RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      a.why = "libcufile.so.0 not found";
      return a;
    }
    a.driver_open = reinterpret_cast<CUfileError_t (*)(void)>(
        dlsym(h, "cuFileDriverOpen"));
    a.handle_register =
        reinterpret_cast<CUfileError_t (*)(CUfileHandle_t*, CUfileDescr_t*)>(
            dlsym(h, "cuFileHandleRegister"));
    a.handle_deregister = reinterpret_cast<void (*)(CUfileHandle_t)>(
        dlsym(h, "cuFileHandleDeregister"));
    a.read = reinterpret_cast<ssize_t (*)(CUfileHandle_t, void*, size_t,
                                          off_t, off_t)>(
        dlsym(h, "cuFileRead"));
    if (!a.driver_open || !a.handle_register || !a.handle_deregister ||
        !a.read) {
      a.why = "libcufile lacks the cuFile entry points";
      return a;
    }
    const CUfileError_t e = a.driver_open();
    if (e.err != CU_FILE_SUCCESS) {
      a.why = "cuFileDriverOpen failed (" + std::to_string((int)e.err) + ")";
      return a;
    }
    a.ok = true;
    return a;
  }();
  return api;
}

// pinned bounce buffers of one reader thread: pread into one while the
// other's copy engine transfer runs (own non-blocking stream)
struct Bounce {
  static constexpr size_t kBytes = 8 << 20;
  uint8_t* buf[2] = {nullptr, nullptr};
  cudaEvent_t done[2] = {nullptr, nullptr};
  cudaStream_t stream = nullptr;
  int next = 0;
  bool used[2] = {false, false};
  Bounce() {
    for (int i = 0; i < 2; i++) {
      ATLAS_CUDA(cudaMallocHost(&buf[i], kBytes));
      ATLAS_CUDA(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming));
    }
    ATLAS_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  }
  ~Bounce() {
    if (stream) cudaStreamSynchronize(stream);
    for (int i = 0; i < 2; i++) {
      if (buf[i]) cudaFreeHost(buf[i]);
      if (done[i]) cudaEventDestroy(done[i]);
    }
    if (stream) cudaStreamDestroy(stream);
  }
  // file bytes [off, off + n) -> device dst
  bool move(int fd, uint8_t* dst, size_t n, int64_t off) {
    while (n) {
      const size_t m = std::min(n, kBytes);
      const int b = next;
      next ^= 1;
      if (used[b]) ATLAS_CUDA(cudaEventSynchronize(done[b]));
      if (!pread_all(fd, buf[b], m, off)) return false;
      ATLAS_CUDA(cudaMemcpyAsync(dst, buf[b], m, cudaMemcpyHostToDevice,
                                 stream));
      ATLAS_CUDA(cudaEventRecord(done[b], stream));
      used[b] = true;
      dst += m;
      off += (int64_t)m;
      n -= m;
    }
    return true;
  }
};

// pinned bounce buffers are kept between calls (a cudaMallocHost per
// call and thread cost more than the reads of a small layer directory)
struct BounceLease {
  int dev;
  Bounce* b = nullptr;
  static std::mutex& mu() {
    static std::mutex m;
    return m;
  }
  static std::vector<std::pair<int, Bounce*>>& pool() {
    static std::vector<std::pair<int, Bounce*>> p;  // process lifetime
    return p;
  }
  explicit BounceLease(int d) : dev(d) {}
  Bounce* get() {
    if (b) return b;
    {
      std::lock_guard<std::mutex> lock(mu());
      auto& p = pool();
      for (size_t i = 0; i < p.size(); i++)
        if (p[i].first == dev) {
          b = p[i].second;
          p.erase(p.begin() + i);
          break;
        }
    }
    if (!b) b = new Bounce();
    return b;
  }
  ~BounceLease() {
    if (!b) return;
    std::lock_guard<std::mutex> lock(mu());
    pool().emplace_back(dev, b);
  }
};

}  // namespace
}  // namespace atlas

using namespace atlas;

extern "C" {

int atlas_spill_read(const char* const* paths, int32_t n_files,
                     int32_t dtype, int64_t dim, int64_t num_vertices,
                     void* rows_out, uint16_t* delivery_out, int32_t threads,
                     int64_t* bytes_read) {
  try {
    if ((!paths && n_files) || !rows_out || dim < 1 || num_vertices < 0 ||
        (dtype != ATLAS_F32 && dtype != ATLAS_F16)) {
      set_error("atlas_spill_read: bad arguments");
      return ATLAS_ECONFIG;
    }
    std::vector<std::atomic<uint16_t>> delivery((size_t)num_vertices);
    for (auto& d : delivery) d.store(0, std::memory_order_relaxed);
    std::atomic<int64_t> bytes{0};
    FirstError err;
    uint8_t* out = static_cast<uint8_t*>(rows_out);
    const int64_t row_b = dim * (dtype == ATLAS_F32 ? 4 : 2);
    const RunSink host_sink = [&](int fd, uint64_t id, uint64_t nrows,
                                  int64_t off) {
      return pread_all(fd, out + id * row_b, nrows * row_b, off);
    };
    run_pool(n_files, default_threads(threads), [&](int64_t i) {
      read_one(paths[i], dtype, dim, num_vertices, host_sink, delivery.data(),
               &bytes, &err);
    });
    if (err.code != ATLAS_OK) {
      set_error(err.msg);
      return err.code;
    }
    int64_t bad = 0, first = -1;
    for (int64_t v = 0; v < num_vertices; v++) {
      const uint16_t c = delivery[v].load(std::memory_order_relaxed);
      if (delivery_out) delivery_out[v] = c;
      if (c != 1) {
        if (first < 0) first = v;
        bad++;
      }
    }
    if (bytes_read) *bytes_read = bytes.load();
    if (bad) {
      set_error(std::to_string(bad) + " ids not delivered exactly once, first " +
                std::to_string(first));
      return ATLAS_ECOVERAGE;
    }
    return ATLAS_OK;
  } catch (const std::exception& e) {
    set_error(std::string("atlas_spill_read: ") + e.what());
    return ATLAS_EINVARIANT;
  }
}

int atlas_spill_read_device(const char* const* paths, int32_t n_files,
                            int32_t dtype, int64_t dim, int64_t num_vertices,
                            void* rows_dev, uint16_t* delivery_out,
                            int32_t threads, int64_t* bytes_read,
                            int32_t* used_gds) {
  try {
    if ((!paths && n_files) || dim < 1 || num_vertices < 0 ||
        (dtype != ATLAS_F32 && dtype != ATLAS_F16)) {
      set_error("atlas_spill_read_device: bad arguments");
      return ATLAS_ECONFIG;
    }
    // rows_dev == NULL: validate the directory (headers, sizes, ids,
    // coverage) without reading rows or touching the device
    const bool validate_only = rows_dev == nullptr;
    ATLAS_NVTX("atlas_spill_read_device");
    std::vector<std::atomic<uint16_t>> delivery((size_t)num_vertices);
    for (auto& d : delivery) d.store(0, std::memory_order_relaxed);
    std::atomic<int64_t> bytes{0};
    FirstError err;
    uint8_t* out = static_cast<uint8_t*>(rows_dev);
    const int64_t row_b = dim * (dtype == ATLAS_F32 ? 4 : 2);
    const CuFileApi& cf = cufile();
    const int nthreads = default_threads(threads);
    const int64_t nf = n_files;
    std::atomic<int64_t> next{0};
    int dev = 0;
    if (!validate_only) ATLAS_CUDA(cudaGetDevice(&dev));
    auto worker = [&] {
      try {
        if (!validate_only) cudaSetDevice(dev);
        BounceLease bounce(dev);
        for (int64_t i; (i = next.fetch_add(1)) < nf;) {
          CUfileHandle_t fh = nullptr;
          bool reg = false;
          // rows land at their ids: runs of consecutive ids are one
          // storage -> HBM transfer (cuFileRead) or one bounce stream
          const RunSink sink = [&](int fd, uint64_t id, uint64_t nrows,
                                   int64_t off) -> bool {
            const size_t n = (size_t)(nrows * row_b);
            if (validate_only) return true;
            if (cf.ok) {
              if (!reg) {
                CUfileDescr_t d{};
                d.type = CU_FILE_HANDLE_TYPE_OPAQUE_FD;
                d.handle.fd = fd;
                if (cf.handle_register(&fh, &d).err != CU_FILE_SUCCESS)
                  return false;
                reg = true;
              }
              size_t done = 0;
              while (done < n) {
                const ssize_t r = cf.read(fh, out, n - done,
                                          (off_t)(off + (int64_t)done),
                                          (off_t)(id * row_b + done));
                if (r <= 0) return false;
                done += (size_t)r;
              }
              return true;
            }
            return bounce.get()->move(fd, out + id * row_b, n, off);
          };
          read_one(paths[i], dtype, dim, num_vertices, sink, delivery.data(),
                   &bytes, &err);
          if (reg) cf.handle_deregister(fh);
        }
        if (bounce.b) ATLAS_CUDA(cudaStreamSynchronize(bounce.b->stream));
      } catch (const Error& e) {
        err.set(e.code, e.msg);
      }
    };
    std::vector<std::thread> pool;
    const int t = std::max(1, std::min<int>(nthreads, (int)std::max<int64_t>(nf, 1)));
    for (int k = 0; k < t; k++) pool.emplace_back(worker);
    for (auto& th : pool) th.join();
    if (used_gds) *used_gds = cf.ok && !validate_only ? 1 : 0;
    if (err.code != ATLAS_OK) {
      set_error(err.msg);
      return err.code;
    }
    int64_t bad = 0, first = -1;
    for (int64_t v = 0; v < num_vertices; v++) {
      const uint16_t c = delivery[v].load(std::memory_order_relaxed);
      if (delivery_out) delivery_out[v] = c;
      if (c != 1) {
        if (first < 0) first = v;
        bad++;
      }
    }
    if (bytes_read) *bytes_read = bytes.load();
    if (bad) {
      set_error(std::to_string(bad) + " ids not delivered exactly once, first " +
                std::to_string(first));
      return ATLAS_ECOVERAGE;
    }
    return ATLAS_OK;
  } catch (const std::exception& e) {
    set_error(std::string("atlas_spill_read_device: ") + e.what());
    return ATLAS_EINVARIANT;
  }
}

const char* atlas_gds_status(void) {
  const CuFileApi& cf = cufile();
  static std::string s;
  s = cf.ok ? "cuFile" : "bounce: " + cf.why;
  return s.c_str();
}

int atlas_spill_write(const char* part_dir, const void* rows, int32_t dtype,
                      int64_t dim, int64_t ld, int64_t id_lo, int64_t id_hi,
                      int64_t spill_rows, int32_t threads,
                      int64_t* bytes_written) {
  try {
    if (!part_dir || (!rows && id_hi > id_lo) || dim < 1 || ld < dim ||
        id_lo < 0 || id_hi < id_lo ||
        (dtype != ATLAS_F32 && dtype != ATLAS_F16)) {
      set_error("atlas_spill_write: bad arguments");
      return ATLAS_ECONFIG;
    }
    const int64_t n = id_hi - id_lo;
    const int64_t step = spill_rows > 0 ? spill_rows : std::max<int64_t>(n, 1);
    const int64_t nfiles = n > 0 ? ceil_div(n, step) : 0;
    // rows holds ids [id_lo, id_hi): row of id v at (v - id_lo) * ld
    const auto* src = static_cast<const uint8_t*>(rows) -
                      id_lo * ld * (dtype == ATLAS_F32 ? 4 : 2);
    return write_spills(
        part_dir, src, dtype, dim, ld, nfiles,
        [&](int64_t f, std::vector<uint64_t>& ids) {
          const int64_t lo = id_lo + f * step, hi = std::min(id_hi, lo + step);
          ids.resize(hi - lo);
          for (int64_t i = 0; i < hi - lo; i++) ids[i] = (uint64_t)(lo + i);
        },
        threads, bytes_written);
  } catch (const std::exception& e) {
    set_error(std::string("atlas_spill_write: ") + e.what());
    return ATLAS_EINVARIANT;
  }
}

int atlas_spill_write_runs(const char* part_dir, const void* rows,
                           int32_t dtype, int64_t dim, int64_t ld,
                           const int64_t* ids, const int64_t* spill_start,
                           int64_t nspills, int32_t threads,
                           int64_t* bytes_written) {
  try {
    if (!part_dir || dim < 1 || ld < dim || nspills < 0 ||
        (nspills && (!rows || !ids || !spill_start)) ||
        (dtype != ATLAS_F32 && dtype != ATLAS_F16)) {
      set_error("atlas_spill_write_runs: bad arguments");
      return ATLAS_ECONFIG;
    }
    for (int64_t f = 0; f < nspills; f++) {
      const int64_t a = spill_start[f], b = spill_start[f + 1];
      if (b <= a) {
        set_error("atlas_spill_write_runs: empty spill");
        return ATLAS_EINVARIANT;
      }
      for (int64_t i = a; i < b; i++)
        if (ids[i] < 0 || (i > a && ids[i] <= ids[i - 1])) {
          set_error("atlas_spill_write_runs: spill ids must ascend");
          return ATLAS_EINVARIANT;
        }
    }
    return write_spills(
        part_dir, static_cast<const uint8_t*>(rows), dtype, dim, ld, nspills,
        [&](int64_t f, std::vector<uint64_t>& out) {
          const int64_t a = spill_start[f], b = spill_start[f + 1];
          out.assign(ids + a, ids + b);
        },
        threads, bytes_written);
  } catch (const std::exception& e) {
    set_error(std::string("atlas_spill_write_runs: ") + e.what());
    return ATLAS_EINVARIANT;
  }
}

}  // extern "C"
