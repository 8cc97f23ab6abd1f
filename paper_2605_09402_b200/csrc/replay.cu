// Gather-pattern read replay (the quantity
// oocgnn/bench.py:282-305 `simulate_gather_rows` reports): how many rows a
// destination-major gather engine loads in one layer when every in-neighbour
// row goes through an LRU cache of `cache_rows` rows, fetched in blocks of
// `block_rows` consecutive ids. Host-only code (no device work).
//
// The reference walks the access stream through an OrderedDict. Here the
// answer comes from reuse distances instead: an access hits an LRU cache of
// C blocks iff fewer than C DISTINCT other blocks were touched since the
// previous access to the same block. A Fenwick tree over stream positions
// holds a 1 at the latest access of every block, so the distinct count is a
// range sum -- O(E log E) with no hashing, exact for every C.
//
// Access order: destinations ascending, each destination's in-neighbours in
// ascending source id (the transposed CSR a gather engine walks). A counting
// sort of the CSR by destination gives exactly that order, because sources
// are emitted in ascending id.
#include <cstdint>
#include <vector>

#include "internal.cuh"

namespace atlas {
namespace {

struct Fenwick {
  std::vector<int32_t> t;
  explicit Fenwick(int64_t n) : t(n + 1, 0) {}
  void add(int64_t i, int32_t v) {
    for (++i; i < (int64_t)t.size(); i += i & -i) t[i] += v;
  }
  int64_t prefix(int64_t i) const {  // sum over [0, i)
    int64_t s = 0;
    for (; i > 0; i -= i & -i) s += t[i];
    return s;
  }
};

}  // namespace
}  // namespace atlas

using namespace atlas;

extern "C" {

int atlas_gather_replay(int64_t num_vertices, int64_t num_edges,
                        const int64_t* offsets, const uint32_t* neighbors,
                        int64_t cache_rows, int64_t block_rows,
                        int64_t* rows_loaded) {
  try {
    if (num_vertices < 0 || num_edges < 0 || !rows_loaded ||
        (num_vertices && !offsets) || (num_edges && !neighbors) ||
        block_rows < 1 || cache_rows < 0) {
      set_error("atlas_gather_replay: bad arguments");
      return ATLAS_ECONFIG;
    }
    const int64_t cap = cache_rows / block_rows;
    if (cap == 0 || num_edges == 0) {  // every touch is a load
      *rows_loaded = num_edges * block_rows;
      return ATLAS_OK;
    }
    // transposed CSR by counting sort: per destination, sources ascending
    std::vector<int64_t> start(num_vertices + 1, 0);
    for (int64_t e = 0; e < num_edges; ++e) {
      const uint32_t d = neighbors[e];
      if ((int64_t)d >= num_vertices) {
        set_error("atlas_gather_replay: neighbour id out of range");
        return ATLAS_ECONSISTENCY;
      }
      ++start[d + 1];
    }
    for (int64_t v = 0; v < num_vertices; ++v) start[v + 1] += start[v];
    std::vector<int64_t> fill(start.begin(), start.end() - 1);
    std::vector<int64_t> blocks(num_edges);
    for (int64_t s = 0; s < num_vertices; ++s)
      for (int64_t e = offsets[s]; e < offsets[s + 1]; ++e)
        blocks[fill[neighbors[e]]++] = s / block_rows;

    const int64_t nblocks = (num_vertices + block_rows - 1) / block_rows;
    std::vector<int64_t> last(nblocks, -1);
    Fenwick fw(num_edges);
    int64_t loads = 0;
    for (int64_t i = 0; i < num_edges; ++i) {
      const int64_t b = blocks[i];
      const int64_t p = last[b];
      if (p < 0) {
        ++loads;  // cold miss
      } else {
        // distinct blocks touched strictly between p and i
        const int64_t distinct = fw.prefix(i) - fw.prefix(p + 1);
        if (distinct >= cap) ++loads;
        fw.add(p, -1);
      }
      fw.add(i, 1);
      last[b] = i;
    }
    *rows_loaded = loads * block_rows;
    return ATLAS_OK;
  } catch (const std::exception& ex) {
    set_error(std::string("atlas_gather_replay: ") + ex.what());
    return ATLAS_EINVARIANT;
  }
}

}  // extern "C"
