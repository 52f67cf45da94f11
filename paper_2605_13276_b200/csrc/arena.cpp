// Dual-pool arena allocator (host-side bookkeeping over a device slab).
//
// Reference: pkg/src/dvla/pools.py:72-212 (Pool.alloc / free / _insert_free /
// epoch_reset / stats) and kernels/numba_backend.py:139-247 (alloc_trace_run).
// Placement decisions are integer-exact copies of the reference policy:
// first fit over an offset-sorted free list, aligned start, lead/tail split,
// coalescing free, generation-stamped handles, O(1) epoch reset for ENV_AUX.
// The arena never touches device memory itself: offsets index a cudaMalloc'd
// slab (dvla_dev_alloc) that the Python Pool exposes as zero-copy views.
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/dvla_b200.h"

namespace dvla {
int fail(int code, const char* fmt, ...);
}

namespace {

const char* kind_name(int kind) {
  switch (kind) {
    case DVLA_POOL_MODEL_COMPUTE: return "model_compute";
    case DVLA_POOL_ENV_AUX: return "env_aux";
    default: return "unified_baseline";
  }
}

struct Live {
  int64_t offset, size, generation;
};

}  // namespace

struct dvla_arena {
  int kind;
  int64_t capacity;
  int64_t pool_id;
  int64_t generation = 0;
  std::vector<int64_t> free_off, free_size;
  std::unordered_map<int64_t, Live> live;  // serial -> block
  int64_t next_serial = 1;
  int64_t alloc_count = 0, free_count = 0, failed_allocs = 0, churn_bytes = 0;
  int torch_bound = 0;   // hosting torch's segments (dvla_torch_pool_bind): no epoch reset
  std::mutex mu;
};

static std::atomic<int64_t> g_pool_ids{1};

static std::string handle_repr(int64_t pool_id, int64_t offset, int64_t size, int64_t gen,
                               int64_t serial) {
  char b[192];
  snprintf(b, sizeof(b),
           "PoolHandle(pool_id=%lld, offset=%lld, size=%lld, generation=%lld, serial=%lld)",
           (long long)pool_id, (long long)offset, (long long)size, (long long)gen,
           (long long)serial);
  return b;
}

// first-fit placement (pools.py:98-118); returns offset or -1
static int64_t place(std::vector<int64_t>& fo, std::vector<int64_t>& fs, int64_t size,
                     int64_t align) {
  for (size_t j = 0; j < fo.size(); ++j) {
    const int64_t o = fo[j], s = fs[j];
    const int64_t a = ((o + align - 1) / align) * align;
    if (a + size <= o + s) {
      const int64_t lead = a - o, tail = (o + s) - (a + size);
      if (lead > 0 && tail > 0) {
        fs[j] = lead;
        fo.insert(fo.begin() + j + 1, a + size);
        fs.insert(fs.begin() + j + 1, tail);
      } else if (lead > 0) {
        fs[j] = lead;
      } else if (tail > 0) {
        fo[j] = a + size;
        fs[j] = tail;
      } else {
        fo.erase(fo.begin() + j);
        fs.erase(fs.begin() + j);
      }
      return a;
    }
  }
  return -1;
}

// coalescing insert (pools.py:143-158)
static void insert_free(std::vector<int64_t>& fo, std::vector<int64_t>& fs, int64_t off,
                        int64_t size) {
  const size_t j = std::lower_bound(fo.begin(), fo.end(), off) - fo.begin();
  const bool mp = j > 0 && fo[j - 1] + fs[j - 1] == off;
  const bool mn = j < fo.size() && off + size == fo[j];
  if (mp && mn) {
    fs[j - 1] += size + fs[j];
    fo.erase(fo.begin() + j);
    fs.erase(fs.begin() + j);
  } else if (mp) {
    fs[j - 1] += size;
  } else if (mn) {
    fo[j] = off;
    fs[j] += size;
  } else {
    fo.insert(fo.begin() + j, off);
    fs.insert(fs.begin() + j, size);
  }
}

extern "C" int dvla_arena_create(int kind, int64_t capacity, dvla_arena** out,
                                 int64_t* pool_id_out) {
  if (!out) return dvla::fail(DVLA_ERR_USAGE, "null out pointer");
  if (capacity <= 0)
    return dvla::fail(DVLA_ERR_CONFIG, "pool capacity must be > 0, got %lld", (long long)capacity);
  if (kind < DVLA_POOL_MODEL_COMPUTE || kind > DVLA_POOL_UNIFIED_BASELINE)
    return dvla::fail(DVLA_ERR_USAGE, "unknown pool kind %d", kind);
  dvla_arena* a = new dvla_arena();
  a->kind = kind;
  a->capacity = capacity;
  a->pool_id = g_pool_ids.fetch_add(1);
  a->free_off.push_back(0);
  a->free_size.push_back(capacity);
  *out = a;
  if (pool_id_out) *pool_id_out = a->pool_id;
  return DVLA_OK;
}

extern "C" int dvla_arena_destroy(dvla_arena* a) {
  delete a;
  return DVLA_OK;
}

extern "C" int dvla_arena_alloc(dvla_arena* a, int64_t size, int64_t align, int64_t* offset_out,
                                int64_t* serial_out, int64_t* generation_out) {
  if (!a) return dvla::fail(DVLA_ERR_USAGE, "null arena");
  if (size <= 0) return dvla::fail(DVLA_ERR_CONFIG, "alloc size must be > 0, got %lld", (long long)size);
  if (align < 1 || (align & (align - 1)) != 0)
    return dvla::fail(DVLA_ERR_CONFIG, "align must be a power of two, got %lld", (long long)align);
  std::lock_guard<std::mutex> g(a->mu);
  const int64_t off = place(a->free_off, a->free_size, size, align);
  if (off < 0) {
    a->failed_allocs += 1;
    return dvla::fail(DVLA_ERR_ALLOC_FAILURE, "%s pool cannot place %lld bytes @align %lld",
                      kind_name(a->kind), (long long)size, (long long)align);
  }
  const int64_t serial = a->next_serial++;
  a->live[serial] = Live{off, size, a->generation};
  a->alloc_count += 1;
  a->churn_bytes += size;
  if (offset_out) *offset_out = off;
  if (serial_out) *serial_out = serial;
  if (generation_out) *generation_out = a->generation;
  return DVLA_OK;
}

extern "C" int dvla_arena_free(dvla_arena* a, int64_t pool_id, int64_t offset, int64_t size,
                               int64_t generation, int64_t serial) {
  if (!a) return dvla::fail(DVLA_ERR_USAGE, "null arena");
  std::lock_guard<std::mutex> g(a->mu);
  const std::string h = handle_repr(pool_id, offset, size, generation, serial);
  if (pool_id != a->pool_id)
    return dvla::fail(DVLA_ERR_POOL_USAGE, "handle %s belongs to another pool", h.c_str());
  if (generation != a->generation)
    return dvla::fail(DVLA_ERR_POOL_USAGE, "stale handle %s: generation %lld != %lld", h.c_str(),
                      (long long)generation, (long long)a->generation);
  auto it = a->live.find(serial);
  if (it == a->live.end())
    return dvla::fail(DVLA_ERR_POOL_USAGE, "double free of %s", h.c_str());
  const Live blk = it->second;
  a->live.erase(it);
  insert_free(a->free_off, a->free_size, blk.offset, blk.size);
  a->free_count += 1;
  return DVLA_OK;
}

extern "C" int dvla_arena_epoch_reset(dvla_arena* a) {
  if (!a) return dvla::fail(DVLA_ERR_USAGE, "null arena");
  std::lock_guard<std::mutex> g(a->mu);
  if (a->kind != DVLA_POOL_ENV_AUX)
    return dvla::fail(DVLA_ERR_POOL_USAGE,
                      "epoch_reset on a %s pool; model allocations are long-lived by contract",
                      kind_name(a->kind));
  if (a->torch_bound)
    return dvla::fail(DVLA_ERR_POOL_USAGE,
                      "epoch_reset on a pool that hosts torch's allocations (unbind it first)");
  a->generation += 1;
  a->live.clear();
  a->free_off.assign(1, 0);
  a->free_size.assign(1, a->capacity);
  return DVLA_OK;
}

extern "C" int dvla_arena_is_live(dvla_arena* a, int64_t generation, int64_t serial, int* out) {
  if (!a || !out) return dvla::fail(DVLA_ERR_USAGE, "null pointer argument");
  std::lock_guard<std::mutex> g(a->mu);
  *out = (generation == a->generation && a->live.count(serial)) ? 1 : 0;
  return DVLA_OK;
}

extern "C" int dvla_arena_stats(dvla_arena* a, int64_t* out) {
  if (!a || !out) return dvla::fail(DVLA_ERR_USAGE, "null pointer argument");
  std::lock_guard<std::mutex> g(a->mu);
  int64_t total = 0, largest = 0;
  for (int64_t s : a->free_size) {
    total += s;
    largest = std::max(largest, s);
  }
  out[0] = a->capacity - total;  // live_bytes
  out[1] = total;
  out[2] = largest;
  out[3] = a->failed_allocs;
  out[4] = a->alloc_count;
  out[5] = a->free_count;
  out[6] = a->churn_bytes;
  out[7] = a->generation;
  out[8] = static_cast<int64_t>(a->free_off.size());
  return DVLA_OK;
}

// Batched trace (numba_backend.py:139-247): out_ok 1 placed / 0 failed,
// 3 freed / 2 free skipped (no live block); out_off = offset or -1.
extern "C" int dvla_arena_trace(int64_t capacity, int64_t n, const uint8_t* is_alloc,
                                const int64_t* size, const int64_t* align, const uint64_t* pick,
                                uint8_t* out_ok, int64_t* out_off, int64_t* final_out) {
  if (capacity <= 0) return dvla::fail(DVLA_ERR_CONFIG, "pool capacity must be > 0, got %lld", (long long)capacity);
  if (n < 0 || (n > 0 && (!is_alloc || !size || !align || !pick || !out_ok || !out_off)))
    return dvla::fail(DVLA_ERR_USAGE, "bad trace arguments");
  std::vector<int64_t> fo{0}, fs{capacity};
  std::vector<int64_t> live_ids;  // birth order
  live_ids.reserve(static_cast<size_t>(n));
  std::vector<int64_t> blk_off(static_cast<size_t>(n)), blk_size(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    if (is_alloc[i] == 1) {
      const int64_t al = align[i];
      if (al < 1 || (al & (al - 1)) != 0 || size[i] <= 0)
        return dvla::fail(DVLA_ERR_CONFIG, "trace op %lld: bad size/align", (long long)i);
      const int64_t off = place(fo, fs, size[i], al);
      if (off < 0) {
        out_ok[i] = 0;
        out_off[i] = -1;
        continue;
      }
      out_ok[i] = 1;
      out_off[i] = off;
      live_ids.push_back(i);
      blk_off[i] = off;
      blk_size[i] = size[i];
    } else {
      if (live_ids.empty()) {
        out_ok[i] = 2;
        out_off[i] = -1;
        continue;
      }
      const size_t idx = static_cast<size_t>(pick[i] % static_cast<uint64_t>(live_ids.size()));
      const int64_t tgt = live_ids[idx];
      live_ids.erase(live_ids.begin() + idx);
      insert_free(fo, fs, blk_off[tgt], blk_size[tgt]);
      out_ok[i] = 3;
      out_off[i] = blk_off[tgt];
    }
  }
  if (final_out) {
    int64_t total = 0, largest = 0;
    for (int64_t s : fs) {
      total += s;
      largest = std::max(largest, s);
    }
    final_out[0] = total;
    final_out[1] = largest;
    final_out[2] = static_cast<int64_t>(fs.size());
  }
  return DVLA_OK;
}

// ---- torch's caching allocator on top of an ENV_AUX arena
//
// torch temporaries (activations, concatenations, the
// sampler's observation tensors) belong in the recycled pool, not in
// torch's own cudaMalloc segments.  dvla_torch_alloc / dvla_torch_free have
// the signatures of torch.cuda.memory.CUDAPluggableAllocator; inside a
// torch.cuda.MemPool built on them, every segment torch requests is placed
// by the first-fit arena bound to that device (pools.torch_arena) in that
// arena's device slab.  Torch sub-allocates and caches within its segments.
namespace {
struct TorchBinding {
  dvla_arena* arena = nullptr;
  uintptr_t base = 0;
  std::unordered_map<uintptr_t, std::pair<int64_t, int64_t>> live;  // ptr -> (serial, gen)
  std::mutex mu;
};
TorchBinding g_torch[64];
}  // namespace

extern "C" int dvla_torch_pool_bind(int device, dvla_arena* a, void* base) {
  if (device < 0 || device >= 64) return dvla::fail(DVLA_ERR_USAGE, "device out of range");
  TorchBinding& b = g_torch[device];
  std::lock_guard<std::mutex> g(b.mu);
  if (a && (!base || a->kind != DVLA_POOL_ENV_AUX))
    return dvla::fail(DVLA_ERR_USAGE, "torch allocations bind to an ENV_AUX device pool");
  if (a && b.arena && b.arena != a)
    return dvla::fail(DVLA_ERR_POOL_USAGE, "device %d already hosts torch in another pool",
                      device);
  if (!a && !b.live.empty())
    return dvla::fail(DVLA_ERR_POOL_USAGE, "%zu torch segments still live in the pool",
                      b.live.size());
  if (b.arena) {
    std::lock_guard<std::mutex> ga(b.arena->mu);
    b.arena->torch_bound = 0;
  }
  b.arena = a;
  b.base = reinterpret_cast<uintptr_t>(base);
  if (a) {
    std::lock_guard<std::mutex> ga(a->mu);
    a->torch_bound = 1;
  }
  return DVLA_OK;
}

extern "C" void* dvla_torch_alloc(size_t size, int device, void* stream) {
  (void)stream;
  if (device < 0 || device >= 64 || size == 0) return nullptr;
  TorchBinding& b = g_torch[device];
  std::lock_guard<std::mutex> g(b.mu);
  if (!b.arena) return nullptr;
  int64_t off = 0, serial = 0, gen = 0;
  if (dvla_arena_alloc(b.arena, static_cast<int64_t>(size), 512, &off, &serial, &gen) != DVLA_OK)
    return nullptr;  // torch reports out of memory for the pool
  const uintptr_t p = b.base + static_cast<uintptr_t>(off);
  b.live[p] = {serial, gen};
  return reinterpret_cast<void*>(p);
}

extern "C" void dvla_torch_free(void* ptr, size_t size, int device, void* stream) {
  (void)stream;
  if (device < 0 || device >= 64 || !ptr) return;
  TorchBinding& b = g_torch[device];
  std::lock_guard<std::mutex> g(b.mu);
  auto it = b.live.find(reinterpret_cast<uintptr_t>(ptr));
  if (!b.arena || it == b.live.end()) return;
  const int64_t off = static_cast<int64_t>(reinterpret_cast<uintptr_t>(ptr) - b.base);
  dvla_arena_free(b.arena, b.arena->pool_id, off, static_cast<int64_t>(size), it->second.second,
                  it->second.first);
  b.live.erase(it);
}
