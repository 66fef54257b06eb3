// Common infrastructure for the B200 IFMM library: error handling, device
// arenas, launch helpers and warp/block reductions.  sm_100a only.
#pragma once
#include <cuda_runtime.h>
#include <atomic>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

namespace ifmm {

// ---------------------------------------------------------------- errors
enum Status : int {
  IFMM_OK = 0,
  IFMM_INVALID = 1,         // -> ValueError
  IFMM_SINGULAR_PIVOT = 2,  // -> SingularPivotError(level, index, cond)
  IFMM_CUDA = 3,            // -> RuntimeError
  IFMM_OOM = 4,             // -> MemoryError
  IFMM_NO_DEVICE = 5,       // -> RuntimeError (no CUDA device: no CPU fallback)
};

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

struct SingularPivot : Error {
  int level, index;
  double cond;
  SingularPivot(int lv, int ix, double c, const std::string& m)
      : Error(IFMM_SINGULAR_PIVOT, m), level(lv), index(ix), cond(c) {}
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) {
    char buf[512];
    snprintf(buf, sizeof buf, "CUDA error %s (%s) at %s:%d: %s", cudaGetErrorName(e), what, file, line,
             cudaGetErrorString(e));
    throw Error(e == cudaErrorMemoryAllocation ? IFMM_OOM : IFMM_CUDA, buf);
  }
}
// every kernel launch of the library goes through CK_LAUNCH: count them
inline std::atomic<long long>& launch_counter() {
  static std::atomic<long long> c{0};
  return c;
}
#define CK(x) ::ifmm::cuda_check((x), #x, __FILE__, __LINE__)
#define CK_LAUNCH()                                                                  \
  do {                                                                               \
    ::ifmm::launch_counter().fetch_add(1, std::memory_order_relaxed);                \
    ::ifmm::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__);     \
  } while (0)

[[noreturn]] inline void invalid(const std::string& m) { throw Error(IFMM_INVALID, m); }

// ---------------------------------------------------------------- slab cache
// Process-wide cache of device slabs.  cudaMalloc of multi-GB slabs costs
// tens of ms and cudaFree synchronises the device, so arenas (factorization
// records, per-call workspaces) return their slabs here and later arenas
// reuse them; the cache is flushed when an allocation would otherwise fail.
// A slab is only released after the work using it has been synchronised (the
// C API is synchronous), so reuse needs no stream ordering.
struct SlabCache {
  std::mutex mu;
  std::multimap<std::pair<int, size_t>, void*> free;  // (device, bytes) -> ptr
  size_t cached = 0;
  static constexpr size_t kMaxCached = size_t(64) << 30;
};
inline SlabCache& slab_cache() {
  static SlabCache* c = new SlabCache();  // never destroyed: slabs outlive static teardown
  return *c;
}
inline void slab_cache_flush(int dev) {
  SlabCache& c = slab_cache();
  std::lock_guard<std::mutex> lk(c.mu);
  for (auto it = c.free.begin(); it != c.free.end();) {
    if (it->first.first == dev) {
      cudaFree(it->second);
      c.cached -= it->first.second;
      it = c.free.erase(it);
    } else {
      ++it;
    }
  }
}
// A cached slab of at least `bytes` (and at most 2x), else a new one; *got =
// its size.  Returns nullptr if the device is out of memory even after a flush.
inline void* slab_get(size_t bytes, size_t* got) {
  int dev = 0;
  cudaGetDevice(&dev);
  SlabCache& c = slab_cache();
  {
    std::lock_guard<std::mutex> lk(c.mu);
    auto it = c.free.lower_bound({dev, bytes});
    if (it != c.free.end() && it->first.first == dev && it->first.second <= 2 * bytes) {
      void* p = it->second;
      *got = it->first.second;
      c.cached -= *got;
      c.free.erase(it);
      return p;
    }
  }
  void* p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) {
    cudaGetLastError();
    slab_cache_flush(dev);
    if (cudaMalloc(&p, bytes) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
  }
  *got = bytes;
  return p;
}
inline void slab_put(void* p, size_t bytes) {
  int dev = 0;
  cudaGetDevice(&dev);
  SlabCache& c = slab_cache();
  std::lock_guard<std::mutex> lk(c.mu);
  if (c.cached + bytes > SlabCache::kMaxCached) {
    cudaFree(p);
    return;
  }
  c.free.insert({{dev, bytes}, p});
  c.cached += bytes;
}

// ---------------------------------------------------------------- arena
// Bump allocator over large device slabs (from the slab cache).  Reset releases
// everything at once (per level / per batch workspaces); slabs are kept for
// reuse and go back to the cache when the arena is destroyed.
class Arena {
 public:
  explicit Arena(size_t slab = size_t(256) << 20) : slab_(slab) {}
  ~Arena() { release(); }
  Arena(const Arena&) = delete;
  Arena& operator=(const Arena&) = delete;

  void* alloc(size_t bytes, size_t align = 256) {
    if (bytes == 0) bytes = align;
    for (;;) {
      if (cur_ < slabs_.size()) {
        Slab& s = slabs_[cur_];
        size_t off = (s.used + align - 1) / align * align;
        if (off + bytes <= s.size) {
          s.used = off + bytes;
          in_use_ += bytes;
          if (zero_) zero_upto(s, s.used);
          return static_cast<char*>(s.ptr) + off;
        }
        ++cur_;
        continue;
      }
      size_t sz = bytes > slab_ ? bytes : slab_;
      void* p = slab_get(sz, &sz);
      if (p == nullptr) {
        char buf[256];
        snprintf(buf, sizeof buf, "device allocation of %.3f GB failed (arena holds %.3f GB)", sz / 1e9,
                 reserved() / 1e9);
        throw Error(IFMM_OOM, buf);
      }
      // a slab from the cache holds whatever its last user left: all of it may be non-zero
      slabs_.push_back({p, sz, 0, zero_ ? sz : 0, 0});
      cur_ = slabs_.size() - 1;
    }
  }
  // When set, every allocation starts as zeros: cleared on `s` when it is handed out (lazily, see reset()).
  void set_zero_stream(cudaStream_t s) { zero_stream_ = s; zero_ = true; }
  template <class T>
  T* alloc_n(size_t n) {
    return static_cast<T*>(alloc(n * sizeof(T)));
  }
  // Zeroing is lazy (zero arenas): a reset only notes how far each slab may hold old data; the
  // allocations of the next round clear what they take, 256 MB ahead at a time, stream-ordered
  // before any work that can touch the memory.  A level that needs a quarter of what the level
  // before it used clears a quarter (C3: ~150 GB of memsets per factorization otherwise).
  void reset() {
    for (auto& s : slabs_) {
      const size_t stale = s.zeroed < s.dirty ? s.dirty : 0;  // old data beyond what this round cleared
      s.dirty = zero_ ? (s.used > stale ? s.used : stale) : 0;
      s.zeroed = 0;
      s.used = 0;
    }
    cur_ = 0;
    in_use_ = 0;
  }
  void release() {
    for (auto& s : slabs_) slab_put(s.ptr, s.size);
    slabs_.clear();
    cur_ = 0;
    in_use_ = 0;
  }
  size_t reserved() const {
    size_t t = 0;
    for (auto& s : slabs_) t += s.size;
    return t;
  }
  size_t in_use() const { return in_use_; }

 private:
  struct Slab {
    void* ptr;
    size_t size;
    size_t used;
    size_t dirty;   // zero arenas: bytes [0, dirty) may hold old data, the rest of the slab is zero
    size_t zeroed;  // bytes [0, zeroed) have been cleared since the last reset
  };
  void zero_upto(Slab& s, size_t end) {
    const size_t need = end < s.dirty ? end : s.dirty;
    if (s.zeroed >= need) return;
    constexpr size_t kAhead = size_t(256) << 20;
    size_t to = s.zeroed + kAhead > need ? s.zeroed + kAhead : need;
    if (to > s.dirty) to = s.dirty;
    if (cudaMemsetAsync(static_cast<char*>(s.ptr) + s.zeroed, 0, to - s.zeroed, zero_stream_) != cudaSuccess)
      throw Error(IFMM_CUDA, "cudaMemsetAsync failed on an arena slab");
    s.zeroed = to;
  }
  std::vector<Slab> slabs_;
  size_t cur_ = 0;
  size_t slab_;
  size_t in_use_ = 0;
  cudaStream_t zero_stream_ = nullptr;
  bool zero_ = false;
};

// Host-pinned staging area for descriptor uploads.  Bump-allocated; reset()
// only after the stream has been synchronised (the copies read from it).
class Staging {
 public:
  ~Staging() {
    for (auto& c : chunks_) cudaFreeHost(c.ptr);
  }
  void* get(size_t bytes) {
    bytes = (bytes + 255) / 256 * 256;
    for (;;) {
      if (cur_ < chunks_.size()) {
        Chunk& c = chunks_[cur_];
        if (c.used + bytes <= c.size) {
          void* p = static_cast<char*>(c.ptr) + c.used;
          c.used += bytes;
          return p;
        }
        ++cur_;
        continue;
      }
      size_t sz = bytes > (size_t(64) << 20) ? bytes : (size_t(64) << 20);
      void* p = nullptr;
      CK(cudaMallocHost(&p, sz));
      chunks_.push_back({p, sz, 0});
      cur_ = chunks_.size() - 1;
    }
  }
  void reset() {
    for (auto& c : chunks_) c.used = 0;
    cur_ = 0;
  }

 private:
  struct Chunk {
    void* ptr;
    size_t size;
    size_t used;
  };
  std::vector<Chunk> chunks_;
  size_t cur_ = 0;
};

// Upload a host vector into the arena, async on `s` through pinned staging.
template <class T>
T* upload(Arena& a, const std::vector<T>& v, cudaStream_t s, Staging& st) {
  T* d = a.alloc_n<T>(v.size() ? v.size() : 1);
  if (!v.empty()) {
    void* h = st.get(v.size() * sizeof(T));
    memcpy(h, v.data(), v.size() * sizeof(T));
    CK(cudaMemcpyAsync(d, h, v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  return d;
}

inline int ceil_div(long long a, long long b) { return int((a + b - 1) / b); }

// ---------------------------------------------------------------- device helpers
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum; `red` must hold >= 32 doubles of shared memory.
__device__ inline double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (wid == 0) {
    t = lane < nw ? red[lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) red[0] = t;
  }
  __syncthreads();
  t = red[0];
  __syncthreads();
  return t;
}

// Block-wide argmax of |v| with the smallest index winning ties (numpy/LAPACK
// idamax convention).  Entries with idx < 0 are ignored.  Returns index (or -1)
// and writes the signed value at that index to *val.
struct ArgMax {
  double a;  // |value|, -1 for none
  int i;
};
__device__ __forceinline__ ArgMax argmax_merge(ArgMax x, ArgMax y) {
  if (y.a > x.a || (y.a == x.a && y.i >= 0 && (x.i < 0 || y.i < x.i))) return y;
  return x;
}
__device__ inline ArgMax block_argmax(ArgMax v, ArgMax* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ArgMax w;
    w.a = __shfl_xor_sync(0xffffffffu, v.a, o);
    w.i = __shfl_xor_sync(0xffffffffu, v.i, o);
    v = argmax_merge(v, w);
  }
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  if (wid == 0) {
    ArgMax t = lane < nw ? red[lane] : ArgMax{-1.0, -1};
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ArgMax w;
      w.a = __shfl_xor_sync(0xffffffffu, t.a, o);
      w.i = __shfl_xor_sync(0xffffffffu, t.i, o);
      t = argmax_merge(t, w);
    }
    if (lane == 0) red[0] = t;
  }
  __syncthreads();
  ArgMax r = red[0];
  __syncthreads();
  return r;
}

}  // namespace ifmm
