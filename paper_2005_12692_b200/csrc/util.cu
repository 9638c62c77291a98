// util.cu -- workspace, device sort/scan wrappers.
#include <cub/cub.cuh>

#include <cstdlib>
#include <map>

#include "pipeline.cuh"

namespace cr {

static thread_local std::string g_err_text;
void set_error_text(const std::string& s) { g_err_text = s; }
const char* last_error_text() { return g_err_text.c_str(); }

namespace {
struct Prof {
  bool on = false;
  uint64_t gen = 0, ended = 0;  // calls begun / the last call whose events are complete
  std::vector<cudaEvent_t> pool;
  int used = 0;
  std::vector<const char*> names;
  ~Prof() {
    for (auto e : pool) cudaEventDestroy(e);
  }
  cudaEvent_t next() {
    if (used == int(pool.size())) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
      pool.push_back(e);
    }
    return pool[used++];
  }
};
thread_local Prof g_prof;
}  // namespace

thread_local int64_t g_launch_count = 0;

static thread_local int64_t g_opts[OPT_COUNT] = {};
int64_t opt(int key) { return key > 0 && key < OPT_COUNT ? g_opts[key] : 0; }
bool set_opt(int key, int64_t v) {
  if (key <= 0 || key >= OPT_COUNT) return false;
  g_opts[key] = v;
  return true;
}

void set_profiling(bool on) { g_prof.on = on; }

void prof_begin(cudaStream_t s) {
  g_launch_count = 0;
  ++g_prof.gen;
  g_prof.used = 0;
  g_prof.names.clear();
  if (!g_prof.on) return;
  cudaEvent_t e = g_prof.next();
  if (e) cudaEventRecord(e, s);
  g_prof.names.push_back("begin");
}

void prof_mark(cudaStream_t s, const char* stage) {
  if (!g_prof.on || g_prof.names.empty()) return;
  cudaEvent_t e = g_prof.next();
  if (!e) return;
  cudaEventRecord(e, s);
  g_prof.names.push_back(stage);
}

void prof_end(cr_stats& st) {
  st.launches = g_launch_count;
  st.nstages = 0;
  g_prof.ended = g_prof.gen;  // stage times are read lazily (prof_fill), outside the call
}

uint64_t prof_gen() { return g_prof.gen; }

void prof_fill(cr_stats& st) {
  if (!g_prof.on || g_prof.ended != g_prof.gen) return;
  st.nstages = 0;
  int n = int(g_prof.names.size());
  for (int i = 1; i < n && st.nstages < 16; ++i) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, g_prof.pool[i - 1], g_prof.pool[i]);
    st.stage_ms[st.nstages] = ms;
    strncpy(st.stage_name[st.nstages], g_prof.names[i], 23);
    st.stage_name[st.nstages][23] = 0;
    ++st.nstages;
  }
}

namespace {
struct Arena {
  void* base = nullptr;
  size_t cap = 0;
};
constexpr int MAX_DEV = 64;
thread_local Arena g_arena[MAX_DEV];

// Block cache (per host thread and device): device blocks are kept after a call and handed out
// again by size, so a steady stream of calls makes no allocator calls at all.  The stream-ordered
// pool (cudaMallocAsync) was measured to stall the host for 10-1000 ms on some repeated calls
// (profiles/r01/s5: C5 reduce_d1 1.63 -> 2.72 s, H0 4.5 -> 536 ms) -- fragmentation makes it map
// fresh memory.  A block is reused for a request of size in [size/2, size]; blocks are only freed
// when an allocation fails (then everything cached is returned to the driver and it is retried).
// Calls are blocking and one stream each; a call on another stream first waits on an event
// recorded at the end of the previous call, so cached blocks are never in use by two streams.
struct Cache {
  std::multimap<size_t, void*> free_blocks;  // size -> block
  std::map<void*, size_t> size_of;           // every block this cache owns
  cudaEvent_t done = nullptr;                // recorded at the end of the last call
  cudaStream_t last = nullptr;
  bool pool_set = false;
  size_t bytes = 0;                          // held by this cache (in use or free)
};
struct Caches {
  Cache c[MAX_DEV];
  // A host thread that exits returns its blocks (errors are ignored: at process exit the CUDA
  // runtime may already be gone, and then the driver reclaims everything anyway).
  ~Caches() { release_all(); }
  void release_all();
};
thread_local Caches g_caches;
#define g_cache (g_caches.c)
size_t round_block(size_t b) {
  if (b <= (size_t(1) << 20)) return (b + 511) & ~size_t(511);
  return (b + (size_t(2) << 20) - 1) & ~((size_t(2) << 20) - 1);
}
}  // namespace

void Caches::release_all() {
  int cur = -1;
  if (cudaGetDevice(&cur) != cudaSuccess) {
    cudaGetLastError();
    return;
  }
  for (int d = 0; d < MAX_DEV; ++d) {
    Cache& C = c[d];
    Arena& A = g_arena[d];
    if (C.size_of.empty() && !A.base) continue;
    if (cudaSetDevice(d) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    if (C.done) cudaEventSynchronize(C.done);  // the last call's work is complete
    for (auto& kv : C.size_of) cudaFree(kv.first);
    if (A.base) cudaFree(A.base);
    A.base = nullptr;
    A.cap = 0;
    C.free_blocks.clear();
    C.size_of.clear();
    C.bytes = 0;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, d) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
    cudaGetLastError();
  }
  cudaSetDevice(cur);
  cudaGetLastError();
}

void release_workspace() { g_caches.release_all(); }

size_t workspace_bytes() {
  size_t n = 0;
  for (int d = 0; d < MAX_DEV; ++d) n += g_cache[d].bytes + g_arena[d].cap;
  return n;
}

Workspace::Workspace(cudaStream_t s) : s_(s) {
  if (cudaGetDevice(&dev_) != cudaSuccess || dev_ < 0 || dev_ >= MAX_DEV) dev_ = 0;
  Cache& C = g_cache[dev_];
  if (!C.pool_set) {  // keep freed blocks in the default pool (once per thread and device)
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev_) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    C.pool_set = true;
  }
  if (C.done && C.last != s_) cudaStreamWaitEvent(s_, C.done, 0);
}

Workspace::~Workspace() {
  Cache& C = g_cache[dev_];
  for (void* p : ptrs_)
    if (p) C.free_blocks.emplace(C.size_of[p], p);
  if (!C.done) cudaEventCreateWithFlags(&C.done, cudaEventDisableTiming);
  if (C.done) cudaEventRecord(C.done, s_);
  C.last = s_;
  if (arena_ && need_ > acap_) {  // grow the arena to this call's high-water mark
    Arena& A = g_arena[dev_];
    if (A.base) cudaFreeAsync(A.base, s_);
    A.base = nullptr;
    A.cap = 0;
    const size_t cap = need_ + need_ / 4;
    if (cudaMallocAsync(&A.base, cap, s_) == cudaSuccess) A.cap = cap;
    else A.base = nullptr, cudaGetLastError();
  }
}

void Workspace::use_arena() {
  arena_ = true;
  abase_ = static_cast<char*>(g_arena[dev_].base);
  acap_ = g_arena[dev_].cap;
  aoff_ = need_ = 0;
}

void* Workspace::alloc_bytes(size_t bytes) {
  if (arena_) {
    const size_t b = (bytes + 255) & ~size_t(255);
    need_ += b;
    if (aoff_ + b <= acap_) {
      void* p = abase_ + aoff_;
      aoff_ += b;
      return p;
    }
  }
  Cache& C = g_cache[dev_];
  const size_t want = round_block(bytes < 1 ? 1 : bytes);
  auto it = C.free_blocks.lower_bound(want);
  if (it != C.free_blocks.end() && it->first <= 2 * want) {
    void* p = it->second;
    C.free_blocks.erase(it);
    ptrs_.push_back(p);
    return p;
  }
  void* p = nullptr;
  if (cudaMallocAsync(&p, want, s_) != cudaSuccess) {
    cudaGetLastError();  // out of memory: return the cache to the driver and retry once
    for (auto& kv : C.free_blocks) {
      cudaFreeAsync(kv.second, s_);
      C.bytes -= C.size_of[kv.second];
      C.size_of.erase(kv.second);
    }
    C.free_blocks.clear();
    CR_CUDA(cudaMallocAsync(&p, want, s_));
  }
  C.size_of[p] = want;
  C.bytes += want;
  ptrs_.push_back(p);
  return p;
}

void Workspace::release(void* p) {
  for (auto& q : ptrs_)
    if (q == p) {
      Cache& C = g_cache[dev_];
      C.free_blocks.emplace(C.size_of[q], q);  // reusable by later allocations on this stream
      q = nullptr;
      return;
    }
}

namespace {
// One pinned staging block per host thread, allocated on first use and kept for the life of the
// thread (cudaMallocHost costs milliseconds; a per-call allocation dominated small calls).
struct PinnedBlock {
  unsigned long long* p = nullptr;
  ~PinnedBlock() {
    if (p) cudaFreeHost(p);
  }
};
thread_local PinnedBlock g_pinned;
}  // namespace

HostScalars::HostScalars() : p(nullptr) {
  if (!g_pinned.p) CR_CUDA(cudaMallocHost(&g_pinned.p, 64 * sizeof(unsigned long long)));
  p = g_pinned.p;
}
HostScalars::~HostScalars() {}

void exclusive_sum_u32(const uint32_t* in, uint32_t* out, int64_t n, Workspace& ws) {
  if (n <= 0) return;
  size_t tmp = 0;
  CR_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, int(n), ws.stream()));
  void* t = ws.alloc_bytes(tmp);
  CR_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, in, out, int(n), ws.stream()));
  ws.release(t);
}

}  // namespace cr
