// util.cu -- workspace, device sort/scan wrappers.
#include <cub/cub.cuh>

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
thread_local bool g_pool_set[MAX_DEV] = {};
}  // namespace

Workspace::Workspace(cudaStream_t s) : s_(s) {
  if (cudaGetDevice(&dev_) != cudaSuccess || dev_ < 0 || dev_ >= MAX_DEV) dev_ = 0;
  if (!g_pool_set[dev_]) {  // keep freed blocks in the default pool (once per thread and device)
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev_) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    g_pool_set[dev_] = true;
  }
}

Workspace::~Workspace() {
  for (void* p : ptrs_)
    if (p) cudaFreeAsync(p, s_);
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
  void* p = nullptr;
  CR_CUDA(cudaMallocAsync(&p, bytes, s_));
  ptrs_.push_back(p);
  return p;
}

void Workspace::release(void* p) {
  for (auto& q : ptrs_)
    if (q == p) {
      cudaFreeAsync(q, s_);
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

void sort_keys_u64(uint64_t* keys, int64_t n, bool descending, int end_bit, Workspace& ws) {
  if (n <= 1) return;
  uint64_t* alt = ws.alloc<uint64_t>(n);
  cub::DoubleBuffer<uint64_t> db(keys, alt);
  size_t tmp = 0;
  if (descending)
    CR_CUDA(cub::DeviceRadixSort::SortKeysDescending(nullptr, tmp, db, int(n), 0, end_bit, ws.stream()));
  else
    CR_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, db, int(n), 0, end_bit, ws.stream()));
  void* t = ws.alloc_bytes(tmp);
  if (descending)
    CR_CUDA(cub::DeviceRadixSort::SortKeysDescending(t, tmp, db, int(n), 0, end_bit, ws.stream()));
  else
    CR_CUDA(cub::DeviceRadixSort::SortKeys(t, tmp, db, int(n), 0, end_bit, ws.stream()));
  if (db.Current() != keys)
    CR_CUDA(cudaMemcpyAsync(keys, db.Current(), n * sizeof(uint64_t), cudaMemcpyDeviceToDevice,
                            ws.stream()));
  ws.release(t);
  ws.release(alt);
}

void exclusive_sum_u32(const uint32_t* in, uint32_t* out, int64_t n, Workspace& ws) {
  if (n <= 0) return;
  size_t tmp = 0;
  CR_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, int(n), ws.stream()));
  void* t = ws.alloc_bytes(tmp);
  CR_CUDA(cub::DeviceScan::ExclusiveSum(t, tmp, in, out, int(n), ws.stream()));
  ws.release(t);
}

}  // namespace cr
