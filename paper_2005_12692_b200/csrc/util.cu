// util.cu -- workspace, device sort/scan wrappers.
#include <cub/cub.cuh>

#include "pipeline.cuh"

namespace cr {

static thread_local std::string g_err_text;
void set_error_text(const std::string& s) { g_err_text = s; }
const char* last_error_text() { return g_err_text.c_str(); }

Workspace::Workspace(cudaStream_t s) : s_(s) {
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
}

Workspace::~Workspace() {
  for (void* p : ptrs_)
    if (p) cudaFreeAsync(p, s_);
}

void* Workspace::alloc_bytes(size_t bytes) {
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

HostScalars::HostScalars() : p(nullptr) {
  CR_CUDA(cudaMallocHost(&p, 64 * sizeof(unsigned long long)));
}
HostScalars::~HostScalars() {
  if (p) cudaFreeHost(p);
}

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
