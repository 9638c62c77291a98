// workspace.cuh -- stream-ordered scratch allocations and small host helpers.
#pragma once
#include <vector>

#include "cr_internal.cuh"

namespace cr {

// All scratch is cudaMallocAsync'ed on the call's stream and freed (stream-ordered) on exit.
// The device's default mempool keeps freed blocks (release threshold = max), so repeated
// calls do not return memory to the driver.
//
// Arena mode (use_arena): allocations are carved from a per-thread, per-device device buffer that
// persists across calls (a call is blocking, so the previous call's work is complete when the
// next one starts); what does not fit falls back to cudaMallocAsync and the arena grows to the
// call's high-water mark when the workspace closes.  release() is a no-op for arena memory.  Used
// by the latency-bound paths, where ~20 stream-ordered allocations per call cost more host time
// than the kernels take.
class Workspace {
 public:
  explicit Workspace(cudaStream_t s);
  ~Workspace();
  template <class T>
  T* alloc(int64_t n) {
    return static_cast<T*>(alloc_bytes(size_t(n < 1 ? 1 : n) * sizeof(T)));
  }
  void* alloc_bytes(size_t bytes);
  void release(void* p);  // early stream-ordered free
  void use_arena();
  cudaStream_t stream() const { return s_; }
  int device() const { return dev_; }

 private:
  cudaStream_t s_;
  int dev_ = 0;
  std::vector<void*> ptrs_;
  bool arena_ = false;
  char* abase_ = nullptr;
  size_t acap_ = 0, aoff_ = 0, need_ = 0;
};

// Pinned host staging for small device->host reads.
struct HostScalars {
  HostScalars();
  ~HostScalars();
  unsigned long long* p;  // 64 entries
};

template <class T>
inline T read_scalar(const T* dev, cudaStream_t s, HostScalars& hs) {
  CR_CUDA(cudaMemcpyAsync(hs.p, dev, sizeof(T), cudaMemcpyDeviceToHost, s));
  CR_CUDA(cudaStreamSynchronize(s));
  T v;
  memcpy(&v, hs.p, sizeof(T));
  return v;
}

}  // namespace cr
