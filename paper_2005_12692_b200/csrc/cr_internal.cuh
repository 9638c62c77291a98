// cr_internal.cuh -- shared device/host helpers of libcr.so (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "../../include/cr.h"

namespace cr {

constexpr uint32_t NONE32 = 0xFFFFFFFFu;
constexpr uint64_t NONE64 = 0xFFFFFFFFFFFFFFFFull;
// ord(+inf): +inf cells are absent from K (reading R5); every finite ord is smaller.
constexpr uint32_t ABSENT_ORD = 0xFF800000u;

// Order-preserving map float32 -> uint32 after -0.0 -> +0.0 (reading R7): a < b as floats
// iff ord(a) < ord(b).  NaN never reaches it (rejected first).
__host__ __device__ __forceinline__ uint32_t ord_of(float f) {
#ifdef __CUDA_ARCH__
  uint32_t u = __float_as_uint(f);
#else
  uint32_t u;
  memcpy(&u, &f, 4);
#endif
  u = u == 0x80000000u ? 0u : u;
  // negative: ~u; non-negative: u | sign bit  (branch-free: xor with 0xFFFFFFFF or 0x80000000)
  return u ^ (uint32_t(int32_t(u) >> 31) | 0x80000000u);
}
__host__ __device__ __forceinline__ float float_of_ord(uint32_t o) {
  const uint32_t u = o ^ (~uint32_t(int32_t(o) >> 31) | 0x80000000u);
#ifdef __CUDA_ARCH__
  return __uint_as_float(u);
#else
  float f;
  memcpy(&f, &u, 4);
  return f;
#endif
}
__host__ __device__ __forceinline__ uint64_t make_key(uint32_t ord, uint32_t kidx) {
  return (uint64_t(ord) << 32) | kidx;
}
__host__ __device__ __forceinline__ uint32_t key_ord(uint64_t k) { return uint32_t(k >> 32); }
__host__ __device__ __forceinline__ uint32_t key_kidx(uint64_t k) { return uint32_t(k); }

// Khalimsky geometry.  Cell (X,Y,Z), kidx = (Z*KY + Y)*KX + X.
struct Geom {
  int64_t nx, ny, nz;      // voxels per axis (x fastest)
  int64_t KX, KY, KZ;      // 2n-1
  int64_t ncells;          // KX*KY*KZ
  int64_t nvox;            // nx*ny*nz
  int D;                   // number of axes with extent > 1 (0 for a single voxel)
  __host__ __device__ __forceinline__ int64_t stride(int axis) const {
    return axis == 0 ? 1 : (axis == 1 ? KX : KX * KY);
  }
};

// Per-cell tag (u8): kind in bits 6-7, partner direction in bits 0-2.
//   kind 0: residual (not an apparent pair)
//   kind 1: DOWN  -- upper cell of an apparent pair (partner is a facet)
//   kind 2: UP    -- lower cell of an apparent pair (partner is a cofacet)
//   kind 3: CLEARED -- residual cell that is the death cell of a pair one dimension below
// direction dir = 2*axis + (sign > 0): partner kidx = kidx + (sign)*stride(axis).
constexpr uint8_t KIND_RESIDUAL = 0, KIND_DOWN = 1, KIND_UP = 2, KIND_CLEARED = 3;
__host__ __device__ __forceinline__ uint8_t tag_kind(uint8_t t) { return t >> 6; }
__host__ __device__ __forceinline__ int tag_dir(uint8_t t) { return t & 7; }
__host__ __device__ __forceinline__ uint8_t make_tag(uint8_t kind, int dir) {
  return uint8_t((kind << 6) | dir);
}
__host__ __device__ __forceinline__ int64_t dir_offset(const Geom& g, int dir) {
  int64_t s = g.stride(dir >> 1);
  return (dir & 1) ? s : -s;
}

// Validation / measurement options (cr_set_option; thread-local, 0 = the product default).
enum OptKey {
  OPT_FORCE_GENERAL = 1,     // 1D images through the general path
  OPT_1D_TREE = 2,           // 1D images through the tree path instead of the tiles
  OPT_TOP_REDUCE = 3,        // top dimension by the coboundary reduction instead of duality
  OPT_K5_BLOCKS_PER_SM = 4,  // resident K5 blocks per SM (<= the occupancy limit)
  OPT_K5_JITTER_NS = 5,      // pseudo-random K5 delays: perturb the schedule (tests)
  OPT_DEBUG = 6,             // per-stage counters on stderr
  OPT_KF_TMA = 7,            // filtration ring by TMA instead of per-thread cp.async
  OPT_KF_RCAP = 8,           // residual edges staged per filtration CTA (tests: the overflow path)
  OPT_COUNT = 9
};
int64_t opt(int key);

// Error plumbing (host).
struct Error {
  cr_status st;
  std::string msg;
};
void set_error_text(const std::string& s);

// Per-stage CUDA-event timing (thread-local, enabled by cr_set_profiling).
void prof_begin(cudaStream_t s);
void prof_mark(cudaStream_t s, const char* stage);  // the stage that just ended
void prof_end(cr_stats& st);                         // after the call's final sync
uint64_t prof_gen();                                 // profiled calls begun on this thread
void prof_fill(cr_stats& st);  // stage times of the last call, if no call began since

#define CR_CUDA(call)                                                                       \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess) {                                                                \
      throw ::cr::Error{e_ == cudaErrorMemoryAllocation ? CR_ENOMEM : CR_ECUDA,             \
                        std::string(#call) + ": " + cudaGetErrorString(e_) + " @" +         \
                            __FILE__ + ":" + std::to_string(__LINE__)};                     \
    }                                                                                       \
  } while (0)

// Device-side bounds assertions (build with CR_DEVICE_ASSERTS=1, see build.py): compiled out of
// the normal build.  The pool's compute-sanitizer is closed (profiles/r02/sanitizer), so the
// capacity invariants of the working-column tiers, merges, sort and stores are checked by these
// instead; a failure prints the site and traps (the call fails with CR_ECUDA).
#ifdef CR_DEVICE_ASSERTS
#define CR_DASSERT(c)                                                                  \
  do {                                                                                 \
    if (!(c)) {                                                                        \
      printf("CR_DASSERT failed %s:%d: %s\n", __FILE__, __LINE__, #c);                  \
      __trap();                                                                        \
    }                                                                                  \
  } while (0)
#else
#define CR_DASSERT(c) \
  do {                \
  } while (0)
#endif

extern thread_local int64_t g_launch_count;
#define CR_CHECK_LAUNCH()                \
  do {                                   \
    CR_CUDA(cudaGetLastError());         \
    ++::cr::g_launch_count;              \
  } while (0)

// One thread per voxel: x within a block row, (y, z) from the grid -- no division per voxel.
// Images whose y or z extent exceeds the grid limit fall back to a linear launch with division.
constexpr int VOX_THREADS = 128;  // measured (C5b H0 + sort + top dim): 64: 12.2 ms, 128: 9.6, 256: 10.0, 512: 10.9
inline bool vox_grid_ok(const Geom& g) { return g.ny <= 65535 && g.nz <= 65535; }
inline dim3 vox_grid(const Geom& g) {
  // (measured: a (row, y, z) grid of 128-thread rows was slower on C5b than the linear launch --
  // a million small blocks -- so the linear form with one division pair per voxel is used)
  return dim3(unsigned((g.nvox + VOX_THREADS - 1) / VOX_THREADS), 1, 1);
}
// this thread's voxel (v, x, y, z); false past the row end / the grid
__device__ __forceinline__ bool vox_of_thread(const Geom& g, uint32_t& v, uint32_t& x, uint32_t& y,
                                              uint32_t& z) {
  const uint32_t nx = uint32_t(g.nx), ny = uint32_t(g.ny);
  if (gridDim.y > 1 || gridDim.z > 1) {
    x = blockIdx.x * VOX_THREADS + threadIdx.x;
    y = blockIdx.y;
    z = blockIdx.z;
    v = (z * ny + y) * nx + x;
    return x < nx;
  }
  const uint64_t vv = uint64_t(blockIdx.x) * VOX_THREADS + threadIdx.x;
  v = uint32_t(vv);
  const uint32_t r = v / nx;
  x = v - r * nx;
  z = r / ny;
  y = r - z * ny;
  return vv < uint64_t(g.nvox);
}

// Append up to NI items per thread to out[] behind the counter *n with one atomic per emitting
// warp for all NI slots.  Item order is arbitrary.  Every lane of the warp must call it.
template <class T, int NI>
__device__ __forceinline__ void warp_append(const bool (&emit)[NI], const T (&item)[NI],
                                            T* __restrict__ out, unsigned* __restrict__ n) {
  // one atomic per warp for all NI slots (same-address atomics serialise at the L2 slice)
  const int lane = threadIdx.x & 31;
  unsigned mask[NI], total = 0;
#pragma unroll
  for (int i = 0; i < NI; ++i) {
    mask[i] = __ballot_sync(0xFFFFFFFFu, emit[i]);
    total += __popc(mask[i]);
  }
  if (!total) return;
  unsigned base = 0;
  if (lane == 0) base = atomicAdd(n, total);
  base = __shfl_sync(0xFFFFFFFFu, base, 0);
#pragma unroll
  for (int i = 0; i < NI; ++i) {
    if (emit[i]) out[base + __popc(mask[i] & ((1u << lane) - 1))] = item[i];
    base += __popc(mask[i]);
  }
}

inline unsigned grid_for(int64_t n, int block) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  if (g > 0x7FFFFFFF) g = 0x7FFFFFFF;
  return unsigned(g);
}

}  // namespace cr
