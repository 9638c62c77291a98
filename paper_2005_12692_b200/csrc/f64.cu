// f64.cu -- float64 images (cr_barcodes_f64): the paper's own value precision (PAPER.md:188,
// "pixel values ... stored as double").
//
// Persistence of a sublevel-set filtration depends on the image only through the order of its
// values (the pairing is a function of the total order (birth, dim, kidx), and births are maxima
// of vertex values), so the float64 barcode is computed by the float32 pipeline on an
// order-isomorphic SURROGATE image and the bar endpoints are mapped back:
//   exact case  every finite value is a float32 value: the surrogate is the cast (no rounding),
//               the endpoints are cast back to double.  Cost: one 8 B/voxel read + 4 B/voxel write.
//   rank case   otherwise the values are dense-ranked on the device (radix sort of the
//               order-preserving u64 of each double, -0 -> +0; run-start flags; inclusive scan)
//               and voxel v gets the normal float32 with bit pattern 0x00800000 + rank(v) -- a
//               finite value with the same order and the same ties -- while +inf stays +inf
//               (outside the domain, reading R5).  Endpoint r is mapped back through the table
//               of distinct values.
// Neither case changes the order, so births, deaths, birth cells and the pairing are exactly
// those of the float64 filtration (pinned against oracle_ph_f64 in tests/test_gpu_parity.py).
#include <cub/cub.cuh>

#include "pipeline.cuh"

namespace cr {
namespace {

cr_status fail(const Error& e) {
  set_error_text(e.msg);
  return e.st;
}

constexpr uint32_t SURR_BASE = 0x00800000u;  // bits of the smallest normal float32
constexpr int64_t MAX_RANKS = int64_t(0x7F800000u - SURR_BASE);  // below +inf's bit pattern

__device__ __forceinline__ uint64_t ord64(double x) {
  uint64_t u = uint64_t(__double_as_longlong(x));
  u = u == 0x8000000000000000ull ? 0ull : u;  // -0.0 -> +0.0 (reading R7)
  return u ^ (uint64_t(int64_t(u) >> 63) | 0x8000000000000000ull);
}
__device__ __forceinline__ double double_of_ord64(uint64_t o) {
  const uint64_t u = o ^ (~uint64_t(int64_t(o) >> 63) | 0x8000000000000000ull);
  return __longlong_as_double(int64_t(u));
}

// Pass 1: NaN check, exactness check, and the cast surrogate (used when every value is exact).
// flags[0] |= 1 on NaN, flags[1] |= 1 on a value that float32 does not represent.
__global__ void k_f64_cast(const double* __restrict__ img, int64_t n, float* __restrict__ surr,
                           unsigned* __restrict__ flags) {
  bool nan = false, inexact = false;
  for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < n;
       v += int64_t(gridDim.x) * blockDim.x) {
    const double x = img[v];
    const float f = __double2float_rn(x);
    nan |= x != x;
    inexact |= double(f) != x && x == x;
    surr[v] = f;
  }
  if (__syncthreads_or(nan) && threadIdx.x == 0) atomicOr(flags + 0, 1u);
  if (__syncthreads_or(inexact) && threadIdx.x == 0) atomicOr(flags + 1, 1u);
}

__global__ void k_f64_keys(const double* __restrict__ img, int64_t n, uint64_t* __restrict__ keys,
                           uint32_t* __restrict__ idx) {
  for (int64_t v = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; v < n;
       v += int64_t(gridDim.x) * blockDim.x) {
    keys[v] = ord64(img[v]);
    idx[v] = uint32_t(v);
  }
}

// flag[i] = 1 where sorted key i starts a run of equal values
__global__ void k_f64_runs(const uint64_t* __restrict__ keys, int64_t n, uint32_t* __restrict__ flag) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    flag[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1u : 0u;
}

// rank = inclusive_scan(flag) - 1; surrogate[idx[i]] = normal float of rank (or +inf);
// uniq[rank] = the double of each run.
__global__ void k_f64_scatter(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ idx,
                              const uint32_t* __restrict__ flag, const uint32_t* __restrict__ incl,
                              int64_t n, float* __restrict__ surr, double* __restrict__ uniq) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const uint32_t r = incl[i] - 1u;
    const double x = double_of_ord64(keys[i]);
    const bool pinf = x == __longlong_as_double(0x7FF0000000000000ll);
    surr[idx[i]] = pinf ? __uint_as_float(0x7F800000u) : __uint_as_float(SURR_BASE + r);
    if (flag[i]) uniq[r] = x;
  }
}

__device__ __forceinline__ double back(float f, const double* __restrict__ uniq) {
  if (isinf(f) && f > 0.f) return __longlong_as_double(0x7FF0000000000000ll);
  return uniq ? uniq[__float_as_uint(f) - SURR_BASE] : double(f);
}

__global__ void k_f64_map(const cr_pair* __restrict__ in, int64_t n, const double* __restrict__ uniq,
                          cr_pair64* __restrict__ out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const cr_pair p = in[i];
    cr_pair64 q;
    q.dim = p.dim;
    q.pad = 0;
    q.birth = back(p.birth, uniq);
    q.death = back(p.death, uniq);
    out[i] = q;
  }
}


}  // namespace
}  // namespace cr

using namespace cr;

extern "C" cr_status cr_barcodes_f64(const double* image, const int64_t* shape, int ndim,
                                     int maxdim, cr_pair64* out_pairs, uint32_t* out_birth_cells,
                                     int64_t out_capacity, int64_t* n_pairs, cr_stream_t stream) {
  if (!image || !n_pairs || ndim < 1 || ndim > 3 || !shape || maxdim < 0 || out_capacity < 0 ||
      (out_capacity > 0 && !out_pairs))
    return CR_EINVAL;
  const int64_t ncells = cr_num_cells(shape, ndim);
  if (ncells < 0) return CR_EINVAL;
  try {
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    Geom g = make_geom(shape, ndim);
    const int64_t n = g.nvox;
    Workspace ws(s);
    HostScalars hs;
    cr_stats st{};
    prof_begin(s);
    float* surr = ws.alloc<float>(n);
    unsigned* flags = ws.alloc<unsigned>(2);
    CR_CUDA(cudaMemsetAsync(flags, 0, 2 * sizeof(unsigned), s));
    const int T = 256;
    k_f64_cast<<<grid_for(n, T), T, 0, s>>>(image, n, surr, flags);
    CR_CHECK_LAUNCH();
    CR_CUDA(cudaMemcpyAsync(hs.p, flags, 2 * sizeof(unsigned), cudaMemcpyDeviceToHost, s));
    CR_CUDA(cudaStreamSynchronize(s));
    unsigned hf[2];
    memcpy(hf, hs.p, sizeof(hf));
    if (hf[0]) return CR_EINVAL;  // NaN
    double* uniq = nullptr;
    if (hf[1]) {  // rank case
      if (n > MAX_RANKS) return CR_EINVAL;
      uint64_t* k0 = ws.alloc<uint64_t>(n);
      uint32_t* i0 = ws.alloc<uint32_t>(n);
      uint32_t* flag = ws.alloc<uint32_t>(n);
      uint32_t* incl = ws.alloc<uint32_t>(n);
      uniq = ws.alloc<double>(n);
      k_f64_keys<<<grid_for(n, T), T, 0, s>>>(image, n, k0, i0);
      CR_CHECK_LAUNCH();
      radix_sort<uint64_t, uint32_t>(k0, i0, n, 0, 64, false, ws);
      size_t scan_bytes = 0;
      CR_CUDA(cub::DeviceScan::InclusiveSum(nullptr, scan_bytes, flag, incl, n, s));
      void* tmp = ws.alloc_bytes(scan_bytes);
      k_f64_runs<<<grid_for(n, T), T, 0, s>>>(k0, n, flag);
      CR_CHECK_LAUNCH();
      CR_CUDA(cub::DeviceScan::InclusiveSum(tmp, scan_bytes, flag, incl, n, s));
      k_f64_scatter<<<grid_for(n, T), T, 0, s>>>(k0, i0, flag, incl, n, surr,
                                                 uniq);
      CR_CHECK_LAUNCH();
    }
    prof_mark(s, hf[1] ? "f64_rank" : "f64_cast");
    const int64_t cap = out_capacity > 0 ? out_capacity : 1;
    cr_pair* tmp_pairs = ws.alloc<cr_pair>(cap);
    int64_t m;
    {
      Workspace ws2(s);
      m = barcodes_core(surr, g, maxdim, tmp_pairs, out_birth_cells, out_capacity, ws2, hs, st);
    }
    *n_pairs = m;
    if (m > out_capacity) {
      CR_CUDA(cudaStreamSynchronize(s));
      return CR_ERANGE;
    }
    if (m > 0) {
      k_f64_map<<<grid_for(m, T), T, 0, s>>>(tmp_pairs, m, uniq, out_pairs);
      CR_CHECK_LAUNCH();
    }
    prof_mark(s, "f64_map");
    CR_CUDA(cudaStreamSynchronize(s));
    prof_end(st);
    set_last_stats(st);
    return CR_OK;
  } catch (const Error& e) {
    return fail(e);
  }
}
