// sort.cu -- K3: hand-written stable LSD radix sort of the residual keys (the
// paper's "we have to sort only twice").
//
// Keys are sorted over their significant bits only ([begin_bit, end_bit): e.g. 32 + kidx bits
// for (ord << 32 | kidx) column keys), 8 bits per pass, each pass three kernels:
//   1. k_rs_hist     one block per tile of RS_TILE keys: the tile's digit histogram
//                    (shared-memory atomics), written digit-major: hist[d * nblk + block];
//   2. k_rs_scan     one block per digit: exclusive scan of that digit's per-tile counts, and the
//                    digit's total;
//   3. k_rs_scatter  one block per tile again: digit bases = exclusive scan of the 256 totals + the
//                    tile's offset; the tile is ranked stably in sub-tiles of 256 keys (one per
//                    thread, in input order): within a warp by __match_any_sync peers, across warps
//                    by a per-digit prefix over the 8 warps' counts, across sub-tiles by a running
//                    base -- then keys (and values) are scattered.
// Descending order sorts the complemented digits (a stable ascending sort of ~key).
#include <cub/cub.cuh>

#include "pipeline.cuh"

namespace cr {
namespace {

constexpr int RS_THREADS = 256, RS_IPT = 16, RS_TILE = RS_THREADS * RS_IPT;

template <class K>
__device__ __forceinline__ uint32_t rs_digit(K k, int shift, uint32_t mask, bool desc) {
  return uint32_t((desc ? ~k : k) >> shift) & mask;
}

template <class K>
__global__ void __launch_bounds__(RS_THREADS) k_rs_hist(const K* __restrict__ keys, int64_t n,
                                                        int shift, uint32_t mask, bool desc,
                                                        uint32_t* __restrict__ hist,
                                                        uint32_t nblk) {
  __shared__ uint32_t h[256];
  const int t = threadIdx.x;
  h[t] = 0;
  __syncthreads();
  const int64_t base = int64_t(blockIdx.x) * RS_TILE;
#pragma unroll 4
  for (int i = 0; i < RS_IPT; ++i) {
    const int64_t idx = base + i * RS_THREADS + t;
    if (idx < n) atomicAdd(&h[rs_digit(keys[idx], shift, mask, desc)], 1u);
  }
  __syncthreads();
  hist[uint64_t(t) * nblk + blockIdx.x] = h[t];
}

// hist[d * nblk + b] <- exclusive prefix over b (per digit d = blockIdx.x); total[d] <- the sum
__global__ void __launch_bounds__(1024) k_rs_scan(uint32_t* __restrict__ hist, uint32_t nblk,
                                                  uint32_t* __restrict__ total) {
  typedef cub::BlockScan<uint32_t, 1024> BS;
  __shared__ typename BS::TempStorage s_scan;
  uint32_t* h = hist + uint64_t(blockIdx.x) * nblk;
  uint32_t run = 0;
  for (uint32_t c = 0; c < nblk; c += 1024) {
    const uint32_t i = c + threadIdx.x;
    const uint32_t v = i < nblk ? h[i] : 0u;
    uint32_t pre, tot;
    BS(s_scan).ExclusiveSum(v, pre, tot);
    if (i < nblk) h[i] = run + pre;
    run += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) total[blockIdx.x] = run;
}

template <class K, class V>
__global__ void __launch_bounds__(RS_THREADS) k_rs_scatter(
    const K* __restrict__ kin, const V* __restrict__ vin, K* __restrict__ kout, V* __restrict__ vout,
    int64_t n, int shift, uint32_t mask, bool desc, const uint32_t* __restrict__ hist,
    const uint32_t* __restrict__ total, uint32_t nblk) {
  typedef cub::BlockScan<uint32_t, RS_THREADS> BS;
  __shared__ typename BS::TempStorage s_scan;
  __shared__ uint32_t s_base[256];             // next output position of each digit
  __shared__ uint32_t s_cnt[RS_THREADS / 32][256];
  __shared__ uint32_t s_tot[256];
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  {
    uint32_t pre;
    BS(s_scan).ExclusiveSum(total[t], pre);
    s_base[t] = pre + hist[uint64_t(t) * nblk + blockIdx.x];
  }
  const unsigned lt = (1u << lane) - 1;
  const int64_t base = int64_t(blockIdx.x) * RS_TILE;
  for (int i = 0; i < RS_IPT; ++i) {
    const int64_t idx = base + i * RS_THREADS + t;
    const bool valid = idx < n;
    const K k = valid ? kin[idx] : K(0);
    const uint32_t d = valid ? rs_digit(k, shift, mask, desc) : 256u;
#pragma unroll
    for (int w = 0; w < RS_THREADS / 32; ++w) s_cnt[w][t] = 0;
    __syncthreads();
    const unsigned peers = __match_any_sync(0xFFFFFFFFu, d);
    const uint32_t rank = __popc(peers & lt);
    if (valid && rank == 0) s_cnt[warp][d] = __popc(peers);
    __syncthreads();
    {  // per-digit exclusive prefix over the warps (thread t: digit t)
      uint32_t run = 0;
#pragma unroll
      for (int w = 0; w < RS_THREADS / 32; ++w) {
        const uint32_t c = s_cnt[w][t];
        s_cnt[w][t] = run;
        run += c;
      }
      s_tot[t] = run;
    }
    __syncthreads();
    if (valid) {
      const uint32_t pos = s_base[d] + s_cnt[warp][d] + rank;
      kout[pos] = k;
      if (vin) vout[pos] = vin[idx];
    }
    __syncthreads();
    s_base[t] += s_tot[t];
  }
}

}  // namespace

template <class K, class V>
void radix_sort(K* keys, V* vals, int64_t n, int begin_bit, int end_bit, bool descending,
                Workspace& ws) {
  if (n <= 1 || end_bit <= begin_bit) return;
  if (n >= (int64_t(1) << 32)) throw Error{CR_EINTERNAL, "radix_sort: more than 2^32 keys"};
  cudaStream_t s = ws.stream();
  const uint32_t nblk = uint32_t((n + RS_TILE - 1) / RS_TILE);
  K* kalt = ws.alloc<K>(n);
  V* valt = vals ? ws.alloc<V>(n) : nullptr;
  uint32_t* hist = ws.alloc<uint32_t>(int64_t(256) * nblk);
  uint32_t* total = ws.alloc<uint32_t>(256);
  K *ki = keys, *ko = kalt;
  V *vi = vals, *vo = valt;
  for (int shift = begin_bit; shift < end_bit; shift += 8) {
    const int bits = end_bit - shift < 8 ? end_bit - shift : 8;
    const uint32_t mask = (1u << bits) - 1u;
    k_rs_hist<K><<<nblk, RS_THREADS, 0, s>>>(ki, n, shift, mask, descending, hist, nblk);
    CR_CHECK_LAUNCH();
    k_rs_scan<<<256, 1024, 0, s>>>(hist, nblk, total);
    CR_CHECK_LAUNCH();
    k_rs_scatter<K, V><<<nblk, RS_THREADS, 0, s>>>(ki, vi, ko, vo, n, shift, mask, descending,
                                                   hist, total, nblk);
    CR_CHECK_LAUNCH();
    K* tk = ki;
    ki = ko;
    ko = tk;
    V* tv = vi;
    vi = vo;
    vo = tv;
  }
  if (ki != keys) {
    CR_CUDA(cudaMemcpyAsync(keys, ki, size_t(n) * sizeof(K), cudaMemcpyDeviceToDevice, s));
    if (vals) CR_CUDA(cudaMemcpyAsync(vals, vi, size_t(n) * sizeof(V), cudaMemcpyDeviceToDevice, s));
  }
  ws.release(total);
  ws.release(hist);
  if (valt) ws.release(valt);
  ws.release(kalt);
}

template void radix_sort<uint64_t, uint64_t>(uint64_t*, uint64_t*, int64_t, int, int, bool,
                                             Workspace&);
template void radix_sort<uint64_t, uint32_t>(uint64_t*, uint32_t*, int64_t, int, int, bool,
                                             Workspace&);
template void radix_sort<uint32_t, uint64_t>(uint32_t*, uint64_t*, int64_t, int, int, bool,
                                             Workspace&);

void sort_keys_u64(uint64_t* keys, int64_t n, bool descending, int end_bit, Workspace& ws,
                   int begin_bit) {
  radix_sort<uint64_t, uint32_t>(keys, nullptr, n, begin_bit, end_bit, descending, ws);
}

}  // namespace cr
