// sort.cu -- K3: hand-written stable LSD radix sort of the residual keys (the
// paper's "we have to sort only twice").
//
// One-sweep design: keys are sorted over their significant bits only ([begin_bit, end_bit): e.g.
// 32 + kidx bits for (ord << 32 | kidx) column keys), 8 bits per pass, and a pass reads every
// key (and value) once and writes it once:
//   k_os_hist    one read of the keys for the digit histograms of ALL passes (block-private
//                shared-memory histograms, added into global counters);
//   k_os_scan    per pass: exclusive scan of the 256 digit totals (the digit's first output slot);
//   k_os_pass    per pass: a CTA takes the next tile of OS_TILE keys (tile order from an atomic
//                counter, so every earlier tile is already running), ranks it stably in shared
//                memory -- warp w owns a contiguous chunk and walks it 32 keys at a time, a key's
//                rank among its warp's equal digits from __match_any_sync peers and a per-warp
//                running count -- publishes its per-digit counts and finds the counts of all
//                earlier tiles by decoupled look-back (thread d spins on digit d of the previous
//                tiles' status words until one is an inclusive prefix), stages the tile sorted by
//                digit in shared memory, and writes it out: consecutive threads write consecutive
//                slots of a digit's run (coalesced), instead of one scattered word per key.
// Status words carry the pass number, so one memset serves all passes.  Descending order sorts
// the complemented digits (a stable ascending sort of ~key).
#include <cub/cub.cuh>

#include "pipeline.cuh"

namespace cr {
namespace {

constexpr int OS_THREADS = 256, OS_WARPS = OS_THREADS / 32, OS_IPT = 12;
constexpr int OS_TILE = OS_THREADS * OS_IPT;  // 3072 keys per tile (measured best of 8 / 12 / 16)
constexpr int OS_RADIX = 256;
constexpr int OS_MAXPASS = 8;
// status word of (tile, digit): [63:56] pass + 1, [55:54] 1 = aggregate, 2 = inclusive prefix,
// [53:0] count
constexpr uint64_t OS_AGG = 1ull << 54, OS_INC = 2ull << 54, OS_CNT = (1ull << 54) - 1;

template <class K>
__device__ __forceinline__ uint32_t os_digit(K k, int shift, bool desc) {
  return uint32_t((desc ? ~k : k) >> shift) & (OS_RADIX - 1);
}

// ghist[p * 256 + d] += #keys with digit d in pass p (p = 0 .. npass-1, shift begin_bit + 8p)
template <class K>
__global__ void __launch_bounds__(OS_THREADS) k_os_hist(const K* __restrict__ keys, int64_t n,
                                                        int begin_bit, int npass, bool desc,
                                                        unsigned* __restrict__ ghist) {
  __shared__ unsigned h[OS_MAXPASS][OS_RADIX];
  for (int i = threadIdx.x; i < OS_MAXPASS * OS_RADIX; i += OS_THREADS) (&h[0][0])[i] = 0;
  __syncthreads();
  for (int64_t i = int64_t(blockIdx.x) * OS_THREADS + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * OS_THREADS) {
    const K k = keys[i];
    for (int p = 0; p < npass; ++p) atomicAdd(&h[p][os_digit(k, begin_bit + 8 * p, desc)], 1u);
  }
  __syncthreads();
  for (int p = 0; p < npass; ++p) {
    const unsigned c = h[p][threadIdx.x];
    if (c) atomicAdd(ghist + p * OS_RADIX + threadIdx.x, c);
  }
}

// ghist[p][*] <- exclusive prefix sums (one block per pass)
__global__ void __launch_bounds__(OS_RADIX) k_os_scan(unsigned* __restrict__ ghist) {
  typedef cub::BlockScan<unsigned, OS_RADIX> BS;
  __shared__ typename BS::TempStorage tmp;
  unsigned* h = ghist + blockIdx.x * OS_RADIX;
  unsigned pre;
  BS(tmp).ExclusiveSum(h[threadIdx.x], pre);
  h[threadIdx.x] = pre;
}

template <class K, class V>
struct OsSmem {
  K k[OS_TILE];
  V v[OS_TILE];
  unsigned wcnt[OS_WARPS][OS_RADIX];  // per-warp digit counts, then their exclusive prefixes
  unsigned toff[OS_RADIX];             // tile-local first slot of each digit
  unsigned hist[OS_RADIX];             // the tile's digit counts
  unsigned long long gbase[OS_RADIX];  // global slot of the tile's first key of each digit
  unsigned tile;
};

template <class K, class V, bool HASV>
__global__ void __launch_bounds__(OS_THREADS, 3) k_os_pass(
    const K* __restrict__ kin, const V* __restrict__ vin, K* __restrict__ kout,
    V* __restrict__ vout, int64_t n, int shift, bool desc, int pass,
    const unsigned* __restrict__ gstart, unsigned long long* __restrict__ status,
    unsigned* __restrict__ tile_ctr) {
  extern __shared__ uint4 os_dyn[];
  OsSmem<K, V>& S = *reinterpret_cast<OsSmem<K, V>*>(os_dyn);
  typedef cub::BlockScan<unsigned, OS_THREADS> BS;
  __shared__ typename BS::TempStorage s_scan;
  const int t = threadIdx.x, w = t >> 5, lane = t & 31;
  const bool single = gstart == nullptr;  // one tile: its own counts are the global ones
  if (t == 0) S.tile = single ? 0u : atomicAdd(tile_ctr, 1u);
  for (int i = t; i < OS_WARPS * OS_RADIX; i += OS_THREADS) (&S.wcnt[0][0])[i] = 0;
  S.hist[t] = 0;
  __syncthreads();
  const unsigned tile = S.tile;
  const int64_t base = int64_t(tile) * OS_TILE;
  const unsigned lt = (1u << lane) - 1;
  // 1. load (warp w: keys [w * 32 * IPT, (w + 1) * 32 * IPT) of the tile, 32 at a time) and
  //    rank within the warp
  K k[OS_IPT];
  V v[OS_IPT];
  unsigned rk[OS_IPT];
  unsigned vmask = 0;  // bit r: key r exists (digits are recomputed from the keys: registers)
#pragma unroll
  for (int r = 0; r < OS_IPT; ++r) {
    const int64_t i = base + (w * OS_IPT + r) * 32 + lane;
    const bool valid = i < n;
    k[r] = valid ? kin[i] : K(0);
    if (HASV) v[r] = valid ? vin[i] : V(0);
    vmask |= valid ? 1u << r : 0u;
  }
#define OS_DG(r) (((vmask >> (r)) & 1u) ? os_digit(k[r], shift, desc) : unsigned(OS_RADIX))
  // the tile's digit counts first (shared-memory atomics), published at once as an aggregate:
  // later tiles' look-backs then rarely wait on this tile while it ranks
#pragma unroll
  for (int r = 0; r < OS_IPT; ++r)
    if ((vmask >> r) & 1u) atomicAdd(&S.hist[os_digit(k[r], shift, desc)], 1u);
  __syncthreads();
  const unsigned cnt = S.hist[t];
  const unsigned long long tag = uint64_t(pass + 1) << 56;
  unsigned long long* st = single ? nullptr : status + uint64_t(tile) * OS_RADIX + t;
  if (!single) __stcg(st, tag | (tile == 0 ? OS_INC : OS_AGG) | cnt);
#pragma unroll
  for (int r = 0; r < OS_IPT; ++r) {
    const unsigned d = OS_DG(r);
    // lanes with the same digit: 9 ballots (8 digit bits + "no key") instead of a MATCH, whose
    // result latency stalled the ranking (ncu: 29 % of the pass's stall samples)
    unsigned peers = 0xFFFFFFFFu;
#pragma unroll
    for (int b = 0; b < 9; ++b) {
      const unsigned m = __ballot_sync(0xFFFFFFFFu, (d >> b) & 1u);
      peers &= ((d >> b) & 1u) ? m : ~m;
    }
    const unsigned before = d < OS_RADIX ? S.wcnt[w][d] : 0u;
    __syncwarp();
    if (d < OS_RADIX && (peers & lt) == 0) S.wcnt[w][d] = before + __popc(peers);
    __syncwarp();
    rk[r] = before + __popc(peers & lt);
  }
  __syncthreads();
  // 2. thread t = digit t: per-warp offsets, look-back over the earlier tiles
  {
    unsigned run = 0;
#pragma unroll
    for (int ww = 0; ww < OS_WARPS; ++ww) {
      const unsigned c = S.wcnt[ww][t];
      S.wcnt[ww][t] = run;
      run += c;
    }
  }
  unsigned toff;
  BS(s_scan).ExclusiveSum(cnt, toff);
  S.toff[t] = toff;
  unsigned long long excl = 0;
  for (int64_t j = single ? -1 : int64_t(tile) - 1; j >= 0; --j) {
    const unsigned long long* p = status + uint64_t(j) * OS_RADIX + t;
    unsigned long long s;
    do {
      s = *reinterpret_cast<const volatile unsigned long long*>(p);
    } while ((s >> 56) != uint64_t(pass + 1) || (s & (3ull << 54)) == 0);
    excl += s & OS_CNT;
    if (s & OS_INC) break;
  }
  if (!single && tile != 0) __stcg(st, tag | OS_INC | (excl + cnt));
  S.gbase[t] = single ? toff : gstart[t] + excl;
  __syncthreads();
  // 3. stage the tile sorted by digit
#pragma unroll
  for (int r = 0; r < OS_IPT; ++r) {
    const unsigned d = OS_DG(r);
    if (d < OS_RADIX) {
      const unsigned pos = S.toff[d] + S.wcnt[w][d] + rk[r];
      CR_DASSERT(pos < unsigned(OS_TILE));
      S.k[pos] = k[r];
      if (HASV) S.v[pos] = v[r];
    }
  }
#undef OS_DG
  __syncthreads();
  // 4. write out: slot i of the staged tile goes to gbase[d] + (i - toff[d])
  const int64_t tn64 = n - base < OS_TILE ? n - base : OS_TILE;
  const int tn = int(tn64);
  for (int i = t; i < tn; i += OS_THREADS) {
    const K kk = S.k[i];
    const unsigned d = os_digit(kk, shift, desc);
    const unsigned long long o = S.gbase[d] + unsigned(i - S.toff[d]);
    CR_DASSERT(o < (unsigned long long)n);
    kout[o] = kk;
    if (HASV) vout[o] = S.v[i];
  }
}

template <class K, class V, bool HASV>
void os_set_smem(int dev) {
  static thread_local int done_dev = -1;
  if (done_dev == dev) return;
  CR_CUDA(cudaFuncSetAttribute(k_os_pass<K, V, HASV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               int(sizeof(OsSmem<K, V>))));
  done_dev = dev;
}

template <class K, class V, bool HASV>
void os_sort(K* keys, V* vals, int64_t n, int begin_bit, int end_bit, bool descending,
             Workspace& ws) {
  cudaStream_t s = ws.stream();
  const int npass = (end_bit - begin_bit + 7) / 8;
  if (npass > OS_MAXPASS) throw Error{CR_EINTERNAL, "radix_sort: more than 64 key bits"};
  const int64_t ntiles = (n + OS_TILE - 1) / OS_TILE;
  K* kalt = ws.alloc<K>(n);
  V* valt = HASV ? ws.alloc<V>(n) : nullptr;
  if (ntiles == 1) {  // one tile: no histogram pass, no status words, no look-back
    os_set_smem<K, V, HASV>(ws.device());
    K *ki = keys, *ko = kalt;
    V *vi = vals, *vo = valt;
    for (int p = 0; p < npass; ++p) {
      k_os_pass<K, V, HASV><<<1, OS_THREADS, sizeof(OsSmem<K, V>), s>>>(
          ki, vi, ko, vo, n, begin_bit + 8 * p, descending, p, nullptr, nullptr, nullptr);
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
      if (HASV)
        CR_CUDA(cudaMemcpyAsync(vals, vi, size_t(n) * sizeof(V), cudaMemcpyDeviceToDevice, s));
    }
    if (valt) ws.release(valt);
    ws.release(kalt);
    return;
  }
  // counters: ghist [npass][256], tile counters [npass]; status [ntiles][256]
  unsigned* ghist = ws.alloc<unsigned>(OS_MAXPASS * OS_RADIX + OS_MAXPASS);
  unsigned* tctr = ghist + OS_MAXPASS * OS_RADIX;
  unsigned long long* status = ws.alloc<unsigned long long>(ntiles * OS_RADIX);
  CR_CUDA(cudaMemsetAsync(ghist, 0, (OS_MAXPASS * OS_RADIX + OS_MAXPASS) * sizeof(unsigned), s));
  CR_CUDA(cudaMemsetAsync(status, 0, size_t(ntiles) * OS_RADIX * sizeof(unsigned long long), s));
  {
    int64_t hb = (n + OS_THREADS * 8 - 1) / (OS_THREADS * 8);
    if (hb > 4 * 148) hb = 4 * 148;
    if (hb < 1) hb = 1;
    k_os_hist<K><<<unsigned(hb), OS_THREADS, 0, s>>>(keys, n, begin_bit, npass, descending, ghist);
    CR_CHECK_LAUNCH();
    k_os_scan<<<npass, OS_RADIX, 0, s>>>(ghist);
    CR_CHECK_LAUNCH();
  }
  os_set_smem<K, V, HASV>(ws.device());
  K *ki = keys, *ko = kalt;
  V *vi = vals, *vo = valt;
  for (int p = 0; p < npass; ++p) {
    k_os_pass<K, V, HASV><<<unsigned(ntiles), OS_THREADS, sizeof(OsSmem<K, V>), s>>>(
        ki, vi, ko, vo, n, begin_bit + 8 * p, descending, p, ghist + p * OS_RADIX, status,
        tctr + p);
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
    if (HASV)
      CR_CUDA(cudaMemcpyAsync(vals, vi, size_t(n) * sizeof(V), cudaMemcpyDeviceToDevice, s));
  }
  ws.release(status);
  ws.release(ghist);
  if (valt) ws.release(valt);
  ws.release(kalt);
}

}  // namespace

template <class K, class V>
void radix_sort(K* keys, V* vals, int64_t n, int begin_bit, int end_bit, bool descending,
                Workspace& ws) {
  if (n <= 1 || end_bit <= begin_bit) return;
  if (n >= (int64_t(1) << 32)) throw Error{CR_EINTERNAL, "radix_sort: more than 2^32 keys"};
  if (vals)
    os_sort<K, V, true>(keys, vals, n, begin_bit, end_bit, descending, ws);
  else
    os_sort<K, V, false>(keys, vals, n, begin_bit, end_bit, descending, ws);
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
