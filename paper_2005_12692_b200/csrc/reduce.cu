// reduce.cu -- K5: residual coboundary column reduction of dimension d >= 1.
//
// Columns are the finite d-cells that are neither apparent (K2) nor cleared (death cells of
// dimension d-1), processed in DECREASING key order (the paper's order of
// d-cells, "larger birth-time come first", with ties by kidx, reading R1).
// A column is the coboundary delta(s) -- the finite cofacets of s -- as a set of (d+1)-cell keys;
// its pivot is the minimum key (the earliest coface).  While the pivot is owned, the owner's
// column is added over Z/2 (symmetric difference):
//   - owner is apparent (the pivot t is the upper cell of an apparent pair (s', t)) -> add delta(s')
//     enumerated on the fly (the implicit coboundary of PAPER.md:135-136);
//   - owner is an earlier committed column -> add its stored reduced column.
// A nonzero column with an unowned pivot t gives the pair (s, t): bar [birth s, birth t)
// (PAPER.md:138-140); a zero column gives an essential class.
//
// Working column (one warp per column): a sorted main array M in global memory plus a small
// sorted "fresh" array F in shared memory, both consumed from the front (pivots only move later);
// the column is M xor F, and equal heads cancel lazily when the pivot is taken.  Small addends
// (apparent coboundaries, short stored columns) merge into F at O(|F|) cost; F is merged into M
// only when it fills up, so a long column is not rewritten on every addition.
//
// Parallel schedule (one persistent kernel, no grid-wide rounds).  Warps take columns in
// processing order from a counter (per segment, segments interleaved).  A column publishes its
// current pivot cand(j) -- a lower bound of its final pivot: adding a column with the same pivot
// only moves the pivot later -- after every pivot change.  Column j with an unowned pivot p
// commits once every earlier column i of its segment has cand(i) > p or is finished (then no
// earlier column can end on p, and j's pivot is final); it waits on the first blocking column
// only, and a column committed while j is unfinished has a pivot j can never reach -- the
// sequential reduction's pairs are reproduced exactly (applied per column).
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "pipeline.cuh"

namespace cr {
namespace {

#ifdef K5_TIMING  // measurement builds only: per-phase cycles of the heavy columns, printed
#define KT(...) __VA_ARGS__
#else
#define KT(...)
#endif
constexpr int WPB = 8;  // warps per block
constexpr int THREADS = WPB * 32;
#ifndef K5_FCAP
#define K5_FCAP 512
#endif
// fresh-array capacity per warp (shared memory, x2 ping-pong): 512 since the merges went to merge
// path (profiles/r02/s7: F 256 / 512 / 768 -> C5 169 / 144 / 138 ms, C5b 45.6 / 45.1 / 45.4 ms)
constexpr uint32_t FCAP = K5_FCAP;

// n / d for n, d < 2^32 by one 64-bit high multiply: m = ceil(2^64 / d) makes the quotient exact
// (the error n * (m - 2^64/d) / 2^64 < 2^-32 cannot carry past the fractional part (d-1)/d).
struct FastDiv {
  uint64_t m;
  uint32_t d;
  static FastDiv make(uint32_t d) { return FastDiv{d <= 1 ? 0ull : (~0ull / d) + 1, d}; }
  __device__ __forceinline__ uint32_t div(uint32_t n) const {
    return d <= 1 ? n : uint32_t(__umul64hi(uint64_t(n), m));
  }
};

struct RP {
  Geom g;
  FastDiv fx, fxy;  // by KX and by KX*KY: Khalimsky coordinates of a kidx
  const uint64_t* cols;  // column keys in processing order (grouped by segment)
  uint32_t ncols;
  const uint32_t* births;
  const uint8_t* tags;
  // pivot hash table (open addressing, linear probing, 2^k slots of {key = pivot kidx, val}):
  // val = (pool offset << 24) | length of the committed column owning that pivot, NONE64 until
  // written.  ~2x the columns in slots: L2-resident (C5b 64 MB), where round 1's dense table
  // over every cell took 8.6 GB, a memset per call and a DRAM miss per lookup.
  ulonglong2* otab;
  uint32_t omask;
  uint64_t* pool;
  unsigned long long* pool_top;
  unsigned long long pool_cap;
  uint64_t* work;      // per warp: 2 * mcap main-array entries
  uint32_t mcap;
  uint64_t* gwork;     // per warp: 2 * (GCAP + FCAP) middle-tier entries
  // lv[0][j] = cand(j): 0 before column j starts, then a lower bound of its pivot key, NONE64
  // once it is finished.  lv[L][e] (L = 1..3) = a lower bound of min lv[0] over the 32^L columns
  // [e * 32^L, (e+1) * 32^L): every entry only grows, so a stale bound is still a bound.
  uint64_t* lv[4];
  const uint32_t* seg_off;  // nseg + 1 column offsets (columns are grouped by segment)
  uint32_t nseg;
  unsigned* seg_next;  // per segment: columns handed out
  unsigned long long* fetch;  // fetch counter (spreads warps over the segments)
  uint64_t* rec;  // one record per column, at the column's index
  int* err;
  unsigned long long* stats;  // [0] waits [1] additions [2] sum of lengths [3] max length
                              // [4] cycles waited [5] commits
  unsigned long long* ness;  // essential classes (zero columns)
  unsigned jitter;     // validation: pseudo-random delays (ns) that perturb the schedule
  unsigned long long* colrec;  // debug (option debug >= 2): per column 16 words, see k_reduce
};
constexpr int OI_LEN_BITS = 24;  // owner value: stored column length field

__device__ __forceinline__ uint32_t ohash(uint32_t k, uint32_t mask) {
  return uint32_t((uint64_t(k) * 0x9E3779B97F4A7C15ull) >> 32) & mask;
}
// The owner value of pivot k (NONE64: no committed owner -- or one whose value is not written
// yet, which callers treat as "not yet", re-checking after the owner is published finished).
// All lanes read the same slot (one transaction); warp-uniform.
__device__ __forceinline__ uint64_t owner_of(const ulonglong2* otab, uint32_t mask, uint32_t k) {
  for (uint32_t i = ohash(k, mask);; i = (i + 1) & mask) {
    const ulonglong2 sl = __ldcg(otab + i);
    if (sl.x == k) return sl.y;
    if (sl.x == NONE64) return NONE64;
  }
}
// the same with relaxed (coherent) loads, for the re-checks that order after a fence
__device__ __forceinline__ uint64_t owner_of_rlx(const ulonglong2* otab, uint32_t mask, uint32_t k) {
  for (uint32_t i = ohash(k, mask);; i = (i + 1) & mask) {
    const uint64_t* sl = reinterpret_cast<const uint64_t*>(otab + i);
    uint64_t key, val;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(key) : "l"(sl) : "memory");
    if (key == NONE64) return NONE64;
    if (key == k) {
      asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(val) : "l"(sl + 1) : "memory");
      return val;
    }
  }
}
// one thread: claim k's slot and write its value (every pivot is committed once)
__device__ __forceinline__ void owner_insert(ulonglong2* otab, uint32_t mask, uint32_t k,
                                             uint64_t val) {
  for (uint32_t i = ohash(k, mask);; i = (i + 1) & mask) {
    unsigned long long* key = reinterpret_cast<unsigned long long*>(otab + i);
    const unsigned long long old = atomicCAS(key, NONE64, (unsigned long long)k);
    if (old == NONE64 || old == k) {
      asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(key + 1), "l"(val) : "memory");
      return;
    }
  }
}

__device__ __forceinline__ uint64_t ldcg64(const uint64_t* p) {
  return __ldcg((const unsigned long long*)p);
}
template <bool G>
__device__ __forceinline__ uint64_t ld64(const uint64_t* p) {
  return G ? ldcg64(p) : *p;
}

// Keys of the working columns: (ord << 32 | kidx), pivot = the minimum.
__device__ __forceinline__ uint64_t rkey(const RP&, uint32_t b, uint32_t k) { return make_key(b, k); }
__device__ __forceinline__ uint32_t rkid(const RP&, uint64_t key) { return uint32_t(key); }

// The column of cell s, sorted ascending, written to dst (<= 6 entries): its finite cofacets (the
// implicit coboundary of PAPER.md:135-136).  Warp-collective.
__device__ __forceinline__ uint32_t coboundary(const RP& P, uint32_t s, uint64_t* dst, int lane) {
  const Geom& g = P.g;
  const uint32_t KX = uint32_t(g.KX), KY = uint32_t(g.KY);
  const uint32_t r = P.fx.div(s), z = P.fxy.div(s);
  const uint32_t c[3] = {s - r * KX, r - z * KY, z};
  const uint32_t ext[3] = {KX, KY, uint32_t(g.KZ)};
  uint64_t key = NONE64;
  if (lane < 6) {
    const int a = lane >> 1, sg = lane & 1;
    if (!(c[a] & 1) && (sg ? c[a] + 1 < ext[a] : c[a] > 0)) {
      const int64_t stv = g.stride(a);
      const uint32_t t = uint32_t(int64_t(s) + (sg ? stv : -stv));
      const uint32_t tb = __ldg(P.births + t);
      if (tb != ABSENT_ORD) key = rkey(P, tb, t);
    }
  }
  const unsigned valid = __ballot_sync(0xFFFFFFFFu, key != NONE64);
  int rank = 0;
#pragma unroll
  for (int l = 0; l < 6; ++l) rank += (__shfl_sync(0xFFFFFFFFu, key, l) < key);
  if (key != NONE64) dst[rank] = key;
  __syncwarp();
  return __popc(valid);
}

template <bool G>
__device__ __forceinline__ uint32_t lower_bound(const uint64_t* B, uint32_t n, uint64_t x) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (ld64<G>(B + mid) < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// C = A xor B (sorted, distinct entries each), C distinct from A and B.  Warp-collective.
// Output position of a kept A[i]: (#kept A before i) + (#kept B below A[i]); the number of common
// values below A[i] equals the number of A's duplicates before i.
// C = A xor B for A, B in shared memory (sorted, distinct entries each), C anywhere: merge path.
// Lane l takes the merged positions [l*per, (l+1)*per) (ties A first: an equal pair is adjacent,
// A's copy first); a start falling between an equal pair moves past it, so both copies are in
// one lane and cancel there.  Each lane merges its ranges sequentially twice -- to count, then
// (after a warp scan of the counts) to write.  O(1) shared-memory steps per entry instead of a
// binary search per entry on both sides.  Warp-collective; returns |C|.
__device__ uint32_t merge_xor_path(const uint64_t* A, uint32_t a, const uint64_t* B, uint32_t b,
                                   uint64_t* C, int lane) {
  const uint32_t n = a + b;
  if (n == 0) return 0;
  const uint32_t per = (n + 31) >> 5;
  const uint32_t d = min(uint32_t(lane) * per, n);
  uint32_t lo = d > b ? d - b : 0, hi = d < a ? d : a;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (A[mid] <= B[d - mid - 1]) lo = mid + 1;
    else hi = mid;
  }
  uint32_t is = lo, js = d - lo;
  if (is > 0 && js < b && A[is - 1] == B[js]) ++js;  // keep an equal pair in one lane
  uint32_t ie = __shfl_down_sync(0xFFFFFFFFu, is, 1), je = __shfl_down_sync(0xFFFFFFFFu, js, 1);
  if (lane == 31 || d + per >= n) {
    ie = a;
    je = b;
  }
  if (d >= n) ie = is = a, je = js = b;  // lanes past the end take nothing
  uint32_t cnt = 0;
  {
    uint32_t i = is, j = js;
    while (i < ie || j < je) {
      const uint64_t x = i < ie ? A[i] : NONE64, y = j < je ? B[j] : NONE64;
      if (x == y) {
        ++i;
        ++j;
      } else if (x < y) {
        ++cnt;
        ++i;
      } else {
        ++cnt;
        ++j;
      }
    }
  }
  uint32_t pos = cnt;  // inclusive warp scan
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, pos, o);
    if (lane >= o) pos += v;
  }
  const uint32_t total = __shfl_sync(0xFFFFFFFFu, pos, 31);
  pos -= cnt;
  {
    uint32_t i = is, j = js;
    while (i < ie || j < je) {
      const uint64_t x = i < ie ? A[i] : NONE64, y = j < je ? B[j] : NONE64;
      if (x == y) {
        ++i;
        ++j;
      } else if (x < y) {
        C[pos++] = x;
        ++i;
      } else {
        C[pos++] = y;
        ++j;
      }
    }
  }
  __syncwarp();
  return total;
}

// L1-cached load of a warp-private buffer (G, M): coherent with this SM's own stores (never the
// non-coherent read-only path: the buffers are rewritten in ping-pong by the same warp)
__device__ __forceinline__ uint64_t ld_ca(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.global.ca.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}

// C = A xor F for A in global memory, F in shared memory, C in global memory: merge path with
// each lane merging one contiguous diagonal segment (its reads of A are sequential per lane and
// hit L1 after the first), twice -- count, warp scan, write.  Warp-collective; returns |C|.
__device__ uint32_t merge_xor_path_g(const uint64_t* A, uint32_t a, const uint64_t* F,
                                     uint32_t b, uint64_t* __restrict__ C, int lane) {
  const uint32_t n = a + b;
  if (n == 0) return 0;
  const uint32_t per = (n + 31) >> 5;
  const uint32_t d = min(uint32_t(lane) * per, n);
  uint32_t lo = d > b ? d - b : 0, hi = d < a ? d : a;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (ld_ca(A + mid) <= F[d - mid - 1]) lo = mid + 1;
    else hi = mid;
  }
  uint32_t is = lo, js = d - lo;
  if (is > 0 && js < b && ld_ca(A + is - 1) == F[js]) ++js;
  uint32_t ie = __shfl_down_sync(0xFFFFFFFFu, is, 1), je = __shfl_down_sync(0xFFFFFFFFu, js, 1);
  if (lane == 31 || d + per >= n) {
    ie = a;
    je = b;
  }
  if (d >= n) ie = is = a, je = js = b;
  // Each lane streams its A segment through a 4-deep register queue (the load of A[i + 4] is
  // issued when A[i] is consumed), so a step waits on a compare, not on an L1 round trip.
  auto lda = [&](uint32_t k, uint32_t end) -> uint64_t { return k < end ? ld_ca(A + k) : NONE64; };
  uint32_t cnt = 0;
  {
    uint32_t i = is, j = js;
    uint64_t x0 = lda(i, ie), x1 = lda(i + 1, ie), x2 = lda(i + 2, ie), x3 = lda(i + 3, ie);
    uint64_t y = j < je ? F[j] : NONE64;
    while (i < ie || j < je) {
      if (x0 == y) {
        ++i;
        ++j;
        x0 = x1; x1 = x2; x2 = x3; x3 = lda(i + 3, ie);
        y = j < je ? F[j] : NONE64;
      } else if (x0 < y) {
        ++cnt;
        ++i;
        x0 = x1; x1 = x2; x2 = x3; x3 = lda(i + 3, ie);
      } else {
        ++cnt;
        ++j;
        y = j < je ? F[j] : NONE64;
      }
    }
  }
  uint32_t pos = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, pos, o);
    if (lane >= o) pos += v;
  }
  const uint32_t total = __shfl_sync(0xFFFFFFFFu, pos, 31);
  pos -= cnt;
  {
    uint32_t i = is, j = js;
    uint64_t x0 = lda(i, ie), x1 = lda(i + 1, ie), x2 = lda(i + 2, ie), x3 = lda(i + 3, ie);
    uint64_t y = j < je ? F[j] : NONE64;
    while (i < ie || j < je) {
      if (x0 == y) {
        ++i;
        ++j;
        x0 = x1; x1 = x2; x2 = x3; x3 = lda(i + 3, ie);
        y = j < je ? F[j] : NONE64;
      } else if (x0 < y) {
        C[pos++] = x0;
        ++i;
        x0 = x1; x1 = x2; x2 = x3; x3 = lda(i + 3, ie);
      } else {
        C[pos++] = y;
        ++j;
        y = j < je ? F[j] : NONE64;
      }
    }
  }
  __syncwarp();
  return total;
}

template <bool AG, bool BG>
__device__ uint32_t merge_symdiff(const uint64_t* A, uint32_t a, const uint64_t* B, uint32_t b,
                                  uint64_t* C, int lane) {
  if (!AG && !BG) return merge_xor_path(A, a, B, b, C, lane);
  const unsigned lt = (1u << lane) - 1;
  uint32_t carry = 0;
  for (uint32_t base = 0; base < a; base += 32) {
    const uint32_t i = base + lane;
    const bool valid = i < a;
    const uint64_t x = valid ? ld64<AG>(A + i) : 0;
    const uint32_t r = valid ? lower_bound<BG>(B, b, x) : 0;
    const bool dup = valid && r < b && ld64<BG>(B + r) == x;
    const unsigned m = __ballot_sync(0xFFFFFFFFu, dup);
    const uint32_t cb = carry + __popc(m & lt);
    if (valid && !dup) C[(i - cb) + (r - cb)] = x;
    carry += __popc(m);
  }
  const uint32_t dups = carry;
  carry = 0;
  for (uint32_t base = 0; base < b; base += 32) {
    const uint32_t k = base + lane;
    const bool valid = k < b;
    const uint64_t x = valid ? ld64<BG>(B + k) : 0;
    const uint32_t r = valid ? lower_bound<AG>(A, a, x) : 0;
    const bool dup = valid && r < a && ld64<AG>(A + r) == x;
    const unsigned m = __ballot_sync(0xFFFFFFFFu, dup);
    const uint32_t cb = carry + __popc(m & lt);
    if (valid && !dup) C[(k - cb) + (r - cb)] = x;
    carry += __popc(m);
  }
  __syncwarp();
  return a + b - 2 * dups;
}

// C = A xor B for A in shared memory and a tiny B (nb <= SMALLB, shared memory), C distinct from
// both.  Lane k < nb places B[k] by one binary search in A; every lane then holds all of B in
// registers, so an A entry needs only register compares, and the A chunks are independent:
//   kept A[i] goes to i + #{B < A[i]} - 2 #{common values < A[i]},
//   kept B[k] goes to k + #{A < B[k]} - 2 #{common values < B[k]}.
// Warp-collective; returns |C|.
constexpr uint32_t SMALLB = 8;
__device__ uint32_t merge_small(const uint64_t* A, uint32_t a, const uint64_t* B, uint32_t nb,
                                uint64_t* C, int lane) {
  uint64_t y = NONE64;
  uint32_t la = 0;
  bool ydup = false;
  if (lane < int(nb)) {
    y = B[lane];
    la = lower_bound<false>(A, a, y);
    ydup = la < a && A[la] == y;
  }
  const uint32_t bdup = __ballot_sync(0xFFFFFFFFu, ydup);
  uint64_t bv[SMALLB];
#pragma unroll
  for (int k = 0; k < int(SMALLB); ++k) bv[k] = __shfl_sync(0xFFFFFFFFu, y, k);  // NONE64 past nb
#pragma unroll 2
  for (uint32_t i = lane; i < a; i += 32) {
    const uint64_t x = A[i];
    uint32_t lessB = 0, D = 0;
    bool dup = false;
#pragma unroll
    for (int k = 0; k < int(SMALLB); ++k) {
      const bool lt = bv[k] < x;
      lessB += lt ? 1u : 0u;
      D += (lt && (bdup >> k & 1)) ? 1u : 0u;
      dup |= bv[k] == x;
    }
    if (!dup) C[i + lessB - 2 * D] = x;
  }
  if (lane < int(nb) && !ydup) C[lane + la - 2 * __popc(bdup & ((1u << lane) - 1))] = y;
  __syncwarp();
  return a + nb - 2 * __popc(bdup);
}

// C = A xor B with A in global memory and B in global (BG) or shared memory (!BG: all of B,
// b <= FCAP), for long inputs: windows of up to FCAP entries of A (and of B) are staged in shared
// memory (SA, SB: FCAP entries each) with coalesced loads, and the entries up to
// min(last staged A, last staged B) -- all of one window -- are merged there (merge path, output
// straight to C); the rest of the windows is shifted to their fronts and topped up.  No global
// search per chunk: the cut is found in shared memory.  (Round 2's first form split fixed-size
// chunks by a 32-way merge-path search over global memory: two dependent global round trips per
// chunk before its loads.)  Keys within A and within B are distinct, so an equal pair never
// straddles a cut.
__device__ __forceinline__ uint32_t upper_bound_smem(const uint64_t* S, uint32_t n, uint64_t x) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (S[mid] <= x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}
__device__ __forceinline__ void shift_front(uint64_t* S, uint32_t from, uint32_t n, int lane) {
  // S[0, n) <- S[from, from + n), chunk by chunk (a chunk's reads before its writes)
  for (uint32_t t0 = 0; t0 < n; t0 += 32) {
    const uint32_t t = t0 + lane;
    const uint64_t v = t < n ? S[from + t] : 0;
    __syncwarp();
    if (t < n) S[t] = v;
    __syncwarp();
  }
}
template <bool BG>
__device__ __noinline__ uint32_t merge_chunked(const uint64_t* A, uint32_t a, const uint64_t* B,
                                               uint32_t b, uint64_t* C, uint64_t* SA, uint64_t* SB,
                                               int lane) {
  constexpr uint32_t W = FCAP;
  uint32_t ia = 0, na = 0;  // A[ia, ia + na) sits in SA[0, na)
  uint32_t ib = 0, nb = 0;  // BG: B[ib, ib + nb) in SB[0, nb); !BG: B[ib, b) in place
  uint32_t out = 0;
  while (true) {
    const uint32_t fa = (W - na) < (a - ia - na) ? (W - na) : (a - ia - na);
    for (uint32_t t = lane; t < fa; t += 32) SA[na + t] = ldcg64(A + ia + na + t);
    na += fa;
    const uint64_t* WB;
    uint32_t wnb;
    bool bmore;
    if (BG) {
      const uint32_t fb = (W - nb) < (b - ib - nb) ? (W - nb) : (b - ib - nb);
      for (uint32_t t = lane; t < fb; t += 32) SB[nb + t] = ldcg64(B + ib + nb + t);
      nb += fb;
      WB = SB;
      wnb = nb;
      bmore = ib + nb < b;
    } else {
      WB = B + ib;
      wnb = b - ib;
      bmore = false;
    }
    __syncwarp();
    if (na == 0 && wnb == 0) break;
    const bool amore = ia + na < a;
    const uint64_t la = amore ? SA[na - 1] : NONE64, lb = bmore ? WB[wnb - 1] : NONE64;
    const uint64_t bound = la < lb ? la : lb;
    const uint32_t ca = bound == NONE64 ? na : upper_bound_smem(SA, na, bound);
    const uint32_t cb = bound == NONE64 ? wnb : upper_bound_smem(WB, wnb, bound);
    out += merge_xor_path(SA, ca, WB, cb, C + out, lane);
    shift_front(SA, ca, na - ca, lane);
    ia += ca;
    na -= ca;
    if (BG) {
      shift_front(SB, cb, nb - cb, lane);
      nb -= cb;
    }
    ib += cb;
  }
  return out;
}

// The working column of a warp (DBG: with the debug counters of option debug >= 2).
template <bool DBG>
struct ColT {
  static constexpr bool dbg = DBG;
  // tiers as (current, alternate) buffer pairs -- pointers, never indexed arrays, so that the
  // whole struct stays in registers
  uint64_t *Mc, *Ma;  // global main arrays
  uint64_t *Gc, *Ga;  // global middle arrays (GCAP + FCAP entries each)
  uint32_t ng, g0;
  uint64_t gwin;   // per lane: G[gb][gwb + lane] (valid unless gstale)
  uint32_t gwb;
  bool gstale;
  uint64_t *Fc, *Fa;  // shared fresh arrays
  uint32_t nm, h;
  uint32_t nf, f0;
  uint64_t mwin;   // per lane: M[mb][wb + lane] (valid unless mstale), NONE64 past the end
  uint32_t wb;     // window base
  bool mstale;
  long long fcyc;  // debug: cycles spent in flushes
  unsigned long long fent;  // debug: flushes, entries of M flushed
  unsigned fn;
  unsigned tpi, tpm, tpg;  // debug: take_pivot iterations, M / G window reloads
  unsigned nsp;            // debug: R spills
  long long rcyc, scyc;    // debug: cycles in r_insert, in spills (incl. their flushes)
  uint32_t cap;    // capacity of M[0] and M[1]
  uint64_t* spare; // the second half of a grown pair, installed after the merge that grew it
  uint32_t pt;     // tier of the pivot take_pivot returned: 0 M, 1 G, 2 F, 3 R
  uint64_t rv;     // per lane: one entry of the register bag R (unsorted; NONE64 = empty lane)
  uint32_t nr;     // entries in R
  uint64_t rmin;   // min of R (NONE64 if empty), kept exact
  uint64_t ha, hg, hb;  // cached heads of M[h:], G[g0:], F[f0:] (valid unless hstale)
  bool hstale;
  __device__ uint32_t len() const { return (nm - h) + (ng - g0) + (nf - f0) + nr; }
};
#ifndef K5_GCAP
#define K5_GCAP 8192
#endif
constexpr uint32_t GCAP = K5_GCAP;
#ifndef K5_GK
#define K5_GK 24
#endif  // the middle tier: F merges into G, G into M when it exceeds GCAP

// The working column is M[h:] xor G[g0:] xor F[f0:] xor R: three sorted tiers -- a long main
// array and a middle array in global memory, a fresh array in shared memory -- and a register
// bag R of <= 32 entries (one per lane, unsorted) that takes the small addends (apparent
// coboundaries, short stored columns): an insertion is a push through shared memory and a
// __match_any_sync for the cancellations, its minimum two __reduce_min_sync, instead of a sorted
// insertion.  Equal values in different tiers cancel lazily, when they reach the heads.  The
// heads of M, G and F are cached in registers and refreshed only for the tier that moved.

// head of M[h:] / G[g0:] from the register windows (the next 32 entries, one per lane, reloaded
// with one coalesced load when the head leaves the window or the tier is rewritten)
template <class CT>
__device__ __forceinline__ uint64_t head_m(CT& c, int lane) {
  if (c.mstale || c.h >= c.wb + 32) {
    c.wb = c.h;
    c.mwin = c.h + lane < c.nm ? ldcg64(c.Mc + c.h + lane) : NONE64;
    c.mstale = false;
    if (CT::dbg) ++c.tpm;
  }
  CR_DASSERT(c.h - c.wb < 32);
  return __shfl_sync(0xFFFFFFFFu, c.mwin, c.h - c.wb);
}
template <class CT>
__device__ __forceinline__ uint64_t head_g(CT& c, int lane) {
  if (c.gstale || c.g0 >= c.gwb + 32) {
    c.gwb = c.g0;
    c.gwin = c.g0 + lane < c.ng ? ldcg64(c.Gc + c.g0 + lane) : NONE64;
    c.gstale = false;
    if (CT::dbg) ++c.tpg;
  }
  CR_DASSERT(c.g0 - c.gwb < 32);
  return __shfl_sync(0xFFFFFFFFu, c.gwin, c.g0 - c.gwb);
}
template <class CT>
__device__ __forceinline__ uint64_t head_f(CT& c) {
  return c.f0 < c.nf ? c.Fc[c.f0] : NONE64;
}
template <class CT>
__device__ __forceinline__ void refresh_heads(CT& c, int lane) {
  c.ha = head_m(c, lane);
  c.hg = head_g(c, lane);
  c.hb = head_f(c);
  c.hstale = false;
}

// min over the lanes of a 64-bit key (NONE64 if every lane holds NONE64): two 32-bit reductions
__device__ __forceinline__ uint64_t bag_min(uint64_t v) {
  const uint32_t hi = __reduce_min_sync(0xFFFFFFFFu, uint32_t(v >> 32));
  const uint32_t lo = __reduce_min_sync(0xFFFFFFFFu, uint32_t(v >> 32) == hi ? uint32_t(v) : ~0u);
  return (uint64_t(hi) << 32) | lo;
}
// remove R's minimum
template <class CT>
__device__ __forceinline__ void bag_pop(CT& c) {
  if (c.rv == c.rmin) c.rv = NONE64;
  --c.nr;
  c.rmin = bag_min(c.rv);
}
// R <- R xor Y for the pairwise distinct keys y held by the lanes in vm (requires nr + |vm| <=
// 32): the y's go to the free lanes in order (through `scratch`), then a key present twice (a y
// equal to an R entry) leaves both lanes.  Warp-collective.
template <class CT>
__device__ __forceinline__ void bag_insert(CT& c, uint64_t y, unsigned vm, uint64_t* scratch,
                                           int lane) {
  const unsigned lt = (1u << lane) - 1;
  CR_DASSERT(c.nr + __popc(vm) <= 32);
  const unsigned fm = __ballot_sync(0xFFFFFFFFu, c.rv == NONE64);
  if ((vm >> lane) & 1u) scratch[__popc(vm & lt)] = y;
  __syncwarp();
  const uint32_t ny = __popc(vm);
  const uint32_t j = __popc(fm & lt);
  if (((fm >> lane) & 1u) && j < ny) c.rv = scratch[j];
  __syncwarp();
  const unsigned peers = __match_any_sync(0xFFFFFFFFu, c.rv);
  const bool dup = c.rv != NONE64 && (peers & (peers - 1)) != 0;
  const unsigned dm = __ballot_sync(0xFFFFFFFFu, dup);
  if (dup) c.rv = NONE64;
  c.nr = c.nr + ny - __popc(dm);
  c.rmin = bag_min(c.rv);
}
// the bag sorted ascending across the lanes (empty lanes, NONE64, last): bitonic network
__device__ __forceinline__ uint64_t bag_sorted(uint64_t v, int lane) {
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const uint64_t o = __shfl_xor_sync(0xFFFFFFFFu, v, j);
      const bool takemin = ((lane & j) == 0) == ((lane & k) == 0);
      v = takemin ? (o < v ? o : v) : (o > v ? o : v);
    }
  }
  return v;
}

// pivot = min of the tier heads, cancelling equal pairs; NONE64 if the column is zero.
// c.pt: the tier it heads (3 = R).  Warp-collective.
template <class CT>
__device__ __forceinline__ uint64_t take_pivot(CT& c, int lane) {
  if (c.hstale) refresh_heads(c, lane);
  while (true) {
    if (CT::dbg) ++c.tpi;
    const uint64_t a = c.ha, g = c.hg, b = c.hb, r = c.rmin;
    const uint64_t m1 = a < g ? a : g, m2 = b < r ? b : r;
    const uint64_t m = m1 < m2 ? m1 : m2;
    if (m == NONE64) return NONE64;
    const bool ea = a == m, eg = g == m, eb = b == m, er = r == m;
    const int k = int(ea) + int(eg) + int(eb) + int(er);
    // equal values in several tiers cancel in pairs: an even count removes the value, an odd
    // count (3) leaves one copy, which is the pivot (c.pt: its tier, the last one matching)
    c.pt = er ? 3u : (eb ? 2u : (eg ? 1u : 0u));
    if (k == 1) return m;
    int drop = k == 3 ? 2 : k;
    if (ea && drop) {
      ++c.h;
      c.ha = head_m(c, lane);
      --drop;
    }
    if (eg && drop) {
      ++c.g0;
      c.hg = head_g(c, lane);
      --drop;
    }
    if (eb && drop) {
      ++c.f0;
      c.hb = head_f(c);
      --drop;
    }
    if (er && drop) {
      bag_pop(c);
      --drop;
    }
    if (k == 3) return m;
  }
}

// Remove the pivot take_pivot returned (it is the head of tier c.pt): adding a column whose first
// entry is the pivot then adds only the rest of it -- one take_pivot iteration and one insertion
// fewer per addition than letting the two copies cancel at the heads.
template <class CT>
__device__ __forceinline__ void consume_pivot(CT& c, int lane) {
  if (c.pt == 0) {
    ++c.h;
    c.ha = head_m(c, lane);
  } else if (c.pt == 1) {
    ++c.g0;
    c.hg = head_g(c, lane);
  } else if (c.pt == 2) {
    ++c.f0;
    c.hb = head_f(c);
  } else {
    bag_pop(c);
  }
}

// R <- R xor B for a sorted B of nb <= SMALLB entries in shared memory (nr + nb <= 32).
template <class CT>
__device__ __forceinline__ void r_insert(CT& c, const uint64_t* B, uint32_t nb, uint64_t* scratch,
                                         int lane) {
  const uint64_t y = lane < int(nb) ? B[lane] : NONE64;
  __syncwarp();  // B may be `scratch`'s neighbour: read before the pushes
  bag_insert(c, y, nb >= 32 ? 0xFFFFFFFFu : ((1u << nb) - 1u), scratch, lane);
}

// The apparent-partner coboundary, speculated.  A DOWN pivot t (a (d+1)-cell) is the upper cell
// of an apparent pair (s', t) with s' = t + e_dir, a facet of t; the column then adds delta(s') =
// {t} + the other cofacets of s'.  Before t's tag is known, lane L < 30 loads the birth of member
// L % 5 of facet direction L / 5: member 0 is t + 2 e_dir (across the facet), members 1-4 are
// s' -/+ e_b for the two other axes b (when b is even in t).  The tag, the owner record and these
// births are independent loads, so an addition waits on one memory latency instead of a chain.
struct Spec {
  uint32_t cell;
  uint32_t birth;  // ABSENT_ORD if the member does not exist
};
// The lane's fixed role in spec_issue (depends only on the lane and the grid): member m of facet
// direction f.  The member exists iff t's axis a is odd, the checked axis `chk` stays inside the
// grid after moving by `dchk`, and (members 1-4) axis b is even in t.
struct SpecLane {
  int a, chk, dchk, sa;
  bool need_b_even;
  uint32_t off;      // cell - t (two's complement)
  bool active;
};
__device__ __forceinline__ SpecLane spec_lane(const Geom& g, int lane) {
  SpecLane L{0, 0, 0, 0, false, 0u, false};
  if (lane >= 30) return L;
  const int f = lane / 5, m = lane % 5;
  L.a = f >> 1;
  const int sa = (f & 1) ? 1 : -1;
  L.sa = sa;
  L.active = true;
  if (m == 0) {
    L.chk = L.a;
    L.dchk = 2 * sa;
    L.off = uint32_t(int64_t(2 * sa) * g.stride(L.a));
  } else {
    const int b = (L.a + 1 + ((m - 1) >> 1)) % 3;
    const int sb = (m & 1) ? -1 : 1;  // m = 1, 3: -;  m = 2, 4: +
    L.chk = b;
    L.dchk = sb;
    L.need_b_even = true;
    L.off = uint32_t(int64_t(sa) * g.stride(L.a) + int64_t(sb) * g.stride(b));
  }
  return L;
}
__device__ __forceinline__ Spec spec_issue(const RP& P, const SpecLane& L, uint32_t t) {
  const uint32_t KX = uint32_t(P.g.KX), KY = uint32_t(P.g.KY);
  const uint32_t ty = P.fx.div(t), tz = P.fxy.div(t);
  const uint32_t cx = t - ty * KX, cy = ty - tz * KY, cz = tz;
  const uint32_t ca = L.a == 0 ? cx : (L.a == 1 ? cy : cz);
  const uint32_t cc = L.chk == 0 ? cx : (L.chk == 1 ? cy : cz);
  const uint32_t ec = L.chk == 0 ? KX : (L.chk == 1 ? KY : uint32_t(P.g.KZ));
  const uint32_t moved = cc + uint32_t(L.dchk);  // wraps below 0 to a huge value
  Spec r{0u, ABSENT_ORD};
  const bool up_axis = ca & 1;  // t spans axis a: s' = t + sa e_a is a facet of t
  const bool b_bad = L.need_b_even && (cc & 1);
  if (L.active && up_axis && moved < ec && !b_bad) {
    r.cell = t + L.off;
    r.birth = __ldg(P.births + r.cell);
  }
  return r;
}



// Make room for a merge of `need` entries into M[mb ^ 1]: a column that outgrows its warp's slot
// moves to a larger pair carved from the pool (bump allocation; the few long columns of a launch
// leave their old pairs behind).  False (err 2: the caller retries with a larger pool) if the
// pool is exhausted.
template <class CT>
__device__ __forceinline__ bool grow(CT& c, uint32_t need, const RP& P, int lane) {
  if (need <= c.cap) return true;
  uint64_t ncap = uint64_t(need) * 2;
  if (ncap < uint64_t(c.cap) * 4) ncap = uint64_t(c.cap) * 4;
  unsigned long long off = 0;
  if (lane == 0) off = atomicAdd(P.pool_top, 2ull * ncap);
  off = __shfl_sync(0xFFFFFFFFu, off, 0);
  if (off + 2 * ncap > P.pool_cap || ncap > 0xFFFFFFFFull) {
    if (lane == 0) atomicOr(P.err, 2);
    return false;
  }
  c.Ma = P.pool + off;  // the merge's destination
  c.spare = P.pool + off + ncap;  // replaces the old M[mb] once the merge has read it
  c.cap = uint32_t(ncap);
  return true;
}
template <class CT>
__device__ __forceinline__ void swap_main(CT& c) {
  {
    uint64_t* t = c.Mc;
    c.Mc = c.Ma;
    c.Ma = c.spare ? c.spare : t;
    c.spare = nullptr;
  }
}

// G <- G[g0:] xor F[f0:]; then, if G holds more than GCAP entries, M <- M[h:] xor G (F is empty
// then, so both of its buffers are merge scratch).  Returns false on capacity overflow.
// (The log-structured tiers keep the cost of a flush at O(|G|) -- round 1 merged F straight into
// M, O(|M|) per flush, which dominated the longest columns: 48k-entry M, ~420k cycles a flush.)
template <class CT>
__device__ __forceinline__ bool flush(CT& c, const RP& P, int lane) {
  const uint32_t na = c.ng - c.g0, nb = c.nf - c.f0;
  if (nb == 0) return true;
  c.hstale = true;
  const long long t0 = CT::dbg ? clock64() : 0;
  uint32_t n;
  if (na == 0) {
    for (uint32_t i = lane; i < nb; i += 32) c.Ga[i] = c.Fc[c.f0 + i];
    __syncwarp();
    n = nb;
  } else {
    n = merge_xor_path_g(c.Gc + c.g0, na, c.Fc + c.f0, nb, c.Ga, lane);
  }
  CR_DASSERT(n <= GCAP + FCAP);
  { uint64_t* t = c.Gc; c.Gc = c.Ga; c.Ga = t; }
  c.ng = n;
  c.g0 = 0;
  c.gstale = true;
  c.nf = c.f0 = 0;
  // G moves into M once it outgrows ~K5_GK sqrt(|M|) (at least 2048, at most GCAP): the cost of a
  // flush grows with |G| and that of a G -> M merge with |M|, so the balance point moves with |M|
  uint32_t glim = uint32_t(float(K5_GK) * __fsqrt_rn(float(c.nm - c.h)));
  glim = glim < 2048u ? 2048u : (glim > GCAP ? GCAP : glim);
  if (c.ng > glim) {
    const uint32_t nm = c.nm - c.h;
    if (!grow(c, nm + c.ng, P, lane)) return false;
    const uint32_t n2 = merge_chunked<true>(c.Mc + c.h, nm, c.Gc, c.ng, c.Ma,
                                            c.Fc, c.Fa, lane);
    CR_DASSERT(n2 <= c.cap);
    swap_main(c);
    c.nm = n2;
    c.h = 0;
    c.mstale = true;
    c.ng = c.g0 = 0;
    if (CT::dbg) c.fent += nm;
  }
  if (CT::dbg) {
    c.fcyc += clock64() - t0;
    ++c.fn;
  }
  return true;
}

constexpr uint32_t STAGE = 64;
constexpr unsigned long long POOL_CHUNK = 4096;  // pool entries a warp reserves at a time  // global addends are staged in shared memory, STAGE entries at a time

// F <- F xor R, R emptied (flushing F into M first if it cannot take R).  Warp-collective.
template <class CT>
__device__ __forceinline__ bool spill_r(CT& c, const RP& P, uint64_t* scratch, int lane) {
  const uint32_t live = c.nr;
  if (live > 0) {
    if ((c.nf - c.f0) + live > FCAP && !flush(c, P, lane)) return false;
    const uint64_t v = bag_sorted(c.rv, lane);  // R's entries ascending in lanes [0, live)
    if (uint32_t(lane) < live) scratch[lane] = v;
    __syncwarp();
    if (c.nf == c.f0) {
      if (uint32_t(lane) < live) c.Fc[lane] = scratch[lane];
      c.nf = live;
    } else {
      c.nf = merge_symdiff<false, false>(c.Fc + c.f0, c.nf - c.f0, scratch, live,
                                         c.Fa, lane);
      { uint64_t* t = c.Fc; c.Fc = c.Fa; c.Fa = t; }
    }
    c.f0 = 0;
    CR_DASSERT(c.nf <= FCAP);
    __syncwarp();
    c.hstale = true;
  }
  c.rv = NONE64;
  c.nr = 0;
  c.rmin = NONE64;
  return true;
}

// column += B (sorted; BG: B in global memory).  Returns false on capacity overflow.
template <bool BG, class CT>
__device__ __forceinline__ bool add_column(CT& c, const uint64_t* B, uint32_t nb, const RP& P, int lane,
                           uint64_t* stage, uint64_t* small) {
  if (nb <= SMALLB) {  // into the register list
    if (BG) {
      if (uint32_t(lane) < nb) small[lane] = ldcg64(B + lane);
      __syncwarp();
      B = small;
    }
    const long long t0 = CT::dbg ? clock64() : 0;
    if (c.nr + nb > 32) {
      if (!spill_r(c, P, stage, lane)) return false;
      if (CT::dbg) ++c.nsp;
    }
    const long long t1 = CT::dbg ? clock64() : 0;
    r_insert(c, B, nb, stage, lane);
    if (CT::dbg) {
      c.scyc += t1 - t0;
      c.rcyc += clock64() - t1;
    }
    return true;
  }
  c.hstale = true;  // F or M is rewritten below
  if (BG && (c.nf - c.f0) + nb <= FCAP) {
    // STAGE entries at a time: one coalesced load each instead of a dependent global binary
    // search per F entry (F xor B = F xor B[0:64] xor B[64:128] ...)
    for (uint32_t b0 = 0; b0 < nb; b0 += STAGE) {
      const uint32_t m = nb - b0 < STAGE ? nb - b0 : STAGE;
      for (uint32_t i = lane; i < m; i += 32) stage[i] = ldcg64(B + b0 + i);
      __syncwarp();
      const uint32_t n =
          m <= SMALLB
              ? merge_small(c.Fc + c.f0, c.nf - c.f0, stage, m, c.Fa, lane)
              : merge_symdiff<false, false>(c.Fc + c.f0, c.nf - c.f0, stage, m, c.Fa, lane);
      { uint64_t* t = c.Fc; c.Fc = c.Fa; c.Fa = t; }
      c.nf = n;
      c.f0 = 0;
      CR_DASSERT(c.nf <= FCAP);
    }
    return true;
  }
  if (!BG && nb <= SMALLB && (c.nf - c.f0) + nb <= FCAP) {
    const uint32_t n = merge_small(c.Fc + c.f0, c.nf - c.f0, B, nb, c.Fa, lane);
    { uint64_t* t = c.Fc; c.Fc = c.Fa; c.Fa = t; }
    c.nf = n;
    c.f0 = 0;
    CR_DASSERT(c.nf <= FCAP);
    return true;
  }
  if ((c.nf - c.f0) + nb <= FCAP) {
    const uint32_t n =
        merge_symdiff<false, BG>(c.Fc + c.f0, c.nf - c.f0, B, nb, c.Fa, lane);
    { uint64_t* t = c.Fc; c.Fc = c.Fa; c.Fa = t; }
    c.nf = n;
    c.f0 = 0;
    CR_DASSERT(c.nf <= FCAP);
    return true;
  }
  if (!flush(c, P, lane)) return false;
  if (nb <= FCAP) {  // F is empty now: B becomes F
    for (uint32_t i = lane; i < nb; i += 32) c.Fc[i] = ld64<BG>(B + i);
    __syncwarp();
    c.nf = nb;
    c.f0 = 0;
    return true;
  }
  if (!grow(c, (c.nm - c.h) + nb, P, lane)) return false;
  const uint32_t n = merge_chunked<BG>(c.Mc + c.h, c.nm - c.h, B, nb, c.Ma,
                                       c.Fc, c.Fa, lane);
  CR_DASSERT(n <= c.cap);
  swap_main(c);
  c.nm = n;
  c.h = 0;
  c.mstale = true;
  return true;
}

// ---------------------------------------------------------------- the asynchronous commit rule

// Release / acquire fences at GPU scope.  __threadfence (fence.sc) also invalidates the SM's L1
// (SASS CCTL.IVALL), which drops every warp's cached births and tags; a release needs only the
// MEMBAR (fence.release.gpu, no CCTL), and the one acquire site uses fence.acquire.gpu (CCTL
// only).  Every load of data other warps write (lv, the owner table, the pool) is L2-coherent
// (ld.relaxed.gpu / ld.cg), so L1 holds only read-only data.
#ifndef K5_SLEEP_MAX
#define K5_SLEEP_MAX 2048  // ns: the back-off of a column waiting on an earlier one
#endif
#ifndef K5_SLEEP0
#define K5_SLEEP0 64
#endif
__device__ __forceinline__ void fence_release() {
  asm volatile("fence.release.gpu;" ::: "memory");
}
__device__ __forceinline__ void fence_acquire() {
  asm volatile("fence.acquire.gpu;" ::: "memory");
}

__device__ __forceinline__ uint64_t ld_rlx(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rlx(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ int ld_rlx_i32(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// The first column i in [x, j) whose published candidate is <= p (it may still end on p, or is
// not started), or j if there is none.  Warp-collective.  Chunks of 32^L columns whose bound
// lv[L] exceeds p are skipped whole, 32 chunks per load.  The chunks whose bound does not are
// re-derived from their 32 children in parallel (lane = chunk, 32 independent loads each) and
// their bounds raised with atomicMax -- the children's current values are lower bounds of the
// chunk's later minimum -- and only the first chunk that still fails is entered.  A column found
// > p or finished stays so (candidates only grow), so the caller resumes after a blocker.
// *xfin: every column in [seg_lo, *xfin) is known finished; advanced while the scan starts there.
__device__ __forceinline__ uint32_t find_blocker(const RP& P, uint32_t x, uint32_t j, uint64_t p,
                                                 uint32_t* xfin, int lane) {
  uint32_t desc_end[4] = {0u, 0u, 0u, 0u};  // end of the last level-L chunk entered
  bool fin_run = x == *xfin;                // the scan has seen only finished columns so far
  while (x < j) {
    int L = 0;
#pragma unroll
    for (int l = 3; l >= 1; --l) {
      const uint32_t sz = 1u << (5 * l);
      if (L == 0 && (x & (sz - 1)) == 0 && uint64_t(x) + sz <= j && x >= desc_end[l]) L = l;
    }
    if (L == 0) {  // single columns, up to the next 32-aligned position (where chunks resume)
      const uint32_t to_edge = 32u - (x & 31u);
      const uint32_t n = j - x < to_edge ? j - x : to_edge;
      const uint64_t v = uint32_t(lane) < n ? ld_rlx(P.lv[0] + x + lane) : NONE64;
      const unsigned bad = __ballot_sync(0xFFFFFFFFu, v <= p);
      const unsigned notfin = __ballot_sync(0xFFFFFFFFu, v != NONE64);
      if (fin_run) {
        const uint32_t nf = notfin ? uint32_t(__ffs(notfin) - 1) : n;
        *xfin = x + (nf < n ? nf : n);
        fin_run = !notfin;
      }
      if (bad) return x + __ffs(bad) - 1;
      x += n;
      continue;
    }
    const int sh = 5 * L;
    const uint32_t e = x >> sh;
    // whole chunks in range, up to the next level-(L+1) boundary (so the next step can use it)
    const uint32_t to_edge = 32u - (e & 31u);
    const uint32_t m = ((j - x) >> sh) < to_edge ? ((j - x) >> sh) : to_edge;
    uint64_t v = uint32_t(lane) < m ? ld_rlx(P.lv[L] + e + lane) : NONE64;
    if (__any_sync(0xFFFFFFFFu, v <= p)) {
      if (v <= p) {  // re-derive this lane's chunk from its children
        const uint64_t* ch = P.lv[L - 1] + (uint64_t(e + lane) << 5);
        uint64_t mn = NONE64;
#pragma unroll 8
        for (int k = 0; k < 32; ++k) {
          const uint64_t cv = ld_rlx(ch + k);
          mn = cv < mn ? cv : mn;
        }
        if (mn > v) atomicMax(reinterpret_cast<unsigned long long*>(P.lv[L] + e + lane), mn);
        v = mn;
      }
    }
    const unsigned bad = __ballot_sync(0xFFFFFFFFu, v <= p);
    if (fin_run) {
      const unsigned notfin = __ballot_sync(0xFFFFFFFFu, uint32_t(lane) < m && v != NONE64);
      const uint32_t nf = notfin ? uint32_t(__ffs(notfin) - 1) : m;
      *xfin = x + (nf << sh);
      fin_run = !notfin;
    }
    if (!bad) {
      x += m << sh;
      continue;
    }
    const uint32_t f = __ffs(bad) - 1;
    x += f << sh;
    desc_end[L] = x + (1u << sh);  // enter chunk f: its 32 children are examined next
  }
  return j;
}

// Column j is finished: publish it (after its owner entry / record, fenced) and raise the bounds
// of its chunks -- the level-1 bound to its 32 columns' current minimum, the levels above while
// their chunks are entirely finished.  Warp-collective.
__device__ __forceinline__ void finish_column(const RP& P, uint32_t j, int lane) {
  __syncwarp();
  if (lane == 0) {
    fence_release();  // the owner entry and the record are visible before "finished"
    st_rlx(P.lv[0] + j, NONE64);
  }
  __syncwarp();
  // (no fence before reading the siblings: a bound left stale by two columns finishing at once
  // only costs a later scanner one re-derivation, never correctness)
  uint32_t e = j;
  for (int L = 1; L <= 3; ++L) {
    e >>= 5;
    const uint64_t cv = ld_rlx(P.lv[L - 1] + (uint64_t(e) << 5) + lane);
    const uint64_t mn = bag_min(cv);  // two 32-bit reductions instead of five 64-bit shuffles
    if (lane == 0 && mn > ld_rlx(P.lv[L] + e)) {
      atomicMax(reinterpret_cast<unsigned long long*>(P.lv[L] + e), mn);
      fence_release();
    }
    __syncwarp();
    if (mn != NONE64) break;
  }
}

// Next column for this warp: columns are handed out in processing order within each segment;
// consecutive fetches go to consecutive segments, so independent images progress together.
// Returns (segment, column) or column NONE32 when every segment is exhausted.
__device__ __forceinline__ uint32_t fetch_column(const RP& P, uint32_t& seg, int lane) {
  uint32_t j = NONE32, s = 0;
  if (lane == 0) {
    const unsigned long long c = P.nseg > 1 ? atomicAdd(P.fetch, 1ull) : 0ull;
    for (uint32_t t = 0; t < P.nseg; ++t) {
      s = uint32_t((c + t) % P.nseg);
      const uint32_t lo = __ldg(P.seg_off + s), hi = __ldg(P.seg_off + s + 1);
      if (lo + *reinterpret_cast<volatile unsigned*>(P.seg_next + s) >= hi) continue;
      const uint32_t r = atomicAdd(P.seg_next + s, 1u);
      if (lo + r < hi) {
        j = lo + r;
        break;
      }
    }
  }
  seg = __shfl_sync(0xFFFFFFFFu, s, 0);
  return __shfl_sync(0xFFFFFFFFu, j, 0);
}

__device__ __forceinline__ void jitter_sleep(const RP& P, uint32_t a, uint32_t b) {
  if (!P.jitter) return;
  uint32_t h = a * 0x9E3779B1u ^ (b + 0x7F4A7C15u) * 0x85EBCA6Bu;
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  h ^= h >> 13;
  if ((h & 3) == 0) __nanosleep(h % P.jitter);
}

// 2 resident blocks (16 warps) per SM: 128 registers a thread keep the working column out of
// local memory; measured against 4 / 3 / 1 blocks and F of 256 / 512 / 768 / 1024 entries
// (profiles/r02/s4): C5b 62.5 / 60.3 / 65.0 ms, C5 227 / 223 / 180 ms, C4 31.1 / 30.6 / 26.3 ms
// vs 56.1 / 198 / 26.3 ms here -- the chains of dependent additions, not the number of columns
// in flight, bound the reduction.
#ifndef K5_MINB
#define K5_MINB 2
#endif
constexpr size_t K5_SMEM = sizeof(uint64_t) * WPB * (2 * FCAP + SMALLB + STAGE);
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <bool DBG>
__global__ void __launch_bounds__(THREADS, K5_MINB) k_reduce(RP P) {
  extern __shared__ uint64_t k5_smem[];  // K5Smem
  uint64_t(*s_F)[2][FCAP] = reinterpret_cast<uint64_t(*)[2][FCAP]>(k5_smem);
  uint64_t(*s_small)[SMALLB] = reinterpret_cast<uint64_t(*)[SMALLB]>(k5_smem + WPB * 2 * FCAP);
  uint64_t(*s_stage)[STAGE] = reinterpret_cast<uint64_t(*)[STAGE]>(k5_smem + WPB * (2 * FCAP + SMALLB));
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const uint32_t w = blockIdx.x * WPB + wib;

  ColT<DBG> c;
  using CT = ColT<DBG>;
  uint64_t* const slot = P.work + uint64_t(w) * 2 * P.mcap;
  uint64_t* const gslot = P.gwork + uint64_t(w) * 2 * (GCAP + FCAP);
  const SpecLane sl = spec_lane(P.g, lane);
  c.Fc = s_F[wib][0];
  c.Fa = s_F[wib][1];
  unsigned long long pool_cur = 0, pool_end = 0;  // this warp's current pool chunk
  unsigned adds = 0, waits = 0, maxlen = 0;
  unsigned long long addlen = 0, wcyc = 0, commits = 0;

  for (;;) {
    if (ld_rlx_i32(P.err)) break;
    uint32_t seg;
    const long long tf0 = DBG ? clock64() : 0;
    const uint32_t j = fetch_column(P, seg, lane);
    if (j == NONE32) break;
    const long long tf1 = DBG ? clock64() : 0;
    long long t_scan = 0, t_commit = 0;
    const uint32_t seg_lo = __ldg(P.seg_off + seg);
    const uint32_t cell = rkid(P, P.cols[j]);

    c.h = c.f0 = c.nm = 0;
    c.Mc = slot;  // a column grown into the pool last time starts over in the slot
    c.Ma = slot + P.mcap;
    c.Gc = gslot;
    c.Ga = gslot + (GCAP + FCAP);
    c.ng = c.g0 = 0;
    c.gstale = true;
    c.cap = P.mcap;
    c.spare = nullptr;
    c.rv = NONE64;
    c.nr = 0;
    c.rmin = NONE64;
    c.mstale = true;
    c.hstale = true;
    c.nf = coboundary(P, cell, c.Fc, lane);
    const unsigned long long c_t0 = DBG ? gtimer() : 0;
    unsigned c_pre = 0;     // debug: apparent additions before the first non-apparent pivot
    bool c_inpre = true;
    c.fcyc = 0;
    c.fent = 0;
    c.fn = 0;
    c.tpi = c.tpm = c.tpg = 0;
    c.nsp = 0;
    c.rcyc = c.scyc = 0;
    unsigned long long d_tp = 0, d_lk = 0, d_app = 0, d_pool = 0, d_napp = 0, d_plen = 0;
    unsigned long long c_adds = adds, c_wait = 0, c_waits = waits;
    uint32_t c_blk = NONE32;
    KT(unsigned long long kt_piv = 0, kt_mem = 0, kt_cons = 0, kt_spill = 0, kt_ins = 0, kt_app = 0;
       const long long kt_c0 = clock64();)
    uint64_t pub = 0;      // last published candidate
    uint64_t xp = NONE64;  // the pivot the scan cursor x is valid for
    uint32_t x = seg_lo;
    uint32_t xfin = seg_lo;  // [seg_lo, xfin): known finished
    bool ok = true;
    while (true) {
      const long long q0 = DBG ? clock64() : 0;
      KT(const long long k0 = clock64();)
      const uint64_t piv = take_pivot(c, lane);
      KT(const long long k1 = clock64(); kt_piv += k1 - k0;)
      const long long q1 = CT::dbg ? clock64() : 0;
      d_tp += q1 - q0;
      if (piv == NONE64) {  // zero column: essential (exact given the clearing)
        if (lane == 0) {
          P.rec[j] = (uint64_t(cell) << 32) | NONE32;  // one record per column: no counter
          atomicAdd(P.ness, 1ull);
        }
        break;
      }
      if (piv != pub) {
        if (lane == 0) st_rlx(P.lv[0] + j, piv);
        pub = piv;
      }
      const uint32_t pk = rkid(P, piv);
      // independent loads: the speculated partner coboundary, the tag, the owner record
      const Spec sp = spec_issue(P, sl, pk);
      const uint8_t t = __ldg(P.tags + pk);

      const uint64_t* add;
      uint32_t alen;
      bool glob;
      const long long q2 = CT::dbg ? clock64() : 0;
      d_lk += q2 - q1;
      if (tag_kind(t) == KIND_DOWN) {
        // the pivot is the upper cell of an apparent pair (s', pivot): add delta(s') minus the
        // pivot, straight from the speculated births into the register list R
        const int dir = tag_dir(t);
        const uint64_t y = (lane < 30 && lane / 5 == dir && sp.birth != ABSENT_ORD)
                               ? rkey(P, sp.birth, sp.cell) : NONE64;
        const unsigned vm = __ballot_sync(0xFFFFFFFFu, y != NONE64);
        KT(const long long k2 = clock64(); kt_mem += k2 - k1;)
        consume_pivot(c, lane);
        KT(const long long k3 = clock64(); kt_cons += k3 - k2;)
        if (DBG && c_inpre) ++c_pre;
        const uint32_t ny = __popc(vm);
        addlen += c.len() + ny;
        if (ny) {
          if (c.nr + ny > 32) ok = spill_r(c, P, s_stage[wib], lane);
          if (!ok) break;
          KT(const long long k4 = clock64(); kt_spill += k4 - k3;)
          bag_insert(c, y, vm, s_stage[wib], lane);
          KT(kt_ins += clock64() - k4;)
        }
        KT(++kt_app;)
        ++adds;
        if (DBG) {
          d_app += clock64() - q2;
          ++d_napp;
        }
        const unsigned l = c.len();
        maxlen = l > maxlen ? l : maxlen;
        continue;
      }
      // not apparent: is the pivot owned by a committed column? (probed only now -- apparent
      // pivots, 93 % of them, never touch the table)
      const uint64_t oi = owner_of(P.otab, P.omask, pk);
      if (oi != NONE64) {
        if (DBG) c_inpre = false;
        // the owner's reduced column starts with the pivot itself
        add = P.pool + (oi >> OI_LEN_BITS) + 1;
        alen = uint32_t(oi & ((1u << OI_LEN_BITS) - 1)) - 1;
        glob = true;
        consume_pivot(c, lane);
      } else {
        if (DBG) c_inpre = false;
        // unowned pivot: wait until no earlier column of the segment can end on it
        jitter_sleep(P, j, uint32_t(adds));
        if (xp != piv) {  // a new pivot: earlier columns are checked again, past the finished ones
          x = xfin;
          xp = piv;
        }
        bool owned = false;
        while (!owned) {
          const long long ts0 = DBG ? clock64() : 0;
          const uint32_t b = find_blocker(P, x, j, piv, &xfin, lane);
          if (DBG) t_scan += clock64() - ts0;
          if (b == j) break;
          x = b;
          ++waits;
          c_blk = b;
          const long long t0 = DBG ? clock64() : 0;
          // Waiting must stay cheap: 32 warps share an SM's issue slots with the working ones.
          // All lanes read the same word (one transaction, the same value in every lane: no
          // shuffles); the owner entry and the error flag are looked at every 8th try; the
          // back-off grows to 2 us.
          unsigned ns = K5_SLEEP0;
          for (int it = 1;; ++it) {
            if (ld_rlx(P.lv[0] + b) > piv) break;
            if ((it & 7) == 0) {
              if (ld_rlx_i32(P.err)) {
                ok = false;
                break;
              }
              if (owner_of_rlx(P.otab, P.omask, pk) != NONE64) {  // an earlier column committed it
                owned = true;
                break;
              }
            }
            __nanosleep(ns);
            if (ns < K5_SLEEP_MAX) ns <<= 1;
          }
          if (DBG) {
            wcyc += clock64() - t0;
            c_wait += clock64() - t0;
          }
          if (!ok) break;
          x = b + 1;
        }
        if (!ok) break;
        if (!owned) {  // every earlier column is finished or beyond piv: final check, commit
          uint64_t o = 0;
          if (lane == 0) {
            fence_acquire();  // the owner entries published before the "finished" flags seen
            o = owner_of_rlx(P.otab, P.omask, pk);
          }
          owned = __shfl_sync(0xFFFFFFFFu, o, 0) != NONE64;
        }
        if (owned) continue;  // the owner's column is added on the next pass
        const long long tc0 = DBG ? clock64() : 0;
        ok = spill_r(c, P, s_stage[wib], lane);  // the commit reads M and F
        if (!ok) break;
        const uint32_t L = c.len();
        // pool space from the warp's own chunk (one global atomic per POOL_CHUNK entries, not
        // one per committed column: 2k warps committing 1.5 M columns share the counter)
        if (pool_cur + L > pool_end) {
          const unsigned long long want = L > POOL_CHUNK ? L : POOL_CHUNK;
          unsigned long long base = 0;
          if (lane == 0) base = atomicAdd(P.pool_top, want);
          pool_cur = __shfl_sync(0xFFFFFFFFu, base, 0);
          pool_end = pool_cur + want;
        }
        const unsigned long long off = pool_cur;
        pool_cur += L;
        if (off + L > P.pool_cap) {
          if (lane == 0) atomicOr(P.err, 2);
          ok = false;
          break;
        }
        // reduced column = M[h:] xor G[g0:] xor F[f0:], written straight into the pool
        uint32_t n;
        if (c.nm == c.h && c.ng == c.g0) {  // held in F alone (most columns): a copy
          n = c.nf - c.f0;
          CR_DASSERT(off + n <= P.pool_cap);
          for (uint32_t i = lane; i < n; i += 32) P.pool[off + i] = c.Fc[c.f0 + i];
          __syncwarp();
        } else if (c.ng > c.g0) {
          if (c.nf > c.f0) {
            ok = flush(c, P, lane);  // F into G (G may move into M)
            if (!ok) break;
          }
          n = c.ng > c.g0
                  ? merge_chunked<true>(c.Mc + c.h, c.nm - c.h, c.Gc + c.g0,
                                        c.ng - c.g0, P.pool + off, c.Fc, c.Fa, lane)
                  : merge_chunked<false>(c.Mc + c.h, c.nm - c.h, c.Fc + c.f0,
                                         c.nf - c.f0, P.pool + off, c.Fa, nullptr, lane);
        } else {
          n = merge_chunked<false>(c.Mc + c.h, c.nm - c.h, c.Fc + c.f0, c.nf - c.f0,
                                   P.pool + off, c.Fa, nullptr, lane);
        }
        __syncwarp();  // every lane's pool writes before lane 0's release
        if (lane == 0) {
          if (n >> OI_LEN_BITS) atomicOr(P.err, 4);  // a reduced column of >= 2^24 entries
          fence_release();
          owner_insert(P.otab, P.omask, pk, (uint64_t(off) << OI_LEN_BITS) | n);
          P.rec[j] = (uint64_t(cell) << 32) | pk;  // (birth cell, death cell)
        }
        if (DBG) {
          ++commits;
          t_commit += clock64() - tc0;
        }
        break;
      }
      addlen += c.len() + alen;
      if (alen)
        ok = glob ? add_column<true>(c, add, alen, P, lane, s_stage[wib], s_small[wib])
                  : add_column<false>(c, add, alen, P, lane, s_stage[wib], s_small[wib]);
      if (CT::dbg) {
        const long long q3 = clock64();
        if (glob) {
          d_pool += q3 - q2;
          d_plen += alen;
        } else {
          d_app += q3 - q2;
          ++d_napp;
        }
      }
      if (!ok) break;  // pool exhausted (err 2 set): the launch is retried
      ++adds;
      const unsigned l = c.len();
      maxlen = l > maxlen ? l : maxlen;
    }
    if (!ok) break;
    KT(if (lane == 0 && kt_app > 2000)
         printf("K5T col %u: %llu cycles, %llu apparent adds; per add: pivot %.0f mem %.0f consume %.0f "
                "spill %.0f insert %.0f\n", j, (unsigned long long)(clock64() - kt_c0), kt_app,
                double(kt_piv) / kt_app, double(kt_mem) / kt_app, double(kt_cons) / kt_app,
                double(kt_spill) / kt_app, double(kt_ins) / kt_app);)
    const long long tfin0 = DBG ? clock64() : 0;
    finish_column(P, j, lane);
    if (DBG && lane == 0) {
      unsigned long long* R = P.colrec + 32ull * j;
      R[23] = (uint64_t(seg) << 32) | (j - seg_lo);  // segment, position in it
      R[24] = c_pre;
      R[19] = tf1 - tf0;
      R[20] = t_scan;
      R[21] = t_commit;
      R[22] = clock64() - tfin0;
      R[0] = c_t0;
      R[1] = gtimer();
      R[2] = adds - c_adds;
      R[3] = c_wait;
      R[4] = waits - c_waits;
      R[5] = c_blk;
      R[6] = w;
      {
        R[8] = d_tp;
        R[9] = d_lk;
        R[10] = d_app;
        R[11] = d_pool;
        R[12] = d_napp;
        R[13] = d_plen;
        R[14] = (unsigned long long)c.fcyc;
        R[15] = ((unsigned long long)c.fn << 40) | c.fent;
        R[7] = ((unsigned long long)c.tpi << 40) | ((unsigned long long)c.tpm << 20) | c.tpg;
        R[16] = (unsigned long long)c.rcyc;
        R[17] = (unsigned long long)c.scyc;
        R[18] = c.nsp;
      }
    }
  }
  if (lane == 0) {
    atomicAdd(P.stats + 0, (unsigned long long)waits);
    atomicAdd(P.stats + 1, (unsigned long long)adds);
    atomicAdd(P.stats + 2, addlen);
    atomicMax(P.stats + 3, (unsigned long long)maxlen);
    atomicAdd(P.stats + 4, wcyc);
    atomicAdd(P.stats + 5, commits);
  }
}

// lv[0][i] = 0 for real columns (not started), NONE64 for the padding; chunk bounds likewise.
__global__ void k_levels_init(uint64_t* lv0, uint64_t* lv1, uint64_t* lv2, uint64_t* lv3,
                              uint32_t ncols, uint32_t npad) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= npad) return;
  lv0[i] = i < ncols ? 0ull : NONE64;
  if (i < (npad >> 5)) lv1[i] = (uint64_t(i) << 5) < ncols ? 0ull : NONE64;
  if (i < (npad >> 10)) lv2[i] = (uint64_t(i) << 10) < ncols ? 0ull : NONE64;
  if (i < (npad >> 15)) lv3[i] = (uint64_t(i) << 15) < ncols ? 0ull : NONE64;
}

// Columns of dimension d: finite residual d-cells (not apparent, not cleared), as keys.  One thread
// per voxel v enumerates the d-cells with base voxel v (odd Khalimsky offsets on d of the axes).
__global__ void k_collect_columns(const uint32_t* __restrict__ births,
                                  const uint8_t* __restrict__ tags, Geom g, int d,
                                  uint64_t* __restrict__ cols, unsigned* __restrict__ ncols) {
  uint32_t v, c[3];
  const bool in0 = vox_of_thread(g, v, c[0], c[1], c[2]);
  const uint32_t n[3] = {uint32_t(g.nx), uint32_t(g.ny), uint32_t(g.nz)};
  const uint32_t ks[3] = {1u, uint32_t(g.KX), uint32_t(g.KX * g.KY)};
  const uint32_t kb = (2 * c[2] * uint32_t(g.KY) + 2 * c[1]) * uint32_t(g.KX) + 2 * c[0];
  const bool in = in0 && births[kb] != ABSENT_ORD;  // every cell with base v contains v
  bool emit[3] = {false, false, false};
  uint64_t key[3] = {0, 0, 0};
  int q = 0;
#pragma unroll
  for (int t = 1; t < 8; ++t) {  // cell type: bit a set = odd along axis a
    if (__popc(t) != d || q >= 3) continue;
    if (in) {
      bool ok = true;
      uint32_t k = kb;
#pragma unroll
      for (int a = 0; a < 3; ++a)
        if (t >> a & 1) {
          ok = ok && c[a] + 1 < n[a];
          k += ks[a];
        }
      // the tag first (1 B; ~1 % of the cells are residual), the birth only for residual or
      // absent ones (an absent cell's tag is 0 too)
      if (ok && tag_kind(tags[k]) == KIND_RESIDUAL) {
        const uint32_t b = births[k];
        if (b != ABSENT_ORD) {
          emit[q] = true;
          key[q] = make_key(b, k);
        }
      }
    }
    ++q;
  }
  warp_append(emit, key, cols, ncols);
}

// Dim-1 columns from H0's candidates: the edges whose tag is still residual (not cleared by an
// H0 merge).  One thread per candidate, one append atomic per warp.
__global__ void k_cols_from_cands(const H0Cand* __restrict__ cand, uint32_t n,
                                  const uint8_t* __restrict__ tags, uint64_t* __restrict__ cols,
                                  unsigned* __restrict__ ncols) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  bool emit[1] = {false};
  uint64_t key[1] = {0};
  if (i < n) {
    key[0] = cand[i].key;
    CR_DASSERT(key_ord(key[0]) != ABSENT_ORD);
    emit[0] = tag_kind(tags[key_kidx(key[0])]) == KIND_RESIDUAL;
  }
  warp_append(emit, key, cols, ncols);
}

__global__ void k_seg_keys(const uint64_t* __restrict__ cols, unsigned n, uint32_t seg_cells,
                           uint32_t* __restrict__ segk) {
  unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) segk[i] = key_kidx(cols[i]) / seg_cells;
}

// seg_off[t] = first position i with segk[i] >= t (segk sorted ascending), t = 0..nseg
__global__ void k_seg_offsets(const uint32_t* __restrict__ segk, unsigned n, unsigned nseg,
                              uint32_t* __restrict__ seg_off) {
  const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t > nseg) return;
  unsigned a = 0, b = n;
  while (a < b) {
    const unsigned m = (a + b) >> 1;
    if (segk[m] < t) a = m + 1;
    else b = m;
  }
  seg_off[t] = a;
}

__global__ void k_seg_single(unsigned n, uint32_t* seg_off) {
  if (threadIdx.x < 2) seg_off[threadIdx.x] = threadIdx.x ? n : 0u;
}

__global__ void k_mark_cleared(const uint64_t* __restrict__ rec, int64_t n, uint8_t* tags) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t dk = uint32_t(rec[i]);
  if (dk != NONE32) tags[dk] = make_tag(KIND_CLEARED, 0);
}

}  // namespace

// Debug (option debug >= 2): the chain that ends the launch -- from the last column to finish,
// follow each column's last blocker -- and the busiest columns.
static void debug_critical_path(const unsigned long long* dcol, uint32_t ncols, cudaStream_t s) {
  constexpr int RW = 32;
  std::vector<unsigned long long> R(RW * size_t(ncols));
  CR_CUDA(cudaMemcpyAsync(R.data(), dcol, R.size() * 8, cudaMemcpyDeviceToHost, s));
  CR_CUDA(cudaStreamSynchronize(s));
  unsigned long long t0 = ~0ull, t1 = 0;
  uint32_t last = 0;
  for (uint32_t j = 0; j < ncols; ++j) {
    t0 = std::min(t0, R[RW * j]);
    if (R[RW * j + 1] > t1) t1 = R[RW * j + 1], last = j;
  }
  fprintf(stderr, "[cr] K5 span %.3f ms; chain from the last column (col: start..end us, adds, "
          "wait us, waits, blocker):\n", (t1 - t0) / 1e6);
  uint32_t cur = last;
  for (int k = 0; k < 40 && cur != NONE32 && cur < ncols; ++k) {
    const unsigned long long* r = &R[RW * size_t(cur)];
    fprintf(stderr, "   %u (seg %llu pos %llu): %.1f..%.1f adds %llu wait %.1f waits %llu blk %lld\n",
            cur, r[23] >> 32, r[23] & 0xFFFFFFFFull, (r[0] - t0) / 1e3, (r[1] - t0) / 1e3, r[2],
            r[3] / 1.9e3, r[4], r[5] == NONE32 ? -1ll : (long long)r[5]);
    cur = uint32_t(r[5]);
  }
  std::vector<std::pair<unsigned long long, uint32_t>> busy(ncols);
  for (uint32_t j = 0; j < ncols; ++j) busy[j] = {R[RW * j + 1] - R[RW * j], j};
  std::sort(busy.rbegin(), busy.rend());
  fprintf(stderr, "[cr] longest columns (col: start..end us, adds, wait us):\n");
  for (int k = 0; k < 12 && k < int(ncols); ++k) {
    const uint32_t j = busy[k].second;
    const unsigned long long* r = &R[RW * size_t(j)];
    fprintf(stderr, "   %u: %.1f..%.1f adds %llu (apparent before the first other pivot: %llu) "
            "wait %.1f\n", j, (r[0] - t0) / 1e3, (r[1] - t0) / 1e3, r[2], r[24], r[3] / 1.9e3);
    if (r[8] + r[9] + r[10] + r[11]) {
      const double a = r[2] ? double(r[2]) : 1.0, pa = double(r[2] - r[12]);
      fprintf(stderr, "      take_pivot: %.2f iterations, %.3f M and %.3f G window reloads per call;"
              " r_insert %.0f cycles per apparent add, spills %llu at %.0f cycles (incl. flushes)\n",
              double(r[7] >> 40) / (a + 1), double((r[7] >> 20) & 0xFFFFF) / (a + 1),
              double(r[7] & 0xFFFFF) / (a + 1), r[12] ? r[16] / double(r[12]) : 0.0, r[18],
              r[18] ? r[17] / double(r[18]) : 0.0);
      fprintf(stderr, "      per add cycles: pivot %.0f lookup %.0f | apparent adds %llu at %.0f, "
              "pool adds %.0f at %.0f (avg len %.0f) | flushes %llu: %.0f cycles each, avg M %.0f\n",
              r[8] / a, r[9] / a, r[12], r[12] ? r[10] / double(r[12]) : 0.0, pa,
              pa ? r[11] / pa : 0.0, pa ? r[13] / pa : 0.0, r[15] >> 40,
              (r[15] >> 40) ? r[14] / double(r[15] >> 40) : 0.0,
              (r[15] >> 40) ? double(r[15] & ((1ull << 40) - 1)) / double(r[15] >> 40) : 0.0);
    }
  }
  {
    unsigned long long pre = 0, all = 0;
    for (uint32_t j = 0; j < ncols; ++j) {
      pre += R[RW * size_t(j) + 24];
      all += R[RW * size_t(j) + 2];
    }
    fprintf(stderr, "[cr] additions %llu, apparent ones before a column's first other pivot %llu\n",
            all, pre);
  }
  {  // where the warps' time goes, summed over all columns (cycles -> ms of warp time)
    double tot = 0, add = 0, wait = 0, fetch = 0, scan = 0, commit = 0, fin = 0;
    for (uint32_t j = 0; j < ncols; ++j) {
      const unsigned long long* r = &R[RW * size_t(j)];
      tot += double(r[1] - r[0]) * 1.9;  // ns -> cycles at ~1.9 GHz
      wait += double(r[3]);
      fetch += double(r[19]);
      scan += double(r[20]);
      commit += double(r[21]);
      fin += double(r[22]);
      add += double(r[8] + r[9] + r[10] + r[11]);
    }
    fprintf(stderr, "[cr] column time (sum over columns, %% of column lifetimes): pivot+lookup+adds "
            "%.1f%%, waits %.1f%%, scans %.1f%%, commits %.1f%%, finish %.1f%%, fetch %.3g cycles "
            "total\n", 100 * add / tot, 100 * wait / tot, 100 * scan / tot, 100 * commit / tot,
            100 * fin / tot, fetch);
  }
  // in-flight profile: columns started but unfinished, sampled at 20 instants
  for (int q = 1; q < 20; ++q) {
    const unsigned long long tq = t0 + (t1 - t0) * q / 20;
    uint32_t inflight = 0, done = 0;
    for (uint32_t j = 0; j < ncols; ++j) {
      inflight += R[RW * j] <= tq && R[RW * j + 1] > tq;
      done += R[RW * j + 1] <= tq;
    }
    fprintf(stderr, "   t=%.1f ms: in flight %u, done %u\n", (tq - t0) / 1e6, inflight, done);
  }
}

void reduce_dimension(GeneralState& S, int d, Workspace& ws, HostScalars& hs, cr_stats& st) {
  cudaStream_t s = ws.stream();
  const Geom& g = S.g;
  const int B = 256;
  const int64_t nd = st.cells[d];
  S.R.rec[d] = ws.alloc<uint64_t>(nd + 1);  // at most one record per column
  S.R.n[d] = 0;
  if (nd == 0) return;

  unsigned long long* ctr = ws.alloc<unsigned long long>(16);
  CR_CUDA(cudaMemsetAsync(ctr, 0, 16 * sizeof(unsigned long long), s));
  uint64_t* cols = ws.alloc<uint64_t>(nd + 1);
  if (d == 1 && S.h0_cand) {
    // the residual edges H0 did not clear, from H0's candidate list (every residual edge)
    if (S.h0_ncand)
      k_cols_from_cands<<<grid_for(S.h0_ncand, 256), 256, 0, s>>>(
          S.h0_cand, S.h0_ncand, S.tags, cols, reinterpret_cast<unsigned*>(ctr));
    CR_CHECK_LAUNCH();
    ws.release(const_cast<H0Cand*>(S.h0_cand));
    S.h0_cand = nullptr;
  } else {
    k_collect_columns<<<vox_grid(g), VOX_THREADS, 0, s>>>(S.births, S.tags, g, d, cols,
                                                          reinterpret_cast<unsigned*>(ctr));
    CR_CHECK_LAUNCH();
  }
  const unsigned ncols = read_scalar(reinterpret_cast<unsigned*>(ctr), s, hs);
  st.columns[d] = ncols;
  if (ncols > 0) {
    // decreasing (ord << 32 | kidx): kidx has bits_for(ncells) significant bits, ord all 32 --
    // two stable passes over [0, kb) then [32, 64) skip the zero bits in between
    {
      const int kb = bits_for(uint64_t(g.ncells));
      radix_sort<uint64_t, uint32_t>(cols, nullptr, ncols, 0, kb, /*descending=*/true, ws);
      radix_sort<uint64_t, uint32_t>(cols, nullptr, ncols, 32, 64, /*descending=*/true, ws);
    }
    unsigned nseg = 1;
    uint32_t* seg_off = nullptr;
    if (S.seg_cells) {
      // batched images: group the columns by image (stable, so each image keeps its decreasing
      // key order); images are independent complexes, so their relative order is immaterial
      uint32_t* segk = ws.alloc<uint32_t>(ncols);
      k_seg_keys<<<grid_for(ncols, B), B, 0, s>>>(cols, ncols, S.seg_cells, segk);
      CR_CHECK_LAUNCH();
      const uint64_t nimg = (uint64_t(g.ncells) + S.seg_cells - 1) / S.seg_cells;
      radix_sort<uint32_t, uint64_t>(segk, cols, ncols, 0, bits_for(nimg), false, ws);
      nseg = unsigned((uint64_t(g.ncells) + S.seg_cells - 1) / S.seg_cells);
      seg_off = ws.alloc<uint32_t>(nseg + 1);
      k_seg_offsets<<<grid_for(nseg + 1, B), B, 0, s>>>(segk, ncols, nseg, seg_off);
      CR_CHECK_LAUNCH();
    } else {
      seg_off = ws.alloc<uint32_t>(2);
      k_seg_single<<<1, 32, 0, s>>>(ncols, seg_off);
      CR_CHECK_LAUNCH();
    }

    prof_mark(s, d == 1 ? "sort_d1" : (d == 2 ? "sort_d2" : "sort_d3"));  // collect + sort
    int dev = 0, nsm = 0, per_sm = 0;
    CR_CUDA(cudaGetDevice(&dev));
    CR_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    const bool dbg = opt(OPT_DEBUG) >= 2;
    void* const kfn = dbg ? (void*)k_reduce<true> : (void*)k_reduce<false>;
    static thread_local int attr_dev[2] = {-1, -1};
    if (attr_dev[dbg] != dev) {
      CR_CUDA(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, int(K5_SMEM)));
      attr_dev[dbg] = dev;
    }
    CR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, THREADS, K5_SMEM));
    if (per_sm < 1) throw Error{CR_EINTERNAL, "k_reduce cannot be resident"};
    per_sm = per_sm > K5_MINB ? K5_MINB : per_sm;
    if (opt(OPT_K5_BLOCKS_PER_SM) > 0 && opt(OPT_K5_BLOCKS_PER_SM) < per_sm)
      per_sm = int(opt(OPT_K5_BLOCKS_PER_SM));
    int64_t blocks = int64_t(nsm) * per_sm;
    const int64_t need_blocks = (int64_t(ncols) + WPB - 1) / WPB;  // small problems
    if (need_blocks < blocks) blocks = need_blocks;
    const uint32_t W = uint32_t(blocks * WPB);

    const uint32_t npad = (ncols + 32767u) & ~32767u;
    uint64_t* lv = ws.alloc<uint64_t>(int64_t(npad) + npad / 32 + npad / 1024 + npad / 32768);
    uint32_t obits = 10;
    while ((uint64_t(1) << obits) < 4ull * ncols + 1024) ++obits;  // load <= 1/4: short probes
    const uint32_t oslots = 1u << obits;
    ulonglong2* otab = static_cast<ulonglong2*>(ws.alloc_bytes(size_t(oslots) * sizeof(ulonglong2)));
    unsigned* seg_next = ws.alloc<unsigned>(nseg);
    int* err = reinterpret_cast<int*>(ctr + 3);
    unsigned long long* pool_top = ctr + 5;
    unsigned long long* stats = ctr + 6;   // [6..11]
    unsigned long long* fetch = ctr + 12;

    // main-array slot per warp; longer columns grow into the pool.  The pool (reduced columns +
    // grown main arrays) is sized so that exhausting it -- which reruns the whole launch with 4x --
    // does not happen on realistic inputs: 16 entries per column + 32 Mi entries (256 MB)
    const uint32_t mcap = 4096u;
    unsigned long long pool_cap = 16ull * ncols + (1ull << 25) + uint64_t(W) * POOL_CHUNK;
    uint64_t* work = ws.alloc<uint64_t>(int64_t(W) * 2 * mcap);
    uint64_t* gwork = ws.alloc<uint64_t>(int64_t(W) * 2 * (GCAP + FCAP));
    uint64_t* pool = nullptr;
    unsigned long long* colrec = nullptr;
    for (int attempt = 0;; ++attempt) {
      if (!pool) pool = ws.alloc<uint64_t>(int64_t(pool_cap));
      CR_CUDA(cudaMemsetAsync(otab, 0xFF, size_t(oslots) * sizeof(ulonglong2), s));
      CR_CUDA(cudaMemsetAsync(seg_next, 0, nseg * sizeof(unsigned), s));
      CR_CUDA(cudaMemsetAsync(ctr + 3, 0, 13 * sizeof(unsigned long long), s));
      k_levels_init<<<grid_for(npad, B), B, 0, s>>>(lv, lv + npad, lv + npad + npad / 32,
                                                   lv + npad + npad / 32 + npad / 1024, ncols,
                                                   npad);
      CR_CHECK_LAUNCH();
      RP P;
      P.g = g;
      P.fx = FastDiv::make(uint32_t(g.KX));
      P.fxy = FastDiv::make(uint32_t(g.KX * g.KY));
      P.cols = cols;
      P.ncols = ncols;
      P.births = S.births;
      P.tags = S.tags;
      P.otab = otab;
      P.omask = oslots - 1;
      P.pool = pool;
      P.pool_top = pool_top;
      P.pool_cap = pool_cap;
      P.work = work;
      P.mcap = mcap;
      P.gwork = gwork;
      P.lv[0] = lv;
      P.lv[1] = lv + npad;
      P.lv[2] = lv + npad + npad / 32;
      P.lv[3] = lv + npad + npad / 32 + npad / 1024;
      P.seg_off = seg_off;
      P.nseg = nseg;
      P.seg_next = seg_next;
      P.fetch = fetch;
      P.rec = S.R.rec[d];
      P.err = err;
      P.stats = stats;
      P.ness = ctr + 13;
      P.jitter = unsigned(opt(OPT_K5_JITTER_NS));
      P.colrec = nullptr;
      if (dbg) {
        if (!colrec) colrec = ws.alloc<unsigned long long>(32 * int64_t(ncols));
        P.colrec = colrec;
      }
      void* args[] = {&P};
      // cooperative launch: every warp resident at once (a warp may wait on any other's column)
      CR_CUDA(cudaLaunchCooperativeKernel(kfn, dim3(unsigned(blocks)), dim3(THREADS),
                                          args, K5_SMEM, s));
      ++g_launch_count;
      const int e = read_scalar(err, s, hs);
      if (e == 0) break;
      if (e & 4) throw Error{CR_EINTERNAL, "reduced column longer than 2^24 entries"};
      if (attempt > 12) throw Error{CR_ENOMEM, "reduction buffers exhausted"};
      ws.release(pool);
      pool = nullptr;
      pool_cap *= 4;
    }
    CR_CUDA(cudaMemcpyAsync(hs.p, ctr, 16 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    CR_CUDA(cudaStreamSynchronize(s));
    S.R.n[d] = int64_t(ncols);  // one record per column (a pair or an essential class)
    st.rounds[d] = int64_t(hs.p[6]);  // waits on an earlier column
    st.additions[d] = int64_t(hs.p[7]);
    st.addlen[d] = int64_t(hs.p[8]);
    st.maxlen[d] = int64_t(hs.p[9]);
    st.essential[d] = int64_t(hs.p[13]);
    if (opt(OPT_DEBUG))
      fprintf(stderr, "[cr] dim %d: cols %u warps %u waits %llu adds %llu addlen %llu maxlen %llu "
              "wait-cycles/warp %.3g commits %llu pool %llu/%llu\n", d, ncols, W, hs.p[6], hs.p[7],
              hs.p[8], hs.p[9], double(hs.p[10]) / W, hs.p[11], hs.p[5], pool_cap);
    if (colrec) debug_critical_path(colrec, ncols, s);
    ws.release(work);
    ws.release(gwork);
    ws.release(pool);
    ws.release(otab);
    ws.release(lv);
  }
  if (S.R.n[d] > 0) {
    k_mark_cleared<<<grid_for(S.R.n[d], B), B, 0, s>>>(S.R.rec[d], S.R.n[d], S.tags);
    CR_CHECK_LAUNCH();
  }
  ws.release(cols);
}

}  // namespace cr
