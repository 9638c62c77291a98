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
// Parallel schedule (one persistent cooperative kernel).  Warp w owns columns j = w (mod W), W =
// resident warps; the window is the W columns lo..lo+W-1 (lo = first unfinished), one per warp.
// Each round every warp advances its column by at most max_steps additions and publishes its
// current pivot cand(j) at window position j - lo (a lower bound of its final pivot: adding a
// column with the same pivot only moves the pivot later).  Column j with an unowned pivot commits
// iff cand(j) < min{cand(i) : lo <= i < j}: no earlier column can end on that pivot, so j's pivot
// is final, and any column committed while j is unfinished has a pivot j can never reach -- the
// sequential reduction's pairs are reproduced exactly.
#include <cooperative_groups.h>

#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "pipeline.cuh"

namespace cg = cooperative_groups;

namespace cr {
namespace {

constexpr int WPB = 8;  // warps per block
constexpr int THREADS = WPB * 32;
constexpr uint32_t FCAP = 256;  // fresh-array capacity per warp (shared memory, x2 ping-pong)

struct RP {
  Geom g;
  int d;
  const uint64_t* cols;
  uint32_t ncols;
  const uint32_t* births;
  const uint8_t* tags;
  uint32_t* owner;
  uint64_t* pool;
  unsigned long long* pool_top;
  unsigned long long pool_cap;
  unsigned long long* pool_off;
  uint32_t* pool_len;
  uint64_t* work;      // per warp: 2 * mcap main-array entries
  uint32_t mcap;
  uint64_t* cand;      // per window position
  uint64_t* chunkmin;  // per block (positions [WPB*b, WPB*b+WPB))
  uint32_t* chunkflag; // per block: a segment starts inside the chunk
  uint32_t* segpos;    // per window position: segment (image) of its column
  uint32_t seg_cells;  // cells per segment (batched images), 0: one segment
  unsigned* lo_buf;    // [2]
  uint64_t* rec;
  unsigned long long* nrec;
  int* err;
  int max_steps;
  unsigned long long* stats;  // [0] rounds [1] additions [2] sum of lengths [3] max length
                              // debug: [4] pool additions [5] pool lengths [7]/[8] cycles in
                              // pool/apparent additions [9] cycles in pivot + owner lookups
  int debug;
  unsigned long long* colstat;  // debug: per column (additions, entries touched)
  int prefetch;                 // warm next pivots' lookups (CR_K5_PREFETCH=1; measured no gain)
  int lcache;                   // per-warp lookup cache (CR_K5_CACHE=1; measured no gain: the
                                // rounds wait on the heaviest column's addition chain)
};

__device__ __forceinline__ uint64_t ldcg64(const uint64_t* p) {
  return __ldcg((const unsigned long long*)p);
}
template <bool G>
__device__ __forceinline__ uint64_t ld64(const uint64_t* p) {
  return G ? ldcg64(p) : *p;
}

// Per-warp direct-mapped cache of pivot lookups (tag and owner of a (d+1)-cell), in shared
// memory.  Owners change only in the commit phase, so the cache is cleared at every round start;
// tags never change.  Filled by the coboundary enumeration (the cofacets of an apparent partner
// are the likeliest next pivots) and by the pivot lookups themselves.
constexpr int LC = 32;
struct LookupCache {
  uint32_t key[LC];
  uint32_t val[LC];  // tag << 24 | owner (0xFFFFFF: none)
};
constexpr uint32_t LC_NOOWN = 0xFFFFFFu;
__device__ __forceinline__ uint32_t lc_pack(uint8_t tag, uint32_t owner) {
  return (uint32_t(tag) << 24) | (owner == NONE32 ? LC_NOOWN : (owner & LC_NOOWN));
}

// Finite cofacets of cell s, sorted ascending, written to dst (<= 6 entries).  Warp-collective.
template <bool CACHE = false>
__device__ uint32_t coboundary(const RP& P, uint32_t s, uint64_t* dst, int lane,
                              LookupCache* lc = nullptr) {
  const Geom& g = P.g;
  const uint32_t KX = uint32_t(g.KX), KY = uint32_t(g.KY);
  const uint32_t c[3] = {s % KX, (s / KX) % KY, s / (KX * KY)};
  const uint32_t ext[3] = {KX, KY, uint32_t(g.KZ)};
  uint64_t key = NONE64;
  if (lane < 6) {
    const int a = lane >> 1, sg = lane & 1;
    if (!(c[a] & 1) && (sg ? c[a] + 1 < ext[a] : c[a] > 0)) {
      const int64_t stv = g.stride(a);
      const uint32_t t = uint32_t(int64_t(s) + (sg ? stv : -stv));
      const uint32_t tb = __ldg(P.births + t);
      if (CACHE) {  // the cofacet's lookups ride along with its birth (independent loads)
        const uint8_t tt = __ldg(P.tags + t);
        const uint32_t to = __ldcg(P.owner + t);
        if (tb != ABSENT_ORD) {
          lc->key[t & (LC - 1)] = t;
          lc->val[t & (LC - 1)] = lc_pack(tt, to);
        }
      }
      if (tb != ABSENT_ORD) key = make_key(tb, t);
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
template <bool AG, bool BG>
__device__ uint32_t merge_symdiff(const uint64_t* A, uint32_t a, const uint64_t* B, uint32_t b,
                                  uint64_t* C, int lane) {
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

// C = A xor B with A in global memory and B in global (BG) or shared memory, for long inputs:
// merge-path chunks of <= CH elements are staged in shared memory (SA, SB: CH+1 entries each) and
// merged there, so a long array is read once, coalesced, instead of one global binary search per
// element.  Chunks split by the merge path with ties taken from A first; an equal pair split by a
// chunk boundary is kept together by taking B's copy into the chunk too.
template <bool BG>
__device__ uint32_t merge_chunked(const uint64_t* A, uint32_t a, const uint64_t* B, uint32_t b,
                                  uint64_t* C, uint64_t* SA, uint64_t* SB, int lane) {
  constexpr uint32_t CH = FCAP - 1;
  uint32_t i0 = 0, j0 = 0, out = 0;
  while (i0 < a || j0 < b) {
    const uint32_t ra = a - i0, rb = b - j0;
    const uint32_t k = ra + rb < CH ? ra + rb : CH;
    uint32_t i = 0;
    if (lane == 0) {
      uint32_t lo = k > rb ? k - rb : 0, hi = k < ra ? k : ra;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (ldcg64(A + i0 + mid) <= ld64<BG>(B + j0 + k - mid - 1)) lo = mid + 1;
        else hi = mid;
      }
      i = lo;
    }
    i = __shfl_sync(0xFFFFFFFFu, i, 0);
    uint32_t j = k - i;
    if (i > 0 && j < rb && ldcg64(A + i0 + i - 1) == ld64<BG>(B + j0 + j)) ++j;
    for (uint32_t t = lane; t < i; t += 32) SA[t] = ldcg64(A + i0 + t);
    const uint64_t* Bc = B + j0;
    if (BG) {
      for (uint32_t t = lane; t < j; t += 32) SB[t] = ldcg64(B + j0 + t);
      Bc = SB;
    }
    __syncwarp();
    out += merge_symdiff<false, false>(SA, i, Bc, j, C + out, lane);
    i0 += i;
    j0 += j;
  }
  return out;
}

struct MinOp {
  __device__ __forceinline__ uint64_t operator()(uint64_t a, uint64_t b) const {
    return a < b ? a : b;
  }
};
// segmented minimum: (value, starts-a-segment) pairs
struct SegMin {
  uint64_t v;
  uint32_t f;
};
struct SegOp {
  __device__ __forceinline__ SegMin operator()(const SegMin& a, const SegMin& b) const {
    return SegMin{b.f ? b.v : (a.v < b.v ? a.v : b.v), a.f | b.f};
  }
};
typedef cub::BlockScan<SegMin, THREADS> SScan;

// The working column of a warp.
struct Col {
  uint64_t* M[2];  // global main arrays
  uint64_t* F[2];  // shared fresh arrays
  uint32_t mb, nm, h;
  uint32_t fb, nf, f0;
  uint64_t mhead;  // cached M[mb][h] (valid unless mstale)
  bool mstale;
  __device__ uint32_t len() const { return (nm - h) + (nf - f0); }
};

// pivot = min of (M[h:] xor F[f0:]), cancelling equal heads; NONE64 if the column is zero.
// The head of M is cached in a register (mhead) and reloaded only when h moves or M changes.
__device__ __forceinline__ uint64_t take_pivot(Col& c) {
  while (true) {
    if (c.mstale) {
      c.mhead = c.h < c.nm ? ldcg64(c.M[c.mb] + c.h) : NONE64;
      c.mstale = false;
    }
    const uint64_t a = c.mhead;
    const uint64_t b = c.f0 < c.nf ? c.F[c.fb][c.f0] : NONE64;
    if (a != b) return a < b ? a : b;
    if (a == NONE64) return NONE64;
    ++c.h;
    ++c.f0;
    c.mstale = true;
  }
}

// C = A xor F for a long A (global) and a short F (shared, b <= FCAP), C in global memory, using
// X (FCAP u64 of shared scratch).  Warp-collective; returns |C|.
//  1. positions: P[t] = #{A < F[t]} by a sampled search (<= 256 samples of A in X, then a binary
//     search inside one sample interval; a lane's <= 8 searches run interleaved), dup[t] = (A[P[t]]
//     == F[t]); prefix counts of inserted (non-dup) and cancelled (dup) F entries over t;
//  2. the non-dup F entries go to P[t] + ins_before(t) - dup_before(t);
//  3. A streams through in windows of 256 (8 independent loads per lane): A[i] moves to
//     i + #{non-dup t : P[t] <= i} - #{dup t : P[t] < i}, unless a dup lands on it.  A window that
//     holds no position only shifts (one smem search per window).
__device__ uint32_t merge_long_short(const uint64_t* __restrict__ A, uint32_t a, const uint64_t* F,
                                     uint32_t b, uint64_t* __restrict__ C, uint64_t* X, int lane) {
  constexpr int R = FCAP / 32;  // F entries per lane (t = lane + 32 r)
  constexpr int G = 4;          // searches run interleaved per group
  constexpr uint32_t NS = FCAP / 2;
  const unsigned lt = (1u << lane) - 1;
  uint32_t* XP = reinterpret_cast<uint32_t*>(X + NS);  // P[t]            (upper half of X)
  uint32_t* XC = reinterpret_cast<uint32_t*>(X);       // prefix counts   (lower half, later)
  // ---- 1. <= NS samples of A in X[0, NS)
  const uint32_t S = a > NS ? (a + NS - 1) / NS : 1u;
  const uint32_t ns = a ? (a + S - 1) / S : 0u;
  for (uint32_t sidx = lane; sidx < ns; sidx += 32) X[sidx] = ldcg64(A + uint64_t(sidx) * S);
  __syncwarp();
  uint32_t dupm = 0;
#pragma unroll
  for (int g0 = 0; g0 < R; g0 += G) {
    uint32_t lo[G], hi[G];
    uint64_t f[G];
#pragma unroll
    for (int q = 0; q < G; ++q) {
      const uint32_t t = lane + 32 * (g0 + q);
      f[q] = t < b ? F[t] : NONE64;
      uint32_t l = 0, h = ns;  // l = #samples < f; the answer lies in (l-1)*S+1 .. min(a, l*S)
      while (l < h) {
        const uint32_t m = (l + h) >> 1;
        if (X[m] < f[q]) l = m + 1;
        else h = m;
      }
      lo[q] = l ? (l - 1) * S + 1 : 0u;
      hi[q] = l ? min(a, l * S) : 0u;
      if (t >= b) lo[q] = hi[q] = 0;
    }
    bool busy = true;
    while (busy) {  // interleaved binary searches: lower_bound of f in A[lo, hi)
      busy = false;
      uint64_t v[G];
#pragma unroll
      for (int q = 0; q < G; ++q)
        if (lo[q] < hi[q]) v[q] = ldcg64(A + ((lo[q] + hi[q]) >> 1));
#pragma unroll
      for (int q = 0; q < G; ++q)
        if (lo[q] < hi[q]) {
          const uint32_t m = (lo[q] + hi[q]) >> 1;
          if (v[q] < f[q]) lo[q] = m + 1;
          else hi[q] = m;
          busy |= lo[q] < hi[q];
        }
    }
#pragma unroll
    for (int q = 0; q < G; ++q) {
      const uint32_t t = lane + 32 * (g0 + q);
      if (t < b) {
        if (lo[q] < a && ldcg64(A + lo[q]) == f[q]) dupm |= 1u << (g0 + q);
        XP[t] = lo[q];
      }
    }
  }
  __syncwarp();  // the samples are dead: XC takes the lower half
  uint32_t totI = 0, totD = 0;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const uint32_t t = lane + 32 * r;
    const bool valid = t < b, dup = dupm >> r & 1;
    const unsigned bi = __ballot_sync(0xFFFFFFFFu, valid && !dup);
    const unsigned bd = __ballot_sync(0xFFFFFFFFu, valid && dup);
    const uint32_t ci = totI + __popc(bi & lt), cd = totD + __popc(bd & lt);
    if (valid) {
      XC[t] = (uint32_t(dup) << 31) | (cd << 16) | ci;
      if (!dup) C[XP[t] + ci - cd] = F[t];  // 2. the inserted F entries
    }
    totI += __popc(bi);
    totD += __popc(bd);
  }
  __syncwarp();
  // ---- 3. stream A
  auto lower_p = [&](uint32_t x) {  // #t with P[t] < x
    uint32_t l = 0, h = b;
    while (l < h) {
      const uint32_t m = (l + h) >> 1;
      if (XP[m] < x) l = m + 1;
      else h = m;
    }
    return l;
  };
  for (uint32_t w0 = 0; w0 < a; w0 += 256) {
    uint64_t v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t i = w0 + lane + 32 * k;
      v[k] = i < a ? ldcg64(A + i) : 0ull;
    }
    const uint32_t tl = lower_p(w0), th = lower_p(w0 + 256);
    const uint32_t cl = tl < b ? XC[tl] & 0x7FFFFFFFu : ((totD << 16) | totI);
    const uint32_t baseI = cl & 0xFFFFu, baseD = cl >> 16;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t i = w0 + lane + 32 * k;
      if (i >= a) continue;
      uint32_t ins = baseI, rem = baseD;
      bool removed = false;
      for (uint32_t t = tl; t < th; ++t) {
        const uint32_t pt = XP[t];
        const bool dup = XC[t] >> 31;
        if (!dup && pt <= i) ++ins;
        if (dup && pt < i) ++rem;
        if (dup && pt == i) removed = true;
      }
      if (!removed) C[i + ins - rem] = v[k];
    }
  }
  __syncwarp();
  return a + totI - totD;
}

__device__ int g_k5_dbg = 0;                      // CR_DEBUG_STATS: flush counters below
__device__ unsigned long long g_k5_flush[4];      // flushes, cycles, entries of M, long merges

// M <- M[h:] xor F[f0:]   (returns false on capacity overflow)
__device__ bool flush(Col& c, uint32_t mcap, int lane) {
  const uint32_t na = c.nm - c.h, nb = c.nf - c.f0;
  if (nb == 0) return true;
  if (na + nb > mcap) return false;
  const long long t0 = g_k5_dbg ? clock64() : 0;
  const uint32_t n = merge_long_short(c.M[c.mb] + c.h, na, c.F[c.fb] + c.f0, nb,
                                      c.M[c.mb ^ 1], c.F[c.fb ^ 1], lane);
  if (g_k5_dbg && lane == 0) {
    atomicAdd(g_k5_flush + 0, 1ull);
    atomicAdd(g_k5_flush + 1, (unsigned long long)(clock64() - t0));
    atomicAdd(g_k5_flush + 2, (unsigned long long)na);
  }
  c.mb ^= 1;
  c.nm = n;
  c.h = 0;
  c.nf = c.f0 = 0;
  c.mstale = true;
  return true;
}

// column += B (sorted; BG: B in global memory).  Returns false on capacity overflow.
template <bool BG>
__device__ bool add_column(Col& c, const uint64_t* B, uint32_t nb, uint32_t mcap, int lane) {
  if ((c.nf - c.f0) + nb <= FCAP) {
    const uint32_t n =
        merge_symdiff<false, BG>(c.F[c.fb] + c.f0, c.nf - c.f0, B, nb, c.F[c.fb ^ 1], lane);
    c.fb ^= 1;
    c.nf = n;
    c.f0 = 0;
    return true;
  }
  if (!flush(c, mcap, lane)) return false;
  if (nb <= FCAP) {  // F is empty now: B becomes F
    for (uint32_t i = lane; i < nb; i += 32) c.F[c.fb][i] = ld64<BG>(B + i);
    __syncwarp();
    c.nf = nb;
    c.f0 = 0;
    return true;
  }
  if ((c.nm - c.h) + nb > mcap) return false;
  const uint32_t n = merge_chunked<BG>(c.M[c.mb] + c.h, c.nm - c.h, B, nb, c.M[c.mb ^ 1],
                                       c.F[0], c.F[1], lane);
  c.mb ^= 1;
  c.nm = n;
  c.h = 0;
  c.mstale = true;
  return true;
}

__global__ void __launch_bounds__(THREADS, 4) k_reduce(RP P) {
  cg::grid_group grid = cg::this_grid();
  __shared__ uint64_t s_F[WPB][2][FCAP];
  __shared__ uint64_t s_small[WPB][8];
  __shared__ LookupCache s_lc[WPB];
  __shared__ uint64_t s_pref[4 * THREADS];
  __shared__ typename SScan::TempStorage s_scan;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const uint32_t W = (gridDim.x * blockDim.x) >> 5;
  const uint32_t w = blockIdx.x * WPB + wib;
  const uint32_t nblocks = gridDim.x;

  Col c;
  c.M[0] = P.work + uint64_t(w) * 2 * P.mcap;
  c.M[1] = c.M[0] + P.mcap;
  c.F[0] = s_F[wib][0];
  c.F[1] = s_F[wib][1];
  uint32_t j = w;
  bool started = false, fin = false;
  uint32_t lo = 0;

  LookupCache* lc = &s_lc[wib];
  for (uint32_t round = 0;; ++round) {
    for (int i = lane; i < LC; i += 32) lc->key[i] = NONE32;  // owners may have changed
    __syncwarp();
    // ---------------- phase A: advance my column
    if (fin && j < lo) {
      j += W;
      started = false;
      fin = false;
    }
    uint64_t cval = NONE64;
    bool ready = false;
    if (j < P.ncols && !fin) {
      if (!started) {
        started = true;
        c.mb = c.fb = 0;
        c.h = c.f0 = c.nm = 0;
        c.mstale = true;
        c.nf = coboundary<false>(P, key_kidx(P.cols[j]), c.F[0], lane);
      }
      int steps = 0;
      unsigned long long adds = 0, addlen = 0;
      bool ok = true;
      while (true) {
        const long long tl0 = P.debug ? clock64() : 0;
        const uint64_t piv = take_pivot(c);
        if (piv == NONE64) break;
        const uint32_t pk = key_kidx(piv);
        if (P.prefetch && lane >= 1 && lane <= 12) {
          // warm the lookups of the column's next entries (the likely next pivots): their tag and
          // owner lines, so that the dependent chain of the next additions hits L2
          uint64_t e = NONE64;
          if (lane <= 6) {
            const uint32_t i = c.h + lane;
            if (i < c.nm) e = ldcg64(c.M[c.mb] + i);
          } else {
            const uint32_t i = c.f0 + uint32_t(lane - 6);
            if (i < c.nf) e = c.F[c.fb][i];
          }
          if (e != NONE64) {
            const uint32_t ek = key_kidx(e);
            asm volatile("prefetch.global.L2 [%0];" ::"l"(P.tags + ek));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(P.owner + ek));
          }
        }
        uint8_t t;
        uint32_t ocached = 0;
        bool hit = false;
        if (P.lcache) {
          const uint32_t ck = lc->key[pk & (LC - 1)];
          if (ck == pk) {
            const uint32_t v = lc->val[pk & (LC - 1)];
            t = uint8_t(v >> 24);
            ocached = (v & LC_NOOWN) == LC_NOOWN ? NONE32 : (v & LC_NOOWN);
            hit = true;
          }
        }
        if (!hit) t = __ldg(P.tags + pk);
        const uint64_t* add;
        uint32_t alen;
        bool glob;
        if (tag_kind(t) == KIND_DOWN) {
          // the pivot is the upper cell of an apparent pair (s', pivot): add delta(s')
          const uint32_t sp = uint32_t(int64_t(pk) + dir_offset(P.g, tag_dir(t)));
          alen = P.lcache ? coboundary<true>(P, sp, s_small[wib], lane, lc)
                          : coboundary<false>(P, sp, s_small[wib], lane);
          add = s_small[wib];
          glob = false;
        } else {
          const uint32_t o = hit ? ocached : __ldcg(P.owner + pk);
          if (o == NONE32) {
            ready = true;
            cval = piv;
            break;
          }
          add = P.pool + __ldcg(P.pool_off + o);
          alen = __ldcg(P.pool_len + o);
          glob = true;
        }
        if (steps >= P.max_steps) {
          cval = piv;
          break;
        }
        addlen += c.len() + alen;
        const long long t0 = clock64();
        if (P.debug && lane == 0) atomicAdd(P.stats + 9, (unsigned long long)(t0 - tl0));
        ok = glob ? add_column<true>(c, add, alen, P.mcap, lane)
                  : add_column<false>(c, add, alen, P.mcap, lane);
        if (P.debug && lane == 0) {
          const unsigned long long dt = (unsigned long long)(clock64() - t0);
          if (glob) {
            atomicAdd(P.stats + 4, 1ull);
            atomicAdd(P.stats + 5, (unsigned long long)alen);
            atomicAdd(P.stats + 7, dt);
          } else {
            atomicAdd(P.stats + 8, dt);
          }
        }
        if (!ok) {
          if (lane == 0) atomicOr(P.err, 1);
          break;
        }
        ++steps;
        ++adds;
      }
      if (lane == 0 && adds) {
        atomicAdd(P.stats + 1, adds);
        atomicAdd(P.stats + 2, addlen);
        atomicMax(P.stats + 3, (unsigned long long)c.len());
        if (P.colstat) {
          P.colstat[2 * j] += adds;
          P.colstat[2 * j + 1] += addlen;
        }
      }
      if (ok && !ready && cval == NONE64) {  // zero column: essential (exact given clearing)
        fin = true;
        if (lane == 0) {
          const unsigned long long r = atomicAdd(P.nrec, 1ull);
          P.rec[r] = (uint64_t(key_kidx(P.cols[j])) << 32) | NONE32;
        }
      }
    }
    // publish at my window position (every position is owned by exactly one warp), with the
    // segment (image of a batch) of the column: columns of different images never interact, so
    // a column is blocked only by unfinished earlier columns of its own segment
    const uint32_t q = j - lo;
    if (lane == 0 && q < W) {
      P.cand[q] = (j < P.ncols && !fin) ? cval : NONE64;
      P.segpos[q] = (j < P.ncols && P.seg_cells) ? key_kidx(P.cols[j]) / P.seg_cells : 0xFFFFFFFFu;
    }
    grid.sync();

    // ---------------- phase B: segmented minima of the window's chunks of WPB positions
    if (threadIdx.x == 0) {
      uint64_t m = NONE64;
      uint32_t f = 0;
      for (int k = 0; k < WPB; ++k) {
        const uint32_t p = blockIdx.x * WPB + k;
        if (p == 0 || __ldcg(P.segpos + p) != __ldcg(P.segpos + p - 1)) {
          m = NONE64;  // a segment starts here
          f = 1;
        }
        m = min(m, ldcg64(P.cand + p));
      }
      P.chunkmin[blockIdx.x] = m;
      P.chunkflag[blockIdx.x] = f;
    }
    grid.sync();

    // ---------------- phase C: exclusive segmented prefix-min at my position, commit
    {  // every block scans the chunk aggregates (nblocks <= 4 * THREADS) into s_pref
      SegMin v[4];
      SegMin t{NONE64, 0};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t b = threadIdx.x * 4 + k;
        v[k] = b < nblocks ? SegMin{ldcg64(P.chunkmin + b), __ldcg(P.chunkflag + b)}
                           : SegMin{NONE64, 0};
        t = SegOp()(t, v[k]);
      }
      SegMin run;
      SScan(s_scan).ExclusiveScan(t, run, SegMin{NONE64, 0}, SegOp());
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t b = threadIdx.x * 4 + k;
        if (b < nblocks) s_pref[b] = run.v;  // min over my segment's positions before chunk b
        run = SegOp()(run, v[k]);
      }
    }
    __syncthreads();
    if (j < P.ncols && !fin && ready && q < W) {
      const uint32_t chunk = q / WPB;
      uint64_t prefix = s_pref[chunk];
      for (uint32_t k = chunk * WPB; k <= q; ++k) {
        if (k == 0 || __ldcg(P.segpos + k) != __ldcg(P.segpos + k - 1)) prefix = NONE64;
        if (k < q) prefix = min(prefix, ldcg64(P.cand + k));
      }
      if (cval < prefix) {
        const uint32_t L = c.len();
        unsigned long long off = 0;
        if (lane == 0) off = atomicAdd(P.pool_top, (unsigned long long)L);
        off = __shfl_sync(0xFFFFFFFFu, off, 0);
        if (off + L > P.pool_cap) {
          if (lane == 0) atomicOr(P.err, 2);
        } else {
          // reduced column = M[h:] xor F[f0:], written straight into the pool
          const uint32_t n = merge_chunked<false>(c.M[c.mb] + c.h, c.nm - c.h, c.F[c.fb] + c.f0,
                                                  c.nf - c.f0, P.pool + off, c.F[c.fb ^ 1],
                                                  nullptr, lane);
          if (lane == 0) {
            P.pool_off[j] = off;
            P.pool_len[j] = n;
            __threadfence();
            P.owner[key_kidx(cval)] = j;
            const unsigned long long r = atomicAdd(P.nrec, 1ull);
            P.rec[r] = (uint64_t(key_kidx(P.cols[j])) << 32) | key_kidx(cval);
          }
          fin = true;
        }
      }
    }
    // next lo = min(first unfinished window column, lo + W)
    if (lane == 0 && j < P.ncols && !fin) atomicMin(P.lo_buf + ((round + 1) & 1), j);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      const uint64_t nl = uint64_t(lo) + W;
      atomicMin(P.lo_buf + ((round + 1) & 1), unsigned(nl < P.ncols ? nl : P.ncols));
      P.lo_buf[round & 1] = NONE32;
      atomicAdd(P.stats, 1ull);
    }
    grid.sync();
    lo = __ldcg(P.lo_buf + ((round + 1) & 1));
    if (lo >= P.ncols) break;
    if (__ldcg(P.err)) break;
  }
}

__global__ void k_collect_columns(const uint32_t* __restrict__ births,
                                  const uint8_t* __restrict__ tags, Geom g, int d,
                                  uint64_t* __restrict__ cols, unsigned* __restrict__ ncols) {
  int64_t kk = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  bool emit = false;
  uint64_t key = 0;
  if (kk < g.ncells) {
    uint32_t k = uint32_t(kk);
    uint32_t KX = uint32_t(g.KX), KY = uint32_t(g.KY);
    uint32_t X = k % KX, r = k / KX, Y = r % KY, Z = r / KY;
    int dim = (X & 1) + (Y & 1) + (Z & 1);
    uint32_t b = births[k];
    if (dim == d && b != ABSENT_ORD && tag_kind(tags[k]) == KIND_RESIDUAL) {
      emit = true;
      key = make_key(b, k);
    }
  }
  unsigned mask = __ballot_sync(0xFFFFFFFFu, emit);
  if (!mask) return;
  int lane = threadIdx.x & 31;
  unsigned base = 0;
  if (lane == __ffs(mask) - 1) base = atomicAdd(ncols, __popc(mask));
  base = __shfl_sync(0xFFFFFFFFu, base, __ffs(mask) - 1);
  if (emit) cols[base + __popc(mask & ((1u << lane) - 1))] = key;
}

__global__ void k_seg_keys(const uint64_t* __restrict__ cols, unsigned n, uint32_t seg_cells,
                           uint32_t* __restrict__ segk) {
  unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) segk[i] = key_kidx(cols[i]) / seg_cells;
}

__global__ void k_mark_cleared(const uint64_t* __restrict__ rec, int64_t n, uint8_t* tags) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t dk = uint32_t(rec[i]);
  if (dk != NONE32) tags[dk] = make_tag(KIND_CLEARED, 0);
}

}  // namespace

void reduce_dimension(GeneralState& S, int d, Workspace& ws, HostScalars& hs, cr_stats& st) {
  cudaStream_t s = ws.stream();
  const Geom& g = S.g;
  const int B = 256;
  const int64_t nd = st.cells[d];
  S.R.rec[d] = ws.alloc<uint64_t>(nd);
  S.R.n[d] = 0;
  if (nd == 0) return;

  unsigned long long* ctr = ws.alloc<unsigned long long>(16);
  CR_CUDA(cudaMemsetAsync(ctr, 0, 16 * sizeof(unsigned long long), s));
  uint64_t* cols = ws.alloc<uint64_t>(nd);
  k_collect_columns<<<grid_for(g.ncells, B), B, 0, s>>>(S.births, S.tags, g, d, cols,
                                                        reinterpret_cast<unsigned*>(ctr));
  CR_CHECK_LAUNCH();
  const unsigned ncols = read_scalar(reinterpret_cast<unsigned*>(ctr), s, hs);
  st.columns[d] = ncols;
  if (ncols > 0) {
    sort_keys_u64(cols, ncols, /*descending=*/true, 64, ws);
    if (S.seg_cells) {
      // batched images: group the columns by image (stable, so each image keeps its decreasing
      // key order); images are independent complexes, so their relative order is immaterial
      uint32_t* segk = ws.alloc<uint32_t>(ncols);
      uint32_t* segk2 = ws.alloc<uint32_t>(ncols);
      uint64_t* cols2 = ws.alloc<uint64_t>(ncols);
      k_seg_keys<<<grid_for(ncols, B), B, 0, s>>>(cols, ncols, S.seg_cells, segk);
      CR_CHECK_LAUNCH();
      cub::DoubleBuffer<uint32_t> dk(segk, segk2);
      cub::DoubleBuffer<uint64_t> dv(cols, cols2);
      size_t tmp = 0;
      CR_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, dk, dv, int(ncols), 0, 32, s));
      void* t = ws.alloc_bytes(tmp);
      CR_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, dk, dv, int(ncols), 0, 32, s));
      if (dv.Current() != cols)
        CR_CUDA(cudaMemcpyAsync(cols, dv.Current(), ncols * sizeof(uint64_t),
                                cudaMemcpyDeviceToDevice, s));
    }

    int dev = 0, nsm = 0, per_sm = 0;
    CR_CUDA(cudaGetDevice(&dev));
    CR_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    CR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_reduce, THREADS, 0));
    if (per_sm < 1) throw Error{CR_EINTERNAL, "k_reduce cannot be resident"};
    per_sm = per_sm > 4 ? 4 : per_sm;
    int64_t blocks = int64_t(nsm) * per_sm;
    const int64_t need_blocks = (int64_t(ncols) + WPB - 1) / WPB;  // small problems
    if (need_blocks < blocks) blocks = need_blocks;
    if (blocks > int64_t(THREADS) * 4) blocks = THREADS * 4;
    const uint32_t W = uint32_t(blocks * WPB);

    uint32_t* owner = ws.alloc<uint32_t>(g.ncells);
    unsigned long long* pool_off = ws.alloc<unsigned long long>(ncols);
    uint32_t* pool_len = ws.alloc<uint32_t>(ncols);
    uint64_t* cand = ws.alloc<uint64_t>(W + blocks);
    uint64_t* chunkmin = ws.alloc<uint64_t>(blocks);
    uint32_t* chunkflag = ws.alloc<uint32_t>(blocks);
    uint32_t* segpos = ws.alloc<uint32_t>(W);
    unsigned* lo_buf = reinterpret_cast<unsigned*>(ctr + 2);
    int* err = reinterpret_cast<int*>(ctr + 3);
    unsigned long long* nrec = ctr + 4;
    unsigned long long* pool_top = ctr + 5;
    unsigned long long* stats = ctr + 6;  // [6] rounds [7] additions [8] lengths [9] max length

    uint32_t mcap = 4096;
    unsigned long long pool_cap = std::max<unsigned long long>(8ull * ncols + 4096, 1ull << 20);
    uint64_t* work = nullptr;
    uint64_t* pool = nullptr;
    unsigned long long* P_colstat = nullptr;
    for (int attempt = 0;; ++attempt) {
      if (!work) work = ws.alloc<uint64_t>(int64_t(W) * 2 * mcap);
      if (!pool) pool = ws.alloc<uint64_t>(int64_t(pool_cap));
      CR_CUDA(cudaMemsetAsync(owner, 0xFF, g.ncells * sizeof(uint32_t), s));
      CR_CUDA(cudaMemsetAsync(lo_buf, 0xFF, 2 * sizeof(unsigned), s));
      CR_CUDA(cudaMemsetAsync(err, 0, sizeof(int), s));
      CR_CUDA(cudaMemsetAsync(nrec, 0, 6 * sizeof(unsigned long long), s));
      RP P;
      P.g = g;
      P.d = d;
      P.cols = cols;
      P.ncols = ncols;
      P.births = S.births;
      P.tags = S.tags;
      P.owner = owner;
      P.pool = pool;
      P.pool_top = pool_top;
      P.pool_cap = pool_cap;
      P.pool_off = pool_off;
      P.pool_len = pool_len;
      P.work = work;
      P.mcap = mcap;
      P.cand = cand;
      P.chunkmin = chunkmin;
      P.chunkflag = chunkflag;
      P.segpos = segpos;
      P.seg_cells = S.seg_cells;
      P.lo_buf = lo_buf;
      P.rec = S.R.rec[d];
      P.nrec = nrec;
      P.err = err;
      P.max_steps = 256;
      P.stats = stats;
      P.debug = std::getenv("CR_DEBUG_STATS") != nullptr;
      {
        const int dbg = P.debug ? 1 : 0;
        unsigned long long z[4] = {0, 0, 0, 0};
        CR_CUDA(cudaMemcpyToSymbolAsync(g_k5_dbg, &dbg, sizeof(int), 0, cudaMemcpyHostToDevice, s));
        CR_CUDA(cudaMemcpyToSymbolAsync(g_k5_flush, z, sizeof(z), 0, cudaMemcpyHostToDevice, s));
      }
      P.colstat = nullptr;
      P.prefetch = std::getenv("CR_K5_PREFETCH") != nullptr;
      P.lcache = std::getenv("CR_K5_CACHE") != nullptr;
      if (P.debug) {
        if (!P_colstat) P_colstat = ws.alloc<unsigned long long>(2 * int64_t(ncols));
        P.colstat = P_colstat;
        CR_CUDA(cudaMemsetAsync(P.colstat, 0, 2 * sizeof(unsigned long long) * ncols, s));
      }
      void* args[] = {&P};
      CR_CUDA(cudaLaunchCooperativeKernel((void*)k_reduce, dim3(unsigned(blocks)), dim3(THREADS),
                                          args, 0, s));
      ++g_launch_count;
      const int e = read_scalar(err, s, hs);
      if (e == 0) break;
      if (attempt > 12) throw Error{CR_ENOMEM, "reduction buffers exhausted"};
      if (e & 1) {
        ws.release(work);
        work = nullptr;
        mcap *= 4;
      }
      if (e & 2) {
        ws.release(pool);
        pool = nullptr;
        pool_cap *= 4;
      }
    }
    CR_CUDA(cudaMemcpyAsync(hs.p, ctr, 16 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    CR_CUDA(cudaStreamSynchronize(s));
    S.R.n[d] = int64_t(hs.p[4]);
    st.rounds[d] = int64_t(hs.p[6]);
    st.additions[d] = int64_t(hs.p[7]);
    st.addlen[d] = int64_t(hs.p[8]);
    st.maxlen[d] = int64_t(hs.p[9]);
    if (std::getenv("CR_DEBUG_STATS")) {
      std::vector<unsigned long long> cs(2 * size_t(ncols));
      CR_CUDA(cudaMemcpy(cs.data(), P_colstat, cs.size() * 8, cudaMemcpyDeviceToHost));
      std::vector<std::pair<unsigned long long, uint32_t>> byent(ncols);
      unsigned long long tot = 0;
      for (uint32_t j = 0; j < ncols; ++j) {
        byent[j] = {cs[2 * j + 1], j};
        tot += cs[2 * j + 1];
      }
      std::sort(byent.rbegin(), byent.rend());
      unsigned long long acc = 0;
      const uint32_t marks[5] = {1, 10, 100, 1000, 10000};
      fprintf(stderr, "[cr] dim %d entry work: total %llu;", d, tot);
      for (uint32_t m : marks) {
        if (m > ncols) break;
        acc = 0;
        for (uint32_t q = 0; q < m; ++q) acc += byent[q].first;
        fprintf(stderr, " top%u %.3f", m, tot ? double(acc) / tot : 0.0);
      }
      unsigned long long fl[4];
      CR_CUDA(cudaMemcpyFromSymbol(fl, g_k5_flush, sizeof(fl)));
      fprintf(stderr, " | flushes %llu cycles %llu M-entries %llu", fl[0], fl[1], fl[2]);
      fprintf(stderr, "\n[cr] top columns (pos, adds, entries):");
      for (int q = 0; q < 8 && q < int(ncols); ++q)
        fprintf(stderr, " (%u,%llu,%llu)", byent[q].second, cs[2 * byent[q].second],
                byent[q].first);
      fprintf(stderr, "\n");
      fprintf(stderr,
              "[cr] dim %d: cols %u rounds %llu adds %llu pool_adds %llu pool_len %llu "
              "cyc_pool %llu cyc_app %llu cyc_lookup %llu W %u\n",
              d, ncols, hs.p[6], hs.p[7], hs.p[10], hs.p[11], hs.p[13], hs.p[14], hs.p[15], W);
    }
    ws.release(work);
    ws.release(pool);
    ws.release(owner);
    ws.release(pool_off);
    ws.release(pool_len);
  }
  if (S.R.n[d] > 0) {
    k_mark_cleared<<<grid_for(S.R.n[d], B), B, 0, s>>>(S.R.rec[d], S.R.n[d], S.tags);
    CR_CHECK_LAUNCH();
  }
  ws.release(cols);
}

}  // namespace cr
