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
#ifndef K5_FCAP
#define K5_FCAP 256
#endif
constexpr uint32_t FCAP = K5_FCAP;  // fresh-array capacity per warp (shared memory, x2 ping-pong)

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
  int d;
  int hom;             // 1: homology mode (columns = (d+1)-cells by boundary, keys complemented)
  const uint64_t* cols;
  uint32_t ncols;
  const uint32_t* births;
  const uint8_t* tags;
  uint64_t* owninfo;   // per (d+1)-cell: (pool offset << 24) | length of the column owning it as
                       // pivot, NONE64 if unowned -- one load instead of owner -> offset, length
  uint64_t* pool;
  unsigned long long* pool_top;
  unsigned long long pool_cap;
  uint64_t* work;      // per warp: 2 * mcap main-array entries
  uint32_t mcap;
  uint64_t* cand;      // per window position
  uint64_t* chunkmin;  // per block (positions [WPB*b, WPB*b+WPB))
  uint32_t* chunkflag; // per block: a segment starts inside the chunk
  uint32_t* segpos;    // per window position: its warp group (positions of a group are contiguous)
  uint32_t seg_cells;  // cells per segment (batched images), 0: one segment
  const uint32_t* seg_off;  // nseg + 1 column offsets (columns are grouped by segment)
  uint32_t nseg;
  uint32_t G;          // warps per group; group g reduces segments g, g + ngroups, ...
  uint32_t ngroups;
  unsigned* lo_buf;    // [2 * ngroups]: next window start of each group (double-buffered)
  unsigned* done_buf;  // [2]: groups with no segment left (double-buffered)
  uint64_t* rec;
  unsigned long long* nrec;
  int* err;
  int ahead;           // read-ahead of the next column (see phase A)
  int max_steps;       // additions per warp and round, at most ...
  long long budget;    // ... and until this many cycles of the round have passed (0: no limit)
  unsigned long long* stats;  // [0] rounds [1] additions [2] sum of lengths [3] max length
                              // debug: [4] pool additions [5] pool lengths [7]/[8] cycles in
                              // pool/apparent additions [9] cycles in pivot + owner lookups
  int debug;
  unsigned long long* rdbg;  // debug: per round [max phase-A cycles, max steps, active warps, t]
  uint32_t rdbg_cap;
  unsigned long long* colstat;  // debug: per column (additions, entries touched, cycles in
                                // lookups, apparent adds, pool adds, flushes)
};
constexpr int OI_LEN_BITS = 24;  // owninfo: stored column length field

__device__ __forceinline__ uint64_t ldcg64(const uint64_t* p) {
  return __ldcg((const unsigned long long*)p);
}
template <bool G>
__device__ __forceinline__ uint64_t ld64(const uint64_t* p) {
  return G ? ldcg64(p) : *p;
}

// Keys of the working columns.  Cohomology: (ord << 32 | kidx), pivot = min.  Homology mode: the
// complement ~(ord << 32 | kidx), so that the min-pivot machinery below takes the MAX (latest)
// face as the pivot and processes columns in increasing filtration order (decreasing ~key).
__device__ __forceinline__ uint64_t rkey(const RP& P, uint32_t b, uint32_t k) {
  const uint64_t x = make_key(b, k);
  return P.hom ? ~x : x;
}
__device__ __forceinline__ uint32_t rkid(const RP& P, uint64_t key) {
  return P.hom ? ~uint32_t(key) : uint32_t(key);
}

// The column of cell s, sorted ascending (by rkey), written to dst (<= 6 entries): its finite
// cofacets (cohomology), or its facets (homology mode).  Warp-collective.
__device__ uint32_t coboundary(const RP& P, uint32_t s, uint64_t* dst, int lane) {
  const Geom& g = P.g;
  const uint32_t KX = uint32_t(g.KX), KY = uint32_t(g.KY);
  const uint32_t r = P.fx.div(s), z = P.fxy.div(s);
  const uint32_t c[3] = {s - r * KX, r - z * KY, z};
  const uint32_t ext[3] = {KX, KY, uint32_t(g.KZ)};
  uint64_t key = NONE64;
  if (lane < 6) {
    const int a = lane >> 1, sg = lane & 1;
    if ((P.hom ? (c[a] & 1) : !(c[a] & 1)) && (sg ? c[a] + 1 < ext[a] : c[a] > 0)) {
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
  uint64_t mwin;   // per lane: M[mb][wb + lane] (valid unless mstale), NONE64 past the end
  uint32_t wb;     // window base
  bool mstale;
  long long fcyc;  // debug: cycles spent in flushes
  uint32_t cap;    // capacity of M[0] and M[1]
  uint64_t* spare; // the second half of a grown pair, installed after the merge that grew it
  uint64_t rv;     // per lane: entry `lane` of the register list R (NONE64 at and past nr)
  uint32_t nr, r0; // R holds positions [r0, nr) (consumed from the front)
  __device__ uint32_t len() const { return (nm - h) + (nf - f0) + (nr - r0); }
};

// The working column is M[h:] xor F[f0:] xor R[r0:nr]: three sorted tiers -- a long main array in
// global memory, a fresh array in shared memory, and a register list of <= 32 entries (one per
// lane) that takes the small addends (apparent coboundaries, short stored columns) at a cost of a
// few shuffles instead of rewriting F.  Equal values in different tiers cancel lazily, when they
// reach the heads.
//
// pivot = min of the three heads, cancelling equal pairs; NONE64 if the column is zero.
// Warp-collective.  The next 32 entries of M sit in a register window (one per lane), reloaded
// with one coalesced load when h leaves it or M changes: the head of a long column is not a
// dependent global load per cancellation.
__device__ __forceinline__ uint64_t take_pivot(Col& c, int lane) {
  while (true) {
    if (c.mstale || c.h >= c.wb + 32) {
      c.wb = c.h;
      c.mwin = c.h + lane < c.nm ? ldcg64(c.M[c.mb] + c.h + lane) : NONE64;
      c.mstale = false;
    }
    const uint64_t a = __shfl_sync(0xFFFFFFFFu, c.mwin, c.h - c.wb);
    const uint64_t b = c.f0 < c.nf ? c.F[c.fb][c.f0] : NONE64;
    const uint64_t rr = __shfl_sync(0xFFFFFFFFu, c.rv, c.r0 & 31);
    const uint64_t r = c.r0 < c.nr ? rr : NONE64;
    if (a == b && a != NONE64) {
      ++c.h;
      ++c.f0;
    } else if (a == r && a != NONE64) {
      ++c.h;
      ++c.r0;
    } else if (b == r && b != NONE64) {
      ++c.f0;
      ++c.r0;
    } else {
      const uint64_t m = a < b ? a : b;
      return m < r ? m : r;
    }
  }
}

// R <- R[r0:nr] xor B for a sorted B of nb <= SMALLB entries in shared memory, with
// (nr - r0) + nb <= 32.  Lane k < nb places B[k] by a shuffle binary search over R; every lane
// holds all of B in registers to place its own R entry; the new list goes through `scratch`
// (>= 40 entries).  Warp-collective.
__device__ __forceinline__ void r_insert(Col& c, const uint64_t* B, uint32_t nb, uint64_t* scratch,
                                         int lane) {
  const uint32_t live = c.nr - c.r0;
  const uint64_t y = lane < int(nb) ? B[lane] : NONE64;
  uint32_t lo = c.r0, hi = c.nr;
#pragma unroll
  for (int it = 0; it < 6; ++it) {  // positions [r0, nr] <= 33 values: 6 halvings
    const uint32_t mid = (lo + hi) >> 1;
    const uint64_t v = __shfl_sync(0xFFFFFFFFu, c.rv, mid & 31);
    if (lo < hi) {
      if (v < y) lo = mid + 1;
      else hi = mid;
    }
  }
  const uint64_t at = __shfl_sync(0xFFFFFFFFu, c.rv, lo & 31);
  const bool ydup = lane < int(nb) && lo < c.nr && at == y;
  const uint32_t bdup = __ballot_sync(0xFFFFFFFFu, ydup);
  uint64_t bv[SMALLB];
#pragma unroll
  for (int k = 0; k < int(SMALLB); ++k) bv[k] = __shfl_sync(0xFFFFFFFFu, y, k);
  const uint64_t x = c.rv;
  uint32_t lessB = 0, D = 0;
  bool dup = false;
#pragma unroll
  for (int k = 0; k < int(SMALLB); ++k) {
    const bool lt = bv[k] < x;
    lessB += lt ? 1u : 0u;
    D += (lt && (bdup >> k & 1)) ? 1u : 0u;
    dup |= bv[k] == x;
  }
  if (uint32_t(lane) >= c.r0 && uint32_t(lane) < c.nr && !dup)
    scratch[(lane - c.r0) + lessB - 2 * D] = x;
  if (lane < int(nb) && !ydup) scratch[lane + (lo - c.r0) - 2 * __popc(bdup & ((1u << lane) - 1))] = y;
  __syncwarp();
  const uint32_t n = live + nb - 2 * __popc(bdup);
  c.rv = uint32_t(lane) < n ? scratch[lane] : NONE64;
  c.nr = n;
  c.r0 = 0;
  __syncwarp();
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
  bool need_b_even;  // (homology mode: axis b must be odd in the pivot)
  uint32_t off;      // cell - t (two's complement)
  bool active;
  bool hom;
};
// Homology mode mirrors it: an UP pivot e (a d-cell) is the lower cell of an apparent pair
// (e, s') with s' = e + e_dir a cofacet; the column adds del(s') = {e} + the other facets of s':
// member 0 is e + 2 e_dir, members 1-4 are s' -/+ e_b for the other axes b odd in e.
__device__ __forceinline__ SpecLane spec_lane(const Geom& g, int lane, bool hom) {
  SpecLane L{0, 0, 0, 0, false, 0u, false, hom};
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
  const bool up_axis = L.hom ? !(ca & 1) : (ca & 1);  // t on the pivot side of axis a
  const bool b_bad = L.need_b_even && (L.hom ? !(cc & 1) : (cc & 1));
  // homology: t is even along a and may sit on the border; the partner t + sa e_a must exist
  const uint32_t ea = L.a == 0 ? KX : (L.a == 1 ? KY : uint32_t(P.g.KZ));
  const bool a_ok = !L.hom || ca + uint32_t(L.sa) < ea;
  if (L.active && up_axis && a_ok && moved < ec && !b_bad) {
    r.cell = t + L.off;
    r.birth = __ldg(P.births + r.cell);
  }
  return r;
}
// delta(s') sorted ascending into dst (<= 6 entries) for the partner direction dir; warp-collective.
__device__ __forceinline__ uint32_t spec_finish(const RP& P, const Spec& sp, int dir, uint64_t piv,
                                                uint64_t* dst, int lane) {
  uint64_t key = NONE64;
  if (lane < 30 && lane / 5 == dir && sp.birth != ABSENT_ORD) key = rkey(P, sp.birth, sp.cell);
  if (lane == 31) key = piv;
  const unsigned vm = __ballot_sync(0xFFFFFFFFu, key != NONE64);
  int rank = 0;
  for (unsigned m = vm; m; m &= m - 1) rank += __shfl_sync(0xFFFFFFFFu, key, __ffs(m) - 1) < key;
  if (key != NONE64) dst[rank] = key;
  __syncwarp();
  return __popc(vm);
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
  constexpr int G = R;          // all of a lane's searches run interleaved
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
  // ---- 3. stream A in windows of 256, software-pipelined (the next window's loads are in flight
  // while this one is placed).  The F entries landing in a window, [tl, th), are walked once per
  // window (broadcast shared reads) against all 8 of a lane's entries at once.
  uint64_t nv[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const uint32_t i = lane + 32 * k;
    nv[k] = i < a ? ldcg64(A + i) : 0ull;
  }
  uint32_t tl = 0;
  for (uint32_t w0 = 0; w0 < a; w0 += 256) {
    uint64_t v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      v[k] = nv[k];
      const uint32_t i = w0 + 256 + lane + 32 * k;
      nv[k] = i < a ? ldcg64(A + i) : 0ull;
    }
    uint32_t th = tl;
    while (th < b && XP[th] < w0 + 256) ++th;
    const uint32_t cl = tl < b ? XC[tl] & 0x7FFFFFFFu : ((totD << 16) | totI);
    uint32_t ins[8], rem[8];
    uint32_t removed = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      ins[k] = cl & 0xFFFFu;
      rem[k] = cl >> 16;
    }
    for (uint32_t t = tl; t < th; ++t) {
      const uint32_t pt = XP[t];
      const bool dup = XC[t] >> 31;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t i = w0 + lane + 32 * k;
        ins[k] += (!dup && pt <= i) ? 1u : 0u;
        rem[k] += (dup && pt < i) ? 1u : 0u;
        removed |= (dup && pt == i) ? (1u << k) : 0u;
      }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t i = w0 + lane + 32 * k;
      if (i < a && !(removed >> k & 1)) C[i + ins[k] - rem[k]] = v[k];
    }
    tl = th;
  }
  __syncwarp();
  return a + totI - totD;
}

__device__ int g_k5_dbg = 0;                      // CR_DEBUG_STATS: flush counters below
__device__ unsigned long long g_k5_flush[4];      // flushes, cycles, entries of M, long merges

// Make room for a merge of `need` entries into M[mb ^ 1]: a column that outgrows its warp's slot
// moves to a larger pair carved from the pool (bump allocation; the few long columns of a launch
// leave their old pairs behind).  False (err 2: the caller retries with a larger pool) if the
// pool is exhausted.
__device__ bool grow(Col& c, uint32_t need, const RP& P, int lane) {
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
  c.M[c.mb ^ 1] = P.pool + off;  // the merge's destination
  c.spare = P.pool + off + ncap;  // replaces the old M[mb] once the merge has read it
  c.cap = uint32_t(ncap);
  return true;
}
__device__ __forceinline__ void swap_main(Col& c) {
  c.mb ^= 1;
  if (c.spare) {
    c.M[c.mb ^ 1] = c.spare;
    c.spare = nullptr;
  }
}

// M <- M[h:] xor F[f0:]   (returns false on capacity overflow)
__device__ bool flush(Col& c, const RP& P, int lane) {
  const uint32_t na = c.nm - c.h, nb = c.nf - c.f0;
  if (nb == 0) return true;
  if (!grow(c, na + nb, P, lane)) return false;
  const long long t0 = g_k5_dbg ? clock64() : 0;
  const uint32_t n = merge_long_short(c.M[c.mb] + c.h, na, c.F[c.fb] + c.f0, nb,
                                      c.M[c.mb ^ 1], c.F[c.fb ^ 1], lane);
  if (g_k5_dbg && lane == 0) {
    atomicAdd(g_k5_flush + 0, 1ull);
    atomicAdd(g_k5_flush + 1, (unsigned long long)(clock64() - t0));
    c.fcyc += clock64() - t0;
    atomicAdd(g_k5_flush + 2, (unsigned long long)na);
  }
  swap_main(c);
  c.nm = n;
  c.h = 0;
  c.nf = c.f0 = 0;
  c.mstale = true;
  return true;
}

constexpr uint32_t STAGE = 64;  // short global addends are staged in shared memory first

// F <- F xor R, R emptied (flushing F into M first if it cannot take R).  Warp-collective.
__device__ bool spill_r(Col& c, const RP& P, uint64_t* scratch, int lane) {
  const uint32_t live = c.nr - c.r0;
  if (live > 0) {
    if ((c.nf - c.f0) + live > FCAP && !flush(c, P, lane)) return false;
    if (uint32_t(lane) >= c.r0 && uint32_t(lane) < c.nr) scratch[lane - c.r0] = c.rv;
    __syncwarp();
    if (c.nf == c.f0) {
      if (uint32_t(lane) < live) c.F[c.fb][lane] = scratch[lane];
      c.nf = live;
    } else {
      c.nf = merge_symdiff<false, false>(c.F[c.fb] + c.f0, c.nf - c.f0, scratch, live,
                                         c.F[c.fb ^ 1], lane);
      c.fb ^= 1;
    }
    c.f0 = 0;
    __syncwarp();
  }
  c.rv = NONE64;
  c.nr = c.r0 = 0;
  return true;
}

// column += B (sorted; BG: B in global memory).  Returns false on capacity overflow.
template <bool BG>
__device__ bool add_column(Col& c, const uint64_t* B, uint32_t nb, const RP& P, int lane,
                           uint64_t* stage, uint64_t* small) {
  if (nb <= SMALLB) {  // into the register list
    if (BG) {
      if (uint32_t(lane) < nb) small[lane] = ldcg64(B + lane);
      __syncwarp();
      B = small;
    }
    if ((c.nr - c.r0) + nb > 32 && !spill_r(c, P, stage, lane)) return false;
    r_insert(c, B, nb, stage, lane);
    return true;
  }
  if (BG && nb <= STAGE && (c.nf - c.f0) + nb <= FCAP) {
    // one coalesced load instead of a dependent global binary search per F entry
    for (uint32_t i = lane; i < nb; i += 32) stage[i] = ldcg64(B + i);
    __syncwarp();
    const uint32_t n =
        nb <= SMALLB
            ? merge_small(c.F[c.fb] + c.f0, c.nf - c.f0, stage, nb, c.F[c.fb ^ 1], lane)
            : merge_symdiff<false, false>(c.F[c.fb] + c.f0, c.nf - c.f0, stage, nb,
                                          c.F[c.fb ^ 1], lane);
    c.fb ^= 1;
    c.nf = n;
    c.f0 = 0;
    return true;
  }
  if (!BG && nb <= SMALLB && (c.nf - c.f0) + nb <= FCAP) {
    const uint32_t n = merge_small(c.F[c.fb] + c.f0, c.nf - c.f0, B, nb, c.F[c.fb ^ 1], lane);
    c.fb ^= 1;
    c.nf = n;
    c.f0 = 0;
    return true;
  }
  if ((c.nf - c.f0) + nb <= FCAP) {
    const uint32_t n =
        merge_symdiff<false, BG>(c.F[c.fb] + c.f0, c.nf - c.f0, B, nb, c.F[c.fb ^ 1], lane);
    c.fb ^= 1;
    c.nf = n;
    c.f0 = 0;
    return true;
  }
  if (!flush(c, P, lane)) return false;
  if (nb <= FCAP) {  // F is empty now: B becomes F
    for (uint32_t i = lane; i < nb; i += 32) c.F[c.fb][i] = ld64<BG>(B + i);
    __syncwarp();
    c.nf = nb;
    c.f0 = 0;
    return true;
  }
  if (!grow(c, (c.nm - c.h) + nb, P, lane)) return false;
  const uint32_t n = merge_chunked<BG>(c.M[c.mb] + c.h, c.nm - c.h, B, nb, c.M[c.mb ^ 1],
                                       c.F[0], c.F[1], lane);
  swap_main(c);
  c.nm = n;
  c.h = 0;
  c.mstale = true;
  return true;
}

#ifndef K5_MINB
#define K5_MINB 4
#endif
__global__ void __launch_bounds__(THREADS, K5_MINB) k_reduce(RP P) {
  cg::grid_group grid = cg::this_grid();
  __shared__ uint64_t s_F[WPB][2][FCAP];
  __shared__ uint64_t s_small[WPB][8];
  // phase A stages short addends, phase C scans chunk minima: grid syncs separate them
  __shared__ union {
    uint64_t stage[WPB][STAGE];
    uint64_t pref[4 * THREADS];
  } s_u;
  static_assert(sizeof(uint64_t) * WPB * STAGE <= sizeof(uint64_t) * 4 * THREADS, "alias");
  auto& s_stage = s_u.stage;
  auto& s_pref = s_u.pref;
  __shared__ typename SScan::TempStorage s_scan;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const uint32_t W = (gridDim.x * blockDim.x) >> 5;
  const uint32_t w = blockIdx.x * WPB + wib;
  const uint32_t nblocks = gridDim.x;

  Col c;
  uint64_t* const slot = P.work + uint64_t(w) * 2 * P.mcap;
  const SpecLane sl = spec_lane(P.g, lane, P.hom != 0);
  c.F[0] = s_F[wib][0];
  c.F[1] = s_F[wib][1];
  // Warp groups: group grp (G warps, window positions [grp*G, grp*G + G)) reduces the segments
  // grp, grp + ngroups, ... one after the other; segments (images of a batch) are independent
  // complexes, so each has its own window and the groups progress concurrently.  One image:
  // one group of all W warps.  Warps beyond ngroups * G stay idle.
  const uint32_t G = P.G, grp = w / G, k = w - grp * G;
  uint32_t seg = grp < P.ngroups ? grp : P.nseg;
  uint32_t lo = seg < P.nseg ? __ldg(P.seg_off + seg) : P.ncols;
  uint32_t end = seg < P.nseg ? __ldg(P.seg_off + seg + 1) : P.ncols;
  uint32_t j = lo + k;
  bool started = false, fin = false;
  if (lane == 0) {
    P.segpos[w] = grp < P.ngroups ? grp : 0xFFFFFFFFu;  // idle positions: a segment of their own
    P.cand[w] = NONE64;
  }

  for (uint32_t round = 0;; ++round) {
    // ---------------- phase A: advance my column
    // Read-ahead: a warp whose column is finished takes its next column j + G at once, even if
    // the window has not reached it yet: it reduces it with the owners committed so far (always
    // valid) and only publishes / commits once the column is inside the window.
    if (fin && (j < lo || P.ahead)) {
      j += G;
      started = false;
      fin = false;
    }
    uint64_t cval = NONE64;
    bool ready = false;
    const long long pa0 = P.rdbg ? clock64() : 0;
    int dbg_steps = -1;
    if (j < end && !fin) {
      if (!started) {
        started = true;
        c.mb = c.fb = 0;
        c.h = c.f0 = c.nm = 0;
        c.M[0] = slot;  // a column grown into the pool last time starts over in the slot
        c.M[1] = slot + P.mcap;
        c.cap = P.mcap;
        c.spare = nullptr;
        c.rv = NONE64;
        c.nr = c.r0 = 0;
        c.mstale = true;
        c.nf = coboundary(P, rkid(P, P.cols[j]), c.F[0], lane);
      }
      int steps = 0;
      const long long round_t0 = clock64();
      unsigned long long adds = 0, addlen = 0, cl = 0, ca = 0, cp = 0;
      c.fcyc = 0;
      bool ok = true;
      while (true) {
        const long long tl0 = P.debug ? clock64() : 0;
        const uint64_t piv = take_pivot(c, lane);
        if (piv == NONE64) break;
        const uint32_t pk = rkid(P, piv);
        // independent loads: the speculated partner coboundary, the tag, the owner record
        const Spec sp = spec_issue(P, sl, pk);
        const uint8_t t = __ldg(P.tags + pk);
        const uint64_t oi = ldcg64(P.owninfo + pk);
        const uint64_t* add;
        uint32_t alen;
        bool glob;
        if (tag_kind(t) == (P.hom ? KIND_UP : KIND_DOWN)) {
          // the pivot is the upper cell of an apparent pair (s', pivot): add delta(s')
          // (homology: the lower cell of (pivot, s'): add del(s'))
          alen = spec_finish(P, sp, tag_dir(t), piv, s_small[wib], lane);
          add = s_small[wib];
          glob = false;
        } else {
          if (oi == NONE64) {
            // ready to commit: fold R into F now (phase C's commit reads M and F, and its shared
            // scratch is busy there)
            ok = spill_r(c, P, s_stage[wib], lane);
            ready = ok;
            cval = piv;
            break;
          }
          add = P.pool + (oi >> OI_LEN_BITS);
          alen = uint32_t(oi & ((1u << OI_LEN_BITS) - 1));
          glob = true;
        }
        if (steps >= P.max_steps || (P.budget && clock64() - round_t0 > P.budget)) {
          cval = piv;
          break;
        }
        addlen += c.len() + alen;
        const long long t0 = P.debug ? clock64() : 0;
        if (P.debug && lane == 0) atomicAdd(P.stats + 9, (unsigned long long)(t0 - tl0));
        cl += t0 - tl0;
        ok = glob ? add_column<true>(c, add, alen, P, lane, s_stage[wib], s_small[wib])
                  : add_column<false>(c, add, alen, P, lane, s_stage[wib], s_small[wib]);
        if (P.debug && lane == 0) {
          const unsigned long long dt = (unsigned long long)(clock64() - t0);
          if (glob) {
            atomicAdd(P.stats + 4, 1ull);
            atomicAdd(P.stats + 5, (unsigned long long)alen);
            atomicAdd(P.stats + 7, dt);
            cp += dt;
          } else {
            atomicAdd(P.stats + 8, dt);
            ca += dt;
          }
        }
        if (!ok) break;  // pool exhausted (err 2 set): the launch is retried
        ++steps;
        ++adds;
      }
      dbg_steps = steps;
      if (lane == 0 && adds) {
        atomicAdd(P.stats + 1, adds);
        atomicAdd(P.stats + 2, addlen);
        atomicMax(P.stats + 3, (unsigned long long)c.len());
        if (P.colstat) {
          P.colstat[6 * j] += adds;
          P.colstat[6 * j + 1] += addlen;
          P.colstat[6 * j + 2] += cl;
          P.colstat[6 * j + 3] += ca;
          P.colstat[6 * j + 4] += cp;
          P.colstat[6 * j + 5] += (unsigned long long)c.fcyc;
        }
      }
      if (ok && !ready && cval == NONE64) {  // zero column: essential (exact given clearing)
        fin = true;
        if (lane == 0) {
          if (P.hom) {
            atomicOr(P.err, 8);  // homology: every column left after the clearing is nonzero
          } else {
            const unsigned long long r = atomicAdd(P.nrec, 1ull);
            P.rec[r] = (uint64_t(rkid(P, P.cols[j])) << 32) | NONE32;
          }
        }
      }
    }
    if (P.rdbg && lane == 0 && round < P.rdbg_cap && dbg_steps >= 0) {
      unsigned long long* R = P.rdbg + 4ull * round;
      atomicMax(R + 0, (unsigned long long)(clock64() - pa0));
      atomicMax(R + 1, (unsigned long long)dbg_steps);
      atomicAdd(R + 2, 1ull);
    }
    if (P.rdbg && blockIdx.x == 0 && threadIdx.x == 0 && round < P.rdbg_cap) {
      unsigned long long tnow;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow));
      P.rdbg[4ull * round + 3] = tnow;
    }
    // publish at my window position (every position of a group's window is owned by exactly one
    // of its warps); a column is blocked only by unfinished earlier columns of its own window
    const uint32_t q = j - lo;
    const uint32_t qg = grp * G + q;
    if (lane == 0 && grp < P.ngroups && q < G) P.cand[qg] = (j < end && !fin) ? cval : NONE64;
    // a read-ahead warp still owns its finished previous column's position
    if (lane == 0 && grp < P.ngroups && q >= G && q - G < G) P.cand[qg - G] = NONE64;
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
    if (j < end && !fin && ready && q < G) {
      const uint32_t chunk = qg / WPB;
      uint64_t prefix = s_pref[chunk];
      for (uint32_t kk = chunk * WPB; kk <= qg; ++kk) {
        if (kk == 0 || __ldcg(P.segpos + kk) != __ldcg(P.segpos + kk - 1)) prefix = NONE64;
        if (kk < qg) prefix = min(prefix, ldcg64(P.cand + kk));
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
            if (n >> OI_LEN_BITS) atomicOr(P.err, 4);  // a reduced column of >= 2^24 entries
            __threadfence();
            P.owninfo[rkid(P, cval)] = (uint64_t(off) << OI_LEN_BITS) | n;
            const unsigned long long r = atomicAdd(P.nrec, 1ull);
            // (birth cell, death cell): cohomology (column, pivot), homology (pivot, column)
            const uint64_t cc = rkid(P, P.cols[j]), pc = rkid(P, cval);
            P.rec[r] = P.hom ? ((pc << 32) | cc) : ((cc << 32) | pc);
          }
          fin = true;
        }
      }
    }
    // next lo of my group = min(first unfinished window column, lo + G, end of the segment)
    const unsigned nxt = ((round + 1) & 1) * P.ngroups, cur = (round & 1) * P.ngroups;
    if (grp < P.ngroups) {
      if (lane == 0 && j < end && !fin) atomicMin(P.lo_buf + nxt + grp, j);
      if (k == 0 && lane == 0) {
        const uint64_t nl = uint64_t(lo) + G;
        atomicMin(P.lo_buf + nxt + grp, unsigned(nl < end ? nl : end));
        P.lo_buf[cur + grp] = NONE32;
        if (seg >= P.nseg) atomicAdd(P.done_buf + ((round + 1) & 1), 1u);
      }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      P.done_buf[round & 1] = 0;
      atomicAdd(P.stats, 1ull);
    }
    grid.sync();
    if (__ldcg(P.done_buf + ((round + 1) & 1)) >= P.ngroups) break;
    if (__ldcg(P.err)) break;
    if (grp < P.ngroups && seg < P.nseg) {
      lo = __ldcg(P.lo_buf + nxt + grp);
      if (lo >= end) {  // segment done: the group moves on to its next one
        seg += P.ngroups;
        lo = seg < P.nseg ? __ldg(P.seg_off + seg) : P.ncols;
        end = seg < P.nseg ? __ldg(P.seg_off + seg + 1) : P.ncols;
        j = lo + k;
        started = false;
        fin = false;
      }
    }
  }
}

__global__ void k_collect_columns(const uint32_t* __restrict__ births,
                                  const uint8_t* __restrict__ tags, Geom g, int d, int hom,
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
      key = hom ? ~make_key(b, k) : make_key(b, k);
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
                           int hom, uint32_t* __restrict__ segk) {
  unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) segk[i] = (hom ? ~key_kidx(cols[i]) : key_kidx(cols[i])) / seg_cells;
}

// Homology mode, after the reduction: a residual d-cell (not apparent, not cleared as a death
// cell of dimension d-1) that is no column's pivot is an essential class (birth, +inf).
__global__ void k_hom_essential(const uint32_t* __restrict__ births,
                                const uint8_t* __restrict__ tags, Geom g, int d,
                                const uint64_t* __restrict__ owninfo, uint64_t* rec,
                                unsigned long long* nrec) {
  const int64_t kk = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (kk >= g.ncells) return;
  const uint32_t k = uint32_t(kk);
  const uint32_t KX = uint32_t(g.KX), KY = uint32_t(g.KY);
  const uint32_t X = k % KX, r = k / KX, Y = r % KY, Z = r / KY;
  if (int((X & 1) + (Y & 1) + (Z & 1)) != d) return;
  if (births[k] == ABSENT_ORD || tag_kind(tags[k]) != KIND_RESIDUAL) return;
  if (owninfo && ldcg64(owninfo + k) != NONE64) return;
  rec[atomicAdd(nrec, 1ull)] = (uint64_t(k) << 32) | NONE32;
}

// Clearing for the homology mode: the birth cells of dimension-(d+1) records (cells that create a
// class, paired with a (d+2)-cell or essential) have zero reduced boundary columns.
__global__ void k_mark_cleared_birth(const uint64_t* __restrict__ rec, int64_t n, uint8_t* tags) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) tags[uint32_t(rec[i] >> 32)] = make_tag(KIND_CLEARED, 0);
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

__global__ void k_mark_cleared(const uint64_t* __restrict__ rec, int64_t n, uint8_t* tags) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t dk = uint32_t(rec[i]);
  if (dk != NONE32) tags[dk] = make_tag(KIND_CLEARED, 0);
}

}  // namespace

void reduce_dimension(GeneralState& S, int d, Workspace& ws, HostScalars& hs, cr_stats& st,
                      bool hom) {
  cudaStream_t s = ws.stream();
  const Geom& g = S.g;
  const int B = 256;
  const int dc = hom ? d + 1 : d;  // dimension of the column cells
  const int64_t nd = st.cells[dc];
  // records: at most one per column, plus (homology) the essential d-cells
  S.R.rec[d] = ws.alloc<uint64_t>(nd + (hom ? st.cells[d] : 0) + 1);
  S.R.n[d] = 0;
  if (nd == 0 && !hom) return;

  unsigned long long* ctr = ws.alloc<unsigned long long>(16);
  CR_CUDA(cudaMemsetAsync(ctr, 0, 16 * sizeof(unsigned long long), s));
  uint64_t* cols = ws.alloc<uint64_t>(nd + 1);
  k_collect_columns<<<grid_for(g.ncells, B), B, 0, s>>>(S.births, S.tags, g, dc, hom ? 1 : 0,
                                                        cols, reinterpret_cast<unsigned*>(ctr));
  CR_CHECK_LAUNCH();
  const unsigned ncols = read_scalar(reinterpret_cast<unsigned*>(ctr), s, hs);
  st.columns[d] = ncols;
  if (ncols > 0) {
    sort_keys_u64(cols, ncols, /*descending=*/true, 64, ws);
    unsigned nseg = 1;
    uint32_t* seg_off = nullptr;
    if (S.seg_cells) {
      // batched images: group the columns by image (stable, so each image keeps its decreasing
      // key order); images are independent complexes, so their relative order is immaterial
      uint32_t* segk = ws.alloc<uint32_t>(ncols);
      uint32_t* segk2 = ws.alloc<uint32_t>(ncols);
      uint64_t* cols2 = ws.alloc<uint64_t>(ncols);
      k_seg_keys<<<grid_for(ncols, B), B, 0, s>>>(cols, ncols, S.seg_cells, hom ? 1 : 0, segk);
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
      nseg = unsigned((uint64_t(g.ncells) + S.seg_cells - 1) / S.seg_cells);
      seg_off = ws.alloc<uint32_t>(nseg + 1);
      k_seg_offsets<<<grid_for(nseg + 1, B), B, 0, s>>>(dk.Current(), ncols, nseg, seg_off);
      CR_CHECK_LAUNCH();
    } else {
      seg_off = ws.alloc<uint32_t>(2);
      const uint32_t h[2] = {0u, ncols};
      CR_CUDA(cudaMemcpyAsync(seg_off, h, sizeof(h), cudaMemcpyHostToDevice, s));
      CR_CUDA(cudaStreamSynchronize(s));  // h is on the stack
    }

    int dev = 0, nsm = 0, per_sm = 0;
    CR_CUDA(cudaGetDevice(&dev));
    CR_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    CR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_reduce, THREADS, 0));
    if (per_sm < 1) throw Error{CR_EINTERNAL, "k_reduce cannot be resident"};
    per_sm = per_sm > K5_MINB ? K5_MINB : per_sm;
    if (const char* e = std::getenv("CR_K5_PER_SM")) per_sm = std::max(1, std::min(per_sm, std::atoi(e)));
    int64_t blocks = int64_t(nsm) * per_sm;
    const int64_t need_blocks = (int64_t(ncols) + WPB - 1) / WPB;  // small problems
    if (need_blocks < blocks) blocks = need_blocks;
    if (blocks > int64_t(THREADS) * 4) blocks = THREADS * 4;
    const uint32_t W = uint32_t(blocks * WPB);

    uint64_t* owninfo = ws.alloc<uint64_t>(g.ncells);
    uint64_t* cand = ws.alloc<uint64_t>(W + blocks);
    uint64_t* chunkmin = ws.alloc<uint64_t>(blocks);
    uint32_t* chunkflag = ws.alloc<uint32_t>(blocks);
    uint32_t* segpos = ws.alloc<uint32_t>(W);
    const uint32_t ngroups = nseg < W ? nseg : W, G = W / ngroups;
    unsigned* lo_buf = ws.alloc<unsigned>(2 * int64_t(ngroups));
    unsigned* done_buf = reinterpret_cast<unsigned*>(ctr + 2);
    int* err = reinterpret_cast<int*>(ctr + 3);
    unsigned long long* nrec = ctr + 4;
    unsigned long long* pool_top = ctr + 5;
    unsigned long long* stats = ctr + 6;  // [6] rounds [7] additions [8] lengths [9] max length

    // main-array slot per warp; longer columns grow into the pool.  The pool (reduced columns +
    // grown main arrays) is sized so that exhausting it -- which reruns the whole launch with 4x --
    // does not happen on realistic inputs: 16 entries per column + 32 Mi entries (256 MB)
    const uint32_t mcap = std::getenv("CR_K5_MCAP")
                              ? uint32_t(std::atoi(std::getenv("CR_K5_MCAP")))
                              : 4096u;
    unsigned long long pool_cap = 16ull * ncols + (1ull << 25);
    uint64_t* work = nullptr;
    uint64_t* pool = nullptr;
    unsigned long long* P_colstat = nullptr;
    unsigned long long* P_rdbg = nullptr;
    uint32_t P_rdbg_cap = 0;
    for (int attempt = 0;; ++attempt) {
      if (!work) work = ws.alloc<uint64_t>(int64_t(W) * 2 * mcap);
      if (!pool) pool = ws.alloc<uint64_t>(int64_t(pool_cap));
      CR_CUDA(cudaMemsetAsync(owninfo, 0xFF, g.ncells * sizeof(uint64_t), s));
      CR_CUDA(cudaMemsetAsync(lo_buf, 0xFF, 2 * sizeof(unsigned) * ngroups, s));
      CR_CUDA(cudaMemsetAsync(done_buf, 0, 2 * sizeof(unsigned), s));
      CR_CUDA(cudaMemsetAsync(err, 0, sizeof(int), s));
      CR_CUDA(cudaMemsetAsync(nrec, 0, 6 * sizeof(unsigned long long), s));
      RP P;
      P.g = g;
      P.fx = FastDiv::make(uint32_t(g.KX));
      P.fxy = FastDiv::make(uint32_t(g.KX * g.KY));
      P.d = d;
      P.hom = hom ? 1 : 0;
      P.cols = cols;
      P.ncols = ncols;
      P.births = S.births;
      P.tags = S.tags;
      P.owninfo = owninfo;
      P.pool = pool;
      P.pool_top = pool_top;
      P.pool_cap = pool_cap;
      P.work = work;
      P.mcap = mcap;
      P.cand = cand;
      P.chunkmin = chunkmin;
      P.chunkflag = chunkflag;
      P.segpos = segpos;
      P.seg_cells = S.seg_cells;
      P.lo_buf = lo_buf;
      P.done_buf = done_buf;
      P.seg_off = seg_off;
      P.nseg = nseg;
      P.G = G;
      P.ngroups = ngroups;
      P.rec = S.R.rec[d];
      P.nrec = nrec;
      P.err = err;
      // Round length: a warp stops adding after ~100 us of the round (not after a fixed number
      // of additions): columns blocked on an earlier column's commit resume one round after it,
      // so short rounds speed up chains of dependent columns, while long ones amortise the grid
      // syncs.  Measured (CR_K5_BUDGET_US / CR_K5_STEPS): C4 reduce 168 ms with 256 steps per
      // round -> 103 ms, C5 1.63 -> 1.37 s, C5b 0.62 -> 0.37 s; with read-ahead 100 us is best
      // on C4 (100 / 106 / 118 ms at 100 / 150 / 250 us; C5, C5b within run-to-run noise).
      {
        int clk_khz = 0;
        CR_CUDA(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev));
        const char* bu = std::getenv("CR_K5_BUDGET_US");
        const double us = bu ? std::atof(bu) : 100.0;
        P.budget = (long long)(us * (clk_khz > 0 ? clk_khz : 1900000) / 1e3);
        const char* ah = std::getenv("CR_K5_AHEAD");
        P.ahead = ah ? std::atoi(ah) : 1;
        const char* ms = std::getenv("CR_K5_STEPS");
        P.max_steps = ms ? std::atoi(ms) : (1 << 30);
      }
      P.stats = stats;
      P.debug = std::getenv("CR_DEBUG_STATS") != nullptr;
      {
        const int dbg = P.debug ? 1 : 0;
        unsigned long long z[4] = {0, 0, 0, 0};
        CR_CUDA(cudaMemcpyToSymbolAsync(g_k5_dbg, &dbg, sizeof(int), 0, cudaMemcpyHostToDevice, s));
        CR_CUDA(cudaMemcpyToSymbolAsync(g_k5_flush, z, sizeof(z), 0, cudaMemcpyHostToDevice, s));
      }
      P.colstat = nullptr;
      P.rdbg = nullptr;
      P.rdbg_cap = 0;
      if (P.debug) {
        P.rdbg_cap = 16384;
        P.rdbg = ws.alloc<unsigned long long>(4 * int64_t(P.rdbg_cap));
        CR_CUDA(cudaMemsetAsync(P.rdbg, 0, 32 * sizeof(unsigned long long) * P.rdbg_cap / 8, s));
      }
      if (P.debug) {
        if (!P_colstat) P_colstat = ws.alloc<unsigned long long>(6 * int64_t(ncols));
        P.colstat = P_colstat;
        CR_CUDA(cudaMemsetAsync(P.colstat, 0, 6 * sizeof(unsigned long long) * ncols, s));
      }
      P_rdbg = P.rdbg;
      P_rdbg_cap = P.rdbg_cap;
      void* args[] = {&P};
      CR_CUDA(cudaLaunchCooperativeKernel((void*)k_reduce, dim3(unsigned(blocks)), dim3(THREADS),
                                          args, 0, s));
      ++g_launch_count;
      const int e = read_scalar(err, s, hs);
      if (std::getenv("CR_DEBUG_STATS"))
        fprintf(stderr, "[cr] dim %d attempt %d: err %d (mcap %u, pool %llu)\n", d, attempt, e,
                mcap, pool_cap);
      if (e == 0) break;
      if (e & 4) throw Error{CR_EINTERNAL, "reduced column longer than 2^24 entries"};
      if (e & 8) throw Error{CR_EINTERNAL, "homology reduction: a column reduced to zero"};
      if (attempt > 12) throw Error{CR_ENOMEM, "reduction buffers exhausted"};
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
      std::vector<unsigned long long> cs(6 * size_t(ncols));
      CR_CUDA(cudaMemcpy(cs.data(), P_colstat, cs.size() * 8, cudaMemcpyDeviceToHost));
      std::vector<std::pair<unsigned long long, uint32_t>> byent(ncols);
      unsigned long long tot = 0;
      for (uint32_t j = 0; j < ncols; ++j) {
        byent[j] = {cs[6 * j + 1], j};
        tot += cs[6 * j + 1];
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
      {
        const uint32_t nr = uint32_t(std::min<unsigned long long>(hs.p[6], P_rdbg_cap));
        std::vector<unsigned long long> R(4 * size_t(nr));
        CR_CUDA(cudaMemcpy(R.data(), P_rdbg, R.size() * 8, cudaMemcpyDeviceToHost));
        double cyc = 0, steps_full = 0;
        unsigned long long hist[5] = {0, 0, 0, 0, 0};
        for (uint32_t r = 0; r < nr; ++r) {
          cyc += double(R[4 * r]);
          const unsigned long long ms = R[4 * r + 1];
          hist[ms >= 256 ? 4 : ms >= 64 ? 3 : ms >= 16 ? 2 : ms >= 1 ? 1 : 0]++;
          if (ms >= 256) steps_full += 1;
        }
        const double wall = nr > 1 ? double(R[4 * (nr - 1) + 3] - R[3]) / 1e6 : 0.0;
        fprintf(stderr, "[cr] dim %d rounds %u: sum of max phase-A %.1f ms (at 1.9 GHz), wall %.1f ms;"
                " max-steps hist 0:%llu 1-15:%llu 16-63:%llu 64-255:%llu 256:%llu\n",
                d, nr, cyc / 1.9e6, wall, hist[0], hist[1], hist[2], hist[3], hist[4]);
        for (uint32_t r = 0; r < nr; r += nr / 12 + 1)
          fprintf(stderr, "   round %u: maxA %.1f us steps %llu active %llu\n", r,
                  R[4 * r] / 1.9e3, R[4 * r + 1], R[4 * r + 2]);
      }
      fprintf(stderr, "\n[cr] top columns (pos, adds, entries):");
      for (int q = 0; q < 8 && q < int(ncols); ++q) {
        const uint32_t jj = byent[q].second;
        const double a = double(cs[6 * jj] ? cs[6 * jj] : 1);
        fprintf(stderr, "\n   col %u adds %llu entries %llu | per add cycles: lookup %.0f app %.0f "
                "pool %.0f (flush %.0f)", jj, cs[6 * jj], byent[q].first, cs[6 * jj + 2] / a,
                cs[6 * jj + 3] / a, cs[6 * jj + 4] / a, cs[6 * jj + 5] / a);
      }
      fprintf(stderr, "\n");
      fprintf(stderr,
              "[cr] dim %d: cols %u rounds %llu adds %llu pool_adds %llu pool_len %llu "
              "cyc_pool %llu cyc_app %llu cyc_lookup %llu W %u\n",
              d, ncols, hs.p[6], hs.p[7], hs.p[10], hs.p[11], hs.p[13], hs.p[14], hs.p[15], W);
    }
    if (hom) {
      k_hom_essential<<<grid_for(g.ncells, B), B, 0, s>>>(S.births, S.tags, g, d, owninfo,
                                                         S.R.rec[d], ctr + 4);
      CR_CHECK_LAUNCH();
      S.R.n[d] = int64_t(read_scalar(ctr + 4, s, hs));
    }
    ws.release(work);
    ws.release(pool);
    ws.release(owninfo);
  } else if (hom) {
    k_hom_essential<<<grid_for(g.ncells, B), B, 0, s>>>(S.births, S.tags, g, d, nullptr,
                                                       S.R.rec[d], ctr + 4);
    CR_CHECK_LAUNCH();
    S.R.n[d] = int64_t(read_scalar(ctr + 4, s, hs));
  }
  if (S.R.n[d] > 0 && !hom) {
    k_mark_cleared<<<grid_for(S.R.n[d], B), B, 0, s>>>(S.R.rec[d], S.R.n[d], S.tags);
    CR_CHECK_LAUNCH();
  }
  ws.release(cols);
}

void mark_cleared_births(GeneralState& S, int d, Workspace& ws) {
  if (S.R.n[d] <= 0) return;
  k_mark_cleared_birth<<<grid_for(S.R.n[d], 256), 256, 0, ws.stream()>>>(S.R.rec[d], S.R.n[d],
                                                                          S.tags);
  CR_CHECK_LAUNCH();
}

}  // namespace cr
