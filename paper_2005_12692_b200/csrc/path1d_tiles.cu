// path1d_tiles.cu -- the fused 1D barcode path (H0 of a path).
//
// Basins (vertices older than both neighbours) and barriers (peak edges; an infinite barrier where
// a finite run ends) alternate along the series; every other cell is in a zero-persistence apparent
// pair (path1d.cu).  A basin b dies at min(L, R), where L (R) is the highest barrier between b and
// the nearest older basin on its left (right), +inf if there is none (elder rule: that is the first
// edge joining b's component to an older vertex).
//
// Level 1 streams the series once, one tile of 4096 samples per CTA, all in shared memory:
//   1. ord() of the samples (+1 halo each side), NaN check;
//   2. the tile's basins ("items") and each item's right barrier, compacted by a block scan;
//   3. a min-tree of basin keys and a max-tree of barrier keys; every item searches its nearest
//      older basin on both sides inside the tile (O(log) shared-memory steps, all items in
//      parallel).  A side that leaves the tile only yields a lower bound (the highest barrier seen);
//      the death is decided when the known side is lower than the other side's bound;
//   4. records (birth, death or pending, sample index) of all basins, and the undecided basins as
//      items of a contracted sequence whose barriers are the maxima of the barriers between kept
//      basins (a basin that died inside a tile never changes another basin's answer: its own older
//      neighbour lies between it and anything farther).  Each tile writes its own fixed-size
//      regions, so no tile waits for another.
// Levels 2.. apply the same tile solver to the contracted items until they fit one tile, where both
// ends of the series are known and every death is decided.  A final single-pass compaction writes
// the staged bars (death > birth, or essential) per tile to the output in basin (= birth kidx)
// order; undecided basins that later turn out zero-length become holes that the gather drops.
#include <cooperative_groups.h>

#include <cub/cub.cuh>

#include "pipeline.cuh"

namespace cg = cooperative_groups;

namespace cr {
namespace {

constexpr uint32_t INF_ORD = 0xFFFFFFFFu;  // ord of an infinite (run-end) barrier
constexpr uint64_t INF_KEY = ~0ull;        // normalised exact +inf
constexpr uint32_t DEATH_PENDING = 0xFFFFFFFEu;
constexpr uint32_t DEATH_ESSENTIAL = 0xFFFFFFFFu;
constexpr uint64_t KEY_NONE = 0;  // no barrier / unknown barrier: neutral for max

constexpr int THREADS = 256;
constexpr int MAXITEMS = 512;           // items per CTA buffer (level-1 residual, level-k tile)
#ifndef CR_1D_ITILE
#define CR_1D_ITILE 512
#endif
constexpr int ITILE = CR_1D_ITILE;      // items per level-k tile (<= MAXITEMS)
static_assert(ITILE <= MAXITEMS, "level tiles fit the CTA buffers");
constexpr int L1_WARPS = THREADS / 32;
constexpr int L1_SPW = 512;             // level-1 samples per warp region
constexpr int L1_TILE = L1_WARPS * L1_SPW;  // level-1 samples per CTA
constexpr int L1_IPW = L1_SPW / 2;      // basins per warp region (no two adjacent)
constexpr int SLOTS1 = L1_TILE / 2;     // staging slots per level-1 tile
constexpr int NLEVELS = 5;              // contraction levels after level 1 (last must be final)
constexpr int TREE_CAP = 2 * MAXITEMS;
// dynamic shared memory: two trees, then death / kept-rank / kept-position / id arrays
constexpr size_t SMEM = size_t(TREE_CAP) * 8 * 2 + size_t(MAXITEMS) * 8 + size_t(MAXITEMS) * 4 * 4;

// Shared-memory trees over n <= MAXITEMS items: mn = min of basin keys, mx = max of
// right-barrier keys.  Level l holds ceil(n / 2^l) nodes at offset 2*MAXITEMS - (2*MAXITEMS >> l);
// node p of level l covers items [p 2^l, (p+1) 2^l).  Offsets are arithmetic so that the struct
// stays in registers and every access is a plain LDS.
struct STree {
  uint64_t* mn;
  uint64_t* mx;
  int n;
  int levels;
};
__device__ __forceinline__ int st_off(int l) { return 2 * MAXITEMS - ((2 * MAXITEMS) >> l); }
__device__ __forceinline__ int st_sz(const STree& T, int l) {
  return T.n == 0 ? 0 : ((T.n - 1) >> l) + 1;
}

__device__ __forceinline__ void stree_layout(STree& T, int n) {
  T.n = n;
  int l = 0;
  while (n > 1) {
    n = (n + 1) >> 1;
    ++l;
  }
  T.levels = l + 1;
}

__device__ __forceinline__ void stree_build(STree& T) {
  for (int l = 1; l < T.levels; ++l) {
    const int pc = st_off(l - 1), nc = st_sz(T, l - 1), pp = st_off(l), np = st_sz(T, l);
    for (int p = threadIdx.x; p < np; p += THREADS) {
      const int a = 2 * p, b = 2 * p + 1;
      uint64_t mn = T.mn[pc + a], mx = T.mx[pc + a];
      if (b < nc) {
        mn = min(mn, T.mn[pc + b]);
        mx = max(mx, T.mx[pc + b]);
      }
      T.mn[pp + p] = mn;
      T.mx[pp + p] = mx;
    }
    __syncthreads();
  }
}

// max of mx over items [a, b] (inclusive), KEY_NONE if empty
__device__ __forceinline__ uint64_t stree_rmax(const STree& T, int a, int b) {
  uint64_t r = KEY_NONE;
  for (int l = 0; a <= b && l < T.levels; ++l) {
    if (a & 1) r = max(r, T.mx[st_off(l) + a++]);
    if (!(b & 1)) r = max(r, T.mx[st_off(l) + b--]);
    a >>= 1;
    b = (b + 1) / 2 - 1;  // floor((b-1)/2) for b >= -1 without negative shifts
  }
  return r;
}

// Nearest older basin left of item j.  Found: true, acc = max right barrier of items i..j-1.
// Not found: false, acc = max right barrier of items 0..j-1.
__device__ __forceinline__ bool search_left(const STree& T, int j, uint64_t q, uint64_t& acc) {
  acc = KEY_NONE;
  int l = 0, p = j - 1;
  while (p >= 0) {
    if (T.mn[st_off(l) + p] < q) {
      while (l > 0) {
        --l;
        const int r = 2 * p + 1;
        if (r < st_sz(T, l) && T.mn[st_off(l) + r] < q) {
          p = r;
        } else {
          if (r < st_sz(T, l)) acc = max(acc, T.mx[st_off(l) + r]);
          p = 2 * p;
        }
      }
      acc = max(acc, T.mx[p]);
      return true;
    }
    acc = max(acc, T.mx[st_off(l) + p]);
    if (p & 1) {
      p -= 1;
    } else {
      p = p / 2 - 1;
      ++l;
    }
  }
  return false;
}

// Nearest older basin right of item j.  Found: acc = max right barrier of items j..r-1.
// Not found: acc = max right barrier of items j..n-1.
__device__ __forceinline__ bool search_right(const STree& T, int j, uint64_t q, uint64_t& acc) {
  acc = T.mx[j];
  int l = 0, p = j + 1;
  while (l < T.levels && p < st_sz(T, l)) {
    if (T.mn[st_off(l) + p] < q) {
      while (l > 0) {
        --l;
        const int c = 2 * p;
        if (T.mn[st_off(l) + c] < q) {
          p = c;
        } else {
          acc = max(acc, T.mx[st_off(l) + c]);
          p = c + 1;
        }
      }
      return true;
    }
    acc = max(acc, T.mx[st_off(l) + p]);
    if (!(p & 1)) {
      p += 1;
    } else {
      p = (p + 1) / 2;
      ++l;
    }
  }
  return false;
}

// Decide item j.  left_start: the tile begins at the start of the series.  lead: highest barrier
// left of item 0 that is not an item's right barrier (KEY_NONE if none/unknown).
// Returns the death ord, DEATH_ESSENTIAL, or DEATH_PENDING (undecided in this tile).
__device__ __forceinline__ uint32_t decide(const STree& T, int j, bool left_start, uint64_t lead) {
  const uint64_t q = T.mn[j];
  uint64_t L, R;
  const bool fl = search_left(T, j, q, L);
  const bool fr = search_right(T, j, q, R);
  bool lk = true, rk = true;  // exactly known?
  if (!fl) {
    L = max(L, lead);
    if (left_start) L = INF_KEY;
    else lk = key_ord(L) == INF_ORD;
  }
  if (lk && key_ord(L) == INF_ORD) L = INF_KEY;
  if (!fr) rk = key_ord(R) == INF_ORD;
  if (rk && key_ord(R) == INF_ORD) R = INF_KEY;
  uint64_t d;
  if (lk && rk) d = min(L, R);
  else if (lk && L < R) d = L;        // R is a lower bound of the right side
  else if (rk && R < L) d = R;        // L is a lower bound of the left side
  else return DEATH_PENDING;
  return d == INF_KEY ? DEATH_ESSENTIAL : key_ord(d);
}


__device__ unsigned long long* g_tl = nullptr;  // debug: level-tile timeline (block 0)
__device__ __forceinline__ void tl_mark(int slot) {
  if (g_tl && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_tl[slot] = t;
  }
}
__device__ int g_rounds = 1;      // contraction rounds before the tree (tunable: CR_1D_ROUNDS)
__device__ int g_l1_rounds = 3;   // level-1 warp rounds incl. the register round (CR_1D_L1ROUNDS)

// ------------------------------------------------------------------------------------------
// Per-tile regions.  Level-1 tile t owns staging slots [t*SLOTS1, (t+1)*SLOTS1) for its output
// candidates (bars with death > birth, essential bars, and undecided basins) in basin order, and an
// item region of the same size for its undecided basins (the next level's input).  No tile waits
// for another: the next kernel scans the per-tile counts.
// ------------------------------------------------------------------------------------------
struct Items {
  uint64_t* key;  // basin key (ord << 32 | sample index)
  uint64_t* rb;   // max barrier key up to the next kept item (or the tile end)
  uint32_t* id;   // staging slot of the basin
  uint32_t* cnt;  // per tile: kept items
  uint64_t* lead; // per tile: max barrier before its first kept item (all of it if none kept)
};

struct Stage {
  uint2* st;          // level-1 staging per slot: (birth, death) float bits; birth HOLE: zero
                      // persistence; death BAR_PENDING, then PEND_TAG | rank: undecided
  uint32_t* cell;     // birth kidx per slot (optional)
  uint32_t* rcnt;     // per level-1 region: basins (slots in use)
  uint32_t* holes;    // per level-1 region: zero-persistence basins
  uint32_t* regoff;   // per level-1 region: output offset of its first bar
  cr_pair* out;       // final output (bars in basin order), capacity cap
  uint32_t* out_cells;
  int64_t cap;
  unsigned long long* cnt;    // [0] undecided basins exported, [1] decided later, [2] of them
                              // zero-persistence (holes in the output)
  uint32_t* ltiles0;          // level-1 tile count for the item levels (written by tile 0)
};

constexpr uint32_t BAR_PENDING = 0x7FC00001u;  // NaN payload marking an undecided death
constexpr uint32_t HOLE = 0xFFFFFFFFu;
// An undecided basin's staged death after level 1: a negative-NaN tag with its rank among the
// bars of its region (< L1_IPW), from which a later level finds its output position.
constexpr uint32_t PEND_TAG = 0xFFC00000u, PEND_RANK = 0x003FFFFFu;

// Stage the decision d (death ord or DEATH_ESSENTIAL) of the basin with birth ord bo in its slot.
__device__ __forceinline__ void stage_put(const Stage& G, uint64_t slot, uint32_t bo, uint32_t d) {
  uint2 v;
  if (d == DEATH_ESSENTIAL) {
    v = make_uint2(__float_as_uint(float_of_ord(bo)), 0x7F800000u);
  } else if (d > bo) {
    v = make_uint2(__float_as_uint(float_of_ord(bo)), __float_as_uint(float_of_ord(d)));
  } else {  // zero persistence: a hole that the gather drops
    v = make_uint2(HOLE, 0u);
    atomicAdd(G.holes + slot / L1_IPW, 1u);
  }
  G.st[slot] = v;
}

// The same without the hole counter: returns whether the slot became a hole (the caller counts).
__device__ __forceinline__ uint32_t stage_put_nh(const Stage& G, uint64_t slot, uint32_t bo,
                                                 uint32_t d) {
  const bool ess = d == DEATH_ESSENTIAL;
  const bool hole = !ess && d <= bo;
  const uint32_t bx = hole ? HOLE : __float_as_uint(float_of_ord(bo));
  const uint32_t dy = ess ? 0x7F800000u : __float_as_uint(float_of_ord(d));
  G.st[slot] = make_uint2(bx, dy);
  return hole;
}

// A later level decides an undecided basin; oid = region * L1_IPW + its rank among the region's
// bars.  The gather writes the record's birth; this writes its dim (-1: a hole) and death.
__device__ __forceinline__ void final_put(const Stage& G, uint32_t oid, uint32_t bo, uint32_t d) {
  atomicAdd(G.cnt + 1, 1ull);
  const bool hole = d != DEATH_ESSENTIAL && d <= bo;
  if (hole) atomicAdd(G.cnt + 2, 1ull);  // zero persistence: compacted away by the host's fix-up
  const int64_t pos = int64_t(__ldcg(G.regoff + oid / L1_IPW)) + (oid % L1_IPW);
  if (pos >= G.cap) return;
  G.out[pos].dim = hole ? -1 : 0;
  if (!hole) G.out[pos].death = d == DEATH_ESSENTIAL ? __int_as_float(0x7F800000) : float_of_ord(d);
}

struct Smem {
  STree T;
  uint32_t* death;
  uint32_t* keep;  // staging slot (level 1)
  uint32_t* kpos;  // compacted item positions
  uint32_t* id;
  uint64_t* okey;  // level 1: the original item keys (buffers A/B are reused)
};

__device__ __forceinline__ Smem carve(unsigned char* smem) {
  Smem S;
  S.T.mn = reinterpret_cast<uint64_t*>(smem);
  S.T.mx = S.T.mn + TREE_CAP;
  S.death = reinterpret_cast<uint32_t*>(S.T.mx + TREE_CAP);
  S.keep = S.death + MAXITEMS;
  S.kpos = S.keep + MAXITEMS;
  S.id = S.kpos + MAXITEMS;
  S.okey = reinterpret_cast<uint64_t*>(S.id + MAXITEMS);
  return S;
}

// O(1) rule on the current (possibly contracted) sequence: keys K, right barriers R (R[n-1] may
// be KEY_NONE = beyond the tile), lead = barrier left of item 0 (KEY_NONE if unknown).  An item
// whose older neighbour sits across the lower of its two adjacent barriers dies there (the other
// side's bottleneck is at least the higher one); an item between two infinite barriers is
// essential.  Returns the death ord, DEATH_ESSENTIAL, or DEATH_PENDING (not decided by this rule).
__device__ __forceinline__ uint32_t quick1(const uint64_t* K, const uint64_t* R, int n, int j,
                                           bool left_start, uint64_t lead) {
  const uint64_t q = K[j];
  const uint64_t bl = j > 0 ? R[j - 1] : (left_start ? INF_KEY : lead);
  const uint64_t br = R[j];
  const bool linf = key_ord(bl) == INF_ORD, rinf = key_ord(br) == INF_ORD;
  if (linf && rinf) return DEATH_ESSENTIAL;
  if (j > 0 && K[j - 1] < q && !linf && br != KEY_NONE && bl < br) return key_ord(bl);
  if (j + 1 < n && K[j + 1] < q && !rinf && bl != KEY_NONE && br < bl) return key_ord(br);
  return DEATH_PENDING;
}

// Decide the items of a tile.  (1) Contraction rounds: apply quick1 to every item, drop the decided
// ones and fold their right barriers into the nearest kept item on their left (into the lead if
// none) -- the contracted sequence has the same answers for the items it keeps.  Each round is
// O(1) per item and fully parallel; a random walk's sequence shrinks ~3x per round.  (2) The few
// items left when a round makes no progress get the full nearest-older tree search.
// Buffers: A = (T.mn, T.mx, id) [0, MAXITEMS), B = (T.mn, T.mx)[MAXITEMS, 2 MAXITEMS) + kpos.
// On return the residual sequence is in buffer A with its tree built; pending residual items are
// flagged in s_pend; the tile's lead is returned.  sink(id, key, death) records each decision.
__shared__ uint32_t s_pend[MAXITEMS / 32];

template <class Sink>
__device__ __forceinline__ int decide_tile(Smem& S, int n, bool left_start, uint64_t& lead, Sink sink) {
  typedef cub::BlockScan<uint32_t, THREADS> BS;
  __shared__ typename BS::TempStorage s_scan;
  __shared__ uint64_t s_lead;
  constexpr int CH = MAXITEMS / THREADS;
  // buffer c: keys S.T.mn + c*MAXITEMS, barriers S.T.mx + c*MAXITEMS, ids S.id - c*MAXITEMS
  // (= S.kpos for c = 1); arithmetic on the shared bases keeps every access an LDS/STS
#define KB(c) (S.T.mn + (c) * MAXITEMS)
#define RB(c) (S.T.mx + (c) * MAXITEMS)
#define IB(c) (S.id - (c) * MAXITEMS)
  int cur = 0;
  const int c0 = threadIdx.x * CH;
  for (int round = 0; round < g_rounds && n > 0; ++round) {
    uint32_t kb = 0;
#pragma unroll
    for (int r = 0; r < CH; ++r) {
      const int j = c0 + r;
      if (j >= n) continue;
      const uint32_t d = quick1(KB(cur), RB(cur), n, j, left_start, lead);
      if (d != DEATH_PENDING) sink(IB(cur)[j], KB(cur)[j], d);
      else kb |= 1u << r;
    }
    uint32_t pre, tot;
    BS(s_scan).ExclusiveSum(uint32_t(__popc(kb)), pre, tot);
    if (threadIdx.x == 0) s_lead = lead;
    if (int(tot) == n) break;  // no progress: the tree decides the rest (uniform branch)
    const int nx = cur ^ 1;
    uint32_t p = pre;
#pragma unroll
    for (int r = 0; r < CH; ++r) {  // kept items move to their new slots
      if (!(kb >> r & 1)) continue;
      const int j = c0 + r;
      KB(nx)[p] = KB(cur)[j];
      RB(nx)[p] = RB(cur)[j];
      IB(nx)[p] = IB(cur)[j];
      ++p;
    }
    __syncthreads();
    p = pre;
#pragma unroll
    for (int r = 0; r < CH; ++r) {  // a dropped item's barrier folds into the kept item on its left
      const int j = c0 + r;
      if (j >= n) continue;
      if (kb >> r & 1) {
        ++p;
      } else {
        const unsigned long long rb = RB(cur)[j];
        if (p == 0) atomicMax(reinterpret_cast<unsigned long long*>(&s_lead), rb);
        else atomicMax(reinterpret_cast<unsigned long long*>(RB(nx) + p - 1), rb);
      }
    }
    __syncthreads();
    lead = s_lead;
    n = int(tot);
    cur = nx;
    __syncthreads();  // s_lead is rewritten next round
  }
  if (cur == 1) {  // residual into buffer A (the tree's level 0)
    for (int j = threadIdx.x; j < n; j += THREADS) {
      S.T.mn[j] = KB(1)[j];
      S.T.mx[j] = RB(1)[j];
      S.id[j] = IB(1)[j];
    }
    __syncthreads();
  }
  for (int w = threadIdx.x; w < MAXITEMS / 32; w += THREADS) s_pend[w] = 0;
  __syncthreads();
  tl_mark(8);
  stree_layout(S.T, n);
  stree_build(S.T);
  tl_mark(9);
  for (int j = threadIdx.x; j < n; j += THREADS) {
    const uint32_t d = decide(S.T, j, left_start, lead);
    if (d != DEATH_PENDING) sink(S.id[j], S.T.mn[j], d);
    else atomicOr(&s_pend[j >> 5], 1u << (j & 31));
  }
  __syncthreads();
  return n;
#undef KB
#undef RB
#undef IB
}

// Export the residual's pending items (flags in s_pend) into the tile's item region, with their
// contracted barriers (max up to the next pending item) and the tile's lead.
template <class IdMap>
__device__ __forceinline__ void export_pending(Smem& S, int n, uint64_t lead, const Items& O, uint32_t tile,
                               IdMap idmap) {
  typedef cub::BlockScan<uint32_t, THREADS> BS;
  __shared__ typename BS::TempStorage s_scan;
  __shared__ uint32_t s_nk;
  constexpr int CH = MAXITEMS / THREADS;
  const int c0 = threadIdx.x * CH;
  uint32_t mine = 0;
#pragma unroll
  for (int r = 0; r < CH; ++r) {
    const int j = c0 + r;
    if (j < n) mine += s_pend[j >> 5] >> (j & 31) & 1;
  }
  uint32_t pre, tot;
  BS(s_scan).ExclusiveSum(mine, pre, tot);
#pragma unroll
  for (int r = 0; r < CH; ++r) {
    const int j = c0 + r;
    if (j < n && (s_pend[j >> 5] >> (j & 31) & 1)) S.kpos[pre++] = j;
  }
  if (threadIdx.x == 0) s_nk = tot;
  __syncthreads();
  const uint32_t nk = s_nk;
  const uint64_t base = uint64_t(tile) * MAXITEMS;
  for (uint32_t r = threadIdx.x; r < nk; r += THREADS) {
    const int j = int(S.kpos[r]);
    const int nxt = r + 1 < nk ? int(S.kpos[r + 1]) : n;
    O.key[base + r] = S.T.mn[j];
    O.rb[base + r] = stree_rmax(S.T, j, nxt - 1);
    O.id[base + r] = idmap(S.id[j]);
  }
  if (threadIdx.x == 0) {
    O.cnt[tile] = nk;
    const int fk = nk ? int(S.kpos[0]) : n;
    uint64_t ld = lead;
    if (fk > 0) ld = max(ld, stree_rmax(S.T, 0, fk - 1));
    O.lead[tile] = ld;
  }
}

// ------------------------------------------------------------------------------------------
// Gather one level-1 region (warp-collective): its staged bars minus holes, in basin order, to the
// output from position o.  All of the region's slots are loaded first (<= L1_IPW / 32 per lane);
// bars are staged in shared memory (96 words per warp) so that the 12-byte records go out as
// contiguous 4-byte stores.  An undecided basin's record gets its birth only: the level that
// decides it writes its dim and death (distinct words, so the two may run concurrently).
__device__ __forceinline__ void gather_region(const Stage& G, int r, int64_t o, uint32_t* sb96) {
  constexpr int NCH = L1_IPW / 32;
  const int lane = threadIdx.x & 31;
  const uint32_t nc = G.rcnt[r];
  const uint64_t sb = uint64_t(r) * L1_IPW;
  uint2 v[NCH];
#pragma unroll
  for (int k = 0; k < NCH; ++k) {
    const uint32_t i = 32 * k + lane;
    v[k] = i < nc ? __ldcs(G.st + sb + i) : make_uint2(HOLE, 0u);
  }
#pragma unroll
  for (int k = 0; k < NCH; ++k) {
    if (32u * k >= nc) break;
    const bool keep = v[k].x != HOLE;
    const bool pend = (v[k].y & PEND_TAG) == PEND_TAG;
    const unsigned km = __ballot_sync(0xFFFFFFFFu, keep);
    const unsigned pm = __ballot_sync(0xFFFFFFFFu, keep && pend);
    const uint32_t q = __popc(km & ((1u << lane) - 1));
    if (keep) {
      sb96[3 * q + 0] = 0u;
      sb96[3 * q + 1] = v[k].x;
      sb96[3 * q + 2] = v[k].y;
      if (G.out_cells && o + q < G.cap) G.out_cells[o + q] = G.cell[sb + 32 * k + lane];
    }
    __syncwarp();
    const uint32_t nk = __popc(km);
    const int64_t lim = G.cap - o;
    const uint32_t nw = lim <= 0 ? 0u : (int64_t(nk) < lim ? nk : uint32_t(lim));
    uint32_t* dst = reinterpret_cast<uint32_t*>(G.out + o);
    if (!pm) {
      for (uint32_t t = lane; t < 3 * nw; t += 32) dst[t] = sb96[t];
    } else {  // skip the dim and death words of undecided basins
      for (uint32_t t = lane; t < 3 * nw; t += 32) {
        const uint32_t rec = t / 3, wd = t - 3 * rec;
        const bool p = (sb96[3 * rec + 2] & PEND_TAG) == PEND_TAG;
        if (!p || wd == 1) dst[t] = sb96[t];
      }
    }
    o += nk;
    __syncwarp();
  }
}

// ------------------------------------------------------------------------------------------
// Level 1.  A CTA owns L1_TILE samples; warp w owns the region of L1_SPW samples starting at
// b0 = a + w*L1_SPW, lane l the 16 samples b0 + 16l .. b0 + 16l + 15 (four float4 loads).
//  (a) each lane marks its basins and barriers in registers and exchanges with its neighbour
//      lanes the events next to its chunk ends (the previous lane's last basin and the barrier
//      after it, the next lane's first basin and the barrier before it);
//  (b) each lane streams its basins in order and applies quick1 to each (the contraction rule of
//      decide_tile: an item whose older neighbour lies across the lower of its two barriers dies
//      there; an item between two infinite barriers is essential) -- one round on the raw
//      sequence, in registers.  Decided basins are staged at once as (birth, death) in their
//      slot (region * L1_IPW + basin index); survivors go to the warp's arrays with their right
//      barrier, and a dropped basin's right barrier folds into the survivor on its left;
//  (c) more quick1 rounds on the warp's survivors (shared memory, warp-synchronous);
//  (d) the warps' residuals are concatenated (u64 keys; a barrier is keyed by its item's position,
//      which preserves the order of barriers in distinct gaps) and decided by decide_tile (rounds,
//      then the shared-memory tree search); the basins still undecided are exported to the next
//      level and their slots marked pending.
// Comparisons on 32-bit ords break ties by position: of two basins with equal ord the left one
// is older; of two barriers with equal ord the left one is lower.
// ------------------------------------------------------------------------------------------
constexpr uint32_t ORD_NONE = 0u;  // unknown barrier: neutral for max (every finite ord is > 0)

struct __align__(16) WarpBuf {
  uint32_t K[L1_IPW];   // basin ords of the warp's residual sequence
  uint32_t R[L1_IPW];   // right-barrier ords (ORD_NONE: beyond the region)
  uint32_t PI[L1_IPW];  // (offset in region << 16) | basin index in region
  uint32_t lead;        // max barrier before the first residual item
  uint32_t n;           // residual items
};
struct WarpScratch {  // the lanes' ords, [i][lane]: conflict-free
  uint32_t O[16][32];
};
static_assert(sizeof(WarpScratch) * L1_WARPS <= SMEM, "scratch aliases the CTA item buffers");
constexpr size_t L1_SMEM = SMEM + sizeof(WarpBuf) * L1_WARPS;

__device__ __forceinline__ uint32_t ord_at(const float* __restrict__ x, int64_t n, int64_t q,
                                           bool& nan) {
  if (q < 0 || q >= n) return ABSENT_ORD;
  const float v = __ldg(x + q);
  nan |= v != v;
  return ord_of(v);
}

// quick1 on 32-bit ords: basin ord q, left/right barriers bl/br (ORD_NONE: unknown), neighbour
// basin ords kp/kn (has_p/has_n: they exist).  Returns the death ord, DEATH_ESSENTIAL or
// DEATH_PENDING.
__device__ __forceinline__ uint32_t quick1_ord(uint32_t q, uint32_t bl, uint32_t br, bool has_p,
                                               uint32_t kp, bool has_n, uint32_t kn) {
  const bool linf = bl == INF_ORD, rinf = br == INF_ORD;
  if (linf && rinf) return DEATH_ESSENTIAL;
  if (has_p && kp <= q && !linf && bl != ORD_NONE && br != ORD_NONE && bl <= br) return bl;
  if (has_n && kn < q && !rinf && br != ORD_NONE && bl != ORD_NONE && br < bl) return br;
  return DEATH_PENDING;
}

__global__ void __launch_bounds__(THREADS) k1_level1(const float* __restrict__ x, int64_t n,
                                                     Items O, Stage G, int* nan_flag,
                                                     int* overflow) {
  extern __shared__ __align__(16) unsigned char smem[];
  Smem S = carve(smem);
  WarpBuf* WB = reinterpret_cast<WarpBuf*>(smem + SMEM);
  __shared__ uint32_t s_off[L1_WARPS + 1];
  __shared__ uint64_t s_lead;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1;
  WarpBuf& B = WB[w];
  WarpScratch& SC = reinterpret_cast<WarpScratch*>(smem)[w];
  const uint32_t t = blockIdx.x;
  const int64_t a = int64_t(t) * L1_TILE;
  if (t == 0 && threadIdx.x == 0) *G.ltiles0 = gridDim.x;
  const int64_t b0 = a + int64_t(w) * L1_SPW;                    // region start
  const uint64_t rslot = (uint64_t(t) * L1_WARPS + w) * L1_IPW;  // region's first slot
  const bool left_start = (t == 0 && w == 0);
  bool nan = false;
  if (lane == 0) B.lead = ORD_NONE;

  // ---------------- (a) samples and events
  const int64_t q0 = b0 + 16 * lane;
  uint32_t o[16];
  if ((reinterpret_cast<uintptr_t>(x) & 15) == 0 && q0 + 15 < n) {
    const float4* x4 = reinterpret_cast<const float4*>(x + q0);
    float4 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = __ldcs(x4 + k);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      nan |= (v[k].x != v[k].x) | (v[k].y != v[k].y) | (v[k].z != v[k].z) | (v[k].w != v[k].w);
      o[4 * k + 0] = ord_of(v[k].x);
      o[4 * k + 1] = ord_of(v[k].y);
      o[4 * k + 2] = ord_of(v[k].z);
      o[4 * k + 3] = ord_of(v[k].w);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 16; ++i) o[i] = ord_at(x, n, q0 + i, nan);
  }
  uint32_t um = __shfl_up_sync(0xFFFFFFFFu, o[15], 1);
  if (lane == 0) um = ord_at(x, n, q0 - 1, nan);
  uint32_t up = __shfl_down_sync(0xFFFFFFFFu, o[0], 1);
  if (lane == 31) up = ord_at(x, n, q0 + 16, nan);
  if (nan) atomicOr(nan_flag, 1);
  // Events as bitmasks over my 16 samples: basin at sample i (bm), barrier after sample i (mm:
  // the peak edge (i, i+1), or the end of a finite run, em, an infinite barrier).  Basins and
  // barriers alternate: one barrier between consecutive basins.  The ords stay
  // in shared memory ([i][lane], aliasing the warp's item arrays until the survivors are
  // written) for the per-basin steps below.
  uint32_t (*SO)[32] = SC.O;
  // Dm bit i: o[i] > o[i+1] (a descent after sample i); A bit i: o[i] is absent (+inf).  Then
  //   basin at i:     o[i-1] > o[i] <= o[i+1]                 = Gprev & ~G
  //   peak edge i:    o[i-1] <= o[i] > o[i+1], both finite    = Dm & ~Gprev & ~Aprev & ~A
  //   run end at i:   o[i] finite, o[i+1] absent              = Anext & ~A
  // (ABSENT_ORD exceeds every finite ord, so Dm is never set before an absent sample.)
  uint32_t Dm = 0, A = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const uint32_t c = o[i], r = i == 15 ? up : o[i + 1];
    SO[i][lane] = c;
    Dm |= c > r ? (1u << i) : 0u;
    A |= c == ABSENT_ORD ? (1u << i) : 0u;
  }
  const uint32_t Gprev = (Dm << 1) | (um > o[0] ? 1u : 0u);
  const uint32_t Aprev = (A << 1) | (um == ABSENT_ORD ? 1u : 0u);
  const uint32_t Anext = (A >> 1) | (up == ABSENT_ORD ? 0x8000u : 0u);
  const uint32_t bm = Gprev & ~Dm & 0xFFFFu;
  const uint32_t em = Anext & ~A;
  const uint32_t mm = ((Dm & ~Gprev & ~Aprev & ~A) | em) & 0xFFFFu;
  __syncwarp();
  const uint32_t nb = __popc(bm);
  // the barrier before my first basin (fB; the whole chunk if it has no basin), ORD_NONE if none
  const int fi = nb ? __ffs(bm) - 1 : 16;
  const uint32_t mlo = mm & ((1u << fi) - 1);
  const int fj = mlo ? 31 - __clz(mlo) : 0;
  const uint32_t fB = mlo ? ((em >> fj & 1) ? INF_ORD : SO[fj][lane]) : ORD_NONE;
  // basin indices: exclusive warp scan of the per-lane counts
  uint32_t inc = nb;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, inc, d);
    if (lane >= d) inc += y;
  }
  const uint32_t nbw = __shfl_sync(0xFFFFFFFFu, inc, 31);
  const uint32_t idx0 = inc - nb;

  // ---------------- (b) the warp's item list: basin ord K, right barrier R (ORD_NONE if it lies
  // beyond my chunk; a barrier before a lane's first basin closes the previous item's gap),
  // (offset << 16 | basin index) PI
  {
    uint32_t brem = bm, idx = idx0;
    while (brem) {
      const int i = __ffs(brem) - 1;
      brem &= brem - 1;
      const uint32_t mr = mm >> i;
      const int j = mr ? i + __ffs(mr) - 1 : 32;
      const bool mine = j < 16 && (brem == 0 || j < __ffs(brem) - 1);
      B.K[idx] = SO[i][lane];
      B.R[idx] = mine ? ((em >> j & 1) ? INF_ORD : SO[j][lane]) : ORD_NONE;
      B.PI[idx] = (uint32_t(16 * lane + i) << 16) | idx;
      if (G.cell) G.cell[rslot + idx] = 2u * uint32_t(q0 + i);
      ++idx;
    }
  }
  __syncwarp();
  if (fB != ORD_NONE) {
    if (idx0 > 0) atomicMax(&B.R[idx0 - 1], fB);
    else atomicMax(&B.lead, fB);
  }
  if (lane == 0) G.rcnt[rslot / L1_IPW] = nbw;
  __syncwarp();

  // ---------------- (c) quick1 rounds over the warp's items, 32 per step
  uint32_t nn = nbw, holes = 0;
#pragma unroll 1
  for (int round = 0; round < g_l1_rounds && nn > 0; ++round) {
    const uint32_t lead0 = B.lead;
    uint32_t kept = 0, cK = 0, cR = 0;
#pragma unroll 1
    for (uint32_t c0 = 0; c0 < nn; c0 += 32) {
      const uint32_t j = c0 + lane;
      const bool valid = j < nn;
      const uint32_t q = valid ? B.K[j] : 0u, r = valid ? B.R[j] : 0u;
      const uint32_t pi = valid ? B.PI[j] : 0u;
      uint32_t kp = __shfl_up_sync(0xFFFFFFFFu, q, 1), rp = __shfl_up_sync(0xFFFFFFFFu, r, 1);
      if (lane == 0) {
        kp = cK;
        rp = cR;
      }
      uint32_t kn = __shfl_down_sync(0xFFFFFFFFu, q, 1);
      if (lane == 31 && j + 1 < nn) kn = B.K[j + 1];
      cK = __shfl_sync(0xFFFFFFFFu, q, 31);
      cR = __shfl_sync(0xFFFFFFFFu, r, 31);
      const uint32_t bl = j > 0 ? rp : (left_start ? INF_ORD : lead0);
      const uint32_t d = valid ? quick1_ord(q, bl, r, j > 0, kp, j + 1 < nn, kn) : DEATH_PENDING;
      const bool keep = valid && d == DEATH_PENDING;
      if (valid && !keep) holes += stage_put_nh(G, rslot + (pi & 0xFFFFu), q, d);
      const unsigned km = __ballot_sync(0xFFFFFFFFu, keep);
      const uint32_t p = kept + __popc(km & lt);
      __syncwarp();
      if (keep) {
        B.K[p] = q;
        B.R[p] = r;
        B.PI[p] = pi;
      }
      __syncwarp();
      if (valid && !keep && r != ORD_NONE) {
        if (p == 0) atomicMax(&B.lead, r);
        else atomicMax(&B.R[p - 1], r);
      }
      kept += __popc(km);
      __syncwarp();
    }
    const uint32_t dropped = nn - kept;
    nn = kept;
    if (dropped * 8 < nn + 8) break;  // little progress: the tree search decides the rest
  }
  holes = __reduce_add_sync(0xFFFFFFFFu, holes);
  if (lane == 0 && holes) atomicAdd(G.holes + rslot / L1_IPW, holes);
  if (lane == 0) B.n = nn;
  __syncthreads();  // the scratch (aliasing the CTA buffers) is dead from here on

  // ---------------- (d) CTA residual: concatenation of the warps' residuals
  if (threadIdx.x == 0) {
    uint32_t off = 0;
    for (int v = 0; v < L1_WARPS; ++v) {
      s_off[v] = off;
      off += WB[v].n;
    }
    s_off[L1_WARPS] = off;
    s_lead = KEY_NONE;
    if (off > uint32_t(MAXITEMS)) atomicOr(overflow, 1);
  }
  __syncthreads();
  const uint32_t m = s_off[L1_WARPS];
  if (m > uint32_t(MAXITEMS)) return;  // adversarial input: the caller reruns on the tree path
  {
    const uint32_t off = s_off[w];
    for (uint32_t j = lane; j < nn; j += 32) {
      const uint32_t pi = B.PI[j];
      const uint64_t pos = uint64_t(b0 + (pi >> 16));
      const uint32_t r = B.R[j];
      S.T.mn[off + j] = (uint64_t(B.K[j]) << 32) | pos;
      S.T.mx[off + j] = r == ORD_NONE ? KEY_NONE : ((uint64_t(r) << 32) | pos);
      S.id[off + j] = (uint32_t(w) * L1_IPW) | (pi & 0xFFFFu);  // tile-relative slot
    }
  }
  __syncthreads();
  if (lane == 0 && B.lead != ORD_NONE) {  // my lead closes the gap after the previous item
    const uint64_t key = (uint64_t(B.lead) << 32) | uint64_t(b0);
    const uint32_t off = s_off[w];
    if (off > 0) atomicMax(reinterpret_cast<unsigned long long*>(S.T.mx + off - 1), key);
    else atomicMax(reinterpret_cast<unsigned long long*>(&s_lead), key);
  }
  __syncthreads();
  uint64_t ld = s_lead;
  const uint64_t tslot = uint64_t(t) * SLOTS1;
  const int nres = decide_tile(S, int(m), t == 0, ld, [=](uint32_t id, uint64_t key, uint32_t d) {
    stage_put(G, tslot + id, key_ord(key), d);
  });
  __shared__ uint32_t s_npend, s_nexp;  // undecided basins needing the rank pass; all of them
  if (threadIdx.x == 0) s_npend = s_nexp = 0;
  __syncthreads();
  for (int j = threadIdx.x; j < nres; j += THREADS)
    if (s_pend[j >> 5] >> (j & 31) & 1) {
      // an undecided basin's rank among its region's bars is its index unless the region holds
      // holes (zero-persistence basins); those regions are ranked by the pass below
      const uint64_t slot = tslot + S.id[j];
      const bool holes = __ldcg(G.holes + slot / L1_IPW) != 0;
      G.st[slot] = make_uint2(__float_as_uint(float_of_ord(key_ord(S.T.mn[j]))),
                              holes ? BAR_PENDING : (PEND_TAG | uint32_t(slot % L1_IPW)));
      if (holes) atomicAdd(&s_npend, 1u);
      atomicAdd(&s_nexp, 1u);
    }
  __syncthreads();
  if (threadIdx.x == 0 && s_nexp) atomicAdd(G.cnt + 0, (unsigned long long)s_nexp);
  // ---------------- (e) ranks of the undecided basins among the bars of their region
  if (s_npend && __ldcg(G.holes + rslot / L1_IPW)) {  // the loads below go out together
    constexpr int NCH = L1_IPW / 32;
    uint2 v[NCH];
#pragma unroll
    for (int k = 0; k < NCH; ++k) {
      const uint32_t i = 32 * k + lane;
      v[k] = i < nbw ? __ldcg(G.st + rslot + i) : make_uint2(HOLE, 0u);
    }
    uint32_t run = 0;
#pragma unroll
    for (int k = 0; k < NCH; ++k) {
      const unsigned km = __ballot_sync(0xFFFFFFFFu, v[k].x != HOLE);
      if (v[k].x != HOLE && v[k].y == BAR_PENDING)
        G.st[rslot + 32 * k + lane].y = PEND_TAG | (run + __popc(km & lt));
      run += __popc(km);
    }
  }
  __syncthreads();
  if (gridDim.x > 1)
    export_pending(S, nres, ld, O, t, [=](uint32_t id) {
      const uint64_t slot = tslot + id;
      return uint32_t(slot - slot % L1_IPW) | (__ldcg(&G.st[slot].y) & PEND_RANK);
    });
}

// ------------------------------------------------------------------------------------------
// Level k >= 2: tiles of ITILE items over the concatenation of the previous level's regions.
struct LevelIn {
  const uint64_t* key;
  const uint64_t* rb;
  const uint32_t* id;
  const uint32_t* cnt;
  const uint64_t* lead;
  const uint32_t* prefix;  // exclusive prefix of cnt, ntiles + 1 entries
  int ntiles;              // tiles of the previous level
};


// One tile t (of ntiles) of an item level.
__device__ __forceinline__ void level_tile(const LevelIn& I, const Items& O, const Stage& G,
                                           Smem& S, uint32_t t, uint32_t total,
                                           uint32_t ntiles) {
  const int P = I.ntiles;
  const uint32_t k0 = t * ITILE;
  const int n = int(total - k0 < uint32_t(ITILE) ? total - k0 : uint32_t(ITILE));
  // gather items k0..k0+n-1 (and item k0-1's barrier) from the previous level's tile regions;
  // the source tile of item g is the last i with prefix[i] <= g.  The prefix segment covering the
  // tile's items is staged in shared memory (two global searches instead of one per item).
  constexpr int PSEG = 2048;
  __shared__ uint64_t s_lead0;
  __shared__ uint32_t s_pref[PSEG];
  __shared__ int s_plo, s_pn;
  auto src_tile = [&](uint32_t g) {
    int lo = 0, hi = P - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (__ldcg(I.prefix + mid) <= g) lo = mid; else hi = mid - 1;
    }
    return lo;
  };
  // source tiles of the first and last item: one parallel pass over the prefix (a thread owns a
  // run of entries and recognises the boundary i with prefix[i] <= g < prefix[i+1]); no
  // dependent chain of global loads
  __shared__ int s_pa, s_pb;
  {
    const uint32_t ga = k0 > 0 ? k0 - 1 : 0, gb = k0 + uint32_t(n) - 1;
    for (int i = threadIdx.x; i < P; i += THREADS) {
      const uint32_t pi = __ldcg(I.prefix + i);
      const uint32_t pn = i + 1 < P ? __ldcg(I.prefix + i + 1) : 0xFFFFFFFFu;
      if (pi <= ga && ga < pn) s_pa = i;
      if (pi <= gb && gb < pn) s_pb = i;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int a = s_pa, b = s_pb;
    s_plo = a;
    s_pn = b - a + 1 <= PSEG ? b - a + 1 : 0;  // 0: too wide, search globally
  }
  __syncthreads();
  const int plo = s_plo, pn = s_pn;
  for (int i = threadIdx.x; i < pn; i += THREADS) s_pref[i] = __ldcg(I.prefix + plo + i);
  __syncthreads();
  for (int j = int(threadIdx.x) - 1; j < n; j += THREADS) {
    if (j < 0 && k0 == 0) continue;
    const uint32_t g = k0 + j;  // j = -1: the item left of the tile
    int lo;
    if (pn) {
      int l = 0, h = pn - 1;
      while (l < h) {
        const int mid = (l + h + 1) >> 1;
        if (s_pref[mid] <= g) l = mid; else h = mid - 1;
      }
      lo = plo + l;
    } else {
      lo = src_tile(g);
    }
    const uint32_t r = g - I.prefix[lo];
    const uint64_t src = uint64_t(lo) * MAXITEMS + r;
    uint64_t rb = I.rb[src];
    if (r + 1 == I.cnt[lo]) {  // the last item of its tile also spans the following tiles' leads
      for (int q = lo + 1; q < P; ++q) {
        rb = max(rb, I.lead[q]);
        if (I.cnt[q] > 0) break;
      }
    }
    if (j < 0) {
      s_lead0 = rb;
    } else {
      S.T.mn[j] = I.key[src];
      S.T.mx[j] = rb;
      S.id[j] = I.id[src];
    }
  }
  if (k0 == 0 && threadIdx.x == 0) s_lead0 = KEY_NONE;
  __syncthreads();
  tl_mark(ntiles > 1 ? 7 : 12);
  uint64_t ld = s_lead0;
  const int nres = decide_tile(S, n, t == 0, ld, [=](uint32_t id, uint64_t key, uint32_t d) {
    final_put(G, id, key_ord(key), d);
  });
  tl_mark(ntiles > 1 ? 10 : 13);
  if (ntiles > 1) {
    export_pending(S, nres, ld, O, t, [](uint32_t id) { return id; });
    tl_mark(11);
  } else if (threadIdx.x == 0) {
    O.cnt[t] = 0;
    O.lead[t] = KEY_NONE;
  }
  __syncthreads();  // the shared buffers are reused by the CTA's next tile
}

// Item levels and the gather in one cooperative launch.
//  (0) region offsets: every CTA sums the bar counts of its share of the level-1 regions; after a
//      grid sync each CTA scans its share into G.regoff (a second grid sync publishes them);
//  (1) item levels: per level, block 0 scans the previous level's per-tile counts (grid sync),
//      then the CTAs share the level's tiles (grid sync).  A level whose items fit one tile is
//      final: both series ends are known there and every basin is decided;
//  (2) a CTA gathers its share of the regions as soon as it has no level tile to work on, so the
//      gather overlaps the (few-CTA) item levels.
struct LevelsArgs {
  LevelIn in[NLEVELS];     // in[l].ntiles = capacity; the actual count comes from ltiles
  Items out[NLEVELS];
  uint32_t* ltiles;        // [0] level-1 tiles; [l+1] actual tiles of item level l
  int64_t cap_tiles[NLEVELS];
  Stage G;
  int* overflow;
  int levels;              // 0: one level-1 tile (every basin decided there)
  int nreg;                // level-1 regions
  uint32_t* part;          // per CTA: bars in its regions
  uint32_t* part2;         // per CTA: undecided basins in its share of the level-1 tiles
  unsigned long long* total;
  uint32_t* gctr;          // next gather chunk
  unsigned long long* tl;  // debug timeline (null unless CR_DEBUG_STATS)
  uint32_t* done;          // [l]: level l's count scan done (1); [NLEVELS + l]: its tiles done
  uint32_t* exits;         // CTAs that finished (the last one publishes the control head)
  const unsigned long long* ctl;  // control head (flags, counters, total): CTL_PUB words
  unsigned long long* host_ctl;   // pinned host words receiving it (no separate D2H copy)
};
constexpr int CTL_PUB = 6;

// Gather chunks of THREADS/32 regions (one per warp), taken from a global counter, until the
// chunks run out or *until reaches goal (goal 0: no stop condition).  Returns false once exhausted.
__device__ bool gather_until(const LevelsArgs& A, const uint32_t* until, uint32_t goal,
                             uint32_t (*s_bar)[96], uint32_t* s_chunk) {
  const int w = threadIdx.x >> 5;
  const uint32_t nchunks = uint32_t((A.nreg + THREADS / 32 - 1) / (THREADS / 32));
  while (true) {
    if (threadIdx.x == 0) {
      uint32_t c = 0xFFFFFFFFu;
      if (!goal || *reinterpret_cast<const volatile uint32_t*>(until) < goal)
        c = atomicAdd(A.gctr, 1u);
      *s_chunk = c;
    }
    __syncthreads();
    const uint32_t c = *s_chunk;
    __syncthreads();
    if (c == 0xFFFFFFFFu) return true;  // stop condition met
    if (c >= nchunks) return false;
    const int r = int(c) * (THREADS / 32) + w;
    if (r < A.nreg) gather_region(A.G, r, int64_t(__ldcg(A.G.regoff + r)), s_bar[w]);
  }
}

__device__ __forceinline__ void levels_body(const LevelsArgs& A) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char smem[];
  Smem S = carve(smem);
  typedef cub::BlockScan<uint32_t, THREADS> BS;
  __shared__ typename BS::TempStorage s_scan;
  __shared__ uint32_t s_red[THREADS / 32];
  __shared__ uint32_t s_bar[THREADS / 32][96];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  auto stamp = [&](int slot) {  // debug timeline (CR_DEBUG_STATS): block 0's view
    if (A.tl && blockIdx.x == 0 && threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      A.tl[slot] = t;
    }
  };
  stamp(0);
  // ---- (0) two grid-wide scans at once: the level-1 regions' bar counts (output offsets) and,
  // when there are item levels, the level-1 tiles' undecided counts (the first item level's
  // prefix, so that no single CTA scans it later)
  const int per = (A.nreg + int(gridDim.x) - 1) / int(gridDim.x);
  const int r0 = min(A.nreg, int(blockIdx.x) * per), r1 = min(A.nreg, r0 + per);
  const int P0 = A.levels ? int(__ldcg(A.ltiles)) : 0;
  const int per2 = (P0 + int(gridDim.x) - 1) / int(gridDim.x);
  const int t0 = min(P0, int(blockIdx.x) * per2), t1 = min(P0, t0 + per2);
  auto rsz = [&](int r) { return __ldcg(A.G.rcnt + r) - __ldcg(A.G.holes + r); };
  auto tsz = [&](int t) { return __ldcg(A.in[0].cnt + t); };
  auto block_sum = [&](uint32_t v) {  // block-wide sum, returned to every thread
    v = __reduce_add_sync(0xFFFFFFFFu, v);
    __syncthreads();
    if (lane == 0) s_red[w] = v;
    __syncthreads();
    uint32_t t = 0;
    for (int k = 0; k < THREADS / 32; ++k) t += s_red[k];
    return t;
  };
  {
    uint32_t s1 = 0, s2 = 0;
    for (int r = r0 + threadIdx.x; r < r1; r += THREADS) s1 += rsz(r);
    for (int t = t0 + threadIdx.x; t < t1; t += THREADS) s2 += tsz(t);
    s1 = block_sum(s1);
    s2 = block_sum(s2);
    if (threadIdx.x == 0) {
      A.part[blockIdx.x] = s1;
      A.part2[blockIdx.x] = s2;
    }
  }
  grid.sync(); stamp(1);
  {
    uint32_t v1 = 0, v2 = 0;
    for (uint32_t k = threadIdx.x; k < blockIdx.x; k += THREADS) {
      v1 += __ldcg(A.part + k);
      v2 += __ldcg(A.part2 + k);
    }
    uint32_t base = block_sum(v1), base2 = block_sum(v2);
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
      *A.total = base + __ldcg(A.part + blockIdx.x);
      if (A.levels) {  // the first item level's size (what block 0 used to scan)
        const uint32_t run = base2 + __ldcg(A.part2 + blockIdx.x);
        const_cast<uint32_t*>(A.in[0].prefix)[P0] = run;
        const uint32_t nt = (run + ITILE - 1) / ITILE;
        if (int64_t(nt) > A.cap_tiles[0]) {
          atomicOr(A.overflow, 1);
          A.ltiles[1] = 0;
        } else {
          A.ltiles[1] = nt > 1 ? nt : 0;
        }
      }
    }
    for (int c = r0; c < r1; c += THREADS) {
      const int r = c + threadIdx.x;
      const uint32_t sz = r < r1 ? rsz(r) : 0u;
      uint32_t pre, tot;
      __syncthreads();
      BS(s_scan).ExclusiveSum(sz, pre, tot);
      if (r < r1) A.G.regoff[r] = base + pre;
      base += tot;
    }
    uint32_t* pref0 = const_cast<uint32_t*>(A.in[0].prefix);
    for (int c = t0; c < t1; c += THREADS) {
      const int t = c + threadIdx.x;
      const uint32_t sz = t < t1 ? tsz(t) : 0u;
      uint32_t pre, tot;
      __syncthreads();
      BS(s_scan).ExclusiveSum(sz, pre, tot);
      if (t < t1) pref0[t] = base2 + pre;
      base2 += tot;
    }
  }
  grid.sync(); stamp(2);
  // ---- (1) item levels, (2) the gather when idle
  __shared__ uint32_t s_chunk;
  bool more = true;  // gather chunks left
  for (int l = 0; l < NLEVELS && A.levels; ++l) {
    LevelIn I = A.in[l];
    I.ntiles = int(__ldcg(A.ltiles + l));
    uint32_t* pref = const_cast<uint32_t*>(I.prefix);
    if (l > 0) {  // (level 0's prefix comes from phase (0))
      if (blockIdx.x == 0) {
        constexpr int PT = 16;  // counts per thread per pass
        uint32_t run = 0;
        for (int c = 0; c < I.ntiles; c += THREADS * PT) {
          const int i0 = c + threadIdx.x * PT;
          uint32_t v[PT], sum = 0;
#pragma unroll
          for (int r = 0; r < PT; ++r) {
            v[r] = i0 + r < I.ntiles ? __ldcg(I.cnt + i0 + r) : 0u;
            sum += v[r];
          }
          uint32_t pre, tot;
          BS(s_scan).ExclusiveSum(sum, pre, tot);
          pre += run;
#pragma unroll
          for (int r = 0; r < PT; ++r)
            if (i0 + r < I.ntiles) {
              pref[i0 + r] = pre;
              pre += v[r];
            }
          run += tot;
          __syncthreads();
        }
        if (threadIdx.x == 0) {
          pref[I.ntiles] = run;
          const uint32_t nt = (run + ITILE - 1) / ITILE;
          if (int64_t(nt) > A.cap_tiles[l] || (l == NLEVELS - 1 && nt > 1)) {
            atomicOr(A.overflow, 1);
            A.ltiles[l + 1] = 0;
          } else {
            A.ltiles[l + 1] = nt > 1 ? nt : 0;  // a final (single) tile exports nothing
          }
          __threadfence();
          atomicExch(A.done + l, 1u);
        }
      } else if (more) {  // block 0 scans; the others gather meanwhile
        more = gather_until(A, A.done + l, 1u, s_bar, &s_chunk);
      }
      grid.sync();
    }
    stamp(3 + 3 * l);
    if (__ldcg(A.overflow)) return;
    const uint32_t total = __ldcg(pref + I.ntiles);
    const uint32_t ntiles = (total + ITILE - 1) / ITILE;
    if (ntiles == 0) break;
    if (blockIdx.x < ntiles) {
      for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x)
        level_tile(I, A.out[l], A.G, S, t, total, ntiles);
      stamp(4 + 3 * l);
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(A.done + NLEVELS + l, 1u);
      }
    } else if (more && ntiles > 1) {
      more = gather_until(A, A.done + NLEVELS + l, min(ntiles, gridDim.x), s_bar, &s_chunk);
    }
    if (ntiles == 1) break;
    grid.sync(); stamp(5 + 3 * l);
  }
  stamp(14);
  if (more) gather_until(A, nullptr, 0u, s_bar, &s_chunk);
  stamp(15);
}

__global__ void __launch_bounds__(THREADS) k1_levels_coop(LevelsArgs A) {
  levels_body(A);
  // the last CTA out writes the control head straight into pinned host memory: the host's
  // stream sync then reads it without a separate copy
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(A.exits, 1u) == gridDim.x - 1) {
      __threadfence();
#pragma unroll
      for (int i = 0; i < CTL_PUB; ++i) A.host_ctl[i] = __ldcg(A.ctl + i);
      __threadfence_system();
    }
  }
}

__global__ void k1_hole_flags(const cr_pair* __restrict__ in, int64_t n, uint32_t* flag) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) flag[i] = in[i].dim != -1;
  if (i == n) flag[i] = 0;
}
__global__ void k1_hole_compact(const cr_pair* __restrict__ in, const uint32_t* __restrict__ icell,
                                int64_t n, const uint32_t* __restrict__ flag,
                                const uint32_t* __restrict__ pos, cr_pair* __restrict__ out,
                                uint32_t* __restrict__ ocell) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n || !flag[i]) return;
  out[pos[i]] = in[i];
  if (ocell) ocell[pos[i]] = icell[i];
}

}  // namespace

int64_t barcodes_1d_tiles(const float* x, int64_t n, cr_pair* out, uint32_t* out_cells,
                          int64_t cap, Workspace& ws, HostScalars& hs, cr_stats& st) {
  cudaStream_t s = ws.stream();
  const int nt1 = int((n + L1_TILE - 1) / L1_TILE);
  // level sizes (tiles), assuming each level contracts >= 4x (else: overflow -> tree path)
  int64_t tiles[NLEVELS + 1];
  tiles[0] = nt1;
  // grids sized for >= 16x contraction per level (a random walk contracts ~200x per level);
  // weaker contraction sets the overflow flag and the caller reruns on the tree path
  int64_t items = int64_t(nt1) * MAXITEMS / 16;
  for (int l = 1; l <= NLEVELS; ++l) {
    tiles[l] = std::max<int64_t>(1, (items + ITILE - 1) / ITILE);
    items = std::max<int64_t>(ITILE, items / 16);
  }
  ws.use_arena();
  Stage G;
  const int nreg = nt1 * L1_WARPS;
  // control block, zeroed by one memset and read back by one copy:
  //   [0, 2) u64: flags (int nan, int overflow), [2, 6): counters, total bars,
  //   [6, 7 + NLEVELS): gather chunk counter + level flags (u32), then holes per region (u32)
  constexpr int CTL_HEAD = 7 + NLEVELS;
  const size_t ctl_bytes = CTL_HEAD * sizeof(unsigned long long) + (nreg + 1) * sizeof(uint32_t);
  unsigned long long* ctl = static_cast<unsigned long long*>(ws.alloc_bytes(ctl_bytes));
  CR_CUDA(cudaMemsetAsync(ctl, 0, ctl_bytes, s));
  int* flags = reinterpret_cast<int*>(ctl);  // nan, overflow
  unsigned long long* meta = ctl + 2;
  G.holes = reinterpret_cast<uint32_t*>(ctl + CTL_HEAD);
  G.st = ws.alloc<uint2>(int64_t(nreg) * L1_IPW);
  G.cell = out_cells ? ws.alloc<uint32_t>(int64_t(nreg) * L1_IPW) : nullptr;
  G.rcnt = ws.alloc<uint32_t>(nreg + 1);
  Items L[NLEVELS + 1];
  for (int l = 0; l <= NLEVELS; ++l) {
    const int64_t cap_items = tiles[l] * int64_t(MAXITEMS);
    L[l].key = ws.alloc<uint64_t>(cap_items);
    L[l].rb = ws.alloc<uint64_t>(cap_items);
    L[l].id = ws.alloc<uint32_t>(cap_items);
    L[l].cnt = ws.alloc<uint32_t>(tiles[l]);
    L[l].lead = ws.alloc<uint64_t>(tiles[l]);
  }
  // per-device launch facts, cached per host thread
  struct DevFacts {
    bool ok = false;
    int nsm = 0, per_sm = 0;
  };
  static thread_local DevFacts facts[64];
  DevFacts& F = facts[ws.device() & 63];
  if (!F.ok) {
    CR_CUDA(cudaFuncSetAttribute(k1_level1, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(L1_SMEM)));
    CR_CUDA(cudaFuncSetAttribute(k1_levels_coop, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(SMEM)));
    CR_CUDA(cudaDeviceGetAttribute(&F.nsm, cudaDevAttrMultiProcessorCount, ws.device()));
    CR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&F.per_sm, k1_levels_coop, THREADS,
                                                          SMEM));
    if (F.per_sm < 1) throw Error{CR_EINTERNAL, "k1_levels_coop cannot be resident"};
    F.ok = true;
  }
  G.out = out;
  G.out_cells = out_cells;
  G.cap = cap;
  G.cnt = meta;
  G.regoff = ws.alloc<uint32_t>(nreg);
  LevelsArgs LA{};
  LA.ltiles = ws.alloc<uint32_t>(NLEVELS + 2);  // [0] = nt1, written by k1_level1
  G.ltiles0 = LA.ltiles;
  k1_level1<<<nt1, THREADS, L1_SMEM, s>>>(x, n, L[0], G, flags + 0, flags + 1);
  CR_CHECK_LAUNCH();
  prof_mark(s, "1d_level1");
  for (int l = 1; l <= NLEVELS; ++l) {
    uint32_t* prefix = nt1 > 1 ? ws.alloc<uint32_t>(tiles[l - 1] + 1) : nullptr;
    LA.in[l - 1] = LevelIn{L[l - 1].key, L[l - 1].rb, L[l - 1].id, L[l - 1].cnt, L[l - 1].lead,
                           prefix, int(tiles[l - 1])};
    LA.out[l - 1] = L[l];
    LA.cap_tiles[l - 1] = tiles[l];
  }
  LA.G = G;
  LA.overflow = flags + 1;
  LA.levels = nt1 > 1;
  LA.nreg = nreg;
  LA.total = meta + 3;
  LA.gctr = reinterpret_cast<uint32_t*>(ctl + 6);
  LA.done = LA.gctr + 1;  // 2 * NLEVELS words, then the exit counter, up to the holes
  LA.exits = LA.done + 2 * NLEVELS;
  static_assert(1 + 2 * NLEVELS + 1 <= 2 * (CTL_HEAD - 6), "control words fit the head");
  LA.ctl = ctl;
  LA.host_ctl = hs.p;
  // item levels are small (a random walk leaves ~0.5 % of basins undecided per tile); the gather
  // streams every bar: a few CTAs per SM keep enough loads in flight
  const int64_t blocks = std::max<int64_t>(
      1, std::min<int64_t>(int64_t(F.nsm) * std::min(F.per_sm, 2), (nreg + 7) / 8));
  LA.part = ws.alloc<uint32_t>(blocks);
  LA.part2 = ws.alloc<uint32_t>(blocks);
  LA.tl = nullptr;
  {
    unsigned long long* gt = nullptr;
    if (opt(OPT_DEBUG)) {
      LA.tl = ws.alloc<unsigned long long>(32);
      CR_CUDA(cudaMemsetAsync(LA.tl, 0, 32 * sizeof(unsigned long long), s));
      gt = LA.tl + 16;
    }
    static thread_local bool tl_set[64] = {};  // g_tl is non-null on this device
    if (gt || tl_set[ws.device() & 63]) {       // no per-call copy in the common case
      CR_CUDA(cudaMemcpyToSymbolAsync(g_tl, &gt, sizeof(gt), 0, cudaMemcpyHostToDevice, s));
      tl_set[ws.device() & 63] = gt != nullptr;
    }
  }
  void* args[] = {&LA};
  CR_CUDA(cudaLaunchCooperativeKernel((void*)k1_levels_coop, dim3(unsigned(blocks)),
                                      dim3(THREADS), args, SMEM, s));
  ++g_launch_count;
  prof_mark(s, "1d_levels_gather");
  CR_CUDA(cudaStreamSynchronize(s));  // k1_levels_coop wrote ctl[0, CTL_PUB) into hs.p
  const int* hf = reinterpret_cast<const int*>(hs.p);
  const unsigned long long exported = hs.p[2], decided = hs.p[3], late_holes = hs.p[4];
  int64_t total = int64_t(hs.p[5]);
  if (opt(OPT_DEBUG) && nt1 > 1) {
    uint32_t lt[NLEVELS + 2];
    CR_CUDA(cudaMemcpy(lt, LA.ltiles, sizeof(lt), cudaMemcpyDeviceToHost));
    fprintf(stderr, "[cr] 1d tiles per level:");
    for (int l = 0; l <= NLEVELS; ++l) fprintf(stderr, " %u", lt[l]);
    fprintf(stderr, " | undecided after level 1: %llu, later holes %llu\n", exported, late_holes);
    unsigned long long tl[32];
    CR_CUDA(cudaMemcpy(tl, LA.tl, sizeof(tl), cudaMemcpyDeviceToHost));
    fprintf(stderr, "[cr] coop timeline (us since start, block 0):");
    for (int q = 1; q < 16; ++q)
      if (tl[q]) fprintf(stderr, " [%d]%.1f", q, (tl[q] - tl[0]) / 1000.0);
    for (int q = 16; q < 32; ++q)
      if (tl[q]) fprintf(stderr, " t%d:%.1f", q - 16, (tl[q] - tl[0]) / 1000.0);
    fprintf(stderr, "\n");
  }
  if (hf[0]) throw Error{CR_EINVAL, "NaN in image"};
  if (hf[1] || exported != decided) return -1;  // contraction did not finish (adversarial)
  if (late_holes) {
    // rare: basins undecided at level 1 that turned out zero-length left holes; compact
    const int64_t m = std::min<int64_t>(total, cap);
    cr_pair* tmp = ws.alloc<cr_pair>(m + 1);
    uint32_t* tcell = out_cells ? ws.alloc<uint32_t>(m + 1) : nullptr;
    uint32_t* flag = ws.alloc<uint32_t>(m + 1);
    uint32_t* pos = ws.alloc<uint32_t>(m + 1);
    CR_CUDA(cudaMemcpyAsync(tmp, out, m * sizeof(cr_pair), cudaMemcpyDeviceToDevice, s));
    if (tcell)
      CR_CUDA(cudaMemcpyAsync(tcell, out_cells, m * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
    k1_hole_flags<<<grid_for(m + 1, 256), 256, 0, s>>>(tmp, m, flag);
    CR_CHECK_LAUNCH();
    exclusive_sum_u32(flag, pos, m + 1, ws);
    k1_hole_compact<<<grid_for(m, 256), 256, 0, s>>>(tmp, tcell, m, flag, pos, out, out_cells);
    CR_CHECK_LAUNCH();
    if (total <= cap) total -= int64_t(late_holes);  // else: an upper bound forces a retry
  }
  st.pairs[0] = total;
  return total;
}

}  // namespace cr
