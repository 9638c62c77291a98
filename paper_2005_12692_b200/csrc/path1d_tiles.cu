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

#ifndef CR_1D_TILE
#define CR_1D_TILE 2048
#endif
constexpr int TILE = CR_1D_TILE;        // samples per level-1 tile
constexpr int ITILE = TILE / 2;         // items per level-k tile
constexpr int THREADS = TILE / 8;
constexpr int VPT = TILE / THREADS;
constexpr int MAXITEMS = TILE / 2;  // basins in a level-1 tile (no two adjacent); == ITILE
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


// quick decision (O(1)): an item whose lower adjacent barrier leads to an older neighbour dies there
// when the other adjacent barrier is higher (the other side's bottleneck is at least that barrier).
// Generalised to a bounded outward scan: both sides advance one item per step, each keeping the
// highest barrier crossed (a lower bound of its bottleneck, exact once an older basin is met or an
// infinite barrier is crossed).  The item is decided as soon as one side is exact and lower than
// the other side's bound.  Returns DEATH_PENDING if both sides run out of tile undecided, and
// DEATH_RETRY if the step budget ends first (the tree search then decides).
constexpr uint32_t DEATH_RETRY = 0xFFFFFFFDu;
__device__ int g_scan_steps = 1;  // outward scan budget (tunable: CR_1D_SCAN; 1 measured best)
__device__ int g_rounds = 1;      // contraction rounds before the tree (tunable: CR_1D_ROUNDS)
__device__ int g_dbg = 0;         // phase-skipping mask for timing experiments (CR_1D_DBG)

__device__ __forceinline__ uint32_t decide_quick(const STree& T, int j, bool left_start,
                                                 uint64_t lead) {
  const uint64_t q = T.mn[j];
  const int n = T.n;
  uint64_t aL = KEY_NONE, aR = T.mx[j];
  int pL = j - 1, pR = j + 1;
  bool xL = false, xR = key_ord(aR) == INF_ORD;  // exact?
  bool doneL = false, doneR = xR;                // stopped scanning?
  if (xR) aR = INF_KEY;
  const int budget = g_scan_steps;
  for (int step = 0; step < budget; ++step) {
    if (!doneL) {
      if (pL < 0) {  // out of tile on the left
        doneL = true;
        aL = max(aL, lead);
        if (left_start || key_ord(aL) == INF_ORD) { xL = true; aL = INF_KEY; }
      } else {
        aL = max(aL, T.mx[pL]);
        if (key_ord(aL) == INF_ORD) { xL = doneL = true; aL = INF_KEY; }
        else if (T.mn[pL] < q) { xL = doneL = true; }
        else --pL;
      }
    }
    if (!doneR) {
      if (pR >= n) {
        doneR = true;
      } else if (T.mn[pR] < q) {
        xR = doneR = true;
      } else {
        aR = max(aR, T.mx[pR]);
        if (key_ord(aR) == INF_ORD) { xR = doneR = true; aR = INF_KEY; }
        else ++pR;
      }
    }
    if (xL && (xR || aR > aL)) {
      const uint64_t d = xR ? min(aL, aR) : aL;
      return d == INF_KEY ? DEATH_ESSENTIAL : key_ord(d);
    }
    if (xR && aL > aR) return aR == INF_KEY ? DEATH_ESSENTIAL : key_ord(aR);
    if (doneL && doneR) return DEATH_PENDING;
  }
  return DEATH_RETRY;
}

// ------------------------------------------------------------------------------------------
// Per-tile regions.  Level-1 tile t owns staging slots [t*MAXITEMS, (t+1)*MAXITEMS) for its output
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
  uint32_t* bar;      // 3 words per slot: dim, birth, death (float bits); dim = -1: hole
  uint32_t* cell;     // birth kidx per slot (optional)
  uint32_t* ncand;    // per level-1 tile
  uint32_t* holes;    // per level-1 tile: zero-persistence undecided basins found later
};

constexpr uint32_t BAR_PENDING = 0x7FC00001u;  // NaN payload marking an undecided death

__device__ __forceinline__ void stage_death(const Stage& G, uint32_t id, uint32_t birth_ord,
                                            uint32_t d) {
  if (d == DEATH_ESSENTIAL) {
    G.bar[3 * id + 2] = 0x7F800000u;
  } else if (d > birth_ord) {
    G.bar[3 * id + 2] = __float_as_uint(float_of_ord(d));
  } else {  // zero persistence: becomes a hole
    G.bar[3 * id + 0] = 0xFFFFFFFFu;
    atomicAdd(G.holes + id / MAXITEMS, 1u);
  }
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
  stree_layout(S.T, n);
  stree_build(S.T);
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
__global__ void __launch_bounds__(THREADS) k1_level1(const float* __restrict__ x, int64_t n,
                                                     Items O, Stage G, int* nan_flag) {
  extern __shared__ __align__(16) unsigned char smem[];
  Smem S = carve(smem);
  uint32_t* s_ord = reinterpret_cast<uint32_t*>(S.T.mx);  // aliases the mx tree while loading
  __shared__ uint32_t s_minpos, s_maxpos;
  __shared__ uint64_t s_lead;
  typedef cub::BlockScan<uint32_t, THREADS> BS;
  __shared__ typename BS::TempStorage s_scan1;
  if (threadIdx.x == 0) {
    s_minpos = 0xFFFFFFFFu;
    s_maxpos = 0;
    s_lead = KEY_NONE;
  }
  const uint32_t t = blockIdx.x;
  const int64_t a = int64_t(t) * TILE;
  // ---- 1. ords of samples [a-1, a+TILE]
  bool nan = false;
  {
    const int64_t body = (n - a < int64_t(TILE)) ? n - a : int64_t(TILE);
    if (body == TILE && (reinterpret_cast<uintptr_t>(x + a) & 15) == 0) {
      const float4* x4 = reinterpret_cast<const float4*>(x + a);
      for (int q = threadIdx.x; q < TILE / 4; q += THREADS) {
        const float4 v = __ldcs(x4 + q);
        nan |= (v.x != v.x) | (v.y != v.y) | (v.z != v.z) | (v.w != v.w);
        s_ord[1 + 4 * q] = ord_of(v.x);
        s_ord[2 + 4 * q] = ord_of(v.y);
        s_ord[3 + 4 * q] = ord_of(v.z);
        s_ord[4 + 4 * q] = ord_of(v.w);
      }
    } else {
      for (int q = threadIdx.x; q < TILE; q += THREADS) {
        uint32_t o = ABSENT_ORD;
        if (q < body) {
          const float v = x[a + q];
          nan |= v != v;
          o = ord_of(v);
        }
        s_ord[1 + q] = o;
      }
    }
    if (threadIdx.x == 0) s_ord[0] = a >= 1 ? ord_of(x[a - 1]) : ABSENT_ORD;
    if (threadIdx.x == 1) s_ord[TILE + 1] = a + TILE < n ? ord_of(x[a + TILE]) : ABSENT_ORD;
  }
  if (nan) atomicOr(nan_flag, 1);
  __syncthreads();
  // ---- 2. events of my VPT consecutive samples (registers until the ords are dead)
  const int v0 = threadIdx.x * VPT;
  uint32_t bmask = 0, mmask = 0;
  uint32_t bo[VPT], mo[VPT];
#pragma unroll
  for (int r = 0; r < VPT; ++r) {
    const int q = v0 + r;
    const uint32_t um = s_ord[q], u0 = s_ord[q + 1], u1 = s_ord[q + 2];
    bo[r] = u0;
    mo[r] = INF_ORD;
    if (u0 == ABSENT_ORD || a + q >= n) continue;
    if (um > u0 && u1 >= u0) bmask |= 1u << r;
    if (u1 == ABSENT_ORD) {
      mmask |= 1u << r;  // a finite run ends after this sample
    } else if (u1 < u0 && um != ABSENT_ORD && um <= u0) {
      mmask |= 1u << r;  // peak edge (q, q+1)
      mo[r] = u0;
    }
  }
  uint32_t bpre, mpre, NB, NM;
  {
    const uint32_t packed = (uint32_t(__popc(bmask)) << 16) | uint32_t(__popc(mmask));
    uint32_t pre, tot;
    BS(s_scan1).ExclusiveSum(packed, pre, tot);
    bpre = pre >> 16;
    mpre = pre & 0xFFFF;
    NB = tot >> 16;
    NM = tot & 0xFFFF;
  }
  if (bmask | mmask) {
    const int fb = bmask ? __ffs(bmask) - 1 : 99, fm = mmask ? __ffs(mmask) - 1 : 99;
    const uint32_t first = fb <= fm ? 2 * (v0 + fb) : 2 * (v0 + fm) + 1;
    const int lb = bmask ? 31 - __clz(bmask) : -1, lm = mmask ? 31 - __clz(mmask) : -1;
    const uint32_t last = lm >= lb ? 2 * (v0 + lm) + 1 : 2 * (v0 + lb);
    atomicMin(&s_minpos, first);
    atomicMax(&s_maxpos, last + 1);
  }
  __syncthreads();  // the ords are dead from here on
  const int lead = (NB + NM > 0) && (s_minpos & 1);
  const int open_end = (NB + NM > 0) && !((s_maxpos - 1) & 1);
  stree_layout(S.T, int(NB));
  {
    uint32_t bi = bpre, mi = mpre;
#pragma unroll
    for (int r = 0; r < VPT; ++r) {
      const uint32_t q = uint32_t(a + v0 + r);
      if (bmask >> r & 1) S.T.mn[bi++] = make_key(bo[r], q);
      if (mmask >> r & 1) {
        const uint64_t key = make_key(mo[r], q);
        if (lead && mi == 0) s_lead = key;
        else S.T.mx[mi - lead] = key;
        ++mi;
      }
    }
  }
  __syncthreads();
  if (open_end && threadIdx.x == 0) S.T.mx[NB - 1] = KEY_NONE;  // its right barrier is beyond
  for (int j = threadIdx.x; j < int(NB); j += THREADS) {
    S.id[j] = j;
    S.okey[j] = S.T.mn[j];
    S.death[j] = DEATH_PENDING;
  }
  __syncthreads();
  uint64_t ld = s_lead;
  const int dbg = g_dbg;  // timing experiments only (CR_1D_DBG); 0 in production
  const int nres = (dbg & 1) ? 0 : decide_tile(S, int(NB), t == 0, ld,
                               [=](uint32_t id, uint64_t, uint32_t d) { S.death[id] = d; });
  if (dbg & 8) return;
  // ---- 3. staging: candidates (bar or undecided) get consecutive slots in basin order
  {
    constexpr int CH = MAXITEMS / THREADS;
    const int c0 = threadIdx.x * CH;
    uint32_t mine = 0;
#pragma unroll
    for (int r = 0; r < CH; ++r) {
      const int j = c0 + r;
      if (j < int(NB)) {
        const uint32_t d = S.death[j];
        mine += d == DEATH_PENDING || d == DEATH_ESSENTIAL || d > key_ord(S.okey[j]);
      }
    }
    uint32_t pre, tot;
    __syncthreads();
    BS(s_scan1).ExclusiveSum(mine, pre, tot);
    const uint64_t sb = uint64_t(t) * MAXITEMS;
#pragma unroll
    for (int r = 0; r < CH; ++r) {
      const int j = c0 + r;
      if (j >= int(NB)) continue;
      const uint32_t d = S.death[j];
      const uint32_t bord = key_ord(S.okey[j]);
      if (!(d == DEATH_PENDING || d == DEATH_ESSENTIAL || d > bord)) continue;
      S.keep[j] = pre;
      const uint64_t o = sb + pre;
      if (dbg & 2) { ++pre; continue; }
      G.bar[3 * o + 0] = 0u;
      G.bar[3 * o + 1] = __float_as_uint(float_of_ord(bord));
      G.bar[3 * o + 2] = d == DEATH_PENDING ? BAR_PENDING
                                            : (d == DEATH_ESSENTIAL ? 0x7F800000u
                                                                    : __float_as_uint(float_of_ord(d)));
      if (G.cell) G.cell[o] = 2u * key_kidx(S.okey[j]);
      ++pre;
    }
    if (threadIdx.x == 0) G.ncand[t] = tot;
    __syncthreads();
  }
  if (gridDim.x > 1 && !(dbg & 4))
    export_pending(S, nres, ld, O, t,
                   [=](uint32_t j) { return uint32_t(t) * MAXITEMS + S.keep[j]; });
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

// exclusive prefix of a level's per-tile counts (one CTA; the tile counts are small)
__global__ void __launch_bounds__(1024) k1_level_prefix(const uint32_t* cnt, int P,
                                                        uint32_t* prefix) {
  typedef cub::BlockScan<uint32_t, 1024> BS;
  __shared__ typename BS::TempStorage s_scan;
  uint32_t run = 0;
  for (int c = 0; c < P; c += 1024) {
    const int i = c + threadIdx.x;
    const uint32_t v = i < P ? cnt[i] : 0u;
    uint32_t pre, tot;
    BS(s_scan).ExclusiveSum(v, pre, tot);
    if (i < P) prefix[i] = run + pre;
    run += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) prefix[P] = run;
}

// One tile t (of ntiles) of an item level.
__device__ __forceinline__ void level_tile(const LevelIn& I, const Items& O, const Stage& G,
                                           Smem& S, uint32_t t, uint32_t total,
                                           uint32_t ntiles) {
  const int P = I.ntiles;
  const uint32_t k0 = t * ITILE;
  const int n = int(total - k0 < uint32_t(ITILE) ? total - k0 : uint32_t(ITILE));
  // gather items k0..k0+n-1 (and item k0-1's barrier) from the previous level's tile regions
  __shared__ uint64_t s_lead0;
  for (int j = int(threadIdx.x) - 1; j < n; j += THREADS) {
    if (j < 0 && k0 == 0) continue;
    const uint32_t g = k0 + j;  // j = -1: the item left of the tile
    int lo = 0, hi = P - 1;     // source tile: last i with prefix[i] <= g
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (I.prefix[mid] <= g) lo = mid; else hi = mid - 1;
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
  uint64_t ld = s_lead0;
  const int nres = decide_tile(S, n, t == 0, ld, [=](uint32_t id, uint64_t key, uint32_t d) {
    stage_death(G, id, key_ord(key), d);
  });
  if (ntiles > 1) {
    export_pending(S, nres, ld, O, t, [](uint32_t id) { return id; });
  } else if (threadIdx.x == 0) {
    O.cnt[t] = 0;
    O.lead[t] = KEY_NONE;
  }
  __syncthreads();  // the shared buffers are reused by the CTA's next tile
}

// All item levels in one cooperative launch: per level, block 0 scans the previous level's
// per-tile counts (grid sync), then the CTAs share the level's tiles (grid sync).  A level whose
// items fit one tile is final: both series ends are known there and every basin is decided.
struct LevelsArgs {
  LevelIn in[NLEVELS];     // in[l].ntiles = capacity; the actual count comes from ltiles
  Items out[NLEVELS];
  uint32_t* ltiles;        // [0] level-1 tiles; [l+1] actual tiles of item level l
  int64_t cap_tiles[NLEVELS];
  Stage G;
  int* overflow;
};

__global__ void __launch_bounds__(THREADS) k1_levels_coop(LevelsArgs A) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char smem[];
  Smem S = carve(smem);
  typedef cub::BlockScan<uint32_t, THREADS> BS;
  __shared__ typename BS::TempStorage s_scan;
  for (int l = 0; l < NLEVELS; ++l) {
    LevelIn I = A.in[l];
    I.ntiles = int(__ldcg(A.ltiles + l));
    uint32_t* pref = const_cast<uint32_t*>(I.prefix);
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
      }
    }
    grid.sync();
    if (__ldcg(A.overflow)) return;
    const uint32_t total = __ldcg(pref + I.ntiles);
    const uint32_t ntiles = (total + ITILE - 1) / ITILE;
    if (ntiles == 0) return;
    for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x)
      level_tile(I, A.out[l], A.G, S, t, total, ntiles);
    if (ntiles == 1) return;
    grid.sync();
  }
}

// ------------------------------------------------------------------------------------------
// Gather: per level-1 tile, copy its candidates (minus holes) to the output.
__global__ void k1_tile_sizes(const uint32_t* ncand, const uint32_t* holes, int nt,
                              uint32_t* sizes) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nt) sizes[i] = ncand[i] - holes[i];
  if (i == nt) sizes[i] = 0;
}

__global__ void __launch_bounds__(256) k1_gather(Stage G, const uint32_t* __restrict__ off,
                                                 int64_t cap, cr_pair* __restrict__ out,
                                                 uint32_t* __restrict__ cells, int* bad) {
  typedef cub::BlockScan<uint32_t, 256> BS;
  __shared__ typename BS::TempStorage s_scan;
  __shared__ uint32_t s_run;
  const uint32_t t = blockIdx.x;
  const uint32_t nc = G.ncand[t];
  const uint64_t sb = uint64_t(t) * MAXITEMS;
  const uint64_t o0 = off[t];
  if (G.holes[t] == 0) {
    const int64_t lim = cap - int64_t(o0);
    const uint32_t nw = lim <= 0 ? 0u : (int64_t(nc) < lim ? nc : uint32_t(lim));
    const uint32_t* src = G.bar + 3 * sb;
    uint32_t* dst = reinterpret_cast<uint32_t*>(out + o0);
    for (uint32_t i = threadIdx.x; i < 3 * nw; i += 256) {
      const uint32_t v = src[i];
      if (v == BAR_PENDING) atomicOr(bad, 1);
      dst[i] = v;
    }
    if (cells)
      for (uint32_t i = threadIdx.x; i < nw; i += 256) cells[o0 + i] = G.cell[sb + i];
    return;
  }
  // rare: some undecided basins turned out zero-length; compact
  if (threadIdx.x == 0) s_run = 0;
  __syncthreads();
  for (uint32_t c = 0; c < nc; c += 256) {
    const uint32_t i = c + threadIdx.x;
    const bool keep = i < nc && G.bar[3 * (sb + i)] != 0xFFFFFFFFu;
    uint32_t pre, tot;
    BS(s_scan).ExclusiveSum(uint32_t(keep), pre, tot);
    if (keep) {
      const uint64_t o = o0 + s_run + pre;
      if (int64_t(o) < cap) {
        uint32_t* d = reinterpret_cast<uint32_t*>(out + o);
        d[0] = G.bar[3 * (sb + i)];
        d[1] = G.bar[3 * (sb + i) + 1];
        d[2] = G.bar[3 * (sb + i) + 2];
        if (d[2] == BAR_PENDING) atomicOr(bad, 1);
        if (cells) cells[o] = G.cell[sb + i];
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) s_run += tot;
    __syncthreads();
  }
}

}  // namespace

int64_t barcodes_1d_tiles(const float* x, int64_t n, cr_pair* out, uint32_t* out_cells,
                          int64_t cap, Workspace& ws, HostScalars& hs, cr_stats& st) {
  cudaStream_t s = ws.stream();
  const int nt1 = int((n + TILE - 1) / TILE);
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
  int* flags = ws.alloc<int>(4);  // nan, overflow, bad
  CR_CUDA(cudaMemsetAsync(flags, 0, 4 * sizeof(int), s));
  Stage G;
  G.bar = ws.alloc<uint32_t>(int64_t(nt1) * MAXITEMS * 3);
  G.cell = out_cells ? ws.alloc<uint32_t>(int64_t(nt1) * MAXITEMS) : nullptr;
  G.ncand = ws.alloc<uint32_t>(nt1 + 1);
  G.holes = ws.alloc<uint32_t>(nt1 + 1);
  CR_CUDA(cudaMemsetAsync(G.holes, 0, (nt1 + 1) * sizeof(uint32_t), s));
  Items L[NLEVELS + 1];
  for (int l = 0; l <= NLEVELS; ++l) {
    const int64_t cap_items = tiles[l] * int64_t(MAXITEMS);
    L[l].key = ws.alloc<uint64_t>(cap_items);
    L[l].rb = ws.alloc<uint64_t>(cap_items);
    L[l].id = ws.alloc<uint32_t>(cap_items);
    L[l].cnt = ws.alloc<uint32_t>(tiles[l]);
    L[l].lead = ws.alloc<uint64_t>(tiles[l]);
  }
  CR_CUDA(cudaFuncSetAttribute(k1_level1, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM)));
  CR_CUDA(cudaFuncSetAttribute(k1_levels_coop, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               int(SMEM)));
  if (const char* e = std::getenv("CR_1D_SCAN")) {  // tuning knob (not part of the ABI)
    const int v = std::atoi(e);
    CR_CUDA(cudaMemcpyToSymbolAsync(g_scan_steps, &v, sizeof(int), 0, cudaMemcpyHostToDevice, s));
  }
  {
    const char* e = std::getenv("CR_1D_DBG");  // timing experiments only: skips phases
    const int v = e ? std::atoi(e) : 0;
    CR_CUDA(cudaMemcpyToSymbolAsync(g_dbg, &v, sizeof(int), 0, cudaMemcpyHostToDevice, s));
  }
  if (const char* e = std::getenv("CR_1D_ROUNDS")) {  // tuning knob (not part of the ABI)
    const int v = std::atoi(e);
    CR_CUDA(cudaMemcpyToSymbolAsync(g_rounds, &v, sizeof(int), 0, cudaMemcpyHostToDevice, s));
  }
  k1_level1<<<nt1, THREADS, SMEM, s>>>(x, n, L[0], G, flags + 0);
  CR_CHECK_LAUNCH();
  prof_mark(s, "1d_level1");
  if (nt1 > 1) {
    LevelsArgs LA{};
    for (int l = 1; l <= NLEVELS; ++l) {
      uint32_t* prefix = ws.alloc<uint32_t>(tiles[l - 1] + 1);
      LA.in[l - 1] = LevelIn{L[l - 1].key, L[l - 1].rb, L[l - 1].id, L[l - 1].cnt, L[l - 1].lead,
                             prefix, int(tiles[l - 1])};
      LA.out[l - 1] = L[l];
      LA.cap_tiles[l - 1] = tiles[l];
    }
    LA.ltiles = ws.alloc<uint32_t>(NLEVELS + 2);
    const uint32_t nt1u = uint32_t(nt1);
    CR_CUDA(cudaMemcpyAsync(LA.ltiles, &nt1u, sizeof(uint32_t), cudaMemcpyHostToDevice, s));
    LA.G = G;
    LA.overflow = flags + 1;
    int dev = 0, nsm = 0, per_sm = 0;
    CR_CUDA(cudaGetDevice(&dev));
    CR_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    CR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k1_levels_coop, THREADS, SMEM));
    if (per_sm < 1) throw Error{CR_EINTERNAL, "k1_levels_coop cannot be resident"};
    // item levels are small (a random walk leaves < 1 % of basins undecided per tile): one CTA
    // per SM keeps the grid syncs cheap; CTAs loop over tiles if there are more
    const int64_t blocks = std::min<int64_t>(int64_t(nsm), std::max<int64_t>(1, tiles[1]));
    void* args[] = {&LA};
    CR_CUDA(cudaLaunchCooperativeKernel((void*)k1_levels_coop, dim3(unsigned(blocks)),
                                        dim3(THREADS), args, SMEM, s));
    ++g_launch_count;
  }
  prof_mark(s, "1d_levels");
  uint32_t* sizes = ws.alloc<uint32_t>(nt1 + 1);
  uint32_t* off = ws.alloc<uint32_t>(nt1 + 1);
  k1_tile_sizes<<<grid_for(nt1 + 1, 256), 256, 0, s>>>(G.ncand, G.holes, nt1, sizes);
  CR_CHECK_LAUNCH();
  exclusive_sum_u32(sizes, off, nt1 + 1, ws);
  k1_gather<<<nt1, 256, 0, s>>>(G, off, cap, out, out_cells, flags + 2);
  CR_CHECK_LAUNCH();
  prof_mark(s, "1d_gather");
  CR_CUDA(cudaMemcpyAsync(hs.p, flags, 4 * sizeof(int), cudaMemcpyDeviceToHost, s));
  CR_CUDA(cudaMemcpyAsync(reinterpret_cast<uint32_t*>(hs.p) + 4, off + nt1, sizeof(uint32_t),
                          cudaMemcpyDeviceToHost, s));
  CR_CUDA(cudaStreamSynchronize(s));
  const int* hf = reinterpret_cast<const int*>(hs.p);
  if (hf[0]) throw Error{CR_EINVAL, "NaN in image"};
  if (hf[1] || hf[2]) return -1;  // contraction did not finish (adversarial input)
  const int64_t total = reinterpret_cast<const uint32_t*>(hs.p)[4];
  st.pairs[0] = total;
  return total;
}

}  // namespace cr
