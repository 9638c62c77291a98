// batched.cu -- K7: the whole pipeline for one small 2D image per CTA, in shared memory
// (batches of MNIST-like images, BASELINE config 3).  Same mathematics and the same total order as
// the device-wide path (general.cu / reduce.cu), so both give identical pairings:
//   births -> apparent pairs -> H0 by union-find with the elder rule over the
//   residual edges in key order -> dimension-1 coboundary reduction with clearing over
//   the residual, uncleared edges in decreasing key order -> bars in (dim, birth kidx)
//   order into a per-image staging region.
// Each image is independent, so a CTA never waits for another; a final gather copies the staged
// bars to the output at the scanned per-image offsets.  Images that do not fit (reduced-column
// pool overflow) are flagged and the caller recomputes the batch on the device-wide path.
#include <cub/cub.cuh>

#include <algorithm>
#include <type_traits>

#include "pipeline.cuh"

namespace cr {
namespace {

constexpr int K7_THREADS = 256;
constexpr int K7_IPT = 8;
constexpr int K7_SORT = K7_THREADS * K7_IPT;  // 2048 keys
constexpr int K7_RADIX = 5;  // digit bits of the block radix sort (44-bit keys: 9 passes; 6+ bits
                              // would not leave room for 4 CTAs per SM)
constexpr int K7_MAXCELLS = 3072;  // Khalimsky cells per image (28x28 -> 3025)
constexpr int K7_MAXVOX = 1024;
constexpr int K7_POOL = 1024;  // stored reduced columns (u64 keys)
constexpr int K7_WORK = 256;   // working column capacity (ping-pong)
constexpr uint32_t D_NONE = 0xFFFFFFFFu, D_ZERO = 0xFFFFFFFEu, D_ESS = 0xFFFFFFFDu;

struct K7Args {
  const float* images;
  int64_t batch;
  int ny, nx;
  int maxdim;
  uint32_t* sbar;   // staging: 3 words per bar, cap per image
  uint32_t* scell;  // staging: birth kidx (optional)
  uint32_t* count;  // bars per image
  int cap;          // bars per image region
  int* flags;       // [0] NaN, [1] overflow
  int dual;         // dimension 1 by Alexander duality (union-find over squares); else reduction
};

// Per-CTA shared memory.  DUAL (dimension 1 by duality, the default): no reduction buffers and no
// sort, so 4 CTAs fit an SM.  The union holds, in turn: the codes (step 2), the union-find
// candidates with their per-root minima (steps 3, 4), the scan (step 5), the sort (reduction).
struct K7Red {
  uint16_t owner[K7_MAXCELLS];
  uint64_t pool[K7_POOL];
  uint64_t work[2][K7_WORK];
  uint16_t pool_off[K7_MAXCELLS / 2];
  uint16_t pool_len[K7_MAXCELLS / 2];
};
struct K7Empty {};
template <bool DUAL>
constexpr int k7_cand() { return DUAL ? 1536 : K7_SORT; }  // union-find candidates per image
template <bool DUAL>
struct K7Smem {
  uint32_t ord[K7_MAXVOX + 1];  // voxel ords; later the dual parents (OMEGA = nvox <= MAXVOX)
  uint32_t births[K7_MAXCELLS];
  uint32_t death[K7_MAXCELLS];
  uint16_t vpar[K7_MAXVOX];
  uint8_t tags[K7_MAXCELLS];
  typename std::conditional<DUAL, K7Empty, K7Red>::type red;
  union {  // the keys are held in registers while the sort uses its temporary storage
    typename std::conditional<
        DUAL, K7Empty,
        typename cub::BlockRadixSort<uint64_t, K7_THREADS, K7_IPT, cub::NullType,
                                     K7_RADIX>::TempStorage>::type sort;
    typename cub::BlockScan<uint32_t, K7_THREADS>::TempStorage scan;
    struct {
      uint64_t keys[k7_cand<DUAL>()];  // candidates (compact keys), unsorted
      uint64_t best[K7_MAXVOX + 1];    // per root: the minimum (H0) / maximum (dual) candidate
    };
  } tmp;
  uint32_t nkeys;
  uint32_t changed;
  uint32_t nbars;
};

template <class SM>
__device__ __forceinline__ uint64_t cellkey(const SM& S, uint32_t k) {
  return make_key(S.births[k], k);
}
// compact sort key (ord << 12 | kidx): the same order as cellkey on <= 4096 cells, 44 bits
constexpr int K7_KBITS = 12, K7_SORT_BITS = 32 + K7_KBITS;
static_assert(K7_MAXCELLS <= (1 << K7_KBITS), "kidx field");
template <class SM>
__device__ __forceinline__ uint64_t sortkey(const SM& S, uint32_t k) {
  return (uint64_t(S.births[k]) << K7_KBITS) | k;
}
__device__ __forceinline__ uint32_t sortcell(uint64_t key) {
  return uint32_t(key & ((1u << K7_KBITS) - 1));
}

// sort S.tmp.keys[0..n) ascending (descending if desc) in place, on the compact key's 44 bits
template <class SM>
__device__ void k7_sort(SM& S, uint32_t n, bool desc) {
  uint64_t it[K7_IPT];
#pragma unroll
  for (int r = 0; r < K7_IPT; ++r) {
    const uint32_t i = threadIdx.x * K7_IPT + r;
    it[r] = i < n ? S.tmp.keys[i] : (desc ? 0ull : (1ull << K7_SORT_BITS) - 1);
  }
  __syncthreads();
  typedef cub::BlockRadixSort<uint64_t, K7_THREADS, K7_IPT, cub::NullType, K7_RADIX> BRS;
  if (desc) BRS(S.tmp.sort).SortDescending(it, 0, K7_SORT_BITS);
  else BRS(S.tmp.sort).Sort(it, 0, K7_SORT_BITS);
  __syncthreads();
#pragma unroll
  for (int r = 0; r < K7_IPT; ++r) {
    const uint32_t i = threadIdx.x * K7_IPT + r;
    if (i < n) S.tmp.keys[i] = it[r];
  }
  __syncthreads();
}

__device__ __forceinline__ uint32_t k7_find(uint16_t* par, uint32_t x) {
  while (par[x] != x) {
    par[x] = par[par[x]];
    x = par[x];
  }
  return x;
}

// C = A xor B (sorted arrays), one thread
__device__ uint32_t k7_symdiff(const uint64_t* A, uint32_t a, const uint64_t* B, uint32_t b,
                               uint64_t* C) {
  uint32_t i = 0, j = 0, n = 0;
  while (i < a && j < b) {
    const uint64_t x = A[i], y = B[j];
    if (x < y) { C[n++] = x; ++i; }
    else if (y < x) { C[n++] = y; ++j; }
    else { ++i; ++j; }
  }
  while (i < a) C[n++] = A[i++];
  while (j < b) C[n++] = B[j++];
  return n;
}


// Code of a 2D cell k with parities (OX, OY) (the rule of k_filtration): the first equal-birth
// cofacet in kidx order (-Y < -X < +X < +Y) and the last equal-birth facet; h*: the neighbour in
// that direction is inside the grid (facets of a present cell always are).
template <bool OX, bool OY, class SM>
__device__ __forceinline__ uint32_t k7_code(const SM& S, int k, int KX, bool hxm, bool hxp,
                                            bool hym, bool hyp) {
  const uint32_t b = S.births[k];
  if (b == ABSENT_ORD) return 0x40;
  const uint32_t ym = hym ? S.births[k - KX] : ABSENT_ORD;
  const uint32_t xm = hxm ? S.births[k - 1] : ABSENT_ORD;
  const uint32_t xp = hxp ? S.births[k + 1] : ABSENT_ORD;
  const uint32_t yp = hyp ? S.births[k + KX] : ABSENT_ORD;
  uint32_t mc = 7, mf = 7;
  if (!OY && yp == b) mc = 3;
  if (!OX && xp == b) mc = 1;
  if (!OX && xm == b) mc = 0;
  if (!OY && ym == b) mc = 2;
  if (OY && ym == b) mf = 2;
  if (OX && xm == b) mf = 0;
  if (OX && xp == b) mf = 1;
  if (OY && yp == b) mf = 3;
  return mc | (mf << 3);
}

// Persistent CTAs: CTA b takes images b, b + gridDim.x, ...
template <bool DUAL>
__global__ void __launch_bounds__(K7_THREADS, 4) k7_image(K7Args A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  K7Smem<DUAL>& S = *reinterpret_cast<K7Smem<DUAL>*>(smem_raw);
  const int nx = A.nx, ny = A.ny, nvox = nx * ny;
  const int KX = 2 * nx - 1, KY = 2 * ny - 1, N = KX * KY;
  constexpr int KC = k7_cand<DUAL>() / K7_THREADS;  // candidate slots per thread
  // exact quotient by KX (operands < 2^12) with one multiply-high
  const uint64_t mKX = ((1ull << 32) + KX - 1) / KX;
  auto dKX = [&](int c) { return int((uint64_t(uint32_t(c)) * mKX) >> 32); };
  const uint64_t mNX = ((1ull << 32) + nx - 1) / nx;
  auto dNX = [&](int v) { return int((uint64_t(uint32_t(v)) * mNX) >> 32); };
  auto vox = [&](int c) {  // base voxel of cell c
    const int Y = dKX(c);
    return (Y >> 1) * nx + ((c - Y * KX) >> 1);
  };
  for (int64_t img = blockIdx.x; img < A.batch; img += gridDim.x) {
  // ---- 1. ords, births
  bool nan = false;
  for (int v = threadIdx.x; v < nvox; v += K7_THREADS) {
    const float f = __ldg(A.images + img * nvox + v);
    nan |= f != f;
    S.ord[v] = ord_of(f);
  }
  if (nan) atomicOr(A.flags, 1);
  __syncthreads();
  // per voxel (x, y): its vertex and the edges / square toward x+1, y+1
  for (int v = threadIdx.x; v < nvox; v += K7_THREADS) {
    const int y = dNX(v), x = v - y * nx;
    const bool hx = x + 1 < nx, hy = y + 1 < ny;
    const uint32_t a = S.ord[v], ax = hx ? S.ord[v + 1] : 0u, ay = hy ? S.ord[v + nx] : 0u,
                   axy = (hx && hy) ? S.ord[v + nx + 1] : 0u;
    const int k = 2 * y * KX + 2 * x;
    S.births[k] = a;
    S.death[k] = D_NONE;
    if (hx) {
      S.births[k + 1] = max(a, ax);
      S.death[k + 1] = D_NONE;
    }
    if (hy) {
      S.births[k + KX] = max(a, ay);
      S.death[k + KX] = D_NONE;
      if (hx) {
        S.births[k + KX + 1] = max(max(a, ax), max(ay, axy));
        S.death[k + KX + 1] = D_NONE;
      }
    }
  }
  if constexpr (!DUAL)
    for (int k = threadIdx.x; k < N; k += K7_THREADS) S.red.owner[k] = 0xFFFFu;
  __syncthreads();
  // ---- 2. apparent pairs, as in general.cu's k_filtration: a code per cell
  // (direction of the first equal-birth cofacet, of the last equal-birth facet, in kidx order
  // -Y(2) < -X(0) < +X(1) < +Y(3); 7 = none; reading R17), then UP iff the min cofacet's max
  // facet points back, else DOWN iff the max facet's min cofacet points back.  The codes use the
  // sort buffer (free until the H0 sort).
  uint8_t* code = reinterpret_cast<uint8_t*>(S.tmp.keys);
  // per voxel: its vertex, edges toward x+1 / y+1 and square (static parities, no division)
  for (int v = threadIdx.x; v < nvox; v += K7_THREADS) {
    const int y = dNX(v), x = v - y * nx, k = 2 * y * KX + 2 * x;
    const bool hx = x + 1 < nx, hy = y + 1 < ny, lx = x > 0, ly = y > 0;
    code[k] = uint8_t(k7_code<false, false>(S, k, KX, lx, hx, ly, hy));
    if (hx) code[k + 1] = uint8_t(k7_code<true, false>(S, k + 1, KX, true, true, ly, hy));
    if (hy) {
      code[k + KX] = uint8_t(k7_code<false, true>(S, k + KX, KX, lx, hx, true, true));
      if (hx) code[k + KX + 1] = uint8_t(k7_code<true, true>(S, k + KX + 1, KX, true, true, true, true));
    }
  }
  __syncthreads();
  auto tag_at = [&](int k) {
    const uint32_t c = code[k];
    uint8_t tag = 0;
    if (!(c & 0x40)) {
      const uint32_t mc = c & 7, mf = (c >> 3) & 7;
      auto nbk = [&](uint32_t d) { return k + ((d >> 1) ? KX : 1) * ((d & 1) ? 1 : -1); };
      if (mc != 7 && ((code[nbk(mc)] >> 3) & 7) == (mc ^ 1)) tag = make_tag(KIND_UP, int(mc));
      else if (mf != 7 && (code[nbk(mf)] & 7) == (mf ^ 1)) tag = make_tag(KIND_DOWN, int(mf));
    }
    S.tags[k] = tag;
  };
  for (int v = threadIdx.x; v < nvox; v += K7_THREADS) {
    const int y = dNX(v), x = v - y * nx, k = 2 * y * KX + 2 * x;
    const bool hx = x + 1 < nx, hy = y + 1 < ny;
    tag_at(k);
    if (hx) tag_at(k + 1);
    if (hy) {
      tag_at(k + KX);
      if (hx) tag_at(k + KX + 1);
    }
  }
  __syncthreads();
  // ---- 3. H0: apparent forest, roots, residual edges in key order, elder-rule union-find
  for (int v = threadIdx.x; v < nvox; v += K7_THREADS) {
    const int x = v % nx, y = v / nx, k = 2 * y * KX + 2 * x;
    uint32_t p = v;
    const uint8_t t = S.tags[k];
    if (S.births[k] != ABSENT_ORD && tag_kind(t) == KIND_UP) {
      const int d = tag_dir(t);
      const int vs = (d >> 1) == 0 ? 1 : nx;
      p = (d & 1) ? v + vs : v - vs;
    }
    S.vpar[v] = uint16_t(p);
  }
  if (threadIdx.x == 0) S.nkeys = 0;
  __syncthreads();
  // (no flattening pass: the roots below come from finds with path halving)
  // residual edges joining different basins, enumerated per voxel: (v, v+1) and (v, v+nx)
  for (int v = threadIdx.x; v < nvox; v += K7_THREADS) {
    const int y = dNX(v), x = v - y * nx, kv = 2 * y * KX + 2 * x;
#pragma unroll
    for (int o = 0; o < 2; ++o) {
      if (o == 0 ? x + 1 >= nx : y + 1 >= ny) continue;
      const int k = kv + (o == 0 ? 1 : KX), vb = v + (o == 0 ? 1 : nx);
      if (S.births[k] == ABSENT_ORD || tag_kind(S.tags[k]) != KIND_RESIDUAL) continue;
      if (k7_find(S.vpar, v) != k7_find(S.vpar, vb)) {
        const uint32_t q = atomicAdd(&S.nkeys, 1u);
        if (q < uint32_t(k7_cand<DUAL>())) S.tmp.keys[q] = sortkey(S, k);
      }
    }
  }
  __syncthreads();
  const uint32_t nc = S.nkeys;
  if (nc > uint32_t(k7_cand<DUAL>())) {  // adversarial image: the stacked path takes the batch
    if (threadIdx.x == 0) atomicOr(A.flags + 1, 1);
    continue;
  }
  // Elder-rule Kruskal over the candidates as block-wide merge rounds (the rule of general.cu's
  // k_mm_rounds: an edge commits when it is the minimum candidate at both of its components, or
  // at the younger one alone -- the merges of the sequential Kruskal loop, with no sort: the
  // per-root minima are taken on the compact keys).  Thread t owns candidates t + 256 r.
  {
    // per-root extremum of round `rnd`, round-tagged so that no reset phase is needed:
    // (rnd << 44) | (~key & mask44) under atomicMax = the minimum key of the newest round
    uint64_t* best = S.tmp.best;
    for (int v = threadIdx.x; v < nvox; v += K7_THREADS) best[v] = 0;
    constexpr uint64_t KM = (1ull << K7_SORT_BITS) - 1;
    uint64_t rnd = 0;
    uint32_t alive = 0;  // bit r: candidate t + 256 r undecided
#pragma unroll
    for (int r = 0; r < KC; ++r)
      if (threadIdx.x + K7_THREADS * r < int(nc)) alive |= 1u << r;
    uint16_t ra[KC], rb[KC];
    __syncthreads();
    while (true) {
      bool any = false;
#pragma unroll
      for (int r = 0; r < KC; ++r) {
        if (!(alive >> r & 1)) continue;
        const uint32_t i = threadIdx.x + K7_THREADS * r;
        const uint64_t key = S.tmp.keys[i];
        const uint32_t k = sortcell(key);
        const int s1 = ((int(k) - dKX(int(k)) * KX) & 1) ? 1 : KX;
        const int a = int(k) - s1, b = int(k) + s1;
        const uint32_t va = vox(a), vb = vox(b);
        const uint32_t x = k7_find(S.vpar, va), y = k7_find(S.vpar, vb);
        if (x == y) {  // positive edge: closes a cycle of older edges
          alive &= ~(1u << r);
          continue;
        }
        ra[r] = uint16_t(x);
        rb[r] = uint16_t(y);
        any = true;
        const unsigned long long tk = (rnd << K7_SORT_BITS) | (~key & KM);
        atomicMax((unsigned long long*)(best + x), tk);
        atomicMax((unsigned long long*)(best + y), tk);
      }
      if (!__syncthreads_or(any)) break;
#pragma unroll
      for (int r = 0; r < KC; ++r) {
        if (!(alive >> r & 1)) continue;
        const uint32_t i = threadIdx.x + K7_THREADS * r;
        const uint64_t key = S.tmp.keys[i];
        const uint32_t x = ra[r], y = rb[r];
        const uint64_t tk = (rnd << K7_SORT_BITS) | (~key & KM);
        const bool min_a = best[x] == tk, min_b = best[y] == tk;
        if (!min_a && !min_b) continue;
        const uint32_t kxa = 2 * (x / nx) * KX + 2 * (x % nx), kxb = 2 * (y / nx) * KX + 2 * (y % nx);
        const bool a_young = cellkey(S, kxa) > cellkey(S, kxb);
        if (!(min_a && min_b) && (a_young ? !min_a : !min_b)) continue;
        const uint32_t young = a_young ? x : y, old = a_young ? y : x;
        const uint32_t ky = a_young ? kxa : kxb;
        const uint32_t k = sortcell(key);
        S.vpar[young] = uint16_t(old);  // elder rule
        S.death[ky] = S.births[k] > S.births[ky] ? S.births[k] : D_ZERO;
        S.tags[k] = make_tag(KIND_CLEARED, 0);
        alive &= ~(1u << r);
      }
      ++rnd;
      __syncthreads();
    }
  }
  for (int v = threadIdx.x; v < nvox; v += K7_THREADS) {
    const int k = 2 * (v / nx) * KX + 2 * (v % nx);
    if (S.vpar[v] == v && S.births[k] != ABSENT_ORD) S.death[k] = D_ESS;
  }
  // ---- 4. dimension 1: residual, uncleared edges in decreasing key order
  const bool do_d1 = A.maxdim >= 1 && nx > 1 && ny > 1;
  if (threadIdx.x == 0) S.nkeys = 0;
  __syncthreads();
  if (DUAL && do_d1) {
    // dimension 1 = the top dimension of a 2D image, by Alexander duality (the
    // same construction as general.cu's top_dual): squares and the outside OMEGA are the vertices,
    // residual edges in decreasing key the edges, the root with the larger key survives.  Dual
    // parents live in S.ord (the voxel ords are dead after step 1).
    uint32_t* dp = S.ord;
    const uint32_t OMEGA = uint32_t(nvox);
    auto sq_of = [&](uint32_t v) -> uint32_t {  // square with base voxel v
      return (2 * (v / nx) + 1) * KX + 2 * (v % nx) + 1;
    };
    auto side = [&](int e, int sg) -> uint32_t {  // dual vertex on side sg of edge e
      const int Y = dKX(e), X = e - Y * KX;
      int q;
      if (X & 1) {  // horizontal edge: squares above/below
        if (sg ? Y + 1 >= KY : Y == 0) return OMEGA;
        q = e + (sg ? KX : -KX);
      } else {
        if (sg ? X + 1 >= KX : X == 0) return OMEGA;
        q = e + (sg ? 1 : -1);
      }
      return uint32_t(vox(q));
    };
    for (int v = threadIdx.x; v <= nvox; v += K7_THREADS) {
      uint32_t p = uint32_t(v);
      if (v < nvox && (v % nx) + 1 < nx && (v / nx) + 1 < ny) {
        const uint32_t k = sq_of(uint32_t(v));
        const uint8_t t = S.tags[k];
        if (S.births[k] != ABSENT_ORD && tag_kind(t) == KIND_DOWN) {
          const int d = tag_dir(t), off = (d >> 1) == 0 ? 1 : KX;
          p = side(int(k) + ((d & 1) ? off : -off), d & 1);
        }
      }
      dp[v] = p;
    }
    __syncthreads();
    auto dfind = [&](uint32_t x) {
      while (true) {
        const uint32_t q = *(volatile uint32_t*)(dp + x);
        if (q == x) return x;
        const uint32_t qq = *(volatile uint32_t*)(dp + q);
        if (qq != q) atomicCAS(dp + x, q, qq);
        x = qq;
      }
    };
    // edges enumerated per voxel: (v, v+1) and (v, v+nx)
    for (int v = threadIdx.x; v < nvox; v += K7_THREADS) {  // absent faces join absent sides
      const int y = dNX(v), x = v - y * nx, kv = 2 * y * KX + 2 * x;
      for (int o = 0; o < 2; ++o) {
        if (o == 0 ? x + 1 >= nx : y + 1 >= ny) continue;
        const int k = kv + (o == 0 ? 1 : KX);
        if (S.births[k] != ABSENT_ORD) continue;
        uint32_t a = side(k, 0), b = side(k, 1);
        while (true) {
          a = dfind(a);
          b = dfind(b);
          if (a == b) break;
          if (a > b) { const uint32_t t = a; a = b; b = t; }
          if (atomicCAS(dp + a, a, b) == a) break;
        }
      }
    }
    __syncthreads();
    for (int v = threadIdx.x; v < nvox; v += K7_THREADS) {  // residual edges between components
      const int y = dNX(v), x = v - y * nx, kv = 2 * y * KX + 2 * x;
#pragma unroll
      for (int o = 0; o < 2; ++o) {
        if (o == 0 ? x + 1 >= nx : y + 1 >= ny) continue;
        const int k = kv + (o == 0 ? 1 : KX);
        if (S.births[k] == ABSENT_ORD || tag_kind(S.tags[k]) != KIND_RESIDUAL) continue;
        if (dfind(side(k, 0)) != dfind(side(k, 1))) {
          const uint32_t q = atomicAdd(&S.nkeys, 1u);
          if (q < uint32_t(k7_cand<DUAL>())) S.tmp.keys[q] = sortkey(S, k);
        }
      }
    }
    __syncthreads();
    const uint32_t nc = S.nkeys;
    if (nc > uint32_t(k7_cand<DUAL>())) {
      if (threadIdx.x == 0) atomicOr(A.flags + 1, 1);
      continue;
    }
    // Kruskal over the dual edges in decreasing key order as block-wide merge rounds, the mirror
    // of the H0 rounds above: the per-root extremum is the MAXIMUM candidate key, and the root
    // with the larger key survives.
    {
      auto rkey = [&](uint32_t v) -> uint64_t {
        return v == OMEGA ? NONE64 : cellkey(S, sq_of(v));
      };
      uint64_t* best = S.tmp.best;  // dual vertices 0..nvox (OMEGA = nvox <= K7_MAXVOX)
      for (int v = threadIdx.x; v <= nvox; v += K7_THREADS) best[v] = 0;
      uint64_t rnd = 0;  // round-tagged maxima: (rnd << 44) | key, no reset phase
      uint32_t alive = 0;
#pragma unroll
      for (int r = 0; r < KC; ++r)
        if (threadIdx.x + K7_THREADS * r < int(nc)) alive |= 1u << r;
      uint32_t ra[KC], rb[KC];
      __syncthreads();
      while (true) {
        bool any = false;
#pragma unroll
        for (int r = 0; r < KC; ++r) {
          if (!(alive >> r & 1)) continue;
          const uint32_t i = threadIdx.x + K7_THREADS * r;
          const uint64_t key = S.tmp.keys[i];
          const uint32_t e = sortcell(key);
          const uint32_t x = dfind(side(int(e), 0)), y = dfind(side(int(e), 1));
          if (x == y) {  // closes a cycle (a death of dimension 0)
            alive &= ~(1u << r);
            continue;
          }
          ra[r] = x;
          rb[r] = y;
          any = true;
          const unsigned long long tk = (rnd << K7_SORT_BITS) | key;
          atomicMax((unsigned long long*)(best + x), tk);
          atomicMax((unsigned long long*)(best + y), tk);
        }
        if (!__syncthreads_or(any)) break;
#pragma unroll
        for (int r = 0; r < KC; ++r) {
          if (!(alive >> r & 1)) continue;
          const uint32_t i = threadIdx.x + K7_THREADS * r;
          const uint64_t key = S.tmp.keys[i];
          const uint32_t x = ra[r], y = rb[r];
          const uint64_t tk = (rnd << K7_SORT_BITS) | key;
          const bool min_a = best[x] == tk, min_b = best[y] == tk;
          if (!min_a && !min_b) continue;
          const uint64_t ka = rkey(x), kb = rkey(y);
          const bool a_young = ka < kb;
          if (!(min_a && min_b) && (a_young ? !min_a : !min_b)) continue;
          const uint32_t young = a_young ? x : y, old = a_young ? y : x;
          const uint64_t ky = a_young ? ka : kb;
          const uint32_t e = sortcell(key);
          dp[young] = old;
          if (key_ord(ky) == ABSENT_ORD) {
            S.death[e] = D_ESS;  // two absent regions meet: a hole that never fills
          } else {
            const uint32_t by = key_ord(ky);
            S.death[e] = by > S.births[e] ? by : D_ZERO;
          }
          alive &= ~(1u << r);
        }
        ++rnd;
        __syncthreads();
      }
    }
  } else if (do_d1) {
   if constexpr (!DUAL) {
    auto& R = S.red;
    for (int k = threadIdx.x; k < N; k += K7_THREADS) {
      const int Y = dKX(k), X = k - Y * KX;
      if (((X & 1) + (Y & 1)) == 1 && S.births[k] != ABSENT_ORD &&
          tag_kind(S.tags[k]) == KIND_RESIDUAL)
        S.tmp.keys[atomicAdd(&S.nkeys, 1u)] = sortkey(S, k);
    }
    __syncthreads();
    const uint32_t ncol = S.nkeys;
    k7_sort(S, ncol, true);
    if (threadIdx.x == 0) {
      uint32_t ptop = 0;
      bool overflow = false;
      for (uint32_t ci = 0; ci < ncol && !overflow; ++ci) {
        const uint32_t sk = sortcell(S.tmp.keys[ci]);
        // coboundary: the finite squares on both sides of the edge
        auto cob = [&](uint32_t e, uint64_t* dst) -> uint32_t {
          const int Y = dKX(e), X = e - Y * KX;
          uint32_t n = 0;
          uint64_t c0 = NONE64, c1 = NONE64;
          if (X & 1) {  // horizontal edge: squares above and below
            if (Y > 0 && S.births[e - KX] != ABSENT_ORD) c0 = cellkey(S, e - KX);
            if (Y + 1 < KY && S.births[e + KX] != ABSENT_ORD) c1 = cellkey(S, e + KX);
          } else {
            if (X > 0 && S.births[e - 1] != ABSENT_ORD) c0 = cellkey(S, e - 1);
            if (X + 1 < KX && S.births[e + 1] != ABSENT_ORD) c1 = cellkey(S, e + 1);
          }
          if (c0 > c1) { const uint64_t t = c0; c0 = c1; c1 = t; }
          if (c0 != NONE64) dst[n++] = c0;
          if (c1 != NONE64) dst[n++] = c1;
          return n;
        };
        int cur = 0;
        uint32_t len = cob(sk, R.work[0]);
        uint64_t tmpc[2];
        while (true) {
          if (len == 0) {
            S.death[sk] = D_ESS;
            break;
          }
          const uint64_t p = R.work[cur][0];
          const uint32_t pk = key_kidx(p);
          const uint8_t t = S.tags[pk];
          const uint64_t* add;
          uint32_t alen;
          if (tag_kind(t) == KIND_DOWN) {
            const int d = tag_dir(t);
            const int off = (d >> 1) == 0 ? 1 : KX;
            alen = cob(uint32_t(int(pk) + ((d & 1) ? off : -off)), tmpc);
            add = tmpc;
          } else if (R.owner[pk] != 0xFFFFu) {
            const uint32_t o = R.owner[pk];
            add = R.pool + R.pool_off[o];
            alen = R.pool_len[o];
          } else {  // new pair (edge, square): bar [birth edge, birth square)
            if (ptop + len > K7_POOL || ci >= K7_MAXCELLS / 2) {
              overflow = true;
              break;
            }
            for (uint32_t i = 0; i < len; ++i) R.pool[ptop + i] = R.work[cur][i];
            R.pool_off[ci] = uint16_t(ptop);
            R.pool_len[ci] = uint16_t(len);
            ptop += len;
            R.owner[pk] = uint16_t(ci);
            S.death[sk] = S.births[pk] > S.births[sk] ? S.births[pk] : D_ZERO;
            break;
          }
          if (len + alen > K7_WORK) {
            overflow = true;
            break;
          }
          len = k7_symdiff(R.work[cur], len, add, alen, R.work[cur ^ 1]);
          cur ^= 1;
        }
      }
      if (overflow) atomicOr(A.flags + 1, 1);
    }
   }
  }
  __syncthreads();
  // ---- 5. bars in (dim, birth kidx) order: vertices, then edges.  Thread t owns the cells
  // [CPT t, CPT t + CPT); one block scan of its packed (dim-0 | dim-1 << 16) counts places them.
  typedef cub::BlockScan<uint32_t, K7_THREADS> BS;
  constexpr int CPT = (K7_MAXCELLS + K7_THREADS - 1) / K7_THREADS;
  const int64_t base = img * A.cap;
  const int dmx = do_d1 ? 1 : 0;
  const int k0 = threadIdx.x * CPT;
  uint32_t keepm = 0, cnt = 0;
#pragma unroll
  for (int q = 0; q < CPT; ++q) {
    const int k = k0 + q;
    if (k >= N) break;
    const int Y = dKX(k), X = k - Y * KX, dim = (X & 1) + (Y & 1);
    const uint32_t d = S.death[k];
    if (dim <= dmx && d != D_NONE && d != D_ZERO) {
      keepm |= 1u << q;
      cnt += 1u << (16 * dim);
    }
  }
  uint32_t pre, tot;
  BS(S.tmp.scan).ExclusiveSum(cnt, pre, tot);
  const uint32_t tot0 = tot & 0xFFFFu, nb = (tot & 0xFFFFu) + (tot >> 16);
  uint32_t o0 = pre & 0xFFFFu, o1 = tot0 + (pre >> 16);
#pragma unroll
  for (int q = 0; q < CPT; ++q) {
    if (!(keepm >> q & 1)) continue;
    const int k = k0 + q;
    const int Yk = dKX(k), dim = ((k - Yk * KX) & 1) + (Yk & 1);
    const uint32_t o = dim ? o1++ : o0++;
    if (int(o) < A.cap) {
      const uint32_t d = S.death[k];
      uint32_t* w = A.sbar + 3 * (base + o);
      w[0] = uint32_t(dim);
      w[1] = __float_as_uint(float_of_ord(S.births[k]));
      w[2] = d == D_ESS ? 0x7F800000u : __float_as_uint(float_of_ord(d));
      if (A.scell) A.scell[base + o] = uint32_t(k);
    }
  }
  if (threadIdx.x == 0) {
    if (int(nb) > A.cap) atomicOr(A.flags + 1, 1);
    A.count[img] = nb;
  }
  __syncthreads();  // S is reused by the next image
  }
  asm volatile("cp.async.wait_group 0;\n" ::);
}

__global__ void k7_gather(const uint32_t* __restrict__ sbar, const uint32_t* __restrict__ scell,
                          const uint32_t* __restrict__ count, const int64_t* __restrict__ off,
                          int cap, int64_t out_cap, cr_pair* out, uint32_t* cells) {
  const int64_t img = blockIdx.x;
  const uint32_t n = count[img];
  const int64_t o0 = off[img];
  const uint32_t* src = sbar + 3 * img * cap;
  uint32_t* dst = reinterpret_cast<uint32_t*>(out + o0);
  const int64_t lim = out_cap - o0;
  const uint32_t nw = lim <= 0 ? 0u : (int64_t(n) < lim ? n : uint32_t(lim));
  for (uint32_t i = threadIdx.x; i < 3 * nw; i += blockDim.x) dst[i] = src[i];
  if (cells)
    for (uint32_t i = threadIdx.x; i < nw; i += blockDim.x) cells[o0 + i] = scell[img * cap + i];
}

__global__ void __launch_bounds__(1024) k7_offsets(const uint32_t* __restrict__ count, int64_t batch, int64_t* off) {
  // single block exclusive scan over batch counts (int64)
  typedef cub::BlockScan<int64_t, 1024> BS;
  __shared__ typename BS::TempStorage tmp;
  int64_t run = 0;
  for (int64_t c = 0; c < batch; c += 1024) {
    const int64_t i = c + threadIdx.x;
    const int64_t v = i < batch ? int64_t(count[i]) : 0;
    int64_t pre, tot;
    BS(tmp).ExclusiveSum(v, pre, tot);
    if (i < batch) off[i] = run + pre;
    run += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) off[batch] = run;
}

}  // namespace

bool batched_small_2d_fits(int64_t ny, int64_t nx) {
  return nx * ny <= K7_MAXVOX && (2 * nx - 1) * (2 * ny - 1) <= K7_MAXCELLS &&
         (2 * nx - 1) * (2 * ny - 1) <= 65535;
}

// Returns -1 if some image did not fit the per-CTA buffers (caller falls back).
int64_t barcodes_batched_small_2d(const float* images, int64_t batch, int64_t ny, int64_t nx,
                                  int maxdim, cr_pair* out, uint32_t* out_cells, int64_t cap,
                                  int64_t* out_offsets, Workspace& ws, HostScalars& hs,
                                  cr_stats& st) {
  cudaStream_t s = ws.stream();
  const int cells = int((2 * nx - 1) * (2 * ny - 1));
  const int vox = int(nx * ny);
  // bars per image <= vertices + edges
  const int per = int(std::min<int64_t>(cells, vox + (nx - 1) * ny + nx * (ny - 1)));
  K7Args A;
  A.images = images;
  A.batch = batch;
  A.ny = int(ny);
  A.nx = int(nx);
  A.maxdim = maxdim;
  A.dual = opt(OPT_TOP_REDUCE) == 0;
  A.cap = per;
  A.sbar = ws.alloc<uint32_t>(batch * int64_t(per) * 3);
  A.scell = out_cells ? ws.alloc<uint32_t>(batch * int64_t(per)) : nullptr;
  A.count = ws.alloc<uint32_t>(batch + 1);
  A.flags = ws.alloc<int>(4);
  CR_CUDA(cudaMemsetAsync(A.flags, 0, 4 * sizeof(int), s));
  const bool dual = A.dual && nx > 1 && ny > 1 && vox + 1 <= K7_MAXVOX;
  auto launch = [&](auto kern, size_t smem) {
    CR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    int dev = 0, nsm = 0, per_sm = 0;
    CR_CUDA(cudaGetDevice(&dev));
    CR_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    CR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, K7_THREADS, smem));
    if (per_sm < 1) per_sm = 1;
    const int64_t grid = std::min<int64_t>(batch, int64_t(nsm) * per_sm);
    kern<<<unsigned(grid), K7_THREADS, smem, s>>>(A);
  };
  if (dual) launch(k7_image<true>, sizeof(K7Smem<true>));
  else launch(k7_image<false>, sizeof(K7Smem<false>));
  CR_CHECK_LAUNCH();
  prof_mark(s, "k7_images");
  k7_offsets<<<1, 1024, 0, s>>>(A.count, batch, out_offsets);
  CR_CHECK_LAUNCH();
  CR_CUDA(cudaMemcpyAsync(hs.p, A.flags, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
  CR_CUDA(cudaMemcpyAsync(hs.p + 1, out_offsets + batch, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  CR_CUDA(cudaStreamSynchronize(s));
  const int* hf = reinterpret_cast<const int*>(hs.p);
  if (hf[0]) throw Error{CR_EINVAL, "NaN in image"};
  if (hf[1]) return -1;
  const int64_t total = int64_t(hs.p[1]);
  k7_gather<<<unsigned(batch), 128, 0, s>>>(A.sbar, A.scell, A.count, out_offsets, per, cap, out,
                                            out_cells);
  CR_CHECK_LAUNCH();
  prof_mark(s, "k7_gather");
  st.pairs[0] = total;
  return total;
}

}  // namespace cr
