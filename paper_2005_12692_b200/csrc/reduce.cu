// reduce.cu -- K5: residual coboundary column reduction of dimension d >= 1.
//
// Columns are the finite d-cells that are neither apparent (K2) nor cleared (death cells of
// dimension d-1), processed in DECREASING key order (the paper's order of
// d-cells, "larger birth-time come first", with ties by kidx, reading R1).
// A column is the coboundary delta(s) -- the finite cofacets of s -- kept as a sorted list of
// (d+1)-cell keys; its pivot is the minimum key (the earliest coface).  While the pivot is owned,
// the owner's column is added over Z/2 (symmetric difference):
//   - owner is apparent (the pivot t is the upper cell of an apparent pair (s', t)) -> add delta(s')
//     enumerated on the fly (the implicit coboundary of PAPER.md:135-136);
//   - owner is an earlier committed column -> add its stored reduced column.
// A nonzero column with an unowned pivot t gives the pair (s, t): bar [birth s, birth t)
// (PAPER.md:138-140); a zero column gives an essential class.
//
// Parallel schedule (one persistent cooperative kernel, one warp per window position): the
// window holds the W columns lo..lo+W-1 (lo = first unfinished).  Each round every warp advances
// its column by at most max_steps additions, publishing its current pivot cand(j) (a lower bound
// of the final pivot: adding a column with the same pivot only moves the pivot later).  Column j
// with an unowned pivot commits iff cand(j) < min{cand(i) : i < j unfinished}: no earlier column
// can end on that pivot, so j's pivot is final, and any column committed while j is unfinished has
// a pivot j can never reach -- the sequential reduction's pairs are reproduced exactly.
#include <cooperative_groups.h>

#include <cub/cub.cuh>

#include "pipeline.cuh"

namespace cg = cooperative_groups;

namespace cr {
namespace {

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
  uint64_t* work;
  uint32_t work_cap;
  uint32_t* slot_col;
  uint32_t* slot_len;
  uint32_t* slot_flags;  // bit0: current buffer, bit1: finished
  uint64_t* cand;
  uint64_t* blockmin;
  unsigned* lo_buf;
  uint64_t* rec;
  unsigned long long* nrec;
  int* err;
  int max_steps;
  unsigned long long* stats;  // [0] rounds, [1] additions
};

constexpr int WARPS_PER_BLOCK = 8;
constexpr int THREADS = WARPS_PER_BLOCK * 32;

__device__ __forceinline__ uint64_t ldcg64(const uint64_t* p) { return __ldcg((const unsigned long long*)p); }

// Finite cofacets of cell s, sorted ascending, written to dst (<= 6 entries).  Warp-collective.
__device__ uint32_t coboundary(const RP& P, uint32_t s, uint64_t* dst, int lane) {
  const Geom& g = P.g;
  uint32_t KX = uint32_t(g.KX), KY = uint32_t(g.KY);
  uint32_t c[3] = {s % KX, (s / KX) % KY, s / (KX * KY)};
  uint32_t ext[3] = {KX, KY, uint32_t(g.KZ)};
  uint64_t key = NONE64;
  if (lane < 6) {
    int a = lane >> 1, sg = lane & 1;
    if (!(c[a] & 1) && (sg ? c[a] + 1 < ext[a] : c[a] > 0)) {
      int64_t stv = g.stride(a);
      uint32_t t = uint32_t(int64_t(s) + (sg ? stv : -stv));
      uint32_t tb = __ldg(P.births + t);
      if (tb != ABSENT_ORD) key = make_key(tb, t);
    }
  }
  unsigned valid = __ballot_sync(0xFFFFFFFFu, key != NONE64);
  int rank = 0;
  for (int l = 0; l < 6; ++l) {
    uint64_t o = __shfl_sync(0xFFFFFFFFu, key, l);
    rank += (o < key);
  }
  if (key != NONE64) dst[rank] = key;
  __syncwarp();
  return __popc(valid);
}

__device__ __forceinline__ uint32_t lower_bound(const uint64_t* B, uint32_t n, uint64_t x,
                                                bool cg_load) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    uint64_t v = cg_load ? ldcg64(B + mid) : B[mid];
    if (v < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// C = A xor B (sorted, distinct entries each).  Warp-collective.  Returns |C|.
__device__ uint32_t merge_symdiff(const uint64_t* A, uint32_t a, const uint64_t* B, uint32_t b,
                                  bool b_cg, uint64_t* C, int lane) {
  const unsigned lt = (1u << lane) - 1;
  uint32_t carry = 0;
  for (uint32_t base = 0; base < a; base += 32) {
    uint32_t i = base + lane;
    bool valid = i < a;
    uint64_t x = valid ? ldcg64(A + i) : 0;
    uint32_t r = valid ? lower_bound(B, b, x, b_cg) : 0;
    bool dup = valid && r < b && (b_cg ? ldcg64(B + r) : B[r]) == x;
    unsigned m = __ballot_sync(0xFFFFFFFFu, dup);
    uint32_t cb = carry + __popc(m & lt);
    if (valid && !dup) C[(i - cb) + (r - cb)] = x;
    carry += __popc(m);
  }
  const uint32_t dups = carry;
  carry = 0;
  for (uint32_t base = 0; base < b; base += 32) {
    uint32_t k = base + lane;
    bool valid = k < b;
    uint64_t x = valid ? (b_cg ? ldcg64(B + k) : B[k]) : 0;
    uint32_t r = valid ? lower_bound(A, a, x, true) : 0;
    bool dup = valid && r < a && ldcg64(A + r) == x;
    unsigned m = __ballot_sync(0xFFFFFFFFu, dup);
    uint32_t cb = carry + __popc(m & lt);
    if (valid && !dup) C[(k - cb) + (r - cb)] = x;
    carry += __popc(m);
  }
  __syncwarp();
  return a + b - 2 * dups;
}

__global__ void __launch_bounds__(THREADS) k_reduce(RP P) {
  cg::grid_group grid = cg::this_grid();
  __shared__ uint64_t s_small[WARPS_PER_BLOCK][8];
  __shared__ uint64_t s_red[THREADS / 32];
  __shared__ uint64_t s_wmin[WARPS_PER_BLOCK];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const uint32_t W = (gridDim.x * blockDim.x) >> 5;
  const uint32_t w = blockIdx.x * WARPS_PER_BLOCK + wib;
  uint32_t lo = 0;
  const int sh = P.d;  // unused placeholder to keep P.d referenced
  (void)sh;

  for (uint32_t round = 0;; ++round) {
    // ---------------- phase A: advance my window position's column
    const uint32_t j = lo + w;
    uint64_t cval = NONE64;
    bool ready = false, fin = true;
    uint32_t len = 0, flags = 0, slot = 0;
    uint64_t* wk = nullptr;
    if (j < P.ncols) {
      slot = j % W;
      wk = P.work + uint64_t(slot) * 2 * P.work_cap;
      const uint32_t scol = __ldcg(P.slot_col + slot);
      if (scol != j) {  // a new column enters the window: its coboundary
        uint32_t s = key_kidx(P.cols[j]);
        len = coboundary(P, s, wk, lane);
        flags = 0;
        if (lane == 0) P.slot_col[slot] = j;
      } else {
        len = __ldcg(P.slot_len + slot);
        flags = __ldcg(P.slot_flags + slot);
      }
      fin = flags & 2;
      if (!fin) {
        int steps = 0;
        unsigned long long adds = 0;
        while (true) {
          uint64_t* cur = wk + (flags & 1) * P.work_cap;
          if (len == 0) break;
          const uint64_t piv = ldcg64(cur);
          const uint32_t pk = key_kidx(piv);
          const uint8_t t = __ldg(P.tags + pk);
          const uint64_t* add;
          uint32_t alen;
          bool add_cg;
          if (tag_kind(t) == KIND_DOWN) {
            // pivot is the upper cell of an apparent pair (s', pivot): add delta(s')
            uint32_t sp = uint32_t(int64_t(pk) + dir_offset(P.g, tag_dir(t)));
            alen = coboundary(P, sp, s_small[wib], lane);
            add = s_small[wib];
            add_cg = false;
          } else {
            const uint32_t o = __ldcg(P.owner + pk);
            if (o == NONE32) { ready = true; break; }
            add = P.pool + __ldcg(P.pool_off + o);
            alen = __ldcg(P.pool_len + o);
            add_cg = true;
          }
          if (steps >= P.max_steps) break;
          if (len + alen > P.work_cap) {
            if (lane == 0) atomicOr(P.err, 1);
            break;
          }
          uint64_t* nxt = wk + ((flags & 1) ^ 1) * P.work_cap;
          len = merge_symdiff(cur, len, add, alen, add_cg, nxt, lane);
          flags ^= 1;
          ++steps;
          ++adds;
        }
        if (lane == 0 && adds) atomicAdd(P.stats + 1, adds);
        if (len == 0) {  // zero column: essential class (clearing makes this exact)
          fin = true;
          flags |= 2;
          if (lane == 0) {
            unsigned long long r = atomicAdd(P.nrec, 1ull);
            P.rec[r] = (uint64_t(key_kidx(P.cols[j])) << 32) | NONE32;
          }
        } else {
          cval = ldcg64(wk + (flags & 1) * P.work_cap);
        }
      }
    }
    if (lane == 0) P.cand[w] = fin ? NONE64 : cval;
    // block min of the candidates (for the grid-wide prefix)
    uint64_t mine = fin ? NONE64 : cval;
    if (lane == 0) s_wmin[wib] = mine;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint64_t m = NONE64;
      for (int q = 0; q < WARPS_PER_BLOCK; ++q) m = min(m, s_wmin[q]);
      P.blockmin[blockIdx.x] = m;
    }
    grid.sync();

    // ---------------- phase B: exclusive prefix-min over window positions < w
    uint64_t pm = NONE64;
    for (uint32_t b = threadIdx.x; b < blockIdx.x; b += THREADS) pm = min(pm, (uint64_t)__ldcg((const unsigned long long*)P.blockmin + b));
    for (int off = 16; off > 0; off >>= 1) pm = min(pm, __shfl_xor_sync(0xFFFFFFFFu, pm, off));
    if (lane == 0) s_red[wib] = pm;
    __syncthreads();
    uint64_t prefix = NONE64;
    for (int q = 0; q < WARPS_PER_BLOCK; ++q) prefix = min(prefix, s_red[q]);
    for (int q = 0; q < wib; ++q) prefix = min(prefix, s_wmin[q]);

    // ---------------- phase C: commit
    if (j < P.ncols && !fin && ready && cval < prefix) {
      uint64_t* cur = wk + (flags & 1) * P.work_cap;
      unsigned long long off = 0;
      if (lane == 0) off = atomicAdd(P.pool_top, (unsigned long long)len);
      off = __shfl_sync(0xFFFFFFFFu, off, 0);
      if (off + len > P.pool_cap) {
        if (lane == 0) atomicOr(P.err, 2);
      } else {
        for (uint32_t i = lane; i < len; i += 32) P.pool[off + i] = ldcg64(cur + i);
        if (lane == 0) {
          P.pool_off[j] = off;
          P.pool_len[j] = len;
          __threadfence();
          P.owner[key_kidx(cval)] = j;
          unsigned long long r = atomicAdd(P.nrec, 1ull);
          P.rec[r] = (uint64_t(key_kidx(P.cols[j])) << 32) | key_kidx(cval);
        }
        fin = true;
        flags |= 2;
      }
    }
    if (j < P.ncols && lane == 0) {
      P.slot_len[slot] = len;
      P.slot_flags[slot] = flags;
    }
    // next lo = min(unfinished window column, lo + W)
    if (lane == 0 && j < P.ncols && !fin) atomicMin(P.lo_buf + ((round + 1) & 1), j);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      uint64_t nl = uint64_t(lo) + W;
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

    int dev = 0, nsm = 0, per_sm = 0;
    CR_CUDA(cudaGetDevice(&dev));
    CR_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    CR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_reduce, THREADS, 0));
    if (per_sm < 1) throw Error{CR_EINTERNAL, "k_reduce cannot be resident"};
    per_sm = per_sm > 4 ? 4 : per_sm;
    int64_t blocks = int64_t(nsm) * per_sm;
    // do not launch more warps than columns (small problems)
    int64_t need_blocks = (int64_t(ncols) + WARPS_PER_BLOCK - 1) / WARPS_PER_BLOCK;
    if (need_blocks < blocks) blocks = need_blocks;
    const uint32_t W = uint32_t(blocks * WARPS_PER_BLOCK);

    uint32_t* owner = ws.alloc<uint32_t>(g.ncells);
    unsigned long long* pool_off = ws.alloc<unsigned long long>(ncols);
    uint32_t* pool_len = ws.alloc<uint32_t>(ncols);
    uint32_t* slot_col = ws.alloc<uint32_t>(W);
    uint32_t* slot_len = ws.alloc<uint32_t>(W);
    uint32_t* slot_flags = ws.alloc<uint32_t>(W);
    uint64_t* cand = ws.alloc<uint64_t>(W);
    uint64_t* blockmin = ws.alloc<uint64_t>(blocks);
    unsigned* lo_buf = reinterpret_cast<unsigned*>(ctr + 2);
    int* err = reinterpret_cast<int*>(ctr + 3);
    unsigned long long* nrec = ctr + 4;
    unsigned long long* pool_top = ctr + 5;
    unsigned long long* stats = ctr + 6;  // [6] rounds [7] additions

    uint32_t work_cap = 256;
    unsigned long long pool_cap = std::max<unsigned long long>(4ull * ncols + 1024, 1ull << 20);
    uint64_t* work = nullptr;
    uint64_t* pool = nullptr;
    for (int attempt = 0;; ++attempt) {
      if (!work) work = ws.alloc<uint64_t>(int64_t(W) * 2 * work_cap);
      if (!pool) pool = ws.alloc<uint64_t>(int64_t(pool_cap));
      CR_CUDA(cudaMemsetAsync(owner, 0xFF, g.ncells * sizeof(uint32_t), s));
      CR_CUDA(cudaMemsetAsync(slot_col, 0xFF, W * sizeof(uint32_t), s));
      CR_CUDA(cudaMemsetAsync(lo_buf, 0xFF, 2 * sizeof(unsigned), s));
      CR_CUDA(cudaMemsetAsync(err, 0, sizeof(int), s));
      CR_CUDA(cudaMemsetAsync(nrec, 0, 4 * sizeof(unsigned long long), s));
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
      P.work_cap = work_cap;
      P.slot_col = slot_col;
      P.slot_len = slot_len;
      P.slot_flags = slot_flags;
      P.cand = cand;
      P.blockmin = blockmin;
      P.lo_buf = lo_buf;
      P.rec = S.R.rec[d];
      P.nrec = nrec;
      P.err = err;
      P.max_steps = 64;
      P.stats = stats;
      void* args[] = {&P};
      CR_CUDA(cudaLaunchCooperativeKernel((void*)k_reduce, dim3(unsigned(blocks)), dim3(THREADS),
                                          args, 0, s));
      ++g_launch_count;
      int e = read_scalar(err, s, hs);
      if (e == 0) break;
      if (e & 4) throw Error{CR_EINTERNAL, "reduction invariant violated"};
      if (attempt > 12) throw Error{CR_ENOMEM, "reduction buffers exhausted"};
      if (e & 1) {
        ws.release(work);
        work = nullptr;
        work_cap *= 4;
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
