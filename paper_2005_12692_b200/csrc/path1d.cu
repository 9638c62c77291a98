// path1d.cu -- the 1D path (time series): H0 of a path graph.
//
// In 1D every edge is negative and H0 is the whole barcode.  Vertex i (kidx 2i) has key
// (ord(x_i), i); edge j between i=j and j+1 (kidx 2j+1) has key (ord(max(x_j, x_j+1)), j).
//  * A vertex older than both neighbours is a basin (not apparent); every other vertex is the
//    younger end of its earliest edge and dies there at zero persistence (apparent pair).
//  * An edge that is not the earliest edge of its younger endpoint is a peak (not apparent).
//    Within a finite run basins and peaks alternate: b_0 M_0 b_1 M_1 ... b_k, and a run ends with
//    an infinite barrier.  The compressed sequence keeps exactly these.
//  * Elder rule: basin b dies at the lower of its two bottlenecks -- the highest
//    barrier between b and the nearest older basin on each side (infinite if none) -- because that
//    is the first edge joining b's component to an older vertex.  Both searches (nearest smaller
//    value + range max) run on a min-tree of basin keys and a max-tree of barrier keys, O(log K)
//    per basin with early exit, all basins in parallel.
#include <cub/cub.cuh>

#include "pipeline.cuh"

namespace cr {
namespace {

constexpr int T1 = 256;       // threads per block
constexpr int IPT = 8;        // elements per thread
constexpr int TILE = T1 * IPT;
constexpr uint32_t INF_BAR = 0xFFFFFFFFu;  // ord of a run-end barrier

__device__ __forceinline__ uint32_t uord(const float* x, int64_t i) { return ord_of(__ldg(x + i)); }

struct Flags {
  bool basin, barrier;
  uint32_t bar_ord;
};

// basin(i) and barrier-after-vertex(i)
__device__ __forceinline__ Flags flags_at(const float* x, int64_t n, int64_t i, uint32_t um,
                                          uint32_t u0, uint32_t u1, uint32_t u2) {
  // um = ord(x_{i-1}) (ABSENT if i==0), u0 = ord(x_i), u1 = ord(x_{i+1}), u2 = ord(x_{i+2})
  Flags f;
  const bool fin0 = u0 != ABSENT_ORD;
  f.basin = fin0 && um > u0 && u1 >= u0;
  f.barrier = false;
  f.bar_ord = INF_BAR;
  if (!fin0) return f;
  if (u1 == ABSENT_ORD) {  // run ends after vertex i (or i is the last vertex)
    f.barrier = true;
    return f;
  }
  const uint32_t e = max(u0, u1);  // edge i exists
  // The younger endpoint of edge i is i+1 if u1 >= u0 (ties: larger kidx is younger); then edge i
  // is that endpoint's earliest edge (key (u1, i) < (max(u1,u2), i+1)) and is apparent.  Otherwise
  // the younger endpoint is i, whose other edge i-1 has key (max(um,u0), i-1): it is earlier than
  // (u0, i) iff um <= u0, and then edge i is a peak.
  const bool peak = (u1 < u0) && (um != ABSENT_ORD) && (um <= u0);
  if (peak) {
    f.barrier = true;
    f.bar_ord = e;
  }
  return f;
}

__device__ __forceinline__ void load4(const float* x, int64_t n, int64_t i, uint32_t& um,
                                      uint32_t& u0, uint32_t& u1, uint32_t& u2) {
  um = i >= 1 ? uord(x, i - 1) : ABSENT_ORD;
  u0 = uord(x, i);
  u1 = i + 1 < n ? uord(x, i + 1) : ABSENT_ORD;
  u2 = i + 2 < n ? uord(x, i + 2) : ABSENT_ORD;
}

__global__ void __launch_bounds__(T1) k1_count(const float* __restrict__ x, int64_t n,
                                               uint32_t* __restrict__ cnt_b,
                                               uint32_t* __restrict__ cnt_m, int* nan_flag) {
  typedef cub::BlockReduce<uint32_t, T1> BR;
  __shared__ typename BR::TempStorage tb, tm;
  int64_t base = int64_t(blockIdx.x) * TILE;
  uint32_t nb = 0, nm = 0;
  for (int r = 0; r < IPT; ++r) {
    int64_t i = base + r * T1 + threadIdx.x;
    if (i >= n) break;
    float xv = __ldg(x + i);
    if (xv != xv) atomicOr(nan_flag, 1);
    uint32_t um, u0, u1, u2;
    load4(x, n, i, um, u0, u1, u2);
    Flags f = flags_at(x, n, i, um, u0, u1, u2);
    nb += f.basin;
    nm += f.barrier;
  }
  uint32_t sb = BR(tb).Sum(nb);
  __syncthreads();
  uint32_t sm = BR(tm).Sum(nm);
  if (threadIdx.x == 0) {
    cnt_b[blockIdx.x] = sb;
    cnt_m[blockIdx.x] = sm;
  }
}

__global__ void __launch_bounds__(T1) k1_scatter(const float* __restrict__ x, int64_t n,
                                                 const uint32_t* __restrict__ off_b,
                                                 const uint32_t* __restrict__ off_m,
                                                 uint64_t* __restrict__ bkey,
                                                 uint64_t* __restrict__ mkey,
                                                 uint32_t* __restrict__ bvert,
                                                 uint32_t* __restrict__ medge) {
  typedef cub::BlockScan<uint32_t, T1> BS;
  __shared__ typename BS::TempStorage tb, tm;
  int64_t base = int64_t(blockIdx.x) * TILE;
  uint32_t ob = off_b[blockIdx.x], om = off_m[blockIdx.x];
  for (int r = 0; r < IPT; ++r) {
    int64_t i = base + r * T1 + threadIdx.x;
    Flags f{false, false, INF_BAR};
    uint32_t u0 = 0;
    if (i < n) {
      uint32_t um, u1, u2;
      load4(x, n, i, um, u0, u1, u2);
      f = flags_at(x, n, i, um, u0, u1, u2);
    }
    uint32_t pb, pm, tb_, tm_;
    BS(tb).ExclusiveSum(uint32_t(f.basin), pb, tb_);
    BS(tm).ExclusiveSum(uint32_t(f.barrier), pm, tm_);
    if (f.basin) {
      uint32_t k = ob + pb;
      bkey[k] = make_key(u0, k);
      bvert[k] = uint32_t(2 * i);
    }
    if (f.barrier) {
      uint32_t k = om + pm;
      mkey[k] = make_key(f.bar_ord, k);
      medge[k] = f.bar_ord == INF_BAR ? NONE32 : uint32_t(2 * i + 1);
    }
    ob += tb_;
    om += tm_;
    __syncthreads();
  }
}

// one level of the min-tree (keys of basins) and max-tree (keys of barriers)
__global__ void k1_tree_level(const uint64_t* __restrict__ minc, const uint64_t* __restrict__ maxc,
                              int64_t nc, uint64_t* __restrict__ minp, uint64_t* __restrict__ maxp,
                              int64_t np) {
  int64_t p = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= np) return;
  int64_t a = 2 * p, b = 2 * p + 1;
  uint64_t mn = minc[a], mx = maxc[a];
  if (b < nc) {
    mn = min(mn, minc[b]);
    mx = max(mx, maxc[b]);
  }
  minp[p] = mn;
  maxp[p] = mx;
}

struct Tree {
  const uint64_t* mn[40];
  const uint64_t* mx[40];
  int64_t size[40];
  int levels;
};

// death barrier key of basin i (NONE64 if essential)
__device__ uint64_t basin_death(const Tree& T, int64_t i) {
  const uint64_t q = T.mn[0][i];
  // ---- left: nearest j < i with key < q; barriers j..i-1
  uint64_t L = NONE64;
  {
    uint64_t acc = 0;
    int l = 0;
    int64_t p = i - 1;
    while (p >= 0) {
      if (T.mn[l][p] < q) {
        while (l > 0) {
          --l;
          int64_t r = 2 * p + 1;
          if (r < T.size[l] && T.mn[l][r] < q) {
            p = r;
          } else {
            if (r < T.size[l]) acc = max(acc, T.mx[l][r]);
            p = 2 * p;
          }
        }
        acc = max(acc, T.mx[0][p]);
        L = acc;
        break;
      }
      acc = max(acc, T.mx[l][p]);
      if (key_ord(acc) == INF_BAR) break;  // an infinite barrier separates: no death this side
      if (p & 1) {
        p -= 1;
      } else {
        p = p / 2 - 1;
        ++l;
      }
    }
    if (L != NONE64 && key_ord(L) == INF_BAR) L = NONE64;
  }
  // ---- right: nearest r > i with key < q; barriers i..r-1
  uint64_t R = NONE64;
  {
    uint64_t acc = T.mx[0][i];
    int l = 0;
    int64_t p = i + 1;
    while (key_ord(acc) != INF_BAR && acc < L && p < T.size[l]) {
      if (T.mn[l][p] < q) {
        while (l > 0) {
          --l;
          int64_t c = 2 * p;
          if (T.mn[l][c] < q) {
            p = c;
          } else {
            acc = max(acc, T.mx[l][c]);
            p = c + 1;
          }
        }
        R = acc;
        break;
      }
      acc = max(acc, T.mx[l][p]);
      if (!(p & 1)) {
        p += 1;
      } else {
        p = (p + 1) / 2;
        ++l;
      }
    }
    if (R != NONE64 && key_ord(R) == INF_BAR) R = NONE64;
  }
  return min(L, R);
}

__global__ void k1_deaths(Tree T, int64_t K, uint64_t* __restrict__ death) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= K) return;
  death[i] = basin_death(T, i);
}

__global__ void k1_flags_out(const uint64_t* __restrict__ bkey, const uint64_t* __restrict__ death,
                             int64_t K, uint32_t* __restrict__ flag) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= K) return;
  uint64_t d = death[i];
  flag[i] = (d == NONE64) || (key_ord(d) > key_ord(bkey[i]));
}

__global__ void k1_emit(const uint64_t* __restrict__ bkey, const uint64_t* __restrict__ death,
                        const uint32_t* __restrict__ bvert, const uint32_t* __restrict__ flag,
                        const uint32_t* __restrict__ pos, int64_t K, int64_t cap,
                        cr_pair* __restrict__ out, uint32_t* __restrict__ cells) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= K || !flag[i]) return;
  int64_t o = pos[i];
  if (o >= cap) return;
  uint64_t d = death[i];
  cr_pair p;
  p.dim = 0;
  p.birth = float_of_ord(key_ord(bkey[i]));
  p.death = d == NONE64 ? __int_as_float(0x7F800000) : float_of_ord(key_ord(d));
  out[o] = p;
  if (cells) cells[o] = bvert[i];
}

// partner array: every vertex and edge; apparent pairs by the local rule, basins via deaths.
__global__ void k1_partner_local(const float* __restrict__ x, int64_t n, uint32_t* __restrict__ P) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t um, u0, u1, u2;
  load4(x, n, i, um, u0, u1, u2);
  // vertex 2i
  if (u0 == ABSENT_ORD) {
    P[2 * i] = CR_PARTNER_ABSENT;
  } else if (um > u0 && u1 >= u0) {
    P[2 * i] = CR_PARTNER_ESSENTIAL;  // basin: filled by k1_partner_basins if it dies
  } else {
    // earliest incident edge: (max(um,u0), i-1) vs (max(u0,u1), i)
    bool left_ok = um != ABSENT_ORD, right_ok = u1 != ABSENT_ORD;
    uint64_t kl = left_ok ? make_key(max(um, u0), uint32_t(i - 1)) : NONE64;
    uint64_t kr = right_ok ? make_key(max(u0, u1), uint32_t(i)) : NONE64;
    P[2 * i] = kl < kr ? uint32_t(2 * i - 1) : uint32_t(2 * i + 1);
  }
  // edge 2i+1
  if (i + 1 < n) {
    if (u0 == ABSENT_ORD || u1 == ABSENT_ORD) {
      P[2 * i + 1] = CR_PARTNER_ABSENT;
    } else {
      Flags f = flags_at(x, n, i, um, u0, u1, u2);
      bool peak = f.barrier && f.bar_ord != INF_BAR;
      // apparent: partner is the younger endpoint
      P[2 * i + 1] = peak ? CR_PARTNER_ESSENTIAL : (u1 >= u0 ? uint32_t(2 * i + 2) : uint32_t(2 * i));
    }
  }
}

__global__ void k1_partner_basins(const uint64_t* __restrict__ death,
                                  const uint32_t* __restrict__ bvert,
                                  const uint32_t* __restrict__ medge, int64_t K,
                                  uint32_t* __restrict__ P) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= K) return;
  uint64_t d = death[i];
  if (d == NONE64) return;
  uint32_t e = medge[key_kidx(d)];
  P[bvert[i]] = e;
  P[e] = bvert[i];
}

struct Compressed {
  int64_t K = 0;
  uint64_t* bkey = nullptr;
  uint64_t* mkey = nullptr;
  uint32_t* bvert = nullptr;
  uint32_t* medge = nullptr;
  uint64_t* death = nullptr;
};

void compress_and_solve(const float* x, int64_t n, Workspace& ws, HostScalars& hs, Compressed& C,
                        cr_stats& st) {
  cudaStream_t s = ws.stream();
  const int64_t nb = (n + TILE - 1) / TILE;
  uint32_t* cnt = ws.alloc<uint32_t>(2 * (nb + 1));
  uint32_t* off = ws.alloc<uint32_t>(2 * (nb + 1));
  int* nan_flag = ws.alloc<int>(1);
  CR_CUDA(cudaMemsetAsync(nan_flag, 0, sizeof(int), s));
  CR_CUDA(cudaMemsetAsync(cnt, 0, 2 * (nb + 1) * sizeof(uint32_t), s));
  k1_count<<<unsigned(nb), T1, 0, s>>>(x, n, cnt, cnt + nb + 1, nan_flag);
  CR_CHECK_LAUNCH();
  prof_mark(s, "1d_count");
  exclusive_sum_u32(cnt, off, nb + 1, ws);
  exclusive_sum_u32(cnt + nb + 1, off + nb + 1, nb + 1, ws);
  CR_CUDA(cudaMemcpyAsync(hs.p, off + nb, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  CR_CUDA(cudaMemcpyAsync(reinterpret_cast<uint32_t*>(hs.p) + 2, off + 2 * nb + 1, sizeof(uint32_t),
                          cudaMemcpyDeviceToHost, s));
  CR_CUDA(cudaMemcpyAsync(reinterpret_cast<int*>(hs.p) + 4, nan_flag, sizeof(int),
                          cudaMemcpyDeviceToHost, s));
  CR_CUDA(cudaStreamSynchronize(s));
  if (reinterpret_cast<int*>(hs.p)[4]) throw Error{CR_EINVAL, "NaN in image"};
  const int64_t K = reinterpret_cast<uint32_t*>(hs.p)[0];
  const int64_t KM = reinterpret_cast<uint32_t*>(hs.p)[2];
  if (K != KM) throw Error{CR_EINTERNAL, "1D path: basins and barriers do not alternate"};
  C.K = K;
  st.columns[0] = K;
  if (K == 0) return;
  // tree level 0 is the compressed arrays themselves; allocate levels 1.. contiguously
  int64_t total = 0, sz = K;
  int levels = 1;
  while (sz > 1) {
    sz = (sz + 1) / 2;
    total += sz;
    ++levels;
  }
  if (levels > 40) throw Error{CR_EINTERNAL, "tree too deep"};
  prof_mark(s, "1d_scan");
  C.bkey = ws.alloc<uint64_t>(K + total);
  C.mkey = ws.alloc<uint64_t>(K + total);
  C.bvert = ws.alloc<uint32_t>(K);
  C.medge = ws.alloc<uint32_t>(K);
  k1_scatter<<<unsigned(nb), T1, 0, s>>>(x, n, off, off + nb + 1, C.bkey, C.mkey, C.bvert, C.medge);
  CR_CHECK_LAUNCH();
  prof_mark(s, "1d_scatter");
  Tree T;
  T.levels = levels;
  T.mn[0] = C.bkey;
  T.mx[0] = C.mkey;
  T.size[0] = K;
  int64_t o = K;
  for (int l = 1; l < levels; ++l) {
    T.size[l] = (T.size[l - 1] + 1) / 2;
    T.mn[l] = C.bkey + o;
    T.mx[l] = C.mkey + o;
    k1_tree_level<<<grid_for(T.size[l], 256), 256, 0, s>>>(T.mn[l - 1], T.mx[l - 1], T.size[l - 1],
                                                          C.bkey + o, C.mkey + o, T.size[l]);
    CR_CHECK_LAUNCH();
    o += T.size[l];
  }
  prof_mark(s, "1d_tree");
  C.death = ws.alloc<uint64_t>(K);
  k1_deaths<<<grid_for(K, 256), 256, 0, s>>>(T, K, C.death);
  CR_CHECK_LAUNCH();
  prof_mark(s, "1d_deaths");
}

}  // namespace

int64_t barcodes_1d_tree(const float* x, int64_t n, cr_pair* out, uint32_t* out_cells, int64_t cap,
                    Workspace& ws, HostScalars& hs, cr_stats& st) {
  cudaStream_t s = ws.stream();
  Compressed C;
  compress_and_solve(x, n, ws, hs, C, st);
  if (C.K == 0) return 0;
  uint32_t* flag = ws.alloc<uint32_t>(C.K + 1);
  uint32_t* pos = ws.alloc<uint32_t>(C.K + 1);
  k1_flags_out<<<grid_for(C.K, 256), 256, 0, s>>>(C.bkey, C.death, C.K, flag);
  CR_CHECK_LAUNCH();
  CR_CUDA(cudaMemsetAsync(flag + C.K, 0, sizeof(uint32_t), s));
  exclusive_sum_u32(flag, pos, C.K + 1, ws);
  k1_emit<<<grid_for(C.K, 256), 256, 0, s>>>(C.bkey, C.death, C.bvert, flag, pos, C.K, cap, out,
                                             out_cells);
  CR_CHECK_LAUNCH();
  prof_mark(s, "1d_emit");
  uint32_t cnt = read_scalar(pos + C.K, s, hs);
  st.pairs[0] = cnt;
  return cnt;
}

void pairing_1d(const float* x, int64_t n, uint32_t* partner, Workspace& ws, HostScalars& hs,
                cr_stats& st) {
  cudaStream_t s = ws.stream();
  Compressed C;
  compress_and_solve(x, n, ws, hs, C, st);
  k1_partner_local<<<grid_for(n, 256), 256, 0, s>>>(x, n, partner);
  CR_CHECK_LAUNCH();
  if (C.K > 0) {
    k1_partner_basins<<<grid_for(C.K, 256), 256, 0, s>>>(C.death, C.bvert, C.medge, C.K, partner);
    CR_CHECK_LAUNCH();
  }
}

}  // namespace cr
