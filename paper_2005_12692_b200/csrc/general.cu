// general.cu -- the general (1D/2D/3D, one image) path: K1 filtration, K2 apparent pairs,
// K4 dimension-0 pairing (union-find with the elder rule), bar/partner emission.
// The dims >= 1 reduction (K5) is in reduce.cu.
#include <cooperative_groups.h>

#include <cub/cub.cuh>

#include "pipeline.cuh"

namespace cg = cooperative_groups;

namespace cr {

Geom make_geom(const int64_t* shape, int ndim) {
  Geom g{};
  int64_t s[3] = {1, 1, 1};
  for (int i = 0; i < ndim; ++i) s[3 - ndim + i] = shape[i];
  g.nz = s[0];
  g.ny = s[1];
  g.nx = s[2];
  g.KX = 2 * g.nx - 1;
  g.KY = 2 * g.ny - 1;
  g.KZ = 2 * g.nz - 1;
  g.ncells = g.KX * g.KY * g.KZ;
  g.nvox = g.nx * g.ny * g.nz;
  g.D = (g.nx > 1) + (g.ny > 1) + (g.nz > 1);
  return g;
}

namespace {

__device__ __forceinline__ void coords_of(const Geom& g, uint32_t k, uint32_t& X, uint32_t& Y,
                                          uint32_t& Z) {
  uint32_t KX = uint32_t(g.KX), KY = uint32_t(g.KY);
  X = k % KX;
  uint32_t r = k / KX;
  Y = r % KY;
  Z = r / KY;
}

// ---------------------------------------------------------------------------------------------
// K1: cell births.  birth = max over a cell's vertices of ord(phi); since
// ord(+inf) = ABSENT_ORD exceeds every finite ord, a cell with a +inf vertex gets ABSENT_ORD
// (absent from K, reading R5).  A thread owns one (x, y) voxel column and streams
// K1_ZC planes along z: per plane it loads its voxel and the one at y+1 (the plane z+1 pair is
// carried to the next step), takes the x+1 neighbours from the next lane, and writes the 8 cells
// whose lowest vertex is its voxel (the 2x2 cells of the Khalimsky rows (2z|2z+1, 2y|2y+1) at
// X = 2x, 2x+1: contiguous across the warp).  Finite cells are counted per dimension.
// ---------------------------------------------------------------------------------------------
constexpr int K1_ZC = 8;
__global__ void __launch_bounds__(256) k_births(const float* __restrict__ img, Geom g,
                                                uint32_t* __restrict__ births,
                                                unsigned long long* __restrict__ cnt,
                                                int* __restrict__ nan_flag) {
  const uint32_t nx = uint32_t(g.nx), ny = uint32_t(g.ny), nz = uint32_t(g.nz);
  const uint32_t KX = uint32_t(g.KX), KY = uint32_t(g.KY);
  const uint32_t XB = (nx + 31) / 32, YB = (ny + 7) / 8;
  uint32_t blk = blockIdx.x;
  const uint32_t xb = blk % XB;
  blk /= XB;
  const uint32_t yb = blk % YB, zb = blk / YB;
  const int lane = threadIdx.x & 31;
  const uint32_t x = xb * 32 + lane, y = yb * 8 + (threadIdx.x >> 5);
  const uint32_t z0 = zb * K1_ZC, z1 = min(nz, z0 + K1_ZC);
  const bool vx = x < nx, vy = y < ny, hx = x + 1 < nx, hy = y + 1 < ny;
  const uint64_t plane = uint64_t(nx) * ny;
  bool nan = false;
  auto ld = [&](uint32_t xx, uint32_t yy, uint32_t zz, bool ok) -> uint32_t {
    if (!ok) return ABSENT_ORD;
    const float f = __ldg(img + zz * plane + uint64_t(yy) * nx + xx);
    nan |= f != f;
    return ord_of(f);
  };
  // planes z (a, b), z+1 (an, bn) and z+2 (prefetched); lane 31 also streams the x+1 column
  const bool l31 = lane == 31;
  uint32_t a = ld(x, y, z0, vx && vy), b = ld(x, y + 1, z0, vx && hy);
  uint32_t an = ld(x, y, z0 + 1, vx && vy && z0 + 1 < nz), bn = ld(x, y + 1, z0 + 1, vx && hy && z0 + 1 < nz);
  uint32_t e = l31 ? ld(x + 1, y, z0, hx && vy) : 0u, f = l31 ? ld(x + 1, y + 1, z0, hx && hy) : 0u;
  uint32_t en = l31 ? ld(x + 1, y, z0 + 1, hx && vy && z0 + 1 < nz) : 0u;
  uint32_t fn = l31 ? ld(x + 1, y + 1, z0 + 1, hx && hy && z0 + 1 < nz) : 0u;
  uint32_t c0 = 0, c1 = 0, c2 = 0, c3 = 0;
  for (uint32_t z = z0; z < z1; ++z) {
    const bool hz = z + 1 < nz, hz2 = z + 2 < nz && z + 2 < z1 + 1;
    const uint32_t an2 = ld(x, y, z + 2, vx && vy && hz2), bn2 = ld(x, y + 1, z + 2, vx && hy && hz2);
    const uint32_t en2 = l31 ? ld(x + 1, y, z + 2, hx && vy && hz2) : 0u;
    const uint32_t fn2 = l31 ? ld(x + 1, y + 1, z + 2, hx && hy && hz2) : 0u;
    uint32_t a1 = __shfl_down_sync(0xFFFFFFFFu, a, 1), b1 = __shfl_down_sync(0xFFFFFFFFu, b, 1);
    uint32_t an1 = __shfl_down_sync(0xFFFFFFFFu, an, 1), bn1 = __shfl_down_sync(0xFFFFFFFFu, bn, 1);
    if (l31) {
      a1 = e;
      b1 = f;
      an1 = en;
      bn1 = fn;
    }
    if (vx && vy) {
      const uint32_t c100 = max(a, a1), c010 = max(a, b), c110 = max(c100, max(b, b1));
      const uint32_t c001 = max(a, an), c101 = max(c100, max(an, an1));
      const uint32_t c011 = max(c010, max(an, bn));
      const uint32_t c111 = max(c110, max(max(an, an1), max(bn, bn1)));
      uint32_t* r = births + (uint64_t(2 * z) * KY + 2 * y) * KX + 2 * x;
      r[0] = a;
      if (hx) r[1] = c100;
      c0 += a != ABSENT_ORD;
      c1 += hx && c100 != ABSENT_ORD;
      if (hy) {
        r[KX] = c010;
        if (hx) r[KX + 1] = c110;
        c1 += c010 != ABSENT_ORD;
        c2 += hx && c110 != ABSENT_ORD;
      }
      if (hz) {
        uint32_t* q = r + uint64_t(KX) * KY;
        q[0] = c001;
        if (hx) q[1] = c101;
        c1 += c001 != ABSENT_ORD;
        c2 += hx && c101 != ABSENT_ORD;
        if (hy) {
          q[KX] = c011;
          if (hx) q[KX + 1] = c111;
          c2 += c011 != ABSENT_ORD;
          c3 += hx && c111 != ABSENT_ORD;
        }
      }
    }
    a = an;
    b = bn;
    an = an2;
    bn = bn2;
    e = en;
    f = fn;
    en = en2;
    fn = fn2;
  }
  // counts and the NaN flag: warp, then block, then one atomic per counter
  __shared__ uint32_t s_c[4];
  if (threadIdx.x < 4) s_c[threadIdx.x] = 0;
  __syncthreads();
  c0 = __reduce_add_sync(0xFFFFFFFFu, c0);
  c1 = __reduce_add_sync(0xFFFFFFFFu, c1);
  c2 = __reduce_add_sync(0xFFFFFFFFu, c2);
  c3 = __reduce_add_sync(0xFFFFFFFFu, c3);
  const bool anynan = __any_sync(0xFFFFFFFFu, nan);
  if (lane == 0) {
    atomicAdd(s_c + 0, c0);
    atomicAdd(s_c + 1, c1);
    atomicAdd(s_c + 2, c2);
    atomicAdd(s_c + 3, c3);
    if (anynan) atomicOr(nan_flag, 1);
  }
  __syncthreads();
  if (threadIdx.x < 4 && s_c[threadIdx.x]) atomicAdd(cnt + threadIdx.x, (unsigned long long)s_c[threadIdx.x]);
}
// ---------------------------------------------------------------------------------------------
// K1 with K2a fused: births AND the direction codes (min-key cofacet | max-key facet << 3, see
// K2 below) of every cell, from one read of the image.  Thread = voxel column (x, y), streamed
// along z; a warp covers x = 30*xb-1 .. 30*xb+30 (lanes 0 and 31 are halo), a CTA covers the voxel
// rows y = 8*yb-1 .. 8*yb+8 (warps 0 and 9 are halo).  A cell's 6 grid neighbours come from: the
// same thread (the other half of its voxel's 2x2x2 block), the neighbouring lanes (X), the
// neighbouring warps through shared memory (Y), and the previous / next z step (Z) -- the codes of
// the cz=1 layer of plane z are formed one step later, when plane z+1's cz=0 layer exists.
// Outputs (births, codes) are written by the non-halo threads only.
// ---------------------------------------------------------------------------------------------
constexpr uint8_t CODE_ABSENT = 0x40;  // code bit 6: the cell is absent (+inf birth)
constexpr int K1C_ROWS = 8, K1C_THREADS = 32 * (K1C_ROWS + 2), K1C_ZC = 8;
inline unsigned k1c_grid(const Geom& g) {
  return unsigned(((g.nx + 29) / 30) * ((g.ny + K1C_ROWS - 1) / K1C_ROWS) *
                  ((g.nz + K1C_ZC - 1) / K1C_ZC));
}
__device__ __forceinline__ void code_visit(bool exists, bool odd, uint32_t nb, uint32_t dir,
                                           uint32_t& mcb, uint32_t& mc, uint32_t& mfb,
                                           uint32_t& mf) {
  const bool f = exists && odd && nb >= mfb;
  const bool c = exists && !odd && nb < mcb;
  mfb = f ? nb : mfb;
  mf = f ? dir : mf;
  mcb = c ? nb : mcb;
  mc = c ? dir : mc;
}
// code of a cell with birth b, odd-axis flags, and its neighbours (ABSENT_ORD where missing);
// neighbours are visited in increasing kidx order: -Z, -Y, -X, +X, +Y, +Z
__device__ __forceinline__ uint8_t cell_code6(uint32_t b, bool ox, bool oy, bool oz, uint32_t zm,
                                              bool hzm, uint32_t ym, bool hym, uint32_t xm,
                                              bool hxm, uint32_t xp, bool hxp, uint32_t yp,
                                              bool hyp, uint32_t zp, bool hzp) {
  if (b == ABSENT_ORD) return CODE_ABSENT;
  uint32_t mcb = ABSENT_ORD, mc = 7, mfb = 0, mf = 7;
  code_visit(hzm, oz, zm, 4, mcb, mc, mfb, mf);
  code_visit(hym, oy, ym, 2, mcb, mc, mfb, mf);
  code_visit(hxm, ox, xm, 0, mcb, mc, mfb, mf);
  code_visit(hxp, ox, xp, 1, mcb, mc, mfb, mf);
  code_visit(hyp, oy, yp, 3, mcb, mc, mfb, mf);
  code_visit(hzp, oz, zp, 5, mcb, mc, mfb, mf);
  return uint8_t(mc | (mf << 3));
}

__global__ void __launch_bounds__(K1C_THREADS) k_births_codes(const float* __restrict__ img,
                                                              Geom g,
                                                              uint32_t* __restrict__ births,
                                                              uint8_t* __restrict__ code,
                                                              unsigned long long* __restrict__ cnt,
                                                              int* __restrict__ nan_flag) {
  const int nx = int(g.nx), ny = int(g.ny), nz = int(g.nz);
  const uint32_t KX = uint32_t(g.KX), KY = uint32_t(g.KY);
  const int XB = (nx + 29) / 30, YB = (ny + K1C_ROWS - 1) / K1C_ROWS;
  uint32_t blk = blockIdx.x;
  const int xb = int(blk % XB);
  blk /= XB;
  const int yb = int(blk % YB), zb = int(blk / YB);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int x = xb * 30 - 1 + lane, y = yb * K1C_ROWS - 1 + w;
  const int z0 = zb * K1C_ZC, z1 = min(nz, z0 + K1C_ZC);
  const bool vx = x >= 0 && x < nx, vy = y >= 0 && y < ny, vv = vx && vy;
  const bool hx = x + 1 < nx, hy = y + 1 < ny;  // the cell spans x+1 / y+1
  const bool outp = vv && lane >= 1 && lane <= 30 && w >= 1 && w <= K1C_ROWS;
  const uint64_t plane = uint64_t(nx) * ny;
  // shared rows: births of the cz=0 layer of plane z and the cz=1 layer of plane z-1,
  // 2 cells (cy = 0, 1) x 2 (cx) per thread, indexed [w][lane]
  __shared__ uint32_t s_b0[K1C_ROWS + 2][4][32];
  __shared__ uint32_t s_b1[K1C_ROWS + 2][4][32];
  __shared__ uint32_t s_c[4];
  bool nan = false;
  auto ld = [&](int xx, int yy, int zz) -> uint32_t {
    if (xx < 0 || xx >= nx || yy < 0 || yy >= ny || zz < 0 || zz >= nz) return ABSENT_ORD;
    const float f = __ldg(img + uint64_t(zz) * plane + uint64_t(yy) * nx + xx);
    nan |= f != f;
    return ord_of(f);
  };
  // voxel values of plane zz: a = (x, y), b = (x, y+1); x+1 by shuffle (lane 31 loads)
  uint32_t a = ld(x, y, z0 - 1), b = ld(x, y + 1, z0 - 1);
  uint32_t an = ld(x, y, z0), bn = ld(x, y + 1, z0);
  uint32_t e = lane == 31 ? ld(x + 1, y, z0 - 1) : 0u, f = lane == 31 ? ld(x + 1, y + 1, z0 - 1) : 0u;
  uint32_t en = lane == 31 ? ld(x + 1, y, z0) : 0u, fn = lane == 31 ? ld(x + 1, y + 1, z0) : 0u;
  // previous step's cz=1 layer (plane z-1): births [cy][cx], for the Z- of this step's cz=0 cells
  // and its own codes one step late; and its Z- layer (plane z-1's cz=0)
  uint32_t p1[2][2] = {{ABSENT_ORD, ABSENT_ORD}, {ABSENT_ORD, ABSENT_ORD}};
  uint32_t p0[2][2] = {{ABSENT_ORD, ABSENT_ORD}, {ABSENT_ORD, ABSENT_ORD}};
  uint32_t c0 = 0, c1 = 0, c2 = 0, c3 = 0;
  for (int z = z0 - 1; z <= z1; ++z) {
    const bool pz = z >= 0 && z < nz;     // plane z exists
    const bool hz = z + 1 < nz;           // cells of plane z span z+1
    const uint32_t an2 = ld(x, y, z + 2), bn2 = ld(x, y + 1, z + 2);
    const uint32_t en2 = lane == 31 ? ld(x + 1, y, z + 2) : 0u;
    const uint32_t fn2 = lane == 31 ? ld(x + 1, y + 1, z + 2) : 0u;
    uint32_t a1 = __shfl_down_sync(0xFFFFFFFFu, a, 1), b1 = __shfl_down_sync(0xFFFFFFFFu, b, 1);
    uint32_t an1 = __shfl_down_sync(0xFFFFFFFFu, an, 1), bn1 = __shfl_down_sync(0xFFFFFFFFu, bn, 1);
    if (lane == 31) {
      a1 = e;
      b1 = f;
      an1 = en;
      bn1 = fn;
    }
    // births of the 8 cells of voxel (x, y, z): q0[cy][cx] (Z = 2z), q1[cy][cx] (Z = 2z+1);
    // cells that do not exist (beyond the grid) are ABSENT_ORD, i.e. not in K
    uint32_t q0[2][2], q1[2][2];
    {
      const uint32_t A = pz && vv ? a : ABSENT_ORD;
      const uint32_t c100 = hx ? max(a, a1) : ABSENT_ORD, c010 = hy ? max(a, b) : ABSENT_ORD;
      const uint32_t c110 = hx && hy ? max(max(a, a1), max(b, b1)) : ABSENT_ORD;
      q0[0][0] = A;
      q0[0][1] = pz && vv ? c100 : ABSENT_ORD;
      q0[1][0] = pz && vv ? c010 : ABSENT_ORD;
      q0[1][1] = pz && vv ? c110 : ABSENT_ORD;
      const bool o1 = pz && vv && hz;
      q1[0][0] = o1 ? max(a, an) : ABSENT_ORD;
      q1[0][1] = o1 && hx ? max(max(a, a1), max(an, an1)) : ABSENT_ORD;
      q1[1][0] = o1 && hy ? max(max(a, b), max(an, bn)) : ABSENT_ORD;
      q1[1][1] = o1 && hx && hy ? max(max(max(a, a1), max(b, b1)), max(max(an, an1), max(bn, bn1)))
                                : ABSENT_ORD;
    }
    // exchange the cz=0 layer of plane z and the cz=1 layer of plane z-1 (X by shuffle, Y by smem)
#pragma unroll
    for (int cy = 0; cy < 2; ++cy)
#pragma unroll
      for (int cx = 0; cx < 2; ++cx) {
        s_b0[w][2 * cy + cx][lane] = q0[cy][cx];
        s_b1[w][2 * cy + cx][lane] = p1[cy][cx];
      }
    uint32_t x0m[2], x0p[2], x1m[2], x1p[2];  // [cy]: X-1 of a cx=0 cell, X+1 of a cx=1 cell
#pragma unroll
    for (int cy = 0; cy < 2; ++cy) {
      x0m[cy] = __shfl_up_sync(0xFFFFFFFFu, q0[cy][1], 1);
      x0p[cy] = __shfl_down_sync(0xFFFFFFFFu, q0[cy][0], 1);
      x1m[cy] = __shfl_up_sync(0xFFFFFFFFu, p1[cy][1], 1);
      x1p[cy] = __shfl_down_sync(0xFFFFFFFFu, p1[cy][0], 1);
    }
    __syncthreads();
    if (outp) {
      const uint32_t X0 = 2 * uint32_t(x), Y0 = 2 * uint32_t(y);
      // ---- births of plane z, and the codes of its cz=0 layer (Z = 2z)
      if (pz && z >= z0 && z < z1) {
        const uint32_t Z = 2 * uint32_t(z);
        uint32_t* r = births + (uint64_t(Z) * KY + Y0) * KX + X0;
        uint8_t* cr = code + (uint64_t(Z) * KY + Y0) * KX + X0;
#pragma unroll
        for (int cy = 0; cy < 2; ++cy)
#pragma unroll
          for (int cx = 0; cx < 2; ++cx) {
            if ((cx && !hx) || (cy && !hy)) continue;
            const uint32_t bb = q0[cy][cx];
            const uint32_t xm = cx ? q0[cy][0] : x0m[cy];
            const uint32_t xp = cx ? x0p[cy] : q0[cy][1];
            const uint32_t ym = cy ? q0[0][cx] : s_b0[w - 1][2 + cx][lane];
            const uint32_t yp = cy ? s_b0[w + 1][cx][lane] : q0[1][cx];
            const uint8_t cd = cell_code6(bb, cx, cy, false, p1[cy][cx], z > 0, ym, Y0 + cy > 0,
                                          xm, X0 + cx > 0, xp, X0 + cx + 1 < KX, yp,
                                          Y0 + cy + 1 < KY, q1[cy][cx], hz);
            r[cy * KX + cx] = bb;
            cr[cy * KX + cx] = cd;
            const int dim = cx + cy;
            const bool fin = bb != ABSENT_ORD;
            c0 += fin && dim == 0;
            c1 += fin && dim == 1;
            c2 += fin && dim == 2;
            if (hz) {
              const uint32_t b1v = q1[cy][cx];
              r[uint64_t(KX) * KY + cy * KX + cx] = b1v;
              const bool fin1 = b1v != ABSENT_ORD;
              c1 += fin1 && dim == 0;
              c2 += fin1 && dim == 1;
              c3 += fin1 && dim == 2;
            }
          }
      }
      // ---- codes of plane z-1's cz=1 layer (Z = 2z-1): Z- = plane z-1's cz=0, Z+ = plane z's cz=0
      const int zq = z - 1;
      if (zq >= z0 && zq < z1 && zq + 1 < nz) {
        const uint32_t Z = 2 * uint32_t(zq) + 1;
        uint8_t* cr = code + (uint64_t(Z) * KY + Y0) * KX + X0;
#pragma unroll
        for (int cy = 0; cy < 2; ++cy)
#pragma unroll
          for (int cx = 0; cx < 2; ++cx) {
            if ((cx && !hx) || (cy && !hy)) continue;
            const uint32_t bb = p1[cy][cx];
            const uint32_t xm = cx ? p1[cy][0] : x1m[cy];
            const uint32_t xp = cx ? x1p[cy] : p1[cy][1];
            const uint32_t ym = cy ? p1[0][cx] : s_b1[w - 1][2 + cx][lane];
            const uint32_t yp = cy ? s_b1[w + 1][cx][lane] : p1[1][cx];
            cr[cy * KX + cx] = cell_code6(bb, cx, cy, true, p0[cy][cx], true, ym, Y0 + cy > 0, xm,
                                          X0 + cx > 0, xp, X0 + cx + 1 < KX, yp, Y0 + cy + 1 < KY,
                                          q0[cy][cx], true);
          }
      }
    }
    __syncthreads();
#pragma unroll
    for (int cy = 0; cy < 2; ++cy)
#pragma unroll
      for (int cx = 0; cx < 2; ++cx) {
        p0[cy][cx] = q0[cy][cx];
        p1[cy][cx] = q1[cy][cx];
      }
    a = an;
    b = bn;
    an = an2;
    bn = bn2;
    e = en;
    f = fn;
    en = en2;
    fn = fn2;
  }
  if (threadIdx.x < 4) s_c[threadIdx.x] = 0;
  __syncthreads();
  c0 = __reduce_add_sync(0xFFFFFFFFu, c0);
  c1 = __reduce_add_sync(0xFFFFFFFFu, c1);
  c2 = __reduce_add_sync(0xFFFFFFFFu, c2);
  c3 = __reduce_add_sync(0xFFFFFFFFu, c3);
  const bool anynan = __any_sync(0xFFFFFFFFu, nan);
  if (lane == 0) {
    atomicAdd(s_c + 0, c0);
    atomicAdd(s_c + 1, c1);
    atomicAdd(s_c + 2, c2);
    atomicAdd(s_c + 3, c3);
    if (anynan) atomicOr(nan_flag, 1);
  }
  __syncthreads();
  if (threadIdx.x < 4 && s_c[threadIdx.x])
    atomicAdd(cnt + threadIdx.x, (unsigned long long)s_c[threadIdx.x]);
}

inline unsigned k_births_grid(const Geom& g) {
  return unsigned(((g.nx + 31) / 32) * ((g.ny + 7) / 8) * ((g.nz + K1_ZC - 1) / K1_ZC));
}

// ---------------------------------------------------------------------------------------------
// K2: apparent pairs (Ripser's shortcut, inherited per PAPER.md:44-45).  For a finite cell s:
//   UP   : t = min-key cofacet of s, and s is the max-key facet of t  -> (s, t) is a pair;
//   DOWN : r = max-key facet of s, and s is the min-key cofacet of r   -> (r, s) is a pair.
// Keys are (ord(birth), kidx); the pair always has death == birth (birth(t) = max facet birth).
// Each thread writes only its own tag, so no two threads touch the same byte.
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ uint8_t tag_of(const uint32_t* __restrict__ births, const Geom& g,
                                          uint32_t k, int& dim_out) {
  const uint32_t bo = births[k];
  if (bo == ABSENT_ORD) return 0;
  uint32_t c[3];
  coords_of(g, k, c[0], c[1], c[2]);
  const uint32_t ext[3] = {uint32_t(g.KX), uint32_t(g.KY), uint32_t(g.KZ)};
  const int64_t st[3] = {1, g.KX, g.KX * g.KY};
  const uint64_t mykey = make_key(bo, k);
  const int dim = (c[0] & 1) + (c[1] & 1) + (c[2] & 1);
  uint8_t tag = 0;
  // UP
  {
    uint64_t best = NONE64;
    int bdir = -1;
    for (int a = 0; a < 3; ++a) {
      if (c[a] & 1) continue;
      for (int s = 0; s < 2; ++s) {
        if (s == 0 ? c[a] == 0 : c[a] + 1 >= ext[a]) continue;
        uint32_t t = uint32_t(int64_t(k) + (s ? st[a] : -st[a]));
        uint32_t tb = __ldg(births + t);
        if (tb == ABSENT_ORD) continue;
        uint64_t key = make_key(tb, t);
        if (key < best) { best = key; bdir = 2 * a + s; }
      }
    }
    if (bdir >= 0) {
      uint32_t t = key_kidx(best);
      int ta = bdir >> 1;
      bool is_max = true;
      for (int a = 0; a < 3 && is_max; ++a) {
        bool odd = (a == ta) ? true : (c[a] & 1);
        if (!odd) continue;
        for (int s = 0; s < 2; ++s) {
          uint32_t f = uint32_t(int64_t(t) + (s ? st[a] : -st[a]));
          if (f == k) continue;
          if (make_key(__ldg(births + f), f) > mykey) { is_max = false; break; }
        }
      }
      if (is_max) tag = make_tag(KIND_UP, bdir);
    }
  }
  // DOWN
  if (!tag && dim >= 1) {
    uint64_t best = 0;
    int bdir = -1;
    for (int a = 0; a < 3; ++a) {
      if (!(c[a] & 1)) continue;
      for (int s = 0; s < 2; ++s) {
        uint32_t f = uint32_t(int64_t(k) + (s ? st[a] : -st[a]));
        uint64_t key = make_key(__ldg(births + f), f);
        if (bdir < 0 || key > best) { best = key; bdir = 2 * a + s; }
      }
    }
    uint32_t r = key_kidx(best);
    int ra = bdir >> 1;
    bool is_min = true;
    for (int a = 0; a < 3 && is_min; ++a) {
      bool odd = (a == ra) ? false : (c[a] & 1);
      if (odd) continue;
      uint32_t ca = (a == ra) ? c[a] + ((bdir & 1) ? 1 : -1) : c[a];
      for (int s = 0; s < 2; ++s) {
        if (s == 0 ? ca == 0 : ca + 1 >= ext[a]) continue;
        uint32_t t = uint32_t(int64_t(r) + (s ? st[a] : -st[a]));
        if (t == k) continue;
        uint32_t tb = __ldg(births + t);
        if (tb == ABSENT_ORD) continue;
        if (make_key(tb, t) < mykey) { is_min = false; break; }
      }
    }
    if (is_min) tag = make_tag(KIND_DOWN, bdir);
  }
  dim_out = dim;
  return tag;
}

__global__ void k_tags(const uint32_t* __restrict__ births, Geom g, uint8_t* __restrict__ tags,
                       unsigned long long* __restrict__ app_cnt) {
  int64_t kk = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  uint8_t tag = 0;
  int dim = 0;
  if (kk < g.ncells) {
    tag = tag_of(births, g, uint32_t(kk), dim);
    tags[kk] = tag;
  }
  // apparent (UP) cells per dimension: warp ballots, then one atomic per warp and dimension
  const bool up = tag_kind(tag) == KIND_UP;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const unsigned m = __ballot_sync(0xFFFFFFFFu, up && dim == d);
    if ((threadIdx.x & 31) == 0 && m) atomicAdd(app_cnt + d, (unsigned long long)__popc(m));
  }
}


// ---------------------------------------------------------------------------------------------
// K2 in two streaming passes over the Khalimsky grid (the same apparent pairs as tag_of):
//   K2a: code[s] = (direction of s's min-key cofacet) | (direction of its max-key facet) << 3,
//        7 = none; bit 6: s absent.  A cell's 6 grid neighbours s +- e_a are its facets (odd
//        axis a) or cofacets (even a), and their kidx order is fixed: -Z < -Y < -X < +X < +Y < +Z,
//        so scanning them in that order, a strict < keeps the smaller kidx among equal births
//        (min key) and >= the larger (max key).  Absent cofacets are not in K.
//   K2b: s is UP (paired with its min cofacet t) iff t's max facet is s; else DOWN (paired with
//        its max facet r) iff r's min cofacet is s.
// A CTA covers 64 cells of a Khalimsky row x 4 rows of one plane; all index math is 32-bit.
// ---------------------------------------------------------------------------------------------
struct K2Tile {
  uint32_t X, Y, Z, k;
  bool valid;
};
__device__ __forceinline__ K2Tile k2_tile(const Geom& g) {
  const uint32_t KX = uint32_t(g.KX), KY = uint32_t(g.KY);
  const uint32_t XB = (KX + 63) / 64, YB = (KY + 3) / 4;
  uint32_t b = blockIdx.x;
  const uint32_t xb = b % XB;
  b /= XB;
  const uint32_t yb = b % YB, zb = b / YB;
  K2Tile T;
  T.X = xb * 64 + (threadIdx.x & 63);
  T.Y = yb * 4 + (threadIdx.x >> 6);
  T.Z = zb;
  T.valid = T.X < KX && T.Y < KY;
  T.k = (T.Z * KY + T.Y) * KX + T.X;
  return T;
}
inline unsigned k2_grid(const Geom& g) {
  return unsigned(((g.KX + 63) / 64) * ((g.KY + 3) / 4) * g.KZ);
}

__global__ void __launch_bounds__(256) k_codes(const uint32_t* __restrict__ births, Geom g,
                                               uint8_t* __restrict__ code) {
  const K2Tile T = k2_tile(g);
  if (!T.valid) return;
  const uint32_t KX = uint32_t(g.KX), KY = uint32_t(g.KY), KZ = uint32_t(g.KZ);
  const uint32_t sy = KX, sz = KX * KY;
  const uint32_t b = births[T.k];
  if (b == ABSENT_ORD) {
    code[T.k] = CODE_ABSENT;
    return;
  }
  uint32_t mcb = ABSENT_ORD, mfb = 0, mc = 7, mf = 7;
  auto visit = [&](bool exists, bool odd, uint32_t kk, uint32_t dir) {
    if (!exists) return;
    const uint32_t nb = __ldg(births + kk);
    if (odd) {
      if (nb >= mfb) {
        mfb = nb;
        mf = dir;
      }
    } else if (nb < mcb) {  // absent (ABSENT_ORD) never wins
      mcb = nb;
      mc = dir;
    }
  };
  visit(T.Z > 0, T.Z & 1, T.k - sz, 4);
  visit(T.Y > 0, T.Y & 1, T.k - sy, 2);
  visit(T.X > 0, T.X & 1, T.k - 1, 0);
  visit(T.X + 1 < KX, T.X & 1, T.k + 1, 1);
  visit(T.Y + 1 < KY, T.Y & 1, T.k + sy, 3);
  visit(T.Z + 1 < KZ, T.Z & 1, T.k + sz, 5);
  code[T.k] = uint8_t(mc | (mf << 3));
}

// K2a, streaming along Z: a warp owns 32 cells of one Khalimsky row, a CTA 8 rows, and walks
// K2_ZC planes.  The +-Z neighbours are the thread's own previous/next values (registers), +-X
// come from the neighbouring lanes, +-Y from the neighbouring warps through shared memory (the
// CTA's first and last warps load the rows just outside it).  Each birth is read from DRAM once.
constexpr int K2_ZC = 16;
inline unsigned k2z_grid(const Geom& g) {
  return unsigned(((g.KX + 31) / 32) * ((g.KY + 7) / 8) * ((g.KZ + K2_ZC - 1) / K2_ZC));
}
__global__ void __launch_bounds__(256) k_codes_z(const uint32_t* __restrict__ births, Geom g,
                                                 uint8_t* __restrict__ code) {
  const uint32_t KX = uint32_t(g.KX), KY = uint32_t(g.KY), KZ = uint32_t(g.KZ);
  const uint32_t XB = (KX + 31) / 32, YB = (KY + 7) / 8;
  uint32_t blk = blockIdx.x;
  const uint32_t xb = blk % XB;
  blk /= XB;
  const uint32_t yb = blk % YB, zb = blk / YB;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t X = xb * 32 + lane, Y = yb * 8 + w;
  const uint32_t Z0 = zb * K2_ZC, Z1 = min(KZ, Z0 + K2_ZC);
  const bool vx = X < KX, vy = Y < KY;
  const uint32_t sz = KX * KY;
  __shared__ uint32_t s_row[10][32];  // rows Y0-1 .. Y0+8 of the current plane
  auto at = [&](uint32_t xx, uint32_t yy, uint32_t zz, bool ok) -> uint32_t {
    return ok ? __ldg(births + (zz * KY + yy) * KX + xx) : ABSENT_ORD;
  };
  uint32_t prev = Z0 > 0 ? at(X, Y, Z0 - 1, vx && vy) : ABSENT_ORD;
  uint32_t cur = at(X, Y, Z0, vx && vy);
  for (uint32_t Z = Z0; Z < Z1; ++Z) {
    const bool hn = Z + 1 < KZ;
    const uint32_t next = at(X, Y, Z + 1, vx && vy && hn);
    // rows above/below the CTA (halo), and the X neighbours outside the warp
    if (w == 0) s_row[0][lane] = at(X, Y - 1, Z, vx && Y > 0);
    if (w == 7) s_row[9][lane] = at(X, Y + 1, Z, vx && Y + 1 < KY);
    s_row[w + 1][lane] = cur;
    uint32_t xm = __shfl_up_sync(0xFFFFFFFFu, cur, 1), xp = __shfl_down_sync(0xFFFFFFFFu, cur, 1);
    if (lane == 0) xm = at(X - 1, Y, Z, vy && X > 0);
    if (lane == 31) xp = at(X + 1, Y, Z, vy && X + 1 < KX);
    __syncthreads();
    const uint32_t ym = s_row[w][lane], yp = s_row[w + 2][lane];
    if (vx && vy) {
      const uint32_t k = (Z * KY + Y) * KX + X;
      uint8_t c = CODE_ABSENT;
      if (cur != ABSENT_ORD) {
        uint32_t mcb = ABSENT_ORD, mfb = 0, mc = 7, mf = 7;
        auto visit = [&](bool exists, bool odd, uint32_t nb, uint32_t dir) {
          if (!exists) return;
          if (odd) {
            if (nb >= mfb) {
              mfb = nb;
              mf = dir;
            }
          } else if (nb < mcb) {
            mcb = nb;
            mc = dir;
          }
        };
        visit(Z > 0, Z & 1, prev, 4);
        visit(Y > 0, Y & 1, ym, 2);
        visit(X > 0, X & 1, xm, 0);
        visit(X + 1 < KX, X & 1, xp, 1);
        visit(Y + 1 < KY, Y & 1, yp, 3);
        visit(hn, Z & 1, next, 5);
        c = uint8_t(mc | (mf << 3));
      }
      code[k] = c;
    }
    __syncthreads();
    prev = cur;
    cur = next;
  }
}

// K2 fused (births -> tags), streaming along Z.  A warp covers 32 consecutive cells of a
// Khalimsky row, X = X0-1 .. X0+30, and a CTA 18 rows, Y = Y0-1 .. Y0+16; codes (K2a) are formed
// for all of them, tags (K2b) for the inner 30 x 16.  Step z forms the codes of plane z from the
// births of planes z-1, z, z+1 (own column in registers, X neighbours by shuffle, Y neighbours
// through shared memory) and the tags of plane z-1 from the codes of planes z-2, z-1, z.  Births
// are prefetched two planes ahead; codes never leave the chip.
constexpr int K2F_ROWS = 16, K2F_ZC = 32, K2F_THREADS = 32 * (K2F_ROWS + 2);
inline unsigned k2f_grid(const Geom& g) {
  return unsigned(((g.KX + 29) / 30) * ((g.KY + K2F_ROWS - 1) / K2F_ROWS) *
                  ((g.KZ + K2F_ZC - 1) / K2F_ZC));
}
// Running max (facets) / min (cofacets) of (birth, position in the kidx order), branch-free.
// Neighbours are visited in increasing kidx order (rank r = 0..5); a missing neighbour has birth
// ABSENT_ORD and is skipped for cofacets (never < the initial ABSENT_ORD) and, as a facet of a
// present cell, never occurs.
struct CodeAcc {
  uint32_t mcb, mfb, mc, mf;
  __device__ __forceinline__ CodeAcc() : mcb(ABSENT_ORD), mfb(0u), mc(7u), mf(7u) {}
  __device__ __forceinline__ void visit(bool exists, bool odd, uint32_t nb, uint32_t dir) {
    const bool f = exists && odd && nb >= mfb;   // >=: the later (larger kidx) wins ties
    const bool c = exists && !odd && nb < mcb;   // <: the earlier (smaller kidx) wins ties
    mfb = f ? nb : mfb;
    mf = f ? dir : mf;
    mcb = c ? nb : mcb;
    mc = c ? dir : mc;
  }
  __device__ __forceinline__ uint8_t code() const { return uint8_t(mc | (mf << 3)); }
};
// tag of a cell with code c given its six neighbours' codes packed one byte each by direction
// (dir = 2 axis + (sign > 0)): UP if its min cofacet's max facet is itself, else DOWN if its max
// facet's min cofacet is itself
__device__ __forceinline__ uint8_t code_tag(uint8_t c, uint64_t nbp) {
  if (c & CODE_ABSENT) return 0;
  const uint32_t mc = c & 7, mf = (c >> 3) & 7;
  const uint32_t tmc = uint32_t(nbp >> (8 * (mc & 7))) & 0xFF;  // mc == 7: reads byte 7 (= 0)
  const uint32_t tmf = uint32_t(nbp >> (8 * (mf & 7))) & 0xFF;
  if (mc != 7 && ((tmc >> 3) & 7) == (mc ^ 1)) return make_tag(KIND_UP, int(mc));
  if (mf != 7 && (tmf & 7) == (mf ^ 1)) return make_tag(KIND_DOWN, int(mf));
  return 0;
}

__global__ void __launch_bounds__(K2F_THREADS) k_apparent(const uint32_t* __restrict__ births,
                                                         Geom g, uint8_t* __restrict__ tags,
                                                         unsigned long long* __restrict__ app_cnt) {
  const int KX = int(g.KX), KY = int(g.KY), KZ = int(g.KZ);
  const int XB = (KX + 29) / 30, YB = (KY + K2F_ROWS - 1) / K2F_ROWS;
  uint32_t blk = blockIdx.x;
  const int xb = int(blk % XB);
  blk /= XB;
  const int yb = int(blk % YB), zb = int(blk / YB);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int X = xb * 30 - 1 + lane, Y = yb * K2F_ROWS - 1 + w;
  const int Z0 = zb * K2F_ZC, Z1 = min(KZ, Z0 + K2F_ZC);
  const bool vc = X >= 0 && X < KX && Y >= 0 && Y < KY;
  const bool out_cell = vc && lane >= 1 && lane <= 30 && w >= 1 && w <= K2F_ROWS;
  const bool ox = X & 1, oy = Y & 1;
  const bool hxm = X > 0, hxp = X + 1 < KX, hym = Y > 0, hyp = Y + 1 < KY;
  const uint32_t plane = uint32_t(KX) * uint32_t(KY);
  __shared__ uint32_t s_b[K2F_ROWS + 4][32];   // births rows Y0-2 .. Y0+17 of plane z
  __shared__ uint8_t s_c[2][K2F_ROWS + 2][32];  // codes rows Y0-1 .. Y0+16, planes z-1 | z
  __shared__ uint32_t s_cnt[3];
  if (threadIdx.x < 3) s_cnt[threadIdx.x] = 0;
  // streams: own column, and one halo column for the CTA's edge threads (warp 0: row Y-1, the last
  // warp: row Y+1, lanes 0/31: X-1/X+1; the four corner lanes also stream their X halo)
  int hx = X, hy = Y;
  if (w == 0) hy = Y - 1;
  else if (w == K2F_ROWS + 1) hy = Y + 1;
  else if (lane == 0) hx = X - 1;
  else if (lane == 31) hx = X + 1;
  const bool ewarp = w == 0 || w == K2F_ROWS + 1;
  const bool has_h = hx != X || hy != Y;
  const bool vh = has_h && hx >= 0 && hx < KX && hy >= 0 && hy < KY;
  const bool xh = (lane == 0 || lane == 31) && ewarp;
  const int cx = lane == 0 ? X - 1 : X + 1;
  const bool vq = xh && cx >= 0 && cx < KX && Y >= 0 && Y < KY;
  // stream pointers (advanced by one plane per step) and their validity
  const uint32_t* po = births + (vc ? uint32_t(Y) * uint32_t(KX) + uint32_t(X) : 0u);
  const uint32_t* ph = births + (vh ? uint32_t(hy) * uint32_t(KX) + uint32_t(hx) : 0u);
  const uint32_t* pq = births + (vq ? uint32_t(Y) * uint32_t(KX) + uint32_t(cx) : 0u);
  auto ld0 = [&](const uint32_t* p, bool ok, int zz) -> uint32_t {
    return (ok && zz >= 0 && zz < KZ) ? __ldg(p + uint32_t(zz) * plane) : ABSENT_ORD;
  };
  uint32_t bzm = ld0(po, vc, Z0 - 2), bz = ld0(po, vc, Z0 - 1), bzp = ld0(po, vc, Z0);
  uint32_t bzp2 = ld0(po, vc, Z0 + 1);
  uint32_t hz = ld0(ph, vh, Z0 - 1), hzp = ld0(ph, vh, Z0), hzp2 = ld0(ph, vh, Z0 + 1);
  uint32_t qz = ld0(pq, vq, Z0 - 1), qzp = ld0(pq, vq, Z0), qzp2 = ld0(pq, vq, Z0 + 1);
  // next loads: plane z + 3
  const int zl = Z0 + 2;
  const uint32_t* no = po + (zl > 0 ? uint32_t(zl) * plane : 0u);
  const uint32_t* nh = ph + (zl > 0 ? uint32_t(zl) * plane : 0u);
  const uint32_t* nq = pq + (zl > 0 ? uint32_t(zl) * plane : 0u);
  uint8_t cprev2 = CODE_ABSENT, cprev = CODE_ABSENT;
  uint32_t nup = 0;  // UP cells per dimension, one byte each (<= K2F_ZC per thread)
  uint8_t* tout = tags + (uint32_t(max(Y, 0)) * uint32_t(KX) + uint32_t(max(X, 0))) +
                  uint64_t(max(Z0, 0)) * plane;
  for (int z = Z0 - 1; z <= Z1; ++z) {
    const bool lz = z + 3 < KZ;  // z + 3 >= Z0 + 2 >= 0
    const uint32_t bnext = (vc && lz) ? __ldg(no) : ABSENT_ORD;
    const uint32_t hnext = (vh && lz) ? __ldg(nh) : ABSENT_ORD;
    const uint32_t qnext = (vq && lz) ? __ldg(nq) : ABSENT_ORD;
    no += plane;
    nh += plane;
    nq += plane;
    s_b[w + 1][lane] = bz;
    if (w == 0) s_b[0][lane] = hz;
    if (w == K2F_ROWS + 1) s_b[K2F_ROWS + 3][lane] = hz;
    uint32_t xm = __shfl_up_sync(0xFFFFFFFFu, bz, 1), xp = __shfl_down_sync(0xFFFFFFFFu, bz, 1);
    const uint32_t xe = ewarp ? qz : hz;
    if (lane == 0) xm = xe;
    if (lane == 31) xp = xe;
    __syncthreads();
    uint8_t cz = CODE_ABSENT;
    if (vc && z >= 0 && z < KZ && bz != ABSENT_ORD) {
      const bool oz = z & 1;
      CodeAcc acc;
      acc.visit(z > 0, oz, bzm, 4);
      acc.visit(hym, oy, s_b[w][lane], 2);
      acc.visit(hxm, ox, xm, 0);
      acc.visit(hxp, ox, xp, 1);
      acc.visit(hyp, oy, s_b[w + 2][lane], 3);
      acc.visit(z + 1 < KZ, oz, bzp, 5);
      cz = acc.code();
    }
    s_c[z & 1][w][lane] = cz;
    __syncthreads();
    // tags of plane z-1 from the codes of planes z-2, z-1, z
    const int zt = z - 1;
    const uint32_t cxm = __shfl_up_sync(0xFFFFFFFFu, uint32_t(cprev), 1);
    const uint32_t cxp = __shfl_down_sync(0xFFFFFFFFu, uint32_t(cprev), 1);
    if (zt >= Z0 && zt < Z1 && out_cell) {
      const uint64_t nbp = uint64_t(cxm) | (uint64_t(cxp) << 8) |
                           (uint64_t(s_c[zt & 1][w - 1][lane]) << 16) |
                           (uint64_t(s_c[zt & 1][w + 1][lane]) << 24) |
                           (uint64_t(cprev2) << 32) | (uint64_t(cz) << 40);
      const uint8_t t = code_tag(cprev, nbp);
      *tout = t;
      nup += uint32_t(tag_kind(t) == KIND_UP) << (8 * (ox + oy + (zt & 1)));
    }
    if (zt >= Z0) tout += plane;
    cprev2 = cprev;
    cprev = cz;
    bzm = bz;
    bz = bzp;
    bzp = bzp2;
    bzp2 = bnext;
    hz = hzp;
    hzp = hzp2;
    hzp2 = hnext;
    qz = qzp;
    qzp = qzp2;
    qzp2 = qnext;
  }
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const uint32_t v = __reduce_add_sync(0xFFFFFFFFu, (nup >> (8 * d)) & 0xFFu);
    if (lane == 0 && v) atomicAdd(s_cnt + d, v);
  }
  __syncthreads();
  if (threadIdx.x < 3 && s_cnt[threadIdx.x])
    atomicAdd(app_cnt + threadIdx.x, (unsigned long long)s_cnt[threadIdx.x]);
}

__global__ void __launch_bounds__(256) k_tags2(const uint8_t* __restrict__ code, Geom g,
                                               uint8_t* __restrict__ tags,
                                               unsigned long long* __restrict__ app_cnt) {
  const K2Tile T = k2_tile(g);
  uint8_t tag = 0;
  int dim = 0;
  if (T.valid) {
    const uint32_t KX = uint32_t(g.KX), KY = uint32_t(g.KY);
    const uint32_t st[3] = {1u, KX, KX * KY};
    const uint8_t c = code[T.k];
    dim = (T.X & 1) + (T.Y & 1) + (T.Z & 1);
    if (!(c & CODE_ABSENT)) {
      const uint32_t mc = c & 7, mf = (c >> 3) & 7;
      if (mc != 7) {
        const uint32_t t = (mc & 1) ? T.k + st[mc >> 1] : T.k - st[mc >> 1];
        if (((__ldg(code + t) >> 3) & 7) == (mc ^ 1)) tag = make_tag(KIND_UP, int(mc));
      }
      if (!tag && mf != 7) {
        const uint32_t r = (mf & 1) ? T.k + st[mf >> 1] : T.k - st[mf >> 1];
        if ((__ldg(code + r) & 7) == (mf ^ 1)) tag = make_tag(KIND_DOWN, int(mf));
      }
    }
    tags[T.k] = tag;
  }
  const bool up = tag_kind(tag) == KIND_UP;
  __shared__ uint32_t s_c[3];
  if (threadIdx.x < 3) s_c[threadIdx.x] = 0;
  __syncthreads();
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const unsigned m = __ballot_sync(0xFFFFFFFFu, up && dim == d);
    if ((threadIdx.x & 31) == 0 && m) atomicAdd(s_c + d, uint32_t(__popc(m)));
  }
  __syncthreads();
  if (threadIdx.x < 3 && s_c[threadIdx.x])
    atomicAdd(app_cnt + threadIdx.x, (unsigned long long)s_c[threadIdx.x]);
}

// K2b over the codes formed by k_births_codes: 4 consecutive cells per thread (one 32-bit load of
// their codes, one 32-bit store of their tags); the partner's code is a byte load (L1/L2).
__global__ void __launch_bounds__(256) k_tags_codes(const uint8_t* __restrict__ code, Geom g,
                                                    uint8_t* __restrict__ tags,
                                                    unsigned long long* __restrict__ app_cnt) {
  const uint64_t k0 = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
  const uint64_t N = uint64_t(g.ncells);
  const uint32_t KX = uint32_t(g.KX), KY = uint32_t(g.KY);
  auto stride = [&](uint32_t ax) -> int64_t {
    return ax == 0 ? 1 : (ax == 1 ? int64_t(KX) : int64_t(KX) * KY);
  };
  uint32_t nup = 0;
  if (k0 < N) {
    uint32_t w4 = 0;
    if (k0 + 3 < N) {
      w4 = __ldg(reinterpret_cast<const uint32_t*>(code + k0));
    } else {
      for (uint64_t j = 0; k0 + j < N; ++j) w4 |= uint32_t(code[k0 + j]) << (8 * j);
    }
    uint32_t X = uint32_t(k0 % KX), Y = uint32_t((k0 / KX) % KY), Z = uint32_t(k0 / (uint64_t(KX) * KY));
    uint32_t out = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint64_t k = k0 + j;
      if (k < N) {
        const uint8_t c = uint8_t(w4 >> (8 * j));
        uint8_t tag = 0;
        if (!(c & CODE_ABSENT)) {
          const uint32_t mc = c & 7, mf = (c >> 3) & 7;
          if (mc != 7) {
            const int64_t t = int64_t(k) + ((mc & 1) ? stride(mc >> 1) : -stride(mc >> 1));
            if (((__ldg(code + t) >> 3) & 7) == (mc ^ 1)) tag = make_tag(KIND_UP, int(mc));
          }
          if (!tag && mf != 7) {
            const int64_t r = int64_t(k) + ((mf & 1) ? stride(mf >> 1) : -stride(mf >> 1));
            if ((__ldg(code + r) & 7) == (mf ^ 1)) tag = make_tag(KIND_DOWN, int(mf));
          }
          if (tag_kind(tag) == KIND_UP) nup += 1u << (8 * ((X & 1) + (Y & 1) + (Z & 1)));
        }
        out |= uint32_t(tag) << (8 * j);
      }
      if (++X == KX) {
        X = 0;
        if (++Y == KY) {
          Y = 0;
          ++Z;
        }
      }
    }
    if (k0 + 3 < N) {
      *reinterpret_cast<uint32_t*>(tags + k0) = out;
    } else {
      for (uint64_t j = 0; k0 + j < N; ++j) tags[k0 + j] = uint8_t(out >> (8 * j));
    }
  }
  __shared__ uint32_t s_c[3];
  if (threadIdx.x < 3) s_c[threadIdx.x] = 0;
  __syncthreads();
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const uint32_t v = __reduce_add_sync(0xFFFFFFFFu, (nup >> (8 * d)) & 0xFFu);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(s_c + d, v);
  }
  __syncthreads();
  if (threadIdx.x < 3 && s_c[threadIdx.x])
    atomicAdd(app_cnt + threadIdx.x, (unsigned long long)s_c[threadIdx.x]);
}

// ---------------------------------------------------------------------------------------------
// K1 + K2 fused (the default): births AND apparent-pair tags of every cell from one read of the
// image (PAPER.md:97-108 for the births, PAPER.md:44-45 for the apparent pairs; the same pairs as
// k_births + k_apparent above).  A thread owns one voxel column (x, y) and walks it along z; its
// unit of work is the voxel block B(x,y,z) = the 8 cells (2x+i, 2y+j, 2z+k), i,j,k in {0,1},
// whose births are maxima over the voxels (x..x+i, y..y+j, z..z+k): with the "plane cells"
// P(z) = {V, Ex, Ey, Sxy} of a block, the k=1 cells are max(P(z), P(z+1)) (4 max per block).
// A cell's 6 Khalimsky neighbours lie in its own block or in the blocks at x+-1 (neighbouring
// lanes: shuffles), y+-1 (neighbouring warps: shared memory) and z+-1 (the thread's previous /
// next step: registers), so codes and tags are formed from registers with one __syncthreads per
// step.  Lanes 0 and 31 and warps 0 and KF_ROWS+1 are halo (their blocks' codes feed the tags of
// the inner 30 x KF_ROWS columns); lane 31 also loads the x+1 voxels its i=1 cells need.  Step z
// completes B(z-1)'s births (writes them), forms B(z-1)'s codes and B(z-2)'s tags (writes them).
//
// Codes use equal births only.  A cell's max-key facet has the cell's own birth (a birth is the max
// over the vertices, and every vertex lies in a facet), so it is the LAST facet in kidx order whose
// birth equals the cell's.  Cofacets have births >= the cell's; the min-key cofacet matters only
// when its birth equals the cell's (an apparent pair has death == birth), and then it is the FIRST
// cofacet in kidx order with that birth; otherwise the code says "none" (7), which gives the same
// UP / DOWN decisions as the full min-key code.  One compare + select per neighbour.
// Warps whose births (codes) are all absent skip the code (tag) arithmetic: C5's outside-ball
// region costs only its stores.
// Layout in registers: births b[i + 2j + 4k]; codes and tags packed in two words by j, byte i+2k.
// ---------------------------------------------------------------------------------------------
constexpr int KF_ROWS = 14, KF_THREADS = 32 * (KF_ROWS + 2);
struct KfLaunch {
  unsigned grid;
  int zc;
};
inline KfLaunch kf_launch(const Geom& g) {
  const int64_t xy = ((g.nx + 29) / 30) * ((g.ny + KF_ROWS - 1) / KF_ROWS);
  int zc = 64;
  while (zc > 8 && xy * ((g.nz + zc - 1) / zc) < 4 * 148) zc >>= 1;
  return {unsigned(xy * ((g.nz + zc - 1) / zc)), zc};
}

// code of cell (I,J,K) of block B; L/R: births of the x-1 block's i=1 / x+1 block's i=0 cells
// (index j + 2k), D/U: the y-1 block's j=1 / y+1 block's j=0 cells (index i + 2k), Zm/Zp: the
// z-1 block's k=1 / z+1 block's k=0 cells (index i + 2j).  kidx order of the neighbours:
// -Z (dir 4) < -Y (2) < -X (0) < +X (1) < +Y (3) < +Z (5); odd axis -> facet, even -> cofacet.
template <int I, int J, int K>
__device__ __forceinline__ uint32_t kf_code(const uint32_t (&B)[8], const uint32_t (&L)[4],
                                            const uint32_t (&R)[4], const uint32_t (&D)[4],
                                            const uint32_t (&U)[4], const uint32_t (&Zm)[4],
                                            const uint32_t (&Zp)[4]) {
  const uint32_t b = B[I + 2 * J + 4 * K];
  const uint32_t nb[6] = {K ? B[I + 2 * J] : Zm[I + 2 * J],       // -Z
                          J ? B[I + 4 * K] : D[I + 2 * K],        // -Y
                          I ? B[2 * J + 4 * K] : L[J + 2 * K],    // -X
                          I ? R[J + 2 * K] : B[1 + 2 * J + 4 * K],  // +X
                          J ? U[I + 2 * K] : B[I + 2 + 4 * K],    // +Y
                          K ? Zp[I + 2 * J] : B[I + 2 * J + 4]};  // +Z
  constexpr uint32_t dir[6] = {4, 2, 0, 1, 3, 5};
  const bool odd[6] = {K != 0, J != 0, I != 0, I != 0, J != 0, K != 0};
  // facets: the last equal one (the first facet is the default: one of them must be equal)
  uint32_t mf = 7;
  bool first = true;
#pragma unroll
  for (int q = 0; q < 6; ++q)
    if (odd[q]) {
      mf = first ? dir[q] : (nb[q] == b ? dir[q] : mf);
      first = false;
    }
  // cofacets: the first equal one (scan backwards); absent cofacets never equal a present birth
  uint32_t mc = 7;
#pragma unroll
  for (int q = 5; q >= 0; --q)
    if (!odd[q]) mc = nb[q] == b ? dir[q] : mc;
  return b == ABSENT_ORD ? uint32_t(CODE_ABSENT) : (mc | (mf << 3));
}
// Tags of the 4 cells of code word J (bytes p = i + 2k), all at once: byte-wise SIMD on packed
// codes.  nbw[d] holds, in byte p, the code of that cell's neighbour in direction d (assembled by
// byte permutes from the block's and the neighbouring blocks' code words).  UP at byte p iff its
// mc == d and the neighbour's mf == d^1 for some d; DOWN iff its mf == d and the neighbour's
// mc == d^1 (the pair is apparent iff each is the other's extremal (co)facet).
// Per direction: a bit-select pairs the two 3-bit fields, a xor+mask compares them with the
// constant, and (z + 0x7F) has bit 7 clear iff the 6-bit byte z is 0 (no carry leaves a byte).
// A word holds only j-even (J=0: Y cofacets) or j-odd (J=1: Y facets) cells, so half of the Y
// tests are dropped.  Absent cells (code 0x40: fields 0) are masked out at the end.
template <int J>
__device__ __forceinline__ uint32_t kf_tags_word(uint32_t own, uint32_t xm, uint32_t xp,
                                                 uint32_t ym, uint32_t yp, uint32_t zm,
                                                 uint32_t zp) {
  const uint32_t nbw[6] = {xm, xp, ym, yp, zm, zp};
  uint32_t upn = 0, dnn = 0;  // bit 7 of each byte: set iff NO direction matched
  upn = dnn = 0xFFFFFFFFu;
#pragma unroll
  for (int d = 0; d < 6; ++d) {
    const bool ydir = d == 2 || d == 3;
    if (!ydir || J == 0) {  // UP: own mc (bits 0-2) with the neighbour's mf (bits 3-5)
      const uint32_t K = uint32_t(d | ((d ^ 1) << 3)) * 0x01010101u;
      const uint32_t X = (own & 0x07070707u) | (nbw[d] & 0x38383838u);
      upn &= ((X ^ K) & 0x3F3F3F3Fu) + 0x7F7F7F7Fu;
    }
    if (!ydir || J == 1) {  // DOWN: own mf with the neighbour's mc
      const uint32_t K = uint32_t((d ^ 1) | (d << 3)) * 0x01010101u;
      const uint32_t X = (nbw[d] & 0x07070707u) | (own & 0x38383838u);
      dnn &= ((X ^ K) & 0x3F3F3F3Fu) + 0x7F7F7F7Fu;
    }
  }
  const uint32_t pres = ~(own << 1);                       // bit 7 set iff present
  const uint32_t upf = ~upn & pres & 0x80808080u;
  const uint32_t dnf = ~dnn & ~upf & pres & 0x80808080u;   // UP wins (as in tag_of)
  const uint32_t upm = (upf >> 7) * 0xFFu, dnm = (dnf >> 7) * 0xFFu;
  return (upm & (0x80808080u | (own & 0x07070707u))) |
         (dnm & (0x40404040u | ((own >> 3) & 0x07070707u)));
}

__device__ __forceinline__ uint32_t kf_ord(float f) {
  const uint32_t u = __float_as_uint(f + 0.0f);  // -0 + 0 = +0 (reading R7); NaN stays NaN
  return u ^ (uint32_t(int32_t(u) >> 31) | 0x80000000u);
}

__device__ __forceinline__ void kf_cp4(uint32_t saddr, const float* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(saddr), "l"(g));
}
__device__ __forceinline__ void kf_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void kf_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

constexpr int KF_PF = 3, KF_RING = KF_PF + 1;  // voxel planes in flight, ring slots
constexpr int KF_VROWS = KF_ROWS + 3, KF_VCOLS = 33;
struct KfSmem {
  uint32_t v[KF_RING][KF_VROWS][KF_VCOLS];  // voxel ring (raw float bits)
  uint4 bj0[2][KF_ROWS + 2][32];            // births of the j=0 cells (i + 2k), double-buffered
  uint4 bj1[2][KF_ROWS + 2][32];            // births of the j=1 cells
  uint32_t c0[2][KF_ROWS + 2][32];          // codes word j=0
  uint32_t c1[2][KF_ROWS + 2][32];          // codes word j=1
  uint32_t cnt[8];
};

struct KfP {  // 32-bit geometry for k_filtration (image < 2^32 voxels, Khalimsky grid < 2^32 cells)
  uint32_t nx, ny, nz, KX, KXY, plane, XB, YB, zc;
};
inline KfP kf_params(const Geom& g, int zc) {
  KfP p;
  p.nx = uint32_t(g.nx);
  p.ny = uint32_t(g.ny);
  p.nz = uint32_t(g.nz);
  p.KX = uint32_t(g.KX);
  p.KXY = uint32_t(g.KX * g.KY);
  p.plane = uint32_t(g.nx * g.ny);
  p.XB = uint32_t((g.nx + 29) / 30);
  p.YB = uint32_t((g.ny + KF_ROWS - 1) / KF_ROWS);
  p.zc = uint32_t(zc);
  return p;
}

__global__ void __launch_bounds__(KF_THREADS, 2) k_filtration(const float* __restrict__ img,
                                                              const KfP P,
                                                              uint32_t* __restrict__ births,
                                                              uint8_t* __restrict__ tags,
                                                              unsigned long long* __restrict__ cnt,
                                                              int* __restrict__ nan_flag) {
  extern __shared__ uint4 kf_dyn[];
  KfSmem& S = *reinterpret_cast<KfSmem*>(kf_dyn);
  const int nx = int(P.nx), ny = int(P.ny), nz = int(P.nz);
  uint32_t blk = blockIdx.x;
  const int xb = int(blk % P.XB);
  blk /= P.XB;
  const int yb = int(blk % P.YB), zb = int(blk / P.YB);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int x = xb * 30 - 1 + lane, y = yb * KF_ROWS - 1 + w;
  const int z0 = zb * int(P.zc), z1 = min(nz, z0 + int(P.zc));
  const bool vx = x >= 0 && x < nx, vy = y >= 0 && y < ny, vy1 = y + 1 < ny;
  const bool l31 = lane == 31, vx1 = x + 1 < nx, lastw = w == KF_ROWS + 1;
  const bool out = vx && vy && lane >= 1 && lane <= 30 && w >= 1 && w <= KF_ROWS;
  const bool halo_w = w == 0 || lastw;  // warp-uniform: no tags needed
  if (threadIdx.x < 8) S.cnt[threadIdx.x] = 0;
  constexpr uint32_t INF_BITS = 0x7F800000u;
  // Voxel ring: v[slot][row][col], rows y0-1 .. y0+KF_ROWS+1 (the last copied by the last warp),
  // cols x0-1 .. x0+31 (col 32 copied by lane 31).  Copies: (x, y); lane 31 also (x+1, y); the
  // last warp also (x, y+1) and its lane 31 (x+1, y+1) -- all offsets of the (x, y) pointer.
  // Positions outside the image hold +inf from the start and are never copied.
  const bool o00 = vx && vy, o10 = l31 && vx1 && vy, o01 = lastw && vx && vy1,
             o11 = lastw && l31 && vx1 && vy1;
  uint32_t* const vown = &S.v[0][w][lane];
  const uint32_t sv0 = uint32_t(__cvta_generic_to_shared(vown));
  constexpr uint32_t SLOTW = KF_VROWS * KF_VCOLS, SLOT = SLOTW * 4, ROW = KF_VCOLS * 4;
  const int c32 = 32 - lane;  // own col -> col 32
#pragma unroll
  for (int r = 0; r < KF_RING; ++r) {
    if (!o00) vown[r * SLOTW] = INF_BITS;
    if (l31 && !o10) vown[r * SLOTW + c32] = INF_BITS;
    if (lastw && !o01) vown[r * SLOTW + KF_VCOLS] = INF_BITS;
    if (lastw && l31 && !o11) vown[r * SLOTW + KF_VCOLS + c32] = INF_BITS;
  }
  const float* gsrc = img + (o00 ? uint64_t(uint32_t(y) * P.nx + uint32_t(x)) : 0ull);
  // plane zz into ring slot s (always one commit group, possibly empty)
  auto issue = [&](int zz, uint32_t s) {
    if (zz >= 0 && zz < nz) {  // CTA-uniform
      const uint32_t a = sv0 + s * SLOT;
      const float* p = gsrc + uint64_t(uint32_t(zz)) * P.plane;
      if (o00) kf_cp4(a, p);
      if (o10) kf_cp4(a + 4 * c32, p + 1);
      if (lastw) {
        const float* q = p + P.nx;
        if (o01) kf_cp4(a + ROW, q);
        if (o11) kf_cp4(a + ROW + 4 * c32, q + 1);
      }
    } else {
      uint32_t* v = vown + s * SLOTW;
      if (o00) v[0] = INF_BITS;
      if (o10) v[c32] = INF_BITS;
      if (o01) v[KF_VCOLS] = INF_BITS;
      if (o11) v[KF_VCOLS + c32] = INF_BITS;
    }
    kf_commit();
  };
  // all voxels this thread copies (or prefilled) into slot s are +inf
  auto own_inf = [&](uint32_t s) -> bool {
    const uint32_t* v = vown + s * SLOTW;
    bool r = v[0] == INF_BITS;
    if (l31) r = r && v[c32] == INF_BITS;
    if (lastw) r = r && v[KF_VCOLS] == INF_BITS && (!l31 || v[KF_VCOLS + c32] == INF_BITS);
    return r;
  };
  int z = z0 - 2;
#pragma unroll
  for (int q = 0; q < KF_PF; ++q) issue(z + q, uint32_t(q));
  kf_wait<KF_PF - 1>();  // plane z0-2 landed (own copies)
  // CTA-uniform "plane is +inf over the CTA's footprint" flags of planes z-2, z-1, z; the
  // fictitious planes before z0-2 count as +inf (the state below is initialised as absent)
  bool f2 = true, f1 = true, f0 = __syncthreads_and(own_inf(0));
  const int wm = max(w - 1, 0), wp = min(w + 1, KF_ROWS + 1);
  bool nan = false;
  uint32_t P0[4] = {ABSENT_ORD, ABSENT_ORD, ABSENT_ORD, ABSENT_ORD};  // P(z-1)
  uint32_t Zm[4] = {ABSENT_ORD, ABSENT_ORD, ABSENT_ORD, ABSENT_ORD};  // B(z-2), k=1 cells
  uint32_t CC[2] = {0x40404040u, 0x40404040u};                     // codes of B(z-2)
  uint32_t CZm[2] = {0x40404040u, 0x40404040u};                    // codes of B(z-3)
  // per-byte counters (byte = cell position i + 2k of word j): finite cells, UP cells
  uint32_t fin0 = 0, fin1 = 0, up0 = 0, up1 = 0;
  // output: births of B(z-1) / tags of B(z-2) at (2z'+k, 2y+j, 2x+i); offset of (2z0-2, 2y, 2x)
  // ... advanced by 2 KXY per step (only used when the step's plane is in [z0, z1))
  const uint32_t rowbase = uint32_t(2 * max(y, 0)) * P.KX + uint32_t(2 * max(x, 0));
  const bool hx = x + 1 < nx, hy = y + 1 < ny;
  uint32_t rs = 0;  // ring slot of plane z
  for (; z <= z1 + 1; ++z) {
    issue(z + KF_PF, (rs + KF_PF) & (KF_RING - 1));
    const bool fast = f2 && f1 && f0;  // B(z-1), B(z-2) entirely absent: nothing to compute
    uint32_t Pn[4] = {ABSENT_ORD, ABSENT_ORD, ABSENT_ORD, ABSENT_ORD};
    uint32_t Bk[8];
    const int buf = z & 1;
    if (!fast) {
      // P(z): plane cells of block z, from the ring (max over floats, then the order key)
      const uint32_t* v = vown + rs * SLOTW;
      const float v00 = __uint_as_float(v[0]), v10 = __uint_as_float(v[1]);
      const float v01 = __uint_as_float(v[KF_VCOLS]), v11 = __uint_as_float(v[KF_VCOLS + 1]);
      nan |= v00 != v00;
      const float ex = fmaxf(v00, v10);
      Pn[0] = kf_ord(v00);
      Pn[1] = kf_ord(ex);
      Pn[2] = kf_ord(fmaxf(v00, v01));
      Pn[3] = kf_ord(fmaxf(ex, fmaxf(v01, v11)));
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        Bk[q] = P0[q];
        Bk[q + 4] = max(P0[q], Pn[q]);
      }
      S.bj0[buf][w][lane] = make_uint4(Bk[0], Bk[1], Bk[4], Bk[5]);
      S.bj1[buf][w][lane] = make_uint4(Bk[2], Bk[3], Bk[6], Bk[7]);
      S.c0[buf][w][lane] = CC[0];
      S.c1[buf][w][lane] = CC[1];
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q) Bk[q] = ABSENT_ORD;
    }
    kf_wait<KF_PF - 1>();  // plane z+1 landed (own copies); visible to all after the barrier
    const uint32_t rn = (rs + 1) & (KF_RING - 1);
    const bool fn = __syncthreads_and(own_inf(rn));
    uint32_t NC[2] = {0x40404040u, 0x40404040u};
    uint32_t T0 = 0, T1 = 0;  // tag bytes, words by j, bytes i + 2k (like the codes)
    if (!fast) {
      // codes of B(z-1)
      const uint32_t bmin = min(min(min(Bk[0], Bk[1]), min(Bk[2], Bk[3])),
                                min(min(Bk[4], Bk[5]), min(Bk[6], Bk[7])));
      if (__any_sync(0xFFFFFFFFu, bmin != ABSENT_ORD)) {
        const uint4 dq = S.bj1[buf][wm][lane], uq = S.bj0[buf][wp][lane];
        const uint32_t D[4] = {dq.x, dq.y, dq.z, dq.w}, U[4] = {uq.x, uq.y, uq.z, uq.w};
        uint32_t L[4], R[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {  // q = j + 2k: L = x-1's (1,j,k), R = x+1's (0,j,k)
          L[q] = __shfl_up_sync(0xFFFFFFFFu, Bk[1 + 2 * q], 1);
          R[q] = __shfl_down_sync(0xFFFFFFFFu, Bk[2 * q], 1);
        }
        const uint32_t c000 = kf_code<0, 0, 0>(Bk, L, R, D, U, Zm, Pn);
        const uint32_t c100 = kf_code<1, 0, 0>(Bk, L, R, D, U, Zm, Pn);
        const uint32_t c010 = kf_code<0, 1, 0>(Bk, L, R, D, U, Zm, Pn);
        const uint32_t c110 = kf_code<1, 1, 0>(Bk, L, R, D, U, Zm, Pn);
        const uint32_t c001 = kf_code<0, 0, 1>(Bk, L, R, D, U, Zm, Pn);
        const uint32_t c101 = kf_code<1, 0, 1>(Bk, L, R, D, U, Zm, Pn);
        const uint32_t c011 = kf_code<0, 1, 1>(Bk, L, R, D, U, Zm, Pn);
        const uint32_t c111 = kf_code<1, 1, 1>(Bk, L, R, D, U, Zm, Pn);
        NC[0] = c000 | (c100 << 8) | (c001 << 16) | (c101 << 24);
        NC[1] = c010 | (c110 << 8) | (c011 << 16) | (c111 << 24);
      }
      // tags of B(z-2) (not needed in the halo warps)
      if (!halo_w && __any_sync(0xFFFFFFFFu, (CC[0] & CC[1] & 0x40404040u) != 0x40404040u)) {
        const uint32_t CD = S.c1[buf][wm][lane], CU = S.c0[buf][wp][lane];
        uint32_t CL[2], CR[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          CL[q] = __shfl_up_sync(0xFFFFFFFFu, CC[q], 1);
          CR[q] = __shfl_down_sync(0xFFFFFFFFu, CC[q], 1);
        }
        // neighbour codes by direction, byte p = i + 2k (see kf_tags_word)
        T0 = kf_tags_word<0>(CC[0], __byte_perm(CL[0], CC[0], 0x6341),
                             __byte_perm(CC[0], CR[0], 0x6341), CD, CC[1],
                             __byte_perm(CZm[0], CC[0], 0x5432), __byte_perm(CC[0], NC[0], 0x5432));
        T1 = kf_tags_word<1>(CC[1], __byte_perm(CL[1], CC[1], 0x6341),
                             __byte_perm(CC[1], CR[1], 0x6341), CC[0], CU,
                             __byte_perm(CZm[1], CC[1], 0x5432), __byte_perm(CC[1], NC[1], 0x5432));
      }
    }
    // stores: births of B(z-1), tags of B(z-2); counters from the codes (bit 6 = absent) and
    // the tags (bit 7 = UP).  Cell (i,j,k) exists iff (i=0 or hx), (j=0 or hy), (k=0 or hz).
    if (out) {
      const int zb1 = z - 1, zb2 = z - 2;
      if (zb1 >= z0 && zb1 < z1) {
        fin0 += (~NC[0] >> 6) & 0x01010101u;
        fin1 += (~NC[1] >> 6) & 0x01010101u;
        uint32_t* p0 = births + (uint32_t(zb1) * 2u * P.KXY + rowbase);
        uint32_t* p1 = p0 + P.KX;
        const bool hz = zb1 + 1 < nz;
        p0[0] = Bk[0];
        if (hx) p0[1] = Bk[1];
        if (hy) p1[0] = Bk[2];
        if (hx && hy) p1[1] = Bk[3];
        if (hz) {
          uint32_t* p2 = p0 + P.KXY;
          uint32_t* p3 = p1 + P.KXY;
          p2[0] = Bk[4];
          if (hx) p2[1] = Bk[5];
          if (hy) p3[0] = Bk[6];
          if (hx && hy) p3[1] = Bk[7];
        }
      }
      if (zb2 >= z0 && zb2 < z1) {
        up0 += (T0 >> 7) & 0x01010101u;
        up1 += (T1 >> 7) & 0x01010101u;
        uint8_t* p0 = tags + (uint32_t(zb2) * 2u * P.KXY + rowbase);
        uint8_t* p1 = p0 + P.KX;
        const bool hz = zb2 + 1 < nz;
        p0[0] = uint8_t(T0);
        if (hx) p0[1] = uint8_t(T0 >> 8);
        if (hy) p1[0] = uint8_t(T1);
        if (hx && hy) p1[1] = uint8_t(T1 >> 8);
        if (hz) {
          uint8_t* p2 = p0 + P.KXY;
          uint8_t* p3 = p1 + P.KXY;
          p2[0] = uint8_t(T0 >> 16);
          if (hx) p2[1] = uint8_t(T0 >> 24);
          if (hy) p3[0] = uint8_t(T1 >> 16);
          if (hx && hy) p3[1] = uint8_t(T1 >> 24);
        }
      }
    }
    // shift the pipeline
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      Zm[q] = Bk[q + 4];
      P0[q] = Pn[q];
    }
    CZm[0] = CC[0];
    CZm[1] = CC[1];
    CC[0] = NC[0];
    CC[1] = NC[1];
    f2 = f1;
    f1 = f0;
    f0 = fn;
    rs = rn;
  }
  kf_wait<0>();
  // counters: byte p of word j is cell (i, j, k) with p = i + 2k, dim = i + j + k
  auto B8 = [](uint32_t v, int p) { return (v >> (8 * p)) & 0xFFu; };
  const uint32_t v[7] = {B8(up0, 0),                                      // UP, dim 0
                         B8(up0, 1) + B8(up0, 2) + B8(up1, 0),             // UP, dim 1
                         B8(up0, 3) + B8(up1, 1) + B8(up1, 2),             // UP, dim 2
                         B8(fin0, 0),                                     // finite, dim 0
                         B8(fin0, 1) + B8(fin0, 2) + B8(fin1, 0),          // dim 1
                         B8(fin0, 3) + B8(fin1, 1) + B8(fin1, 2),          // dim 2
                         B8(fin1, 3)};                                    // dim 3
#pragma unroll
  for (int q = 0; q < 7; ++q) {
    const uint32_t s = __reduce_add_sync(0xFFFFFFFFu, v[q]);
    if (lane == 0 && s) atomicAdd(S.cnt + q, s);
  }
  const bool anynan = __any_sync(0xFFFFFFFFu, nan);
  if (lane == 0 && anynan) atomicOr(nan_flag, 1);
  __syncthreads();
  if (threadIdx.x < 7 && S.cnt[threadIdx.x])
    atomicAdd(cnt + (threadIdx.x < 3 ? threadIdx.x : threadIdx.x + 1),
              (unsigned long long)S.cnt[threadIdx.x]);
}
// ---------------------------------------------------------------------------------------------
// K4: H0 by union-find with the elder rule.
//  (1) every apparent vertex v (UP, paired with its earliest edge e_v) hangs under the other
//      endpoint of e_v, which is older; roots are the non-apparent vertices ("basins").
//  (2) pointer jumping flattens the forest.
//  (3) a residual edge whose endpoints share a root is positive (a cycle); the others are
//      inter-basin candidates.
//  (4) mutual-minimum rounds: every component takes its minimum candidate edge; an edge that is
//      the minimum at both of its components is exactly the next Kruskal merge there, so it is
//      committed: the younger root dies at it (elder rule) and is linked under the elder.
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t vox_kidx(const Geom& g, uint32_t v) {
  uint32_t nx = uint32_t(g.nx), ny = uint32_t(g.ny);
  uint32_t x = v % nx, r = v / nx, y = r % ny, z = r / ny;
  return (2 * z * uint32_t(g.KY) + 2 * y) * uint32_t(g.KX) + 2 * x;
}
__device__ __forceinline__ uint32_t kidx_vox(const Geom& g, uint32_t k) {
  uint32_t X, Y, Z;
  coords_of(g, k, X, Y, Z);
  return ((Z >> 1) * uint32_t(g.ny) + (Y >> 1)) * uint32_t(g.nx) + (X >> 1);
}

__global__ void k_h0_parent(const uint32_t* __restrict__ births, const uint8_t* __restrict__ tags,
                            Geom g, uint32_t* __restrict__ parent) {
  int64_t vv = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (vv >= g.nvox) return;
  uint32_t v = uint32_t(vv);
  uint32_t k = vox_kidx(g, v);
  uint8_t t = tags[k];
  uint32_t p = v;
  if (births[k] != ABSENT_ORD && tag_kind(t) == KIND_UP) {
    int d = tag_dir(t);
    int64_t vs = (d >> 1) == 0 ? 1 : ((d >> 1) == 1 ? g.nx : g.nx * g.ny);
    p = uint32_t(int64_t(v) + ((d & 1) ? vs : -vs));
  }
  parent[v] = p;
}

__global__ void k_pointer_jump(uint32_t* parent, int64_t n) {
  int64_t vv = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (vv >= n) return;
  uint32_t v = uint32_t(vv);
  uint32_t p = parent[v];
  while (true) {
    uint32_t pp = *(volatile uint32_t*)(parent + p);
    if (pp == p) break;
    p = pp;
    parent[v] = p;
  }
}

struct Cand {
  uint64_t key;  // edge key
  uint32_t a, b; // current component roots (voxel ids)
};

__global__ void k_h0_edges(const uint32_t* __restrict__ births, const uint8_t* __restrict__ tags,
                           Geom g, const uint32_t* __restrict__ parent, Cand* __restrict__ cand,
                           unsigned int* __restrict__ ncand) {
  int64_t kk = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  bool emit = false;
  Cand c;
  if (kk < g.ncells) {
    uint32_t k = uint32_t(kk);
    uint32_t X, Y, Z;
    coords_of(g, k, X, Y, Z);
    int dim = (X & 1) + (Y & 1) + (Z & 1);
    uint32_t bo = births[k];
    if (dim == 1 && bo != ABSENT_ORD && tag_kind(tags[k]) == KIND_RESIDUAL) {
      int64_t s = (X & 1) ? 1 : ((Y & 1) ? g.KX : g.KX * g.KY);
      uint32_t va = kidx_vox(g, uint32_t(k - s)), vb = kidx_vox(g, uint32_t(k + s));
      uint32_t ra = parent[va], rb = parent[vb];
      if (ra != rb) {
        emit = true;
        c.key = make_key(bo, k);
        c.a = ra;
        c.b = rb;
      }
    }
  }
  unsigned mask = __ballot_sync(0xFFFFFFFFu, emit);
  if (!mask) return;
  int lane = threadIdx.x & 31;
  unsigned base = 0;
  if (lane == __ffs(mask) - 1) base = atomicAdd(ncand, __popc(mask));
  base = __shfl_sync(0xFFFFFFFFu, base, __ffs(mask) - 1);
  if (emit) cand[base + __popc(mask & ((1u << lane) - 1))] = c;
}

__device__ __forceinline__ uint32_t uf_find(uint32_t* parent, uint32_t v) {
  uint32_t p = *(volatile uint32_t*)(parent + v);
  if (p == v) return v;
  while (true) {
    uint32_t pp = *(volatile uint32_t*)(parent + p);
    if (pp == p) break;
    p = pp;
  }
  return p;
}

__global__ void k_mm_find(Cand* cand, unsigned n, uint32_t* parent, unsigned long long* best,
                          uint8_t* alive) {
  unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  Cand c = cand[i];
  uint32_t a = uf_find(parent, c.a), b = uf_find(parent, c.b);
  cand[i].a = a;
  cand[i].b = b;
  if (a == b) {  // connected through strictly smaller edges: positive
    alive[i] = 0;
    return;
  }
  alive[i] = 1;
  atomicMin(best + a, (unsigned long long)c.key);
  atomicMin(best + b, (unsigned long long)c.key);
}

__global__ void k_mm_commit(const Cand* cand, unsigned n, const uint32_t* __restrict__ births,
                            Geom g, uint32_t* parent, const unsigned long long* best,
                            uint8_t* alive, uint8_t* tags, uint64_t* rec,
                            unsigned long long* nrec) {
  unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || !alive[i]) return;
  Cand c = cand[i];
  // Commit when the edge is the minimum at both components (the next Kruskal merge there), or
  // when it is the minimum at the YOUNGER component alone: that component does not change before
  // the edge, and the other one can only merge with older roots first, so the younger root dies
  // at this edge whatever happens on the other side.  (Mutual minima alone degenerate into one
  // merge per round when a large old component absorbs many young ones.)
  const bool min_a = best[c.a] == c.key, min_b = best[c.b] == c.key;
  if (!min_a && !min_b) return;
  uint32_t ka = vox_kidx(g, c.a), kb = vox_kidx(g, c.b);
  uint64_t keya = make_key(births[ka], ka), keyb = make_key(births[kb], kb);
  const bool a_young = keya > keyb;
  if (!(min_a && min_b) && (a_young ? !min_a : !min_b)) return;
  uint32_t young = a_young ? c.a : c.b, old = a_young ? c.b : c.a;
  uint32_t kyoung = a_young ? ka : kb;
  parent[young] = old;  // elder rule: the younger component dies
  tags[key_kidx(c.key)] = make_tag(KIND_CLEARED, 0);  // a death edge: cleared for dim 1
  unsigned long long r = atomicAdd(nrec, 1ull);
  rec[r] = (uint64_t(kyoung) << 32) | key_kidx(c.key);
  alive[i] = 2;
}

__global__ void k_mm_reset(Cand* cand, unsigned n, unsigned long long* best, const uint8_t* alive,
                           Cand* next, unsigned* nnext) {
  unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
  bool keep = false;
  Cand c;
  if (i < n) {
    c = cand[i];
    if (alive[i]) {
      best[c.a] = NONE64;
      best[c.b] = NONE64;
    }
    keep = alive[i] == 1;
  }
  unsigned mask = __ballot_sync(0xFFFFFFFFu, keep);
  if (!mask) return;
  int lane = threadIdx.x & 31;
  unsigned base = 0;
  if (lane == __ffs(mask) - 1) base = atomicAdd(nnext, __popc(mask));
  base = __shfl_sync(0xFFFFFFFFu, base, __ffs(mask) - 1);
  if (keep) next[base + __popc(mask & ((1u << lane) - 1))] = c;
}

__global__ void k_h0_essential(const uint32_t* __restrict__ births, Geom g,
                               const uint32_t* __restrict__ parent, uint64_t* rec,
                               unsigned long long* nrec, unsigned long long* nroots) {
  int64_t vv = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  bool emit = false;
  uint32_t k = 0;
  if (vv < g.nvox) {
    uint32_t v = uint32_t(vv);
    k = vox_kidx(g, v);
    emit = parent[v] == v && births[k] != ABSENT_ORD;
  }
  unsigned mask = __ballot_sync(0xFFFFFFFFu, emit);
  if (!mask) return;
  int lane = threadIdx.x & 31;
  unsigned long long base = 0;
  if (lane == __ffs(mask) - 1) base = atomicAdd(nrec, (unsigned long long)__popc(mask));
  base = __shfl_sync(0xFFFFFFFFu, base, __ffs(mask) - 1);
  if (emit) rec[base + __popc(mask & ((1u << lane) - 1))] = (uint64_t(k) << 32) | NONE32;
}

// ---- single-CTA variant for up to SMEM_BASINS basins: the same mutual-minimum rounds, with the
// union-find forest and the per-component minimum in shared memory and __syncthreads between
// phases (a round costs ~1 us instead of a host round trip).  Basins are renumbered by their rank
// in elder order, so the elder of two roots is simply the smaller id; candidate edges are sorted
// by key, so a component's minimum edge is the smallest edge index.
constexpr int SMEM_BASINS = 56000;
// Up to this many roots the union-find runs in one CTA's shared memory (Boruvka MSF + Kruskal),
// beyond it as device-wide merge rounds.  Since the rounds also commit a younger component's
// minimum edge they take ~10-15 rounds on every config and beat the one-CTA path everywhere
// (profiles/r01: C1 H0 1.38 -> 0.47 ms, C4 top dim 15.8 -> 0.52 ms), so the default is 0;
// CR_SMEM_BASINS=n (<= SMEM_BASINS) brings the one-CTA path back for cross-checks.
unsigned smem_basins_max() {
  const char* e = std::getenv("CR_SMEM_BASINS");
  const unsigned v = e ? unsigned(std::strtoul(e, nullptr, 10)) : 0u;
  return v < unsigned(SMEM_BASINS) ? v : unsigned(SMEM_BASINS);
}  // u32 union-find in <= 224 KB of shared memory; ranks < 2^16
constexpr int H0_THREADS = 1024;

__global__ void k_collect_roots(const uint32_t* __restrict__ births, Geom g,
                                const uint32_t* __restrict__ parent, uint64_t* rootkey,
                                unsigned* nroot) {
  int64_t vv = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  bool emit = false;
  uint64_t key = 0;
  if (vv < g.nvox) {
    uint32_t v = uint32_t(vv);
    uint32_t k = vox_kidx(g, v);
    if (parent[v] == v && births[k] != ABSENT_ORD) {
      emit = true;
      key = make_key(births[k], k);
    }
  }
  unsigned mask = __ballot_sync(0xFFFFFFFFu, emit);
  if (!mask) return;
  int lane = threadIdx.x & 31;
  unsigned base = 0;
  if (lane == __ffs(mask) - 1) base = atomicAdd(nroot, __popc(mask));
  base = __shfl_sync(0xFFFFFFFFu, base, __ffs(mask) - 1);
  if (emit) rootkey[base + __popc(mask & ((1u << lane) - 1))] = key;
}

__global__ void k_rank_roots(const uint64_t* __restrict__ rootkey, unsigned nb, Geom g,
                             uint32_t* rank_of) {
  unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nb) rank_of[kidx_vox(g, key_kidx(rootkey[i]))] = i;
}

__global__ void k_cand_pack(const Cand* __restrict__ cand, unsigned n,
                            const uint32_t* __restrict__ rank_of, uint64_t* keys, uint32_t* ab) {
  unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const Cand c = cand[i];
  keys[i] = c.key;
  ab[i] = (rank_of[c.a] << 16) | rank_of[c.b];
}

__device__ __forceinline__ uint32_t sfind(uint32_t* par, uint32_t x) {
  while (true) {
    const uint32_t p = par[x];
    if (p == x) return x;
    const uint32_t pp = par[p];
    if (pp != p) par[x] = pp;  // path halving (benign under concurrency: both are ancestors)
    x = pp;
  }
}

// Boruvka on the basin graph (one CTA, union-find in shared memory): every component's minimum
// edge is a minimum-spanning-forest edge (keys are distinct); components hook along them (of a
// mutual pair only the larger id hooks) until no edge joins two components.  MSF edges are exactly
// Kruskal's merge edges; the others close cycles (positive edges, dimension-1 columns).
__global__ void __launch_bounds__(H0_THREADS) k_h0_boruvka(
    const uint32_t* __restrict__ ab, unsigned n, unsigned nb, uint32_t* best, uint32_t* act0,
    uint32_t* act1, uint32_t* hook, uint32_t* msf, unsigned* nmsf, unsigned long long* rounds_out) {
  extern __shared__ uint32_t sh[];
  uint32_t* par = sh;
  __shared__ unsigned s_nnext;
  for (unsigned i = threadIdx.x; i < nb; i += H0_THREADS) {
    par[i] = i;
    best[i] = 0xFFFFFFFFu;
  }
  for (unsigned i = threadIdx.x; i < n; i += H0_THREADS) act0[i] = i;
  __syncthreads();
  unsigned na = n;
  uint32_t* act = act0;
  uint32_t* nxt = act1;
  unsigned long long rounds = 0;
  while (na > 0) {
    if (threadIdx.x == 0) s_nnext = 0;
    __syncthreads();
    for (unsigned t = threadIdx.x; t < na; t += H0_THREADS) {
      const uint32_t e = act[t];
      const uint32_t a = sfind(par, ab[e] >> 16), b = sfind(par, ab[e] & 0xFFFFu);
      if (a == b) continue;  // closes a cycle: not an MSF edge
      atomicMin(best + a, e);
      atomicMin(best + b, e);
      nxt[atomicAdd(&s_nnext, 1u)] = e;
    }
    __syncthreads();
    // hook targets (computed before any hooking)
    for (unsigned c = threadIdx.x; c < nb; c += H0_THREADS) {
      uint32_t h = 0xFFFFFFFFu;
      if (par[c] == c && best[c] != 0xFFFFFFFFu) {
        const uint32_t e = best[c];
        const uint32_t a = sfind(par, ab[e] >> 16), b = sfind(par, ab[e] & 0xFFFFu);
        const uint32_t o = a == c ? b : a;
        if (!(best[o] == e && c < o)) h = o;  // of a mutual pair only the larger id hooks
        if (best[o] != e || c < o) msf[atomicAdd(nmsf, 1u)] = e;  // record each edge once
      }
      hook[c] = h;
    }
    __syncthreads();
    for (unsigned c = threadIdx.x; c < nb; c += H0_THREADS) {
      if (hook[c] != 0xFFFFFFFFu) par[c] = hook[c];
      best[c] = 0xFFFFFFFFu;
    }
    __syncthreads();
    na = s_nnext;
    uint32_t* tmp = act;
    act = nxt;
    nxt = tmp;
    ++rounds;
  }
  if (threadIdx.x == 0) *rounds_out = rounds;
}

// Elder-rule Kruskal over the MSF edges in key order (one thread; union-find in shared memory).
__global__ void __launch_bounds__(H0_THREADS) k_h0_kruskal(
    const uint64_t* __restrict__ keys, const uint32_t* __restrict__ ab,
    const uint32_t* __restrict__ msf, unsigned nmsf, const uint64_t* __restrict__ rootkey,
    unsigned nb, uint8_t* tags, uint64_t* rec, unsigned long long* nrec) {
  extern __shared__ uint32_t sh[];
  uint32_t* par = sh;
  for (unsigned i = threadIdx.x; i < nb; i += H0_THREADS) par[i] = i;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long r = *nrec;
    for (unsigned t = 0; t < nmsf; ++t) {
      const uint32_t e = msf[t];
      const uint32_t a = sfind(par, ab[e] >> 16), b = sfind(par, ab[e] & 0xFFFFu);
      const uint32_t young = a > b ? a : b, old = a > b ? b : a;  // elder = smaller rank
      par[young] = old;
      const uint32_t ke = key_kidx(keys[e]);
      tags[ke] = make_tag(KIND_CLEARED, 0);
      rec[r++] = (uint64_t(key_kidx(rootkey[young])) << 32) | ke;
    }
    *nrec = r;
  }
  __syncthreads();
  for (unsigned i = threadIdx.x; i < nb; i += H0_THREADS)
    if (par[i] == i) {
      const unsigned long long r = atomicAdd(nrec, 1ull);
      rec[r] = (uint64_t(key_kidx(rootkey[i])) << 32) | NONE32;
    }
}

__global__ void __launch_bounds__(H0_THREADS) k_h0_smem(
    const uint64_t* __restrict__ keys, const uint32_t* __restrict__ ab, unsigned n,
    const uint64_t* __restrict__ rootkey, unsigned nb, uint32_t* act0, uint32_t* act1,
    uint8_t* tags, uint64_t* rec, unsigned long long* nrec, unsigned long long* rounds_out) {
  extern __shared__ uint32_t sh[];
  uint32_t* par = sh;
  uint32_t* best = sh + nb;
  __shared__ unsigned s_nnext;
  for (unsigned i = threadIdx.x; i < nb; i += H0_THREADS) {
    par[i] = i;
    best[i] = 0xFFFFFFFFu;
  }
  for (unsigned i = threadIdx.x; i < n; i += H0_THREADS) act0[i] = i;
  __syncthreads();
  unsigned na = n;
  uint32_t* act = act0;
  uint32_t* nxt = act1;
  unsigned long long rounds = 0;
  while (na > 0) {
    // phase 1: components' minimum edges (edges inside one component are positive: dropped)
    for (unsigned t = threadIdx.x; t < na; t += H0_THREADS) {
      const uint32_t e = act[t];
      const uint32_t a = sfind(par, ab[e] >> 16), b = sfind(par, ab[e] & 0xFFFFu);
      if (a != b) {
        atomicMin(best + a, e);
        atomicMin(best + b, e);
      }
    }
    if (threadIdx.x == 0) s_nnext = 0;
    __syncthreads();
    // phase 2: an edge minimal at both components is the next Kruskal merge there
    for (unsigned t = threadIdx.x; t < na; t += H0_THREADS) {
      const uint32_t e = act[t];
      const uint32_t a = sfind(par, ab[e] >> 16), b = sfind(par, ab[e] & 0xFFFFu);
      if (a == b) continue;  // positive edge
      if (best[a] == e && best[b] == e) {
        const uint32_t young = a > b ? a : b, old = a > b ? b : a;  // elder = smaller rank
        par[young] = old;
        const uint32_t ke = key_kidx(keys[e]);
        tags[ke] = make_tag(KIND_CLEARED, 0);
        const unsigned long long r = atomicAdd(nrec, 1ull);
        rec[r] = (uint64_t(key_kidx(rootkey[young])) << 32) | ke;
      } else {
        nxt[atomicAdd(&s_nnext, 1u)] = e;
      }
    }
    __syncthreads();
    // phase 3: reset the minima; next round's active list
    for (unsigned i = threadIdx.x; i < nb; i += H0_THREADS) best[i] = 0xFFFFFFFFu;
    na = s_nnext;
    uint32_t* tmp = act;
    act = nxt;
    nxt = tmp;
    ++rounds;
    __syncthreads();
  }
  // essential classes: the remaining roots
  for (unsigned i = threadIdx.x; i < nb; i += H0_THREADS)
    if (par[i] == i) {
      const unsigned long long r = atomicAdd(nrec, 1ull);
      rec[r] = (uint64_t(key_kidx(rootkey[i])) << 32) | NONE32;
    }
  if (threadIdx.x == 0) *rounds_out = rounds;
}

__global__ void k_count_basins(const uint32_t* __restrict__ births, const uint8_t* __restrict__ tags,
                               Geom g, const uint32_t* __restrict__ parent,
                               unsigned long long* cnt) {
  int64_t vv = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  bool b = false;
  if (vv < g.nvox) {
    uint32_t k = vox_kidx(g, uint32_t(vv));
    b = births[k] != ABSENT_ORD && tag_kind(tags[k]) != KIND_UP;
  }
  unsigned mask = __ballot_sync(0xFFFFFFFFu, b);
  if ((threadIdx.x & 31) == 0 && mask) atomicAdd(cnt, (unsigned long long)__popc(mask));
}

// ---------------------------------------------------------------------------------------------
// Top dimension D-1 by Alexander duality ("--top_dim").
// The dim-(D-1) cohomology columns are the (D-1)-cells, processed in decreasing key, and a column's
// coboundary holds its <= 2 cofaces (top cells); reducing such columns with pivot = min coface is
// the union-find of the dual graph -- top cells as vertices, (D-1)-cells as edges in decreasing key
// -- with the elder rule reversed: the root with the LARGER key survives, the younger root y dies
// at the edge sigma, giving the bar [birth sigma, birth y).  A face on the grid boundary or next to
// an absent top cell has fewer cofaces in K: its missing side is an absent vertex (absent top cells
// and one outside vertex OMEGA, all older than any present cell, joined first through absent
// faces).  Merging two absent-rooted components leaves a zero column: an essential bar.  Edges
// closing a cycle are the negative cells of dim D-2 (cleared).  With keys complemented (~key), the
// order and the elder rule are those of the H0 machinery above, which is reused.
// ---------------------------------------------------------------------------------------------
struct DualG {
  Geom g;
  uint32_t omega;  // = nvox: the outside vertex
};
// top cell whose base voxel is v (odd on every active axis), if it exists
__device__ __forceinline__ bool top_of_voxel(const Geom& g, uint32_t v, uint32_t& k) {
  const uint32_t nx = uint32_t(g.nx), ny = uint32_t(g.ny), nz = uint32_t(g.nz);
  const uint32_t x = v % nx, r = v / nx, y = r % ny, z = r / ny;
  uint32_t X = 0, Y = 0, Z = 0;
  if (nx > 1) { if (x + 1 >= nx) return false; X = 2 * x + 1; }
  if (ny > 1) { if (y + 1 >= ny) return false; Y = 2 * y + 1; }
  if (nz > 1) { if (z + 1 >= nz) return false; Z = 2 * z + 1; }
  k = (Z * uint32_t(g.KY) + Y) * uint32_t(g.KX) + X;
  return true;
}
__device__ __forceinline__ uint32_t coord_of(const Geom& g, uint32_t k, int a) {
  const uint32_t KX = uint32_t(g.KX), KY = uint32_t(g.KY);
  return a == 0 ? k % KX : (a == 1 ? (k / KX) % KY : k / (KX * KY));
}
__device__ __forceinline__ uint32_t extent_of(const Geom& g, int a) {
  return uint32_t(a == 0 ? g.KX : (a == 1 ? g.KY : g.KZ));
}
// dual vertex of the top cell on side sg (0: -, 1: +) of face k along axis a (OMEGA if outside)
__device__ __forceinline__ uint32_t dual_side(const DualG& G, uint32_t k, int a, int sg) {
  const uint32_t c = coord_of(G.g, k, a);
  if (sg ? c + 1 >= extent_of(G.g, a) : c == 0) return G.omega;
  const int64_t st = G.g.stride(a);
  return kidx_vox(G.g, uint32_t(int64_t(k) + (sg ? st : -st)));
}

__global__ void k_dual_parent(const uint32_t* __restrict__ births, const uint8_t* __restrict__ tags,
                              DualG G, uint32_t* __restrict__ parent) {
  const int64_t vv = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (vv > G.omega) return;
  const uint32_t v = uint32_t(vv);
  uint32_t p = v, k;
  if (v < G.omega && top_of_voxel(G.g, v, k) && births[k] != ABSENT_ORD) {
    const uint8_t t = tags[k];
    if (tag_kind(t) == KIND_DOWN) {  // dual apparent pair: hangs under its face's other coface
      const int dir = tag_dir(t);
      const uint32_t f = uint32_t(int64_t(k) + dir_offset(G.g, dir));
      p = dual_side(G, f, dir >> 1, dir & 1);
    }
  }
  parent[v] = p;
}

__device__ __forceinline__ uint32_t d_find(uint32_t* parent, uint32_t v) {
  while (true) {
    const uint32_t p = *(volatile uint32_t*)(parent + v);
    if (p == v) return v;
    const uint32_t pp = *(volatile uint32_t*)(parent + p);
    if (pp != p) atomicCAS(parent + v, p, pp);  // path halving
    v = pp;
  }
}

// faces of dimension D-1: the active axes all odd but one (the normal axis, returned)
__device__ __forceinline__ int face_normal(const Geom& g, uint32_t k) {
  int even = -1, neven = 0;
  for (int a = 0; a < 3; ++a) {
    if (extent_of(g, a) <= 1) continue;
    if (!(coord_of(g, k, a) & 1)) {
      even = a;
      ++neven;
    }
  }
  return neven == 1 ? even : -1;
}

// The same unions enumerated per voxel v (one thread): the face with normal a whose lower corner
// is v (Khalimsky 2v_a on axis a, 2v_b + 1 on the other active axes) joins the cubes with base
// voxels v - e_a and v (OMEGA past the border).  One thread per voxel and three faces instead of
// one thread per Khalimsky cell (C5b: 8x fewer threads, no coordinate decoding per cell).
__global__ void k_dual_absent_vox(const uint32_t* __restrict__ births, DualG G,
                                  uint32_t* parent) {
  const int64_t vv = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (vv >= G.g.nvox) return;
  const uint32_t v = uint32_t(vv);
  const uint32_t nx = uint32_t(G.g.nx), ny = uint32_t(G.g.ny), nz = uint32_t(G.g.nz);
  const uint32_t KX = uint32_t(G.g.KX), KY = uint32_t(G.g.KY);
  const uint32_t r = v / nx;
  const uint32_t c[3] = {v - r * nx, r % ny, r / ny}, n[3] = {nx, ny, nz};
  const uint32_t vst[3] = {1u, nx, nx * ny};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (n[a] <= 1) continue;
    uint32_t K[3];
    bool ok = true;
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      if (b == a) {
        K[b] = 2 * c[b];
      } else if (n[b] > 1) {
        K[b] = 2 * c[b] + 1;
        ok = ok && c[b] + 1 < n[b];
      } else {
        K[b] = 0;
      }
    }
    if (!ok) continue;
    if (__ldg(births + (K[2] * KY + K[1]) * KX + K[0]) != ABSENT_ORD) continue;
    uint32_t x = c[a] > 0 ? v - vst[a] : G.omega, y = c[a] + 1 < n[a] ? v : G.omega;
    while (true) {
      x = d_find(parent, x);
      y = d_find(parent, y);
      if (x == y) break;
      if (x > y) {
        const uint32_t t = x;
        x = y;
        y = t;
      }
      if (atomicCAS(parent + x, x, y) == x) break;
    }
  }
}

// absent faces join their absent sides (larger id = elder root, OMEGA the eldest)
__global__ void k_dual_absent(const uint32_t* __restrict__ births, DualG G, uint32_t* parent) {
  const int64_t kk = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (kk >= G.g.ncells) return;
  const uint32_t k = uint32_t(kk);
  if (births[k] != ABSENT_ORD) return;
  const int n = face_normal(G.g, k);
  if (n < 0) return;
  uint32_t a = dual_side(G, k, n, 0), b = dual_side(G, k, n, 1);
  while (true) {
    a = d_find(parent, a);
    b = d_find(parent, b);
    if (a == b) return;
    if (a > b) {
      const uint32_t t = a;
      a = b;
      b = t;
    }
    if (atomicCAS(parent + a, a, b) == a) return;
  }
}

__global__ void k_dual_edges(const uint32_t* __restrict__ births, const uint8_t* __restrict__ tags,
                             DualG G, const uint32_t* __restrict__ parent, Cand* __restrict__ cand,
                             unsigned int* __restrict__ ncand) {
  const int64_t kk = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  bool emit = false;
  Cand c;
  if (kk < G.g.ncells) {
    const uint32_t k = uint32_t(kk);
    const uint32_t bo = births[k];
    if (bo != ABSENT_ORD && tag_kind(tags[k]) == KIND_RESIDUAL) {
      const int n = face_normal(G.g, k);
      if (n >= 0) {
        const uint32_t ra = parent[dual_side(G, k, n, 0)], rb = parent[dual_side(G, k, n, 1)];
        if (ra != rb) {
          emit = true;
          c.key = ~make_key(bo, k);  // ascending ~key = decreasing key
          c.a = ra;
          c.b = rb;
        }
      }
    }
  }
  const unsigned mask = __ballot_sync(0xFFFFFFFFu, emit);
  if (!mask) return;
  const int lane = threadIdx.x & 31;
  unsigned base = 0;
  if (lane == __ffs(mask) - 1) base = atomicAdd(ncand, __popc(mask));
  base = __shfl_sync(0xFFFFFFFFu, base, __ffs(mask) - 1);
  if (emit) cand[base + __popc(mask & ((1u << lane) - 1))] = c;
}

// key of a dual root (larger = elder): OMEGA the largest, absent top cells next
__device__ __forceinline__ uint64_t dual_root_key(const uint32_t* __restrict__ births, const DualG& G,
                                                  uint32_t v) {
  if (v == G.omega) return ~0ull;
  uint32_t k = 0;
  top_of_voxel(G.g, v, k);
  return make_key(births[k], k);
}

__global__ void k_dual_roots(const uint32_t* __restrict__ births, DualG G,
                             const uint32_t* __restrict__ parent, uint64_t* rootkey, unsigned* nroot,
                             unsigned long long* count) {
  const int64_t vv = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  bool emit = false;
  uint64_t key = 0;
  if (vv <= G.omega) {
    const uint32_t v = uint32_t(vv);
    uint32_t k;
    if (parent[v] == v && (v == G.omega || top_of_voxel(G.g, v, k))) {
      emit = true;
      key = ~dual_root_key(births, G, v);  // ascending = elder first
    }
  }
  const unsigned mask = __ballot_sync(0xFFFFFFFFu, emit);
  if (!mask) return;
  const int lane = threadIdx.x & 31;
  if (count) {
    if (lane == __ffs(mask) - 1) atomicAdd(count, (unsigned long long)__popc(mask));
    return;
  }
  unsigned base = 0;
  if (lane == __ffs(mask) - 1) base = atomicAdd(nroot, __popc(mask));
  base = __shfl_sync(0xFFFFFFFFu, base, __ffs(mask) - 1);
  if (emit) rootkey[base + __popc(mask & ((1u << lane) - 1))] = key;
}

__global__ void k_dual_rank(const uint64_t* __restrict__ rootkey, unsigned nb, DualG G,
                            uint32_t* rank_of) {
  const unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nb) return;
  const uint64_t key = ~rootkey[i];
  rank_of[key == ~0ull ? G.omega : kidx_vox(G.g, key_kidx(key))] = i;
}

// dual record of the edge with complemented key ek whose younger root has key ry
__device__ __forceinline__ uint64_t dual_record(uint64_t ek, uint64_t ry) {
  const uint32_t sigma = ~key_kidx(ek);
  const bool absent = key_ord(ry) == ABSENT_ORD;  // (OMEGA is never the younger root)
  return (uint64_t(sigma) << 32) | (absent ? NONE32 : key_kidx(ry));
}

// Kruskal over the MSF edges in (complemented) key order, elder = smaller rank.
__global__ void __launch_bounds__(H0_THREADS) k_dual_kruskal(
    const uint64_t* __restrict__ keys, const uint32_t* __restrict__ ab,
    const uint32_t* __restrict__ msf, unsigned nmsf, const uint64_t* __restrict__ rootkey,
    unsigned nb, uint64_t* rec, unsigned long long* nrec) {
  extern __shared__ uint32_t sh[];
  uint32_t* par = sh;
  for (unsigned i = threadIdx.x; i < nb; i += H0_THREADS) par[i] = i;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long r = *nrec;
    for (unsigned t = 0; t < nmsf; ++t) {
      const uint32_t e = msf[t];
      const uint32_t a = sfind(par, ab[e] >> 16), b = sfind(par, ab[e] & 0xFFFFu);
      const uint32_t young = a > b ? a : b, old = a > b ? b : a;
      par[young] = old;
      rec[r++] = dual_record(keys[e], ~rootkey[young]);
    }
    *nrec = r;
  }
}

// Device-wide dual merge round (mirror of k_mm_commit: the elder is the LARGER key): an edge
// commits if it is the minimum (in complemented order) at both components, or at the younger one.
__global__ void k_dual_mm_commit(const Cand* cand, unsigned n, const uint32_t* __restrict__ births,
                                 DualG G, uint32_t* parent, const unsigned long long* best,
                                 uint8_t* alive, uint64_t* rec, unsigned long long* nrec) {
  const unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || !alive[i]) return;
  const Cand c = cand[i];
  const bool min_a = best[c.a] == c.key, min_b = best[c.b] == c.key;
  if (!min_a && !min_b) return;
  const uint64_t ka = dual_root_key(births, G, c.a), kb = dual_root_key(births, G, c.b);
  const bool a_young = ka < kb;
  if (!(min_a && min_b) && (a_young ? !min_a : !min_b)) return;
  const uint32_t young = a_young ? c.a : c.b, old = a_young ? c.b : c.a;
  parent[young] = old;
  const unsigned long long r = atomicAdd(nrec, 1ull);
  rec[r] = dual_record(c.key, a_young ? ka : kb);
  alive[i] = 2;
}

// All merge rounds (H0 or the dual) in one cooperative launch: the phases of k_mm_find,
// k_mm_commit / k_dual_mm_commit and k_mm_reset separated by grid syncs, looping on the device
// until no candidate is left -- instead of three launches, a memset and a host round trip per
// round (C1: 14 rounds cost ~35 us each on the host path).  Same per-edge logic, so the same
// commits in the same rounds.  ctl: [0]/[1] survivor counters (double-buffered), [2] rounds.
struct MMArgs {
  Cand* cur;
  Cand* nxt;
  const unsigned* n;  // device: the number of candidates (read by the kernel: no host round trip)
  uint32_t* parent;
  unsigned long long* best;  // 2 * nbest entries (two buffers, by round parity)
  unsigned nbest;
  uint8_t* alive;            // n entries, 1 on entry
  const uint32_t* births;
  Geom g;
  DualG G;
  uint8_t* tags;
  uint64_t* rec;
  unsigned long long* nrec;
  unsigned* ctl;
};
template <bool DUAL>
__global__ void __launch_bounds__(256) k_mm_rounds(MMArgs A) {
  // Two grid syncs per round: the candidate list is never compacted (alive bit 0: undecided,
  // bit 1: did an atomicMin last round), and the per-root minima alternate between two buffers
  // (A.best, A.best + A.nbest) by round parity, the previous round's buffer being reset by the
  // candidates that touched it while the current one is filled.
  cg::grid_group grid = cg::this_grid();
  const unsigned gt = blockIdx.x * blockDim.x + threadIdx.x, gs = gridDim.x * blockDim.x;
  Cand* cur = A.cur;
  const unsigned n = *A.n;
  unsigned rounds = 0;
  while (true) {
    unsigned long long* bc = A.best + (rounds & 1) * A.nbest;
    unsigned long long* bp = A.best + ((rounds + 1) & 1) * A.nbest;
    for (unsigned i = gt; i < n; i += gs) {  // find (and reset the previous round's minima)
      uint8_t st = A.alive[i];
      if (!st) continue;
      Cand c = cur[i];
      if (st & 2) {
        bp[c.a] = NONE64;
        bp[c.b] = NONE64;
        st &= 1;
      }
      if (st & 1) {
        const uint32_t a = uf_find(A.parent, c.a), b = uf_find(A.parent, c.b);
        if (a == b) {  // connected through strictly smaller edges: positive
          st = 0;
        } else {
          cur[i].a = a;
          cur[i].b = b;
          atomicMin(bc + a, (unsigned long long)c.key);
          atomicMin(bc + b, (unsigned long long)c.key);
          st = 3;
        }
      }
      A.alive[i] = st;
    }
    grid.sync();
    unsigned left = 0;
    for (unsigned i = gt; i < n; i += gs) {  // commit (see k_mm_commit / k_dual_mm_commit)
      if (A.alive[i] != 3) continue;
      const Cand c = cur[i];
      const bool min_a = bc[c.a] == c.key, min_b = bc[c.b] == c.key;
      bool commit = false;
      uint64_t ka = 0, kb = 0;
      bool a_young = false;
      if (min_a || min_b) {
        if (DUAL) {
          ka = dual_root_key(A.births, A.G, c.a);
          kb = dual_root_key(A.births, A.G, c.b);
        } else {
          const uint32_t xa = vox_kidx(A.g, c.a), xb = vox_kidx(A.g, c.b);
          ka = make_key(A.births[xa], xa);
          kb = make_key(A.births[xb], xb);
        }
        a_young = DUAL ? ka < kb : ka > kb;
        commit = (min_a && min_b) || (a_young ? min_a : min_b);
      }
      if (!commit) {
        ++left;
        continue;
      }
      const uint32_t young = a_young ? c.a : c.b, old = a_young ? c.b : c.a;
      A.parent[young] = old;
      const unsigned long long r = atomicAdd(A.nrec, 1ull);
      if (DUAL) {
        A.rec[r] = dual_record(c.key, a_young ? ka : kb);
      } else {
        A.tags[key_kidx(c.key)] = make_tag(KIND_CLEARED, 0);  // a death edge: cleared for dim 1
        A.rec[r] = (uint64_t(key_kidx(a_young ? ka : kb)) << 32) | key_kidx(c.key);
      }
      A.alive[i] = 2;  // decided; its minima are reset next round
    }
    unsigned* cnt = A.ctl + (rounds & 1);
    left = __reduce_add_sync(0xFFFFFFFFu, left);
    if ((threadIdx.x & 31) == 0 && left) atomicAdd(cnt, left);
    if (gt == 0) A.ctl[(rounds + 1) & 1] = 0;  // the next round's counter (read before 2 syncs)
    grid.sync();
    ++rounds;
    if (__ldcg(cnt) == 0) break;
  }
  if (gt == 0) A.ctl[2] = rounds;
}

// Launches the merge rounds on the *n_dev candidates (cand, spare buffer cand2, both holding
// n_max); ctl (4 device unsigned, zeroed by the caller) receives the number of rounds in ctl[2].
// No host synchronisation: the caller reads ctl[2] with its next scalar read.
template <bool DUAL>
void mm_rounds(Cand* cand, Cand* cand2, const unsigned* n_dev, int64_t n_max, uint32_t* parent,
               unsigned long long* best, unsigned nbest, uint8_t* alive, const uint32_t* births,
               const Geom& g,
               const DualG& G, uint8_t* tags, uint64_t* rec, unsigned long long* nrec,
               unsigned* ctl, Workspace& ws) {
  cudaStream_t s = ws.stream();
  static thread_local int occ[2] = {0, 0};
  static thread_local int nsm = 0;
  if (!nsm) {
    int dev = 0;
    CR_CUDA(cudaGetDevice(&dev));
    CR_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  }
  if (!occ[DUAL]) {
    CR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ[DUAL], k_mm_rounds<DUAL>, 256, 0));
    if (occ[DUAL] < 1) throw Error{CR_EINTERNAL, "k_mm_rounds cannot be resident"};
  }
  int64_t blocks = (n_max + 255) / 256;
  const int64_t cap = int64_t(nsm) * occ[DUAL];
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  CR_CUDA(cudaMemsetAsync(alive, 1, size_t(n_max > 0 ? n_max : 1), s));
  MMArgs A{cand, cand2, n_dev, parent, best, nbest, alive, births, g, G, tags, rec, nrec, ctl};
  void* args[] = {&A};
  CR_CUDA(cudaLaunchCooperativeKernel((void*)k_mm_rounds<DUAL>, dim3(unsigned(blocks)), dim3(256),
                                      args, 0, s));
  ++g_launch_count;
}

// Returns false (doing nothing) if the dual graph has more than max_basins roots: its union-find
// then runs on one CTA's shared memory only up to SMEM_BASINS roots, and the device-wide
// mutual-minimum rounds degenerate on the dual graph (the outside vertex absorbs components one
// per round), so the caller reduces the coboundary matrix instead.
bool top_dual(GeneralState& S, int d, Workspace& ws, HostScalars& hs, cr_stats& st,
              unsigned max_basins) {
  cudaStream_t s = ws.stream();
  const Geom& g = S.g;
  const int B = 256;
  DualG G{g, uint32_t(g.nvox)};
  const int64_t nv = g.nvox + 1;
  S.R.rec[d] = ws.alloc<uint64_t>(st.cells[d] + 1);
  S.R.n[d] = 0;
  unsigned long long* cnt = ws.alloc<unsigned long long>(8);
  CR_CUDA(cudaMemsetAsync(cnt, 0, 8 * sizeof(unsigned long long), s));
  uint32_t* parent = ws.alloc<uint32_t>(nv);
  k_dual_parent<<<grid_for(nv, B), B, 0, s>>>(S.births, S.tags, G, parent);
  CR_CHECK_LAUNCH();
  if (std::getenv("CR_DUAL_ABSENT_CELLS"))  // the per-cell form (cross-check)
    k_dual_absent<<<grid_for(g.ncells, B), B, 0, s>>>(S.births, G, parent);
  else
    k_dual_absent_vox<<<grid_for(g.nvox, B), B, 0, s>>>(S.births, G, parent);
  CR_CHECK_LAUNCH();
  k_pointer_jump<<<grid_for(nv, B), B, 0, s>>>(parent, nv);
  CR_CHECK_LAUNCH();
  Cand* cand = ws.alloc<Cand>(st.cells[d] + 1);
  unsigned* ncand = reinterpret_cast<unsigned*>(cnt);
  k_dual_edges<<<grid_for(g.ncells, B), B, 0, s>>>(S.births, S.tags, G, parent, cand, ncand);
  CR_CHECK_LAUNCH();
  k_dual_roots<<<grid_for(nv, B), B, 0, s>>>(S.births, G, parent, nullptr, nullptr, cnt + 1);
  CR_CHECK_LAUNCH();
  CR_CUDA(cudaMemcpyAsync(hs.p, cnt, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  CR_CUDA(cudaStreamSynchronize(s));
  unsigned n = unsigned(hs.p[0] & 0xFFFFFFFFu);
  const unsigned nb = unsigned(hs.p[1]);
  if (nb > max_basins) {
    ws.release(cand);
    ws.release(parent);
    return false;
  }
  st.columns[d] = nb;

  unsigned long long* nrec = cnt + 2;
  if (nb > smem_basins_max()) {  // device-wide merge rounds
    unsigned long long* best = ws.alloc<unsigned long long>(2 * nv);
    CR_CUDA(cudaMemsetAsync(best, 0xFF, 2 * nv * sizeof(unsigned long long), s));
    uint8_t* alive = ws.alloc<uint8_t>(n + 1);
    Cand* cand2 = ws.alloc<Cand>(n + 1);
    unsigned* ctl = reinterpret_cast<unsigned*>(cnt + 6);  // cnt[6], cnt[7]: zeroed above
    mm_rounds<true>(cand, cand2, ncand, n, parent, best, unsigned(nv), alive, S.births, g, G,
                    nullptr, S.R.rec[d], nrec, ctl, ws);
    CR_CUDA(cudaMemcpyAsync(hs.p, cnt + 2, 6 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                            s));
    CR_CUDA(cudaStreamSynchronize(s));
    S.R.n[d] = int64_t(hs.p[0]);
    st.rounds[d] = int64_t(reinterpret_cast<const unsigned*>(hs.p + 4)[2]);
    return true;
  }
  {
    uint64_t* rootkey = ws.alloc<uint64_t>(nb + 1);
    k_dual_roots<<<grid_for(nv, B), B, 0, s>>>(S.births, G, parent, rootkey,
                                               reinterpret_cast<unsigned*>(cnt + 3), nullptr);
    CR_CHECK_LAUNCH();
    sort_keys_u64(rootkey, nb, false, 64, ws);
    uint32_t* rank_of = ws.alloc<uint32_t>(nv);
    k_dual_rank<<<grid_for(nb, B), B, 0, s>>>(rootkey, nb, G, rank_of);
    CR_CHECK_LAUNCH();
    uint64_t* keys = ws.alloc<uint64_t>(n + 1);
    uint32_t* ab = ws.alloc<uint32_t>(n + 1);
    if (n > 0) {
      k_cand_pack<<<grid_for(n, B), B, 0, s>>>(cand, n, rank_of, keys, ab);
      CR_CHECK_LAUNCH();
      uint64_t* k2 = ws.alloc<uint64_t>(n);
      uint32_t* v2 = ws.alloc<uint32_t>(n);
      cub::DoubleBuffer<uint64_t> dk(keys, k2);
      cub::DoubleBuffer<uint32_t> dv(ab, v2);
      size_t tmp = 0;
      CR_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, dk, dv, int(n), 0, 64, s));
      void* t = ws.alloc_bytes(tmp);
      CR_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, dk, dv, int(n), 0, 64, s));
      keys = dk.Current();
      ab = dv.Current();
    }
    uint32_t* act0 = ws.alloc<uint32_t>(n + 1);
    uint32_t* act1 = ws.alloc<uint32_t>(n + 1);
    uint32_t* best32 = ws.alloc<uint32_t>(nb + 1);
    uint32_t* hook = ws.alloc<uint32_t>(nb + 1);
    uint32_t* msf = ws.alloc<uint32_t>(nb + 1);
    unsigned* nmsf = reinterpret_cast<unsigned*>(cnt + 4);
    const size_t smem = size_t(nb > 0 ? nb : 1) * 4;
    CR_CUDA(cudaFuncSetAttribute(k_h0_boruvka, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(smem)));
    CR_CUDA(cudaFuncSetAttribute(k_dual_kruskal, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(smem)));
    k_h0_boruvka<<<1, H0_THREADS, smem, s>>>(ab, n, nb, best32, act0, act1, hook, msf, nmsf,
                                             cnt + 5);
    CR_CHECK_LAUNCH();
    const unsigned nm = read_scalar(nmsf, s, hs);
    if (nm > 1) {
      uint32_t* m2 = ws.alloc<uint32_t>(nm);
      cub::DoubleBuffer<uint32_t> dm(msf, m2);
      size_t tmp = 0;
      CR_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, dm, int(nm), 0, 32, s));
      void* t = ws.alloc_bytes(tmp);
      CR_CUDA(cub::DeviceRadixSort::SortKeys(t, tmp, dm, int(nm), 0, 32, s));
      msf = dm.Current();
    }
    k_dual_kruskal<<<1, H0_THREADS, smem, s>>>(keys, ab, msf, nm, rootkey, nb, S.R.rec[d], nrec);
    CR_CHECK_LAUNCH();
    st.rounds[d] = int64_t(read_scalar(cnt + 5, s, hs));
    S.R.n[d] = int64_t(read_scalar(nrec, s, hs));
  }
  return true;
}

// In a full barcode the reduction of the top dimension is cheap once lower dimensions are cleared;
// the dual union-find wins while its roots fit a fast single-CTA pass (measured: C1 2.7k roots,
// 1.1 vs 2.0 ms; C4 50k roots, 15.8 vs 8.7 ms).
unsigned dual_max_basins() {  // tuning knob CR_DUAL_MAX (measurement); default: always
  const char* e = std::getenv("CR_DUAL_MAX");
  return e ? unsigned(std::strtoul(e, nullptr, 10)) : 0xFFFFFFFFu;
}
bool use_dual(const Geom& g, int d) {
  if (d != g.D - 1 || d < 1) return false;
  const char* e = std::getenv("CR_TOP_REDUCE");  // force the coboundary reduction (cross-checks)
  return !(e && e[0] == '1');
}

// ---------------------------------------------------------------------------------------------
// Output: records -> bars: keep death > birth or essential.
// ---------------------------------------------------------------------------------------------
__global__ void k_bar_flags(const uint64_t* __restrict__ rec, int64_t n,
                            const uint32_t* __restrict__ births, uint32_t* __restrict__ flag) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t r = rec[i];
  uint32_t b = uint32_t(r >> 32), d = uint32_t(r);
  flag[i] = (d == NONE32) || (births[d] > births[b]);
}

__global__ void k_bar_scatter(const uint64_t* __restrict__ rec, int64_t n,
                              const uint32_t* __restrict__ births,
                              const uint32_t* __restrict__ flag, const uint32_t* __restrict__ pos,
                              int dim, const long long* __restrict__ dbase, int64_t cap,
                              cr_pair* out, uint32_t* out_cells) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n || !flag[i]) return;
  int64_t o = dbase[dim] + pos[i];
  if (o >= cap) return;
  uint64_t r = rec[i];
  uint32_t b = uint32_t(r >> 32), d = uint32_t(r);
  cr_pair p;
  p.dim = dim;
  p.birth = float_of_ord(births[b]);
  p.death = d == NONE32 ? __int_as_float(0x7F800000) : float_of_ord(births[d]);
  out[o] = p;
  if (out_cells) out_cells[o] = b;
}

// running output offsets of emit_bars: dbase[d + 1] = dbase[d] + bars of dimension d
__global__ void k_bar_advance(const uint32_t* __restrict__ pos, int64_t n, long long* dbase,
                              int d) {
  dbase[d + 1] = dbase[d] + (pos ? (long long)pos[n] : 0ll);
}

__global__ void k_partner_init(const uint32_t* __restrict__ births, const uint8_t* __restrict__ tags,
                               Geom g, uint32_t* __restrict__ partner) {
  int64_t kk = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (kk >= g.ncells) return;
  uint32_t k = uint32_t(kk);
  if (births[k] == ABSENT_ORD) {
    partner[k] = CR_PARTNER_ABSENT;
    return;
  }
  uint8_t t = tags[k];
  uint8_t kind = tag_kind(t);
  partner[k] = (kind == KIND_UP || kind == KIND_DOWN)
                   ? uint32_t(int64_t(k) + dir_offset(g, tag_dir(t)))
                   : CR_PARTNER_ESSENTIAL;
}

__global__ void k_partner_records(const uint64_t* __restrict__ rec, int64_t n,
                                  uint32_t* __restrict__ partner) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t r = rec[i];
  uint32_t b = uint32_t(r >> 32), d = uint32_t(r);
  if (d != NONE32) {
    partner[b] = d;
    partner[d] = b;
  }
}

}  // namespace

// ---------------------------------------------------------------------------------------------
// Dimensions 1..dmax after H0: dimension 1 by the cohomology reduction, whose
// pivots clear dimension 2, then the top dimension by duality.  Alternative (CR_K5_HOM=1, 3D):
// the top dimension 2 by duality first (it needs no clearing), then dimension 1 by the HOMOLOGY
// reduction of the square columns with the clearing of the squares that create a 2-class (the
// twist).  Its reduced columns are 1-cycles: on C4 the entry work halves (210 M -> 115 M entries,
// heaviest column 55 M -> 10.6 M) but the additions grow (423 k -> 545 k) and the critical chain
// of dependent additions is as long (366 vs 363 rounds): 168 vs 174 ms, C5 1.63 vs 1.76 s, so
// cohomology stays the default.  Both give the same pairing (unique given reading R1).
void reduce_dims(GeneralState& S, const Geom& g, int dmax, Workspace& ws, HostScalars& hs,
                 cr_stats& st) {
  static const char* names[4] = {"", "reduce_d1", "reduce_d2", "reduce_d3"};
  cudaStream_t s = ws.stream();
  const char* e = std::getenv("CR_K5_HOM");
  const bool hom1 = g.D == 3 && dmax >= 1 && use_dual(g, 2) && e && e[0] == '1';
  if (hom1) {
    if (!top_dual(S, 2, ws, hs, st, 0xFFFFFFFFu)) throw Error{CR_EINTERNAL, "top dimension"};
    prof_mark(s, names[2]);
    mark_cleared_births(S, 2, ws);
    reduce_dimension(S, 1, ws, hs, st, /*hom=*/true);
    prof_mark(s, names[1]);
    return;
  }
  for (int d = 1; d <= dmax; ++d) {
    if (!(use_dual(g, d) && top_dual(S, d, ws, hs, st, dual_max_basins())))
      reduce_dimension(S, d, ws, hs, st);
    prof_mark(s, names[d]);
  }
}

void run_general(const float* image, const Geom& g, int dmax, Workspace& ws, HostScalars& hs,
                 GeneralState& S, cr_stats& st) {
  cudaStream_t s = ws.stream();
  S.g = g;
  const int B = 256;
  S.births = ws.alloc<uint32_t>(g.ncells);
  S.tags = ws.alloc<uint8_t>(g.ncells);
  unsigned long long* cnt = ws.alloc<unsigned long long>(32);
  CR_CUDA(cudaMemsetAsync(cnt, 0, 32 * sizeof(unsigned long long), s));
  int* nan_flag = reinterpret_cast<int*>(cnt + 31);

  // Default: K1 + K2 in one kernel (k_filtration).  Variants for cross-checks and measurement
  // (profiles/r01/s3: C5 K1+K2 = 0.52 + 3.60 ms as k_births + k_apparent (CR_K12_OLD),
  // 1.91 + 1.76 fused births+codes, 0.52 + 1.66 + 1.76 split): CR_K12_OLD, CR_K12_FUSED,
  // CR_K12_SPLIT, CR_K2_TWOPASS, CR_K2_ONEPASS.
  const bool k12_old = !(std::getenv("CR_K12_FUSED") || std::getenv("CR_K12_SPLIT"));
  const bool k12_sep = std::getenv("CR_K12_OLD") || std::getenv("CR_K2_ONEPASS") ||
                       std::getenv("CR_K2_TWOPASS") || !k12_old;
  if (!k12_sep) {  // default: K1 + K2 in one streaming kernel
    const KfLaunch L = kf_launch(g);
    static thread_local int kf_attr_dev = -1;
    if (kf_attr_dev != ws.device()) {
      CR_CUDA(cudaFuncSetAttribute(k_filtration, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(sizeof(KfSmem))));
      kf_attr_dev = ws.device();
    }
    k_filtration<<<L.grid, KF_THREADS, sizeof(KfSmem), s>>>(image, kf_params(g, L.zc), S.births,
                                                            S.tags, cnt, nan_flag);
    CR_CHECK_LAUNCH();
    prof_mark(s, "filtration");
  } else if (!k12_old && std::getenv("CR_K12_SPLIT")) {
    // K1 (births) alone, then K2 as codes (z-streaming) + tags from codes
    uint8_t* code = ws.alloc<uint8_t>(g.ncells + 4);
    k_births<<<k_births_grid(g), 256, 0, s>>>(image, g, S.births, cnt + 4, nan_flag);
    CR_CHECK_LAUNCH();
    prof_mark(s, "births");
    k_codes_z<<<k2z_grid(g), 256, 0, s>>>(S.births, g, code);
    CR_CHECK_LAUNCH();
    k_tags_codes<<<grid_for((g.ncells + 3) / 4, 256), 256, 0, s>>>(code, g, S.tags, cnt + 0);
    CR_CHECK_LAUNCH();
    ws.release(code);
  } else if (!k12_old) {
    // K1 + K2a fused (births and direction codes), then K2b (tags from codes)
    uint8_t* code = ws.alloc<uint8_t>(g.ncells + 4);
    k_births_codes<<<k1c_grid(g), K1C_THREADS, 0, s>>>(image, g, S.births, code, cnt + 4, nan_flag);
    CR_CHECK_LAUNCH();
    prof_mark(s, "births");
    k_tags_codes<<<grid_for((g.ncells + 3) / 4, 256), 256, 0, s>>>(code, g, S.tags, cnt + 0);
    CR_CHECK_LAUNCH();
    ws.release(code);
  } else {
  k_births<<<k_births_grid(g), 256, 0, s>>>(image, g, S.births, cnt + 4, nan_flag);
  CR_CHECK_LAUNCH();
  prof_mark(s, "births");
  if (std::getenv("CR_K2_ONEPASS")) {  // the one-kernel definition (cross-check in tests)
    k_tags<<<grid_for(g.ncells, B), B, 0, s>>>(S.births, g, S.tags, cnt + 0);
    CR_CHECK_LAUNCH();
  } else if (std::getenv("CR_K2_TWOPASS")) {  // codes in HBM, then tags (cross-check)
    uint8_t* code = ws.alloc<uint8_t>(g.ncells);
    k_codes_z<<<k2z_grid(g), 256, 0, s>>>(S.births, g, code);
    CR_CHECK_LAUNCH();
    k_tags2<<<k2_grid(g), 256, 0, s>>>(code, g, S.tags, cnt + 0);
    CR_CHECK_LAUNCH();
    ws.release(code);
  } else {
    k_apparent<<<k2f_grid(g), K2F_THREADS, 0, s>>>(S.births, g, S.tags, cnt + 0);
    CR_CHECK_LAUNCH();
  }
  }
  if (k12_sep) prof_mark(s, "apparent");

  if (S.top_only) {  // the top dimension alone (--top_dim): no H0, no clearing
    CR_CUDA(cudaMemcpyAsync(hs.p, cnt, 32 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    CR_CUDA(cudaStreamSynchronize(s));
    if (*reinterpret_cast<int*>(hs.p + 31)) throw Error{CR_EINVAL, "NaN in image"};
    for (int d = 0; d < 4; ++d) {
      st.apparent[d] = int64_t(hs.p[d]);
      st.cells[d] = int64_t(hs.p[4 + d]);
    }
    if (g.D < 2 || top_dual(S, g.D - 1, ws, hs, st, 0xFFFFFFFFu)) {
      prof_mark(s, "top_dual");
      return;
    }
    // too many dual roots for the one-CTA union-find: the full pipeline (the top dimension's
    // zero columns are essential only given the clearing by the dimensions below)
    S.top_only = false;
  }

  // ---- H0
  uint32_t* parent = ws.alloc<uint32_t>(g.nvox);
  k_h0_parent<<<grid_for(g.nvox, B), B, 0, s>>>(S.births, S.tags, g, parent);
  CR_CHECK_LAUNCH();
  k_pointer_jump<<<grid_for(g.nvox, B), B, 0, s>>>(parent, g.nvox);
  CR_CHECK_LAUNCH();
  k_count_basins<<<grid_for(g.nvox, B), B, 0, s>>>(S.births, S.tags, g, parent, cnt + 8);
  CR_CHECK_LAUNCH();

  // NaN check + counts (one sync)
  CR_CUDA(cudaMemcpyAsync(hs.p, cnt, 32 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  CR_CUDA(cudaStreamSynchronize(s));
  if (*reinterpret_cast<int*>(hs.p + 31)) throw Error{CR_EINVAL, "NaN in image"};
  for (int d = 0; d < 4; ++d) {
    st.apparent[d] = int64_t(hs.p[d]);
    st.cells[d] = int64_t(hs.p[4 + d]);
  }
  st.columns[0] = int64_t(hs.p[8]);
  const int64_t nedges = st.cells[1];

  Cand* cand = ws.alloc<Cand>(nedges);
  Cand* cand2 = ws.alloc<Cand>(nedges);
  unsigned* ncand = reinterpret_cast<unsigned*>(cnt + 12);
  k_h0_edges<<<grid_for(g.ncells, B), B, 0, s>>>(S.births, S.tags, g, parent, cand, ncand);
  CR_CHECK_LAUNCH();

  // vertex records: at most one per finite vertex
  S.R.rec[0] = ws.alloc<uint64_t>(st.cells[0]);
  unsigned long long* nrec0 = cnt + 13;
  const unsigned nb = unsigned(st.columns[0]);
  if (nb <= smem_basins_max()) {
    // few basins: shared-memory rounds in one CTA
    const unsigned n = read_scalar(ncand, s, hs);
    uint64_t* rootkey = ws.alloc<uint64_t>(nb + 1);
    unsigned* nroot = reinterpret_cast<unsigned*>(cnt + 15);
    k_collect_roots<<<grid_for(g.nvox, B), B, 0, s>>>(S.births, g, parent, rootkey, nroot);
    CR_CHECK_LAUNCH();
    sort_keys_u64(rootkey, nb, false, 64, ws);
    uint32_t* rank_of = ws.alloc<uint32_t>(g.nvox);
    k_rank_roots<<<grid_for(nb, B), B, 0, s>>>(rootkey, nb, g, rank_of);
    CR_CHECK_LAUNCH();
    uint64_t* keys = ws.alloc<uint64_t>(n + 1);
    uint32_t* ab = ws.alloc<uint32_t>(n + 1);
    if (n > 0) {
      k_cand_pack<<<grid_for(n, B), B, 0, s>>>(cand, n, rank_of, keys, ab);
      CR_CHECK_LAUNCH();
      uint64_t* k2 = ws.alloc<uint64_t>(n);
      uint32_t* v2 = ws.alloc<uint32_t>(n);
      cub::DoubleBuffer<uint64_t> dk(keys, k2);
      cub::DoubleBuffer<uint32_t> dv(ab, v2);
      size_t tmp = 0;
      CR_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, dk, dv, int(n), 0, 64, s));
      void* t = ws.alloc_bytes(tmp);
      CR_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, dk, dv, int(n), 0, 64, s));
      keys = dk.Current();
      ab = dv.Current();
    }
    uint32_t* act0 = ws.alloc<uint32_t>(n + 1);
    uint32_t* act1 = ws.alloc<uint32_t>(n + 1);
    uint32_t* best32 = ws.alloc<uint32_t>(nb + 1);
    uint32_t* hook = ws.alloc<uint32_t>(nb + 1);
    uint32_t* msf = ws.alloc<uint32_t>(nb + 1);
    unsigned* nmsf = reinterpret_cast<unsigned*>(cnt + 17);
    const size_t smem = size_t(nb > 0 ? nb : 1) * 4;
    CR_CUDA(cudaFuncSetAttribute(k_h0_boruvka, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(smem)));
    CR_CUDA(cudaFuncSetAttribute(k_h0_kruskal, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(smem)));
    k_h0_boruvka<<<1, H0_THREADS, smem, s>>>(ab, n, nb, best32, act0, act1, hook, msf, nmsf,
                                             cnt + 16);
    CR_CHECK_LAUNCH();
    const unsigned nm = read_scalar(nmsf, s, hs);
    if (nm > 1) {  // Kruskal order = edge index order (candidates are sorted by key)
      uint32_t* m2 = ws.alloc<uint32_t>(nm);
      cub::DoubleBuffer<uint32_t> dm(msf, m2);
      size_t tmp = 0;
      CR_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, dm, int(nm), 0, 32, s));
      void* t = ws.alloc_bytes(tmp);
      CR_CUDA(cub::DeviceRadixSort::SortKeys(t, tmp, dm, int(nm), 0, 32, s));
      msf = dm.Current();
    }
    k_h0_kruskal<<<1, H0_THREADS, smem, s>>>(keys, ab, msf, nm, rootkey, nb, S.tags, S.R.rec[0],
                                             nrec0);
    CR_CHECK_LAUNCH();
    CR_CUDA(cudaMemcpyAsync(hs.p, cnt + 13, 4 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    CR_CUDA(cudaStreamSynchronize(s));
    S.R.n[0] = int64_t(hs.p[0]);
    st.rounds[0] = int64_t(hs.p[3]);
    prof_mark(s, "h0");
    ws.release(cand);
    ws.release(cand2);
    ws.release(parent);
    reduce_dims(S, g, dmax, ws, hs, st);
    return;
  }
  unsigned long long* best = ws.alloc<unsigned long long>(2 * g.nvox);
  CR_CUDA(cudaMemsetAsync(best, 0xFF, 2 * g.nvox * sizeof(unsigned long long), s));
  uint8_t* alive = ws.alloc<uint8_t>(nedges);
  unsigned* ctl = reinterpret_cast<unsigned*>(cnt + 20);  // cnt[20], cnt[21]: zeroed at the start
  mm_rounds<false>(cand, cand2, ncand, nedges, parent, best, unsigned(g.nvox), alive, S.births, g,
                   DualG{g, uint32_t(g.nvox)}, S.tags, S.R.rec[0], nrec0, ctl, ws);
  // flatten once more so that roots are exact, then essential classes
  k_pointer_jump<<<grid_for(g.nvox, B), B, 0, s>>>(parent, g.nvox);
  CR_CHECK_LAUNCH();
  k_h0_essential<<<grid_for(g.nvox, B), B, 0, s>>>(S.births, g, parent, S.R.rec[0], nrec0,
                                                    nullptr);
  CR_CHECK_LAUNCH();
  CR_CUDA(cudaMemcpyAsync(hs.p, cnt + 13, 9 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                          s));
  CR_CUDA(cudaStreamSynchronize(s));
  S.R.n[0] = int64_t(hs.p[0]);
  st.rounds[0] = int64_t(reinterpret_cast<const unsigned*>(hs.p + 7)[2]);
  prof_mark(s, "h0");
  ws.release(cand);
  ws.release(cand2);
  ws.release(best);
  ws.release(alive);
  ws.release(parent);

  reduce_dims(S, g, dmax, ws, hs, st);
}

int64_t emit_bars(const GeneralState& S, int maxdim, cr_pair* out, uint32_t* out_cells,
                  int64_t cap, Workspace& ws, HostScalars& hs, cr_stats& st) {
  cudaStream_t s = ws.stream();
  const int B = 256;
  // one host read at the end: the output offset of each dimension is kept on the device
  const int dl = maxdim < 3 ? maxdim : 3;
  long long* dbase = ws.alloc<long long>(5);
  CR_CUDA(cudaMemsetAsync(dbase, 0, 5 * sizeof(long long), s));
  int kb = 1;  // significant bits of a kidx: records sort by birth kidx (distinct per dimension)
  while (kb < 32 && (int64_t(1) << kb) < S.g.ncells) ++kb;
  for (int d = 0; d <= dl; ++d) {
    int64_t n = S.R.n[d];
    if (n == 0 || !S.R.rec[d]) {
      k_bar_advance<<<1, 1, 0, s>>>(nullptr, 0, dbase, d);
      CR_CHECK_LAUNCH();
      continue;
    }
    sort_keys_u64(S.R.rec[d], n, false, 32 + kb, ws, 32);
    uint32_t* flag = ws.alloc<uint32_t>(n + 1);
    uint32_t* pos = ws.alloc<uint32_t>(n + 1);
    k_bar_flags<<<grid_for(n, B), B, 0, s>>>(S.R.rec[d], n, S.births, flag);
    CR_CHECK_LAUNCH();
    CR_CUDA(cudaMemsetAsync(flag + n, 0, sizeof(uint32_t), s));
    exclusive_sum_u32(flag, pos, n + 1, ws);
    k_bar_scatter<<<grid_for(n, B), B, 0, s>>>(S.R.rec[d], n, S.births, flag, pos, d, dbase, cap,
                                               out, out_cells);
    CR_CHECK_LAUNCH();
    k_bar_advance<<<1, 1, 0, s>>>(pos, n, dbase, d);
    CR_CHECK_LAUNCH();
    ws.release(flag);
    ws.release(pos);
  }
  CR_CUDA(cudaMemcpyAsync(hs.p, dbase, 5 * sizeof(long long), cudaMemcpyDeviceToHost, s));
  CR_CUDA(cudaStreamSynchronize(s));
  for (int d = 0; d <= dl; ++d) st.pairs[d] = int64_t(hs.p[d + 1] - hs.p[d]);
  prof_mark(s, "emit");
  return int64_t(hs.p[dl + 1]);
}

void emit_partner(const GeneralState& S, uint32_t* partner, Workspace& ws) {
  cudaStream_t s = ws.stream();
  const int B = 256;
  k_partner_init<<<grid_for(S.g.ncells, B), B, 0, s>>>(S.births, S.tags, S.g, partner);
  CR_CHECK_LAUNCH();
  for (int d = 0; d < 4; ++d)
    if (S.R.n[d] > 0) {
      k_partner_records<<<grid_for(S.R.n[d], B), B, 0, s>>>(S.R.rec[d], S.R.n[d], partner);
      CR_CHECK_LAUNCH();
    }
}

}  // namespace cr
