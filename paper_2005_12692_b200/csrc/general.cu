// general.cu -- the general (1D/2D/3D, one image) path: K1 filtration, K2 apparent pairs,
// K4 dimension-0 pairing (union-find with the elder rule), bar/partner emission.
// The dims >= 1 reduction (K5) is in reduce.cu.
#include <cooperative_groups.h>

#include <cuda.h>
#include <cudaTypedefs.h>

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


// ---------------------------------------------------------------------------------------------
// K1 + K2 fused (the default): births AND apparent-pair tags of every cell from one read of the
// image (PAPER.md:97-108 for the births, PAPER.md:44-45 for the apparent pairs).  A thread owns
// two voxel columns (x, y) and (x, y+1) and walks them along z; its unit of work is the voxel
// block B(x,y,z) = the 8 cells (2x+i, 2y+j, 2z+k), i,j,k in {0,1},
// whose births are maxima over the voxels (x..x+i, y..y+j, z..z+k): with the "plane cells"
// P(z) = {V, Ex, Ey, Sxy} of a block, the k=1 cells are max(P(z), P(z+1)) (4 max per block).
// A cell's 6 Khalimsky neighbours lie in its own block or in the blocks at x+-1 (neighbouring
// lanes: shuffles), y+-1 (the thread's other row, or the neighbouring warp's: shared memory) and
// z+-1 (the thread's previous / next step: registers), so codes and tags are formed from
// registers with one __syncthreads per step.  Lanes 0 and 31, warp 0's first row and the last
// warp's second row are halo (their blocks' codes feed the tags of the inner 30 x K2_ROWS
// columns); lane 31 also loads the x+1 voxels its i=1 cells need.  Step z completes B(z-1)'s
// births (writes them), forms B(z-1)'s codes and B(z-2)'s tags (writes them).
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
constexpr uint8_t CODE_ABSENT = 0x40;  // code bit 6: the cell is absent (+inf birth)
struct KfLaunch {
  unsigned grid;
  int zc;
};
#ifndef KF_ZC0
#define KF_ZC0 64  // planes a CTA walks (halved while the grid is below 4 CTAs per SM)
#endif
inline KfLaunch kf_launch(const Geom& g, int rows) {
  const int64_t xy = ((g.nx + 29) / 30) * ((g.ny + rows - 1) / rows);
  int zc = KF_ZC0;
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
  // a (positive) NaN would order above +inf and make the cells past the grid present: it is
  // clamped to +inf's key (the call fails with CR_EINVAL anyway; this keeps it memory-safe)
  return min(u ^ (uint32_t(int32_t(u) >> 31) | 0x80000000u), ABSENT_ORD);
}

__device__ __forceinline__ void kf_cp4(uint32_t saddr, const float* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(saddr), "l"(g));
}
__device__ __forceinline__ void kf_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void kf_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

constexpr int KF_PF = 3, KF_RING = KF_PF + 1;  // voxel planes in flight, ring slots
constexpr uint32_t KF_RCAP = 1024;  // residual edges a CTA stages in shared memory

// TMA ring (nx % 4 == 0: the tensor map's row pitch must be a multiple of 16 B): one elected
// thread loads a CTA's (KF_TCOLS x K2_VROWS) voxel box of a plane with cp.async.bulk.tensor
// against the slot's mbarrier; out-of-image voxels arrive as 0 and are replaced by +inf on read.
__device__ __forceinline__ void kf_mbar_init(uint32_t bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar));
}
__device__ __forceinline__ void kf_tma_plane(uint32_t dst, const CUtensorMap* map, int x, int y,
                                             int z, uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(dst),
      "l"(map), "r"(x), "r"(y), "r"(z), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void kf_mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra W;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}

struct KfP {  // 32-bit geometry for k_filtration (image < 2^32 voxels, Khalimsky grid < 2^32 cells)
  uint32_t nx, ny, nz, KX, KXY, plane, XB, YB, zc;
  uint32_t zb0;  // first z-chunk of this launch
  // batches read unstacked: stacked plane zz is plane (zz % zper) of image zz / zper, and the
  // separator (+inf) when zz % zper == zimg (zper = zimg + 1); zper == 0: planes as they are
  uint32_t zper, zimg;
  // residual present edges (dimension 1) found by the tags pass: their kidx are appended to res1
  // (count *nres1) -- the H0 candidates and, uncleared, the dim-1 columns; nullptr: none kept
  uint32_t* res1;
  unsigned* nres1;
  uint32_t rcap;  // residual edges staged per CTA (<= KF_RCAP; smaller only to test the overflow)
  // residual present squares (dimension 2; 3D: the faces of the top-dimension dual), likewise
  uint32_t* res2;
  unsigned* nres2;
  // the forests, from the tags of B(z-2): H0 (h0par[v] = the partner edge's other vertex for an
  // apparent (UP) vertex v, else v; the non-apparent present vertices, the basins, appended to
  // basins / *nbasins) and the top-dimension dual (dpar[v] for the top cell with base voxel v:
  // the top cell across its apparent face, OMEGA = nvox past the border or for an absent top
  // cell, else v); nullptr: not built here
  uint32_t* h0par;
  uint32_t* basins;
  unsigned long long* nbasins;
  uint32_t* dpar;
  uint32_t topw, topb;  // the top cell's tag: word j, byte i + 2k of (i, j, k) = active axes
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
  p.YB = 1;  // set by the launcher (rows per CTA)
  p.zc = uint32_t(zc);
  p.zb0 = 0;
  p.zper = p.zimg = 0;
  p.res1 = nullptr;
  p.nres1 = nullptr;
  p.rcap = KF_RCAP;
  p.res2 = nullptr;
  p.nres2 = nullptr;
  p.h0par = p.basins = p.dpar = nullptr;
  p.nbasins = nullptr;
  p.topw = g.ny > 1 ? 1u : 0u;
  p.topb = (g.nx > 1 ? 1u : 0u) + (g.nz > 1 ? 2u : 0u);
  return p;
}

// The kernel: TWO voxel rows per warp (rows y0-1+2w and y0+2w of warp w): the y-neighbour of a
// warp's second row is its first row (registers), so shared memory carries only the rows at warp
// boundaries, and a step's barrier covers twice the voxels.  Small CTAs measured fastest: NW = 4
// warps, 8 rows (6 output rows) x 30 columns per CTA, 128 registers, many CTAs per SM to cover
// each other's barrier waits (round 2's first form: one row per warp, 16 warps, 14 output rows:
// C5b 3.20 ms, C5 1.21 ms -> 2.70 ms, 1.05 ms).
#ifndef K2_NWARPS
#define K2_NWARPS 4  // measured (C5b filtration): 3: 2.98 ms, 4: 2.70, 5: 2.82, 6: 2.93, 8: 2.85, 12: 3.16
#endif
constexpr int K2_NW = K2_NWARPS, K2_THREADS = 32 * K2_NW, K2_ROWS = 2 * K2_NW - 2;
constexpr int K2_VROWS = 2 * K2_NW + 1;
// ring slot: K2_VROWS rows of VCOLS voxels (33 used; the TMA box's rows are 36 wide = 144 B, a
// multiple of 16 B, from a 16-B aligned column: the 33 start at column 1 or 3; slots start on
// 128 B)
template <bool TMA>
struct KfRing {
  static constexpr int VCOLS = TMA ? 36 : 33;
  static constexpr int SLOTW = TMA ? ((K2_VROWS * VCOLS * 4 + 127) / 128) * 32 : K2_VROWS * VCOLS;
  static constexpr uint32_t BOX_BYTES = K2_VROWS * VCOLS * 4;
};
template <bool TMA>
struct alignas(128) Kf2Smem {
  uint32_t v[KF_RING][KfRing<TMA>::SLOTW];  // voxel ring (raw float bits)
  unsigned long long bar[KF_RING];           // TMA: the slots' mbarriers
  uint4 b0[2][K2_NW][32];    // row 0's j=0 births (i + 2k), for the warp below's row 1 (its U)
  uint4 b1[2][K2_NW][32];    // row 1's j=1 births, for the warp above's row 0 (its D)
  uint32_t c0[2][K2_NW][32];  // row 0's j=0 code word
  uint32_t c1[2][K2_NW][32];  // row 1's j=1 code word
  uint32_t cnt[8];
  uint32_t rcnt, rcnt2;       // residual edges / squares listed by the CTA (rbuf* hold the first
  uint32_t rbase, rbase2;     // rcap), their offsets in the global lists
  uint32_t rbuf[KF_RCAP];
  uint32_t rbuf2[KF_RCAP];
  uint32_t bcnt, bbase;       // basins listed by the CTA (bbuf holds the first rcap)
  uint32_t doff[8];           // voxel offset of each direction (the forests)
  uint32_t bbuf[KF_RCAP];
};
inline KfP kf2_params(const Geom& g, int zc) {
  KfP p = kf_params(g, zc);
  p.YB = uint32_t((g.ny + K2_ROWS - 1) / K2_ROWS);
  return p;
}

// The image as a 3D tensor (nx, ny, nzsrc) of float32 for the TMA ring: box = one ring slot
// (36 x K2_VROWS x 1), out-of-bounds voxels zero-filled.  false (-> the cp.async ring) when the
// row pitch is not a multiple of 16 B, the base is not 16-B aligned, or the driver refuses.
bool kf_tensor_map(CUtensorMap* map, const float* image, int64_t nx, int64_t ny, int64_t nzsrc) {
  if (nx % 4 != 0 || (reinterpret_cast<uintptr_t>(image) & 15) != 0) return false;
  static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  if (!encode) return false;
  const cuuint64_t dims[3] = {cuuint64_t(nx), cuuint64_t(ny), cuuint64_t(nzsrc)};
  const cuuint64_t strides[2] = {cuuint64_t(nx) * 4, cuuint64_t(nx * ny) * 4};
  const cuuint32_t box[3] = {cuuint32_t(KfRing<true>::VCOLS), cuuint32_t(K2_VROWS), 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(image), dims, strides,
                box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <bool TMA>
#ifndef K2_MINB
#define K2_MINB 4  // 4 CTAs of 4 warps per SM: <= 128 registers
#endif
__global__ void __launch_bounds__(K2_THREADS, K2_MINB) k_filtration(const float* __restrict__ img,
                                                               const KfP P,
                                                               uint32_t* __restrict__ births,
                                                               uint8_t* __restrict__ tags,
                                                               unsigned long long* __restrict__ cnt,
                                                               int* __restrict__ nan_flag,
                                                               const __grid_constant__ CUtensorMap tmap) {
  extern __shared__ __align__(128) uint4 kf_dyn[];
  Kf2Smem<TMA>& S = *reinterpret_cast<Kf2Smem<TMA>*>(kf_dyn);
  constexpr int VC = KfRing<TMA>::VCOLS;
  const int nx = int(P.nx), ny = int(P.ny), nz = int(P.nz);
  uint32_t blk = blockIdx.x;
  const int xb = int(blk % P.XB);
  blk /= P.XB;
  const int yb = int(blk % P.YB), zb = int(P.zb0 + blk / P.YB);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int x = xb * 30 - 1 + lane;
  const int y0 = yb * K2_ROWS - 1 + 2 * w;  // row 0 of this warp; row 1 is y0 + 1
  const int z0 = zb * int(P.zc), z1 = min(nz, z0 + int(P.zc));
  const bool vx = x >= 0 && x < nx, vx1 = x + 1 < nx, l31 = lane == 31;
  const bool lastw = w == K2_NW - 1;
  bool vy[2], out[2], halo[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int yr = y0 + r;
    vy[r] = yr >= 0 && yr < ny;
    halo[r] = (w == 0 && r == 0) || (lastw && r == 1);  // warp-uniform
    out[r] = vx && vy[r] && lane >= 1 && lane <= 30 && !halo[r];
  }
  const bool vy2 = y0 + 2 < ny;  // the extra ring row (last warp)
  if (threadIdx.x < 8) S.cnt[threadIdx.x] = 0;
  if (threadIdx.x == 0) S.rcnt = S.rcnt2 = S.bcnt = 0;
  if (threadIdx.x < 8) {  // voxel offset of direction d: -x +x -y +y -z +z (two's complement)
    const uint32_t d = threadIdx.x, o = d < 2 ? 1u : (d < 4 ? P.nx : P.plane);
    S.doff[d] = d < 6 ? ((d & 1) ? o : 0u - o) : 0u;
  }
  if (P.dpar && blockIdx.x == 0 && threadIdx.x == 0) P.dpar[P.nx * P.ny * P.nz] = P.nx * P.ny * P.nz;
  constexpr uint32_t INF_BITS = 0x7F800000u;
  // Voxel ring: rows y0(w=0) .. y0(w=0) + 2 NW (the last copied by the last warp), cols x0-1 ..
  // x0+31 (col 32 copied by lane 31).  cp.async ring: a thread copies (x, y0 + r), lane 31 also
  // (x+1, y0 + r); the last warp also the row after its row 1; outside the image: +inf, never
  // copied.  TMA ring: thread 0 loads the whole box; the voxels a thread "owns" (checks for
  // all-+inf planes) are the same.
  const bool o0 = vx && vy[0], o1 = vx && vy[1], o0x = l31 && vx1 && vy[0],
             o1x = l31 && vx1 && vy[1], o2 = lastw && vx && vy2, o2x = lastw && l31 && vx1 && vy2;
  // TMA: the box's first column must be 16-B aligned (x % 4 == 0; measured: other x fault), so
  // it starts at xs = floor4(x0 - 1) and the CTA's columns sit at offset co = x0 - 1 - xs (1 or 3)
  const int xs = (xb * 30 - 1) & ~3, co = TMA ? xb * 30 - 1 - xs : 0;
  uint32_t* const vown = &S.v[0][2 * w * VC + lane + co];
  const uint32_t sv0 = uint32_t(__cvta_generic_to_shared(vown));
  constexpr uint32_t SLOTW = KfRing<TMA>::SLOTW, SLOT = SLOTW * 4, ROW = VC * 4;
  const int c32 = 32 - lane;
  const uint32_t bar0 = uint32_t(__cvta_generic_to_shared(&S.bar[0]));
  const uint32_t ring0 = uint32_t(__cvta_generic_to_shared(&S.v[0][0]));
  uint32_t rmask = 0, phase = 0;  // TMA: slots holding a loaded plane; their mbarrier parities
  if constexpr (TMA) {
    if (threadIdx.x == 0) {
#pragma unroll
      for (int q = 0; q < KF_RING; ++q) kf_mbar_init(bar0 + 8 * q);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
  } else {
#pragma unroll
    for (int q = 0; q < KF_RING; ++q) {
      uint32_t* v = vown + q * SLOTW;
      if (!o0) v[0] = INF_BITS;
      if (!o1) v[VC] = INF_BITS;
      if (l31 && !o0x) v[c32] = INF_BITS;
      if (l31 && !o1x) v[VC + c32] = INF_BITS;
      if (lastw && !o2) v[2 * VC] = INF_BITS;
      if (lastw && l31 && !o2x) v[2 * VC + c32] = INF_BITS;
    }
  }
  const int ys = y0 >= 0 ? y0 : 0;  // copies of row 0 / 1 are offsets of (x, ys) when valid
  const float* gsrc = img + (vx ? uint64_t(uint32_t(ys) * P.nx + uint32_t(x)) : 0ull);
  const int d0 = y0 >= 0 ? 0 : 1;   // y0 = -1 only for warp 0's halo row 0 (never copied)
  // source plane of the next stacked plane >= 0 this thread issues (issue() is called for
  // consecutive planes): image pb, plane pl of its period (one division here, increments after)
  const int zfirst = z0 - 2 > 0 ? z0 - 2 : 0;
  uint32_t pb = P.zper ? uint32_t(zfirst) / P.zper : 0u;
  uint32_t pl = P.zper ? uint32_t(zfirst) - pb * P.zper : uint32_t(zfirst);
  auto issue = [&](int zz, uint32_t sl) {
    bool real = zz >= 0 && zz < nz;  // CTA-uniform
    uint32_t src = 0;
    if (zz >= 0) {
      if (P.zper) {
        real = real && pl != P.zimg;  // a separator plane is +inf
        src = pb * P.zimg + pl;
        if (++pl == P.zper) {
          pl = 0;
          ++pb;
        }
      } else {
        src = pl++;
      }
    }
    if constexpr (TMA) {
      real = real && zz <= z1 + 2;  // the last plane the walk reads
      rmask = real ? rmask | (1u << sl) : rmask & ~(1u << sl);
      if (real && threadIdx.x == 0)
        kf_tma_plane(ring0 + sl * SLOT, &tmap, xs, yb * K2_ROWS - 1, int(src),
                     bar0 + 8 * sl, KfRing<TMA>::BOX_BYTES);
    } else {
      if (real) {
        const uint32_t a = sv0 + sl * SLOT;
        const float* p = gsrc + uint64_t(src) * P.plane - (d0 ? P.nx : 0u);
        if (o0) kf_cp4(a, p);
        if (o0x) kf_cp4(a + 4 * c32, p + 1);
        if (o1) kf_cp4(a + ROW, p + P.nx);
        if (o1x) kf_cp4(a + ROW + 4 * c32, p + P.nx + 1);
        if (lastw) {
          if (o2) kf_cp4(a + 2 * ROW, p + 2 * P.nx);
          if (o2x) kf_cp4(a + 2 * ROW + 4 * c32, p + 2 * P.nx + 1);
        }
      } else {
        uint32_t* v = vown + sl * SLOTW;
        if (o0) v[0] = INF_BITS;
        if (o1) v[VC] = INF_BITS;
        if (o0x) v[c32] = INF_BITS;
        if (o1x) v[VC + c32] = INF_BITS;
        if (o2) v[2 * VC] = INF_BITS;
        if (o2x) v[2 * VC + c32] = INF_BITS;
      }
      kf_commit();
    }
  };
  // wait until slot sl's plane has arrived (cp.async: the oldest but KF_PF - 1 groups)
  auto arrive = [&](uint32_t sl) {
    if constexpr (TMA) {
      if (rmask >> sl & 1) {
        kf_mbar_wait(bar0 + 8 * sl, phase >> sl & 1);
        phase ^= 1u << sl;
      }
    } else {
      kf_wait<KF_PF - 1>();
    }
  };
  // TMA: the 4 voxels a row's blocks read are valid (in the image) -- else +inf
  bool m4[2][4];
  m4[0][0] = vx && vy[0], m4[0][1] = vx1 && vy[0], m4[0][2] = vx && vy[1], m4[0][3] = vx1 && vy[1];
  m4[1][0] = vx && vy[1], m4[1][1] = vx1 && vy[1], m4[1][2] = vx && vy2, m4[1][3] = vx1 && vy2;
  const bool mall = m4[0][0] && m4[0][1] && m4[1][0] && m4[1][1] && m4[1][2] && m4[1][3];
  int z = z0 - 2;
#pragma unroll
  for (int q = 0; q < KF_PF; ++q) issue(z + q, uint32_t(q));
  arrive(0);
  __syncthreads();
  // warp-uniform all-absent steps: g1 / g2 = every thread's own voxels (x, y0), (x, y0 + 1) of
  // plane z-1 / z-2 were +inf (then all its cells with base voxel there are absent)
  bool g2 = true, g1 = true;
  const int wm = max(w - 1, 0), wp = min(w + 1, K2_NW - 1);
  bool nan = false;
  uint32_t P0[2][4], Zm[2][4], CC[2][2], CZm[2][2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
#pragma unroll
    for (int q = 0; q < 4; ++q) P0[r][q] = Zm[r][q] = ABSENT_ORD;
    CC[r][0] = CC[r][1] = CZm[r][0] = CZm[r][1] = 0x40404040u;
  }
  uint32_t fin0 = 0, fin1 = 0, up0 = 0, up1 = 0;
  uint32_t rowbase[2];
#pragma unroll
  for (int r = 0; r < 2; ++r)
    rowbase[r] = uint32_t(2 * max(y0 + r, 0)) * P.KX + uint32_t(2 * max(x, 0));
  const bool hx = x + 1 < nx;
  const bool hy[2] = {y0 + 1 < ny, y0 + 2 < ny};
  // the forests: the row's voxel index in its plane; the top cell exists in x / y; the
  // directions (bit = dir: -x +x -y +y) whose top cell two steps away exists
  uint32_t vrow[2], dok[2];
  bool dtop[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int yr = y0 + r;
    vrow[r] = uint32_t(max(yr, 0)) * P.nx + uint32_t(max(x, 0));
    dtop[r] = (nx == 1 || hx) && (ny == 1 || hy[r]);
    dok[r] = (x > 0 ? 1u : 0u) | (x + 2 < nx ? 2u : 0u) | (yr > 0 ? 4u : 0u) |
             (yr + 2 < ny ? 8u : 0u);
  }
  uint32_t rs = 0;
  for (; z <= z1 + 1; ++z) {
    issue(z + KF_PF, (rs + KF_PF) & (KF_RING - 1));
    const uint32_t* v = vown + rs * SLOTW;
    const bool sr = !TMA || (rmask >> rs & 1);
    uint32_t u0[2] = {v[0], v[VC]};  // own voxels (x, y0 + r) of plane z
    if (TMA && !(sr && mall)) {
      u0[0] = sr && m4[0][0] ? u0[0] : INF_BITS;
      u0[1] = sr && m4[1][0] ? u0[1] : INF_BITS;
    }
    const bool g0 = __all_sync(0xFFFFFFFFu, u0[0] == INF_BITS && u0[1] == INF_BITS);
    // a fast step: B(z-2), B(z-1) and plane z's cells of the whole warp are absent, so its births
    // are ABSENT, codes 0x40, tags 0 -- no arithmetic, only the stores and the y-exchange
    const bool fast = g2 && g1 && g0;
    uint32_t Pn[2][4], Bk[2][8];
    const int buf = z & 1;
    if (!fast) {
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const uint32_t* vr = v + r * VC;
        uint32_t u[4] = {u0[r], vr[1], vr[VC], vr[VC + 1]};
        if (TMA && !(sr && mall)) {
#pragma unroll
          for (int q = 0; q < 4; ++q) u[q] = sr && m4[r][q] ? u[q] : INF_BITS;
        }
        const float v00 = __uint_as_float(u[0]), v10 = __uint_as_float(u[1]);
        const float v01 = __uint_as_float(u[2]), v11 = __uint_as_float(u[3]);
        nan |= v00 != v00;
        const float ex = fmaxf(v00, v10);
        Pn[r][0] = kf_ord(v00);
        Pn[r][1] = kf_ord(ex);
        Pn[r][2] = kf_ord(fmaxf(v00, v01));
        Pn[r][3] = kf_ord(fmaxf(ex, fmaxf(v01, v11)));
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          Bk[r][q] = P0[r][q];
          Bk[r][q + 4] = max(P0[r][q], Pn[r][q]);
        }
      }
    } else {
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          Pn[r][q] = ABSENT_ORD;
          Bk[r][q] = Bk[r][q + 4] = ABSENT_ORD;
        }
    }
    // the y-exchange, also from fast warps (their neighbours may not be fast)
    S.b0[buf][w][lane] = make_uint4(Bk[0][0], Bk[0][1], Bk[0][4], Bk[0][5]);
    S.b1[buf][w][lane] = make_uint4(Bk[1][2], Bk[1][3], Bk[1][6], Bk[1][7]);
    S.c0[buf][w][lane] = CC[0][0];
    S.c1[buf][w][lane] = CC[1][1];
    const uint32_t rn = (rs + 1) & (KF_RING - 1);
    arrive(rn);
    __syncthreads();
    uint32_t NC[2][2], T[2][2];
#pragma unroll
    for (int r = 0; r < 2; ++r) NC[r][0] = NC[r][1] = 0x40404040u, T[r][0] = T[r][1] = 0u;
    if (!fast) {
      // codes of B(z-1), both rows
      uint32_t bmin = ABSENT_ORD;
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int q = 0; q < 8; ++q) bmin = min(bmin, Bk[r][q]);
      if (__any_sync(0xFFFFFFFFu, bmin != ABSENT_ORD)) {
        const uint4 dq = S.b1[buf][wm][lane], uq = S.b0[buf][wp][lane];
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          uint32_t D[4], U[4];
          if (r == 0) {  // below: the warp below's row 1; above: own row 1
            D[0] = dq.x; D[1] = dq.y; D[2] = dq.z; D[3] = dq.w;
            U[0] = Bk[1][0]; U[1] = Bk[1][1]; U[2] = Bk[1][4]; U[3] = Bk[1][5];
          } else {       // below: own row 0; above: the warp above's row 0
            D[0] = Bk[0][2]; D[1] = Bk[0][3]; D[2] = Bk[0][6]; D[3] = Bk[0][7];
            U[0] = uq.x; U[1] = uq.y; U[2] = uq.z; U[3] = uq.w;
          }
          uint32_t L[4], R[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            L[q] = __shfl_up_sync(0xFFFFFFFFu, Bk[r][1 + 2 * q], 1);
            R[q] = __shfl_down_sync(0xFFFFFFFFu, Bk[r][2 * q], 1);
          }
          const uint32_t c000 = kf_code<0, 0, 0>(Bk[r], L, R, D, U, Zm[r], Pn[r]);
          const uint32_t c100 = kf_code<1, 0, 0>(Bk[r], L, R, D, U, Zm[r], Pn[r]);
          const uint32_t c010 = kf_code<0, 1, 0>(Bk[r], L, R, D, U, Zm[r], Pn[r]);
          const uint32_t c110 = kf_code<1, 1, 0>(Bk[r], L, R, D, U, Zm[r], Pn[r]);
          const uint32_t c001 = kf_code<0, 0, 1>(Bk[r], L, R, D, U, Zm[r], Pn[r]);
          const uint32_t c101 = kf_code<1, 0, 1>(Bk[r], L, R, D, U, Zm[r], Pn[r]);
          const uint32_t c011 = kf_code<0, 1, 1>(Bk[r], L, R, D, U, Zm[r], Pn[r]);
          const uint32_t c111 = kf_code<1, 1, 1>(Bk[r], L, R, D, U, Zm[r], Pn[r]);
          NC[r][0] = c000 | (c100 << 8) | (c001 << 16) | (c101 << 24);
          NC[r][1] = c010 | (c110 << 8) | (c011 << 16) | (c111 << 24);
        }
      }
      // tags of B(z-2), rows that are not halo
      const uint32_t CDw = S.c1[buf][wm][lane], CUw = S.c0[buf][wp][lane];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        if (halo[r] ||
            !__any_sync(0xFFFFFFFFu, (CC[r][0] & CC[r][1] & 0x40404040u) != 0x40404040u))
          continue;
        const uint32_t CD = r == 0 ? CDw : CC[0][1], CU = r == 0 ? CC[1][0] : CUw;
        uint32_t CL[2], CR[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          CL[q] = __shfl_up_sync(0xFFFFFFFFu, CC[r][q], 1);
          CR[q] = __shfl_down_sync(0xFFFFFFFFu, CC[r][q], 1);
        }
        T[r][0] = kf_tags_word<0>(CC[r][0], __byte_perm(CL[0], CC[r][0], 0x6341),
                                  __byte_perm(CC[r][0], CR[0], 0x6341), CD, CC[r][1],
                                  __byte_perm(CZm[r][0], CC[r][0], 0x5432),
                                  __byte_perm(CC[r][0], NC[r][0], 0x5432));
        T[r][1] = kf_tags_word<1>(CC[r][1], __byte_perm(CL[1], CC[r][1], 0x6341),
                                  __byte_perm(CC[r][1], CR[1], 0x6341), CC[r][0], CU,
                                  __byte_perm(CZm[r][1], CC[r][1], 0x5432),
                                  __byte_perm(CC[r][1], NC[r][1], 0x5432));
      }
    }
    // stores (as in k_filtration), per row
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      if (!out[r]) continue;
      const int zb1 = z - 1, zb2 = z - 2;
      if (zb1 >= z0 && zb1 < z1) {
        fin0 += (~NC[r][0] >> 6) & 0x01010101u;
        fin1 += (~NC[r][1] >> 6) & 0x01010101u;
        uint32_t* p0 = births + (uint32_t(zb1) * 2u * P.KXY + rowbase[r]);
        uint32_t* p1 = p0 + P.KX;
        const bool hz = zb1 + 1 < nz;
        p0[0] = Bk[r][0];
        if (hx) p0[1] = Bk[r][1];
        if (hy[r]) p1[0] = Bk[r][2];
        if (hx && hy[r]) p1[1] = Bk[r][3];
        if (hz) {
          uint32_t* p2 = p0 + P.KXY;
          uint32_t* p3 = p1 + P.KXY;
          p2[0] = Bk[r][4];
          if (hx) p2[1] = Bk[r][5];
          if (hy[r]) p3[0] = Bk[r][6];
          if (hx && hy[r]) p3[1] = Bk[r][7];
        }
      }
      if (zb2 >= z0 && zb2 < z1) {
        up0 += (T[r][0] >> 7) & 0x01010101u;
        up1 += (T[r][1] >> 7) & 0x01010101u;
        uint8_t* p0 = tags + (uint32_t(zb2) * 2u * P.KXY + rowbase[r]);
        uint8_t* p1 = p0 + P.KX;
        const bool hz = zb2 + 1 < nz;
        p0[0] = uint8_t(T[r][0]);
        if (hx) p0[1] = uint8_t(T[r][0] >> 8);
        if (hy[r]) p1[0] = uint8_t(T[r][1]);
        if (hx && hy[r]) p1[1] = uint8_t(T[r][1] >> 8);
        if (hz) {
          uint8_t* p2 = p0 + P.KXY;
          uint8_t* p3 = p1 + P.KXY;
          p2[0] = uint8_t(T[r][0] >> 16);
          if (hx) p2[1] = uint8_t(T[r][0] >> 24);
          if (hy[r]) p3[0] = uint8_t(T[r][1] >> 16);
          if (hx && hy[r]) p3[1] = uint8_t(T[r][1] >> 24);
        }
        if (P.h0par) {  // (branch-free but for the rare basin staging)
          const uint32_t v = uint32_t(zb2) * P.plane + vrow[r];
          const uint32_t OMEGA = P.nx * P.ny * P.nz;
          const bool has_top = dtop[r] && (P.nz == 1 || hz);
          if (fast) {  // the warp's cells of B(z-2) are all absent (warp-uniform)
            P.h0par[v] = v;
            if (P.dpar) P.dpar[v] = has_top ? OMEGA : v;
          } else {
            // H0: an apparent vertex hangs under its partner edge's other vertex (absent cells
            // have tag 0: never UP); S.doff[dir] = the voxel offset of direction dir
            const uint32_t vt = T[r][0] & 0xFFu;
            const bool vup = (vt >> 6) == KIND_UP;
            P.h0par[v] = vup ? v + S.doff[vt & 7u] : v;
            if (!vup && !(CC[r][0] & 0x40u)) {  // a present basin (rare)
              const uint32_t i = atomicAdd(&S.bcnt, 1u);
              if (i < P.rcap) S.bbuf[i] = v;
              else P.basins[atomicAdd(P.nbasins, 1ull)] = v;
            }
            if (P.dpar) {  // the dual: a top cell hangs under the top cell across its apparent face
              // (3D: the cube, byte 3 of word 1; else the top cell's word and byte)
              const bool d3 = P.topw == 1 && P.topb == 3;
              const uint32_t tw = d3 ? T[r][1] >> 24 : ((P.topw ? T[r][1] : T[r][0]) >> (8 * P.topb));
              const uint32_t cw = d3 ? CC[r][1] >> 24 : ((P.topw ? CC[r][1] : CC[r][0]) >> (8 * P.topb));
              const uint32_t tt = tw & 0xFFu;
              const bool tabs = cw & 0x40u;
              const bool tdown = (tt >> 6) == KIND_DOWN;
              // directions whose top cell two steps away exists: x / y bits per row, z per plane
              const uint32_t okm = dok[r] | (zb2 > 0 ? 0x10u : 0u) |
                                   (uint32_t(zb2) + 2 < P.nz ? 0x20u : 0u);
              const uint32_t across = (okm >> (tt & 7u)) & 1u ? v + S.doff[tt & 7u] : OMEGA;
              // absent top cells hang under OMEGA (a cavity call rebuilds the forest)
              P.dpar[v] = !has_top ? v : (tabs ? OMEGA : (tdown ? across : v));
            }
          }
        }
      }
    }
    // residual present edges of B(z-2): a byte of q is 0 iff its cell is present (code bit 6
    // clear) and residual (tag kind 0); cells past the grid are absent in the codes
    // (rare: ~1 % of the edges; staged per CTA in shared memory, flushed at the end, the
    // overflow past KF_RCAP appended to the global list directly)
    if (!fast && P.res1 && z - 2 >= z0 && z - 2 < z1) {
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        if (!out[r]) continue;
        const uint32_t q0 = (T[r][0] & 0xC0C0C0C0u) | (CC[r][0] & 0x40404040u);
        const uint32_t q1 = (T[r][1] & 0xC0C0C0C0u) | (CC[r][1] & 0x40404040u);
        // bit 7 of a byte: the byte is 0 (its bytes are 0x00 / 0x40 / 0x80 / 0xC0); word 0:
        // x-edge (1,0,0) byte 1, z-edge (0,0,1) byte 2, xz-square (1,0,1) byte 3; word 1: y-edge
        // (0,1,0) byte 0, xy-square (1,1,0) byte 1, yz-square (0,1,1) byte 2
        const uint32_t z0 = ~(q0 | (q0 << 1)) & (P.res2 ? 0x80808000u : 0x00808000u);
        const uint32_t z1 = ~(q1 | (q1 << 1)) & (P.res2 ? 0x00808080u : 0x00000080u);
        if (!(z0 | z1)) continue;  // the common case
        const uint32_t kv = uint32_t(z - 2) * 2u * P.KXY + rowbase[r];
        auto put = [&](uint32_t k) {
          const uint32_t i = atomicAdd(&S.rcnt, 1u);
          if (i < P.rcap) S.rbuf[i] = k;
          else P.res1[atomicAdd(P.nres1, 1u)] = k;
        };
        auto put2 = [&](uint32_t k) {
          const uint32_t i = atomicAdd(&S.rcnt2, 1u);
          if (i < P.rcap) S.rbuf2[i] = k;
          else P.res2[atomicAdd(P.nres2, 1u)] = k;
        };
        if (z0 & 0x00008000u) put(kv + 1);                // x-edge
        if (z0 & 0x00800000u) put(kv + P.KXY);            // z-edge
        if (z1 & 0x00000080u) put(kv + P.KX);             // y-edge
        if (z0 & 0x80000000u) put2(kv + P.KXY + 1);       // xz-square
        if (z1 & 0x00008000u) put2(kv + P.KX + 1);        // xy-square
        if (z1 & 0x00800000u) put2(kv + P.KX + P.KXY);    // yz-square
      }
    }
#pragma unroll
    for (int r = 0; r < 2; ++r) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        Zm[r][q] = Bk[r][q + 4];
        P0[r][q] = Pn[r][q];
      }
      CZm[r][0] = CC[r][0];
      CZm[r][1] = CC[r][1];
      CC[r][0] = NC[r][0];
      CC[r][1] = NC[r][1];
    }
    g2 = g1;
    g1 = g0;
    rs = rn;
  }
  if constexpr (!TMA) kf_wait<0>();
  auto B8 = [](uint32_t v, int p) { return (v >> (8 * p)) & 0xFFu; };
  const uint32_t vv[7] = {B8(up0, 0),
                          B8(up0, 1) + B8(up0, 2) + B8(up1, 0),
                          B8(up0, 3) + B8(up1, 1) + B8(up1, 2),
                          B8(fin0, 0),
                          B8(fin0, 1) + B8(fin0, 2) + B8(fin1, 0),
                          B8(fin0, 3) + B8(fin1, 1) + B8(fin1, 2),
                          B8(fin1, 3)};
#pragma unroll
  for (int q = 0; q < 7; ++q) {
    const uint32_t sm = __reduce_add_sync(0xFFFFFFFFu, vv[q]);
    if (lane == 0 && sm) atomicAdd(S.cnt + q, sm);
  }
  const bool anynan = __any_sync(0xFFFFFFFFu, nan);
  if (lane == 0 && anynan) atomicOr(nan_flag, 1);
  __syncthreads();
  if (P.res1) {  // the CTA's staged residual cells and basins: one global atomic per list
    const uint32_t nr = min(S.rcnt, P.rcap), nr2 = P.res2 ? min(S.rcnt2, P.rcap) : 0u;
    const uint32_t nb = P.h0par ? min(S.bcnt, P.rcap) : 0u;
    if (nr | nr2 | nb) {
      if (threadIdx.x == 0 && nr) S.rbase = atomicAdd(P.nres1, nr);
      if (threadIdx.x == 32 && nr2) S.rbase2 = atomicAdd(P.nres2, nr2);
      if (threadIdx.x == 64 && nb) S.bbase = uint32_t(atomicAdd(P.nbasins, (unsigned long long)nb));
      __syncthreads();
      const uint32_t rb = S.rbase, rb2 = S.rbase2, bb = S.bbase;
      for (uint32_t i = threadIdx.x; i < nr; i += K2_THREADS) P.res1[rb + i] = S.rbuf[i];
      for (uint32_t i = threadIdx.x; i < nr2; i += K2_THREADS) P.res2[rb2 + i] = S.rbuf2[i];
      for (uint32_t i = threadIdx.x; i < nb; i += K2_THREADS) P.basins[bb + i] = S.bbuf[i];
    }
  }
  if (threadIdx.x < 7 && S.cnt[threadIdx.x])
    atomicAdd(cnt + (threadIdx.x < 3 ? threadIdx.x : threadIdx.x + 1),
              (unsigned long long)S.cnt[threadIdx.x]);
}
// ---------------------------------------------------------------------------------------------
// K4: H0 by union-find with the elder rule.
//  (1) every apparent vertex v (UP, paired with its earliest edge e_v) hangs under the other
//      endpoint of e_v, which is older; roots are the non-apparent vertices ("basins").
//  (2) the forest is not flattened: the endpoints of residual edges find their roots on demand
//      (path halving), ~1 % of the edges.
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

// parent of every voxel in the apparent-pair forest, and the number of basins (present vertices
// that are not the lower cell of an apparent pair) into *nbasins
// Essential H0 classes: the listed basins that are still roots after the merge rounds.
__global__ void k_h0_roots(const uint32_t* __restrict__ basins,
                           const unsigned long long* __restrict__ nbasins,
                           const uint32_t* __restrict__ births, Geom g,
                           const uint32_t* __restrict__ parent, uint64_t* rec,
                           unsigned long long* nrec, unsigned long long* nroots) {
  const unsigned long long n = *nbasins;
  const unsigned long long stride = uint64_t(gridDim.x) * blockDim.x;
  const int lane = threadIdx.x & 31;
  for (unsigned long long i0 = uint64_t(blockIdx.x) * blockDim.x; i0 < n; i0 += stride) {
    const unsigned long long i = i0 + threadIdx.x;
    bool emit = false;
    uint32_t k = 0;
    if (i < n) {
      const uint32_t v = basins[i];
      emit = parent[v] == v;
      const uint32_t nx = uint32_t(g.nx), ny = uint32_t(g.ny);
      const uint32_t r = v / nx, x = v - r * nx, z = r / ny, y = r - z * ny;
      k = (2 * z * uint32_t(g.KY) + 2 * y) * uint32_t(g.KX) + 2 * x;
    }
    const unsigned mask = __ballot_sync(0xFFFFFFFFu, emit);
    if (!mask) continue;
    unsigned long long base = 0;
    if (lane == __ffs(mask) - 1) {
      base = atomicAdd(nrec, (unsigned long long)__popc(mask));
      atomicAdd(nroots, (unsigned long long)__popc(mask));
    }
    base = __shfl_sync(0xFFFFFFFFu, base, __ffs(mask) - 1);
    if (emit) rec[base + __popc(mask & ((1u << lane) - 1))] = (uint64_t(k) << 32) | NONE32;
  }
}


// Root of x in a forest whose links only ever point to ancestors, with path halving (plain
// stores: a racing writer also stores an ancestor).  Used instead of flattening the whole forest:
// only the endpoints of the few residual edges need roots (C5b: ~2 M of 172 M edges).
__device__ __forceinline__ uint32_t find_halve(uint32_t* parent, uint32_t x) {
  uint32_t p = *(volatile uint32_t*)(parent + x);
  while (p != x) {
    const uint32_t pp = *(volatile uint32_t*)(parent + p);
    if (pp == p) return p;
    *(volatile uint32_t*)(parent + x) = pp;
    x = pp;
    p = *(volatile uint32_t*)(parent + x);
  }
  return x;
}

using Cand = H0Cand;  // key: the edge's (dual: complemented face's) key; a, b: endpoints / roots



// H0 candidates from the filtration's list of residual present edges: key and endpoints (the
// lower voxel and its neighbour along the edge's odd axis); k_mm_rounds finds the roots.
__global__ void k_h0_cands(const uint32_t* __restrict__ list, const unsigned* __restrict__ n,
                           const uint32_t* __restrict__ births, Geom g, Cand* __restrict__ cand) {
  const unsigned N = *n;
  const uint32_t KX = uint32_t(g.KX), KXY = uint32_t(g.KX * g.KY);
  const uint32_t nx = uint32_t(g.nx), nxy = uint32_t(g.nx * g.ny);
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
    const uint32_t k = list[i];
    const uint32_t Z = k / KXY, rm = k - Z * KXY, Y = rm / KX, X = rm - Y * KX;
    const uint32_t v = (Z >> 1) * nxy + (Y >> 1) * nx + (X >> 1);
    const uint32_t vs = (X & 1) ? 1u : ((Y & 1) ? nx : nxy);
    CR_DASSERT(uint64_t(k) < uint64_t(g.ncells) && ((X & 1) + (Y & 1) + (Z & 1)) == 1);
    CR_DASSERT(uint64_t(v) + vs < uint64_t(g.nvox));
    cand[i] = Cand{make_key(births[k], k), v, v + vs};
  }
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
// absent_to_omega: no +inf cavity is enclosed (Euler count, see top_dual), so every absent top
// cell lies in the outside vertex's component and hangs under it directly.
__global__ void k_dual_parent(const uint32_t* __restrict__ births, const uint8_t* __restrict__ tags,
                              DualG G, uint32_t* __restrict__ parent, int absent_to_omega,
                              unsigned long long* __restrict__ nroots) {
  uint32_t v, x, y, z;
  if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && threadIdx.x == 0)
    parent[G.omega] = G.omega;
  const bool in = vox_of_thread(G.g, v, x, y, z);
  if (nroots) {  // top cells that are roots (final when absent ones hang under OMEGA)
    bool root = false;
    if (in) {
      const uint32_t c[3] = {x, y, z};
      const uint32_t n[3] = {uint32_t(G.g.nx), uint32_t(G.g.ny), uint32_t(G.g.nz)};
      bool has_top = true;
      uint32_t K[3];
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        has_top = has_top && (n[a] == 1 || c[a] + 1 < n[a]);
        K[a] = n[a] > 1 ? 2 * c[a] + 1 : 0;
      }
      if (has_top) {
        const uint32_t k = (K[2] * uint32_t(G.g.KY) + K[1]) * uint32_t(G.g.KX) + K[0];
        root = births[k] != ABSENT_ORD && tag_kind(tags[k]) != KIND_DOWN;
      }
    }
    const unsigned mask = __ballot_sync(0xFFFFFFFFu, root);
    if ((threadIdx.x & 31) == 0 && mask) atomicAdd(nroots, (unsigned long long)__popc(mask));
  }
  if (!in) return;
  // the top cell with base voxel v (odd on every active axis), from v's coordinates (no second
  // decode of v or of the cell's kidx)
  const uint32_t c[3] = {x, y, z};
  const uint32_t n[3] = {uint32_t(G.g.nx), uint32_t(G.g.ny), uint32_t(G.g.nz)};
  const uint32_t vs[3] = {1u, n[0], n[0] * n[1]};
  bool has_top = true;
  uint32_t K[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (n[a] > 1) {
      has_top = has_top && c[a] + 1 < n[a];
      K[a] = 2 * c[a] + 1;
    } else {
      K[a] = 0;
    }
  }
  uint32_t p = v;
  if (has_top) {
    const uint32_t k = (K[2] * uint32_t(G.g.KY) + K[1]) * uint32_t(G.g.KX) + K[0];
    if (births[k] == ABSENT_ORD) {
      if (absent_to_omega) p = G.omega;
    } else {
      const uint8_t t = tags[k];
      if (tag_kind(t) == KIND_DOWN) {
        // dual apparent pair (face f = k + dir, top cell k): k hangs under f's other coface, the
        // top cell two steps along the axis -- base voxel v -/+ e_a, or OMEGA past the border
        const int dir = tag_dir(t), a = dir >> 1;
        if (dir & 1) p = c[a] + 2 < n[a] ? v + vs[a] : G.omega;
        else p = c[a] > 0 ? v - vs[a] : G.omega;
      }
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
// Dual candidate edges: residual (D-1)-cells whose two cofaces (top cells, OMEGA past the border)
// have different roots.  One thread per voxel v enumerates the (D-1)-cells with base voxel v (one
// per active normal axis a: even on a, odd on the other active axes), whose cofaces are the top
// cells with base voxels v - e_a and v.  The same threads count the dual roots into *nroots.
// Top cells that are roots after the absent cells' union-find (the cavity case).
__global__ void k_dual_roots(DualG G, const uint32_t* __restrict__ parent,
                             unsigned long long* __restrict__ nroots) {
  uint32_t v, x, y, z;
  const bool in = vox_of_thread(G.g, v, x, y, z);
  const uint32_t c[3] = {x, y, z};
  const uint32_t n[3] = {uint32_t(G.g.nx), uint32_t(G.g.ny), uint32_t(G.g.nz)};
  bool has_top = in;
#pragma unroll
  for (int a = 0; a < 3; ++a) has_top = has_top && (n[a] == 1 || c[a] + 1 < n[a]);
  const bool root = has_top && parent[v] == v;
  const unsigned mask = __ballot_sync(0xFFFFFFFFu, root);
  if ((threadIdx.x & 31) == 0 && mask) atomicAdd(nroots, (unsigned long long)__popc(mask));
}

// Dual candidates from the filtration's list of residual present (D-1)-cells: faces not cleared
// by the dimension below, whose two sides (the top cells across the face's normal axis, or OMEGA
// past the border) have different roots (path halving).  OMEGA is always a root: the absent
// cells' union-find links smaller indices under larger ones.
__global__ void k_dual_cands(const uint32_t* __restrict__ list, const unsigned* __restrict__ n_dev,
                             const uint32_t* __restrict__ births, const uint8_t* __restrict__ tags,
                             DualG G, uint32_t* parent, Cand* __restrict__ cand,
                             unsigned* __restrict__ ncand, unsigned long long* nroots) {
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(nroots, 1ull);  // OMEGA
  const unsigned N = *n_dev;
  const Geom& g = G.g;
  const uint32_t KX = uint32_t(g.KX), KXY = uint32_t(g.KX * g.KY);
  const uint32_t n[3] = {uint32_t(g.nx), uint32_t(g.ny), uint32_t(g.nz)};
  const uint32_t vs[3] = {1u, n[0], n[0] * n[1]};
  const unsigned stride = gridDim.x * blockDim.x;
  for (unsigned i0 = blockIdx.x * blockDim.x; i0 < N; i0 += stride) {  // warp-uniform trips
    const unsigned i = i0 + threadIdx.x;
    bool emit[1] = {false};
    Cand cd[1];
    if (i < N) {
      const uint32_t k = list[i];
      CR_DASSERT(uint64_t(k) < uint64_t(g.ncells));
      if (tag_kind(tags[k]) == KIND_RESIDUAL) {  // not cleared by the dimension below
        const uint32_t Z = k / KXY, rm = k - Z * KXY, Y = rm / KX, X = rm - Y * KX;
        const uint32_t C[3] = {X, Y, Z};
        int a = 0;  // the normal axis: the active axis along which the face is even
#pragma unroll
        for (int b = 2; b >= 0; --b)
          if (n[b] > 1 && !(C[b] & 1)) a = b;
        const uint32_t v = (Z >> 1) * vs[2] + (Y >> 1) * vs[1] + (X >> 1);
        const uint32_t ca = C[a] >> 1;
        CR_DASSERT(v < G.omega && ca < n[a] && births[k] != ABSENT_ORD);
        const uint32_t ra = ca > 0 ? find_halve(parent, v - vs[a]) : G.omega;
        const uint32_t rb = ca + 1 < n[a] ? find_halve(parent, v) : G.omega;
        if (ra != rb) {
          emit[0] = true;
          cd[0].key = ~make_key(births[k], k);  // ascending ~key = decreasing key
          cd[0].a = ra;
          cd[0].b = rb;
        }
      }
    }
    warp_append(emit, cd, cand, ncand);
  }
}


// key of a dual root (larger = elder): OMEGA the largest, absent top cells next
__device__ __forceinline__ uint64_t dual_root_key(const uint32_t* __restrict__ births, const DualG& G,
                                                  uint32_t v) {
  if (v == G.omega) return ~0ull;
  uint32_t k = 0;
  top_of_voxel(G.g, v, k);
  return make_key(births[k], k);
}


// dual record of the edge with complemented key ek whose younger root has key ry
__device__ __forceinline__ uint64_t dual_record(uint64_t ek, uint64_t ry) {
  const uint32_t sigma = ~key_kidx(ek);
  const bool absent = key_ord(ry) == ABSENT_ORD;  // (OMEGA is never the younger root)
  return (uint64_t(sigma) << 32) | (absent ? NONE32 : key_kidx(ry));
}

struct MMArgs {
  Cand* cur;
  const unsigned* n;  // device: the number of candidates (read by the kernel: no host round trip)
  uint32_t* parent;
  unsigned long long* best;  // 2 * nbest entries (two buffers, by round parity)
  unsigned nbest;
  uint8_t* alive;            // n entries (set to 1 by the kernel)
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
  // Initialise the two minima buffers at the roots the candidates touch, and the alive flags,
  // instead of memsetting 2 x nbest words (2.2 GB on C5b): every root a later find returns is
  // an endpoint root of some candidate (links only join two candidates' endpoint roots).
  // The candidates arrive with their endpoints (H0: voxels; the dual's k_dual_cands already
  // passes roots): their roots in the apparent forest are found here (path halving), the
  // same-root ones dropped (H0: the edge closes a cycle of older edges).
  for (unsigned i = gt; i < n; i += gs) {
    const Cand c = cur[i];
    const uint32_t a = find_halve(A.parent, c.a), b = find_halve(A.parent, c.b);
    if (a == b) {
      A.alive[i] = 0;
      continue;
    }
    cur[i].a = a;
    cur[i].b = b;
    A.best[a] = NONE64;
    A.best[b] = NONE64;
    A.best[A.nbest + a] = NONE64;
    A.best[A.nbest + b] = NONE64;
    A.alive[i] = 1;
  }
  grid.sync();
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
        // path halving (only ancestor pointers are written in the find phase; links are made
        // in the commit phase, after the grid barrier): C5b H0 1.26 -> 1.09 ms over plain finds
        const uint32_t a = find_halve(A.parent, c.a), b = find_halve(A.parent, c.b);
        if (a == b) {  // connected through strictly smaller edges: positive
          st = 0;
        } else {
          cur[i].a = a;
          cur[i].b = b;
          // test before the atomic: a root's minimum only decreases within the round, so a key
          // not below the value read cannot be it (the true minimum always reads a larger value:
          // keys are unique); the atomics on a large component's root no longer serialise
          if (c.key < __ldcg(bc + a)) atomicMin(bc + a, (unsigned long long)c.key);
          if (c.key < __ldcg(bc + b)) atomicMin(bc + b, (unsigned long long)c.key);
          st = 3;
        }
      }
      A.alive[i] = st;
    }
    grid.sync();
    unsigned left = 0;
    // commit: an edge that is the minimum at both of its components is the next Kruskal merge
    // there; one that is the minimum at the younger component alone also commits -- that
    // component does not change before the edge, so its root dies at this edge whatever the
    // other side does first (the elder rule).  Dual graph: the
    // same with the elder rule reversed (the root with the larger key survives).
    for (unsigned i = gt; i < n; i += gs) {
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

// Launches the merge rounds on the *n_dev candidates (cand, holding n_max); ctl (4 device unsigned, zeroed by the caller) receives the number of rounds in ctl[2].
// No host synchronisation: the caller reads ctl[2] with its next scalar read.
template <bool DUAL>
void mm_rounds(Cand* cand, const unsigned* n_dev, int64_t n_max, uint32_t* parent,
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
  MMArgs A{cand, n_dev, parent, best, nbest, alive, births, g, G, tags, rec, nrec, ctl};
  void* args[] = {&A};
  CR_CUDA(cudaLaunchCooperativeKernel((void*)k_mm_rounds<DUAL>, dim3(unsigned(blocks)), dim3(256),
                                      args, 0, s));
  ++g_launch_count;
}

// The top dimension d = D-1 by Alexander duality: a union-find with the
// reversed elder rule on the dual graph (top cells + the outside vertex, (D-1)-cells as edges),
// run as device-wide merge rounds.  Always succeeds (returns true).
bool top_dual(GeneralState& S, int d, Workspace& ws, HostScalars& hs, cr_stats& st) {
  cudaStream_t s = ws.stream();
  const Geom& g = S.g;
  const int B = 256;
  DualG G{g, uint32_t(g.nvox)};
  const int64_t nv = g.nvox + 1;
  S.R.rec[d] = ws.alloc<uint64_t>(st.cells[d] + 1);
  S.R.n[d] = 0;
  unsigned long long* cnt = ws.alloc<unsigned long long>(8);
  CR_CUDA(cudaMemsetAsync(cnt, 0, 8 * sizeof(unsigned long long), s));
  // the dual forest: the filtration's (absent top cells under OMEGA), rebuilt below when an
  // enclosed cavity is possible
  uint32_t* parent = S.dual_parent ? S.dual_parent : ws.alloc<uint32_t>(nv);
  // Enclosed +inf cavities (absent components that do not reach the outside) give the essential
  // classes of the top dimension d = D-1, and by the Euler-Poincare relation their number is
  //   ess[d] = (-1)^d (chi - sum_{e<d} (-1)^e ess[e]),  chi = sum_e (-1)^e #(finite e-cells),
  // known here when the dimensions below were computed in this call.  With none, every absent
  // top cell belongs to the outside vertex's component: no union-find over the absent cells.
  bool no_cavity = false;
  if (S.lower_essential_known) {
    int64_t chi = 0, low = 0;
    for (int e = 0; e <= g.D; ++e) chi += (e & 1) ? -st.cells[e] : st.cells[e];
    for (int e = 0; e < d; ++e) low += (e & 1) ? -st.essential[e] : st.essential[e];
    const int64_t ess_top = (d & 1) ? low - chi : chi - low;
    no_cavity = ess_top == 0;
  }
  if (!S.res_faces) throw Error{CR_EINTERNAL, "top_dual: the residual faces were not listed"};
  // with the filtration's forest the roots among the top cells are counted from its counters:
  // the present top cells that are not the upper cell of an apparent pair (face, top)
  const bool forest_given = S.dual_parent != nullptr && no_cavity && d == g.D - 1;
  if (!forest_given) {
    k_dual_parent<<<vox_grid(g), VOX_THREADS, 0, s>>>(S.births, S.tags, G, parent,
                                                      no_cavity ? 1 : 0,
                                                      no_cavity ? cnt + 1 : nullptr);
    CR_CHECK_LAUNCH();
  }
  if (!no_cavity) {
    k_dual_absent_vox<<<grid_for(g.nvox, B), B, 0, s>>>(S.births, G, parent);
    CR_CHECK_LAUNCH();
    k_dual_roots<<<vox_grid(g), VOX_THREADS, 0, s>>>(G, parent, cnt + 1);
    CR_CHECK_LAUNCH();
  }
  // the residual faces listed by the filtration (no per-voxel face scan); the roots of their
  // sides found on demand (no flattening)
  Cand* cand = ws.alloc<Cand>(st.cells[d] + 1);
  unsigned* ncand = reinterpret_cast<unsigned*>(cnt);
  k_dual_cands<<<148 * 8, 256, 0, s>>>(S.res_faces, S.nres_faces, S.births, S.tags, G, parent,
                                       cand, ncand, cnt + 1);
  CR_CHECK_LAUNCH();
  // candidates <= the finite d-cells (known since H0's read): no host read before the rounds
  const int64_t n = st.cells[d] + 1;
  unsigned long long* nrec = cnt + 2;
  unsigned long long* best = ws.alloc<unsigned long long>(2 * nv);  // set in k_mm_rounds
  uint8_t* alive = ws.alloc<uint8_t>(n + 1);
  unsigned* ctl = reinterpret_cast<unsigned*>(cnt + 6);  // cnt[6], cnt[7]: zeroed above
  mm_rounds<true>(cand, ncand, n, parent, best, unsigned(nv), alive, S.births, g, G, nullptr,
                  S.R.rec[d], nrec, ctl, ws);
  CR_CUDA(cudaMemcpyAsync(hs.p, cnt, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  CR_CUDA(cudaStreamSynchronize(s));
  st.columns[d] = int64_t(hs.p[1]);  // dual roots
  if (forest_given) st.columns[d] += st.cells[d + 1] - st.apparent[d];
  S.R.n[d] = int64_t(hs.p[2]);
  st.rounds[d] = int64_t(reinterpret_cast<const unsigned*>(hs.p + 6)[2]);
  ws.release(best);
  ws.release(alive);
  ws.release(cand);
  ws.release(parent);
  if (parent == S.dual_parent) S.dual_parent = nullptr;
  return true;
}

bool use_dual(const Geom& g, int d) {
  if (d != g.D - 1 || d < 1) return false;
  return opt(OPT_TOP_REDUCE) == 0;  // the coboundary reduction instead (cross-checks)
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

// emit_bars for a dimension with n <= BAR1_MAX records, in ONE block: keep-flags, block-wide
// exclusive scan, scatter and the output-offset advance (instead of five launches)
constexpr int BAR1_THREADS = 1024, BAR1_IPT = 8, BAR1_MAX = BAR1_THREADS * BAR1_IPT;
__global__ void __launch_bounds__(BAR1_THREADS) k_bar_one_block(
    const uint64_t* __restrict__ rec, int n, const uint32_t* __restrict__ births, int dim,
    long long* dbase, int64_t cap, cr_pair* out, uint32_t* out_cells) {
  typedef cub::BlockScan<unsigned, BAR1_THREADS> BS;
  __shared__ typename BS::TempStorage tmp;
  const int t = threadIdx.x;
  uint64_t r[BAR1_IPT];
  unsigned keep = 0, cnt = 0;
#pragma unroll
  for (int q = 0; q < BAR1_IPT; ++q) {  // blocked: thread t holds records [t IPT, (t + 1) IPT)
    const int i = t * BAR1_IPT + q;
    r[q] = i < n ? rec[i] : 0ull;
    if (i < n) {
      const uint32_t b = uint32_t(r[q] >> 32), d = uint32_t(r[q]);
      if (d == NONE32 || births[d] > births[b]) {
        keep |= 1u << q;
        ++cnt;
      }
    }
  }
  unsigned pos, total;
  BS(tmp).ExclusiveSum(cnt, pos, total);
  const long long base = dbase[dim];
#pragma unroll
  for (int q = 0; q < BAR1_IPT; ++q)
    if (keep >> q & 1u) {
      const int64_t o = base + pos++;
      if (o < cap) {
        const uint32_t b = uint32_t(r[q] >> 32), d = uint32_t(r[q]);
        cr_pair p;
        p.dim = dim;
        p.birth = float_of_ord(births[b]);
        p.death = d == NONE32 ? __int_as_float(0x7F800000) : float_of_ord(births[d]);
        out[o] = p;
        if (out_cells) out_cells[o] = b;
      }
    }
  if (t == 0) dbase[dim + 1] = base + total;
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
// pivots clear dimension 2, then the top dimension by duality.  (Round 1 also measured dimension 1
// by the homology reduction of the square columns after the top dimension: half the entry work on
// C4 but more additions and an equally long critical chain -- 174 vs 168 ms, C5 1.76 vs 1.63 s --
// and removed it.)
void reduce_dims(GeneralState& S, const Geom& g, int dmax, Workspace& ws, HostScalars& hs,
                 cr_stats& st) {
  static const char* names[4] = {"", "reduce_d1", "reduce_d2", "reduce_d3"};
  cudaStream_t s = ws.stream();
  S.lower_essential_known = true;  // H0 and each reduced dimension count their essential classes
  for (int d = 1; d <= dmax; ++d) {
    if (!(use_dual(g, d) && top_dual(S, d, ws, hs, st)))
      reduce_dimension(S, d, ws, hs, st);
    prof_mark(s, names[d]);
  }
}

void run_general(const float* image, const Geom& g, int dmax, Workspace& ws, HostScalars& hs,
                 GeneralState& S, cr_stats& st) {
  cudaStream_t s = ws.stream();
  S.g = g;
  S.births = ws.alloc<uint32_t>(g.ncells);
  S.tags = ws.alloc<uint8_t>(g.ncells);
  unsigned long long* cnt = ws.alloc<unsigned long long>(32);
  CR_CUDA(cudaMemsetAsync(cnt, 0, 32 * sizeof(unsigned long long), s));
  int* nan_flag = reinterpret_cast<int*>(cnt + 31);
  uint32_t* parent = ws.alloc<uint32_t>(g.nvox);  // H0 basin forest
  uint32_t* basins = ws.alloc<uint32_t>(g.nvox);  // the forest's roots (non-apparent vertices)
  // H0 candidate edges, room for every edge of the grid (a bound known without reading the
  // finite-cell counts back: no host sync before the merge rounds, and pieces of a host batch
  // enumerate their candidates as they arrive)
  int64_t nedges_max = 0;
  {
    const int64_t n3[3] = {g.nx, g.ny, g.nz};
    for (int a = 0; a < 3; ++a)
      if (n3[a] > 1) nedges_max += (n3[a] - 1) * (g.nvox / n3[a]);
  }
  Cand* cand = S.nready ? ws.alloc<Cand>(nedges_max > 0 ? nedges_max : 1) : nullptr;
  unsigned* ncand = reinterpret_cast<unsigned*>(cnt + 12);
  // residual present edges, listed by the filtration (kidx; at most every edge of the grid), and
  // in 3D the residual present squares (the top-dimension dual's faces; in 2D those are edges)
  uint32_t* res1 = ws.alloc<uint32_t>(nedges_max > 0 ? nedges_max : 1);
  uint32_t* res2 = nullptr;
  if (g.D == 3) res2 = ws.alloc<uint32_t>(3 * g.nvox);
  // the top-dimension dual forest, written by the filtration (OMEGA = nvox)
  S.dual_parent = g.D >= 2 ? ws.alloc<uint32_t>(g.nvox + 1) : nullptr;
  S.res_faces = g.D == 3 ? res2 : (g.D == 2 ? res1 : nullptr);
  S.nres_faces = reinterpret_cast<const unsigned*>(g.D == 3 ? cnt + 14 : cnt + 12);

  // K1 + K2 in one streaming kernel (round 1 measured the split alternatives, profiles/r01/s3:
  // C5 0.52 + 3.60 ms as separate births + apparent-pair kernels)
  {
    const KfLaunch L = kf_launch(g, K2_ROWS);
    static thread_local int kf_attr_dev = -1;
    if (kf_attr_dev != ws.device()) {
      CR_CUDA(cudaFuncSetAttribute(k_filtration<false>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(sizeof(Kf2Smem<false>))));
      CR_CUDA(cudaFuncSetAttribute(k_filtration<true>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   int(sizeof(Kf2Smem<true>))));
      kf_attr_dev = ws.device();
    }
    KfP kp = kf2_params(g, L.zc);
    kp.zper = S.img_zper;
    kp.zimg = S.img_zimg;
    kp.res1 = res1;
    kp.nres1 = ncand;
    kp.res2 = res2;
    kp.nres2 = reinterpret_cast<unsigned*>(cnt + 14);
    kp.h0par = parent;
    kp.basins = basins;
    kp.nbasins = cnt + 8;
    kp.dpar = S.dual_parent;
    if (opt(OPT_KF_RCAP) > 0 && opt(OPT_KF_RCAP) < KF_RCAP) kp.rcap = uint32_t(opt(OPT_KF_RCAP));
    // the source planes the filtration reads (a batch read unstacked has no separator planes)
    const int64_t nzsrc = kp.zper ? (g.nz + 1) / kp.zper * kp.zimg : g.nz;
    CUtensorMap tmap;
    // TMA ring only on request: measured slower than the per-thread cp.async ring (C5b 2.94 vs
    // 2.74 ms: 2.24 G vs 2.06 G warp instructions -- the +inf selects for the zero-filled
    // out-of-image voxels and the mbarrier bookkeeping cost more than the 4-byte copies they
    // replace; profiles/r02/s17)
    const bool tma = opt(OPT_KF_TMA) != 0 && kf_tensor_map(&tmap, image, g.nx, g.ny, nzsrc);
    st.kf_tma = tma ? 1 : 0;
    auto launch_kf = [&](unsigned grid) {
      if (tma)
        k_filtration<true><<<grid, K2_THREADS, sizeof(Kf2Smem<true>), s>>>(
            image, kp, S.births, S.tags, cnt, nan_flag, tmap);
      else
        k_filtration<false><<<grid, K2_THREADS, sizeof(Kf2Smem<false>), s>>>(
            image, kp, S.births, S.tags, cnt, nan_flag, tmap);
    };
    const uint32_t nzc = uint32_t((g.nz + L.zc - 1) / L.zc), xy = kp.XB * kp.YB;
    if (S.nready == 0) {
      launch_kf(L.grid);
      CR_CHECK_LAUNCH();
    } else {
      // input arriving in pieces: z-chunk c reads planes up to (c + 1) zc + 4; launch the chunks
      // whose planes are in as each piece lands (the copies run on another stream)
      uint32_t c0 = 0;
      for (int i = 0; i < S.nready && c0 < nzc; ++i) {
        uint32_t c1 = c0;
        while (c1 < nzc && (i == S.nready - 1 ||
                            int64_t(c1 + 1) * L.zc + 4 < S.ready_z[i]))
          ++c1;
        if (c1 == c0) continue;
        CR_CUDA(cudaStreamWaitEvent(s, S.ready_ev[i], 0));
        kp.zb0 = c0;
        launch_kf((c1 - c0) * xy);
        CR_CHECK_LAUNCH();
        c0 = c1;
      }
    }
    prof_mark(s, "filtration");
  }

  if (S.top_only) {  // the top dimension alone (--top_dim): no H0, no clearing
    CR_CUDA(cudaMemcpyAsync(hs.p, cnt, 32 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    CR_CUDA(cudaStreamSynchronize(s));
    if (*reinterpret_cast<int*>(hs.p + 31)) throw Error{CR_EINVAL, "NaN in image"};
    for (int d = 0; d < 4; ++d) {
      st.apparent[d] = int64_t(hs.p[d]);
      st.cells[d] = int64_t(hs.p[4 + d]);
    }
    if (g.D < 2 || top_dual(S, g.D - 1, ws, hs, st)) {
      prof_mark(s, "top_dual");
      return;
    }
    // too many dual roots for the one-CTA union-find: the full pipeline (the top dimension's
    // zero columns are essential only given the clearing by the dimensions below)
    S.top_only = false;
  }

  // ---- H0
  // basin forest, not flattened: k_mm_rounds finds the roots of the residual edges' endpoints
  // (a pointer-jumping pass over every voxel took longer: C5b h0 4.23 -> 4.13 ms without it);
  // the residual edges come listed from the filtration (no per-voxel edge scan: 3.25 -> 1.91 ms).
  // Pieces of a batch arriving from the host were done in the filtration loop above.
  if (!cand) cand = ws.alloc<Cand>(nedges_max > 0 ? nedges_max : 1);
  // (the basin forest and its basins list were written by the filtration)
  // H0 candidates: every residual present edge (the filtration's list) with its endpoints
  k_h0_cands<<<148 * 8, 256, 0, s>>>(res1, ncand, S.births, g, cand);
  CR_CHECK_LAUNCH();
  if (S.res_faces != res1) ws.release(res1);  // (2D: the dual's faces)
  const int64_t nedges = nedges_max;

  // vertex records: at most one per vertex
  S.R.rec[0] = ws.alloc<uint64_t>(g.nvox);
  unsigned long long* nrec0 = cnt + 13;
  unsigned long long* best = ws.alloc<unsigned long long>(2 * g.nvox);  // set in k_mm_rounds
  uint8_t* alive = ws.alloc<uint8_t>(nedges);
  unsigned* ctl = reinterpret_cast<unsigned*>(cnt + 20);  // cnt[20], cnt[21]: zeroed at the start
  mm_rounds<false>(cand, ncand, nedges, parent, best, unsigned(g.nvox), alive, S.births, g,
                   DualG{g, uint32_t(g.nvox)}, S.tags, S.R.rec[0], nrec0, ctl, ws);
  // essential classes: the final roots (parent[v] == v holds exactly for them; no flattening)
  k_h0_roots<<<148 * 8, 256, 0, s>>>(basins, cnt + 8, S.births, g, parent, S.R.rec[0], nrec0,
                                     cnt + 22);
  CR_CHECK_LAUNCH();
  // the one read of H0: NaN flag, cell / apparent / basin counts, records, roots, rounds
  CR_CUDA(cudaMemcpyAsync(hs.p, cnt, 32 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  CR_CUDA(cudaStreamSynchronize(s));
  if (*reinterpret_cast<int*>(hs.p + 31)) throw Error{CR_EINVAL, "NaN in image"};
  for (int d = 0; d < 4; ++d) {
    st.apparent[d] = int64_t(hs.p[d]);
    st.cells[d] = int64_t(hs.p[4 + d]);
  }
  st.columns[0] = int64_t(hs.p[8]);
  S.R.n[0] = int64_t(hs.p[13]);
  st.essential[0] = int64_t(hs.p[22]);
  st.rounds[0] = int64_t(reinterpret_cast<const unsigned*>(hs.p + 20)[2]);
  prof_mark(s, "h0");
  // the candidates (all residual edges) stay for the dim-1 columns if K5 reduces dimension 1
  const bool keep_cand = dmax >= 1 && !use_dual(g, 1);
  if (keep_cand) {
    S.h0_cand = cand;
    S.h0_ncand = reinterpret_cast<const unsigned*>(hs.p + 12)[0];
  } else {
    ws.release(cand);
  }
  ws.release(best);
  ws.release(alive);
  ws.release(parent);
  ws.release(basins);

  reduce_dims(S, g, dmax, ws, hs, st);
  if (S.h0_cand) {  // (not consumed: an error path)
    ws.release(const_cast<Cand*>(S.h0_cand));
    S.h0_cand = nullptr;
  }
  if (S.res_faces) {
    ws.release(S.res_faces);
    S.res_faces = nullptr;
  }
  if (S.dual_parent) {
    ws.release(S.dual_parent);
    S.dual_parent = nullptr;
  }
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
    if (n <= BAR1_MAX) {  // small: one block does the flags, the scan and the scatter
      k_bar_one_block<<<1, BAR1_THREADS, 0, s>>>(S.R.rec[d], int(n), S.births, d, dbase, cap, out,
                                                 out_cells);
      CR_CHECK_LAUNCH();
      continue;
    }
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
