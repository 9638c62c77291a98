// Micro-benchmark of the K5 per-addition building blocks (one warp, clock64): not part of libcr.
// Build: see tools/micro/build.sh.  Checks merge_small against merge_symdiff, then times both.
#include <vector>
#include "../../paper_2005_12692_b200/csrc/reduce.cu"

namespace cr {
// C = A xor F for a long A (global) and a short F (shared, b <= FCAP), C in global memory, using
// X (FCAP u64 of shared scratch).  Warp-collective; returns |C|.
//  1. positions: P[t] = #{A < F[t]} by a sampled search (<= 256 samples of A in X, then a binary
//     search inside one sample interval; a lane's <= 8 searches run interleaved), dup[t] = (A[P[t]]
//     == F[t]); prefix counts of inserted (non-dup) and cancelled (dup) F entries over t;
//  2. the non-dup F entries go to P[t] + ins_before(t) - dup_before(t);
//  3. A streams through in windows of 256 (8 independent loads per lane): A[i] moves to
//     i + #{non-dup t : P[t] <= i} - #{dup t : P[t] < i}, unless a dup lands on it.  A window that
//     holds no position only shifts (one smem search per window).
__device__ uint32_t merge_long_short_ref(const uint64_t* __restrict__ A, uint32_t a, const uint64_t* F,
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


__global__ void k_micro(unsigned long long* out, int na, int nb, int iters, int which) {
  __shared__ uint64_t A[2][FCAP];
  __shared__ uint64_t B[64];
  const int lane = threadIdx.x & 31;
  for (int i = lane; i < FCAP; i += 32) A[0][i] = uint64_t(i) * 1000 + 7;
  for (int i = lane; i < 64; i += 32) B[i] = uint64_t(i) * 37000 + 500;  // distinct from A
  __syncwarp();
  int cur = 0;
  unsigned n = na;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    unsigned m;
    if (which == 0) m = merge_small(A[cur], n, B, nb, A[cur ^ 1], lane);
    else m = merge_symdiff<false, false>(A[cur], n, B, nb, A[cur ^ 1], lane);
    cur ^= 1;
    n = m;
    if (n + nb > FCAP) n = na;
  }
  const long long t1 = clock64();
  if (lane == 0) {
    out[0] = (unsigned long long)(t1 - t0) / iters;
    out[1] = n;
  }
}

__global__ void k_check(int* bad, unsigned seed) {
  __shared__ uint64_t A[FCAP], B[8], C1[FCAP + 8], C2[FCAP + 8];
  const int lane = threadIdx.x & 31;
  for (int t = 0; t < 200; ++t) {
    const unsigned h = seed * 2654435761u + t * 40503u;
    const unsigned na = (h >> 8) % 250, nb = 1 + (h >> 4) % 8;
    for (unsigned i = lane; i < na; i += 32) A[i] = 3ull * i + (h & 1);
    if (lane == 0) {
      unsigned v = (h >> 12) % 5;
      for (unsigned k = 0; k < nb; ++k) {
        v += 1 + ((h >> (k * 3)) & 3);
        B[k] = v;
      }
    }
    __syncwarp();
    const unsigned m1 = merge_small(A, na, B, nb, C1, lane);
    const unsigned m2 = merge_symdiff<false, false>(A, na, B, nb, C2, lane);
    bool ok = m1 == m2;
    for (unsigned i = lane; ok && i < m1; i += 32) ok = C1[i] == C2[i];
    if (!__all_sync(0xFFFFFFFFu, ok) && lane == 0) atomicAdd(bad, 1);
    __syncwarp();
  }
}
// merge_long_short: A (global, na) xor F (shared, nb) -> C (global)
__global__ void k_mls(const uint64_t* A, unsigned na, uint64_t* C, unsigned nb, int iters,
                      unsigned long long* out) {
  __shared__ uint64_t F[FCAP], X[FCAP];
  const int lane = threadIdx.x & 31;
  for (unsigned i = lane; i < nb; i += 32) F[i] = uint64_t(i) * (uint64_t(na) * 4 / nb) + 1;
  __syncwarp();
  unsigned m = 0;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) m = merge_long_short(A, na, F, nb, C, X, lane);
  const long long t1 = clock64();
  if (lane == 0) {
    out[0] = (unsigned long long)(t1 - t0) / iters;
    out[1] = m;
  }
}
__global__ void k_mls_check(const uint64_t* A, unsigned na, uint64_t* C1, uint64_t* C2,
                            int* bad, unsigned seed) {
  __shared__ uint64_t F[FCAP], X[FCAP];
  const int lane = threadIdx.x & 31;
  for (int t = 0; t < 40; ++t) {
    const unsigned h = seed * 2654435761u + t * 97u;
    const unsigned a = (h >> 4) % (na + 1), b = (h >> 16) % (FCAP + 1);
    // F: sorted distinct values in [0, 4a+8), some equal to A entries (A = multiples of 4)
    if (lane == 0) {
      uint64_t v = (h >> 7) % 3;
      for (unsigned i = 0; i < b; ++i) {
        F[i] = v;
        v += 1 + ((h >> (i % 13)) + i * 7) % 9;
      }
    }
    __syncwarp();
    const unsigned m1 = merge_long_short(A, a, F, b, C1, X, lane);
    const unsigned m2 = merge_long_short_ref(A, a, F, b, C2, X, lane);
    __syncwarp();
    bool ok = m1 == m2;
    for (unsigned i = lane; ok && i < m1; i += 32) ok = C1[i] == C2[i];
    if (!__all_sync(0xFFFFFFFFu, ok) && lane == 0) atomicAdd(bad, 1);
    __syncwarp();
  }
}
}  // namespace cr

int main() {
  {
    const unsigned na = 3000;
    std::vector<uint64_t> h(na);
    for (unsigned i = 0; i < na; ++i) h[i] = 4ull * i;
    uint64_t *A, *C1, *C2;
    cudaMalloc(&A, na * 8);
    cudaMalloc(&C1, (na + 512) * 8);
    cudaMalloc(&C2, (na + 512) * 8);
    cudaMemcpy(A, h.data(), na * 8, cudaMemcpyHostToDevice);
    int* bad;
    cudaMalloc(&bad, 4);
    cudaMemset(bad, 0, 4);
    for (unsigned s = 0; s < 100; ++s) cr::k_mls_check<<<1, 32>>>(A, na, C1, C2, bad, s);
    int hb = -1;
    cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
    printf("merge_long_short vs reference: %d mismatching cases of 4000\n", hb);
  }
  {
    const unsigned na = 10000;
    std::vector<uint64_t> h(na);
    for (unsigned i = 0; i < na; ++i) h[i] = 4ull * i;  // F values 1 mod 4: never equal
    uint64_t *A, *C;
    cudaMalloc(&A, na * 8);
    cudaMalloc(&C, (na + 512) * 8);
    cudaMemcpy(A, h.data(), na * 8, cudaMemcpyHostToDevice);
    unsigned long long* o;
    cudaMalloc(&o, 16);
    for (unsigned nb : {32u, 128u, 256u})
      for (unsigned a : {1000u, 10000u}) {
        cr::k_mls<<<1, 32>>>(A, a, C, nb, 20, o);
        unsigned long long hh[2];
        cudaMemcpy(hh, o, 16, cudaMemcpyDeviceToHost);
        printf("merge_long_short a=%u b=%u: %llu cycles (n=%llu)\n", a, nb, hh[0], hh[1]);
      }
  }
  int* bad;
  cudaMalloc(&bad, 4);
  cudaMemset(bad, 0, 4);
  for (unsigned s = 0; s < 50; ++s) cr::k_check<<<1, 32>>>(bad, s);
  int hb = -1;
  cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
  printf("merge_small vs merge_symdiff: %d mismatching cases of 10000\n", hb);
  unsigned long long* d;
  cudaMalloc(&d, 16);
  for (int which = 0; which < 2; ++which)
    for (int na : {32, 128, 250}) {
      cr::k_micro<<<1, 32>>>(d, na, 6, 2000, which);
      unsigned long long h[2];
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
      printf("%s na=%d nb=6: %llu cycles per merge (n=%llu)\n",
             which ? "merge_symdiff" : "merge_small", na, h[0], h[1]);
    }
  return 0;
}
