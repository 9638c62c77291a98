// Micro-benchmark of the K5 per-addition building blocks (one warp, clock64): not part of libcr.
// Build: see tools/micro/build.sh.  Checks merge_small against merge_symdiff, then times both.
#include "../../paper_2005_12692_b200/csrc/reduce.cu"

namespace cr {
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
}  // namespace cr

int main() {
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
