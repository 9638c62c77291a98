// Minimal TMA probe: load one (36 x 9 x 1) box of a float tensor into shared memory.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
__global__ void k(const __grid_constant__ CUtensorMap tmap0, const CUtensorMap* gmap, float* out, int x, int y, int z, int mode) {
  const CUtensorMap* tm = (mode & 4) ? gmap : &tmap0;
  extern __shared__ __align__(128) float sm[];
  __shared__ unsigned long long bar;
  const unsigned b = unsigned(__cvta_generic_to_shared(&bar));
  const unsigned d = unsigned(__cvta_generic_to_shared(sm));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(b));
    if (!(mode & 2)) asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (!(mode & 1))
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(b), "r"(36 * 9 * 4) : "memory");
    else {
      unsigned long long st;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 %0, [%1], %2;\n" : "=l"(st) : "r"(b), "r"(36 * 9 * 4) : "memory");
    }
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
                 " [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(d), "l"(tm), "r"(x), "r"(y), "r"(z), "r"(b) : "memory");
  }
  asm volatile("{\n .reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}\n" ::"r"(b), "r"(0) : "memory");
  for (int i = threadIdx.x; i < 36 * 9; i += blockDim.x) out[i] = sm[i];
}
#include <cstdlib>
int main(int argc, char** argv) {
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  printf("entry %p q=%d\n", (void*)enc, int(q));
  int shapes[][3] = {{64, 40, 5}, {4, 4, 1}, {128, 128, 128}};
  int mode = atoi(argv[1]);
  for (auto& s : shapes) {
    {
      size_t n = size_t(s[0]) * s[1] * s[2];
      float *img, *out;
      cudaMalloc(&img, n * 4); cudaMalloc(&out, 36 * 9 * 4);
      float* h = new float[n];
      for (size_t i = 0; i < n; ++i) h[i] = float(i);
      cudaMemcpy(img, h, n * 4, cudaMemcpyHostToDevice);
      CUtensorMap m;
      cuuint64_t dims[3] = {cuuint64_t(s[0]), cuuint64_t(s[1]), cuuint64_t(s[2])};
      cuuint64_t str[2] = {cuuint64_t(s[0]) * 4, cuuint64_t(s[0]) * s[1] * 4};
      cuuint32_t box[3] = {36, 9, 1}, es[3] = {1, 1, 1};
      CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, img, dims, str, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      CUtensorMap* gm;
      cudaMalloc(&gm, sizeof(CUtensorMap));
      cudaMemcpy(gm, &m, sizeof m, cudaMemcpyHostToDevice);
      k<<<1, 128, 36 * 9 * 4>>>(m, gm, out, atoi(argv[2]), atoi(argv[3]), 0, mode);
      cudaError_t e = cudaDeviceSynchronize();
      float ho[36 * 9];
      cudaMemcpy(ho, out, sizeof ho, cudaMemcpyDeviceToHost);
      printf("shape %d %d %d mode %d encode %d -> %s; out[0..3] %g %g %g %g row1 %g\n", s[0], s[1], s[2], mode, int(r),
             cudaGetErrorString(e), ho[0], ho[1], ho[2], ho[37], ho[36 + 1]);
      if (e != cudaSuccess) return 1;
    }
  }
}
