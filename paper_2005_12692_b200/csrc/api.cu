// api.cu -- the extern "C" boundary of libcr.so (include/cr.h).
#include <cub/cub.cuh>

#include <cstdlib>
#include <cstring>

#include "pipeline.cuh"

namespace cr {
const char* last_error_text();
void set_profiling(bool on);
bool set_opt(int key, int64_t v);
void release_workspace();
size_t workspace_bytes();
static thread_local cr_stats g_last_stats;
static thread_local uint64_t g_stats_gen = 0;  // prof_gen() when g_last_stats was committed
static void commit_stats(const cr_stats& st) {
  g_last_stats = st;
  g_stats_gen = prof_gen();
}

namespace {

bool valid_shape(const int64_t* shape, int ndim) {
  if (!shape || ndim < 1 || ndim > 3) return false;
  int64_t n = 1;
  for (int i = 0; i < ndim; ++i) {
    if (shape[i] < 1 || shape[i] > (int64_t(1) << 32)) return false;
    n *= 2 * shape[i] - 1;
    if (n >= (int64_t(1) << 32) - 2) return false;
  }
  return true;
}

bool force_general() { return opt(OPT_FORCE_GENERAL) != 0; }

// death cell of each bar: the partner of its birth cell ("or optionally, killed")
__global__ void k_death_cells(const uint32_t* __restrict__ birth_cells, int64_t n,
                              const uint32_t* __restrict__ partner, uint32_t* __restrict__ out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = partner[birth_cells[i]];
}

// lifetime-enhanced image: channel 0 = the image, channel 1 + d = per voxel the
// largest lifetime of the dim-d bars born at a cell whose base voxel (X/2, Y/2, Z/2) it is.
// Lifetimes are >= 0, so their float bits order like the values (integer atomicMax).
__global__ void k_lifetime_scatter(const cr_pair* __restrict__ bars, const uint32_t* __restrict__ cells,
                                   int64_t n, const int64_t* __restrict__ offsets, int64_t batch,
                                   Geom g, int nch, float inf_value, float* __restrict__ out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t b = 0;
  if (offsets) {  // image of bar i: last b with offsets[b] <= i
    int64_t lo = 0, hi = batch - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (offsets[mid] <= i) lo = mid; else hi = mid - 1;
    }
    b = lo;
  }
  const cr_pair p = bars[i];
  const float death = isinf(p.death) ? inf_value : p.death;
  float life = death - p.birth;
  if (!(life > 0.f)) life = 0.f;
  const uint32_t k = cells[i];
  const uint32_t KX = uint32_t(g.KX), KY = uint32_t(g.KY);
  const uint32_t X = k % KX, Y = (k / KX) % KY, Z = k / (KX * KY);
  const int64_t v = (int64_t(Z >> 1) * g.ny + (Y >> 1)) * g.nx + (X >> 1);
  float* ch = out + (b * nch + 1 + p.dim) * g.nvox;
  atomicMax(reinterpret_cast<int*>(ch + v), __float_as_int(life));
}

__global__ void k_lifetime_init(const float* __restrict__ img, int64_t nvox, int64_t batch, int nch,
                                float* __restrict__ out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= nvox * batch) return;
  const int64_t b = i / nvox, v = i - b * nvox;
  out[(b * nch) * nvox + v] = img[i];
  for (int c = 1; c < nch; ++c) out[(b * nch + c) * nvox + v] = 0.f;
}

cr_status fail(const Error& e) {
  set_error_text(e.msg);
  return e.st;
}

// Stack `batch` images along the slowest axis with one +inf separator layer between them, so the
// complexes are disjoint (cells touching a separator are absent, reading R5).


__global__ void k_stack(const float* __restrict__ src, int64_t per_img, int64_t layer,
                        int64_t layers_per_img, int64_t nlayers, float* __restrict__ dst) {
  // one stacked layer per blockIdx.y step (its image and slot computed once per block, not per
  // element), 16-byte copies when the layer allows them
  const bool v4 = (layer & 3) == 0 && ((reinterpret_cast<uintptr_t>(src) |
                                        reinterpret_cast<uintptr_t>(dst)) & 15) == 0;
  for (int64_t L = blockIdx.y; L < nlayers; L += gridDim.y) {
    const int64_t b = L / (layers_per_img + 1), l = L % (layers_per_img + 1);
    float* d = dst + L * layer;
    const float* sp = src + b * per_img + l * layer;
    const bool sep = l == layers_per_img;
    const int64_t t0 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t st = int64_t(gridDim.x) * blockDim.x;
    if (v4) {
      const float inf = __int_as_float(0x7F800000);
      float4* d4 = reinterpret_cast<float4*>(d);
      const float4* s4 = reinterpret_cast<const float4*>(sp);
      for (int64_t i = t0; i < (layer >> 2); i += st)
        d4[i] = sep ? make_float4(inf, inf, inf, inf) : __ldg(s4 + i);
    } else {
      for (int64_t i = t0; i < layer; i += st) d[i] = sep ? __int_as_float(0x7F800000) : __ldg(sp + i);
    }
  }
}

// +inf in the separator layers of a stacked batch (layer L of image b: stacked layer
// (b + 1)(L + 1) - 1, for b < batch - 1)
__global__ void k_separators(float* __restrict__ dst, int64_t layer, int64_t layers_per_img,
                             int64_t nsep) {
  for (int64_t b = blockIdx.y; b < nsep; b += gridDim.y) {
    float* d = dst + ((b + 1) * (layers_per_img + 1) - 1) * layer;
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < layer;
         i += int64_t(gridDim.x) * blockDim.x)
      d[i] = __int_as_float(0x7F800000);
  }
}

// Batched emission: keep bars, sort by (image, dim, local kidx), write CSR offsets.
__global__ void k_batch_keys(const uint64_t* __restrict__ rec, int64_t n, int dim,
                             const uint32_t* __restrict__ births, uint32_t cells_per_layer_k,
                             uint32_t klayers_per_img, uint64_t* __restrict__ keys,
                             uint64_t* __restrict__ vals, unsigned* __restrict__ nkeep) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  bool keep = false;
  uint64_t key = 0, val = 0;
  if (i < n) {
    uint64_t r = rec[i];
    uint32_t b = uint32_t(r >> 32), d = uint32_t(r);
    uint32_t bo = births[b];
    uint32_t dor = d == NONE32 ? 0xFFFFFFFFu : births[d];
    keep = (d == NONE32) || (dor > bo);
    // Khalimsky layer of the birth cell along the stacking axis -> image, local kidx
    uint32_t KL = b / cells_per_layer_k;
    uint32_t img = KL / klayers_per_img;
    uint32_t local = b - img * klayers_per_img * cells_per_layer_k;
    key = (uint64_t(img) << 34) | (uint64_t(dim) << 32) | local;
    val = (uint64_t(bo) << 32) | dor;
  }
  unsigned mask = __ballot_sync(0xFFFFFFFFu, keep);
  if (!mask) return;
  int lane = threadIdx.x & 31;
  unsigned base = 0;
  if (lane == __ffs(mask) - 1) base = atomicAdd(nkeep, __popc(mask));
  base = __shfl_sync(0xFFFFFFFFu, base, __ffs(mask) - 1);
  if (keep) {
    unsigned o = base + __popc(mask & ((1u << lane) - 1));
    keys[o] = key;
    vals[o] = val;
  }
}

__global__ void k_batch_write(const uint64_t* __restrict__ keys, const uint64_t* __restrict__ vals,
                              int64_t n, int64_t cap, cr_pair* out, uint32_t* out_cells,
                              unsigned* __restrict__ count) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool in = i < n;
  const uint64_t k = in ? keys[i] : ~0ull, v = in ? vals[i] : 0ull;
  const uint32_t img = uint32_t(k >> 34);
  // per-image counts: the keys are sorted by image, so a warp holds a few runs of equal images;
  // the first lane of each run adds the run's length (one atomic per run, not per bar -- the
  // per-bar atomics on 64 counters serialised: C5b 211 us)
  const int lane = threadIdx.x & 31;
  const uint32_t prev = __shfl_up_sync(0xFFFFFFFFu, img, 1);
  const unsigned heads = __ballot_sync(0xFFFFFFFFu, in && (lane == 0 || prev != img));
  const unsigned inm = __ballot_sync(0xFFFFFFFFu, in);
  if ((heads >> lane) & 1u) {
    const unsigned later = heads & ~((2u << lane) - 1u);  // heads after this lane (lane < 31)
    const int end = lane == 31 || !later ? 32 - __clz(inm) : __ffs(later) - 1;
    atomicAdd(count + img, unsigned(end - lane));
  }
  if (!in || i >= cap) return;
  cr_pair p;
  p.dim = int32_t((k >> 32) & 3);
  p.birth = float_of_ord(uint32_t(v >> 32));
  uint32_t dor = uint32_t(v);
  p.death = dor == 0xFFFFFFFFu ? __int_as_float(0x7F800000) : float_of_ord(dor);
  out[i] = p;
  if (out_cells) out_cells[i] = uint32_t(k);
}

__global__ void k_offsets(const unsigned* __restrict__ count_scan, int64_t batch, int64_t total,
                          int64_t* __restrict__ offsets) {
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < batch) offsets[i] = count_scan[i];
  if (i == batch) offsets[i] = total;
}

int report_dmax(const Geom& g, int maxdim) {
  int top = g.D - 1;
  if (top < 0) top = 0;
  return maxdim < top ? maxdim : top;
}

}  // namespace

// The float32 barcode of one image on the caller's workspace (no profiling brackets, no sync):
// the body of cr_barcodes, shared with cr_barcodes_f64's surrogate pass.
int64_t barcodes_core(const float* image, const Geom& g, int maxdim, cr_pair* out_pairs,
                      uint32_t* out_birth_cells, int64_t out_capacity, Workspace& ws,
                      HostScalars& hs, cr_stats& st) {
  if (g.D <= 1 && !force_general()) {
    st.path = 1;
    return barcodes_1d(image, g.nvox, out_pairs, out_birth_cells, out_capacity, ws, hs, st);
  }
  st.path = 2;
  GeneralState S;
  int dm = report_dmax(g, maxdim);
  run_general(image, g, dm, ws, hs, S, st);
  return emit_bars(S, dm, out_pairs, out_birth_cells, out_capacity, ws, hs, st);
}

void set_last_stats(const cr_stats& st) { commit_stats(st); }

// cr_barcodes_batched_host: copy the host batch straight into the stacked layout on a second
// stream, in up to 8 pieces, each piece's event telling run_general's filtration which z-planes
// have arrived (the filtration of the first pieces overlaps the copy of the later ones).
static void stage_host_batch(const float* host, int64_t batch, int64_t L, int64_t layer,
                             float* simg, GeneralState& S, cudaStream_t s, bool stacked) {
  int dev = 0;
  CR_CUDA(cudaGetDevice(&dev));
  // the copy stream and its events: one set per host thread, re-made on a device change and
  // destroyed when the thread exits
  struct CopyStream {
    int dev = -1;
    cudaStream_t cs = nullptr;
    cudaEvent_t ev[17] = {};
    void destroy() {
      if (dev < 0) return;
      int cur = 0;
      cudaGetDevice(&cur);
      cudaSetDevice(dev);
      cudaStreamSynchronize(cs);
      cudaStreamDestroy(cs);
      for (auto& e : ev) cudaEventDestroy(e);
      cudaSetDevice(cur);
      dev = -1;
    }
    ~CopyStream() { destroy(); }
  };
  static thread_local CopyStream C;
  if (C.dev != dev) {
    C.destroy();
    CR_CUDA(cudaStreamCreateWithFlags(&C.cs, cudaStreamNonBlocking));
    for (auto& e : C.ev) CR_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    C.dev = dev;
  }
  cudaStream_t cs = C.cs;
  cudaEvent_t* ev = C.ev;
  CR_CUDA(cudaEventRecord(ev[16], s));  // the buffer's previous users on s come first
  CR_CUDA(cudaStreamWaitEvent(cs, ev[16], 0));
  if (stacked && batch > 1) {  // 2D: separator rows written in place
    int64_t bx = (layer + 255) / 256;
    if (bx > 64) bx = 64;
    const unsigned by = unsigned(batch - 1 < 65535 ? batch - 1 : 65535);
    k_separators<<<dim3(unsigned(bx), by), 256, 0, s>>>(simg, layer, L, batch - 1);
    CR_CHECK_LAUNCH();
  }
  const int G = int(batch < 8 ? batch : 8);
  const int64_t per = (batch + G - 1) / G;
  S.nready = 0;
  for (int64_t b0 = 0; b0 < batch; b0 += per) {
    const int64_t b1 = b0 + per < batch ? b0 + per : batch;
    if (stacked)
      CR_CUDA(cudaMemcpy2DAsync(simg + b0 * (L + 1) * layer, size_t((L + 1) * layer) * sizeof(float),
                                host + b0 * L * layer, size_t(L * layer) * sizeof(float),
                                size_t(L * layer) * sizeof(float), size_t(b1 - b0),
                                cudaMemcpyHostToDevice, cs));
    else
      CR_CUDA(cudaMemcpyAsync(simg + b0 * L * layer, host + b0 * L * layer,
                              size_t((b1 - b0) * L * layer) * sizeof(float),
                              cudaMemcpyHostToDevice, cs));
    const int i = S.nready++;
    CR_CUDA(cudaEventRecord(ev[i], cs));
    S.ready_ev[i] = ev[i];
    // 3D: the stacked planes of its images (+ the virtual separator after them); 2D: one plane,
    // so the filtration waits for the last piece
    S.ready_z[i] = stacked ? (b1 == batch ? 1 : 0) : b1 * (L + 1);
  }
}

}  // namespace cr

using namespace cr;

extern "C" {

int64_t cr_num_cells(const int64_t* shape, int ndim) {
  if (!valid_shape(shape, ndim)) return -1;
  return make_geom(shape, ndim).ncells;
}

int64_t cr_max_pairs(const int64_t* shape, int ndim, int maxdim) {
  if (!valid_shape(shape, ndim) || maxdim < 0) return -1;
  Geom g = make_geom(shape, ndim);
  int64_t n = 0;
  for (int Z = 0; Z < 2; ++Z)
    for (int Y = 0; Y < 2; ++Y)
      for (int X = 0; X < 2; ++X)
        if (X + Y + Z <= maxdim)
          n += ((g.KZ - Z + 1) / 2) * ((g.KY - Y + 1) / 2) * ((g.KX - X + 1) / 2);
  return n;
}

const char* cr_status_string(cr_status s) {
  switch (s) {
    case CR_OK: return "ok";
    case CR_EINVAL: return "invalid argument (null pointer, bad shape/ndim/maxdim, or NaN in image)";
    case CR_ERANGE: return "output capacity too small (n_pairs holds the required count)";
    case CR_ENOMEM: return "device allocation failed";
    case CR_ECUDA:
    case CR_EINTERNAL: return cr::last_error_text();
  }
  return "unknown status";
}

void cr_last_stats(cr_stats* out) {
  if (!out) return;
  *out = g_last_stats;
  if (g_stats_gen == prof_gen()) prof_fill(*out);
}

void cr_set_profiling(int enable) { cr::set_profiling(enable != 0); }

void cr_release_workspace(void) { cr::release_workspace(); }

int64_t cr_workspace_bytes(void) { return int64_t(cr::workspace_bytes()); }

cr_status cr_set_option(int option, int64_t value) {
  return cr::set_opt(option, value) ? CR_OK : CR_EINVAL;
}

cr_status cr_barcodes(const float* image, const int64_t* shape, int ndim, int maxdim,
                      cr_pair* out_pairs, uint32_t* out_birth_cells, int64_t out_capacity,
                      int64_t* n_pairs, cr_stream_t stream) {
  if (!image || !n_pairs || !valid_shape(shape, ndim) || maxdim < 0 || out_capacity < 0 ||
      (out_capacity > 0 && !out_pairs))
    return CR_EINVAL;
  try {
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    Geom g = make_geom(shape, ndim);
    Workspace ws(s);
    HostScalars hs;
    cr_stats st{};
    prof_begin(s);
    const int64_t n = barcodes_core(image, g, maxdim, out_pairs, out_birth_cells, out_capacity, ws,
                                    hs, st);
    CR_CUDA(cudaStreamSynchronize(s));
    prof_end(st);
    *n_pairs = n;
    if (n > out_capacity) return CR_ERANGE;
    commit_stats(st);
    return CR_OK;
  } catch (const Error& e) {
    return fail(e);
  }
}

cr_status cr_barcodes_topdim(const float* image, const int64_t* shape, int ndim,
                             cr_pair* out_pairs, uint32_t* out_birth_cells, int64_t out_capacity,
                             int64_t* n_pairs, cr_stream_t stream) {
  if (!image || !n_pairs || !valid_shape(shape, ndim) || out_capacity < 0 ||
      (out_capacity > 0 && !out_pairs))
    return CR_EINVAL;
  try {
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    Geom g = make_geom(shape, ndim);
    if (g.D < 2) return CR_EINVAL;  // the top dimension of a 1D image is H0: use cr_barcodes
    Workspace ws(s);
    HostScalars hs;
    cr_stats st{};
    prof_begin(s);
    st.path = 6;
    GeneralState S;
    S.top_only = true;
    run_general(image, g, g.D - 1, ws, hs, S, st);
    const int64_t n = emit_bars(S, g.D - 1, out_pairs, out_birth_cells, out_capacity, ws, hs, st);
    CR_CUDA(cudaStreamSynchronize(s));
    prof_end(st);
    *n_pairs = n;
    if (n > out_capacity) return CR_ERANGE;
    commit_stats(st);
    return CR_OK;
  } catch (const Error& e) {
    return fail(e);
  }
}

cr_status cr_barcodes_host(const float* host_image, const int64_t* shape, int ndim, int maxdim,
                           cr_pair* host_out_pairs, uint32_t* host_out_birth_cells,
                           int64_t out_capacity, int64_t* n_pairs, cr_stream_t stream) {
  if (!host_image || !n_pairs || !valid_shape(shape, ndim) || maxdim < 0 || out_capacity < 0 ||
      (out_capacity > 0 && !host_out_pairs))
    return CR_EINVAL;
  try {
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    Geom g = make_geom(shape, ndim);
    float* dimg = nullptr;
    cr_pair* dout = nullptr;
    uint32_t* dcells = nullptr;
    CR_CUDA(cudaMallocAsync(&dimg, g.nvox * sizeof(float), s));
    int64_t cap = out_capacity > 0 ? out_capacity : 1;
    cudaError_t e1 = cudaMallocAsync(&dout, cap * sizeof(cr_pair), s);
    cudaError_t e2 = host_out_birth_cells ? cudaMallocAsync(&dcells, cap * sizeof(uint32_t), s)
                                          : cudaSuccess;
    cr_status rs = CR_OK;
    if (e1 != cudaSuccess || e2 != cudaSuccess) {
      rs = CR_ENOMEM;
    } else {
      CR_CUDA(cudaMemcpyAsync(dimg, host_image, g.nvox * sizeof(float), cudaMemcpyHostToDevice, s));
      rs = cr_barcodes(dimg, shape, ndim, maxdim, dout, dcells, out_capacity, n_pairs, stream);
      if (rs == CR_OK && *n_pairs > 0) {
        CR_CUDA(cudaMemcpyAsync(host_out_pairs, dout, *n_pairs * sizeof(cr_pair),
                                cudaMemcpyDeviceToHost, s));
        if (host_out_birth_cells)
          CR_CUDA(cudaMemcpyAsync(host_out_birth_cells, dcells, *n_pairs * sizeof(uint32_t),
                                  cudaMemcpyDeviceToHost, s));
      }
    }
    cudaFreeAsync(dimg, s);
    if (dout) cudaFreeAsync(dout, s);
    if (dcells) cudaFreeAsync(dcells, s);
    CR_CUDA(cudaStreamSynchronize(s));
    return rs;
  } catch (const Error& e) {
    return fail(e);
  }
}

// cr_barcodes_batched with the batch on the device (images) or, for the stacked general path,
// in host memory (host_images: copied in pieces straight into the stacked layout).
static cr_status batched_impl(const float* images, const float* host_images, int64_t batch,
                              const int64_t* shape, int ndim, int maxdim, cr_pair* out_pairs,
                              uint32_t* out_birth_cells, int64_t out_capacity,
                              int64_t* out_offsets, int64_t* n_pairs, cr_stream_t stream) {
  if (!n_pairs || !out_offsets || batch < 0 || !valid_shape(shape, ndim) || maxdim < 0 ||
      out_capacity < 0 || (out_capacity > 0 && !out_pairs) ||
      (batch > 0 && !images && !host_images))
    return CR_EINVAL;
  try {
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    Geom g1 = make_geom(shape, ndim);
    if (batch == 0) {
      CR_CUDA(cudaMemsetAsync(out_offsets, 0, sizeof(int64_t), s));
      CR_CUDA(cudaStreamSynchronize(s));
      *n_pairs = 0;
      return CR_OK;
    }
    if (images && g1.nz == 1 && batched_small_2d_fits(g1.ny, g1.nx) && !force_general()) {
      // small 2D images: one CTA per image, everything in shared memory
      Workspace ws(s);
      HostScalars hs;
      cr_stats st{};
      st.path = 5;
      prof_begin(s);
      const int64_t n = barcodes_batched_small_2d(images, batch, g1.ny, g1.nx, maxdim, out_pairs,
                                                  out_birth_cells, out_capacity, out_offsets, ws,
                                                  hs, st);
      if (n >= 0) {
        CR_CUDA(cudaStreamSynchronize(s));
        prof_end(st);
        *n_pairs = n;
        if (n > out_capacity) return CR_ERANGE;
        commit_stats(st);
        return CR_OK;
      }
    }
    // Stack the images along their own slowest axis with one +inf separator layer between
    // consecutive images: the stacked complex is the disjoint union of the images' complexes
    // (every cell touching a separator is absent, reading R5), so its bars are theirs.
    const int64_t L = shape[0];
    int64_t layer = 1;
    for (int i = 1; i < ndim; ++i) layer *= shape[i];
    int64_t stacked[3];
    for (int i = 0; i < ndim; ++i) stacked[i] = shape[i];
    stacked[0] = batch * (L + 1) - 1;
    if (!valid_shape(stacked, ndim)) return CR_EINVAL;
    Geom g = make_geom(stacked, ndim);
    Workspace ws(s);
    HostScalars hs;
    cr_stats st{};
    st.path = 3;
    prof_begin(s);
    // 3D: the filtration reads the volumes unstacked (the separator planes are virtual:
    // KfP::zper), so the batch is never copied into the stacked layout.  2D batches stack along
    // y, which the filtration's plane walk does not see: they are copied into the stacked layout.
    GeneralState S;
    const bool unstacked = ndim == 3;
    const float* simg = images;
    float* staged = nullptr;
    if (unstacked) {
      S.img_zper = uint32_t(L + 1);
      S.img_zimg = uint32_t(L);
      if (host_images) {
        staged = ws.alloc<float>(batch * L * layer);
        stage_host_batch(host_images, batch, L, layer, staged, S, s, false);
        simg = staged;
      }
    } else {
      staged = ws.alloc<float>(g.nvox);
      if (host_images) {
        stage_host_batch(host_images, batch, L, layer, staged, S, s, true);
      } else {
        const int64_t nlayers = g.nvox / layer;
        int64_t bx = (layer / 4 + 255) / 256;
        if (bx < 1) bx = 1;
        if (bx > 64) bx = 64;
        const unsigned by = unsigned(nlayers < 65535 ? nlayers : 65535);
        k_stack<<<dim3(unsigned(bx), by), 256, 0, s>>>(images, L * layer, layer, L, nlayers,
                                                       staged);
        CR_CHECK_LAUNCH();
      }
      simg = staged;
      prof_mark(s, "stack");
    }
    {  // Khalimsky cells per image period along the stacking axis: kidx / seg_cells = image
      uint64_t cl = 1;
      for (int i = 1; i < ndim; ++i) cl *= uint64_t(2 * shape[i] - 1);
      S.seg_cells = uint32_t(cl * uint64_t(2 * (shape[0] + 1)));
    }
    int dm = report_dmax(g1, maxdim);
    run_general(simg, g, dm, ws, hs, S, st);
    if (staged) ws.release(staged);
    // batched emission
    int64_t nrec = 0;
    for (int d = 0; d <= dm; ++d) nrec += S.R.n[d];
    uint64_t* keys = ws.alloc<uint64_t>(nrec + 1);
    uint64_t* vals = ws.alloc<uint64_t>(nrec + 1);
    unsigned* nkeep = ws.alloc<unsigned>(1);
    CR_CUDA(cudaMemsetAsync(nkeep, 0, sizeof(unsigned), s));
    // Khalimsky cells per layer of the stacking axis, and Khalimsky layers per image period
    uint32_t CL = 1;
    for (int i = 1; i < ndim; ++i) CL *= uint32_t(2 * shape[i] - 1);
    const uint32_t KPI = uint32_t(2 * (L + 1));
    for (int d = 0; d <= dm; ++d)
      if (S.R.n[d] > 0) {
        k_batch_keys<<<grid_for(S.R.n[d], 256), 256, 0, s>>>(S.R.rec[d], S.R.n[d], d, S.births,
                                                             CL, KPI, keys, vals, nkeep);
        CR_CHECK_LAUNCH();
      }
    unsigned nk = read_scalar(nkeep, s, hs);
    // sort (image, dim, local kidx) with values
    if (nk > 1)  // key = (image << 34) | (dim << 32) | local kidx: 34 + bits(batch) significant bits
      radix_sort<uint64_t, uint64_t>(keys, vals, nk, 0, 34 + bits_for(uint64_t(batch)), false, ws);
    unsigned* count = ws.alloc<unsigned>(batch + 1);
    unsigned* scan = ws.alloc<unsigned>(batch + 1);
    CR_CUDA(cudaMemsetAsync(count, 0, (batch + 1) * sizeof(unsigned), s));
    if (nk > 0) {
      k_batch_write<<<grid_for(nk, 256), 256, 0, s>>>(keys, vals, nk, out_capacity, out_pairs,
                                                      out_birth_cells, count);
      CR_CHECK_LAUNCH();
    }
    exclusive_sum_u32(count, scan, batch + 1, ws);
    prof_mark(s, "batch_emit");
    k_offsets<<<grid_for(batch + 1, 256), 256, 0, s>>>(scan, batch, nk, out_offsets);
    CR_CHECK_LAUNCH();
    CR_CUDA(cudaStreamSynchronize(s));
    prof_end(st);
    *n_pairs = nk;
    if (int64_t(nk) > out_capacity) return CR_ERANGE;
    commit_stats(st);
    return CR_OK;
  } catch (const Error& e) {
    return fail(e);
  }
}

cr_status cr_barcodes_batched(const float* images, int64_t batch, const int64_t* shape, int ndim,
                              int maxdim, cr_pair* out_pairs, uint32_t* out_birth_cells,
                              int64_t out_capacity, int64_t* out_offsets, int64_t* n_pairs,
                              cr_stream_t stream) {
  if (batch > 0 && !images) return CR_EINVAL;
  return batched_impl(images, nullptr, batch, shape, ndim, maxdim, out_pairs, out_birth_cells,
                      out_capacity, out_offsets, n_pairs, stream);
}

cr_status cr_barcodes_batched_host(const float* host_images, int64_t batch, const int64_t* shape,
                                   int ndim, int maxdim, cr_pair* host_out_pairs,
                                   uint32_t* host_out_birth_cells, int64_t out_capacity,
                                   int64_t* host_out_offsets, int64_t* n_pairs,
                                   cr_stream_t stream) {
  if (!n_pairs || !host_out_offsets || batch < 0 || !valid_shape(shape, ndim) || maxdim < 0 ||
      out_capacity < 0 || (out_capacity > 0 && !host_out_pairs) || (batch > 0 && !host_images))
    return CR_EINVAL;
  try {
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const Geom g = make_geom(shape, ndim);
    const size_t in_bytes = size_t(batch) * size_t(g.nvox) * sizeof(float);
    const int64_t cap = out_capacity > 0 ? out_capacity : 1;
    float* dimg = nullptr;
    cr_pair* dout = nullptr;
    uint32_t* dcells = nullptr;
    int64_t* doff = nullptr;
    cr_status rs = CR_OK;
    // the stacked general path takes the host batch in pieces (overlapping the copy with the
    // filtration); the one-CTA-per-image 2D path and 1D batches take it whole
    const bool staged = batch > 1 && ndim >= 2 &&
                        !(g.nz == 1 && batched_small_2d_fits(g.ny, g.nx) && !force_general());
    if ((!staged && cudaMallocAsync(&dimg, in_bytes > 0 ? in_bytes : 4, s) != cudaSuccess) ||
        cudaMallocAsync(&dout, size_t(cap) * sizeof(cr_pair), s) != cudaSuccess ||
        cudaMallocAsync(&doff, size_t(batch + 1) * sizeof(int64_t), s) != cudaSuccess ||
        (host_out_birth_cells &&
         cudaMallocAsync(&dcells, size_t(cap) * sizeof(uint32_t), s) != cudaSuccess)) {
      cudaGetLastError();
      rs = CR_ENOMEM;
    } else {
      if (staged) {
        rs = batched_impl(nullptr, host_images, batch, shape, ndim, maxdim, dout, dcells,
                          out_capacity, doff, n_pairs, stream);
      } else {
        if (in_bytes)
          CR_CUDA(cudaMemcpyAsync(dimg, host_images, in_bytes, cudaMemcpyHostToDevice, s));
        rs = cr_barcodes_batched(dimg, batch, shape, ndim, maxdim, dout, dcells, out_capacity,
                                 doff, n_pairs, stream);
      }
      if (rs == CR_OK) {
        CR_CUDA(cudaMemcpyAsync(host_out_offsets, doff, size_t(batch + 1) * sizeof(int64_t),
                                cudaMemcpyDeviceToHost, s));
        if (*n_pairs > 0) {
          CR_CUDA(cudaMemcpyAsync(host_out_pairs, dout, size_t(*n_pairs) * sizeof(cr_pair),
                                  cudaMemcpyDeviceToHost, s));
          if (host_out_birth_cells)
            CR_CUDA(cudaMemcpyAsync(host_out_birth_cells, dcells, size_t(*n_pairs) * sizeof(uint32_t),
                                    cudaMemcpyDeviceToHost, s));
        }
      }
    }
    if (dimg) cudaFreeAsync(dimg, s);
    if (dout) cudaFreeAsync(dout, s);
    if (doff) cudaFreeAsync(doff, s);
    if (dcells) cudaFreeAsync(dcells, s);
    CR_CUDA(cudaStreamSynchronize(s));
    return rs;
  } catch (const Error& e) {
    return fail(e);
  }
}

cr_status cr_pairing(const float* image, const int64_t* shape, int ndim, uint32_t* partner,
                     cr_stream_t stream) {
  if (!image || !partner || !valid_shape(shape, ndim)) return CR_EINVAL;
  try {
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    Geom g = make_geom(shape, ndim);
    Workspace ws(s);
    HostScalars hs;
    cr_stats st{};
    if (g.D <= 1 && !force_general()) {
      st.path = 1;
      pairing_1d(image, g.nvox, partner, ws, hs, st);
    } else {
      st.path = 2;
      GeneralState S;
      run_general(image, g, g.D - 1, ws, hs, S, st);
      emit_partner(S, partner, ws);
    }
    CR_CUDA(cudaStreamSynchronize(s));
    commit_stats(st);
    return CR_OK;
  } catch (const Error& e) {
    return fail(e);
  }
}

cr_status cr_death_cells(const float* image, const int64_t* shape, int ndim,
                         const uint32_t* birth_cells, int64_t n, uint32_t* out_death_cells,
                         cr_stream_t stream) {
  if (!image || n < 0 || (n > 0 && (!birth_cells || !out_death_cells)) || !valid_shape(shape, ndim))
    return CR_EINVAL;
  try {
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int64_t nc = cr_num_cells(shape, ndim);
    uint32_t* partner = nullptr;
    CR_CUDA(cudaMallocAsync(&partner, size_t(nc) * sizeof(uint32_t), s));
    cr_status r = cr_pairing(image, shape, ndim, partner, stream);
    if (r == CR_OK && n > 0) {
      k_death_cells<<<grid_for(n, 256), 256, 0, s>>>(birth_cells, n, partner, out_death_cells);
      if (cudaGetLastError() != cudaSuccess) r = CR_ECUDA;
    }
    cudaFreeAsync(partner, s);
    if (r == CR_OK) CR_CUDA(cudaStreamSynchronize(s));
    return r;
  } catch (const Error& e) {
    return fail(e);
  }
}

static cr_status lifetime_common(const float* images, int64_t batch, const int64_t* shape,
                                 int ndim, int maxdim, float inf_value, float* out,
                                 cudaStream_t s) {
  const Geom g = make_geom(shape, ndim);
  const int nch = 2 + report_dmax(g, maxdim);
  const int64_t cap = cr_max_pairs(shape, ndim, maxdim) * batch;
  cr_pair* bars = nullptr;
  uint32_t* cells = nullptr;
  int64_t* offs = nullptr;
  CR_CUDA(cudaMallocAsync(&bars, size_t(cap + 1) * sizeof(cr_pair), s));
  CR_CUDA(cudaMallocAsync(&cells, size_t(cap + 1) * sizeof(uint32_t), s));
  if (batch > 1) CR_CUDA(cudaMallocAsync(&offs, size_t(batch + 1) * sizeof(int64_t), s));
  int64_t n = 0;
  cr_status r = batch > 1
                    ? cr_barcodes_batched(images, batch, shape, ndim, maxdim, bars, cells, cap, offs,
                                          &n, reinterpret_cast<cr_stream_t>(s))
                    : cr_barcodes(images, shape, ndim, maxdim, bars, cells, cap, &n,
                                  reinterpret_cast<cr_stream_t>(s));
  if (r == CR_OK) {
    k_lifetime_init<<<grid_for(g.nvox * batch, 256), 256, 0, s>>>(images, g.nvox, batch, nch, out);
    if (n > 0)
      k_lifetime_scatter<<<grid_for(n, 256), 256, 0, s>>>(bars, cells, n, offs, batch, g, nch,
                                                          inf_value, out);
    if (cudaGetLastError() != cudaSuccess) r = CR_ECUDA;
  }
  cudaFreeAsync(bars, s);
  cudaFreeAsync(cells, s);
  if (offs) cudaFreeAsync(offs, s);
  if (r == CR_OK) CR_CUDA(cudaStreamSynchronize(s));
  return r;
}

cr_status cr_lifetime_image(const float* images, int64_t batch, const int64_t* shape, int ndim,
                            int maxdim, float inf_value, float* out, cr_stream_t stream) {
  if (!images || !out || batch < 1 || maxdim < 0 || !valid_shape(shape, ndim) ||
      inf_value != inf_value)
    return CR_EINVAL;
  try {
    return lifetime_common(images, batch, shape, ndim, maxdim, inf_value, out,
                           reinterpret_cast<cudaStream_t>(stream));
  } catch (const Error& e) {
    return fail(e);
  }
}

}  // extern "C"
