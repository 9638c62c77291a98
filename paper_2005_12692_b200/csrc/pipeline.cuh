// pipeline.cuh -- host-side stages of the general (1D/2D/3D) path and the 1D path.
#pragma once
#include <cstdlib>

#include "workspace.cuh"

namespace cr {

// Pair records: (birth cell kidx << 32) | death cell kidx, death = NONE32 for essential classes.
struct Records {
  uint64_t* rec[4] = {nullptr, nullptr, nullptr, nullptr};
  int64_t n[4] = {0, 0, 0, 0};
};

struct H0Cand {   // an H0 candidate edge (general.cu): its key and two current component roots
  uint64_t key;
  uint32_t a, b;
};

struct GeneralState {
  Geom g;
  uint32_t* births = nullptr;  // ord(birth) per kidx, ABSENT_ORD for +inf
  uint8_t* tags = nullptr;     // see cr_internal.cuh
  uint32_t seg_cells = 0;      // batched: Khalimsky cells per image period (kidx / seg_cells =
                               // image); 0 for a single image
  bool top_only = false;       // compute only dimension D-1, by duality (cr_barcodes_topdim)
  bool lower_essential_known = false;  // cr_stats.essential[e] holds every e < current dim
  // Input arriving in pieces (cr_barcodes_batched_host): planes [0, ready_z[i]) of the image are
  // on the device once event ready_ev[i] has fired; the filtration launches its z-chunks as their
  // planes (and the 4 after them it reads) arrive instead of waiting for the whole copy.
  // a stacked batch read unstacked by the filtration (see KfP::zper): planes per image period
  // (images + separator) and per image; 0 = the image is laid out as the geometry says
  uint32_t img_zper = 0, img_zimg = 0;
  // H0's candidate list, kept for the dim-1 columns: every residual edge is an H0 candidate
  // (listed by k_filtration), and the residual edges that H0 did not clear are exactly the dim-1
  // columns, so reduce_dimension(1) compacts this list instead of scanning the grid (nullptr:
  // scan)
  const H0Cand* h0_cand = nullptr;
  uint32_t h0_ncand = 0;
  // the residual present (D-1)-cells listed by the filtration (kidx; device count): the faces of
  // the top-dimension dual (cleared ones are skipped there); nullptr: not listed
  uint32_t* res_faces = nullptr;
  const unsigned* nres_faces = nullptr;
  uint32_t* dual_parent = nullptr;  // the top-dimension dual forest built by the filtration
  int nready = 0;
  int64_t ready_z[16];
  cudaEvent_t ready_ev[16];
  Records R;
};

Geom make_geom(const int64_t* shape, int ndim);

// K1 + K2 + H0 + reductions for dims 1..dmax (dmax <= D-1).  Throws Error.
void run_general(const float* image, const Geom& g, int dmax, Workspace& ws, HostScalars& hs,
                 GeneralState& S, cr_stats& st);

// Residual coboundary column reduction of dimension d (reduce.cu): columns = residual d-cells in
// decreasing key order; appends records to R.rec[d] and marks the pivots cleared for d+1.
void reduce_dimension(GeneralState& S, int d, Workspace& ws, HostScalars& hs, cr_stats& st);

// Records (dims 0..maxdim) -> bars with death > birth plus essentials, ordered (dim, birth kidx).
// Writes at most cap entries; returns the count needed.
int64_t emit_bars(const GeneralState& S, int maxdim, cr_pair* out, uint32_t* out_cells,
                  int64_t cap, Workspace& ws, HostScalars& hs, cr_stats& st);

// Full pairing from tags + records.
void emit_partner(const GeneralState& S, uint32_t* partner, Workspace& ws);

// 1D path (path1d.cu).  image has n voxels along one axis; cell kidx = 2i (vertex), 2i+1 (edge).
// Fused tile path (path1d_tiles.cu); returns -1 if its contraction levels did not finish
// (adversarial inputs), in which case barcodes_1d falls back to the tree path (path1d.cu).
int64_t barcodes_1d_tiles(const float* image, int64_t n, cr_pair* out, uint32_t* out_cells,
                          int64_t cap, Workspace& ws, HostScalars& hs, cr_stats& st);
int64_t barcodes_1d_tree(const float* image, int64_t n, cr_pair* out, uint32_t* out_cells,
                         int64_t cap, Workspace& ws, HostScalars& hs, cr_stats& st);
inline int64_t barcodes_1d(const float* image, int64_t n, cr_pair* out, uint32_t* out_cells,
                           int64_t cap, Workspace& ws, HostScalars& hs, cr_stats& st) {
  if (opt(OPT_1D_TREE) == 0) {
    int64_t r = barcodes_1d_tiles(image, n, out, out_cells, cap, ws, hs, st);
    if (r >= 0) return r;
    st.path = 4;  // tile levels did not converge: tree path
  }
  return barcodes_1d_tree(image, n, out, out_cells, cap, ws, hs, st);
}
void pairing_1d(const float* image, int64_t n, uint32_t* partner, Workspace& ws, HostScalars& hs,
                cr_stats& st);

// Batches of small 2D images, one CTA per image (batched.cu).  Returns -1 if an image did not fit
// the per-CTA buffers (the caller then uses the stacked device-wide path).
bool batched_small_2d_fits(int64_t ny, int64_t nx);
int64_t barcodes_batched_small_2d(const float* images, int64_t batch, int64_t ny, int64_t nx,
                                  int maxdim, cr_pair* out, uint32_t* out_cells, int64_t cap,
                                  int64_t* out_offsets, Workspace& ws, HostScalars& hs,
                                  cr_stats& st);

// The float32 barcode on the caller's workspace, no profiling brackets (api.cu).
int64_t barcodes_core(const float* image, const Geom& g, int maxdim, cr_pair* out_pairs,
                      uint32_t* out_birth_cells, int64_t out_capacity, Workspace& ws,
                      HostScalars& hs, cr_stats& st);
void set_last_stats(const cr_stats& st);

// Hand-written stable LSD radix sort (sort.cu) over key bits [begin_bit, end_bit), values optional
// (vals == nullptr); instantiated for (u64, u64), (u64, u32), (u32, u64).
template <class K, class V>
void radix_sort(K* keys, V* vals, int64_t n, int begin_bit, int end_bit, bool descending,
                Workspace& ws);
void sort_keys_u64(uint64_t* keys, int64_t n, bool descending, int end_bit, Workspace& ws,
                   int begin_bit = 0);
inline int bits_for(uint64_t v) {  // significant bits of values < v (v >= 1)
  int b = 0;
  while (b < 64 && (uint64_t(1) << b) < v) ++b;
  return b;
}
// Device-wide helpers (util.cu).
void exclusive_sum_u32(const uint32_t* in, uint32_t* out, int64_t n, Workspace& ws);

}  // namespace cr
