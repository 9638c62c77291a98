/* cr.h -- C ABI of libcr.so: Z/2 persistence barcodes of the weighted cubical complex
 * (V-construction) of a 1D/2D/3D float32 image, computed on a B200 (sm_100a).
 *
 * The operation:
 *   - an image phi is a float32 array over a regular grid; voxels with value +inf lie
 *     outside the (possibly non-rectangular) domain X (reading R5 in DESIGN.md);
 *   - K(phi) has one d-cell per d-dimensional unit cube whose 2^d vertex voxels are all in X;
 *     its birth is the max of its vertex values;
 *   - the barcode lists, per dimension d = 0..min(maxdim, ndim-1), the intervals [birth, death)
 *     of the sublevel-set filtration, death = +inf for classes that never die.
 *
 * Cell index (kidx).  With shape (nz, ny, nx) -- x is the LAST, fastest axis; 1D/2D images get
 * leading sizes of 1 -- a cell is a point (X, Y, Z) of the Khalimsky grid
 * 0 <= X <= 2nx-2, 0 <= Y <= 2ny-2, 0 <= Z <= 2nz-2; axis a is spanned iff its coordinate is odd,
 * and kidx = (Z*(2ny-1) + Y)*(2nx-1) + X.  The voxel of a 0-cell is (X/2, Y/2, Z/2).
 *
 * Total order (reading R1): (birth, dim, kidx) ascending.  The barcode multiset does not depend
 * on it; the cell pairing returned by cr_pairing does, and is unique given it.
 *
 * Conventions for every call:
 *   - pointers documented "device" are CUDA device pointers on the current device; "host" are
 *     ordinary (pageable or pinned) host pointers.  The library never frees or retains them.
 *   - work is enqueued on `stream` (a cudaStream_t; NULL means the legacy default stream) on the
 *     current device.  Calls are blocking: they return after the result is complete.
 *   - workspace: device scratch comes from a per-host-thread, per-device block cache.  Blocks
 *     are handed out again to later calls of the same thread (a steady stream of calls makes no
 *     allocator calls) and are KEPT after a call returns -- a C5-size call leaves a few GB
 *     cached.  cr_release_workspace() returns this thread's blocks to the driver (also done
 *     automatically when the thread exits); cr_workspace_bytes() reports what is held.  If an
 *     allocation fails, the thread's free blocks are released and the allocation retried once.
 *   - synchronisation: a call synchronises with `stream` a few times to size its buffers from
 *     device-side counts (e.g. residual columns), and once at the end to learn n_pairs.
 *   - no state shared between host threads; calls on different streams/devices from different
 *     host threads are safe.  cr_status_string's CUDA error text, cr_last_stats, the options
 *     of cr_set_option and the workspace cache are thread-local.
 *   - on any error, outputs are unspecified; nothing is thrown across the ABI.
 */
#ifndef CR_H_
#define CR_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* cr_stream_t; /* == cudaStream_t */

typedef enum {
  CR_OK = 0,
  CR_EINVAL = -1,   /* null pointer, ndim not in {1,2,3}, shape entry < 1, Khalimsky size >= 2^32-2,
                       maxdim < 0, batch < 0, or a NaN in the image                              */
  CR_ERANGE = -2,   /* out_capacity too small; *n_pairs holds the required count                 */
  CR_ENOMEM = -3,   /* device allocation failed                                                  */
  CR_ECUDA = -4,    /* CUDA runtime error; see cr_status_string                                  */
  CR_EINTERNAL = -5 /* internal invariant violated (a bug); see cr_status_string                 */
} cr_status;

/* One bar [birth, death) of dimension dim.  death = +INFINITY for essential classes.
 * birth is always finite.  12 bytes, packed. */
typedef struct {
  int32_t dim;
  float birth;
  float death;
} cr_pair;

/* Barcode of one image (computePH(arr, maxdim) -> rows (dim, birth, death, ...)).
 *   image           device, float32, C-contiguous, prod(shape) values.  May contain +inf (outside the
 *                   domain) and -inf; -0.0 is treated as +0.0; NaN -> CR_EINVAL.
 *   shape           host, ndim int64 entries, slowest axis first (x last).
 *   ndim            1, 2 or 3.
 *   maxdim          >= 0; dimensions 0..min(maxdim, ndim-1) are reported.
 *   out_pairs       device, out_capacity entries, caller-owned.  Receives the bars with
 *                   death > birth plus all essential bars, ordered by (dim, birth cell kidx)
 *                   ascending -- each bar has a distinct birth cell, so the order is total.
 *   out_birth_cells device or NULL; if non-NULL, out_capacity uint32 entries receiving the kidx of
 *                   each bar's birth cell (the "location" of PAPER.md:331, 438-441).
 *   out_capacity    entries available; cr_max_pairs() is always enough.
 *   n_pairs         host; number of bars written, or the required count on CR_ERANGE.  */
cr_status cr_barcodes(const float* image, const int64_t* shape, int ndim, int maxdim,
                      cr_pair* out_pairs, uint32_t* out_birth_cells, int64_t out_capacity,
                      int64_t* n_pairs, cr_stream_t stream);

/* The top dimension alone (dim D-1 for an image with D axes of extent > 1, D >= 2): the paper's
 * "--top_dim" mode, computed by Alexander duality as a union-find on the dual
 * graph (top cells and the outside as vertices, (D-1)-cells as edges in decreasing birth) -- no
 * H0 and no lower-dimensional reduction.  Arguments and output order as for cr_barcodes; the bars
 * equal cr_barcodes' dim-(D-1) bars.  CR_EINVAL if D < 2.  cr_stats.path = 6. */
cr_status cr_barcodes_topdim(const float* image, const int64_t* shape, int ndim,
                             cr_pair* out_pairs, uint32_t* out_birth_cells, int64_t out_capacity,
                             int64_t* n_pairs, cr_stream_t stream);

/* One bar of a float64 image (cr_barcodes_f64).  24 bytes; pad is 0. */
typedef struct {
  int32_t dim;
  int32_t pad;
  double birth;
  double death;
} cr_pair64;

/* Barcode of a float64 image -- the paper's own value precision ("pixel values ... stored as
 * double").  Arguments, output order and errors as for cr_barcodes, with a device
 * float64 image and cr_pair64 bars whose endpoints are the image's own double values.  The
 * filtration order compares doubles exactly: values that differ only below float32 resolution
 * stay distinct.  Implementation: an order-isomorphic float32 surrogate (the cast when every value
 * is a float32 value, else dense ranks from a device radix sort) run through cr_barcodes, bars
 * mapped back; CR_EINVAL also when ranking is needed and prod(shape) >= 0x7F000000.
 * cr_last_stats describes the float32 pass. */
cr_status cr_barcodes_f64(const double* image, const int64_t* shape, int ndim, int maxdim,
                          cr_pair64* out_pairs, uint32_t* out_birth_cells, int64_t out_capacity,
                          int64_t* n_pairs, cr_stream_t stream);

/* Same as cr_barcodes with HOST image and HOST outputs: the library copies the image in and the
 * bars out on `stream` (end-to-end entry point; pinned host memory is fastest). */
cr_status cr_barcodes_host(const float* host_image, const int64_t* shape, int ndim, int maxdim,
                           cr_pair* host_out_pairs, uint32_t* host_out_birth_cells,
                           int64_t out_capacity, int64_t* n_pairs, cr_stream_t stream);

/* Barcodes of `batch` independent images of identical shape stored back to back -- a batch of
 * images as in the paper's CNN application to (Reduced) MNIST; each image's
 * bars are exactly cr_barcodes' for that image (the complexes are disjoint, reading R16)
 * (images: device, batch*prod(shape) float32).  Bars of image b occupy
 * out_pairs[out_offsets[b] .. out_offsets[b+1]) in the per-image order of cr_barcodes;
 * out_birth_cells (optional) holds kidx within the image.
 * out_offsets: device, batch+1 int64.  n_pairs: host, total bars (or required on CR_ERANGE). */
cr_status cr_barcodes_batched(const float* images, int64_t batch, const int64_t* shape, int ndim,
                              int maxdim, cr_pair* out_pairs, uint32_t* out_birth_cells,
                              int64_t out_capacity, int64_t* out_offsets, int64_t* n_pairs,
                              cr_stream_t stream);

/* cr_barcodes_batched with HOST buffers (the end-to-end batch entry point, BASELINE config 5's
 * batch): host_images (batch*prod(shape) float32, pinned memory is fastest) are copied in, the
 * bars (and birth cells, if host_out_birth_cells is non-NULL) and the batch+1 CSR offsets are
 * copied back to the host buffers before return.  Batches of 2D/3D images on the stacked path
 * are copied in up to 8 pieces, straight into the stacked layout, on a library-owned stream;
 * `stream` waits on each piece before the filtration and H0 forest of its planes run, so the copy
 * overlaps them.  host_images must stay unchanged until return.  Arguments,
 * output order and errors as for cr_barcodes_batched; device staging is allocated stream-ordered
 * and freed before return. */
cr_status cr_barcodes_batched_host(const float* host_images, int64_t batch, const int64_t* shape,
                                   int ndim, int maxdim, cr_pair* host_out_pairs,
                                   uint32_t* host_out_birth_cells, int64_t out_capacity,
                                   int64_t* host_out_offsets, int64_t* n_pairs,
                                   cr_stream_t stream);

/* Full cell pairing, all dimensions (validation): the pairs (birth cell, death cell) of the
 * reduction PAPER.md:130-142 (plus the H0 union-find pairs, and the
 * zero-persistence apparent pairs), unique given the total order R1.
 * partner: device, Khalimsky-size uint32:
 * partner[k] = kidx of the cell paired with cell k (zero-length pairs included),
 * CR_PARTNER_ESSENTIAL if k never dies / is never killed, CR_PARTNER_ABSENT if k has a +inf vertex. */
#define CR_PARTNER_ESSENTIAL 0xFFFFFFFFu
#define CR_PARTNER_ABSENT 0xFFFFFFFEu
cr_status cr_pairing(const float* image, const int64_t* shape, int ndim, uint32_t* partner,
                     cr_stream_t stream);

/* Death cells of bars (the "location ... where it is killed" option of PAPER.md:326-331, 438-441).
 *   image, shape, ndim  as for cr_barcodes (the same image the bars were computed from).
 *   birth_cells         device, n uint32: birth-cell kidx of each bar (cr_barcodes' out_birth_cells).
 *   out_death_cells     device, n uint32: kidx of the cell that kills each bar, CR_PARTNER_ESSENTIAL
 *                       for essential bars.  Computed from the cell pairing (cr_pairing), so the
 *                       call costs about one more barcode computation.  The location is unique
 *                       given the total order (reading R1, R13). */
cr_status cr_death_cells(const float* image, const int64_t* shape, int ndim,
                         const uint32_t* birth_cells, int64_t n, uint32_t* out_death_cells,
                         cr_stream_t stream);

/* Lifetime-enhanced images of `batch` images of identical shape (back to back).
 *   out    device float32, batch * C * prod(shape), C = 2 + min(maxdim, ndim-1): for image b,
 *          channel 0 is the image itself and channel 1+d holds, at each voxel, the largest lifetime
 *          (death - birth) of the dim-d bars whose birth cell has that voxel as its base corner
 *          (X/2, Y/2, Z/2) -- 0 where no bar is born.  Essential bars use death = inf_value.
 *   inf_value  the death assigned to essential bars (e.g. the image maximum); NaN -> CR_EINVAL. */
cr_status cr_lifetime_image(const float* images, int64_t batch, const int64_t* shape, int ndim,
                            int maxdim, float inf_value, float* out, cr_stream_t stream);

/* Number of cells of dims 0..min(maxdim, ndim-1) of the V-construction grid:
 * a safe out_capacity (each bar has a distinct birth cell).  Returns -1 on invalid shape. */
int64_t cr_max_pairs(const int64_t* shape, int ndim, int maxdim);

/* Number of Khalimsky cells prod(2*shape[i]-1) -- every cube of the grid --
 * the partner array length; -1 on invalid shape. */
int64_t cr_num_cells(const int64_t* shape, int ndim);

/* Static description of a status code, or (for CR_ECUDA / CR_EINTERNAL) the thread-local text of
 * the last such error raised on this thread. */
const char* cr_status_string(cr_status s);

/* Counters of the last successful call on this host thread (thread-local). */
typedef struct {
  int64_t cells[4];       /* finite cells per dim                                   */
  int64_t apparent[4];    /* apparent pairs whose lower cell has dim d              */
  int64_t columns[4];     /* residual columns reduced in dim d (d >= 1); basins in [0] */
  int64_t rounds[4];      /* parallel rounds: H0 merge rounds in [0], reduction rounds in [d] */
  int64_t pairs[4];       /* bars with death > birth per dim                        */
  int64_t essential[4];   /* essential bars per dim                                 */
  int64_t path;           /* 1 = 1D tiles, 2 = general, 3 = batched (stacked), 4 = 1D tree,
                             5 = batched small 2D (one CTA per image), 6 = top dimension only */
  int32_t nstages;        /* stages timed (only when profiling is enabled)            */
  float stage_ms[16];     /* device time of each stage, CUDA events on the call's stream */
  char stage_name[16][24];
  int64_t launches;       /* hand-written kernels launched by the call (CUB's not counted) */
  int64_t additions[4];   /* column additions in the dim-d reduction                  */
  int64_t addlen[4];      /* sum over additions of the working column length          */
  int64_t maxlen[4];      /* longest working column in the dim-d reduction             */
  int64_t kf_tma;         /* 1 if the filtration loaded its voxel planes by TMA       */
} cr_stats;
void cr_last_stats(cr_stats* out);

/* Enable (1) / disable (0) per-stage CUDA-event timing on this host thread (default off).
 * When on, each call records an event after every pipeline stage on its stream and fills
 * cr_stats.stage_ms / stage_name; the events add no synchronisation beyond the call's own. */
void cr_set_profiling(int enable);

/* Return this host thread's cached device workspace (every device) to the driver and trim the
 * device memory pools; the next call allocates afresh.  Never fails. */
void cr_release_workspace(void);
/* Device bytes held by this host thread's workspace cache (all devices). */
int64_t cr_workspace_bytes(void);

/* Validation and measurement options of this host thread (thread-local; every option defaults to
 * 0 = the product path).  They select cross-check variants that must give identical results --
 * the tests use them to pin one path against another -- or perturb the schedule of the
 * parallel reduction, whose result does not depend on it.  Returns CR_EINVAL for
 * an unknown option.  Not read from the environment. */
typedef enum {
  CR_OPT_FORCE_GENERAL = 1,    /* 1D images through the general 3D path (not the 1D tiles)      */
  CR_OPT_1D_TREE = 2,          /* 1D images through the tree path (not the tiles)               */
  CR_OPT_TOP_REDUCE = 3,       /* top dimension by the coboundary reduction (not duality)       */
  CR_OPT_K5_BLOCKS_PER_SM = 4, /* resident blocks per SM of the reduction (0: occupancy limit)  */
  CR_OPT_K5_JITTER_NS = 5,     /* pseudo-random delays up to this many ns inside the reduction   */
  CR_OPT_DEBUG = 6,            /* per-stage counters printed to stderr                          */
  CR_OPT_KF_TMA = 7,           /* filtration voxel ring by TMA (cp.async.bulk.tensor) when the row
                                  pitch allows it, not per-thread cp.async (measured slower)      */
  CR_OPT_KF_RCAP = 8           /* residual edges a filtration CTA stages in shared memory before
                                  appending to the global list directly (0: 1024; tests)         */
} cr_option;
cr_status cr_set_option(int option, int64_t value);

#ifdef __cplusplus
}
#endif
#endif /* CR_H_ */
