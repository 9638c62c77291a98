// cr_oracle.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A plain, slow, obviously-correct CPU computation of the Z/2 persistence barcode of
// the weighted cubical complex K(phi) (V-construction) of a 1D/2D/3D float32 image (and, with the
// same code instantiated for double, of a float64 image: the paper's own precision).
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
// load this library.  It shares no code, header or table with the CUDA path
// (paper_2005_12692_b200/csrc); the product never links or imports it.
//
// What it computes, step by step (each step cites the passage it follows):
//   1. validate, map -0.0 -> +0.0, reject NaN                      (reading R7)
//   2. enumerate every cubical cell; birth = max of its vertex values
//      a cell with a +inf vertex lies outside the domain X and is absent (R5)
//   3. order the cells by (birth, dim, kidx) ascending                    (reading R1)
//   4. build the explicit boundary matrix over Z/2 (facets of each cell)  (transposed)
//   5. reduce it left to right: add an earlier column while the lowest
//      entries coincide; a pivot (i, j) is the bar [birth_i, birth_j)
//      "twist" mode processes dimensions top-down and skips the column of every
//      pivot row, which the D^2 = 0 argument shows is zero
//   6. read out: pairs with death > birth plus essential classes (death = +inf),
//      dims 0..maxdim, and the full cell pairing (partner array)
//
// The homology reduction of the boundary matrix and the cohomology reduction of the
// coboundary matrix that the paper describes produce the same
// pairs for the same total order (the paper defers to [cohomology] for this).
//
// Pins (tests/test_oracle.py): brute-force persistent Betti numbers from GF(2) ranks,
// an independent cohomology reduction, elder-rule union-find, closed forms and the
// paper's worked examples (tests/golden/).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

namespace {

constexpr uint32_t NONE = 0xFFFFFFFFu;
constexpr uint32_t PARTNER_ESSENTIAL = 0xFFFFFFFFu;
constexpr uint32_t PARTNER_ABSENT = 0xFFFFFFFEu;

struct Grid {
  int64_t nx = 1, ny = 1, nz = 1;  // voxels per axis; x is the fastest (last) axis
  int64_t KX = 1, KY = 1, KZ = 1;  // Khalimsky extents 2n-1
  int64_t ncells() const { return KX * KY * KZ; }
  int64_t kidx(int64_t X, int64_t Y, int64_t Z) const { return (Z * KY + Y) * KX + X; }
};

template <class T>
struct Cell {
  T birth;
  int dim;
  uint32_t kidx;
};

// Step 1+2: cell births over the Khalimsky grid; returns false on NaN.
template <class T>
bool cell_births(const T* image, const Grid& g, std::vector<T>& birth) {
  const int64_t nvox = g.nx * g.ny * g.nz;
  std::vector<T> v(nvox);
  for (int64_t i = 0; i < nvox; ++i) {
    T f = image[i];
    if (std::isnan(f)) return false;
    if (f == T(0)) f = T(0);  // -0.0 -> +0.0 (reading R7)
    v[i] = f;
  }
  birth.assign(g.ncells(), T(0));
  for (int64_t Z = 0; Z < g.KZ; ++Z)
    for (int64_t Y = 0; Y < g.KY; ++Y)
      for (int64_t X = 0; X < g.KX; ++X) {
        // vertices: floor/ceil of half the Khalimsky coordinate on every odd axis
        T b = -T(INFINITY);
        for (int64_t z = Z / 2; z <= (Z + 1) / 2; ++z)
          for (int64_t y = Y / 2; y <= (Y + 1) / 2; ++y)
            for (int64_t x = X / 2; x <= (X + 1) / 2; ++x) {
              T f = v[(z * g.ny + y) * g.nx + x];
              if (f > b) b = f;  // birth = max over the cell's vertices
            }
        birth[g.kidx(X, Y, Z)] = b;
      }
  return true;
}

int cell_dim(const Grid& g, int64_t k) {
  int64_t X = k % g.KX, Y = (k / g.KX) % g.KY, Z = k / (g.KX * g.KY);
  return int(X & 1) + int(Y & 1) + int(Z & 1);
}

// facets of cell k: Khalimsky coordinate -1 and +1 on every odd axis
void facets(const Grid& g, int64_t k, std::vector<int64_t>& out) {
  out.clear();
  int64_t X = k % g.KX, Y = (k / g.KX) % g.KY, Z = k / (g.KX * g.KY);
  if (X & 1) { out.push_back(g.kidx(X - 1, Y, Z)); out.push_back(g.kidx(X + 1, Y, Z)); }
  if (Y & 1) { out.push_back(g.kidx(X, Y - 1, Z)); out.push_back(g.kidx(X, Y + 1, Z)); }
  if (Z & 1) { out.push_back(g.kidx(X, Y, Z - 1)); out.push_back(g.kidx(X, Y, Z + 1)); }
}

using Column = std::vector<uint32_t>;  // sorted filtration positions

void add_column(Column& dst, const Column& src) {  // Z/2 sum = symmetric difference
  Column r;
  r.reserve(dst.size() + src.size());
  std::set_symmetric_difference(dst.begin(), dst.end(), src.begin(), src.end(),
                                std::back_inserter(r));
  dst.swap(r);
}

bool setup_grid(const int64_t* shape, int ndim, Grid& g) {
  if (ndim < 1 || ndim > 3 || !shape) return false;
  int64_t s[3] = {1, 1, 1};  // (nz, ny, nx)
  for (int i = 0; i < ndim; ++i) {
    if (shape[i] < 1) return false;
    s[3 - ndim + i] = shape[i];
  }
  g.nz = s[0]; g.ny = s[1]; g.nx = s[2];
  g.KX = 2 * g.nx - 1; g.KY = 2 * g.ny - 1; g.KZ = 2 * g.nz - 1;
  if (g.ncells() >= (int64_t(1) << 32) - 2) return false;
  return true;
}

// Steps 3-6 for either value type (float32 product precision, float64 paper precision).
//   out_dim/out_birth/out_death/out_cell: capacity `cap` entries (may be NULL if cap == 0);
//     pairs with death > birth and essential classes (death = +inf), dims <= maxdim,
//     ordered by (dim, birth-cell kidx) ascending.
//   partner: NULL or Khalimsky-size uint32: paired cell's kidx, 0xFFFFFFFF essential,
//     0xFFFFFFFE absent (+inf birth).  Always covers all dimensions.
//   stats: NULL or int64[12]: per dim d in 0..3: [3d] positive pairs, [3d+1] zero pairs,
//     [3d+2] essential classes (all dims, independent of maxdim).
// Returns the number of output pairs (may exceed cap; nothing beyond cap is written),
// or -1 on invalid input (NaN, bad shape, maxdim < 0).
template <class T>
int64_t ph_impl(const T* image, const int64_t* shape, int ndim, int maxdim, int twist,
                int32_t* out_dim, T* out_birth, T* out_death, uint32_t* out_cell,
                int64_t cap, uint32_t* partner, int64_t* stats) {
  Grid g;
  if (!image || maxdim < 0 || !setup_grid(shape, ndim, g)) return -1;
  std::vector<T> birth;
  if (!cell_births(image, g, birth)) return -1;
  const int64_t N = g.ncells();

  // Step 3: the present cells in filtration order (birth, dim, kidx).
  std::vector<Cell<T>> cells;
  cells.reserve(N);
  for (int64_t k = 0; k < N; ++k)
    if (birth[k] != T(INFINITY)) cells.push_back({birth[k], cell_dim(g, k), uint32_t(k)});
  std::sort(cells.begin(), cells.end(), [](const Cell<T>& a, const Cell<T>& b) {
    if (a.birth != b.birth) return a.birth < b.birth;
    if (a.dim != b.dim) return a.dim < b.dim;
    return a.kidx < b.kidx;
  });
  const uint32_t M = uint32_t(cells.size());
  std::vector<uint32_t> pos(N, NONE);
  for (uint32_t r = 0; r < M; ++r) pos[cells[r].kidx] = r;

  // Step 4: boundary columns (in filtration positions, sorted ascending).
  std::vector<Column> col(M);
  std::vector<int64_t> f;
  for (uint32_t r = 0; r < M; ++r) {
    facets(g, cells[r].kidx, f);
    for (int64_t k : f) col[r].push_back(pos[k]);  // a facet of a present cell is present
    std::sort(col[r].begin(), col[r].end());
  }

  // Step 5: left-to-right reduction.  owner[i] = column whose lowest entry is i.
  std::vector<uint32_t> owner(M, NONE), paired_with(M, NONE);
  std::vector<char> cleared(M, 0);
  auto reduce = [&](uint32_t j) {
    Column& c = col[j];
    while (!c.empty() && owner[c.back()] != NONE) add_column(c, col[owner[c.back()]]);
    if (!c.empty()) {
      uint32_t low = c.back();
      owner[low] = j;
      paired_with[low] = j;
      paired_with[j] = low;
      cleared[low] = 1;  // twist: column `low` reduces to zero
    }
  };
  if (twist) {
    for (int d = 3; d >= 1; --d)
      for (uint32_t j = 0; j < M; ++j)
        if (cells[j].dim == d && !cleared[j]) reduce(j);
  } else {
    for (uint32_t j = 0; j < M; ++j)
      if (cells[j].dim >= 1) reduce(j);
  }

  // Step 6: read out.
  if (partner) {
    for (int64_t k = 0; k < N; ++k) partner[k] = PARTNER_ABSENT;
    for (uint32_t r = 0; r < M; ++r)
      partner[cells[r].kidx] =
          paired_with[r] == NONE ? PARTNER_ESSENTIAL : cells[paired_with[r]].kidx;
  }
  struct Out { int32_t dim; T b, d; uint32_t cell; };
  std::vector<Out> outs;
  int64_t st[12] = {0};
  for (uint32_t r = 0; r < M; ++r) {
    const Cell<T>& c = cells[r];
    if (paired_with[r] == NONE) {
      st[3 * c.dim + 2]++;
      if (c.dim <= maxdim) outs.push_back({c.dim, c.birth, T(INFINITY), c.kidx});
    } else if (paired_with[r] > r) {  // r is the birth (lower) cell of its pair
      T death = cells[paired_with[r]].birth;
      if (death > c.birth) {
        st[3 * c.dim]++;
        if (c.dim <= maxdim) outs.push_back({c.dim, c.birth, death, c.kidx});
      } else {
        st[3 * c.dim + 1]++;
      }
    }
  }
  std::sort(outs.begin(), outs.end(), [](const Out& a, const Out& b) {
    if (a.dim != b.dim) return a.dim < b.dim;
    return a.cell < b.cell;
  });
  for (int64_t i = 0; i < int64_t(outs.size()) && i < cap; ++i) {
    if (out_dim) out_dim[i] = outs[i].dim;
    if (out_birth) out_birth[i] = outs[i].b;
    if (out_death) out_death[i] = outs[i].d;
    if (out_cell) out_cell[i] = outs[i].cell;
  }
  if (stats) std::memcpy(stats, st, sizeof(st));
  return int64_t(outs.size());
}

}  // namespace

extern "C" {

// Khalimsky-grid births (float32, +inf for absent cells).  0 on success, -1 on bad input/NaN.
int oracle_births(const float* image, const int64_t* shape, int ndim, float* out) {
  Grid g;
  if (!image || !out || !setup_grid(shape, ndim, g)) return -1;
  std::vector<float> b;
  if (!cell_births(image, g, b)) return -1;
  std::memcpy(out, b.data(), sizeof(float) * b.size());
  return 0;
}

// Full persistence computation (float32 image; births and deaths are float32).
//   out_dim/out_birth/out_death/out_cell: capacity `cap` entries (may be NULL if cap == 0);
//     pairs with death > birth and essential classes (death = +inf), dims <= maxdim,
//     ordered by (dim, birth-cell kidx) ascending.
//   partner: NULL or Khalimsky-size uint32: paired cell's kidx, 0xFFFFFFFF essential,
//     0xFFFFFFFE absent (+inf birth).  Always covers all dimensions.
//   stats: NULL or int64[12]: per dim d in 0..3: [3d] positive pairs, [3d+1] zero pairs,
//     [3d+2] essential classes (all dims, independent of maxdim).
// Returns the number of output pairs (may exceed cap; nothing beyond cap is written),
// or -1 on invalid input (NaN, bad shape, maxdim < 0).
int64_t oracle_ph(const float* image, const int64_t* shape, int ndim, int maxdim, int twist,
                  int32_t* out_dim, float* out_birth, float* out_death, uint32_t* out_cell,
                  int64_t cap, uint32_t* partner, int64_t* stats) {
  return ph_impl<float>(image, shape, ndim, maxdim, twist, out_dim, out_birth, out_death,
                        out_cell, cap, partner, stats);
}

// The same computation on a float64 image (the paper's own precision): the
// filtration order compares doubles, births and deaths are doubles.  Same contract as oracle_ph.
int64_t oracle_ph_f64(const double* image, const int64_t* shape, int ndim, int maxdim, int twist,
                      int32_t* out_dim, double* out_birth, double* out_death, uint32_t* out_cell,
                      int64_t cap, uint32_t* partner, int64_t* stats) {
  return ph_impl<double>(image, shape, ndim, maxdim, twist, out_dim, out_birth, out_death,
                         out_cell, cap, partner, stats);
}

// Khalimsky-grid births of a float64 image.  0 on success, -1 on bad input/NaN.
int oracle_births_f64(const double* image, const int64_t* shape, int ndim, double* out) {
  Grid g;
  if (!image || !out || !setup_grid(shape, ndim, g)) return -1;
  std::vector<double> b;
  if (!cell_births(image, g, b)) return -1;
  std::memcpy(out, b.data(), sizeof(double) * b.size());
  return 0;
}

}  // extern "C"
