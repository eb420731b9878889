// mg_lgf.cpp — lattice Green's functions of the multigrid operator (host, setup only).
//
// PAPER.md §2.2: the coarse solve convolves with the LGF of the same
// difference operator, ℒG = δ; §3.3: compatibility is required for
// convergence.  Construction (reading R-LGF): solve ℒG = δ exactly in
// the box |n|_inf <= R, with the continuum Green's function on the box shell
// (3D: -1/(4π|n|); 2D: ln|n|/(2π), then G[0,0] := 0), by the sine transform
// (DST-I) that diagonalises every polynomial in the 1D second differences.
// Written independently of the oracle (plain O(n^2) DST per line, no FFT).
#include <cmath>
#include <vector>

namespace mg {

static double op_symbol(const double* lam, int dim, int order) {
  double s = 0.0;
  for (int a = 0; a < dim; ++a) s += lam[a];
  if (order >= 4) {
    double p = 0.0;
    for (int a = 0; a < dim; ++a)
      for (int b = a + 1; b < dim; ++b) p += lam[a] * lam[b];
    s += p / 6.0;
  }
  if (order == 6 && dim == 3) s += lam[0] * lam[1] * lam[2] / 30.0;  // E13 (reading Z24)
  return s;
}

// stencil weight of ℒ (dimensionless) at offset with `nz` non-zero components
static double op_weight(int dim, int order, int nz) {
  if (order == 2) return nz == 0 ? -2.0 * dim : (nz == 1 ? 1.0 : 0.0);
  if (dim == 3 && order == 6)  // fig:stencils M=6: {-128, 14, 3, 1} / 30
    return nz == 0 ? -128.0 / 30.0 : (nz == 1 ? 14.0 / 30.0 : (nz == 2 ? 3.0 / 30.0 : 1.0 / 30.0));
  if (dim == 3) return nz == 0 ? -4.0 : (nz == 1 ? 1.0 / 3.0 : (nz == 2 ? 1.0 / 6.0 : 0.0));
  return nz == 0 ? -10.0 / 3.0 : (nz == 1 ? 2.0 / 3.0 : 1.0 / 6.0);   // 2D Mehrstellen
}

// in-place orthonormal DST-I along one axis of an m^dim array (stride/len given)
static void dst1_lines(std::vector<double>& a, int m, int dim, int axis, const std::vector<double>& S) {
  std::vector<double> line(m), out(m);
  const long stride = (axis == 0) ? 1 : (axis == 1 ? m : (long)m * m);
  const long total = dim == 2 ? (long)m * m : (long)m * m * m;
  for (long base = 0; base < total; ++base) {
    // base must have index 0 along `axis`
    if ((base / stride) % m != 0) continue;
    for (int j = 0; j < m; ++j) line[j] = a[base + j * stride];
    for (int k = 0; k < m; ++k) {
      double acc = 0.0;
      const double* row = &S[(size_t)k * m];
      for (int j = 0; j < m; ++j) acc += row[j] * line[j];
      out[k] = acc;
    }
    for (int j = 0; j < m; ++j) a[base + j * stride] = out[j];
  }
}

// G on [-R, R]^dim, index (n + R) with x fastest
std::vector<double> box_lgf(int dim, int order, int R) {
  const int n = 2 * R + 1, m = n - 2;
  const long tot = dim == 2 ? (long)n * n : (long)n * n * n;
  std::vector<double> G(tot, 0.0);
  auto idx = [&](int x, int y, int z) -> long { return dim == 2 ? (long)y * n + x : ((long)z * n + y) * n + x; };
  // shell values
  for (long i = 0; i < tot; ++i) {
    const int x = (int)(i % n), y = (int)((i / n) % n), z = dim == 3 ? (int)(i / ((long)n * n)) : R;
    const bool shell = x == 0 || x == n - 1 || y == 0 || y == n - 1 || (dim == 3 && (z == 0 || z == n - 1));
    if (!shell) continue;
    const double X = x - R, Y = y - R, Z = dim == 3 ? z - R : 0.0;
    const double r = std::sqrt(X * X + Y * Y + Z * Z);
    G[i] = dim == 3 ? -1.0 / (4.0 * M_PI * r) : std::log(r) / (2.0 * M_PI);
  }
  // right-hand side on the interior: δ - ℒ(shell)
  const long mt = dim == 2 ? (long)m * m : (long)m * m * m;
  std::vector<double> b(mt, 0.0);
  for (long i = 0; i < mt; ++i) {
    const int x = (int)(i % m) + 1, y = (int)((i / m) % m) + 1, z = dim == 3 ? (int)(i / ((long)m * m)) + 1 : 0;
    double acc = 0.0;
    for (int dz = (dim == 3 ? -1 : 0); dz <= (dim == 3 ? 1 : 0); ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          const int xx = x + dx, yy = y + dy, zz = z + dz;
          const bool shell = xx == 0 || xx == n - 1 || yy == 0 || yy == n - 1 || (dim == 3 && (zz == 0 || zz == n - 1));
          if (!shell) continue;
          const int nz = (dx != 0) + (dy != 0) + (dz != 0);
          acc += op_weight(dim, order, nz) * G[idx(xx, yy, zz)];
        }
    b[i] = -acc;
    if (x == R && y == R && (dim == 2 || z == R)) b[i] += 1.0;
  }
  std::vector<double> S((size_t)m * m), lam(m);
  const double sc = std::sqrt(2.0 / (m + 1));
  for (int k = 0; k < m; ++k) {
    lam[k] = 2.0 * std::cos(M_PI * (k + 1) / (m + 1)) - 2.0;
    for (int j = 0; j < m; ++j) S[(size_t)k * m + j] = sc * std::sin(M_PI * (double)(j + 1) * (k + 1) / (m + 1));
  }
  for (int a = 0; a < dim; ++a) dst1_lines(b, m, dim, a, S);
  for (long i = 0; i < mt; ++i) {
    double l[3];
    l[0] = lam[i % m];
    l[1] = lam[(i / m) % m];
    l[2] = dim == 3 ? lam[i / ((long)m * m)] : 0.0;
    b[i] /= op_symbol(l, dim, order);
  }
  for (int a = 0; a < dim; ++a) dst1_lines(b, m, dim, a, S);
  for (long i = 0; i < mt; ++i) {
    const int x = (int)(i % m) + 1, y = (int)((i / m) % m) + 1, z = dim == 3 ? (int)(i / ((long)m * m)) + 1 : 0;
    G[idx(x, y, z)] = b[i];
  }
  if (dim == 2) {
    const double g0 = G[idx(R, R, 0)];
    for (auto& v : G) v -= g0;
  }
  return G;
}

}  // namespace mg
