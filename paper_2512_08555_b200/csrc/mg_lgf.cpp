// mg_lgf.cpp — lattice Green's functions of the multigrid operator (host, setup only).
//
// PAPER.md §2.2: the coarse solve convolves with the LGF of the same
// difference operator, ℒG = δ; §3.3: compatibility is required for
// convergence.  Construction (reading R-LGF): solve ℒG = δ exactly in
// the box |n|_inf <= R, with the continuum Green's function on the box shell
// (3D: -1/(4π|n|); 2D: ln|n|/(2π), then G[0,0] := 0), by the sine transform
// (DST-I) that diagonalises every polynomial in the 1D second differences.
// Written independently of the oracle (an O(n^2) DST per line, no FFT).
#include <cublas_v2.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <thread>
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

// in-place orthonormal DST-I along one axis of an m^dim array: out[k] = Σ_j S[k][j] in[j]
// per line.  S is symmetric, so a line is accumulated as Σ_j in[j] S[j][:] (contiguous
// rows of S: vectorisable without reassociating a reduction), lines split over host
// threads (setup only; O(m^4) for a 3-D box, the 3-D LGF of a padded semi-unbounded
// coarse level has m ≈ 285).
static void dst1_lines(std::vector<double>& a, int m, int dim, int axis, const std::vector<double>& S) {
  const long stride = (axis == 0) ? 1 : (axis == 1 ? m : (long)m * m);
  const long nlines = dim == 2 ? (long)m : (long)m * m;
  // line l -> base offset: the line index enumerates the other axes, x fastest
  auto base_of = [&](long l) -> long {
    if (axis == 0) return l * m;
    if (axis == 1) return (l % m) + (l / m) * (long)m * m;
    return l;  // axis 2: (x, y) = l
  };
  auto work = [&](long l0, long l1) {
    std::vector<double> line(m), out(m);
    for (long l = l0; l < l1; ++l) {
      const long base = base_of(l);
      for (int j = 0; j < m; ++j) line[j] = a[base + j * stride];
      std::fill(out.begin(), out.end(), 0.0);
      for (int j = 0; j < m; ++j) {
        const double v = line[j];
        const double* row = &S[(size_t)j * m];
        for (int k = 0; k < m; ++k) out[k] += v * row[k];
      }
      for (int j = 0; j < m; ++j) a[base + j * stride] = out[j];
    }
  };
  unsigned nt = std::thread::hardware_concurrency();
  nt = nt == 0 ? 1 : (nt > 32 ? 32 : nt);
  if (nlines < 64 || nt == 1) {
    work(0, nlines);
    return;
  }
  std::vector<std::thread> th;
  const long chunk = (nlines + nt - 1) / nt;
  for (unsigned t = 0; t < nt; ++t) {
    const long l0 = t * chunk, l1 = std::min(nlines, l0 + chunk);
    if (l0 < l1) th.emplace_back(work, l0, l1);
  }
  for (auto& x : th) x.join();
}

// The three DST-I passes of an m^3 array (x fastest) as DGEMMs on the device (S is
// symmetric): along x, X' = S X with X the m x m^2 column-major view; along y, per z
// slice Z' = Z S (strided batch); along z, W' = W S with W the m^2 x m view.  The
// symbol division `divide` runs on the host between the forward and inverse passes.
// For the 3-D LGF of a padded semi-unbounded coarse level (m ≈ 285, 8e10 flop) this
// replaces ~5 s of host time by ~0.1 s.  false (host path) if CUDA or cuBLAS fails.
template <class F>
static bool dst3_gpu(std::vector<double>& a, int m, const std::vector<double>& S, F&& divide) {
  const size_t n3 = (size_t)m * m * m, n2 = (size_t)m * m;
  double *dA = nullptr, *dB = nullptr, *dS = nullptr;
  cublasHandle_t hb = nullptr;
  bool ok = cudaMalloc(&dA, n3 * sizeof(double)) == cudaSuccess && cudaMalloc(&dB, n3 * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&dS, n2 * sizeof(double)) == cudaSuccess && cublasCreate(&hb) == CUBLAS_STATUS_SUCCESS;
  const double one = 1.0, zero = 0.0;
  auto passes = [&]() -> bool {
    if (cudaMemcpy(dA, a.data(), n3 * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess) return false;
    bool r = cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, m, (int)n2, m, &one, dS, m, dA, m, &zero, dB, m) ==
             CUBLAS_STATUS_SUCCESS;
    r = r && cublasDgemmStridedBatched(hb, CUBLAS_OP_N, CUBLAS_OP_N, m, m, m, &one, dB, m, (long long)n2, dS, m, 0,
                                       &zero, dA, m, (long long)n2, m) == CUBLAS_STATUS_SUCCESS;
    r = r && cublasDgemm(hb, CUBLAS_OP_N, CUBLAS_OP_N, (int)n2, m, m, &one, dA, (int)n2, dS, m, &zero, dB, (int)n2) ==
             CUBLAS_STATUS_SUCCESS;
    return r && cudaMemcpy(a.data(), dB, n3 * sizeof(double), cudaMemcpyDeviceToHost) == cudaSuccess;
  };
  if (ok) ok = cudaMemcpy(dS, S.data(), n2 * sizeof(double), cudaMemcpyHostToDevice) == cudaSuccess;
  std::vector<double> keep;
  if (ok) keep = a;
  if (ok) ok = passes();
  if (ok) divide();
  if (ok) ok = passes();
  if (!ok && !keep.empty()) a.swap(keep);  // the host path starts again from the input
  if (hb) cublasDestroy(hb);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dS);
  if (!ok) cudaGetLastError();
  return ok;
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
  auto divide = [&] {
    for (long i = 0; i < mt; ++i) {
      double l[3];
      l[0] = lam[i % m];
      l[1] = lam[(i / m) % m];
      l[2] = dim == 3 ? lam[i / ((long)m * m)] : 0.0;
      b[i] /= op_symbol(l, dim, order);
    }
  };
  if (!(dim == 3 && m >= 96 && dst3_gpu(b, m, S, divide))) {
    for (int a = 0; a < dim; ++a) dst1_lines(b, m, dim, a, S);
    divide();
    for (int a = 0; a < dim; ++a) dst1_lines(b, m, dim, a, S);
  }
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
