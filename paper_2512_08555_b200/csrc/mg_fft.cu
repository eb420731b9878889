// mg_fft.cu — fused transforms of the pruned coarse solve (x periodic, y and z unbounded:
// cfg4, cfg5; DESIGN.md §6 "pruned coarse solve"), the opt-in mg_desc.coarse_pruning = 2.
// Measured on B200 (cfg4's 128 x 270 x 270 level 0): 221 µs for the three kernels against
// ≈ 198 µs for the cuFFT passes they replace, although they move a quarter of the bytes —
// the shared-memory Stockham passes are latency bound (one barrier per pass, 24 warps per
// SM); kept as a tested variant, not the default.
//
// The padded convolution of P:367-398 (generalised E14, reading Z22) on the level-0
// lattice: after the R2C along x (cuFFT), every kx plane is a 2-D problem whose source
// occupies y < Ny, z < Nz of a Py x Pz padded lattice and whose output is read only on
// the window y, z in [-GE, N + GE).  Three kernels replace the eight passes of the cuFFT
// version (zero padding, y FFT, z FFT, multiplier, inverse z, two inverse y, window):
//   k_fft_y_fwd    y FFT of the zero-padded source lines (the padding is never stored);
//   k_fft_z_conv   z FFT of the Nz source rows, the multiplier, inverse z FFT, and only
//                  the Nz + 2 GE window rows written back (the other rows are never read);
//   k_fft_y_inv    inverse y FFT and the window, straight into the C2R input layout.
// Each CTA transforms TC columns in shared memory with a mixed-radix (2, 3, 4, 5, 7)
// Stockham FFT, unnormalised like cuFFT (forward e^{-2πi jk/n}, inverse e^{+...}; the
// 1 / (Px Py Pz) is in the multiplier).  Twiddles come from the host in long double.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <vector>

#include "mg_internal.h"

namespace mg {

namespace {

constexpr int FT_TC = 8;     // columns per CTA
constexpr int FT_NT = 256;   // threads per CTA
constexpr int FT_MAXN = 880; // longest transform: 2 x 8 columns x 881 x 16 B <= 227 KB of shared memory

__constant__ double2 c_root[8][8];  // c_root[r][j] = e^{-2πi j / r}, r in {2, 3, 4, 5, 7}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {  // a * conj(b)
  return make_double2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}

// radix-R DFT of x into y (forward roots e^{-2πi tu/R}; inverse the conjugates)
template <int R, bool INV>
__device__ __forceinline__ void dft_small(const double2 (&x)[R], double2 (&y)[R]) {
  if (R == 2) {
    y[0] = make_double2(x[0].x + x[1].x, x[0].y + x[1].y);
    y[1] = make_double2(x[0].x - x[1].x, x[0].y - x[1].y);
  } else if (R == 4) {
    const double2 s02 = make_double2(x[0].x + x[2].x, x[0].y + x[2].y);
    const double2 d02 = make_double2(x[0].x - x[2].x, x[0].y - x[2].y);
    const double2 s13 = make_double2(x[1].x + x[3].x, x[1].y + x[3].y);
    const double2 d13 = make_double2(x[1].x - x[3].x, x[1].y - x[3].y);
    // forward: y1 = d02 - i d13, y3 = d02 + i d13 (inverse: the conjugate roots)
    const double2 id13 = INV ? make_double2(-d13.y, d13.x) : make_double2(d13.y, -d13.x);
    y[0] = make_double2(s02.x + s13.x, s02.y + s13.y);
    y[2] = make_double2(s02.x - s13.x, s02.y - s13.y);
    y[1] = make_double2(d02.x + id13.x, d02.y + id13.y);
    y[3] = make_double2(d02.x - id13.x, d02.y - id13.y);
  } else {
#pragma unroll
    for (int u = 0; u < R; ++u) {
      double2 acc = x[0];
#pragma unroll
      for (int t = 1; t < R; ++t) {
        const double2 w = c_root[R][(t * u) % R];
        const double2 v = INV ? cmulc(x[t], w) : cmul(x[t], w);
        acc.x += v.x;
        acc.y += v.y;
      }
      y[u] = acc;
    }
  }
}

// one radix-R Stockham pass over ncol columns (pitch NP) of length n: a -> b
template <int R, bool INV>
__device__ __forceinline__ void fft_pass(const double2* __restrict__ a, double2* __restrict__ b, int ncol, int NP,
                                         int n, int p, const double2* __restrict__ tw) {
  const int m = n / R;
  for (int e = threadIdx.x; e < ncol * m; e += blockDim.x) {
    const int c = e / m, i = e - c * m, k = i % p;
    const double2* src = a + c * NP + i;
    double2 x[R];
#pragma unroll
    for (int t = 0; t < R; ++t) x[t] = src[t * m];
    if (p > 1) {
#pragma unroll
      for (int t = 1; t < R; ++t) {
        const double2 w = __ldg(tw + k * (R - 1) + t - 1);
        x[t] = INV ? cmulc(x[t], w) : cmul(x[t], w);
      }
    }
    double2 y[R];
    dft_small<R, INV>(x, y);
    double2* dst = b + c * NP + (i - k) * R + k;
#pragma unroll
    for (int u = 0; u < R; ++u) dst[u * p] = y[u];
  }
}

// the next radix of a compile-time plan (the host's order: 4s, then 2, 3, 5, 7)
__host__ __device__ constexpr int next_radix(int rem) {
  return rem % 4 == 0 ? 4 : rem % 2 == 0 ? 2 : rem % 3 == 0 ? 3 : rem % 5 == 0 ? 5 : 7;
}

// compile-time length N: one pass of radix R after the radices whose product is P (m, p
// and the index arithmetic are constants), then the rest
template <bool INV, int N, int P, int REM, int TOFF>
__device__ __forceinline__ double2* fft_ct(double2* a, double2* b, int ncol, int NP, const double2* __restrict__ tw) {
  if constexpr (REM == 1) {
    return a;
  } else {
    constexpr int R = next_radix(REM), M = N / R;
    for (int e = threadIdx.x; e < ncol * M; e += blockDim.x) {
      const int c = e / M, i = e - c * M, k = i % P;
      const double2* src = a + c * NP + i;
      double2 x[R];
#pragma unroll
      for (int t = 0; t < R; ++t) x[t] = src[t * M];
      if (P > 1) {
#pragma unroll
        for (int t = 1; t < R; ++t) {
          const double2 w = __ldg(tw + TOFF + k * (R - 1) + t - 1);
          x[t] = INV ? cmulc(x[t], w) : cmul(x[t], w);
        }
      }
      double2 y[R];
      dft_small<R, INV>(x, y);
      double2* dst = b + c * NP + (i - k) * R + k;
#pragma unroll
      for (int u = 0; u < R; ++u) dst[u * P] = y[u];
    }
    __syncthreads();
    return fft_ct<INV, N, P * R, REM / R, TOFF + P * (R - 1)>(b, a, ncol, NP, tw);
  }
}

// the whole transform of ncol columns; returns the buffer holding the result
template <bool INV>
__device__ double2* fft_cols(double2* a, double2* b, int ncol, int NP, const FFTPlan& P,
                             const double2* __restrict__ tw) {
  // the production length (cfg4 / cfg5: 2 x 128 + 2 GE - 1 -> 270) with a compile-time plan
  if (P.n == 270) return fft_ct<INV, 270, 1, 270, 0>(a, b, ncol, NP, tw);
  for (int f = 0; f < P.nf; ++f) {
    const double2* t = tw + P.toff[f];
    switch (P.r[f]) {
      case 2: fft_pass<2, INV>(a, b, ncol, NP, P.n, P.p[f], t); break;
      case 3: fft_pass<3, INV>(a, b, ncol, NP, P.n, P.p[f], t); break;
      case 4: fft_pass<4, INV>(a, b, ncol, NP, P.n, P.p[f], t); break;
      case 5: fft_pass<5, INV>(a, b, ncol, NP, P.n, P.p[f], t); break;
      default: fft_pass<7, INV>(a, b, ncol, NP, P.n, P.p[f], t); break;
    }
    __syncthreads();
    double2* s = a;
    a = b;
    b = s;
  }
  return a;
}

// y FFT of the zero-padded source: C1 [c][z][y < Ny][kx] -> C2 [c][z][kx][y < Py]
__global__ void __launch_bounds__(FT_NT) k_fft_y_fwd(const double2* __restrict__ c1, double2* __restrict__ c2, int Ny,
                                                     int Nz, int Hx, int Pz, FFTPlan py,
                                                     const double2* __restrict__ twy) {
  extern __shared__ double2 fsm[];
  const int Py = py.n, NP = Py + 1;
  const int z = blockIdx.x, kx0 = blockIdx.y * FT_TC, cc = blockIdx.z;
  c1 += ((int64_t)cc * Nz + z) * Ny * Hx;
  c2 += (int64_t)cc * Pz * Hx * Py;
  double2* a = fsm;
  double2* b = fsm + FT_TC * NP;
  for (int e = threadIdx.x; e < Py * FT_TC; e += blockDim.x) {
    const int y = e / FT_TC, c = e - y * FT_TC, kx = kx0 + c;
    a[c * NP + y] = (y < Ny && kx < Hx) ? c1[(int64_t)y * Hx + kx] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  const double2* res = fft_cols<false>(a, b, FT_TC, NP, py, twy);
  for (int e = threadIdx.x; e < FT_TC * Py; e += blockDim.x) {
    const int c = e / Py, y = e - c * Py, kx = kx0 + c;
    if (kx < Hx) c2[(((int64_t)z) * Hx + kx) * Py + y] = res[c * NP + y];
  }
}

// z FFT of the Nz source rows, multiplier, inverse z FFT, window rows only, in place on
// C2 [c][z < Pz][q = kx Py + y]
__global__ void __launch_bounds__(FT_NT) k_fft_z_conv(double2* __restrict__ c2, const double* __restrict__ mult, int Q,
                                                      int Nz, int GE, FFTPlan pz, const double2* __restrict__ twz) {
  extern __shared__ double2 fsm[];
  const int Pz = pz.n, NP = Pz + 1;
  const int q0 = blockIdx.x * FT_TC;
  c2 += (int64_t)blockIdx.y * Pz * Q;
  double2* a = fsm;
  double2* b = fsm + FT_TC * NP;
  for (int e = threadIdx.x; e < Pz * FT_TC; e += blockDim.x) {
    const int z = e / FT_TC, c = e - z * FT_TC, q = q0 + c;
    a[c * NP + z] = (z < Nz && q < Q) ? c2[(int64_t)z * Q + q] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  double2* s = fft_cols<false>(a, b, FT_TC, NP, pz, twz);
  for (int e = threadIdx.x; e < Pz * FT_TC; e += blockDim.x) {
    const int kz = e / FT_TC, c = e - kz * FT_TC, q = q0 + c;
    const double mlt = q < Q ? __ldg(mult + (int64_t)kz * Q + q) : 0.0;
    s[c * NP + kz].x *= mlt;
    s[c * NP + kz].y *= mlt;
  }
  __syncthreads();
  const double2* res = fft_cols<true>(s, s == a ? b : a, FT_TC, NP, pz, twz);
  const int nrow = Nz + 2 * GE;
  for (int e = threadIdx.x; e < nrow * FT_TC; e += blockDim.x) {
    const int r = e / FT_TC, c = e - r * FT_TC, q = q0 + c;
    const int z = r < Nz + GE ? r : Pz - nrow + r;
    if (q < Q) c2[(int64_t)z * Q + q] = res[c * NP + z];
  }
}

// inverse y FFT of the window planes and the window itself:
// C2 [c][z][kx][y] -> C3 [c][zw < Wz][yw < Wy][kx]
__global__ void __launch_bounds__(FT_NT) k_fft_y_inv(const double2* __restrict__ c2, double2* __restrict__ c3, int Hx,
                                                     int Pz, int Wy, int Wz, int GE, FFTPlan py,
                                                     const double2* __restrict__ twy) {
  extern __shared__ double2 fsm[];
  const int Py = py.n, NP = Py + 1;
  const int zw = blockIdx.x, kx0 = blockIdx.y * FT_TC, cc = blockIdx.z;
  const int z = (zw - GE + Pz) % Pz;
  c2 += (int64_t)cc * Pz * Hx * Py;
  c3 += (int64_t)cc * Wz * Wy * Hx;
  double2* a = fsm;
  double2* b = fsm + FT_TC * NP;
  for (int e = threadIdx.x; e < FT_TC * Py; e += blockDim.x) {
    const int c = e / Py, y = e - c * Py, kx = kx0 + c;
    a[c * NP + y] = kx < Hx ? c2[((int64_t)z * Hx + kx) * Py + y] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  const double2* res = fft_cols<true>(a, b, FT_TC, NP, py, twy);
  for (int e = threadIdx.x; e < Wy * FT_TC; e += blockDim.x) {
    const int yw = e / FT_TC, c = e - yw * FT_TC, kx = kx0 + c;
    const int y = (yw - GE + Py) % Py;
    if (kx < Hx) c3[((int64_t)zw * Wy + yw) * Hx + kx] = res[c * NP + y];
  }
}

size_t ft_smem(int n) { return sizeof(double2) * 2 * (size_t)FT_TC * (n + 1); }

}  // namespace

// radix plan of a 7-smooth length (4s first, then 2, 3, 5, 7) and its twiddles
// tw[toff[f] + k (r-1) + t-1] = e^{-2πi t k / (p r)}, k < p (long double on the host)
bool fft_plan(int n, FFTPlan& P, std::vector<double>& tw) {
  P = FFTPlan{};
  P.n = n;
  int m = n;
  std::vector<int> rs;
  while (m % 4 == 0) { rs.push_back(4); m /= 4; }
  for (int r : {2, 3, 5, 7})
    while (m % r == 0) { rs.push_back(r); m /= r; }
  if (m != 1 || (int)rs.size() > FFTPlan::MAXF) return false;
  P.nf = (int)rs.size();
  tw.clear();
  int p = 1;
  for (int f = 0; f < P.nf; ++f) {
    const int r = rs[f];
    P.r[f] = r;
    P.p[f] = p;
    P.toff[f] = (int)(tw.size() / 2);
    for (int k = 0; k < p; ++k)
      for (int t = 1; t < r; ++t) {
        const long double ang = -2.0L * 3.14159265358979323846264338327950288L * (long double)(t * k) /
                                (long double)(p * r);
        tw.push_back((double)std::cos(ang));
        tw.push_back((double)std::sin(ang));
      }
    p *= r;
  }
  if (tw.empty()) tw.assign(2, 0.0);
  return true;
}

void prepare_fft_kernels() {
  double2 roots[8][8] = {};
  for (int r = 2; r <= 7; ++r)
    for (int j = 0; j < r; ++j) {
      const long double ang = -2.0L * 3.14159265358979323846264338327950288L * j / r;
      roots[r][j] = make_double2((double)std::cos(ang), (double)std::sin(ang));
    }
  cudaMemcpyToSymbol(c_root, roots, sizeof(roots));
  const int mx = (int)ft_smem(FT_MAXN);
  cudaFuncSetAttribute(k_fft_y_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_fft_z_conv, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
  cudaFuncSetAttribute(k_fft_y_inv, cudaFuncAttributeMaxDynamicSharedMemorySize, mx);
}

void launch_fft_y_fwd(const void* c1, void* c2, int Ny, int Nz, int Hx, int Pz, const FFTPlan& py, const double* twy,
                      int nc, cudaStream_t s) {
  const dim3 grid(Nz, (Hx + FT_TC - 1) / FT_TC, nc);
  k_fft_y_fwd<<<grid, FT_NT, ft_smem(py.n), s>>>((const double2*)c1, (double2*)c2, Ny, Nz, Hx, Pz, py,
                                                  (const double2*)twy);
  note_launch();
}

void launch_fft_z_conv(void* c2, const double* mult, int Q, int Nz, int GE, const FFTPlan& pz, const double* twz,
                       int nc, cudaStream_t s) {
  const dim3 grid((Q + FT_TC - 1) / FT_TC, nc);
  k_fft_z_conv<<<grid, FT_NT, ft_smem(pz.n), s>>>((double2*)c2, mult, Q, Nz, GE, pz, (const double2*)twz);
  note_launch();
}

void launch_fft_y_inv(const void* c2, void* c3, int Hx, int Pz, int Wy, int Wz, int GE, const FFTPlan& py,
                      const double* twy, int nc, cudaStream_t s) {
  const dim3 grid(Wz, (Hx + FT_TC - 1) / FT_TC, nc);
  k_fft_y_inv<<<grid, FT_NT, ft_smem(py.n), s>>>((const double2*)c2, (double2*)c3, Hx, Pz, Wy, Wz, GE, py,
                                                  (const double2*)twy);
  note_launch();
}

}  // namespace mg
