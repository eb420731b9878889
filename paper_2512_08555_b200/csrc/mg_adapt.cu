// mg_adapt.cu — detail coefficients of leaf blocks for grid adaptation (
// PAPER.md §2.1 P:65 "a so-called detail coefficient γ"; reading A1).
//
// γ of a block = max over its nodes of |u - P u|, P u the order-W polynomial
// interpolation of the block's all-even nodes (every-other-node coarse samples):
// along an axis an odd local index j takes the W-point Lagrange interpolant of the
// even positions j-(W-1), …, j+(W-1), shifted by steps of 2 to stay inside the block
// (one-sided near its last node); tensor product applied x, then y, then z.
//
// One CTA per leaf block: every thread loads its 16 (B = 16) nodes into registers at
// once, the even-(y, z) rows go to shared memory, the separable passes run from there
// (x on those rows, y on even z planes), the z pass compares with the register values,
// and the max |u - Pu| is a warp-shuffle reduction; 32 KB of shared memory per CTA.
// HBM traffic: 8 B per node read once (the kernel's roofline).
#include <cuda_runtime.h>

#include <cstdint>

#include "mg.h"
#include "mg_internal.h"

namespace mg {

namespace {

constexpr int DT_NT = 256;

template <int B, int W>
__global__ void __launch_bounds__(DT_NT) k_detail(const double* __restrict__ field, double* __restrict__ gamma) {
  constexpr int B3 = B * B * B, H = B / 2;
  extern __shared__ __align__(16) double sm[];
  double* A = sm;                 // [H][H][B]  the block's even-(z, y) rows
  double* P1 = A + H * H * B;     // [H][H][B]  x-pass on even (z, y)
  double* P2 = P1 + H * H * B;    // [H][B][B]  y-pass on even z
  __shared__ int s_lo[B];
  __shared__ double s_w[B][W];
  const int tid = threadIdx.x;
  const double* src = field + (size_t)blockIdx.x * B3;
  // the whole block into registers at once (one memory latency, coalesced); the
  // even-(z, y) rows also go to shared memory for the x pass
  constexpr int PER = B3 / DT_NT;
  double uv[PER];
#pragma unroll
  for (int k = 0; k < PER; ++k) uv[k] = __ldg(src + tid + k * DT_NT);
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int i = tid + k * DT_NT;
    const int x = i % B, y = (i / B) % B, z = i / (B * B);
    if (((y | z) & 1) == 0) A[((z >> 1) * H + (y >> 1)) * B + x] = uv[k];
  }
  // 1D rules: even j -> itself; odd j -> W taps from lo(j), Lagrange weights
  if (tid < B) {
    const int j = tid;
    if ((j & 1) == 0) {
      s_lo[j] = j;
    } else {
      int lo = j - (W - 1);
      lo = lo < 0 ? 0 : lo;
      lo = lo > B - 2 - 2 * (W - 1) ? B - 2 - 2 * (W - 1) : lo;
      s_lo[j] = lo;
#pragma unroll
      for (int t = 0; t < W; ++t) {
        double num = 1.0, den = 1.0;
#pragma unroll
        for (int s = 0; s < W; ++s) {
          if (s == t) continue;
          num *= (double)(j - (lo + 2 * s));
          den *= (double)((lo + 2 * t) - (lo + 2 * s));
        }
        s_w[j][t] = num / den;
      }
    }
  }
  __syncthreads();
  // the 1D rule at position j over values v(e) with stride `st` from base pointer p
  auto rule = [&](int j, const double* p, int st) {
    if ((j & 1) == 0) return 0.0 + 1.0 * p[j * st];
    const int lo = s_lo[j];
    double s = 0.0;
#pragma unroll
    for (int t = 0; t < W; ++t) s += s_w[j][t] * p[(lo + 2 * t) * st];
    return s;
  };
  // pass x: P1[z/2][y/2][x] on even z, y
  for (int i = tid; i < H * H * B; i += DT_NT) {
    const int x = i % B, yh = (i / B) % H, zh = i / (B * H);
    P1[i] = rule(x, A + (zh * H + yh) * B, 1);
  }
  __syncthreads();
  // pass y: P2[z/2][y][x] on even z, from the even-y rows of P1
  for (int i = tid; i < H * B * B; i += DT_NT) {
    const int x = i % B, y = (i / B) % B, zh = i / (B * B);
    // P1 rows are stored for y/2: position e (even) -> row e/2
    const double* col = P1 + (zh * H) * B + x;  // element (y'=e) at col[(e/2) * B]
    double v;
    if ((y & 1) == 0) {
      v = 0.0 + 1.0 * col[(y >> 1) * B];
    } else {
      const int lo = s_lo[y];
      double s = 0.0;
#pragma unroll
      for (int t = 0; t < W; ++t) s += s_w[y][t] * col[((lo >> 1) + t) * B];
      v = s;
    }
    P2[i] = v;
  }
  __syncthreads();
  // pass z and the detail
  double m = 0.0;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int i = tid + k * DT_NT;
    const int x = i % B, y = (i / B) % B, z = i / (B * B);
    const double* col = P2 + y * B + x;  // plane z' = e at col[(e/2) * B * B]
    double p;
    if ((z & 1) == 0) {
      p = 0.0 + 1.0 * col[(z >> 1) * B * B];
    } else {
      const int lo = s_lo[z];
      double s = 0.0;
#pragma unroll
      for (int t = 0; t < W; ++t) s += s_w[z][t] * col[((lo >> 1) + t) * B * B];
      p = s;
    }
    const double d = fabs(uv[k] - p);
    m = d > m ? d : m;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double t = __shfl_xor_sync(0xffffffffu, m, o);
    m = t > m ? t : m;
  }
  __shared__ double red[DT_NT / 32];
  if ((tid & 31) == 0) red[tid >> 5] = m;
  __syncthreads();
  if (tid == 0) {
    double r = 0.0;
    for (int w = 0; w < DT_NT / 32; ++w) r = red[w] > r ? red[w] : r;
    gamma[blockIdx.x] = r;
  }
}

template <int B, int W>
size_t detail_smem() {
  return sizeof(double) * (size_t)(2 * (B / 2) * (B / 2) * B + (B / 2) * B * B);
}

template <int B, int W>
void launch_detail_bw(const double* f, int n, double* g, cudaStream_t s) {
  static bool ready = false;
  if (!ready) {
    cudaFuncSetAttribute(k_detail<B, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)detail_smem<B, W>());
    ready = true;
  }
  k_detail<B, W><<<n, DT_NT, detail_smem<B, W>(), s>>>(f, g);
  note_launch();
}

}  // namespace

}  // namespace mg

extern "C" int mg_detail(const double* field_dev, int32_t n_leaf, int32_t B, int32_t W, double* gamma_dev,
                         void* stream) {
  using namespace mg;
  if (n_leaf < 0 || (n_leaf > 0 && (!field_dev || !gamma_dev))) return MG_ERR_ARG;
  if (!(B == 8 || B == 16) || !(W == 2 || W == 4 || W == 6)) return MG_ERR_ARG;
  if (2 * (W - 1) > B - 2) return MG_ERR_ARG;  // the W even taps must fit in the block (B = 8: W <= 4)
  if (n_leaf == 0) return MG_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (B == 16) {
    if (W == 2) launch_detail_bw<16, 2>(field_dev, n_leaf, gamma_dev, s);
    else if (W == 4) launch_detail_bw<16, 4>(field_dev, n_leaf, gamma_dev, s);
    else launch_detail_bw<16, 6>(field_dev, n_leaf, gamma_dev, s);
  } else {
    if (W == 2) launch_detail_bw<8, 2>(field_dev, n_leaf, gamma_dev, s);
    else launch_detail_bw<8, 4>(field_dev, n_leaf, gamma_dev, s);
  }
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? MG_OK : MG_ERR_CUDA;
}
