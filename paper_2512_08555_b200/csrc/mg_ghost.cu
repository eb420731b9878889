// mg_ghost.cu — coarse-to-fine boundary-ghost interpolation (a1-iii).
//
// Every boundary-ghost node J of a fine level (resolution jump, or beyond an
// unbounded face under reading U1) takes the tensor product over axes of the 1D
// rule (reading Z7): J_d even -> coarse J_d/2; J_d odd -> I-point centred Lagrange
// midpoint weights on coarse (J_d-1)/2 - I/2 + 1 … (J_d-1)/2 + I/2, I = M + 2.
//
// The per-node form costs I^3 = 216 scattered coarse reads for an odd-odd-odd node.
// Here one CTA handles one ghost box (the bounding box of the needed nodes of one
// ghost block): it stages the coarse support of the box in shared memory once and
// applies the rule separably, x then y then z — the same nesting and summation
// order as the per-node definition (Σ_z w_z Σ_y w_y Σ_x w_x W), so results are
// identical to it, with ~3I multiply-adds per node.
#include <cuda_runtime.h>

#include <cstdint>

#include "mg_internal.h"

namespace mg {

namespace {

constexpr int GB_NT = 256;
// coarse extent per axis of a 16-wide box: 7 + I (13 for I = 6, 15 for I = 8)
template <int I> struct GB {
  static constexpr int MAXC = 7 + I;
  static constexpr int SZ_A = 16 * 16 * MAXC;        // >= MAXC^3 (coarse box) and 16*16*MAXC (pass-y output)
  static constexpr int SZ_B = 16 * MAXC * MAXC;      // pass-x output
};

__device__ __forceinline__ int fdiv2(int a) { return a >> 1; }  // floor(a / 2) (arithmetic shift)

template <int I>
__device__ __forceinline__ void taps(int J, int c0, int& first, int& n, double* w) {
  // 1D rule at fine index J; first = coarse start relative to the box origin c0
  if ((J & 1) == 0) {
    n = 1;
    first = fdiv2(J) - c0;
    w[0] = 1.0;
  } else {
    n = I;
    first = fdiv2(J - 1) - I / 2 + 1 - c0;
    if (I == 4) {
      w[0] = -1.0 / 16; w[1] = 9.0 / 16; w[2] = 9.0 / 16; w[3] = -1.0 / 16;
    } else if (I == 8) {
      w[0] = -5.0 / 2048; w[1] = 49.0 / 2048; w[2] = -245.0 / 2048; w[3] = 1225.0 / 2048;
      w[4] = 1225.0 / 2048; w[5] = -245.0 / 2048; w[6] = 49.0 / 2048; w[7] = -5.0 / 2048;
    } else {
      w[0] = 3.0 / 256; w[1] = -25.0 / 256; w[2] = 150.0 / 256;
      w[3] = 150.0 / 256; w[4] = -25.0 / 256; w[5] = 3.0 / 256;
    }
  }
}

}  // namespace

// box record (12 int32): dst block, lo[3], hi[3] (fine block-local, hi exclusive),
// org[3] = level-global fine index of the block's node (0,0,0), 2 unused.
// Every stage iterates a 3-D index box with the 256 threads laid out as a 16 x 16 tile
// over its two largest axes and a loop over the smallest one (ghost boxes are thin
// slabs: 2 x 16 x 16 faces, 2 x 2 x 16 edges), so that the index arithmetic is adds
// and every thread has work.
template <typename Fn>
__device__ __forceinline__ void box_for(const int D[3], Fn&& fn) {
  int L = 2;  // loop axis: the smallest extent
  if (D[0] < D[L]) L = 0;
  if (D[1] < D[L]) L = 1;
  const int A = L == 0 ? 1 : 0, Bx = L == 2 ? 1 : 2;
  const int ta = threadIdx.x & 15, tb = threadIdx.x >> 4;
  if (ta >= D[A] || tb >= D[Bx]) return;
  int k[3];
  k[A] = ta;
  k[Bx] = tb;
  for (int l = 0; l < D[L]; ++l) {
    k[L] = l;
    fn(k[0], k[1], k[2]);
  }
}

template <int I>
__global__ void __launch_bounds__(GB_NT) k_c2f_box(const int32_t* __restrict__ boxes, LevelView F, LevelView C,
                                                   double* __restrict__ ff, const double* __restrict__ cf,
                                                   bool ext_zero) {
  extern __shared__ double sm[];
  const int32_t* bx = boxes + 12 * blockIdx.x;
  const int blk = bx[0];
  const int lo[3] = {bx[1], bx[2], bx[3]}, hi[3] = {bx[4], bx[5], bx[6]};
  const int B = F.B;
  int g0[3], nf[3], c0[3], nc[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    g0[a] = bx[7 + a] + lo[a];         // first fine global index of the box
    nf[a] = hi[a] - lo[a];
    c0[a] = fdiv2(g0[a]) - I / 2 + 1;  // first coarse tap of the box (odd or even first node)
    nc[a] = fdiv2(g0[a] + nf[a] - 1) + I / 2 - c0[a] + 1;
  }
  double* Cs = sm;                   // [nc2][nc1][nc0]
  double* T1 = sm + GB<I>::SZ_A;     // [nc2][nc1][nf0]
  double* T2 = Cs;                   // [nc2][nf1][nf0] (reuses Cs after pass x)
  // coarse block / local index along one axis (periodic wrap); -1 outside the block map
  // (no runtime-extent divisions: B is a power of two, periodic wraps are conditional adds)
  const int bsh = __ffs(C.B) - 1, bmask = C.B - 1;
  auto cidx = [&](int a, int ci, int& b, int& l) {
    if (C.per[a]) {
      while (ci < 0) ci += C.N[a];
      while (ci >= C.N[a]) ci -= C.N[a];
    }
    l = ci & bmask;
    b = (ci >> bsh) - C.bmap_lo[a];  // arithmetic shift: floor(ci / B)
    if (b < 0 || b >= C.bmap_n[a]) b = -1;
  };
  // ---- stage the coarse support (nodes outside the coarse level -> 0, only reached
  // by non-needed nodes of the box)
  box_for(nc, [&](int qx, int qy, int qz) {
    int b[3], l[3];
    cidx(0, c0[0] + qx, b[0], l[0]);
    cidx(1, c0[1] + qy, b[1], l[1]);
    cidx(2, c0[2] + qz, b[2], l[2]);
    double v = 0.0;
    if (b[0] >= 0 && b[1] >= 0 && b[2] >= 0) {
      const int cblk = __ldg(C.bmap + ((size_t)b[2] * C.bmap_n[1] + b[1]) * C.bmap_n[0] + b[0]);
      if (cblk >= 0) v = cf[(size_t)cblk * C.B3 + (l[2] * C.B + l[1]) * C.B + l[0]];
    }
    Cs[(qz * nc[1] + qy) * nc[0] + qx] = v;
  });
  __syncthreads();
  // ---- pass x: T1[cz][cy][fx]
  {
    const int D[3] = {nf[0], nc[1], nc[2]};
    box_for(D, [&](int fx, int cy, int cz) {
      double w[I];
      int first, n;
      taps<I>(g0[0] + fx, c0[0], first, n, w);
      const double* row = Cs + (cz * nc[1] + cy) * nc[0] + first;
      double sx = 0.0;
      for (int t = 0; t < n; ++t) sx += w[t] * row[t];
      T1[(cz * nc[1] + cy) * nf[0] + fx] = sx;
    });
  }
  __syncthreads();
  // ---- pass y: T2[cz][fy][fx]
  {
    const int D[3] = {nf[0], nf[1], nc[2]};
    box_for(D, [&](int fx, int fy, int cz) {
      double w[I];
      int first, n;
      taps<I>(g0[1] + fy, c0[1], first, n, w);
      const double* col = T1 + (cz * nc[1] + first) * nf[0] + fx;
      double sy = 0.0;
      for (int t = 0; t < n; ++t) sy += w[t] * col[t * nf[0]];
      T2[(cz * nf[1] + fy) * nf[0] + fx] = sy;
    });
  }
  __syncthreads();
  // ---- pass z -> ghost block
  double* dst = ff + (size_t)blk * F.B3;
  box_for(nf, [&](int fx, int fy, int fz) {
    const int J[3] = {g0[0] + fx, g0[1] + fy, g0[2] + fz};
    bool ext = false;
#pragma unroll
    for (int a = 0; a < 3; ++a) ext = ext || (!F.per[a] && (J[a] < 0 || J[a] >= F.N[a]));
    double v;
    if (ext_zero && ext) {
      v = 0.0;
    } else {
      double w[I];
      int first, n;
      taps<I>(J[2], c0[2], first, n, w);
      const double* col = T2 + (first * nf[1] + fy) * nf[0] + fx;
      double sz = 0.0;
      for (int t = 0; t < n; ++t) sz += w[t] * col[t * nf[0] * nf[1]];
      v = sz;
    }
    dst[((lo[2] + fz) * B + (lo[1] + fy)) * B + (lo[0] + fx)] = v;
  });
}

template <int I>
size_t c2f_box_smem() { return sizeof(double) * (size_t)(GB<I>::SZ_A + GB<I>::SZ_B); }

void prepare_ghost_kernels() {
  cudaFuncSetAttribute(k_c2f_box<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c2f_box_smem<4>());
  cudaFuncSetAttribute(k_c2f_box<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c2f_box_smem<6>());
  cudaFuncSetAttribute(k_c2f_box<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c2f_box_smem<8>());
}

void launch_c2f_box(const LevelView& fine, const LevelView& coarse, const int32_t* boxes, int nbox,
                    double* fine_field, const double* coarse_field, int I, bool ext_zero, cudaStream_t s) {
  if (nbox <= 0) return;
  if (I == 4)
    k_c2f_box<4><<<nbox, GB_NT, c2f_box_smem<4>(), s>>>(boxes, fine, coarse, fine_field, coarse_field, ext_zero);
  else if (I == 6)
    k_c2f_box<6><<<nbox, GB_NT, c2f_box_smem<6>(), s>>>(boxes, fine, coarse, fine_field, coarse_field, ext_zero);
  else
    k_c2f_box<8><<<nbox, GB_NT, c2f_box_smem<8>(), s>>>(boxes, fine, coarse, fine_field, coarse_field, ext_zero);
  note_launch();
}

}  // namespace mg
