// mg_ghost.cu — coarse-to-fine boundary-ghost interpolation (a1-iii).
//
// Every boundary-ghost node J of a fine level (resolution jump, or beyond an
// unbounded face under reading U1) takes the tensor product over axes of the 1D
// rule (reading Z7): J_d even -> coarse J_d/2; J_d odd -> I-point centred Lagrange
// midpoint weights on coarse (J_d-1)/2 - I/2 + 1 … (J_d-1)/2 + I/2, I = M + 2.
//
// The per-node form costs I^3 = 216 scattered coarse reads for an odd-odd-odd node.
// Here one CTA handles one ghost box (a box of needed nodes of one ghost block; the
// host splits every block's needed nodes into disjoint thin boxes): it stages the coarse support of the box in shared memory once and
// applies the rule separably, x then y then z — the same nesting and summation
// order as the per-node definition (Σ_z w_z Σ_y w_y Σ_x w_x W), so results are
// identical to it, with ~3I multiply-adds per node.
#include <cuda_runtime.h>

#include <cstdint>

#include "mg_internal.h"

namespace mg {

namespace {

#ifndef MG_GB_NT
#define MG_GB_NT 256
#endif
constexpr int GB_NT = MG_GB_NT;  // threads per ghost box (a 16-wide tile of GB_NT/16 rows)
// coarse extent per axis of a 16-wide box: 7 + I (13 for I = 6, 15 for I = 8)
template <int I> struct GB {
  static constexpr int MAXC = 7 + I;
  static constexpr int SZ_A = 16 * 16 * MAXC;        // >= MAXC^3 (coarse box) and 16*16*MAXC (pass-y output)
  static constexpr int SZ_B = 16 * MAXC * MAXC;      // pass-x output
};

__device__ __forceinline__ int fdiv2(int a) { return a >> 1; }  // floor(a / 2) (arithmetic shift)
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cpa_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

// 1D rule at fine index J: coarse start relative to the box origin c0; odd -> the
// I-point midpoint weights, even -> injection (weight 1)
template <int I>
__device__ __forceinline__ bool taps(int J, int c0, int& first) {
  const bool odd = J & 1;
  first = odd ? fdiv2(J - 1) - I / 2 + 1 - c0 : fdiv2(J) - c0;
  return odd;
}

template <int I>
__device__ __forceinline__ double wt(int t) {
  if (I == 4) {
    constexpr double w[4] = {-1.0 / 16, 9.0 / 16, 9.0 / 16, -1.0 / 16};
    return w[t];
  } else if (I == 8) {
    constexpr double w[8] = {-5.0 / 2048, 49.0 / 2048, -245.0 / 2048, 1225.0 / 2048,
                             1225.0 / 2048, -245.0 / 2048, 49.0 / 2048, -5.0 / 2048};
    return w[t];
  } else {
    constexpr double w[6] = {3.0 / 256, -25.0 / 256, 150.0 / 256, 150.0 / 256, -25.0 / 256, 3.0 / 256};
    return w[t];
  }
}

// Σ_t w_t p[t * stride] in tap order (the per-node definition's summation order);
// an even node is the single coarse value
template <int I>
__device__ __forceinline__ double apply_taps(const double* p, int stride, bool odd) {
  if (!odd) return p[0];
  double s = 0.0;
#pragma unroll
  for (int t = 0; t < I; ++t) s += wt<I>(t) * p[t * stride];
  return s;
}

}  // namespace

// box record: GBOX_REC int32 (mg_internal.h).
// Every stage iterates a 3-D index box with the GB_NT threads laid out as a 16-wide tile
// over its two largest axes and a loop over the smallest one (ghost boxes are thin
// slabs: 2 x 16 x 16 faces, 2 x 2 x 16 edges), so that the index arithmetic is adds
// and every thread has work.
template <typename Fn>
__device__ __forceinline__ void box_for(const int D[3], Fn&& fn) {
  constexpr int TB = GB_NT / 16;  // rows of the 16-wide thread tile
  const int ta = threadIdx.x & 15;
  if (D[0] <= D[1] && D[0] <= D[2]) {         // loop over x
    if (ta >= D[1]) return;
    for (int tb = threadIdx.x >> 4; tb < D[2]; tb += TB)
      for (int l = 0; l < D[0]; ++l) fn(l, ta, tb);
  } else if (D[1] <= D[2]) {                  // loop over y
    if (ta >= D[0]) return;
    for (int tb = threadIdx.x >> 4; tb < D[2]; tb += TB)
      for (int l = 0; l < D[1]; ++l) fn(ta, l, tb);
  } else {                                    // loop over z
    if (ta >= D[0]) return;
    for (int tb = threadIdx.x >> 4; tb < D[1]; tb += TB)
      for (int l = 0; l < D[2]; ++l) fn(ta, tb, l);
  }
}

// Box geometry decoded from a record (all threads, registers).
template <int I>
struct BoxGeo {
  int blk, lo[3], g0[3], nf[3], c0[3], nc[3], cw0[3];
  __device__ void decode(const int* r, const LevelView& C) {
    blk = r[0];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      lo[a] = r[1 + a];
      g0[a] = r[7 + a] + lo[a];          // first fine global index of the box
      nf[a] = r[4 + a] - lo[a];
      c0[a] = fdiv2(g0[a]) - I / 2 + 1;  // first coarse tap of the box (odd or even first node)
      nc[a] = fdiv2(g0[a] + nf[a] - 1) + I / 2 - c0[a] + 1;
      int cf0 = c0[a];
      if (C.per[a]) {
        while (cf0 < 0) cf0 += C.N[a];
        while (cf0 >= C.N[a]) cf0 -= C.N[a];
      }
      cw0[a] = cf0 >> (__ffs(C.B) - 1);
    }
  }
};

__device__ __forceinline__ void cpa8_zfill(void* smem, const void* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(valid ? 8 : 0));
}

// Pipelined over boxes: each CTA walks the boxes blockIdx.x, blockIdx.x + gridDim.x, …;
// the coarse support of the next box is staged by cp.async (zero-filled outside the
// coarse level) into the other half of a double buffer while the current box runs its
// three passes, so the gather latency (the limiter of one box per CTA: record and
// staging loads, then three barrier-separated passes) overlaps the arithmetic.
template <int I>
__global__ void __launch_bounds__(GB_NT) k_c2f_box(const int32_t* __restrict__ boxes, int nbox, LevelView F,
                                                   LevelView C, double* __restrict__ ff,
                                                   const double* __restrict__ cf, bool ext_zero, int szA) {
  extern __shared__ double sm[];
  __shared__ int rec[2][GBOX_REC];
  ff += (int64_t)blockIdx.y * F.cs;  // component blockIdx.y
  cf += (int64_t)blockIdx.y * C.cs;
  const int tid = threadIdx.x;
  const int B = F.B;
  const int CB = C.B, bsh = __ffs(C.B) - 1, bmask = C.B - 1;
  double* T1 = sm + 2 * szA;  // [nc2][nc1][nf0]
  // stage the coarse support of a box (nodes outside the coarse level -> 0, only reached
  // by non-needed nodes of the box).  A box's coarse support spans <= 15 taps per axis,
  // i.e. at most 2 coarse blocks per axis (3 when the coarse level has B/2 blocks); the
  // record carries the coarse block index of every slot combination
  auto stage = [&](const BoxGeo<I>& g, const int* r, double* Cs) {
    auto axis = [&](int a, int q, int& l, int& slot) {
      int ci = g.c0[a] + q;
      if (C.per[a]) {
        if (ci < 0) ci += C.N[a];
        if (ci >= C.N[a]) ci -= C.N[a];
      }
      l = ci & bmask;
      slot = (ci >> bsh) - g.cw0[a];
      if (slot < 0) slot += C.N[a] >> bsh;
    };
    box_for(g.nc, [&](int qx, int qy, int qz) {
      int l0, l1, l2, s0, s1, s2;
      axis(0, qx, l0, s0);
      axis(1, qy, l1, s1);
      axis(2, qz, l2, s2);
      const int cblk = r[12 + s0 + 3 * s1 + 9 * s2];
      cpa8_zfill(Cs + (qz * g.nc[1] + qy) * g.nc[0] + qx,
                 cf + (size_t)(cblk >= 0 ? cblk : 0) * C.B3 + (l2 * CB + l1) * CB + l0, cblk >= 0);
    });
  };
  int b = blockIdx.x;
  if (b >= nbox) return;
  if (tid < GBOX_REC) rec[0][tid] = __ldg(boxes + (size_t)b * GBOX_REC + tid);
  __syncthreads();
  BoxGeo<I> g;
  g.decode(rec[0], C);
  stage(g, rec[0], sm);
  cpa_commit();
  for (int it = 0;; ++it) {
    const int cur = it & 1, bn = b + gridDim.x;
    double* Cs = sm + cur * szA;  // [nc2][nc1][nc0] of box b; T2 [nc2][nf1][nf0] reuses it
    if (bn < nbox && tid < GBOX_REC) rec[cur ^ 1][tid] = __ldg(boxes + (size_t)bn * GBOX_REC + tid);
    __syncthreads();  // rec[cur ^ 1]; the previous box's passes are done with the other buffer
    BoxGeo<I> gn;
    if (bn < nbox) {
      gn.decode(rec[cur ^ 1], C);
      stage(gn, rec[cur ^ 1], sm + (cur ^ 1) * szA);
    }
    cpa_commit();
    cpa_wait1();      // box b's staging has landed (this thread's copies) …
    __syncthreads();  // … and everyone's
    // ---- pass x: T1[cz][cy][fx]
    {
      const int D[3] = {g.nf[0], g.nc[1], g.nc[2]};
      box_for(D, [&](int fx, int cy, int cz) {
        int first;
        const bool odd = taps<I>(g.g0[0] + fx, g.c0[0], first);
        T1[(cz * g.nc[1] + cy) * g.nf[0] + fx] = apply_taps<I>(Cs + (cz * g.nc[1] + cy) * g.nc[0] + first, 1, odd);
      });
    }
    __syncthreads();
    // ---- pass y: T2[cz][fy][fx]
    double* T2 = Cs;
    {
      const int D[3] = {g.nf[0], g.nf[1], g.nc[2]};
      box_for(D, [&](int fx, int fy, int cz) {
        int first;
        const bool odd = taps<I>(g.g0[1] + fy, g.c0[1], first);
        T2[(cz * g.nf[1] + fy) * g.nf[0] + fx] =
            apply_taps<I>(T1 + (cz * g.nc[1] + first) * g.nf[0] + fx, g.nf[0], odd);
      });
    }
    __syncthreads();
    // ---- pass z -> ghost block
    double* dst = ff + (size_t)g.blk * F.B3;
    box_for(g.nf, [&](int fx, int fy, int fz) {
      const int J[3] = {g.g0[0] + fx, g.g0[1] + fy, g.g0[2] + fz};
      bool ext = false;
#pragma unroll
      for (int a = 0; a < 3; ++a) ext = ext || (!F.per[a] && (J[a] < 0 || J[a] >= F.N[a]));
      double v;
      if (ext_zero && ext) {
        v = 0.0;
      } else {
        int first;
        const bool odd = taps<I>(J[2], g.c0[2], first);
        v = apply_taps<I>(T2 + (first * g.nf[1] + fy) * g.nf[0] + fx, g.nf[0] * g.nf[1], odd);
      }
      dst[((g.lo[2] + fz) * B + (g.lo[1] + fy)) * B + (g.lo[0] + fx)] = v;
    });
    if (bn >= nbox) break;
    b = bn;
    g = gn;
  }
}

template <int I>
size_t c2f_box_smem() { return sizeof(double) * (size_t)(2 * GB<I>::SZ_A + GB<I>::SZ_B); }

void prepare_ghost_kernels() {
  cudaFuncSetAttribute(k_c2f_box<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c2f_box_smem<4>());
  cudaFuncSetAttribute(k_c2f_box<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c2f_box_smem<6>());
  cudaFuncSetAttribute(k_c2f_box<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c2f_box_smem<8>());
}

size_t c2f_box_smem_max(int I) {
  return I == 4 ? c2f_box_smem<4>() : I == 6 ? c2f_box_smem<6>() : c2f_box_smem<8>();
}

void launch_c2f_box(const LevelView& fine, const LevelView& coarse, const int32_t* boxes, int nbox, int szA,
                    int szB, double* fine_field, const double* coarse_field, int I, bool ext_zero, cudaStream_t s) {
  if (nbox <= 0) return;
  const size_t smem = sizeof(double) * (size_t)(2 * szA + szB);
  // persistent grid: the resident CTAs of the device (occupancy at this shared-memory
  // size, queried once per size), each walking its share of the boxes
  static int dev_sms = 0;
  if (!dev_sms) {
    int d = 0;
    cudaGetDevice(&d);
    cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, d);
    if (dev_sms <= 0) dev_sms = 148;
  }
  int per_sm = 1;
  auto kern = I == 4 ? k_c2f_box<4> : I == 6 ? k_c2f_box<6> : k_c2f_box<8>;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, GB_NT, smem);
  if (per_sm < 1) per_sm = 1;
  const int grid = nbox < dev_sms * per_sm ? nbox : dev_sms * per_sm;
  kern<<<dim3(grid, fine.nc), GB_NT, smem, s>>>(boxes, nbox, fine, coarse, fine_field, coarse_field, ext_zero, szA);
  note_launch();
}

}  // namespace mg
