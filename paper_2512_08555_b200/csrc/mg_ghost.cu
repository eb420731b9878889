// mg_ghost.cu — coarse-to-fine boundary-ghost interpolation (a1-iii).
//
// Every boundary-ghost node J of a fine level (resolution jump, or beyond an
// unbounded face under reading U1) takes the tensor product over axes of the 1D
// rule (reading Z7): J_d even -> coarse J_d/2; J_d odd -> I-point centred Lagrange
// midpoint weights on coarse (J_d-1)/2 - I/2 + 1 … (J_d-1)/2 + I/2, I = M + 2.
//
// The per-node form costs I^3 = 216 scattered coarse reads for an odd-odd-odd node.
// The host splits every ghost block's needed nodes into disjoint boxes, and two kernels
// apply the rule separably:
//   k_c2f_box:  one CTA per box; stages the box's coarse support in shared memory once
//               and applies the rule x, then y, then z — the per-node definition's
//               nesting and summation order (Σ_z w_z Σ_y w_y Σ_x w_x W), ~3I
//               multiply-adds per node;
//   k_c2f_thin: one warp per box <= 2 nodes thick along some axis (the 1-thick face,
//               edge and corner layers of the distance-1 halo), thin axis first, no
//               staging and no CTA barriers (used on levels with many such boxes).
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

template <int I>
__global__ void __launch_bounds__(GB_NT) k_c2f_box(const int32_t* __restrict__ boxes, LevelView F, LevelView C,
                                                   double* __restrict__ ff, const double* __restrict__ cf,
                                                   bool ext_zero, int t1_off) {
  extern __shared__ double sm[];
  ff += (int64_t)blockIdx.y * F.cs;  // component blockIdx.y
  cf += (int64_t)blockIdx.y * C.cs;
  const int32_t* bx = boxes + GBOX_REC * blockIdx.x;
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
  double* T1 = sm + t1_off;           // [nc2][nc1][nf0]
  double* T2 = Cs;                   // [nc2][nf1][nf0] (reuses Cs after pass x)
  // ---- stage the coarse support (nodes outside the coarse level -> 0, only reached
  // by non-needed nodes of the box).  A box's coarse support spans <= 15 taps per axis,
  // i.e. at most 2 coarse blocks per axis (3 when the coarse level has B/2 blocks); the
  // record carries the coarse block index of every slot combination; each element
  // computes its block-local index and slot inline (no extra barrier)
  const int CB = C.B, bsh = __ffs(C.B) - 1, bmask = C.B - 1;
  int cw0[3], nblk[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    int cf0 = c0[a];
    if (C.per[a]) {
      while (cf0 < 0) cf0 += C.N[a];
      while (cf0 >= C.N[a]) cf0 -= C.N[a];
    }
    cw0[a] = cf0 >> bsh;
    nblk[a] = C.N[a] >> bsh;
  }
  auto axis = [&](int a, int q, int& l, int& slot) {
    int ci = c0[a] + q;
    if (C.per[a]) {
      if (ci < 0) ci += C.N[a];
      if (ci >= C.N[a]) ci -= C.N[a];
    }
    l = ci & bmask;
    slot = (ci >> bsh) - cw0[a];
    if (slot < 0) slot += nblk[a];
  };
  box_for(nc, [&](int qx, int qy, int qz) {
    int l0, l1, l2, s0, s1, s2;
    axis(0, qx, l0, s0);
    axis(1, qy, l1, s1);
    axis(2, qz, l2, s2);
    const int cblk = __ldg(bx + 12 + s0 + 3 * s1 + 9 * s2);
    double v = 0.0;
    if (cblk >= 0) v = cf[(size_t)cblk * C.B3 + (l2 * CB + l1) * CB + l0];
    Cs[(qz * nc[1] + qy) * nc[0] + qx] = v;
  });
  __syncthreads();
  // ---- pass x: T1[cz][cy][fx]
  {
    const int D[3] = {nf[0], nc[1], nc[2]};
    box_for(D, [&](int fx, int cy, int cz) {
      int first;
      const bool odd = taps<I>(g0[0] + fx, c0[0], first);
      T1[(cz * nc[1] + cy) * nf[0] + fx] = apply_taps<I>(Cs + (cz * nc[1] + cy) * nc[0] + first, 1, odd);
    });
  }
  __syncthreads();
  // ---- pass y: T2[cz][fy][fx]
  {
    const int D[3] = {nf[0], nf[1], nc[2]};
    box_for(D, [&](int fx, int fy, int cz) {
      int first;
      const bool odd = taps<I>(g0[1] + fy, c0[1], first);
      T2[(cz * nf[1] + fy) * nf[0] + fx] = apply_taps<I>(T1 + (cz * nc[1] + first) * nf[0] + fx, nf[0], odd);
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
      int first;
      const bool odd = taps<I>(J[2], c0[2], first);
      v = apply_taps<I>(T2 + (first * nf[1] + fy) * nf[0] + fx, nf[0] * nf[1], odd);
    }
    dst[((lo[2] + fz) * B + (lo[1] + fy)) * B + (lo[0] + fx)] = v;
  });
}

// ---------------------------------------------------------------------------------
// Thin boxes (some axis one or two nodes thick: the 1-thick face, edge and corner
// layers of the distance-1 ghost halo, the bulk of every adaptive level's boxes), one
// warp per box, no CTA barriers.  Per 1-thick layer J_a of the thin axis a (b < c the
// other two axes):
//   P[qc][qb] = rule_a(C)(J_a, qb, qc)      coarse plane, the I (odd J_a) or 1 tap(s)
//                                           along a read straight from the coarse level
//   T[fc][qb] = rule_c(P)(fc)               along c
//   u(J)      = rule_b(T)(fb)               along b
// i.e. the same tensor-product rule (reading Z7) with the thin axis first: a layer costs
// (7 + I)^2 + 16 (7 + I) + 256 rule evaluations instead of the x-first passes over the
// I-thick coarse support.  Coarse addresses come from per-axis (slot, offset) tables of
// the box's coarse taps and the record's 27 coarse block indices (zero outside the
// coarse level, only reached by unused plane entries).
// ---------------------------------------------------------------------------------
// warps (boxes) per CTA and CTAs per SM at 80 registers: one-warp CTAs fill the SMs most
// evenly (cfg5 refresh of level 3 / 4, us: 8 x 3: 45.4 / 86.7, 4 x 6: 42.5 / 82.3, 2 x 12:
// 39.4 / 80.2, 1 x 24: 35.6 / 76.5; 64 registers (8 x 4) spill: 48 / 100)
constexpr int GT_W = 1, GT_MINB = 24;

template <int I>
struct GT {
  static constexpr int NC = 7 + I;  // coarse taps per axis of a <= 16-node run
  static constexpr int PS = NC * NC, TS = 16 * NC;
};

template <int I>
__global__ void __launch_bounds__(GT_W * 32, GT_MINB) k_c2f_thin(const int32_t* __restrict__ boxes, int nbox, LevelView F,
                                                        LevelView C, double* __restrict__ ff,
                                                        const double* __restrict__ cf, bool ext_zero) {
  using S = GT<I>;
  __shared__ double sP[GT_W][S::PS];
  __shared__ double sT[GT_W][S::TS];
  __shared__ int srec[GT_W][GBOX_REC];
  __shared__ int sslot[GT_W][3][S::NC], soff[GT_W][3][S::NC];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x * GT_W + w;
  if (b >= nbox) return;  // warp-uniform; only warp-level synchronisation below
  ff += (int64_t)blockIdx.y * F.cs;
  cf += (int64_t)blockIdx.y * C.cs;
  int* rec = srec[w];
  for (int i = lane; i < GBOX_REC; i += 32) rec[i] = __ldg(boxes + (size_t)b * GBOX_REC + i);
  __syncwarp();
  const int CB = C.B, bsh = __ffs(C.B) - 1, bmask = C.B - 1;
  int lo[3], g0[3], nf[3], c0[3], nc[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    lo[a] = rec[1 + a];
    g0[a] = rec[7 + a] + lo[a];
    nf[a] = rec[4 + a] - lo[a];
    c0[a] = fdiv2(g0[a]) - I / 2 + 1;
    nc[a] = fdiv2(g0[a] + nf[a] - 1) + I / 2 - c0[a] + 1;
  }
  // per axis and coarse tap q: block slot (times 1, 3, 9) and offset inside the block
  for (int i = lane; i < 3 * S::NC; i += 32) {
    const int a = i / S::NC, q = i % S::NC;
    if (q >= nc[a]) continue;
    int cf0 = c0[a];
    if (C.per[a]) {
      while (cf0 < 0) cf0 += C.N[a];
      while (cf0 >= C.N[a]) cf0 -= C.N[a];
    }
    int ci = c0[a] + q;
    if (C.per[a]) {
      if (ci < 0) ci += C.N[a];
      if (ci >= C.N[a]) ci -= C.N[a];
    }
    int slot = (ci >> bsh) - (cf0 >> bsh);
    if (slot < 0) slot += C.N[a] >> bsh;
    sslot[w][a][q] = slot * (a == 0 ? 1 : a == 1 ? 3 : 9);
    soff[w][a][q] = (ci & bmask) * (a == 0 ? 1 : a == 1 ? CB : CB * CB);
  }
  __syncwarp();
  // thin axis a (the thinnest; ties: lowest), b < c the others; per-role scalars (no
  // runtime-indexed local arrays)
  const int a = (nf[0] <= nf[1] && nf[0] <= nf[2]) ? 0 : (nf[1] <= nf[2] ? 1 : 2);
  const int ab = a == 0 ? 1 : 0, ac = a == 2 ? 1 : 2;
  auto pick = [](const int v[3], int i) { return i == 0 ? v[0] : (i == 1 ? v[1] : v[2]); };
  const int FB = F.B;
  const int fstr[3] = {1, FB, FB * FB};
  const int per3[3] = {F.per[0], F.per[1], F.per[2]}, N3[3] = {F.N[0], F.N[1], F.N[2]};
  const int nfa = pick(nf, a), nfb = pick(nf, ab), nfc = pick(nf, ac);
  const int ncb = pick(nc, ab), ncc = pick(nc, ac);
  const int g0a = pick(g0, a), g0b = pick(g0, ab), g0c = pick(g0, ac);
  const int c0a = pick(c0, a), c0b = pick(c0, ab), c0c = pick(c0, ac);
  const int doff = pick(lo, a) * pick(fstr, a) + pick(lo, ab) * pick(fstr, ab) + pick(lo, ac) * pick(fstr, ac);
  const int sa = pick(fstr, a), sb = pick(fstr, ab), sc = pick(fstr, ac);
  const bool pera = pick(per3, a), perb = pick(per3, ab), perc = pick(per3, ac);
  const int Na = pick(N3, a), Nb = pick(N3, ab), Nc = pick(N3, ac);
  const int* slb = sslot[w][ab];
  const int* ofb = soff[w][ab];
  const int* slc = sslot[w][ac];
  const int* ofc = soff[w][ac];
  const int* sla = sslot[w][a];
  const int* ofa = soff[w][a];
  // e / n for the flattened loops below as a multiply-high: exact for e * n < 2^32 (n >= 2;
  // ncb >= I always, nfb = 1 for edge and corner boxes)
  const unsigned mb = 0xFFFFFFFFu / (unsigned)ncb + 1u, mfb = nfb > 1 ? 0xFFFFFFFFu / (unsigned)nfb + 1u : 0u;
  double* P = sP[w];
  double* T = sT[w];
  double* dst = ff + (size_t)rec[0] * F.B3 + doff;
  for (int la = 0; la < nfa; ++la) {
    int fa;
    const bool odda = taps<I>(g0a + la, c0a, fa);
    // P[qc][qb]: the rule along a, straight from the coarse level; K entries per lane at a
    // time with all their loads issued before the sums (memory-level parallelism)
    constexpr int K = I == 4 ? 4 : (I == 6 ? 3 : 2);
    const int npl = ncb * ncc;
    for (int e0 = lane; e0 < npl; e0 += K * 32) {
      double cv[K][I];
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int e = e0 + 32 * k;
        if (e >= npl) continue;
        const int qc = (int)__umulhi((unsigned)e, mb), qb = e - qc * ncb;
        const int s0 = 12 + slb[qb] + slc[qc];
        const double* src = cf + ofb[qb] + ofc[qc];
#pragma unroll
        for (int t = 0; t < I; ++t) {
          if (t > 0 && !odda) break;
          const int blk = rec[s0 + sla[fa + t]];
          cv[k][t] = blk >= 0 ? __ldg(src + (size_t)blk * C.B3 + ofa[fa + t]) : 0.0;
        }
      }
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int e = e0 + 32 * k;
        if (e >= npl) continue;
        double v = cv[k][0];
        if (odda) {
          v = 0.0;
#pragma unroll
          for (int t = 0; t < I; ++t) v += wt<I>(t) * cv[k][t];
        }
        P[e] = v;
      }
    }
    __syncwarp();
    // T[fc][qb]: the rule along c
    for (int e = lane; e < nfc * ncb; e += 32) {
      const int fc = (int)__umulhi((unsigned)e, mb), qb = e - fc * ncb;
      int first;
      const bool odd = taps<I>(g0c + fc, c0c, first);
      T[e] = apply_taps<I>(P + first * ncb + qb, ncb, odd);
    }
    __syncwarp();
    // the rule along b -> ghost node
    const int Ja = g0a + la;
    const bool exta = !pera && (Ja < 0 || Ja >= Na);
    for (int e = lane; e < nfc * nfb; e += 32) {
      const int fc = nfb > 1 ? (int)__umulhi((unsigned)e, mfb) : e, fb = e - fc * nfb;
      const int Jb = g0b + fb, Jc = g0c + fc;
      const bool ext = exta || (!perb && (Jb < 0 || Jb >= Nb)) || (!perc && (Jc < 0 || Jc >= Nc));
      double v;
      if (ext_zero && ext) {
        v = 0.0;
      } else {
        int first;
        const bool odd = taps<I>(Jb, c0b, first);
        v = apply_taps<I>(T + fc * ncb + first, 1, odd);
      }
      dst[la * sa + fb * sb + fc * sc] = v;
    }
    __syncwarp();
  }
}

template <int I>
size_t c2f_box_smem() { return sizeof(double) * (size_t)(GB<I>::SZ_A + GB<I>::SZ_B); }

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
  const size_t smem = sizeof(double) * (size_t)(szA + szB);
  if (I == 4)
    k_c2f_box<4><<<dim3(nbox, fine.nc), GB_NT, smem, s>>>(boxes, fine, coarse, fine_field, coarse_field, ext_zero, szA);
  else if (I == 6)
    k_c2f_box<6><<<dim3(nbox, fine.nc), GB_NT, smem, s>>>(boxes, fine, coarse, fine_field, coarse_field, ext_zero, szA);
  else
    k_c2f_box<8><<<dim3(nbox, fine.nc), GB_NT, smem, s>>>(boxes, fine, coarse, fine_field, coarse_field, ext_zero, szA);
  note_launch();
}


void launch_c2f_thin(const LevelView& fine, const LevelView& coarse, const int32_t* boxes, int nbox, double* fine_field,
                     const double* coarse_field, int I, bool ext_zero, cudaStream_t s) {
  if (nbox <= 0) return;
  const dim3 grid((nbox + GT_W - 1) / GT_W, fine.nc);
  if (I == 4) k_c2f_thin<4><<<grid, GT_W * 32, 0, s>>>(boxes, nbox, fine, coarse, fine_field, coarse_field, ext_zero);
  else if (I == 6) k_c2f_thin<6><<<grid, GT_W * 32, 0, s>>>(boxes, nbox, fine, coarse, fine_field, coarse_field, ext_zero);
  else k_c2f_thin<8><<<grid, GT_W * 32, 0, s>>>(boxes, nbox, fine, coarse, fine_field, coarse_field, ext_zero);
  note_launch();
}

}  // namespace mg
