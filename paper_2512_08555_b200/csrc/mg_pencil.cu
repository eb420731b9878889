// mg_pencil.cu — z-marching stencil kernels for B = 16 levels (the hot path).
//
// Why: a 3-D halo tile per 16^3 block evaluated from shared memory costs 19
// shared-memory reads per node and pass; on B200 that makes the red-black sweep
// L1/shared-memory bound at ~1.7 TB/s (profiles/r01_s2_baseline_ncu.md).  These
// kernels instead walk a *pencil* (a run of consecutive real blocks along z) one
// z-plane at a time with one thread per (x,y) column:
//   * each thread keeps its column's centre values and in-plane face sums S4 of
//     the last planes in registers, so a 19-point Mehrstellen node (E12)
//     reads only its 4 in-plane face and 4 in-plane diagonal neighbours from
//     shared memory (the z-neighbours and the z±1 edge sums come from registers);
//   * only xy planes (with an x/y halo) are staged in shared memory, through a
//     cp.async ring that keeps D planes in flight ahead of the compute;
//   * the red and black half-sweeps of one RB sweep (reading Z10: colour = parity
//     of the level-global index, red = even first, each colour from a snapshot)
//     come out of one pass: red at plane s-1 and black at plane s-2 while plane s
//     arrives, so u and f are read from HBM once per sweep (24 B / unknown).
// Boundary-ghost nodes (ghost blocks: c2f at resolution jumps, exterior band) are
// frozen during a sweep (reading Z9): halo nodes in non-real blocks keep their value.
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <type_traits>

#include "mg_internal.h"

namespace mg {

namespace {

constexpr int PB = 16;             // block edge
constexpr int PB3 = PB * PB * PB;
constexpr int PMAXL = 16;          // longest pencil (blocks)
constexpr int D6 = 2;              // M = 6 sweep: planes staged ahead
constexpr int RB6_NREG = 96;       // M = 6 sweep register cap

__device__ __forceinline__ int reg16(int x) { return x < 0 ? -1 : (x >= PB ? 1 : 0); }

__device__ __forceinline__ void cpa16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ---- TMA (cp.async.bulk.tensor) + mbarrier helpers (sm_90+/sm_100a PTX)
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
// generic-proxy accesses of shared memory ordered before later async-proxy (TMA) ones
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
// 4-D tiled TMA load: box at (c0, c1, c2, c3) of the tensor map into shared memory,
// completion counted on the mbarrier in bytes
__device__ __forceinline__ void tma_load4(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];\n" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}

// TMA plane tile: the 20 x 20 halo tile of one z-plane (x, y in [-2, 18)) as 9 dense
// pieces, one per (sx, sy) in {-1, 0, 1}^2 = the neighbour block it comes from (sx =
// -1: x in [14, 16) of the left block, ...): TMA writes boxes densely, so each piece
// has its own row pitch (its box width) and starts 128-byte aligned.  448 doubles
// (3584 B) per field and plane.
struct TmaTile {
  static constexpr int N = 448;
  // piece p = (sx + 1) + 3 (sy + 1): offset (doubles) and row pitch
  __host__ __device__ static constexpr int off(int p) {
    return p == 0 ? 384 : p == 1 ? 320 : p == 2 ? 400 : p == 3 ? 256 : p == 4 ? 0 : p == 5 ? 288 : p == 6 ? 416
                                                                                                 : p == 7 ? 352 : 432;
  }
  __host__ __device__ static constexpr int pitch(int p) { return (p % 3 == 1) ? 16 : 2; }
  // tile position (x, y) in [-2, 18)^2 -> doubles from the field's piece-set base
  __device__ static int at(int x, int y) {
    const int sx = x < 0 ? -1 : (x >= PB ? 1 : 0), sy = y < 0 ? -1 : (y >= PB ? 1 : 0);
    const int p = (sx + 1) + 3 * (sy + 1);
    const int lx = sx < 0 ? x + 2 : (sx > 0 ? x - PB : x), ly = sy < 0 ? y + 2 : (sy > 0 ? y - PB : y);
    return off(p) + ly * pitch(p) + lx;
  }
};

// Source block / z-local index of plane z of a pencil of `len` blocks (planes
// [-H, 16 len + H)): below the pencil -> neighbour slot dz = -1 of its first block,
// above -> dz = +1 of its last block.
__device__ __forceinline__ void plane_src(int z, int nz, int len, int& k, int& dz, int& zl) {
  dz = z < 0 ? -1 : (z >= nz ? 1 : 0);
  k = z < 0 ? 0 : (z >= nz ? len - 1 : (z >> 4));
  zl = z - PB * k - PB * dz;
}

}  // namespace

// ---------------------------------------------------------------------------------
// Red-black sweep.  Plane tile of old u: x, y in [-2, 18) (halo 2), 20 x 20 doubles,
// staged by 16-byte cp.async into an R-plane ring D planes ahead (f likewise, one
// pair per thread).  Each thread owns a pair of columns (a, b) = (x0, x0+1), x0 even
// in [-2, 16], on a row y in [-1, 17); at every plane one of the two is red and the
// other black.  Which one is red at even planes depends only on the row parity, so
// warps hold rows of one parity (warps 0-2: even y, 3-5: odd y), 3 whole rows of 10
// pairs each (lanes 30, 31 idle): the red and black phases run without divergence,
// and the in-row neighbours x0-1, x0+2 come from the adjacent lanes by shuffles
// instead of strided shared-memory loads.  The step loop is unrolled by 4 so that
// every per-column history (planes s … s-3) is a compile-time-indexed register ring.
// Per step s:
//   load plane s | red at plane s-1 on x, y in [-1, 17) | black at s-2 on [0, 16)^2.
// Δ_h^M of a node = (2F + E - 24c)/(6h^2) (M=4) or (F - 6c)/h^2 (M=2), with
//   F = S4(z) + c(z-1) + c(z+1)  (6 faces),  E = D4(z) + S4(z-1) + S4(z+1)  (12 edges),
// S4/D4 the sums of the 4 in-plane face / diagonal neighbours.  For a red node all
// operands are old values; for a black node the faces are red (new, after the red
// phase) and the edges and centre black (old).
// ---------------------------------------------------------------------------------
template <int D, int RR, bool TMA = false>
struct RBShape {
  static constexpr int T = PB + 4;                 // 20: x, y in [-2, 18)
  // row pitch 26 doubles: a warp's 3 same-parity rows (2 apart, 416 B ≡ 32 mod 128)
  // read with 16-byte loads are bank-conflict free
  static constexpr int TW = 26;
  static constexpr int TP = T * TW;                // 520 doubles per plane
  static constexpr int R = RR;                     // plane ring (power of 2)
  static constexpr int NT = 192;                   // 6 warps x (30 pair-threads + 2 idle)
  static constexpr int NPAIR = T * T / 2;          // 200 16-byte u pairs per plane
  static constexpr int NLD = (NPAIR + NT - 1) / NT;  // 2
  // red-phase values, one per pair: [2 planes][18 rows][pitch 13] (conflict-free)
  static constexpr int SNW = 13, SNP = 18 * SNW;
  // cp.async: [R][TP] old u | [2][SNP] red-phase values | [R][NT] f pairs
  // TMA:      [R][u pieces | f pieces] (R x 7168 B, 128-B aligned) | [2][SNP] red-phase values
  static constexpr int SLOT = 2 * TmaTile::N;  // TMA: doubles per ring slot
  static constexpr size_t SMEM = TMA ? sizeof(double) * (size_t)(R * SLOT + 2 * SNP) + 128
                                     : sizeof(double) * (size_t)(R * TP + 2 * SNP + R * NT * 2);
  static constexpr unsigned PLANE_BYTES = 2 * 400 * sizeof(double);  // TMA bytes per plane (u and f tiles)
  static_assert(D + 2 <= R, "ring too small for the prefetch depth");
};

struct RBCtx {
  const int* snb;
  uint64_t* bar;     // TMA: one mbarrier per ring slot
  const TileMaps* tm;
  const uint32_t* sreal;
  double* su;
  double* sn;
  double2* sf;
  int len, nz;       // pencil blocks, interior planes of this pencil (16 len, or a part of one block)
  int z0, nzb;       // first interior plane relative to the first block, 16 len
  const int* glen;   // shared copy of len
  int ld_xy[2], ld_sxy[2], ld_dst[2];
};

__device__ __forceinline__ double shfl_up1(double v) { return __shfl_up_sync(0xffffffffu, v, 1); }
__device__ __forceinline__ double shfl_dn1(double v) { return __shfl_down_sync(0xffffffffu, v, 1); }

template <int ORDER, int D, int RR, int RP, bool SW, bool TMA>
__device__ __forceinline__ void rb_body(const LevelView& L, const RBCtx& cx, int wg, int lane, double omega,
                                        double inv_h2, double inv_d) {
  using S = RBShape<D, RR, TMA>;
  constexpr int TW = S::TW, TP = S::TP, R = S::R, NT = S::NT, NLD = S::NLD, SNW = S::SNW, SNP = S::SNP;
  constexpr int PC = RP;  // column (0 = a = x0, 1 = b = x0+1) that is red at even planes
  const int* snb = cx.snb;
  // planes are indexed relative to the pencil's first block: interior [zlo, zhi);
  // zlo ∈ {0, 8} keeps zlo ≡ 0 (mod 4), which the unrolled step loop relies on
  const int zlo = SW ? cx.z0 : 0, zhi = SW ? cx.z0 + cx.nz : PB * cx.len;
  double* su = cx.su;
  double* sn = cx.sn;
  const int tid = threadIdx.x;
  double2* sfme = cx.sf + tid;  // this thread's f pair, slot stride NT
  const bool valid = lane < 30;  // lanes 30, 31 mirror lane 29 (broadcast reads), write nothing
  const int ri = valid ? 3 * wg + lane / 10 : 3 * wg + 2;
  const int pi = valid ? lane % 10 : 9;
  const int cy = 2 * ri - RP, x0 = 2 * pi - 2;
  const int i0 = (cy + 2) * TW + (x0 + 2);
  double* snme = sn + (cy + 1) * SNW + pi;  // this pair's red value (row cy) in the compact planes
  const int dxc = reg16(x0), dyc = reg16(cy);
  const int sxy = (dxc + 1) + 3 * (dyc + 1);
  const int fxy = (cy - PB * dyc) * PB + (x0 - PB * dxc);
  const bool inner = valid && dxc == 0 && dyc == 0;
  // TMA tile: offsets (< 448, 9 bits each) of this pair's rows cy-1, cy, cy+1 in a
  // plane's u pieces, packed in one register (the f pair sits at the cy offset of the f
  // pieces, which follow the u pieces in a slot)
  const unsigned ro = TMA ? (unsigned)TmaTile::at(x0, cy - 1) | ((unsigned)TmaTile::at(x0, cy) << 9) |
                                ((unsigned)TmaTile::at(x0, cy + 1) << 18)
                          : 0u;

  // ---- plane cursors: source pointers change only at block boundaries (z % 16 == 0)
  // and at the pencil ends; between them they advance by one plane (PB^2 doubles).
  const double* ip[NLD];
  const double* fp = nullptr;
  auto seek_issue = [&](int z) {
    int k, dz, zl;
    const int len = *cx.glen;  // pencil geometry from shared memory (rare path: spare registers)
    plane_src(z, PB * len, len, k, dz, zl);
    const int o = zl * (PB * PB);
#pragma unroll
    for (int d = 0; d < NLD; ++d)
      ip[d] = cx.ld_sxy[d] < 0 ? nullptr
                               : L.u + (size_t)snb[k * 27 + cx.ld_sxy[d] + 9 * (dz + 1)] * PB3 + o + cx.ld_xy[d];
    fp = L.f + (size_t)snb[k * 27 + sxy + 9 * (dz + 1)] * PB3 + o + fxy;
  };
  // stage plane z (called for z = zlo-2, zlo-1, … in order) into ring slot (z+2) & (R-1).
  // In the step loop z = 4 (zq + t) + j + D - 2 with j, D compile-time, so the slot and
  // the block-boundary test fold to constants (zlo ≡ 0 mod 4).
  // TMA staging: lanes 0..17 of warp 0 each load one of the 9 u / 9 f pieces of plane z
  // (lane 0 arms the slot's mbarrier with the plane's byte count first)
  auto issue_tma = [&](int z, auto checked) {
    if (decltype(checked)::value && z >= zhi + 2) return;
    if (tid >= 18) return;
    const int slot = (z + 2) & (R - 1);
    int k, dz, zl;
    const int len = *cx.glen;
    plane_src(z, PB * len, len, k, dz, zl);
    const int p = tid % 9, sx = p % 3 - 1, sy = p / 3 - 1;
    const int mi = (sx != 0) + 2 * (sy != 0);
    const CUtensorMap* map = tid < 9 ? &cx.tm->u[mi] : &cx.tm->f[mi];
    const int blk = snb[k * 27 + p + 9 * (dz + 1)] + (int)blockIdx.y * L.ntot;  // component c: blocks c ntot + .
    if (tid == 0) {
      fence_proxy_async();
      mbar_expect_tx(cx.bar + slot, S::PLANE_BYTES);
    }
    __syncwarp(0x3ffffu);
    tma_load4(su + slot * S::SLOT + (tid < 9 ? 0 : TmaTile::N) + TmaTile::off(p), map, sx < 0 ? 14 : 0,
              sy < 0 ? 14 : 0, zl, blk, cx.bar + slot);
  };
  auto issue = [&](int z, auto checked) {
    if constexpr (TMA) {
      issue_tma(z, checked);
      return;
    }
    if (!decltype(checked)::value || z < zhi + 2) {
      if ((z & 15) == 0) seek_issue(z);
      const int slot = (z + 2) & (R - 1);
      double* dst = su + slot * TP;
#pragma unroll
      for (int d = 0; d < NLD; ++d) {
        if (cx.ld_sxy[d] < 0) continue;
        cpa16(dst + cx.ld_dst[d], ip[d]);
        ip[d] += PB * PB;
      }
      if (valid && (!decltype(checked)::value || (z >= zlo - 1 && z <= zhi))) cpa16(sfme + slot * NT, fp);
      fp += PB * PB;
    }
    cpa_commit();
  };
  bool live = false;  // red-phase liveness of this pair's columns at plane r
  auto seek_live = [&](int z) {
    int k, dz, zl;
    const int len = *cx.glen;
    plane_src(z, PB * len, len, k, dz, zl);
    live = valid && ((cx.sreal[k] >> (sxy + 9 * (dz + 1))) & 1u);
  };
  if (!TMA) seek_issue(zlo - 2);
  seek_live(zlo - 1);
#pragma unroll
  for (int q = 0; q < D; ++q) issue(zlo - 2 + q, std::true_type{});

  // Per-column accumulators (column q = a, b).  With α(z) = 2c(z) + S4(z),
  // β(z) = 2S4(z) + D4(z) - 24c(z), γ(z) = 2n(z) + S4(z) (n = value after the red
  // phase), the Mehrstellen operator times 6h^2 is
  //   red node at r:   α(r-1) + β(r) + α(r+1)                   (all old values)
  //   black node at b: γ(b-1) + 2 S4n(b) + D4(b) - 24c(b) + γ(b+1)  (S4n: red, new)
  // so each column carries only partial sums between steps.
  double accR[2] = {0, 0}, cR[2] = {0, 0};  // red plane: α(r-1) + β(r), c(r)
  double accB[2] = {0, 0}, cB[2] = {0, 0};  // black plane: D4(b) - 24c(b) + γ(b-1), c(b)
  double s4r[2] = {0, 0};                   // S4 at the column's last red plane
  double nl[2] = {0, 0};                    // value after the red phase at the last red plane
  const double h6 = inv_h2 * (1.0 / 6.0);
  const double wd = omega * inv_d;
  double2 fr = make_double2(0.0, 0.0);  // f pair at the plane of the last red phase
  double fb = 0.0;                      // f of the column black at plane s-2

  // output offset of this pair at the black plane b = s-2 (advanced by one plane per
  // step, re-seeked at block starts)
  int ooff = snb[(zlo >> 4) * 27 + 13] * PB3 + ((zlo & 15) - 4) * (PB * PB) + fxy;
  // One group = 4 steps s = base-2 … base+1 (base a multiple of 4, so ring slots and
  // block-boundary tests are compile-time).  The first group holds the pipeline start:
  // red from its third step on, no black; later groups run both.  Only the last group
  // stages planes past the pencil end (bounds-checked issue); elsewhere the staging
  // pointers advance unconditionally.
  auto group = [&](const int base, auto mode) {
    constexpr bool FIRST = decltype(mode)::value == 0, LAST = decltype(mode)::value == 2;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int s = base - 2 + j;
      const int X = (j & 1) ? PC : 1 - PC;  // red at s-1 (black at s and s-2); base even
      const int O = 1 - X;                  // red at s (and s-2)
      if constexpr (TMA) {
        // plane s: slot (s+2) & (R-1), used for the ((s+2) >> 2)-th time (R = 4)
        if (!LAST || s < zhi + 2) mbar_wait(cx.bar + ((s + 2) & (R - 1)), ((s + 2 - (zlo & ~3)) >> 2) & 1);
      } else {
        cpa_wait<D - 1>();
      }
      __syncthreads();
      issue(s + D, std::integral_constant<bool, LAST>{});
      double cq[2], s4q[2], d4q[2];
      {
        const double* Us = su + ((s + 2) & (R - 1)) * (TMA ? S::SLOT : TP);
        const double* U = Us + (TMA ? (ro >> 9) & 511u : i0);
        const double2 m = *reinterpret_cast<const double2*>(TMA ? Us + (ro & 511u) : U - TW);
        const double2 cc = *reinterpret_cast<const double2*>(U);
        const double2 p = *reinterpret_cast<const double2*>(TMA ? Us + (ro >> 18) : U + TW);
        const double l = shfl_up1(cc.y), r = shfl_dn1(cc.x);  // u(x0-1), u(x0+2)
        // rows y-1 + y+1 per column: the diagonal sums need one shuffle per column
        // (u(x0-1, y-1) + u(x0-1, y+1) is the left lane's qy)
        const double qx = m.x + p.x, qy = m.y + p.y;
        cq[0] = cc.x;
        cq[1] = cc.y;
        s4q[0] = (l + cc.y) + qx;
        s4q[1] = (cc.x + r) + qy;
        if (ORDER == 4) {
          d4q[0] = shfl_up1(qy) + qy;
          d4q[1] = qx + shfl_dn1(qx);
        } else {
          d4q[0] = d4q[1] = 0.0;
        }
      }
      // in-row red neighbour of the black node at s-2 held by the adjacent lane
      const double nx = X ? shfl_dn1(nl[0]) : shfl_up1(nl[1]);
      // column X: black at plane s
      const double alpha = ORDER == 4 ? 2.0 * cq[X] + s4q[X] : cq[X];
      if (!FIRST || j >= 2) {  // red half-sweep at plane r = s-1 in [zlo-1, zhi] (column X)
        if (((s - 1) & 15) == 0) seek_live(s - 1);
        fb = X ? fr.y : fr.x;                 // f at plane s-2 of column X (pair read last step)
        // f pair at plane s-1
        fr = TMA ? *reinterpret_cast<const double2*>(su + ((s + 1) & (R - 1)) * S::SLOT + TmaTile::N + ((ro >> 9) & 511u))
                 : sfme[((s + 1) & (R - 1)) * NT];
        double v = cR[X];
        if (live) {
          const double Lu = ORDER == 4 ? (accR[X] + alpha) * h6 : (accR[X] + alpha) * inv_h2;
          v = cR[X] + wd * ((X ? fr.y : fr.x) - Lu);
        }
        if (valid) snme[(j & 1) * SNP] = v;  // new-plane slot = parity of s
        const double g = ORDER == 4 ? 2.0 * v + s4r[X] : v;  // γ(s-1) of column X
        if (!FIRST) {
          const int b = s - 2;
          if ((b & 15) == 0) ooff = snb[(b >> 4) * 27 + 13] * PB3 + fxy;
          if (inner) {  // black half-sweep at plane b (column X)
            const double* N = snme + ((j & 1) ^ 1) * SNP;  // rows cy±1 hold the red node at x of X
            const double S4n = (nl[O] + nx) + (N[-SNW] + N[SNW]);
            const double Lu = ORDER == 4 ? (accB[X] + 2.0 * S4n + g) * h6 : (accB[X] + S4n + g) * inv_h2;
            const double vb = cB[X] + wd * (fb - Lu);
            *reinterpret_cast<double2*>(L.u_out + (size_t)ooff) =
                X ? make_double2(nl[O], vb) : make_double2(vb, nl[O]);
          }
        }
        accB[X] = (ORDER == 4 ? d4q[X] - 24.0 * cq[X] : -6.0 * cq[X]) + g;
        nl[X] = v;
      }
      ooff += PB * PB;
      cB[X] = cq[X];
      accR[X] = alpha;  // α(s): first term of the red node at s+1
      // column O: red at plane s
      accR[O] += ORDER == 4 ? 2.0 * s4q[O] + d4q[O] - 24.0 * cq[O] : s4q[O] - 6.0 * cq[O];
      cR[O] = cq[O];
      s4r[O] = s4q[O];
    }
  };
  const int zq = zlo >> 2, nt = (zhi - zlo + 4) >> 2;
  group(4 * zq, std::integral_constant<int, 0>{});
  for (int t = 1; t < nt - 1; ++t) group(4 * (zq + t), std::integral_constant<int, 1>{});
  group(4 * (zq + nt - 1), std::integral_constant<int, 2>{});
  if (!TMA) cpa_wait<0>();
}

template <int ORDER, int D, int RR, int NREG, bool SW, bool TMA>
__global__ void __maxnreg__(NREG)
    k_rb_pencil(LevelView L, double omega, double inv_h2, double inv_d, const __grid_constant__ TileMaps tm) {
  using S = RBShape<D, RR, TMA>;
  comp_view(L);
  constexpr int T = S::T, TW = S::TW, TP = S::TP, R = S::R, NT = S::NT, NPAIR = S::NPAIR, NLD = S::NLD;
  extern __shared__ __align__(16) double smraw[];
  __shared__ int snb[PMAXL * 27];
  __shared__ uint32_t sreal[PMAXL];
  __shared__ int slen;
  __shared__ __align__(8) uint64_t sbar[R];
  // TMA destinations must be 128-byte aligned
  double* sm = TMA ? reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(smraw) + 127) & ~uintptr_t(127)) : smraw;
  const int tid = threadIdx.x;
  RBCtx cx;
  cx.bar = sbar;
  cx.tm = &tm;
  if (TMA && tid < R) mbar_init(sbar + tid, 1);
  // sweep pencils (sw_*: may split a block into z-parts on small levels) or block pencils
  const bool sw = SW;
  cx.len = __ldg((sw ? L.sw_pen_len : L.pen_len) + blockIdx.x);
  cx.nzb = PB * cx.len;
  if (sw) {
    const int zr = __ldg(L.sw_pen_z + blockIdx.x);
    cx.z0 = zr & 0xff;
    cx.nz = zr >> 8;
  } else {
    cx.z0 = 0;
    cx.nz = cx.nzb;
  }
  cx.snb = snb;
  cx.sreal = sreal;
  cx.glen = &slen;
  if (tid == 0) slen = cx.len;
  cx.su = sm;
  cx.sn = sm + R * (TMA ? S::SLOT : TP);
  cx.sf = reinterpret_cast<double2*>(sm + R * TP + 2 * S::SNP);
  const int32_t* pb = sw ? L.sw_pen_blk + (size_t)blockIdx.x * L.sw_pen_lmax
                         : L.pen_blk + (size_t)blockIdx.x * L.pen_lmax;
  for (int i = tid; i < cx.len * 27; i += NT) snb[i] = __ldg(L.nbr + (size_t)__ldg(pb + i / 27) * 27 + i % 27);
  if (tid < cx.len) sreal[tid] = __ldg(L.nbr_real + __ldg(pb + tid));
  // load items: 0-159 = the 16-wide interior part of the 20 tile rows, 8 lanes per row
  // (each group of 8 lanes fetches one aligned 128-byte line); 160-199 = the 16-byte
  // halo pieces x in [-2, 0) and [16, 18) of every row
#pragma unroll
  for (int d = 0; d < NLD; ++d) {
    const int j = tid + d * NT;
    int py, px;
    if (j < 8 * T) {
      py = j / 8;
      px = 2 + 2 * (j % 8);
    } else {
      const int hh = j - 8 * T;
      py = hh / 2;
      px = (hh & 1) ? PB + 2 : 0;
    }
    const int x = px - 2, y = py - 2, dx = reg16(x), dy = reg16(y);
    cx.ld_xy[d] = (y - PB * dy) * PB + (x - PB * dx);
    cx.ld_sxy[d] = j < NPAIR ? (dx + 1) + 3 * (dy + 1) : -1;
    cx.ld_dst[d] = py * TW + px;
  }
  if (TMA && tid < R) asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");  // inits -> async proxy
  __syncthreads();  // snb / sreal / mbarriers
  // warp-uniform row parity: warps 0-2 even rows, 3-5 odd rows
  const int w = tid >> 5, lane = tid & 31;
  if (w < 3) rb_body<ORDER, D, RR, 0, SW, TMA>(L, cx, w, lane, omega, inv_h2, inv_d);
  else rb_body<ORDER, D, RR, 1, SW, TMA>(L, cx, w - 3, lane, omega, inv_h2, inv_d);
}

// ---------------------------------------------------------------------------------
// Red-black sweep, M = 6 (27-point LHS, E13 / fig:stencils): same tile, pair threads
// and partial-sum scheme as the M = 2/4 sweep, but the black update also reads the
// new red values at its 8 corners (planes b±1, rows y±1), which other warps compute
// one step after the red plane is staged; the black half-sweep therefore runs three
// planes behind the loads instead of two:
//   step s: load plane s | red at s-1 | γ of the red column at s-2 | black at s-3.
// With (times 30 h^2)  α = 14c + 3 S4 + D4,  β = 14 S4 + 3 D4 - 128 c  (old values),
//   γ(z) = 14 n(z) + 3 S4(z) + D4n(z)  (n, D4n: new red values; S4: old black faces):
//   red node at r:   α(r-1) + β(r) + α(r+1)
//   black node at b: -128 c(b) + 3 D4(b) + 14 S4n(b) + γ(b-1) + γ(b+1).
// Steps run in groups of 8 (base ≡ 0 mod 8), so the plane rings (u: 4 planes, red
// values: 4, f: 8 — the black update reads f three planes back) have compile-time
// slots; the last group takes one extra step (black at the last plane).
// ---------------------------------------------------------------------------------
struct RB6Shape {
  static constexpr int T = PB + 4, TW = 26, TP = T * TW;
  static constexpr int R = 4, FR = 8;
  static constexpr int NT = 192;
  static constexpr int NPAIR = T * T / 2, NLD = (NPAIR + NT - 1) / NT;
  static constexpr int SNW = 13, SNP = 18 * SNW, SNR = 4;
  static constexpr size_t SMEM = sizeof(double) * (size_t)(R * TP + SNR * SNP + FR * NT * 2);
};

template <int RP, bool SW>
__device__ __forceinline__ void rb6_body(const LevelView& L, const RBCtx& cx, int wg, int lane, double omega,
                                         double inv_h2, double inv_d) {
  using S = RB6Shape;
  constexpr int TW = S::TW, TP = S::TP, R = S::R, FR = S::FR, NT = S::NT, NLD = S::NLD, SNW = S::SNW,
                SNP = S::SNP;
  constexpr int PC = RP;  // column red at even planes
  const int* snb = cx.snb;
  const int zlo = SW ? cx.z0 : 0, zhi = SW ? cx.z0 + cx.nz : PB * cx.len;  // zlo ≡ 0 (mod 8)
  double* su = cx.su;
  const int tid = threadIdx.x;
  double2* sfme = cx.sf + tid;
  const bool valid = lane < 30;
  const int ri = valid ? 3 * wg + lane / 10 : 3 * wg + 2;
  const int pi = valid ? lane % 10 : 9;
  const int cy = 2 * ri - RP, x0 = 2 * pi - 2;
  const int i0 = (cy + 2) * TW + (x0 + 2);
  double* snme = cx.sn + (cy + 1) * SNW + pi;
  const int dxc = reg16(x0), dyc = reg16(cy);
  const int sxy = (dxc + 1) + 3 * (dyc + 1);
  const int fxy = (cy - PB * dyc) * PB + (x0 - PB * dxc);
  const bool inner = valid && dxc == 0 && dyc == 0;

  const double* ip[NLD];
  const double* fp = nullptr;
  auto seek_issue = [&](int z) {
    int k, dz, zl;
    const int len = *cx.glen;
    plane_src(z, PB * len, len, k, dz, zl);
    const int o = zl * (PB * PB);
#pragma unroll
    for (int d = 0; d < NLD; ++d)
      ip[d] = cx.ld_sxy[d] < 0 ? nullptr
                               : L.u + (size_t)snb[k * 27 + cx.ld_sxy[d] + 9 * (dz + 1)] * PB3 + o + cx.ld_xy[d];
    fp = L.f + (size_t)snb[k * 27 + sxy + 9 * (dz + 1)] * PB3 + o + fxy;
  };
  auto issue = [&](int z, auto checked) {
    if (!decltype(checked)::value || z < zhi + 2) {
      if ((z & 15) == 0) seek_issue(z);
      double* dst = su + ((z + 2) & (R - 1)) * TP;
#pragma unroll
      for (int d = 0; d < NLD; ++d) {
        if (cx.ld_sxy[d] < 0) continue;
        cpa16(dst + cx.ld_dst[d], ip[d]);
        ip[d] += PB * PB;
      }
      if (valid && (!decltype(checked)::value || (z >= zlo - 1 && z <= zhi)))
        cpa16(sfme + ((z + 2) & (FR - 1)) * NT, fp);
      fp += PB * PB;
    }
    cpa_commit();
  };
  bool live = false;
  auto seek_live = [&](int z) {
    int k, dz, zl;
    const int len = *cx.glen;
    plane_src(z, PB * len, len, k, dz, zl);
    live = valid && ((cx.sreal[k] >> (sxy + 9 * (dz + 1))) & 1u);
  };
  seek_issue(zlo - 2);
  seek_live(zlo - 1);
#pragma unroll
  for (int q = 0; q < D6; ++q) issue(zlo - 2 + q, std::true_type{});

  double accR[2] = {0, 0}, cR[2] = {0, 0};  // red plane in flight: α(r-1) + β(r), c(r)
  double s4r[2] = {0, 0};                   // S4 (old) at the column's last red plane
  double nv[2] = {0, 0};                    // the column's last new red value
  double accB[2][2] = {{0, 0}, {0, 0}};     // black planes in flight (slot (b >> 1) & 1)
  double cB[2][2] = {{0, 0}, {0, 0}};
  const double h30 = inv_h2 * (1.0 / 30.0);
  const double wd = omega * inv_d;
  // output offset of this pair at plane b = s-3 (one plane per step, re-seeked at block starts)
  int ooff = snb[(zlo >> 4) * 27 + 13] * PB3 + ((zlo & 15) - 5) * (PB * PB) + fxy;

  auto group = [&](const int base, auto mode) {
    constexpr int MODE = decltype(mode)::value;
    constexpr bool FIRST = MODE == 0, LAST = MODE == 2;
    constexpr int NSTEP = LAST ? 5 : 8;
#pragma unroll
    for (int j = 0; j < NSTEP; ++j) {
      const int s = base - 2 + j;
      const int X = (j & 1) ? PC : 1 - PC;  // black at s, red at s-1
      const int O = 1 - X;                  // red at s and s-2, black at s-1 and s-3
      const bool plane = !LAST || j <= 3;   // plane s exists (s <= zhi+1)
      cpa_wait<D6 - 1>();
      __syncthreads();
      issue(s + D6, std::integral_constant<bool, LAST>{});
      double cq[2] = {0, 0}, s4q[2] = {0, 0}, d4q[2] = {0, 0};
      if (plane) {
        const double* U = su + ((s + 2) & (R - 1)) * TP + i0;
        const double2 m = *reinterpret_cast<const double2*>(U - TW);
        const double2 cc = *reinterpret_cast<const double2*>(U);
        const double2 p = *reinterpret_cast<const double2*>(U + TW);
        const double l = shfl_up1(cc.y), r = shfl_dn1(cc.x);
        const double qx = m.x + p.x, qy = m.y + p.y;  // rows y±1 per column (diagonals: one shuffle)
        cq[0] = cc.x;
        cq[1] = cc.y;
        s4q[0] = (l + cc.y) + qx;
        s4q[1] = (cc.x + r) + qy;
        d4q[0] = shfl_up1(qy) + qy;
        d4q[1] = qx + shfl_dn1(qx);
      }
      // γ of column O at its red plane s-2 (red values of plane s-2 written last step)
      double gam;
      {
        const double* Nz = snme + ((s - 2) & 3) * SNP;
        const double wv = Nz[-SNW] + Nz[SNW];               // rows y±1 at x_O ± 1: own pair …
        const double wn = O == 0 ? shfl_up1(wv) : shfl_dn1(wv);  // … and the adjacent pair
        gam = (14.0 * nv[O] + 3.0 * s4r[O]) + (wv + wn);
      }
      // black half-sweep at plane b = s-3 (column O): S4n from the own pair's red column,
      // the adjacent lane's, and rows y±1 of the red plane b
      {
        const double nxn = O == 0 ? shfl_up1(nv[X]) : shfl_dn1(nv[X]);
        const int b = s - 3;
        if (!FIRST || j >= 5) {
          if ((b & 15) == 0) ooff = snb[(b >> 4) * 27 + 13] * PB3 + fxy;
          if (inner) {
            const double* Nb = snme + (b & 3) * SNP;
            const int sl = (b >> 1) & 1;
            const double S4n = (nv[X] + nxn) + (Nb[-SNW] + Nb[SNW]);
            const double Lu = ((accB[O][sl] + gam) + 14.0 * S4n) * h30;
            const double2 fb2 = sfme[((b + 2) & (FR - 1)) * NT];
            const double vb = cB[O][sl] + wd * ((O ? fb2.y : fb2.x) - Lu);
            *reinterpret_cast<double2*>(L.u_out + (size_t)ooff) =
                O ? make_double2(nv[X], vb) : make_double2(vb, nv[X]);
          }
        }
        ooff += PB * PB;
      }
      accB[O][((s - 1) >> 1) & 1] += gam;  // γ(b-1) of O's black plane b = s-1
      // red half-sweep at plane r = s-1 (column X)
      if ((!FIRST || j >= 2) && plane) {
        if (((s - 1) & 15) == 0) seek_live(s - 1);
        const double2 fr = sfme[((s + 1) & (FR - 1)) * NT];
        const double alpha = (14.0 * cq[X] + 3.0 * s4q[X]) + d4q[X];
        double v = cR[X];
        if (live) {
          const double Lu = (accR[X] + alpha) * h30;
          v = cR[X] + wd * ((X ? fr.y : fr.x) - Lu);
        }
        if (valid) snme[((s - 1) & 3) * SNP] = v;
        nv[X] = v;
      }
      if (plane) {
        // column X black at s: start its black partial sum
        accB[X][(s >> 1) & 1] = 3.0 * d4q[X] - 128.0 * cq[X];
        cB[X][(s >> 1) & 1] = cq[X];
        accR[X] = (14.0 * cq[X] + 3.0 * s4q[X]) + d4q[X];  // α(s): first term of X's red plane s+1
        // column O red at s
        accR[O] += (14.0 * s4q[O] + 3.0 * d4q[O]) - 128.0 * cq[O];
        cR[O] = cq[O];
        s4r[O] = s4q[O];
      }
    }
  };
  // bases written as 8 * (…) so that the compiler sees base ≡ 0 (mod 8)
  const int zq = zlo >> 3, zr = zhi >> 3;
  group(8 * zq, std::integral_constant<int, 0>{});
  for (int t = zq + 1; t < zr; ++t) group(8 * t, std::integral_constant<int, 1>{});
  group(8 * zr, std::integral_constant<int, 2>{});
  cpa_wait<0>();
}

template <int NREG, bool SW>
__global__ void __maxnreg__(NREG) k_rb6_pencil(LevelView L, double omega, double inv_h2, double inv_d) {
  using S = RB6Shape;
  comp_view(L);
  constexpr int T = S::T, TW = S::TW, TP = S::TP, R = S::R, NT = S::NT, NPAIR = S::NPAIR, NLD = S::NLD;
  extern __shared__ __align__(16) double sm[];
  __shared__ int snb[PMAXL * 27];
  __shared__ uint32_t sreal[PMAXL];
  __shared__ int slen;
  const int tid = threadIdx.x;
  RBCtx cx;
  cx.len = __ldg((SW ? L.sw_pen_len : L.pen_len) + blockIdx.x);
  cx.nzb = PB * cx.len;
  if (SW) {
    const int zr = __ldg(L.sw_pen_z + blockIdx.x);
    cx.z0 = zr & 0xff;
    cx.nz = zr >> 8;
  } else {
    cx.z0 = 0;
    cx.nz = cx.nzb;
  }
  cx.snb = snb;
  cx.sreal = sreal;
  cx.glen = &slen;
  if (tid == 0) slen = cx.len;
  cx.su = sm;
  cx.sn = sm + R * TP;
  cx.sf = reinterpret_cast<double2*>(sm + R * TP + S::SNR * S::SNP);
  const int32_t* pb = SW ? L.sw_pen_blk + (size_t)blockIdx.x * L.sw_pen_lmax
                         : L.pen_blk + (size_t)blockIdx.x * L.pen_lmax;
  for (int i = tid; i < cx.len * 27; i += NT) snb[i] = __ldg(L.nbr + (size_t)__ldg(pb + i / 27) * 27 + i % 27);
  if (tid < cx.len) sreal[tid] = __ldg(L.nbr_real + __ldg(pb + tid));
#pragma unroll
  for (int d = 0; d < NLD; ++d) {
    const int j = tid + d * NT;
    int py, px;
    if (j < 8 * T) {
      py = j / 8;
      px = 2 + 2 * (j % 8);
    } else {
      const int hh = j - 8 * T;
      py = hh / 2;
      px = (hh & 1) ? PB + 2 : 0;
    }
    const int x = px - 2, y = py - 2, dx = reg16(x), dy = reg16(y);
    cx.ld_xy[d] = (y - PB * dy) * PB + (x - PB * dx);
    cx.ld_sxy[d] = j < NPAIR ? (dx + 1) + 3 * (dy + 1) : -1;
    cx.ld_dst[d] = py * TW + px;
  }
  __syncthreads();
  const int w = tid >> 5, lane = tid & 31;
  if (w < 3) rb6_body<0, SW>(L, cx, w, lane, omega, inv_h2, inv_d);
  else rb6_body<1, SW>(L, cx, w - 3, lane, omega, inv_h2, inv_d);
}

// ---------------------------------------------------------------------------------
// Residual r = f - Δ_h^M u (Alg. 1) on every node of the pencil's blocks.
// Plane tile of u: x, y in [-2, 18) (halo 1 used; pairs keep 16-byte alignment);
// f: the block's own 16 x 16 plane.  One thread per interior column (256).
// ---------------------------------------------------------------------------------
template <int D>
struct ResShape {
  static constexpr int T = PB + 4, TP = T * T;  // 20, 400
  static constexpr int FP = PB * PB;            // 256
  static constexpr int R = D + 2;
  static constexpr int NT = PB * PB;            // 256
  static constexpr int NUP = TP / 2, NFP = FP / 2;  // 200 + 128 pairs
  static constexpr size_t SMEM = sizeof(double) * (size_t)(R * (TP + FP));
};

// MODE 0: r = f - Δ_h^M u (residual, Alg. 1) on every node of the pencil.
// MODE 1: f = r + Δ_h^M u (FAS right-hand side on the coarse level, Alg. 1) on
//         the nodes of octants covered by the finer level (covmask); others untouched;
//         and û = u on every node of the pencil (the snapshot of Alg. 1).
// MODE 3: r = R_h^4 f = f + (1/12) Σ δ² f (the right-hand side of E12; M = 4)
//         on leaf nodes and r = f on covered nodes, from the plane tiles of f (its ghosts
//         filled); the caller copies r into f (f* stored once).
// MODE 2: max |f - Δ_h^M u| over the nodes of uncovered octants (the composite residual
//         norm of the stopping test) as the bit pattern of a non-negative double
//         (NaN -> quiet-NaN pattern, above +Inf), atomicMax-ed into *out; nothing written.
template <int ORDER, int D, int MODE = 0>
__global__ void __launch_bounds__(ResShape<D>::NT, 4)
    k_res_pencil(LevelView L, double inv_h2, unsigned long long* out = nullptr) {
  using S = ResShape<D>;
  comp_view(L);
  constexpr int T = S::T, TP = S::TP, FP = S::FP, R = S::R, NT = S::NT;
  extern __shared__ __align__(16) double sm[];
  double* su = sm;           // [R][TP]
  double* sf = sm + R * TP;  // [R][FP]
  __shared__ int snb[PMAXL * 27];
  const int tid = threadIdx.x;
  const int len = __ldg(L.pen_len + blockIdx.x);
  const int32_t* pb = L.pen_blk + (size_t)blockIdx.x * L.pen_lmax;
  for (int i = tid; i < len * 27; i += NT) snb[i] = __ldg(L.nbr + (size_t)__ldg(pb + i / 27) * 27 + i % 27);
  __shared__ uint8_t scov[PMAXL];
  if (MODE != 0 && tid < len) scov[tid] = __ldg(L.covmask + __ldg(pb + tid));
  const int nz = PB * len;
  const double* __restrict__ fin = MODE == 1 ? L.r : L.f;  // the right-hand operand staged per plane
  const double* __restrict__ tsrc = MODE == 3 ? L.f : L.u;  // the field of the plane tiles
  unsigned long long nmax = 0ull;                            // MODE 2

  int ld_xy[2], ld_sxy[2], ld_dst[2];
  bool ld_on[2], ld_f[2];
#pragma unroll
  for (int d = 0; d < 2; ++d) {
    const int j = tid + d * NT;
    ld_on[d] = j < S::NUP + S::NFP;
    ld_f[d] = j >= S::NUP;
    if (ld_f[d]) {
      const int jj = j - S::NUP;
      ld_xy[d] = 2 * jj;
      ld_sxy[d] = 4;  // own block (dx = dy = 0)
      ld_dst[d] = R * TP + 2 * jj;
    } else {
      const int py = j / (T / 2), px = 2 * (j % (T / 2));
      const int x = px - 2, y = py - 2, dx = reg16(x), dy = reg16(y);
      ld_xy[d] = (y - PB * dy) * PB + (x - PB * dx);
      ld_sxy[d] = (dx + 1) + 3 * (dy + 1);
      ld_dst[d] = py * T + px;
    }
  }
  __syncthreads();
  if (MODE == 2) {  // a pencil of fully covered blocks holds no leaf node: nothing to reduce
    bool all = true;
    for (int k = 0; k < len; ++k) all = all && scov[k] == 0xff;
    if (all) return;
  }

  auto issue = [&](int z) {
    if (z < nz + 1) {
      int k, dz, zl;
      plane_src(z, nz, len, k, dz, zl);
      const int slot = (z + 1) % R;
#pragma unroll
      for (int d = 0; d < 2; ++d) {
        // MODE 1: r is read only on blocks with a covered octant
        if (!ld_on[d] || (ld_f[d] && (dz != 0 || MODE == 3 || (MODE == 1 && scov[k] == 0)))) continue;
        const int blk = snb[k * 27 + ld_sxy[d] + 9 * (dz + 1)];
        const double* src = (ld_f[d] ? fin : tsrc) + (size_t)blk * PB3 + zl * (PB * PB) + ld_xy[d];
        cpa16(sm + ld_dst[d] + slot * (ld_f[d] ? FP : TP), src);
      }
    }
    cpa_commit();
  };

  const int cx = tid % PB, cy = tid / PB;
  const int ci = (cy + 2) * T + (cx + 2);
#pragma unroll
  for (int q = 0; q < D; ++q) issue(-1 + q);

  double c0 = 0, c1 = 0, c2 = 0, a0 = 0, a1 = 0, a2 = 0, d0 = 0, d1 = 0, d2 = 0;
  const double h6 = inv_h2 * (1.0 / 6.0);
  for (int s = -1; s < nz + 1; ++s) {
    cpa_wait<D - 1>();
    __syncthreads();
    issue(s + D);
    c2 = c1; c1 = c0;
    a2 = a1; a1 = a0;
    d2 = d1; d1 = d0;
    // MODE 1 (FAS): the operator is evaluated only on blocks with a covered octant, so the
    // in-plane sums of plane s are needed only if the block of plane s-1, s or s+1 has one;
    // elsewhere the pass just copies u into û (CTA-uniform branches)
    bool sums = true, lap = true;
    if (MODE == 1) {
      const int kl = min(max((s - 1) >> 4, 0), len - 1), km = min(max(s >> 4, 0), len - 1),
                kh = min(max((s + 1) >> 4, 0), len - 1);
      sums = (scov[kl] | scov[km] | scov[kh]) != 0;
      lap = s >= 1 && scov[(s - 1) >> 4] != 0;
    }
    {
      const double* U = su + ((s + 1) % R) * TP + ci;
      c0 = U[0];
      if (sums) {
        a0 = (U[-1] + U[1]) + (U[-T] + U[T]);
        if (ORDER == 6) d0 = (U[-T - 1] + U[-T + 1]) + (U[T - 1] + U[T + 1]);
      }
    }
    if (MODE == 1 && s >= 1 && !lap) {
      const int r = s - 1;
      L.uhat[(size_t)snb[(r >> 4) * 27 + 13] * PB3 + (r & 15) * (PB * PB) + tid] = c1;
    } else if (MODE == 3 && s >= 1) {
      // f* at plane r = s-1: δ² along x, y from the tile, along z from the carried centres,
      // summed as ((δ²x + δ²y) + δ²z) / 12 (the generic kernel's order)
      const int r = s - 1;
      const double* U = su + ((r + 1) % R) * TP + ci;
      const double dx = (U[-1] - 2.0 * c1) + U[1], dy = (U[-T] - 2.0 * c1) + U[T], dz = (c2 - 2.0 * c1) + c0;
      const size_t o = (size_t)snb[(r >> 4) * 27 + 13] * PB3 + (r & 15) * (PB * PB) + tid;
      const int oct = (cx >= PB / 2) | ((cy >= PB / 2) << 1) | (((r & 15) >= PB / 2) << 2);
      L.r[o] = ((scov[r >> 4] >> oct) & 1) ? c1 : c1 + ((dx + dy) + dz) / 12.0;
    } else if (s >= 1) {
      const int r = s - 1;
      const int sl = (r + 1) % R;
      const double f = sf[sl * FP + tid];
      double Lu;
      if (ORDER == 2) {
        Lu = ((a1 + (c2 + c0)) - 6.0 * c1) * inv_h2;
      } else if (ORDER == 4) {
        const double* U = su + sl * TP + ci;
        const double Dg = (U[-T - 1] + U[-T + 1]) + (U[T - 1] + U[T + 1]);
        const double F = a1 + (c2 + c0);
        const double E = Dg + (a2 + a0);
        Lu = (2.0 * F + E - 24.0 * c1) * h6;
      } else {
        // M = 6 (E13, fig:stencils): (14 faces + 3 edges + corners - 128 c) / (30 h^2)
        const double F = a1 + (c2 + c0);
        const double E = d1 + (a2 + a0);
        const double K = d2 + d0;
        Lu = ((14.0 * F + 3.0 * E) + K - 128.0 * c1) * (inv_h2 * (1.0 / 30.0));
      }
      const size_t o = (size_t)snb[(r >> 4) * 27 + 13] * PB3 + (r & 15) * (PB * PB) + tid;
      if (MODE == 0) {
        L.r[o] = f - Lu;
      } else {
        const int oct = (cx >= PB / 2) | ((cy >= PB / 2) << 1) | (((r & 15) >= PB / 2) << 2);
        const bool cov = (scov[r >> 4] >> oct) & 1;
        if (MODE == 1) {
          if (cov) L.f[o] = f + Lu;
          L.uhat[o] = c1;  // the û snapshot (Alg. 1) of every real node, from the staged plane
        } else if (!cov) {
          const double v = fabs(f - Lu);
          unsigned long long bits = (unsigned long long)__double_as_longlong(v);
          if (v != v) bits = 0x7ff8000000000000ull;
          nmax = bits > nmax ? bits : nmax;
        }
      }
    }
  }
  cpa_wait<0>();
  if (MODE == 2) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long t = __shfl_xor_sync(0xffffffffu, nmax, o);
      nmax = t > nmax ? t : nmax;
    }
    __shared__ unsigned long long sred[NT / 32];
    if ((tid & 31) == 0) sred[tid >> 5] = nmax;
    __syncthreads();
    if (tid == 0) {
      unsigned long long m = 0ull;
      for (int w = 0; w < NT / 32; ++w) m = sred[w] > m ? sred[w] : m;
      atomicMax(out, m);
    }
  }
}

// ---------------------------------------------------------------------------------
// Fused residual + restriction (Alg. 1), column-pair version: the residual
// of the pencil and its halo ring [-1, 17)^2 (the full-weighting footprint; r := 0 at
// fine positions outside the level's blocks, reading Z14) is computed as in the RB
// sweep (pairs of columns, shuffles for the in-row neighbours, Mehrstellen partial
// sums per column: r(z) = f(z) - h6 [α(z-1) + β(z) + α(z+1)]); each pair also forms
// the x-weighted sum at its even column (one shuffle) into a 2-plane shared ring.
// Warps hold rows of one parity (0-2 even, 3-5 odd, as in the sweep), so the coarse
// work stays in the even-row warps: the pair at (x0, y) = (2 qx, 2 qy) writes the
// coarse u(qx, qy) at even planes from its own centre value (injection, E7) and forms
// the y- and z-weights of the coarse residual (E6) from its own x-weighted sum (kept
// in a register) and rows y±1 of the ring.  No extra warps: 6 warps, 4 CTAs per SM.
// The fine residual is never written to HBM.
// Step s: load plane s | r at plane s-1 | y weights of r(s-2) | coarse r at s-3.
struct RR2Shape {
  static constexpr int T = PB + 4, TW = 26, TP = T * TW;  // u tile as in the RB sweep
  static constexpr int D = 2, R = 4;
  static constexpr int NT = 192;                           // 6 warps of 30 pair threads
  static constexpr int NPAIR = T * T / 2;                  // 200 u pairs per plane
  static constexpr int NLD = (NPAIR + NT - 1) / NT;        // 2
  // x-weighted residual rows sx (one per pair, at its even column): rows [-1, 17),
  // pairs 0..9, odd pitch
  static constexpr int SXW = 11, SXP = 18 * SXW;
  // [R][TP] u | [R][NT] f pairs | [2][SXP] sx
  static constexpr size_t SMEM = sizeof(double) * (size_t)(R * TP + R * NT * 2 + 2 * SXP);
};

template <int ORDER, int RP>
__device__ __forceinline__ void rr2_body(const LevelView& L, const LevelView& C, const int* snb, const uint32_t* sreal,
                                         const int* spar, double* sm, const int (&ld_xy)[2], const int (&ld_sxy)[2],
                                         const int (&ld_dst)[2], int wg, int lane, int len, double inv_h2) {
  using S = RR2Shape;
  constexpr int TW = S::TW, TP = S::TP, D = S::D, R = S::R, NT = S::NT, NLD = S::NLD, SXW = S::SXW, SXP = S::SXP;
  double* su = sm;
  double2* sf = reinterpret_cast<double2*>(sm + R * TP);  // [R][NT]
  double* sxr = sm + R * TP + R * NT * 2;                  // [2][SXP]
  const int tid = threadIdx.x;
  const int nz = PB * len;
  const bool valid = lane < 30;  // lanes 30, 31 mirror lane 29 (broadcast reads), write nothing
  const int ri = valid ? 3 * wg + lane / 10 : 3 * wg + 2;
  const int pi = valid ? lane % 10 : 9;
  const int ry = 2 * ri - RP, x0 = 2 * pi - 2;
  const int i0 = (ry + 2) * TW + (x0 + 2);
  const int dxc = reg16(x0), dyc = reg16(ry);
  const int sxy = (dxc + 1) + 3 * (dyc + 1);
  const int fxy = (ry - PB * dyc) * PB + (x0 - PB * dxc);
  double2* sfme = sf + tid;
  double* sxme = sxr + (ry + 1) * SXW + pi;
  // coarse pair: even row, even column inside the block (RP = 0 warps only)
  const bool cthr = RP == 0 && valid && pi >= 1 && pi <= 8 && ry <= 14;
  const int qx = pi - 1, qy = ry >> 1;

  const double* ip[NLD];
  const double* fp = nullptr;
  auto seek_issue = [&](int z) {
    int k, dz, zl;
    plane_src(z, nz, len, k, dz, zl);
    const int o = zl * (PB * PB);
#pragma unroll
    for (int d = 0; d < NLD; ++d)
      ip[d] = ld_sxy[d] < 0 ? nullptr : L.u + (size_t)snb[k * 27 + ld_sxy[d] + 9 * (dz + 1)] * PB3 + o + ld_xy[d];
    fp = L.f + (size_t)snb[k * 27 + sxy + 9 * (dz + 1)] * PB3 + o + fxy;
  };
  // stage plane z (called for z = -2, -1, … in order) into ring slot (z+2) & (R-1)
  auto issue = [&](int z, auto checked) {
    if (!decltype(checked)::value || z < nz + 2) {
      if ((z & 15) == 0) seek_issue(z);
      const int slot = (z + 2) & (R - 1);
#pragma unroll
      for (int d = 0; d < NLD; ++d) {
        if (ld_sxy[d] < 0) continue;
        cpa16(su + slot * TP + ld_dst[d], ip[d]);
        ip[d] += PB * PB;
      }
      if (valid && (!decltype(checked)::value || (z >= -1 && z <= nz))) cpa16(sfme + slot * NT, fp);
      fp += PB * PB;
    }
    cpa_commit();
  };
  bool live = false;
  auto seek_live = [&](int z) {
    int k, dz, zl;
    plane_src(z, nz, len, k, dz, zl);
    live = valid && ((sreal[k] >> (sxy + 9 * (dz + 1))) & 1u);
  };
  seek_issue(-2);
  seek_live(-1);
#pragma unroll
  for (int q = 0; q < D; ++q) issue(-2 + q, std::true_type{});

  double aA[2] = {0, 0}, aP[2] = {0, 0};  // per column: α(s-1); α(s-2) + β(s-1)
  double sxp = 0.0;                       // this pair's x-weighted residual at plane s-2
  double t0 = 0, t1 = 0, t2 = 0;          // coarse pairs: y-weighted sums at planes s-2, s-3, s-4
  const double h6 = ORDER == 4 ? inv_h2 * (1.0 / 6.0) : ORDER == 6 ? inv_h2 * (1.0 / 30.0) : inv_h2;
  // per column: α = 2c + S4, β = 2S4 + D4 - 24c (M = 4, times 6h^2); α = 14c + 3S4 + D4,
  // β = 14S4 + 3D4 - 128c (M = 6, times 30h^2; the corners enter through D4 in α)
  auto alpha_of = [&](double c, double s4, double d4) {
    return ORDER == 4 ? 2.0 * c + s4 : ORDER == 6 ? (14.0 * c + 3.0 * s4) + d4 : c;
  };
  auto beta_of = [&](double c, double s4, double d4) {
    return ORDER == 4 ? 2.0 * s4 + d4 - 24.0 * c : ORDER == 6 ? (14.0 * s4 + 3.0 * d4) - 128.0 * c : s4 - 6.0 * c;
  };
  // Steps s = -2 … nz+1 (the last coarse node, fine plane nz-2, needs residual planes
  // up to nz-1) in groups of 4, s = base-2+j with base a multiple of 4: ring slots,
  // plane parities and block-boundary tests are compile-time; only the first and last
  // groups test the pencil ends.
  auto group = [&](const int base, auto mode) {
    constexpr bool EDGE = decltype(mode)::value != 1, LAST = decltype(mode)::value == 2;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int s = base - 2 + j;
      cpa_wait<D - 1>();
      __syncthreads();
      issue(s + D, std::integral_constant<bool, LAST>{});
      // plane s (shuffles: every lane takes part)
      const double* U = su + ((s + 2) & (R - 1)) * TP + i0;
      const double2 m = *reinterpret_cast<const double2*>(U - TW);
      const double2 cc = *reinterpret_cast<const double2*>(U);
      const double2 p = *reinterpret_cast<const double2*>(U + TW);
      const double l = shfl_up1(cc.y), r = shfl_dn1(cc.x);
      const double qxs = m.x + p.x, qys = m.y + p.y;  // rows y±1 per column (diagonals: one shuffle)
      double cq[2] = {cc.x, cc.y};
      double s4q[2] = {(l + cc.y) + qxs, (cc.x + r) + qys};
      double d4q[2] = {0, 0};
      if (ORDER >= 4) {
        d4q[0] = shfl_up1(qys) + qys;
        d4q[1] = qxs + shfl_dn1(qxs);
      }
      double sxc = 0.0;
      if (!EDGE || s >= 0) {  // residual at plane s-1 in [-1, nz]
        if (((s - 1) & 15) == 0) seek_live(s - 1);
        const double2 fq = sfme[((s + 1) & (R - 1)) * NT];
        double2 rr = make_double2(0.0, 0.0);  // r := 0 outside the level's blocks (Z14)
        if (live) {
          rr.x = fq.x - (aP[0] + alpha_of(cq[0], s4q[0], d4q[0])) * h6;
          rr.y = fq.y - (aP[1] + alpha_of(cq[1], s4q[1], d4q[1])) * h6;
        }
        // full weighting along x at this pair's even column x0: r(x0-1) is the left
        // lane's second column (the definition's order: 0.25 r(-1) + 0.5 r(0) + 0.25 r(1))
        const double rl = shfl_up1(rr.y);
        sxc = 0.25 * rl + 0.5 * rr.x + 0.25 * rr.y;
        if (valid) sxme[((s - 1) & 1) * SXP] = sxc;
      }
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        aP[q] = aA[q] + beta_of(cq[q], s4q[q], d4q[q]);  // α(s-1) + β(s): the node at s, completed at step s+1
        aA[q] = alpha_of(cq[q], s4q[q], d4q[q]);
      }
      if (cthr) {
        // coarse u = fine u(2i) at even interior planes (E7): this pair's centre value
        if ((j & 1) == 0 && (!EDGE || (s >= 0 && s < nz))) {
          const int k = s >> 4, qz = (s & 15) >> 1;
          const int* pr = spar + 4 * k;
          C.u[(size_t)pr[0] * C.B3 + ((pr[3] + qz) * C.B + (pr[2] + qy)) * C.B + (pr[1] + qx)] = cq[0];
        }
        // full weighting of the residual plane s-2 along y (rows y±1 written last step,
        // row y this pair's own), then along z
        if (!EDGE || s >= 1) {
          const double* rp = sxme + ((s - 2) & 1) * SXP;
          double sy = 0.0;
          sy += 0.25 * rp[-SXW];
          sy += 0.5 * sxp;
          sy += 0.25 * rp[SXW];
          t2 = t1; t1 = t0; t0 = sy;
          const int zc = s - 3;  // even when j is odd
          if ((j & 1) == 1 && zc >= 0 && zc < nz) {
            const double sz = (0.25 * t2 + 0.5 * t1) + 0.25 * t0;
            const int k = zc >> 4, qz = (zc & 15) >> 1;
            const int* pr = spar + 4 * k;
            C.r[(size_t)pr[0] * C.B3 + ((pr[3] + qz) * C.B + (pr[2] + qy)) * C.B + (pr[1] + qx)] = sz;
          }
        }
      }
      sxp = sxc;
    }
  };
  const int nt = (nz + 4) >> 2;
  group(0, std::integral_constant<int, 0>{});
  for (int t = 1; t < nt - 1; ++t) group(4 * t, std::integral_constant<int, 1>{});
  group(4 * (nt - 1), std::integral_constant<int, 2>{});
  cpa_wait<0>();
}

template <int ORDER>
__global__ void __maxnreg__(80)
    k_rr2_pencil(LevelView L, LevelView C, double inv_h2) {
  using S = RR2Shape;
  comp_view(L);
  comp_view(C);
  constexpr int T = S::T, TW = S::TW, NT = S::NT, NLD = S::NLD;
  extern __shared__ __align__(16) double sm[];
  __shared__ int snb[PMAXL * 27];
  __shared__ uint32_t sreal[PMAXL];
  __shared__ int spar[PMAXL * 4];
  const int tid = threadIdx.x;
  const int len = __ldg(L.pen_len + blockIdx.x);
  const int32_t* pb = L.pen_blk + (size_t)blockIdx.x * L.pen_lmax;
  for (int i = tid; i < len * 27; i += NT) snb[i] = __ldg(L.nbr + (size_t)__ldg(pb + i / 27) * 27 + i % 27);
  if (tid < len) sreal[tid] = __ldg(L.nbr_real + __ldg(pb + tid));
  if (tid < 4 * len) spar[tid] = __ldg(L.parent + 4 * (size_t)__ldg(pb + tid / 4) + tid % 4);
  // u load items (interior 128-byte lines first, then halo pieces), as in the RB sweep
  int ld_xy[2], ld_sxy[2], ld_dst[2];
#pragma unroll
  for (int d = 0; d < NLD; ++d) {
    const int j = tid + d * NT;
    int py, px;
    if (j < 8 * T) {
      py = j / 8;
      px = 2 + 2 * (j % 8);
    } else {
      const int hh = j - 8 * T;
      py = hh / 2;
      px = (hh & 1) ? PB + 2 : 0;
    }
    const int x = px - 2, y = py - 2, dx = reg16(x), dy = reg16(y);
    ld_xy[d] = (y - PB * dy) * PB + (x - PB * dx);
    ld_sxy[d] = j < S::NPAIR ? (dx + 1) + 3 * (dy + 1) : -1;
    ld_dst[d] = py * TW + px;
  }
  __syncthreads();
  const int w = tid >> 5, lane = tid & 31;
  if (w < 3) rr2_body<ORDER, 0>(L, C, snb, sreal, spar, sm, ld_xy, ld_sxy, ld_dst, w, lane, len, inv_h2);
  else rr2_body<ORDER, 1>(L, C, snb, sreal, spar, sm, ld_xy, ld_sxy, ld_dst, w - 3, lane, len, inv_h2);
}

bool launch_res_restrict_pencil(const LevelView& fine, const LevelView& coarse, int order, cudaStream_t s) {
  if (fine.B != PB || fine.npen <= 0 || fine.pen_lmax > PMAXL) return false;
  const double inv_h2 = 1.0 / (fine.h * fine.h);
  if (order == 2) k_rr2_pencil<2><<<dim3(fine.npen, fine.nc), RR2Shape::NT, RR2Shape::SMEM, s>>>(fine, coarse, inv_h2);
  else if (order == 4) k_rr2_pencil<4><<<dim3(fine.npen, fine.nc), RR2Shape::NT, RR2Shape::SMEM, s>>>(fine, coarse, inv_h2);
  else k_rr2_pencil<6><<<dim3(fine.npen, fine.nc), RR2Shape::NT, RR2Shape::SMEM, s>>>(fine, coarse, inv_h2);
  note_launch();
  return true;
}

// ---------------------------------------------------------------------------------
constexpr int RES_D = 3;

// RB sweep variant (prefetch depth D, ring R, register cap): cfg2 256^3 finest sweep on
// B200 (tools/time_ops.py): <2,4,80> 108.7 us (4 CTAs/SM), <2,4,96> 116.5, <5,8,96> 120.9,
// <2,4,72> 124.6 (spills), <3,8,80> 129.4 (smem: 3 CTAs/SM), <3,5,80> 115.3, <4,6,80>
// 112.9, <3,6,80> 116.7 us (deeper rings do not help).  After the 4-step-group rewrite:
// <2,4,80> 96.8 us, <2,4,72> 102.4 (spills, still 4 CTAs/SM), <2,4,64> 100.6 (5 CTAs/SM,
// 88 B of spills).
constexpr int RB_D = 2, RB_R = 4, RB_NREG = 80;
using RBS = RBShape<RB_D, RB_R, false>;
using RBT = RBShape<RB_D, RB_R, true>;

bool encode_tile_maps(const double* base, int ntot, CUtensorMap out[4]) {
  static PFN_cuTensorMapEncodeTiled_v12000 enc = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }();
  if (!enc || !base || ntot <= 0) return false;
  const cuuint64_t dims[4] = {PB, PB, PB, (cuuint64_t)ntot};
  const cuuint64_t strides[3] = {PB * sizeof(double), PB * PB * sizeof(double), (cuuint64_t)PB3 * sizeof(double)};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  for (int mi = 0; mi < 4; ++mi) {
    const cuuint32_t box[4] = {(mi & 1) ? 2u : 16u, (mi & 2) ? 2u : 16u, 1u, 1u};
    if (enc(&out[mi], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  return true;
}

void prepare_pencil_kernels() {
  // the whole unified L1 as shared memory: several pencil CTAs per SM
  auto setup = [](const void* k, size_t smem) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  };
  setup((const void*)k_rb_pencil<2, RB_D, RB_R, RB_NREG, false, false>, RBS::SMEM);
  setup((const void*)k_rb_pencil<4, RB_D, RB_R, RB_NREG, false, false>, RBS::SMEM);
  setup((const void*)k_rb_pencil<2, RB_D, RB_R, RB_NREG, true, false>, RBS::SMEM);
  setup((const void*)k_rb_pencil<4, RB_D, RB_R, RB_NREG, true, false>, RBS::SMEM);
  setup((const void*)k_rb_pencil<2, RB_D, RB_R, RB_NREG, false, true>, RBT::SMEM);
  setup((const void*)k_rb_pencil<4, RB_D, RB_R, RB_NREG, false, true>, RBT::SMEM);
  setup((const void*)k_rb_pencil<2, RB_D, RB_R, RB_NREG, true, true>, RBT::SMEM);
  setup((const void*)k_rb_pencil<4, RB_D, RB_R, RB_NREG, true, true>, RBT::SMEM);
  setup((const void*)k_rb6_pencil<RB6_NREG, false>, RB6Shape::SMEM);
  setup((const void*)k_rb6_pencil<RB6_NREG, true>, RB6Shape::SMEM);
  setup((const void*)k_rr2_pencil<2>, RR2Shape::SMEM);
  setup((const void*)k_rr2_pencil<4>, RR2Shape::SMEM);
  setup((const void*)k_rr2_pencil<6>, RR2Shape::SMEM);
  setup((const void*)k_res_pencil<2, RES_D, 0>, ResShape<RES_D>::SMEM);
  setup((const void*)k_res_pencil<2, RES_D, 1>, ResShape<RES_D>::SMEM);
  setup((const void*)k_res_pencil<2, RES_D, 2>, ResShape<RES_D>::SMEM);
  setup((const void*)k_res_pencil<4, RES_D, 0>, ResShape<RES_D>::SMEM);
  setup((const void*)k_res_pencil<4, RES_D, 1>, ResShape<RES_D>::SMEM);
  setup((const void*)k_res_pencil<4, RES_D, 2>, ResShape<RES_D>::SMEM);
  setup((const void*)k_res_pencil<6, RES_D, 0>, ResShape<RES_D>::SMEM);
  setup((const void*)k_res_pencil<6, RES_D, 1>, ResShape<RES_D>::SMEM);
  setup((const void*)k_res_pencil<6, RES_D, 2>, ResShape<RES_D>::SMEM);
  setup((const void*)k_res_pencil<4, RES_D, 3>, ResShape<RES_D>::SMEM);
}

// residual-type pencil launch (MODE 0 residual, 1 FAS right-hand side, 2 norm)
template <int MODE>
static bool res_pencil_launch(const LevelView& L, int order, unsigned long long* out, cudaStream_t s) {
  if (L.B != PB || L.npen <= 0 || L.pen_lmax > PMAXL) return false;
  const double inv_h2 = 1.0 / (L.h * L.h);
  constexpr int NT = ResShape<RES_D>::NT;
  constexpr size_t SM = ResShape<RES_D>::SMEM;
  if (order == 2) k_res_pencil<2, RES_D, MODE><<<dim3(L.npen, L.nc), NT, SM, s>>>(L, inv_h2, out);
  else if (order == 4) k_res_pencil<4, RES_D, MODE><<<dim3(L.npen, L.nc), NT, SM, s>>>(L, inv_h2, out);
  else k_res_pencil<6, RES_D, MODE><<<dim3(L.npen, L.nc), NT, SM, s>>>(L, inv_h2, out);
  note_launch();
  return true;
}

bool launch_rb_pencil(const LevelView& L, int order, double omega, const TileMaps* tm, cudaStream_t s) {
  if (L.B != PB || L.npen <= 0 || L.pen_lmax > PMAXL) return false;
  if (order == 6) {
    const double inv_h2 = 1.0 / (L.h * L.h);
    const double inv_d = 1.0 / ((-128.0 / 30.0) * inv_h2);
    if (L.sw_npen > 0) k_rb6_pencil<RB6_NREG, true><<<dim3(L.sw_npen, L.nc), 192, RB6Shape::SMEM, s>>>(L, omega, inv_h2, inv_d);
    else k_rb6_pencil<RB6_NREG, false><<<dim3(L.npen, L.nc), 192, RB6Shape::SMEM, s>>>(L, omega, inv_h2, inv_d);
    note_launch();
    return true;
  }
  const double inv_h2 = 1.0 / (L.h * L.h);
  const double inv_d = 1.0 / ((order == 2 ? -6.0 : -4.0) * inv_h2);
  const int grid = L.sw_npen > 0 ? L.sw_npen : L.npen;
  // tile staging by TMA (tensor maps given) or by cp.async
  static const TileMaps none{};
  const TileMaps& m = tm ? *tm : none;
  if (tm) {
    if (L.sw_npen > 0)
      (order == 2 ? k_rb_pencil<2, RB_D, RB_R, RB_NREG, true, true> : k_rb_pencil<4, RB_D, RB_R, RB_NREG, true, true>)
          <<<dim3(grid, L.nc), RBT::NT, RBT::SMEM, s>>>(L, omega, inv_h2, inv_d, m);
    else
      (order == 2 ? k_rb_pencil<2, RB_D, RB_R, RB_NREG, false, true> : k_rb_pencil<4, RB_D, RB_R, RB_NREG, false, true>)
          <<<dim3(grid, L.nc), RBT::NT, RBT::SMEM, s>>>(L, omega, inv_h2, inv_d, m);
  } else if (L.sw_npen > 0) {
    (order == 2 ? k_rb_pencil<2, RB_D, RB_R, RB_NREG, true, false> : k_rb_pencil<4, RB_D, RB_R, RB_NREG, true, false>)
        <<<dim3(grid, L.nc), RBS::NT, RBS::SMEM, s>>>(L, omega, inv_h2, inv_d, m);
  } else {
    (order == 2 ? k_rb_pencil<2, RB_D, RB_R, RB_NREG, false, false> : k_rb_pencil<4, RB_D, RB_R, RB_NREG, false, false>)
        <<<dim3(grid, L.nc), RBS::NT, RBS::SMEM, s>>>(L, omega, inv_h2, inv_d, m);
  }
  note_launch();
  return true;
}

bool launch_rhs_pencil(const LevelView& L, int order, cudaStream_t s) {
  if (order != 4 || L.B != PB || L.npen <= 0 || L.pen_lmax > PMAXL) return false;
  const double inv_h2 = 1.0 / (L.h * L.h);
  k_res_pencil<4, RES_D, 3><<<dim3(L.npen, L.nc), ResShape<RES_D>::NT, ResShape<RES_D>::SMEM, s>>>(L, inv_h2, nullptr);
  note_launch();
  return true;
}

bool launch_fas_pencil(const LevelView& L, int order, cudaStream_t s) {
  return res_pencil_launch<1>(L, order, nullptr, s);
}

bool launch_res_pencil(const LevelView& L, int order, cudaStream_t s) { return res_pencil_launch<0>(L, order, nullptr, s); }

bool launch_norm_pencil(const LevelView& L, int order, unsigned long long* out, cudaStream_t s) {
  return res_pencil_launch<2>(L, order, out, s);
}

}  // namespace mg
