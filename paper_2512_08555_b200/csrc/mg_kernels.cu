// mg_kernels.cu — sm_100a kernels of the adaptive FAS V-cycle (Alg. 1).
//
// Data layout: each level stores fields as [ntot][B^3] fp64
// blocks, x fastest.  A block's 26 neighbours come from a per-block table; a
// neighbour that is not a real block of the level is a *ghost block* whose
// needed nodes hold boundary-ghost values (c2f at resolution jumps, exterior
// band), so every stencil kernel reads halos uniformly through the table.
//
// All arithmetic is fp64 on the CUDA cores: the path is HBM-bound (≈1 flop/B),
// so there is no tensor-core work here by design (north star).
#include <cuComplex.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "mg_internal.h"

namespace mg {

static unsigned long long g_nlaunch = 0;  // kernels launched by this library (bench evidence)

unsigned long long launches_issued() { return g_nlaunch; }
void note_launch() { ++g_nlaunch; }

__device__ __forceinline__ int region(int x, int B) { return x < 0 ? -1 : (x >= B ? 1 : 0); }

// Value of a level field at block-local coords (x,y,z) in [-B, 2B) of block `b`.
__device__ __forceinline__ double fetch(const double* __restrict__ a, const int32_t* __restrict__ nb, int B,
                                        int x, int y, int z) {
  const int dx = region(x, B), dy = region(y, B), dz = region(z, B);
  const int blk = __ldg(nb + (dx + 1) + 3 * (dy + 1) + 9 * (dz + 1));
  return a[(size_t)blk * (B * B * B) + ((z - dz * B) * B + (y - dy * B)) * B + (x - dx * B)];
}

// ---------------------------------------------------------------------------------
// Stencils on a shared-memory tile (strides 1, T, T*T).  M=2: cross stencil E8;
// M=4: 19-point Mehrstellen E12 (fig:stencils, weights {-24, 2, 1}/6).
// ---------------------------------------------------------------------------------
template <int ORDER, int T>
__device__ __forceinline__ double lap_tile(const double* t, int i, double inv_h2) {
  constexpr int SY = T, SZ = T * T;
  const double c = t[i];
  const double F = ((t[i - 1] + t[i + 1]) + (t[i - SY] + t[i + SY])) + (t[i - SZ] + t[i + SZ]);
  if (ORDER == 2) return (F - 6.0 * c) * inv_h2;
  const double E = (((t[i - 1 - SY] + t[i + 1 - SY]) + (t[i - 1 + SY] + t[i + 1 + SY])) +
                    ((t[i - 1 - SZ] + t[i + 1 - SZ]) + (t[i - 1 + SZ] + t[i + 1 + SZ]))) +
                   ((t[i - SY - SZ] + t[i + SY - SZ]) + (t[i - SY + SZ] + t[i + SY + SZ]));
  if (ORDER == 4) return (2.0 * F + E - 24.0 * c) * (inv_h2 * (1.0 / 6.0));
  // M = 6 (E13, fig:stencils: centre -128, faces 14, edges 3, corners 1, / 30h^2)
  const double K = ((t[i - 1 - SY - SZ] + t[i + 1 - SY - SZ]) + (t[i - 1 + SY - SZ] + t[i + 1 + SY - SZ])) +
                   ((t[i - 1 - SY + SZ] + t[i + 1 - SY + SZ]) + (t[i - 1 + SY + SZ] + t[i + 1 + SY + SZ]));
  return ((14.0 * F + 3.0 * E + K) - 128.0 * c) * (inv_h2 * (1.0 / 30.0));
}

template <int ORDER>
__device__ __forceinline__ double lap_fetch(const double* __restrict__ u, const int32_t* __restrict__ nb, int B,
                                            int x, int y, int z, double inv_h2) {
  auto g = [&](int a, int b, int c) { return fetch(u, nb, B, x + a, y + b, z + c); };
  const double c = g(0, 0, 0);
  const double F = ((g(-1, 0, 0) + g(1, 0, 0)) + (g(0, -1, 0) + g(0, 1, 0))) + (g(0, 0, -1) + g(0, 0, 1));
  if (ORDER == 2) return (F - 6.0 * c) * inv_h2;
  const double E = (((g(-1, -1, 0) + g(1, -1, 0)) + (g(-1, 1, 0) + g(1, 1, 0))) +
                    ((g(-1, 0, -1) + g(1, 0, -1)) + (g(-1, 0, 1) + g(1, 0, 1)))) +
                   ((g(0, -1, -1) + g(0, 1, -1)) + (g(0, -1, 1) + g(0, 1, 1)));
  if (ORDER == 4) return (2.0 * F + E - 24.0 * c) * (inv_h2 * (1.0 / 6.0));
  const double K = ((g(-1, -1, -1) + g(1, -1, -1)) + (g(-1, 1, -1) + g(1, 1, -1))) +
                   ((g(-1, -1, 1) + g(1, -1, 1)) + (g(-1, 1, 1) + g(1, 1, 1)));
  return ((14.0 * F + 3.0 * E + K) - 128.0 * c) * (inv_h2 * (1.0 / 30.0));
}

// ---------------------------------------------------------------------------------
// Fused smoother (+ residual).  One CTA per real block.  The block and a halo of
// H = (#update passes) + (residual ? 1 : 0) nodes are staged in shared memory;
// each pass updates the live nodes (own block or real neighbour block; ghost-block
// nodes are frozen, reading Z9) of a region that shrinks by one node per pass, so
// red, black and the residual all come out of one HBM read of u and f.
// Jacobi: u += ω (f - Δu)/d on all nodes of the region from the snapshot.
// RB:     red (even level-global parity) then black, each from a snapshot (Z10).
// The smoothed block goes to u_out (ping-pong: neighbours read the old u).
// ---------------------------------------------------------------------------------
template <int B, int ORDER, int MODE, bool RES, int NT>
__global__ void __launch_bounds__(NT) k_smooth(LevelView L, double omega, double inv_h2, double inv_d) {
  comp_view(L);
  constexpr int NS = MODE == SM_RB ? 2 : (MODE == SM_JACOBI ? 1 : 0);
  constexpr int H = NS + (RES ? 1 : 0);
  constexpr int T = B + 2 * H;
  constexpr int B3 = B * B * B;
  // staged updates per thread for the largest pass
  constexpr int R0 = B + 2 * (H - 1);
  constexpr int MAXU = MODE == SM_RB ? (R0 * R0 * R0 / 2 + NT - 1) / NT : (R0 * R0 * R0 + NT - 1) / NT;
  extern __shared__ double tile[];
  const int b = blockIdx.x;
  const int32_t* nb = L.nbr + (size_t)b * 27;
  const uint32_t realbits = L.nbr_real[b];

  for (int i = threadIdx.x; i < T * T * T; i += NT) {
    const int x = i % T - H, y = (i / T) % T - H, z = i / (T * T) - H;
    tile[i] = fetch(L.u, nb, B, x, y, z);
  }
  __syncthreads();

#pragma unroll
  for (int p = 0; p < NS; ++p) {
    const int e = H - 1 - p;  // region [-e, B+e)^3
    const int R = B + 2 * e;
    const int colour = p;     // RB: pass 0 = red (even), pass 1 = black (odd)
    const int cnt = MODE == SM_RB ? R * R * R / 2 : R * R * R;
    double stage[MAXU];
#pragma unroll
    for (int k = 0; k < MAXU; ++k) {
      const int i = threadIdx.x + k * NT;
      stage[k] = 0.0;
      if (i < cnt) {
        int x, y, z;
        if (MODE == SM_RB) {
          const int R2 = R / 2;
          z = i / (R * R2);
          const int rem = i - z * R * R2;
          y = rem / R2;
          const int xi = rem - y * R2;
          x = 2 * xi + ((colour + y + z + e) & 1);
        } else {
          z = i / (R * R);
          const int rem = i - z * R * R;
          y = rem / R;
          x = rem - y * R;
        }
        x -= e; y -= e; z -= e;
        const int s = (region(x, B) + 1) + 3 * (region(y, B) + 1) + 9 * (region(z, B) + 1);
        if ((realbits >> s) & 1u) {
          const int ti = ((z + H) * T + (y + H)) * T + (x + H);
          const double c = tile[ti];
          const double f = fetch(L.f, nb, B, x, y, z);
          stage[k] = c + omega * (f - lap_tile<ORDER, T>(tile, ti, inv_h2)) * inv_d;
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < MAXU; ++k) {
      const int i = threadIdx.x + k * NT;
      if (i < cnt) {
        int x, y, z;
        if (MODE == SM_RB) {
          const int R2 = R / 2;
          z = i / (R * R2);
          const int rem = i - z * R * R2;
          y = rem / R2;
          const int xi = rem - y * R2;
          x = 2 * xi + ((colour + y + z + e) & 1);
        } else {
          z = i / (R * R);
          const int rem = i - z * R * R;
          y = rem / R;
          x = rem - y * R;
        }
        x -= e; y -= e; z -= e;
        const int s = (region(x, B) + 1) + 3 * (region(y, B) + 1) + 9 * (region(z, B) + 1);
        if ((realbits >> s) & 1u) tile[((z + H) * T + (y + H)) * T + (x + H)] = stage[k];
      }
    }
    __syncthreads();
  }

  double* uo = (NS > 0) ? L.u_out + (size_t)b * B3 : nullptr;
  for (int i = threadIdx.x; i < B3; i += NT) {
    const int x = i % B, y = (i / B) % B, z = i / (B * B);
    const int ti = ((z + H) * T + (y + H)) * T + (x + H);
    if (NS > 0) uo[i] = tile[ti];
    if (RES) L.r[(size_t)b * B3 + i] = L.f[(size_t)b * B3 + i] - lap_tile<ORDER, T>(tile, ti, inv_h2);
  }
}

// ---------------------------------------------------------------------------------
// Optimised smoother for B = 16 blocks (the hot path).  Same semantics as k_smooth,
// with: the 27-entry neighbour table in shared memory; the halo tile loaded with
// cp.async (8-byte LDGSTS, no register staging); a colour-split tile layout (each
// tile row stores its even-x then its odd-x nodes) so that the red/black passes,
// whose lanes walk same-colour nodes two apart in x, read shared memory without
// bank conflicts; and f for each pass prefetched into registers before the barrier
// that precedes the pass.
// ---------------------------------------------------------------------------------
__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::); }

// Colour-split tile: the T^3 tile nodes are stored in two dense arrays by tile
// parity (x+y+z)&1, each row-major in (z, y, x>>1) with row pitch T/2.  The odd
// array starts at an offset ≡ 8 (mod 16) doubles, so a warp walking same-colour
// nodes of consecutive rows, or all nodes of a row, hits distinct 8-byte banks.
template <int T>
struct CTile {
  static constexpr int W = T / 2;
  static constexpr int HALF = T * T * T / 2;
  static constexpr int BOFF = HALF + ((8 - HALF % 16) % 16 + 16) % 16;
  static constexpr int SIZE = BOFF + HALF;  // doubles
};

// Δ_h^M at a node of a colour-split tile, given its packed position: rel = row-major
// index (z*T+y)*W + (x>>1) inside its colour array, q = tile parity, xpar = x & 1.
// All 19 operands are immediate offsets from four base pointers; same summation
// order as lap_tile.
template <int ORDER, int T>
__device__ __forceinline__ double lap_t(const double* t, int rel, int q, int xpar, double inv_h2) {
  constexpr int W = CTile<T>::W, SZ = T * W;
  const double* S = t + (q ? CTile<T>::BOFF : 0) + rel;  // same colour: centre, edges
  const double* O = t + (q ? 0 : CTile<T>::BOFF) + rel;  // other colour: faces
  const double* Om = O + xpar - 1;                       // (x-1) at Om[0], (x+1) at Om[1]
  const double* Sm = S + xpar - 1;
  const double c = S[0];
  const double F = ((Om[0] + Om[1]) + (O[-W] + O[W])) + (O[-SZ] + O[SZ]);
  if (ORDER == 2) return (F - 6.0 * c) * inv_h2;
  const double E = (((Sm[-W] + Sm[1 - W]) + (Sm[W] + Sm[1 + W])) + ((Sm[-SZ] + Sm[1 - SZ]) + (Sm[SZ] + Sm[1 + SZ]))) +
                   ((S[-W - SZ] + S[W - SZ]) + (S[-W + SZ] + S[W + SZ]));
  return (2.0 * F + E - 24.0 * c) * (inv_h2 * (1.0 / 6.0));
}

// ---- per-variant node tables (identical for every block, built once on the host) ----
// node entry: rel (bits 0-12) | q (13) | xpar (14) | neighbour slot (15-19) | offset in
// that neighbour block (20-31).  load entry: tile index (0-13) | slot (14-18) | offset (19-30).
template <int B, int MODE, bool RES>
struct SmoothShape {
  static constexpr int NS = MODE == SM_RB ? 2 : (MODE == SM_JACOBI ? 1 : 0);
  static constexpr int H = NS + (RES ? 1 : 0);
  static constexpr int T = B + 2 * H;
  static constexpr int B3 = B * B * B;
  // Pass p walks whole rows of the colour-split tile (RB: the W slots of the pass
  // colour's array; Jacobi: all T slots) over the R(p)^2 rows of its region, so that
  // consecutive lanes read consecutive shared-memory words; slots outside the region
  // are idle (invalid table entries).
  __host__ __device__ static constexpr int R(int p) { return B + 2 * (H - 1 - p); }
  __host__ __device__ static constexpr int CNT(int p) { return R(p) * R(p) * (MODE == SM_RB ? T / 2 : T); }
  __host__ __device__ static constexpr int OFF(int p) { return p == 0 ? 0 : OFF(p - 1) + CNT(p - 1); }
  static constexpr int INT_OFF = NS > 0 ? OFF(NS - 1) + CNT(NS - 1) : 0;              // interior, x fastest
  static constexpr int LOAD_OFF = INT_OFF + B3;
  static constexpr int TOTAL = LOAD_OFF + T * T * T;
};

static int host_region(int x, int B) { return x < 0 ? -1 : (x >= B ? 1 : 0); }

template <int B, int MODE, bool RES>
static const uint32_t* smooth_table() {
  using S = SmoothShape<B, MODE, RES>;
  static uint32_t* d = nullptr;
  if (d) return d;
  constexpr int T = S::T, H = S::H, W = CTile<T>::W;
  std::vector<uint32_t> t;
  t.reserve(S::TOTAL);
  auto node = [&](int x, int y, int z) {  // block-local coords (halo allowed)
    const int tx = x + H, ty = y + H, tz = z + H;
    const int dx = host_region(x, B), dy = host_region(y, B), dz = host_region(z, B);
    const uint32_t rel = (uint32_t)((tz * T + ty) * W + (tx >> 1));
    const uint32_t q = (uint32_t)((tx + ty + tz) & 1), xpar = (uint32_t)(tx & 1);
    const uint32_t slot = (uint32_t)((dx + 1) + 3 * (dy + 1) + 9 * (dz + 1));
    const uint32_t floc = (uint32_t)(((z - dz * B) * B + (y - dy * B)) * B + (x - dx * B));
    return rel | (q << 13) | (xpar << 14) | (slot << 15) | (floc << 20);
  };
  for (int p = 0; p < S::NS; ++p) {
    const int e = H - 1 - p;
    for (int z = -e; z < B + e; ++z)
      for (int y = -e; y < B + e; ++y) {
        const int ty = y + H, tz = z + H;
        for (int s = 0; s < (MODE == SM_RB ? W : T); ++s) {
          // RB: slot s of the colour-p row holds tile x with parity making (x+y+z) even for
          // red (p = 0, global parity) / odd for black; Jacobi: tile x = s
          int tx = s;
          if (MODE == SM_RB) {
            const int want = ((p & 1) + H) & 1;  // tile parity of the pass colour
            tx = 2 * s + ((want - ty - tz) & 1);
          }
          const int x = tx - H;
          if (x >= -e && x < B + e) t.push_back(node(x, y, z));
          else t.push_back(0xffffffffu);
        }
      }
  }
  for (int i = 0; i < S::B3; ++i) t.push_back(node(i % B, (i / B) % B, i / (B * B)));
  for (int i = 0; i < T * T * T; ++i) {
    const int tx = i % T, ty = (i / T) % T, tz = i / (T * T);
    const uint32_t e = node(tx - H, ty - H, tz - H);
    const uint32_t dst = ((e >> 13) & 1u ? CTile<T>::BOFF : 0) + (e & 0x1fffu);
    t.push_back(dst | (((e >> 15) & 31u) << 14) | ((e >> 20) << 19));
  }
  if ((int)t.size() != S::TOTAL) return nullptr;
  cudaMalloc(&d, t.size() * sizeof(uint32_t));
  cudaMemcpy(d, t.data(), t.size() * sizeof(uint32_t), cudaMemcpyHostToDevice);
  return d;
}

template <int B, int ORDER, int MODE, bool RES, int NT>
__global__ void __launch_bounds__(NT, (MODE == SM_RB && RES) ? 2 : (MODE < 0 ? 4 : 3))
    k_smooth2(LevelView L, const uint32_t* __restrict__ tab, double omega, double inv_h2, double inv_d) {
  comp_view(L);
  using SH = SmoothShape<B, MODE, RES>;
  constexpr int NS = SH::NS, T = SH::T, B3 = SH::B3;
  constexpr int MAXU = (SH::CNT(0) + NT - 1) / NT;  // pass 0 is the largest
  constexpr int MAXR = (B3 + NT - 1) / NT;
  constexpr int MAXF = MAXU > MAXR ? MAXU : MAXR;
  extern __shared__ double tile[];
  __shared__ int snb[27];
  const int b = blockIdx.x;
  const int tid = threadIdx.x;
  if (tid < 27) snb[tid] = L.nbr[(size_t)b * 27 + tid];
  const uint32_t realbits = L.nbr_real[b];
  __syncthreads();

  // ---- async halo tile load (global reads coalesced along x)
  {
    const uint32_t* lt = tab + SH::LOAD_OFF;
#pragma unroll 4
    for (int i = tid; i < T * T * T; i += NT) {
      const uint32_t e = __ldg(lt + i);
      cp_async8(&tile[e & 0x3fffu], L.u + (size_t)snb[(e >> 14) & 31u] * B3 + (e >> 19));
    }
    asm volatile("cp.async.commit_group;\n" ::);
  }

  double fv[MAXF];
  auto prefetch = [&](int off, int cnt) {
#pragma unroll
    for (int k = 0; k < MAXF; ++k) {
      const int i = tid + k * NT;
      fv[k] = 0.0;
      if (i < cnt) {
        const uint32_t e = __ldg(tab + off + i);
        const uint32_t s = (e >> 15) & 31u;
        if (e != 0xffffffffu && ((realbits >> s) & 1u)) fv[k] = __ldg(L.f + (size_t)snb[s] * B3 + (e >> 20));
      }
    }
  };
  if (NS > 0) prefetch(SH::OFF(0), SH::CNT(0));
  cp_async_wait_all();
  __syncthreads();

#pragma unroll
  for (int p = 0; p < NS; ++p) {
    const int cnt = SH::CNT(p);
    const uint32_t* pt = tab + SH::OFF(p);
    double stage[MAXU];
    uint32_t ent[MAXU];
#pragma unroll
    for (int k = 0; k < MAXU; ++k) {
      const int i = tid + k * NT;
      stage[k] = 0.0;
      ent[k] = 0xffffffffu;
      if (i < cnt) {
        const uint32_t e = __ldg(pt + i);
        if (e != 0xffffffffu && ((realbits >> ((e >> 15) & 31u)) & 1u)) {
          ent[k] = e;
          const int rel = e & 0x1fff, q = (e >> 13) & 1, xp = (e >> 14) & 1;
          const double c = tile[(q ? CTile<T>::BOFF : 0) + rel];
          stage[k] = c + omega * (fv[k] - lap_t<ORDER, T>(tile, rel, q, xp, inv_h2)) * inv_d;
        }
      }
    }
    if (p + 1 < NS) prefetch(SH::OFF(p + 1), SH::CNT(p + 1));
    else if (RES) {
#pragma unroll
      for (int k = 0; k < MAXF; ++k) {
        const int i = tid + k * NT;
        fv[k] = i < B3 ? __ldg(L.f + (size_t)b * B3 + i) : 0.0;
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < MAXU; ++k) {
      const uint32_t e = ent[k];
      if (e != 0xffffffffu) tile[(((e >> 13) & 1u) ? CTile<T>::BOFF : 0) + (e & 0x1fffu)] = stage[k];
    }
    __syncthreads();
  }

  double* uo = L.u_out + (size_t)b * B3;
  const uint32_t* it = tab + SH::INT_OFF;
#pragma unroll
  for (int k = 0; k < MAXR; ++k) {
    const int i = tid + k * NT;
    if (i < B3) {
      const uint32_t e = __ldg(it + i);
      const int rel = e & 0x1fff, q = (e >> 13) & 1, xp = (e >> 14) & 1;
      if (NS > 0) uo[i] = tile[(q ? CTile<T>::BOFF : 0) + rel];
      if (RES) {
        const double fi = NS > 0 ? fv[k] : __ldg(L.f + (size_t)b * B3 + i);
        L.r[(size_t)b * B3 + i] = fi - lap_t<ORDER, T>(tile, rel, q, xp, inv_h2);
      }
    }
  }
}

template <int B, int ORDER, int MODE, bool RES>
static void smooth_inst_v1(const LevelView& L, double omega, double inv_h2, double inv_d, cudaStream_t s,
                           bool prepare_only);

template <int B, int ORDER, int MODE, bool RES>
static void smooth_inst(const LevelView& L, double omega, double inv_h2, double inv_d, cudaStream_t s,
                        bool prepare_only = false) {
  if constexpr (B == 16 && ORDER != 6) {
    constexpr int NT = 256;
    constexpr int NS = MODE == SM_RB ? 2 : (MODE == SM_JACOBI ? 1 : 0);
    constexpr int H = NS + (RES ? 1 : 0);
    constexpr int T = B + 2 * H;
    const size_t smem = sizeof(double) * CTile<T>::SIZE;
    auto k = k_smooth2<B, ORDER, MODE, RES, NT>;
    if (prepare_only) {
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      smooth_table<B, MODE, RES>();
      return;
    }
    const uint32_t* tab = smooth_table<B, MODE, RES>();
    if (L.nreal > 0) { k<<<dim3(L.nreal, L.nc), NT, smem, s>>>(L, tab, omega, inv_h2, inv_d); ++g_nlaunch; }
    return;
  }
  smooth_inst_v1<B, ORDER, MODE, RES>(L, omega, inv_h2, inv_d, s, prepare_only);
}

template <int B, int ORDER, int MODE, bool RES>
static void smooth_inst_v1(const LevelView& L, double omega, double inv_h2, double inv_d, cudaStream_t s,
                           bool prepare_only) {
  constexpr int NT = B >= 16 ? 256 : (B >= 8 ? 128 : 64);
  constexpr int NS = MODE == SM_RB ? 2 : (MODE == SM_JACOBI ? 1 : 0);
  constexpr int H = NS + (RES ? 1 : 0);
  constexpr int T = B + 2 * H;
  const size_t smem = sizeof(double) * T * T * T;
  auto k = k_smooth<B, ORDER, MODE, RES, NT>;
  if (prepare_only) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    return;
  }
  if (L.nreal > 0) { k<<<dim3(L.nreal, L.nc), NT, smem, s>>>(L, omega, inv_h2, inv_d); ++g_nlaunch; }
}

template <int B, int ORDER>
static void prepare_b() {
  LevelView L{};
  smooth_inst<B, ORDER, SM_RB, true>(L, 0, 0, 0, 0, true);
  smooth_inst<B, ORDER, SM_RB, false>(L, 0, 0, 0, 0, true);
  smooth_inst<B, ORDER, SM_JACOBI, true>(L, 0, 0, 0, 0, true);
  smooth_inst<B, ORDER, SM_JACOBI, false>(L, 0, 0, 0, 0, true);
  smooth_inst<B, ORDER, -1, true>(L, 0, 0, 0, 0, true);
}

template <int B, int ORDER>
static void smooth_dispatch_b(const LevelView& L, int mode, double omega, bool res, double inv_h2, double inv_d,
                              cudaStream_t s) {
  if (mode == SM_RB) {
    if (res) smooth_inst<B, ORDER, SM_RB, true>(L, omega, inv_h2, inv_d, s);
    else smooth_inst<B, ORDER, SM_RB, false>(L, omega, inv_h2, inv_d, s);
  } else if (mode == SM_JACOBI) {
    if (res) smooth_inst<B, ORDER, SM_JACOBI, true>(L, omega, inv_h2, inv_d, s);
    else smooth_inst<B, ORDER, SM_JACOBI, false>(L, omega, inv_h2, inv_d, s);
  } else {
    smooth_inst<B, ORDER, -1, true>(L, omega, inv_h2, inv_d, s);
  }
}

template <int ORDER>
static void smooth_dispatch(const LevelView& L, int mode, double omega, bool res, cudaStream_t s) {
  const double inv_h2 = 1.0 / (L.h * L.h);
  const double d = (ORDER == 2 ? -6.0 : (ORDER == 4 ? -4.0 : -128.0 / 30.0)) * inv_h2;  // centre of Δ_h^M
  const double inv_d = 1.0 / d;
  switch (L.B) {
    case 16: smooth_dispatch_b<16, ORDER>(L, mode, omega, res, inv_h2, inv_d, s); break;
    case 8: smooth_dispatch_b<8, ORDER>(L, mode, omega, res, inv_h2, inv_d, s); break;
    case 4: smooth_dispatch_b<4, ORDER>(L, mode, omega, res, inv_h2, inv_d, s); break;
    default: break;
  }
}

void prepare_kernels() {
  prepare_pencil_kernels();
  prepare_ghost_kernels();
  prepare_fft_kernels();
  prepare_b<16, 2>(); prepare_b<16, 4>(); prepare_b<16, 6>();
  prepare_b<8, 2>(); prepare_b<8, 4>(); prepare_b<8, 6>();
  prepare_b<4, 2>(); prepare_b<4, 4>(); prepare_b<4, 6>();
}

void launch_smooth(const LevelView& L, int order, int mode, double omega, bool with_residual, cudaStream_t s) {
  if (order == 2) smooth_dispatch<2>(L, mode, omega, with_residual, s);
  else if (order == 4) smooth_dispatch<4>(L, mode, omega, with_residual, s);
  else smooth_dispatch<6>(L, mode, omega, with_residual, s);
}

void launch_residual(const LevelView& L, int order, cudaStream_t s) {
  if (order == 2) smooth_dispatch<2>(L, -1, 0.0, true, s);
  else if (order == 4) smooth_dispatch<4>(L, -1, 0.0, true, s);
  else smooth_dispatch<6>(L, -1, 0.0, true, s);
}

__global__ void k_copy_list(int n, const int32_t* __restrict__ dst, const int32_t* __restrict__ src,
                            double* __restrict__ d, const double* __restrict__ sv, int64_t csd, int64_t css) {
  d += (int64_t)blockIdx.y * csd;
  sv += (int64_t)blockIdx.y * css;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) d[dst[i]] = sv[src[i]];
}

struct ChainFields {
  double* f[MAX_CHAIN_LEVELS];
  int64_t cs[MAX_CHAIN_LEVELS];
};

__global__ void k_copy_chain(int n, const int32_t* __restrict__ lev, const int32_t* __restrict__ dst,
                             const int32_t* __restrict__ src, ChainFields F) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const int l = lev[i];
    const int c = blockIdx.y;
    F.f[l & 15][c * F.cs[l & 15] + dst[i]] = F.f[l >> 4][c * F.cs[l >> 4] + src[i]];
  }
}

void launch_inject_chain(int n, const int32_t* lev, const int32_t* dst, const int32_t* src,
                         double* const fields[MAX_CHAIN_LEVELS], const int64_t cs[MAX_CHAIN_LEVELS], int nc,
                         cudaStream_t s) {
  if (n <= 0) return;
  ChainFields F;
  for (int j = 0; j < MAX_CHAIN_LEVELS; ++j) {
    F.f[j] = fields[j];
    F.cs[j] = cs[j];
  }
  k_copy_chain<<<dim3((n + 255) / 256, nc), 256, 0, s>>>(n, lev, dst, src, F);
  ++g_nlaunch;
}

void launch_inject_list(const InjList& l, double* coarse_field, const double* fine_field, int nc, int64_t cs_coarse,
                        int64_t cs_fine, cudaStream_t s) {
  if (l.n == 0) return;
  k_copy_list<<<dim3((l.n + 255) / 256, nc), 256, 0, s>>>(l.n, l.dst, l.src, coarse_field, fine_field, cs_coarse, cs_fine);
  ++g_nlaunch;
}

// ---------------------------------------------------------------------------------
// Restriction (Alg. 1): per fine real block, over the coarse sub-box it
// covers in its parent: u_c <- u_f(2i) (E7), r_c <- FW(r_f) (E6); r of ghost blocks
// is never written and stays 0 (reading Z14).
// ---------------------------------------------------------------------------------
__global__ void k_restrict(LevelView F, LevelView C) {
  comp_view(F);
  comp_view(C);
  const int b = blockIdx.x;
  const int B = F.B, Bh = B / 2;
  const int32_t* nb = F.nbr + (size_t)b * 27;
  const int p = F.parent[4 * b], ox = F.parent[4 * b + 1], oy = F.parent[4 * b + 2], oz = F.parent[4 * b + 3];
  for (int i = threadIdx.x; i < Bh * Bh * Bh; i += blockDim.x) {
    const int cx = i % Bh, cy = (i / Bh) % Bh, cz = i / (Bh * Bh);
    const int x = 2 * cx, y = 2 * cy, z = 2 * cz;
    const size_t ci = (size_t)p * C.B3 + ((oz + cz) * C.B + (oy + cy)) * C.B + (ox + cx);
    C.u[ci] = F.u[(size_t)b * F.B3 + (z * B + y) * B + x];
    double sz = 0.0;
    for (int dz = -1; dz <= 1; ++dz) {
      double sy = 0.0;
      for (int dy = -1; dy <= 1; ++dy) {
        const double sx = 0.25 * fetch(F.r, nb, B, x - 1, y + dy, z + dz) + 0.5 * fetch(F.r, nb, B, x, y + dy, z + dz) +
                          0.25 * fetch(F.r, nb, B, x + 1, y + dy, z + dz);
        sy += (dy == 0 ? 0.5 : 0.25) * sx;
      }
      sz += (dz == 0 ? 0.5 : 0.25) * sy;
    }
    C.r[ci] = sz;
  }
}

// Same operation with the fine residual tile (block + 1-node halo) staged in shared
// memory by cp.async; FW evaluated with the same nesting/rounding as k_restrict.
template <int B>
__global__ void __launch_bounds__(256) k_restrict2(LevelView F, LevelView C) {
  comp_view(F);
  comp_view(C);
  constexpr int T = B + 2, Bh = B / 2, B3 = B * B * B;
  __shared__ double rt[T * T * T];
  __shared__ int snb[27];
  const int b = blockIdx.x, tid = threadIdx.x;
  if (tid < 27) snb[tid] = F.nbr[(size_t)b * 27 + tid];
  __syncthreads();
  for (int i = tid; i < T * T * T; i += 256) {
    const int x = i % T - 1, y = (i / T) % T - 1, z = i / (T * T) - 1;
    const int dx = region(x, B), dy = region(y, B), dz = region(z, B);
    const int blk = snb[(dx + 1) + 3 * (dy + 1) + 9 * (dz + 1)];
    cp_async8(&rt[i], F.r + (size_t)blk * B3 + ((z - dz * B) * B + (y - dy * B)) * B + (x - dx * B));
  }
  asm volatile("cp.async.commit_group;\n" ::);
  const int p = F.parent[4 * b], ox = F.parent[4 * b + 1], oy = F.parent[4 * b + 2], oz = F.parent[4 * b + 3];
  double uinj[(Bh * Bh * Bh + 255) / 256];
#pragma unroll
  for (int k = 0; k < (Bh * Bh * Bh + 255) / 256; ++k) {
    const int i = tid + k * 256;
    if (i < Bh * Bh * Bh) {
      const int cx = i % Bh, cy = (i / Bh) % Bh, cz = i / (Bh * Bh);
      uinj[k] = __ldg(F.u + (size_t)b * B3 + ((2 * cz) * B + 2 * cy) * B + 2 * cx);
    }
  }
  cp_async_wait_all();
  __syncthreads();
#pragma unroll
  for (int k = 0; k < (Bh * Bh * Bh + 255) / 256; ++k) {
    const int i = tid + k * 256;
    if (i >= Bh * Bh * Bh) continue;
    const int cx = i % Bh, cy = (i / Bh) % Bh, cz = i / (Bh * Bh);
    const int x = 2 * cx + 1, y = 2 * cy + 1, z = 2 * cz + 1;  // tile coords of the coincident fine node
    double sz = 0.0;
#pragma unroll
    for (int dz = -1; dz <= 1; ++dz) {
      double sy = 0.0;
#pragma unroll
      for (int dy = -1; dy <= 1; ++dy) {
        const double* row = rt + ((z + dz) * T + (y + dy)) * T + x;
        const double sx = 0.25 * row[-1] + 0.5 * row[0] + 0.25 * row[1];
        sy += (dy == 0 ? 0.5 : 0.25) * sx;
      }
      sz += (dz == 0 ? 0.5 : 0.25) * sy;
    }
    const size_t ci = (size_t)p * C.B3 + ((oz + cz) * C.B + (oy + cy)) * C.B + (ox + cx);
    C.u[ci] = uinj[k];
    C.r[ci] = sz;
  }
}

void launch_restrict(const LevelView& fine, const LevelView& coarse, cudaStream_t s) {
  if (!fine.nreal) return;
  if (fine.B == 16) { k_restrict2<16><<<dim3(fine.nreal, fine.nc), 256, 0, s>>>(fine, coarse); ++g_nlaunch; }
  else { k_restrict<<<dim3(fine.nreal, fine.nc), 256, 0, s>>>(fine, coarse); ++g_nlaunch; }
}

// FAS right-hand side on the covered coarse nodes (Alg. 1): f = r + Δ u.
template <int ORDER>
__global__ void k_fas_rhs(LevelView F, LevelView C) {
  comp_view(F);
  comp_view(C);
  const int b = blockIdx.x;
  const int Bh = F.B / 2;
  const int p = F.parent[4 * b], ox = F.parent[4 * b + 1], oy = F.parent[4 * b + 2], oz = F.parent[4 * b + 3];
  const int32_t* nb = C.nbr + (size_t)p * 27;
  const double inv_h2 = 1.0 / (C.h * C.h);
  for (int i = threadIdx.x; i < Bh * Bh * Bh; i += blockDim.x) {
    const int x = ox + i % Bh, y = oy + (i / Bh) % Bh, z = oz + i / (Bh * Bh);
    const size_t ci = (size_t)p * C.B3 + (z * C.B + y) * C.B + x;
    C.f[ci] = C.r[ci] + lap_fetch<ORDER>(C.u, nb, C.B, x, y, z, inv_h2);
  }
}

void launch_fas_rhs(const LevelView& fine, const LevelView& coarse, int order, cudaStream_t s) {
  if (!fine.nreal) return;
  if (order == 2) { k_fas_rhs<2><<<dim3(fine.nreal, fine.nc), 256, 0, s>>>(fine, coarse); ++g_nlaunch; }
  else if (order == 4) { k_fas_rhs<4><<<dim3(fine.nreal, fine.nc), 256, 0, s>>>(fine, coarse); ++g_nlaunch; }
  else { k_fas_rhs<6><<<dim3(fine.nreal, fine.nc), 256, 0, s>>>(fine, coarse); ++g_nlaunch; }
}

// Prolongation of the correction (Alg. 1): u_f += trilinear(u_c - û_c).
__global__ void k_prolong(LevelView F, LevelView C) {
  comp_view(F);
  comp_view(C);
  const int b = blockIdx.x;
  const int B = F.B;
  const int p = F.parent[4 * b], ox = F.parent[4 * b + 1], oy = F.parent[4 * b + 2], oz = F.parent[4 * b + 3];
  const int32_t* nb = C.nbr + (size_t)p * 27;
  for (int i = threadIdx.x; i < F.B3; i += blockDim.x) {
    const int x = i % B, y = (i / B) % B, z = i / (B * B);
    const int cx = ox + (x >> 1), cy = oy + (y >> 1), cz = oz + (z >> 1);
    const int nx = (x & 1) ? 2 : 1, ny = (y & 1) ? 2 : 1, nzc = (z & 1) ? 2 : 1;
    double vz[2];
    for (int tz = 0; tz < nzc; ++tz) {
      double vy[2];
      for (int ty = 0; ty < ny; ++ty) {
        double vx[2];
        for (int tx = 0; tx < nx; ++tx) {
          const int X = cx + tx, Y = cy + ty, Z = cz + tz;
          const int slot = (region(X, C.B) + 1) + 3 * (region(Y, C.B) + 1) + 9 * (region(Z, C.B) + 1);
          // ε := 0 outside the coarse level's blocks (reading Z13-W)
          vx[tx] = (((C.nbr_real[p] | C.nbr_ext[p]) >> slot) & 1u)
                       ? fetch(C.u, nb, C.B, X, Y, Z) - fetch(C.uhat, nb, C.B, X, Y, Z) : 0.0;
        }
        vy[ty] = nx == 2 ? 0.5 * (vx[0] + vx[1]) : vx[0];
      }
      vz[tz] = ny == 2 ? 0.5 * (vy[0] + vy[1]) : vy[0];
    }
    const double e = nzc == 2 ? 0.5 * (vz[0] + vz[1]) : vz[0];
    double* uf = F.u + (size_t)b * F.B3 + i;
    *uf = *uf + e;
  }
}

// Same operation with ε = u_c - û_c on the (B/2+1)^3 coarse nodes under the fine
// block staged once in shared memory; same nesting/rounding as k_prolong.
template <int B>
__global__ void __launch_bounds__(256, 5) k_prolong2(LevelView F, LevelView C) {
  comp_view(F);
  comp_view(C);
  constexpr int E = B / 2 + 1, B3 = B * B * B;
  __shared__ double eps[E * E * E];
  __shared__ int snb[27];
  const int b = blockIdx.x, tid = threadIdx.x;
  const int p = F.parent[4 * b], ox = F.parent[4 * b + 1], oy = F.parent[4 * b + 2], oz = F.parent[4 * b + 3];
  if (tid < 27) snb[tid] = C.nbr[(size_t)p * 27 + tid];
  // prefetch the fine values this thread updates
  double uf[B3 / 256];
#pragma unroll
  for (int k = 0; k < B3 / 256; ++k) uf[k] = F.u[(size_t)b * B3 + tid + k * 256];
  __syncthreads();
  const int CB = C.B;
  // ε is taken on real coarse nodes and on the exterior band (U1); 0 at jump ghosts (Z13-W)
  const uint32_t creal = C.nbr_real[p] | C.nbr_ext[p];
  for (int i = tid; i < E * E * E; i += 256) {
    const int x = ox + i % E, y = oy + (i / E) % E, z = oz + i / (E * E);
    const int dx = region(x, CB), dy = region(y, CB), dz = region(z, CB);
    const int slot = (dx + 1) + 3 * (dy + 1) + 9 * (dz + 1);
    const size_t g = (size_t)snb[slot] * C.B3 + ((z - dz * CB) * CB + (y - dy * CB)) * CB + (x - dx * CB);
    // ε := 0 at coarse nodes outside the level's blocks (jump / exterior ghosts, reading Z13-W)
    eps[i] = ((creal >> slot) & 1u) ? __ldg(C.u + g) - __ldg(C.uhat + g) : 0.0;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < B3 / 256; ++k) {
    const int i = tid + k * 256;
    const int x = i % B, y = (i / B) % B, z = i / (B * B);
    const int cx = x >> 1, cy = y >> 1, cz = z >> 1;
    const int nx = (x & 1) ? 2 : 1, ny = (y & 1) ? 2 : 1, nzc = (z & 1) ? 2 : 1;
    double vz[2];
    for (int tz = 0; tz < nzc; ++tz) {
      double vy[2];
      for (int ty = 0; ty < ny; ++ty) {
        const double* row = eps + ((cz + tz) * E + (cy + ty)) * E + cx;
        vy[ty] = nx == 2 ? 0.5 * (row[0] + row[1]) : row[0];
      }
      vz[tz] = ny == 2 ? 0.5 * (vy[0] + vy[1]) : vy[0];
    }
    const double e = nzc == 2 ? 0.5 * (vz[0] + vz[1]) : vz[0];
    F.u[(size_t)b * B3 + i] = uf[k] + e;
  }
}

void launch_prolong(const LevelView& fine, const LevelView& coarse, cudaStream_t s) {
  if (!fine.nreal) return;
  if (fine.B == 16) { k_prolong2<16><<<dim3(fine.nreal, fine.nc), 256, 0, s>>>(fine, coarse); ++g_nlaunch; }
  else { k_prolong<<<dim3(fine.nreal, fine.nc), 256, 0, s>>>(fine, coarse); ++g_nlaunch; }
}

__global__ void k_inject_up(LevelView F, LevelView C, double* cu) {
  comp_view(F);
  cu += (int64_t)blockIdx.y * C.cs;
  const int b = blockIdx.x;
  const int B = F.B, Bh = B / 2;
  const int p = F.parent[4 * b], ox = F.parent[4 * b + 1], oy = F.parent[4 * b + 2], oz = F.parent[4 * b + 3];
  for (int i = threadIdx.x; i < Bh * Bh * Bh; i += blockDim.x) {
    const int cx = i % Bh, cy = (i / Bh) % Bh, cz = i / (Bh * Bh);
    cu[(size_t)p * C.B3 + ((oz + cz) * C.B + (oy + cy)) * C.B + (ox + cx)] =
        F.u[(size_t)b * F.B3 + ((2 * cz) * B + 2 * cy) * B + 2 * cx];
  }
}

void launch_inject_up(const LevelView& fine, const LevelView& coarse, double* coarse_u, cudaStream_t s) {
  if (fine.nreal) { k_inject_up<<<dim3(fine.nreal, fine.nc), 256, 0, s>>>(fine, coarse, coarse_u); ++g_nlaunch; }
}

// ---------------------------------------------------------------------------------
// Norms over leaf nodes (a9): max |f - Δu| (residual) or max |f| (‖f*‖∞); warp
// shuffle max, one 64-bit atomicMax per CTA on the bit pattern (non-negative
// doubles order like their bit patterns; NaN patterns sort above +Inf).
// ---------------------------------------------------------------------------------
template <int ORDER>
__global__ void k_norm(LevelView L, bool residual, unsigned long long* out) {
  comp_view(L);
  const int b = blockIdx.x;
  const int B = L.B, Bh = B / 2;
  const int32_t* nb = L.nbr + (size_t)b * 27;
  const uint8_t cov = L.covmask[b];
  const double inv_h2 = 1.0 / (L.h * L.h);
  unsigned long long m = 0ull;
  for (int i = threadIdx.x; i < L.B3; i += blockDim.x) {
    const int x = i % B, y = (i / B) % B, z = i / (B * B);
    const int oct = (x >= Bh) | ((y >= Bh) << 1) | ((z >= Bh) << 2);
    if ((cov >> oct) & 1) continue;
    double v = L.f[(size_t)b * L.B3 + i];
    if (residual) v -= lap_fetch<ORDER>(L.u, nb, B, x, y, z, inv_h2);
    v = fabs(v);
    unsigned long long bits = (unsigned long long)__double_as_longlong(v);
    if (v != v) bits = 0x7ff8000000000000ull;
    m = bits > m ? bits : m;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long t = __shfl_xor_sync(0xffffffffu, m, o);
    m = t > m ? t : m;
  }
  __shared__ unsigned long long sm[32];
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long r = 0ull;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r = sm[w] > r ? sm[w] : r;
    atomicMax(out, r);
  }
}

void launch_norm(const LevelView& L, int order, bool residual, unsigned long long* out, cudaStream_t s) {
  if (!L.nreal) return;
  if (order == 2) { k_norm<2><<<dim3(L.nreal, L.nc), 256, 0, s>>>(L, residual, out); ++g_nlaunch; }
  else if (order == 4) { k_norm<4><<<dim3(L.nreal, L.nc), 256, 0, s>>>(L, residual, out); ++g_nlaunch; }
  else { k_norm<6><<<dim3(L.nreal, L.nc), 256, 0, s>>>(L, residual, out); ++g_nlaunch; }
}

// R_h^M f on all real nodes into tmp (M=4: f + (1/12)Σδ²f, right side of E12), then
// f <- tmp on leaf nodes only (reading Z16).
template <int ORDER>
__global__ void k_rhs_apply(LevelView L, double* tmp) {
  comp_view(L);
  tmp += (int64_t)blockIdx.y * L.cs;
  const int b = blockIdx.x;
  const int B = L.B;
  const int32_t* nb = L.nbr + (size_t)b * 27;
  for (int i = threadIdx.x; i < L.B3; i += blockDim.x) {
    const int x = i % B, y = (i / B) % B, z = i / (B * B);
    auto g = [&](int a, int bb, int cc) { return fetch(L.f, nb, B, x + a, y + bb, z + cc); };
    const double c = L.f[(size_t)b * L.B3 + i];
    // δ² along each axis (dimensionless), at (x,y,z) and, for M = 6, at its neighbours
    auto d2x = [&](int yo, int zo) { return (g(-1, yo, zo) - 2.0 * g(0, yo, zo)) + g(1, yo, zo); };
    auto d2y = [&](int xo, int zo) { return (g(xo, -1, zo) - 2.0 * g(xo, 0, zo)) + g(xo, 1, zo); };
    auto d2z = [&](int xo, int yo) { return (g(xo, yo, -1) - 2.0 * g(xo, yo, 0)) + g(xo, yo, 1); };
    const double dx = d2x(0, 0), dy = d2y(0, 0), dz = d2z(0, 0);
    if (ORDER == 4) {
      tmp[(size_t)b * L.B3 + i] = c + ((dx + dy) + dz) / 12.0;
    } else {
      // R_h^6 f = f + (1/12) Σ δ² f + (1/90) Σ_{d<e} δ²_d δ²_e f - (1/240) Σ δ⁴ f (E13, Z24)
      const double dxy = (d2x(-1, 0) - 2.0 * dx) + d2x(1, 0);
      const double dyz = (d2y(0, -1) - 2.0 * dy) + d2y(0, 1);
      const double dzx = (d2z(-1, 0) - 2.0 * dz) + d2z(1, 0);
      const double dxx = ((g(-2, 0, 0) - 4.0 * g(-1, 0, 0)) + 6.0 * c) + (g(2, 0, 0) - 4.0 * g(1, 0, 0));
      const double dyy = ((g(0, -2, 0) - 4.0 * g(0, -1, 0)) + 6.0 * c) + (g(0, 2, 0) - 4.0 * g(0, 1, 0));
      const double dzz = ((g(0, 0, -2) - 4.0 * g(0, 0, -1)) + 6.0 * c) + (g(0, 0, 2) - 4.0 * g(0, 0, 1));
      tmp[(size_t)b * L.B3 + i] = ((c + ((dx + dy) + dz) / 12.0) + ((dxy + dyz) + dzx) / 90.0) -
                                  ((dxx + dyy) + dzz) / 240.0;
    }
  }
}

__global__ void k_rhs_commit(LevelView L, const double* tmp) {
  comp_view(L);
  tmp += (int64_t)blockIdx.y * L.cs;
  const int b = blockIdx.x;
  const int B = L.B, Bh = B / 2;
  const uint8_t cov = L.covmask[b];
  for (int i = threadIdx.x; i < L.B3; i += blockDim.x) {
    const int x = i % B, y = (i / B) % B, z = i / (B * B);
    const int oct = (x >= Bh) | ((y >= Bh) << 1) | ((z >= Bh) << 2);
    if (!((cov >> oct) & 1)) L.f[(size_t)b * L.B3 + i] = tmp[(size_t)b * L.B3 + i];
  }
}

void launch_correct_rhs(const LevelView& L, int order, double* tmp, cudaStream_t s) {
  if (!L.nreal || order == 2) return;
  if (order == 4) { k_rhs_apply<4><<<dim3(L.nreal, L.nc), 256, 0, s>>>(L, tmp); ++g_nlaunch; }
  else { k_rhs_apply<6><<<dim3(L.nreal, L.nc), 256, 0, s>>>(L, tmp); ++g_nlaunch; }
  { k_rhs_commit<<<dim3(L.nreal, L.nc), 256, 0, s>>>(L, tmp); ++g_nlaunch; }
}

// leaf-ordered [n_leaf][B^3] <-> level block storage
__global__ void k_leaf_scatter(int B3, const int64_t* __restrict__ map, const double* __restrict__ src,
                               double* const* __restrict__ dst, const int64_t* __restrict__ lev_cs, bool to_levels) {
  const int n = blockIdx.x, c = blockIdx.y;
  const int64_t m = map[n];
  const int lev = (int)(m >> 32), blk = (int)(m & 0xffffffff);
  double* d = dst[lev] + c * lev_cs[lev] + (size_t)blk * B3;
  const double* sl = src + ((size_t)c * gridDim.x + n) * B3;
  if (to_levels) {
    for (int i = threadIdx.x; i < B3; i += blockDim.x) d[i] = sl[i];
  } else {
    double* o = const_cast<double*>(sl);
    for (int i = threadIdx.x; i < B3; i += blockDim.x) o[i] = d[i];
  }
}

void launch_leaf_scatter(int nleaf, int B3, const int64_t* map, const double* src, double* const* dst_by_level,
                         const int64_t* lev_cs, int nc, bool to_levels, cudaStream_t s) {
  if (nleaf) { k_leaf_scatter<<<dim3(nleaf, nc), 256, 0, s>>>(B3, map, src, dst_by_level, lev_cs, to_levels); ++g_nlaunch; }
}

// Field transfer onto an adapted grid (reading A3): one CTA per destination block.
// rec = (dst block, src block, ox, oy, oz): ox < 0 -> copy the source block (same level
// and position); else trilinear interpolation of the source level's u on the
// octant (ox, oy, oz) of source block `src` and the next coarse node beyond it (real or
// ghost block, refreshed), per axis even -> copy, odd -> mean (the oracle's order).
__global__ void k_transfer(const int32_t* __restrict__ rec, double* __restrict__ dst, int64_t dcs,
                           const double* __restrict__ src, int64_t scs, const int32_t* __restrict__ snbr, int B) {
  const int32_t* r = rec + 5 * blockIdx.x;
  const int B3 = B * B * B, Bh = B / 2, E = Bh + 1;
  dst += (int64_t)blockIdx.y * dcs + (size_t)r[0] * B3;
  src += (int64_t)blockIdx.y * scs;
  if (r[2] < 0) {
    const double* s = src + (size_t)r[1] * B3;
    for (int i = threadIdx.x; i < B3; i += blockDim.x) dst[i] = s[i];
    return;
  }
  extern __shared__ double cw[];  // [E][E][E] coarse window
  const int32_t* nb = snbr + (size_t)r[1] * 27;
  for (int i = threadIdx.x; i < E * E * E; i += blockDim.x) {
    const int x = r[2] + i % E, y = r[3] + (i / E) % E, z = r[4] + i / (E * E);
    cw[i] = fetch(src, nb, B, x, y, z);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < B3; i += blockDim.x) {
    const int x = i % B, y = (i / B) % B, z = i / (B * B);
    const int cx = x >> 1, cy = y >> 1, cz = z >> 1;
    const int nx = (x & 1) ? 2 : 1, ny = (y & 1) ? 2 : 1, nz = (z & 1) ? 2 : 1;
    double vz[2];
    for (int tz = 0; tz < nz; ++tz) {
      double vy[2];
      for (int ty = 0; ty < ny; ++ty) {
        const double* row = cw + ((cz + tz) * E + (cy + ty)) * E + cx;
        vy[ty] = nx == 2 ? 0.5 * (row[0] + row[1]) : row[0];
      }
      vz[tz] = ny == 2 ? 0.5 * (vy[0] + vy[1]) : vy[0];
    }
    dst[i] = nz == 2 ? 0.5 * (vz[0] + vz[1]) : vz[0];
    (void)Bh;
  }
}

void launch_transfer(int n, const int32_t* rec, double* dst, int64_t dcs, const double* src, int64_t scs,
                     const int32_t* snbr, int B, int nc, cudaStream_t s) {
  if (n <= 0) return;
  const int E = B / 2 + 1;
  k_transfer<<<dim3(n, nc), 256, sizeof(double) * E * E * E, s>>>(rec, dst, dcs, src, scs, snbr, B);
  ++g_nlaunch;
}

// Cauchy increment of one V-cycle (E20) over the leaf nodes, on the device:
// out[0] <- max |u_new - u_old|, out[1] <- max |u_new| (bit patterns of non-negative
// doubles, atomicMax; NaN -> the quiet-NaN pattern), and prev <- u_new for the next cycle.
__global__ void k_leaf_cauchy(int B3, const int64_t* __restrict__ map, double* __restrict__ prev,
                              double* const* __restrict__ lev_u, const int64_t* __restrict__ lev_cs,
                              unsigned long long* out) {
  const int n = blockIdx.x, c = blockIdx.y;
  const int64_t m = map[n];
  const int lev = (int)(m >> 32);
  const double* u = lev_u[lev] + c * lev_cs[lev] + (size_t)(m & 0xffffffff) * B3;
  double* p = prev + ((size_t)c * gridDim.x + n) * B3;
  unsigned long long dm = 0ull, um = 0ull;
  for (int i = threadIdx.x; i < B3; i += blockDim.x) {
    const double v = u[i], d = fabs(v - p[i]), a = fabs(v);
    p[i] = v;
    const unsigned long long bd = d != d ? 0x7ff8000000000000ull : (unsigned long long)__double_as_longlong(d);
    const unsigned long long ba = a != a ? 0x7ff8000000000000ull : (unsigned long long)__double_as_longlong(a);
    dm = bd > dm ? bd : dm;
    um = ba > um ? ba : um;
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long t0 = __shfl_xor_sync(0xffffffffu, dm, o), t1 = __shfl_xor_sync(0xffffffffu, um, o);
    dm = t0 > dm ? t0 : dm;
    um = t1 > um ? t1 : um;
  }
  __shared__ unsigned long long sm[2][32];
  if ((threadIdx.x & 31) == 0) {
    sm[0][threadIdx.x >> 5] = dm;
    sm[1][threadIdx.x >> 5] = um;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
      dm = sm[0][w] > dm ? sm[0][w] : dm;
      um = sm[1][w] > um ? sm[1][w] : um;
    }
    atomicMax(out, dm);
    atomicMax(out + 1, um);
  }
}

void launch_leaf_cauchy(int nleaf, int B3, const int64_t* map, double* prev, double* const* lev_u,
                        const int64_t* lev_cs, int nc, unsigned long long* out, cudaStream_t s) {
  if (nleaf) { k_leaf_cauchy<<<dim3(nleaf, nc), 256, 0, s>>>(B3, map, prev, lev_u, lev_cs, out); ++g_nlaunch; }
}

// ---------------------------------------------------------------------------------
// Coarse direct solve (a6) around cuFFT (library call, timed separately).
// ---------------------------------------------------------------------------------
// Gather of level-0 f into the dense transform array.  Per axis, dense index q maps to
// level node J: periodic / unbounded axes J = q (q < N; padding 0); semi-unbounded axes
// (reading S1) hold the mirror-extended source on x = q - (N-1) in [-(N-1), N-1]:
// J = |x|, times the face's sign for x < 0, and 0 at x = 0 for an odd face.
struct CoarseAxes {
  int P[3], sym[3], hi_odd[3], hi_even[3], off[3];
};

__global__ void k_coarse_gather(LevelView L, double* dense, CoarseAxes A) {
  comp_view(L);
  dense += (int64_t)blockIdx.y * A.P[0] * A.P[1] * A.P[2];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n = (int64_t)A.P[0] * A.P[1] * A.P[2];
  if (i >= n) return;
  const int q[3] = {(int)(i % A.P[0]), (int)((i / A.P[0]) % A.P[1]), (int)(i / ((int64_t)A.P[0] * A.P[1]))};
  int J[3];
  double sg = 1.0;
  bool ok = true;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (A.hi_even[a]) {
      // walls at nodes 0 and N-1: even extension of period 2(N-1) (reading S3)
      const int n = L.N[a], p = q[a];
      J[a] = p < n ? p : 2 * (n - 1) - p;
    } else if (A.hi_odd[a]) {
      // both faces symmetric: periodic extension of period 2N (odd/odd) or 4N (even/odd)
      const int n = L.N[a], p = q[a];
      if (A.sym[a] < 0) {
        ok = ok && p != 0 && p != n;
        J[a] = p < n ? p : 2 * n - p;
        if (p > n) sg = -sg;
      } else {
        ok = ok && p != n && p != 3 * n;
        if (p < n) J[a] = p;
        else if (p <= 2 * n) { J[a] = 2 * n - p; sg = -sg; }
        else if (p < 3 * n) { J[a] = p - 2 * n; sg = -sg; }
        else J[a] = 4 * n - p;
      }
    } else if (A.sym[a]) {
      const int x = q[a] - A.off[a];
      ok = ok && x > -L.N[a] && x < L.N[a] && !(A.sym[a] < 0 && x == 0);
      J[a] = x < 0 ? -x : x;
      if (x < 0) sg *= (double)A.sym[a];
    } else {
      ok = ok && q[a] < L.N[a];
      J[a] = q[a];
    }
  }
  double v = 0.0;
  if (ok) {
    const int bx = J[0] / L.B, by = J[1] / L.B, bz = J[2] / L.B;
    const int blk = L.bmap[((bz - L.bmap_lo[2]) * L.bmap_n[1] + (by - L.bmap_lo[1])) * L.bmap_n[0] + (bx - L.bmap_lo[0])];
    v = sg * L.f[(size_t)blk * L.B3 + ((J[2] - bz * L.B) * L.B + (J[1] - by * L.B)) * L.B + (J[0] - bx * L.B)];
  }
  dense[i] = v;
}

void launch_coarse_gather(const LevelView& L, double* dense, const int* P, const int* sym, const int* hi_odd,
                          const int* hi_even, const int* off, cudaStream_t s) {
  CoarseAxes A{};
  for (int a = 0; a < 3; ++a) {
    A.P[a] = P[a];
    A.sym[a] = sym[a];
    A.hi_odd[a] = hi_odd[a];
    A.hi_even[a] = hi_even[a];
    A.off[a] = off[a];
  }
  const int64_t n = (int64_t)P[0] * P[1] * P[2];
  { k_coarse_gather<<<dim3((unsigned)((n + 255) / 256), L.nc), 256, 0, s>>>(L, dense, A); ++g_nlaunch; }
}

__global__ void k_coarse_scatter_nodes(LevelView L, const double* __restrict__ dense, CoarseAxes A) {
  comp_view(L);
  dense += (int64_t)blockIdx.y * A.P[0] * A.P[1] * A.P[2];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n = (int64_t)L.N[0] * L.N[1] * L.N[2];
  if (i >= n) return;
  const int x = (int)(i % L.N[0]), y = (int)((i / L.N[0]) % L.N[1]), z = (int)(i / ((int64_t)L.N[0] * L.N[1]));
  const int bx = x / L.B, by = y / L.B, bz = z / L.B;
  const int blk = L.bmap[((bz - L.bmap_lo[2]) * L.bmap_n[1] + (by - L.bmap_lo[1])) * L.bmap_n[0] + (bx - L.bmap_lo[0])];
  L.u[(size_t)blk * L.B3 + ((z - bz * L.B) * L.B + (y - by * L.B)) * L.B + (x - bx * L.B)] =
      dense[((int64_t)(z + A.off[2]) * A.P[1] + (y + A.off[1])) * A.P[0] + (x + A.off[0])];
}

__global__ void k_coarse_band(C2FList g, double* u, int64_t cs, const double* __restrict__ dense, CoarseAxes A) {
  u += (int64_t)blockIdx.y * cs;
  dense += (int64_t)blockIdx.y * A.P[0] * A.P[1] * A.P[2];
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= g.n) return;
  int q[3];
  for (int a = 0; a < 3; ++a) q[a] = ((g.J[3 * i + a] + A.off[a]) % A.P[a] + A.P[a]) % A.P[a];
  u[g.dst[i]] = dense[((int64_t)q[2] * A.P[1] + q[1]) * A.P[0] + q[0]];
}

void launch_coarse_scatter(const LevelView& L, const double* dense, const int* P, const int* off, const C2FList& band,
                           cudaStream_t s) {
  CoarseAxes A{};
  for (int a = 0; a < 3; ++a) {
    A.P[a] = P[a];
    A.off[a] = off[a];
  }
  const int64_t n = (int64_t)L.N[0] * L.N[1] * L.N[2];
  { k_coarse_scatter_nodes<<<dim3((unsigned)((n + 255) / 256), L.nc), 256, 0, s>>>(L, dense, A); ++g_nlaunch; }
  if (band.n) { k_coarse_band<<<dim3((band.n + 127) / 128, L.nc), 128, 0, s>>>(band, L.u, L.cs, dense, A); ++g_nlaunch; }
}

__global__ void k_fill_list(int n, const int32_t* __restrict__ idx, double* d, double v, int64_t cs) {
  d += (int64_t)blockIdx.y * cs;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) d[idx[i]] = v;
}

void launch_fill_list(int n, const int32_t* idx, double* d, double v, int nc, int64_t cs, cudaStream_t s) {
  if (n <= 0) return;
  k_fill_list<<<dim3((n + 255) / 256, nc), 256, 0, s>>>(n, idx, d, v, cs);
  ++g_nlaunch;
}

__global__ void k_copy_signed(int n, const int32_t* __restrict__ dst, const int32_t* __restrict__ src,
                              const int8_t* __restrict__ sgn, double* d, const double* sv, int64_t cs) {
  d += (int64_t)blockIdx.y * cs;
  sv += (int64_t)blockIdx.y * cs;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) d[dst[i]] = (double)sgn[i] * sv[src[i]];
}

void launch_copy_signed(int n, const int32_t* dst, const int32_t* src, const int8_t* sgn, double* d, const double* sv,
                        int nc, int64_t cs, cudaStream_t s) {
  if (n <= 0) return;
  k_copy_signed<<<dim3((n + 255) / 256, nc), 256, 0, s>>>(n, dst, src, sgn, d, sv, cs);
  ++g_nlaunch;
}

// spectral symbol σ_M(θ) h² from ŝ = 2cosθ - 2
__device__ __forceinline__ double symbol_h2(int order, double sx, double sy, double sz) {
  double s = sx + sy + sz;
  if (order >= 4) s += (sx * sy + sy * sz + sz * sx) * (1.0 / 6.0);
  if (order == 6) s += sx * sy * sz * (1.0 / 30.0);
  return s;
}

// periodic: û /= σ, zero mode -> 0; includes the 1/(PxPyPz) inverse scale
__global__ void k_mul_periodic(cuDoubleComplex* spec, int Px, int Py, int Pz, int order, double h2) {
  const int Hx = Px / 2 + 1;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n = (int64_t)Hx * Py * Pz;
  if (i >= n) return;
  spec += (int64_t)blockIdx.y * n;
  const int kx = (int)(i % Hx), ky = (int)((i / Hx) % Py), kz = (int)(i / ((int64_t)Hx * Py));
  const double tw = 6.283185307179586476925286766559;
  const double sx = 2.0 * cos(tw * kx / Px) - 2.0, sy = 2.0 * cos(tw * ky / Py) - 2.0, sz = 2.0 * cos(tw * kz / Pz) - 2.0;
  const double sig = symbol_h2(order, sx, sy, sz);
  const double scale = 1.0 / ((double)Px * Py * Pz);
  const double m = (kx == 0 && ky == 0 && kz == 0) ? 0.0 : h2 / sig * scale;
  spec[i] = make_cuDoubleComplex(cuCreal(spec[i]) * m, cuCimag(spec[i]) * m);
}

void launch_coarse_mul_periodic(void* spec, const int* P, int order, double h, int nc, cudaStream_t s) {
  const int64_t n = (int64_t)(P[0] / 2 + 1) * P[1] * P[2];
  { k_mul_periodic<<<dim3((unsigned)((n + 255) / 256), nc), 256, 0, s>>>((cuDoubleComplex*)spec, P[0], P[1], P[2], order, h * h); ++g_nlaunch; }
}

__global__ void k_mul_table(cuDoubleComplex* spec, const double* __restrict__ mult, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  spec += (int64_t)blockIdx.y * n;
  const double m = mult[i];
  spec[i] = make_cuDoubleComplex(cuCreal(spec[i]) * m, cuCimag(spec[i]) * m);
}

void launch_coarse_mul_table(void* spec, const double* mult, int64_t n, int nc, cudaStream_t s) {
  { k_mul_table<<<dim3((unsigned)((n + 255) / 256), nc), 256, 0, s>>>((cuDoubleComplex*)spec, mult, n); ++g_nlaunch; }
}

// Multiplier of a mixed periodic / unbounded coarse solve on the R2C spectrum (x halved):
// modes whose periodic wavenumbers are all zero take the transform of the LGF of the
// operator restricted to the unbounded axes (`low`, already x h^2 / (Px Py Pz)); all
// others h^2 / σ_M(k) / (Px Py Pz) (generalised E14, reading Z22).
__global__ void k_build_mult(double* __restrict__ mult, int Px, int Py, int Pz, int perx, int pery, int perz,
                             int ua, int ub, const double* __restrict__ low, int order, double h2, double scale,
                             int layout) {
  const int Hx = Px / 2 + 1;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n = (int64_t)Hx * Py * Pz;
  if (i >= n) return;
  // layout 0: [kz][ky][kx] (the 3-D R2C spectrum); 1: [kz][kx][ky] (the pruned solve)
  int k[3];
  if (layout == 0) {
    k[0] = (int)(i % Hx);
    k[1] = (int)((i / Hx) % Py);
  } else {
    k[1] = (int)(i % Py);
    k[0] = (int)((i / Py) % Hx);
  }
  k[2] = (int)(i / ((int64_t)Hx * Py));
  const int P[3] = {Px, Py, Pz}, per[3] = {perx, pery, perz};
  bool zero_per = true;
  for (int a = 0; a < 3; ++a)
    if (per[a] && k[a] != 0) zero_per = false;
  double m;
  if (zero_per) {
    m = ub >= 0 ? low[(int64_t)k[ub] * P[ua] + k[ua]] : low[k[ua]];
  } else {
    const double tw = 6.283185307179586476925286766559;
    const double sx = 2.0 * cos(tw * k[0] / Px) - 2.0, sy = 2.0 * cos(tw * k[1] / Py) - 2.0,
                 sz = 2.0 * cos(tw * k[2] / Pz) - 2.0;
    m = h2 / symbol_h2(order, sx, sy, sz) * scale;
  }
  mult[i] = m;
}

void launch_build_mult(double* mult, const int* P, const int* per, int ua, int ub, const double* low, int order,
                       double h2, double scale, int layout, cudaStream_t s) {
  const int64_t n = (int64_t)(P[0] / 2 + 1) * P[1] * P[2];
  k_build_mult<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(mult, P[0], P[1], P[2], per[0], per[1], per[2], ua, ub,
                                                             low, order, h2, scale, layout);
  ++g_nlaunch;
}

// Pruned coarse solve (x periodic, y and z unbounded): the y-transform input
// [c][z < Nz][kx][y < Py] from the x-spectrum [c][z][y < Ny][kx], zero for y >= Ny
__global__ void k_spec_pad_y(const cuDoubleComplex* __restrict__ c1, cuDoubleComplex* __restrict__ c2, int Nz, int Ny,
                             int Hx, int Py, int Pz) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // over z < Nz, kx, y < Py
  const int64_t n = (int64_t)Nz * Hx * Py;
  if (i >= n) return;
  const int y = (int)(i % Py), kx = (int)((i / Py) % Hx), z = (int)(i / ((int64_t)Py * Hx));
  const int c = blockIdx.y;
  c2 += (int64_t)c * Pz * Hx * Py;
  c1 += (int64_t)c * Nz * Ny * Hx;
  c2[((int64_t)z * Hx + kx) * Py + y] = y < Ny ? c1[((int64_t)z * Ny + y) * Hx + kx] : make_cuDoubleComplex(0.0, 0.0);
}

// the output window (z, y in [-GE, N + GE), periodic images in the padded lattice) of the
// inverse-transformed [c][z][kx][y] as x-spectra [c][zw][yw][kx] for the final C2R along x
__global__ void k_spec_window(const cuDoubleComplex* __restrict__ c2, cuDoubleComplex* __restrict__ c3, int Wz, int Wy,
                              int Hx, int Py, int Pz, int ge) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;   // over zw, yw, kx
  const int64_t n = (int64_t)Wz * Wy * Hx;
  if (i >= n) return;
  const int kx = (int)(i % Hx), yw = (int)((i / Hx) % Wy), zw = (int)(i / ((int64_t)Hx * Wy));
  const int c = blockIdx.y;
  const int z = (zw - ge + Pz) % Pz, y = (yw - ge + Py) % Py;
  c3[(int64_t)c * Wz * Wy * Hx + i] = c2[(int64_t)c * Pz * Hx * Py + ((int64_t)z * Hx + kx) * Py + y];
}

void launch_spec_pad_y(const void* c1, void* c2, int Nz, int Ny, int Hx, int Py, int Pz, int nc, cudaStream_t s) {
  const int64_t n = (int64_t)Nz * Hx * Py;
  k_spec_pad_y<<<dim3((unsigned)((n + 255) / 256), nc), 256, 0, s>>>((const cuDoubleComplex*)c1, (cuDoubleComplex*)c2, Nz,
                                                                    Ny, Hx, Py, Pz);
  ++g_nlaunch;
}

void launch_spec_window(const void* c2, void* c3, int Wz, int Wy, int Hx, int Py, int Pz, int ge, int nc,
                        cudaStream_t s) {
  const int64_t n = (int64_t)Wz * Wy * Hx;
  k_spec_window<<<dim3((unsigned)((n + 255) / 256), nc), 256, 0, s>>>((const cuDoubleComplex*)c2, (cuDoubleComplex*)c3, Wz,
                                                                     Wy, Hx, Py, Pz, ge);
  ++g_nlaunch;
}

__global__ void k_real_part_scale(const cuDoubleComplex* c, double* out, int64_t n, double a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = cuCreal(c[i]) * a;
}

void launch_real_part_scale(const void* cplx, double* out, int64_t n, double a, cudaStream_t s) {
  if (n) { k_real_part_scale<<<(unsigned)((n + 255) / 256), 256, 0, s>>>((const cuDoubleComplex*)cplx, out, n, a); ++g_nlaunch; }
}

}  // namespace mg
