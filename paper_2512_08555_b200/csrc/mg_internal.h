// mg_internal.h — device-side level description shared by the host runtime
// (mg_host.cpp) and the sm_100a kernels (mg_kernels.cu).  Not part of the ABI.
#pragma once
#include <cstdint>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>

namespace mg {

enum SmoothMode { SM_JACOBI = 0, SM_RB = 1 };

// One multigrid level in HBM.  Every field array is [ntot][B^3] fp64, x fastest;
// blocks [0, nreal) are the level's real blocks (leaves + parents, Morton order),
// blocks [nreal, ntot) are ghost blocks whose needed nodes hold boundary-ghost
// values (resolution-jump c2f, exterior band).  See DESIGN.md §Layout.
struct LevelView {
  int B, B3, nreal, ntot;
  // components (right-hand sides solved together, mg_desc.ncomp): every field array holds
  // nc copies [nc][ntot][B^3]; component c of a batched launch is blockIdx.y (comp_view)
  int nc;
  int64_t cs;           // component stride (doubles) = ntot * B3
  int N[3];             // nodes per axis of the level lattice
  double h;
  double* u;            // current solution buffer (ping-pong, see mg_host.cpp)
  double* u_out;        // the other buffer (smoother output)
  double* f;
  double* r;
  double* uhat;
  const int32_t* nbr;       // [nreal][27], slot (dx+1)+3(dy+1)+9(dz+1) -> block index
  const uint32_t* nbr_real; // [nreal] bit s set iff slot s is a real block
  const uint32_t* nbr_ext;  // [nreal] bit s set iff slot s is a ghost block beyond an unbounded face
  const uint8_t* covmask;   // [nreal] octant o covered by the finer level (bit o)
  const int32_t* parent;    // [nreal][4] (parent block in level-1, ox, oy, oz); m >= 1
  const int32_t* bmap;      // dense block-coordinate map (real+ghost) of this level
  int bmap_lo[3], bmap_n[3];
  int per[3];               // periodic axes
  // pencils: runs of consecutive real blocks along z (same bx, by), <= pen_lmax long;
  // the z-marching stencil kernels (mg_pencil.cu) walk one pencil per CTA
  int npen, pen_lmax;
  const int32_t* pen_blk;   // [npen][pen_lmax] real block indices, bottom to top (-1 padded)
  const int32_t* pen_len;   // [npen]
  // sweep pencils (k_rb_pencil only): like the above, plus (z0 | nplanes << 8) so that
  // small levels can split a block into several z-parts for more CTAs; sw_npen = 0: use pen_*
  int sw_npen, sw_pen_lmax;
  const int32_t* sw_pen_blk;
  const int32_t* sw_pen_len;
  const int32_t* sw_pen_z;
};

// TMA tensor maps of one B = 16 level's u (current buffer) and f arrays, each viewed as a
// 4-D tensor [ntot][16][16][16] fp64 (x fastest), one map per box shape of the plane-tile
// pieces (mg_pencil.cu TmaTile): 0 = 16 x 16, 1 = 2 x 16, 2 = 16 x 2, 3 = 2 x 2 (x by y, one
// plane, one block).  Passed to the kernels by value (__grid_constant__).
struct TileMaps {
  CUtensorMap u[4];
  CUtensorMap f[4];
};
// encode the 4 maps of an array of `ntot` 16^3 blocks; false if the driver lacks TMA
bool encode_tile_maps(const double* base, int ntot, CUtensorMap out[4]);

#ifdef __CUDACC__
// the field pointers of component blockIdx.y (batched launches: gridDim.y = nc)
__device__ __forceinline__ void comp_view(LevelView& L) {
  const int64_t o = (int64_t)blockIdx.y * L.cs;
  L.u += o;
  L.u_out += o;
  L.f += o;
  L.r += o;
  L.uhat += o;
}
#endif

struct C2FList {           // boundary-ghost entries of one level
  int n;
  const int32_t* dst;      // flat index into the level arrays
  const int32_t* J;        // [n][3] level-global node index (exterior allowed)
  const uint8_t* ext;      // 1 = beyond an unbounded face
};

struct InjList {           // f2c injection pairs feeding a level's c2f stencils
  int n;
  const int32_t* dst;      // flat index into level m-1 arrays
  const int32_t* src;      // flat index into level m arrays
};

// ---- launchers (mg_kernels.cu) ----
void prepare_kernels();  // constants + shared-memory attributes (call before any capture)
unsigned long long launches_issued();  // running count of this library's kernel launches
void note_launch();                   // count one launch made outside mg_kernels.cu
void launch_smooth(const LevelView& L, int order, int mode, double omega, bool with_residual,
                   cudaStream_t s);
void launch_residual(const LevelView& L, int order, cudaStream_t s);
// z-marching pencil kernels (B = 16 levels); return false if the level is not eligible
bool launch_rb_pencil(const LevelView& L, int order, double omega, const TileMaps* tm, cudaStream_t s);
bool launch_norm_pencil(const LevelView& L, int order, unsigned long long* out, cudaStream_t s);
bool launch_res_pencil(const LevelView& L, int order, cudaStream_t s);
// f* = R_h^4 f into L.r on the leaf nodes (raw f on covered nodes) (B = 16, M = 4)
bool launch_rhs_pencil(const LevelView& L, int order, cudaStream_t s);
// FAS right-hand side f = r + Δu on the covered nodes of a coarse level (B = 16)
bool launch_fas_pencil(const LevelView& L, int order, cudaStream_t s);
// fused fine residual + full-weighting restriction + u injection into the coarse level
bool launch_res_restrict_pencil(const LevelView& fine, const LevelView& coarse, int order, cudaStream_t s);
void prepare_pencil_kernels();
// separable box c2f (mg_ghost.cu): boxes = [nbox][12] int32 records (see mg_host.cpp)
// c2f ghost-box record (int32): dst block, lo[3], hi[3] (fine block-local, hi exclusive),
// org[3] (level-global fine index of the block's node (0,0,0)), 2 unused, then the
// coarse block index of each of the 3 x 3 x 3 block slots the box's taps meet
// (slot sx + 3 sy + 9 sz; -1 = none), 1 unused
constexpr int GBOX_REC = 40;
// mixed-radix FFT plan of the fused pruned coarse solve (mg_fft.cu): radices r[f], the
// product p[f] of the earlier ones, twiddle offset toff[f] (complex entries)
struct FFTPlan {
  static constexpr int MAXF = 12;
  int n = 0, nf = 0;
  int r[MAXF] = {}, p[MAXF] = {}, toff[MAXF] = {};
};
bool fft_plan(int n, FFTPlan& P, std::vector<double>& tw);
void prepare_fft_kernels();
void launch_fft_y_fwd(const void* c1, void* c2, int Ny, int Nz, int Hx, int Pz, const FFTPlan& py, const double* twy,
                      int nc, cudaStream_t s);
void launch_fft_z_conv(void* c2, const double* mult, int Q, int Nz, int GE, const FFTPlan& pz, const double* twz,
                       int nc, cudaStream_t s);
void launch_fft_y_inv(const void* c2, void* c3, int Hx, int Pz, int Wy, int Wz, int GE, const FFTPlan& py,
                      const double* twy, int nc, cudaStream_t s);
size_t c2f_box_smem_max(int I);
void launch_c2f_thin(const LevelView& fine, const LevelView& coarse, const int32_t* boxes, int nbox, double* fine_field,
                     const double* coarse_field, int I, bool ext_zero, cudaStream_t s);
void launch_c2f_box(const LevelView& fine, const LevelView& coarse, const int32_t* boxes, int nbox, int szA,
                    int szB, double* fine_field, const double* coarse_field, int I, bool ext_zero, cudaStream_t s);
void prepare_ghost_kernels();
void launch_inject_list(const InjList& l, double* coarse_field, const double* fine_field, int nc, int64_t cs_coarse,
                        int64_t cs_fine, cudaStream_t s);
// composed exterior-chain injections: fields[lev] = current u of level lev; entry e copies
// fields[lev_e >> 4][src_e] to fields[lev_e & 15][dst_e]
constexpr int MAX_CHAIN_LEVELS = 16;
void launch_inject_chain(int n, const int32_t* lev, const int32_t* dst, const int32_t* src,
                         double* const fields[MAX_CHAIN_LEVELS], const int64_t cs[MAX_CHAIN_LEVELS], int nc,
                         cudaStream_t s);
void launch_restrict(const LevelView& fine, const LevelView& coarse, cudaStream_t s);
void launch_fas_rhs(const LevelView& fine, const LevelView& coarse, int order, cudaStream_t s);
void launch_prolong(const LevelView& fine, const LevelView& coarse, cudaStream_t s);
void launch_inject_up(const LevelView& fine, const LevelView& coarse, double* coarse_u, cudaStream_t s);
void launch_norm(const LevelView& L, int order, bool residual, unsigned long long* out, cudaStream_t s);
void launch_correct_rhs(const LevelView& L, int order, double* tmp, cudaStream_t s);
// leaf arrays [nc][nleaf][B3]; lev_cs[level] = component stride of that level's fields
void launch_leaf_scatter(int nleaf, int B3, const int64_t* map, const double* src, double* const* dst_by_level,
                         const int64_t* lev_cs, int nc, bool to_levels, cudaStream_t s);
// E20 Cauchy increment on leaf nodes: out[0] max|u - prev|, out[1] max|u|; prev <- u
void launch_leaf_cauchy(int nleaf, int B3, const int64_t* map, double* prev, double* const* lev_u,
                        const int64_t* lev_cs, int nc, unsigned long long* out, cudaStream_t s);
// field transfer (mg_transfer): n records (dst block, src block, ox, oy, oz), ox < 0 = copy
void launch_transfer(int n, const int32_t* rec, double* dst, int64_t dcs, const double* src, int64_t scs,
                     const int32_t* snbr, int B, int nc, cudaStream_t s);
// coarse solve helpers
void launch_coarse_gather(const LevelView& L, double* dense, const int* P, const int* sym, const int* hi_odd,
                          const int* hi_even, const int* off, cudaStream_t s);
void launch_coarse_scatter(const LevelView& L, const double* dense, const int* P, const int* off, const C2FList& band,
                           cudaStream_t s);
// d[c cs + idx[i]] = v for every component c < nc
void launch_fill_list(int n, const int32_t* idx, double* d, double v, int nc, int64_t cs, cudaStream_t s);
void launch_copy_signed(int n, const int32_t* dst, const int32_t* src, const int8_t* sgn, double* d, const double* sv,
                        int nc, int64_t cs, cudaStream_t s);
// spectra of the nc components stored one after the other, (P0/2+1) P1 P2 each
void launch_coarse_mul_periodic(void* spec, const int* P, int order, double h, int nc, cudaStream_t s);
void launch_coarse_mul_table(void* spec, const double* mult, int64_t n, int nc, cudaStream_t s);
// full multiplier table of a mixed periodic / unbounded coarse solve (R2C layout)
// layout 0: [kz][ky][kx] (3-D R2C spectrum), 1: [kz][kx][ky] (pruned solve)
void launch_build_mult(double* mult, const int* P, const int* per, int ua, int ub, const double* low, int order,
                       double h2, double scale, int layout, cudaStream_t s);
// pruned coarse solve (x periodic, y, z unbounded): transposes around the 1-D transforms
void launch_spec_pad_y(const void* c1, void* c2, int Nz, int Ny, int Hx, int Py, int Pz, int nc, cudaStream_t s);
void launch_spec_window(const void* c2, void* c3, int Wz, int Wy, int Hx, int Py, int Pz, int ge, int nc,
                        cudaStream_t s);
void launch_real_part_scale(const void* cplx, double* out, int64_t n, double a, cudaStream_t s);

}  // namespace mg
