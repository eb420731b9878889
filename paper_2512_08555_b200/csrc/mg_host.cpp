// mg_host.cpp — host runtime and C-ABI of the B200 adaptive multigrid solver.
//
// Builds the multigrid level hierarchy from a leaf list (§2.1, P:58-65;
// §3), the per-level neighbour / ghost / transfer tables, the coarse
// FFT-LGF solver, and runs Alg. 1 as a fixed
// schedule of sm_100a kernel launches (optionally one CUDA graph per V-cycle).
#include <cuda_runtime.h>
#include <cufft.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <memory>
#include <queue>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "../../include/mg.h"
#include "mg_internal.h"

namespace mg {
std::vector<double> box_lgf(int dim, int order, int R);
}

using namespace mg;

namespace {

// exterior band width produced by the coarse solve (reading Z21/U1): 5 nodes, or 7 for
// M = 6 under U1 (the I = 8 c2f chain reaches 6 nodes beyond the unbounded faces)
constexpr int GE_M4 = 5, GE_M6U1 = 7;

struct MgError : std::runtime_error {
  int code;
  MgError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CUDA_OK(x)                                                                              \
  do {                                                                                          \
    cudaError_t e_ = (x);                                                                       \
    if (e_ != cudaSuccess)                                                                      \
      throw MgError(e_ == cudaErrorMemoryAllocation ? MG_ERR_OOM : MG_ERR_CUDA,                 \
                    std::string(#x) + ": " + cudaGetErrorString(e_));                           \
  } while (0)
#define CUFFT_OK(x)                                                                             \
  do {                                                                                          \
    cufftResult r_ = (x);                                                                       \
    if (r_ != CUFFT_SUCCESS) throw MgError(MG_ERR_CUDA, std::string(#x) + " failed: " + std::to_string(r_)); \
  } while (0)

thread_local std::string g_err = "";

inline int64_t key3(int x, int y, int z) {
  return (((int64_t)(z + 4096)) << 40) | (((int64_t)(y + 4096)) << 20) | (int64_t)(x + 4096);
}

inline int fdiv(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

uint64_t morton(int x, int y, int z) {
  uint64_t m = 0;
  for (int i = 0; i < 21; ++i) {
    m |= (uint64_t)((x >> i) & 1) << (3 * i);
    m |= (uint64_t)((y >> i) & 1) << (3 * i + 1);
    m |= (uint64_t)((z >> i) & 1) << (3 * i + 2);
  }
  return m;
}

template <class T>
T* dev_upload(const std::vector<T>& v) {
  if (v.empty()) return nullptr;
  T* p = nullptr;
  CUDA_OK(cudaMalloc(&p, v.size() * sizeof(T)));
  CUDA_OK(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return p;
}

struct Level {
  int B = 0, B3 = 0, nreal = 0, nghost = 0, amr = 0;
  int N[3] = {0, 0, 0};
  double h = 0;
  std::vector<std::array<int, 3>> coords;  // real, then ghost
  std::unordered_map<int64_t, int> index;
  std::vector<std::vector<uint64_t>> need;  // per ghost block: B^3 bitset of needed nodes
  std::vector<uint8_t> ghost_ext;           // per ghost block: beyond an unbounded face
  bool ext_chain = false;                   // exterior ghosts filled by c2f (reading U1)
  // host tables
  std::vector<int32_t> nbr, parent, bmap, c2f_dst, c2f_J, inj_dst, inj_src, pen_blk, pen_len, gbox;
  // exterior chains: the injections of refresh(this level) composed into one list of
  // (dst level | src level << 4, dst index, src index), every source on the finest level
  std::vector<int32_t> chain_lev, chain_dst, chain_src;
  int32_t *d_chain_lev = nullptr, *d_chain_dst = nullptr, *d_chain_src = nullptr;
  int gbox_szA = 0, gbox_szB = 0;  // c2f box kernel shared memory (doubles), max over the level's thick boxes
  int gbox_nthin = 0;              // boxes [0, gbox_nthin) go to the warp-per-box thin kernel
  std::vector<int32_t> sw_blk, sw_len, sw_z;  // sweep pencils (z-split blocks on small levels)
  int pen_lmax = 0;
  std::vector<uint32_t> nbr_real, nbr_ext;
  bool has_ext_ghosts = false;  // some real block has a ghost neighbour beyond an unbounded face
  std::vector<uint8_t> covmask, c2f_ext;
  int64_t n_c2f = 0;  // needed boundary-ghost nodes (the per-node lists c2f_* are kept for level 0 only)
  int bmap_lo[3] = {0, 0, 0}, bmap_n[3] = {1, 1, 1};
  // device
  double* u[2] = {nullptr, nullptr};
  double *f = nullptr, *r = nullptr, *uhat = nullptr;
  int cur = 0;
  // TMA tensor maps of the RB sweep, per ping-pong parity: (u[cur], f)
  TileMaps tmaps[2];
  bool has_tmaps = false;
  int32_t *d_nbr = nullptr, *d_parent = nullptr, *d_bmap = nullptr, *d_c2f_dst = nullptr, *d_c2f_J = nullptr,
          *d_inj_dst = nullptr, *d_inj_src = nullptr, *d_pen_blk = nullptr, *d_pen_len = nullptr,
          *d_gbox = nullptr, *d_sw_blk = nullptr, *d_sw_len = nullptr, *d_sw_z = nullptr;
  uint32_t* d_nbr_real = nullptr;
  uint32_t* d_nbr_ext = nullptr;
  uint8_t *d_covmask = nullptr, *d_c2f_ext = nullptr;

  int ntot() const { return nreal + nghost; }
  int find(int x, int y, int z) const {
    auto it = index.find(key3(x, y, z));
    return it == index.end() ? -1 : it->second;
  }
};

}  // namespace

struct mg_handle {
  mg_desc d{};
  double setup_ms[6] = {0, 0, 0, 0, 0, 0};  // mg_create phases (mg_setup_times)
  int per[3] = {1, 1, 1};
  int sym[3] = {0, 0, 0};  // symmetric low face: mirror sign (+1 even, -1 odd), 0 none
  int hi_odd[3] = {0, 0, 0};  // odd high face (mirror about the unstored node N; reading S2)
  int hi_even[3] = {0, 0, 0}; // (EVEN, EVEN) axis: walls at nodes 0 and N-1 (reading S3)
  int fper[3] = {1, 1, 1};    // axis periodic in the coarse-solve transform (P, or both faces symmetric)
  std::vector<int32_t> fwall;  // level-0 nodes on an odd low face: f := 0 there (u = 0)
  int32_t* d_fwall = nullptr;
  int coff[3] = {0, 0, 0};  // coarse solve: level-0 node J is extended node J + coff
  // level 0: exterior f ghosts beyond symmetric faces = signed mirror copies (reading S1)
  std::vector<int32_t> fm_dst, fm_src;
  std::vector<int8_t> fm_sgn;
  int32_t *d_fm_dst = nullptr, *d_fm_src = nullptr;
  int8_t* d_fm_sgn = nullptr;
  int order = 4, I = 6, GE = 5, smoother = 1, eta1 = 2, eta2 = 2;
  double omega = 1.0;
  int nsub = 0;
  std::vector<Level> L;
  std::vector<std::array<int, 4>> leaves;
  cudaStream_t s = nullptr;
  int64_t* d_leafmap = nullptr;
  double** d_lvl_ptrs = nullptr;  // per-level pointer table for the leaf scatter
  std::vector<double*> h_lvl_ptrs;
  unsigned long long* d_norm = nullptr;
  double* d_leafbuf = nullptr;   // [n_leaf][B^3] scratch (host e2e path, Cauchy)
  double* d_leafbuf2 = nullptr;
  bool rhs_set = false;
  bool canonical = true;  // coarse covered nodes hold the injected fine values (a8)
  double fstar_norm = 0.0;
  // coarse solve
  int coarse_kind = 0;  // 0 all periodic, 1 all unbounded, 2 any mix (see setup_coarse)
  int P[3] = {0, 0, 0};
  cufftHandle plan_f = 0, plan_b = 0;
  // pruned coarse solve (x periodic, y and z unbounded, the cfg4 / cfg5 / tube-like mixes):
  // 1-D transforms that skip the zero half of the padded source and the outputs outside
  // the [-GE, N + GE) window (see coarse_solve_pruned)
  bool pruned = false;
  cufftHandle pr_xf = 0, pr_y = 0, pr_z = 0, pr_y1 = 0, pr_y2 = 0, pr_xb = 0;
  double *pr_X = nullptr, *pr_R = nullptr, *pr_mult = nullptr;
  // fused y / z transforms of the pruned solve (mg_fft.cu): plans and device twiddles
  FFTPlan fp_y, fp_z;
  double *d_twy = nullptr, *d_twz = nullptr;
  bool fused_fft = false;
  void *pr_C1 = nullptr, *pr_C2 = nullptr, *pr_C3 = nullptr;
  int pr_W[3] = {0, 0, 0};  // window (x periodic: N; y, z: N + 2 GE)
  std::vector<cufftHandle*> plans() {
    return {&plan_f, &plan_b, &pr_xf, &pr_y, &pr_z, &pr_y1, &pr_y2, &pr_xb};
  }
  double* d_dense = nullptr;
  void* d_spec = nullptr;
  double* d_mult = nullptr;  // kinds 1, 2: full multiplier table on the R2C spectrum
  // per-stage CUDA-event profiling (non-graph launches only)
  bool prof_on = false;
  struct Ev { cudaEvent_t a, b; int st, lv; };
  std::vector<Ev> prof_pending;
  std::vector<cudaEvent_t> evpool;
  std::vector<double> prof_ms;      // [stage][level]
  std::vector<int64_t> prof_n;
  int nsm = 148;  // SMs of the device (grid sizing of the pencil kernels)
  int nc = 1;     // components solved together (mg_desc.ncomp): fields [nc][ntot][B^3]
  int64_t* d_lvl_cs = nullptr;  // per level: component stride (doubles) of its fields
  // graph
  bool use_graph = false;
  cudaGraphExec_t gexec = nullptr;
  int graph_cur_sig = -1;
  std::string err;
};

namespace {

enum Stage { ST_SMOOTH = 0, ST_SMOOTH_RES, ST_RESIDUAL, ST_GHOST, ST_RESTRICT, ST_PROLONG, ST_COARSE, ST_INJECT_UP,
             ST_NORM, ST_FAS, ST_COUNT };

cudaEvent_t get_ev(mg_handle* h) {
  if (!h->evpool.empty()) {
    cudaEvent_t e = h->evpool.back();
    h->evpool.pop_back();
    return e;
  }
  cudaEvent_t e;
  CUDA_OK(cudaEventCreate(&e));
  return e;
}

const char* const kStageName[ST_COUNT] = {"mg smooth", "mg smooth+residual", "mg residual", "mg ghost fill",
                                          "mg restrict", "mg prolong", "mg coarse solve", "mg inject-up",
                                          "mg norm", "mg FAS rhs"};

// RAII around one stage: an NVTX range (host timeline, for nsys / ncu --nvtx filters)
// and, when profiling, a CUDA event pair on the handle's stream.
struct Prof {
  mg_handle* h;
  int st, lv;
  cudaEvent_t a = nullptr;
  bool on;
  Prof(mg_handle* hh, int stage, int level) : h(hh), st(stage), lv(level), on(hh->prof_on) {
    nvtxRangePushA(kStageName[stage]);
    if (on) {
      a = get_ev(h);
      cudaEventRecord(a, h->s);
    }
  }
  ~Prof() {
    nvtxRangePop();
    if (!on) return;
    cudaEvent_t b = get_ev(h);
    cudaEventRecord(b, h->s);
    h->prof_pending.push_back({a, b, st, lv});
  }
};

void prof_flush(mg_handle* h) {
  if (h->prof_pending.empty()) return;
  CUDA_OK(cudaStreamSynchronize(h->s));
  const int nl = (int)h->L.size();
  for (auto& e : h->prof_pending) {
    float ms = 0;
    cudaEventElapsedTime(&ms, e.a, e.b);
    h->prof_ms[e.st * nl + e.lv] += ms;
    h->prof_n[e.st * nl + e.lv] += 1;
    h->evpool.push_back(e.a);
    h->evpool.push_back(e.b);
  }
  h->prof_pending.clear();
}

LevelView view(mg_handle* h, int m) {
  Level& l = h->L[m];
  LevelView v{};
  v.B = l.B;
  v.B3 = l.B3;
  v.nreal = l.nreal;
  v.ntot = l.ntot();
  for (int a = 0; a < 3; ++a) {
    v.N[a] = l.N[a];
    v.bmap_lo[a] = l.bmap_lo[a];
    v.bmap_n[a] = l.bmap_n[a];
    v.per[a] = h->per[a];
  }
  v.h = l.h;
  v.u = l.u[l.cur];
  v.u_out = l.u[1 - l.cur];
  v.f = l.f;
  v.r = l.r;
  v.uhat = l.uhat;
  v.nbr = l.d_nbr;
  v.nbr_real = l.d_nbr_real;
  v.nbr_ext = l.d_nbr_ext;
  v.covmask = l.d_covmask;
  v.parent = l.d_parent;
  v.bmap = l.d_bmap;
  v.npen = (int)l.pen_len.size();
  v.pen_lmax = l.pen_lmax;
  v.pen_blk = l.d_pen_blk;
  v.pen_len = l.d_pen_len;
  v.sw_npen = (int)l.sw_len.size();
  v.sw_pen_lmax = 1;
  v.sw_pen_blk = l.d_sw_blk;
  v.sw_pen_len = l.d_sw_len;
  v.sw_pen_z = l.d_sw_z;
  v.nc = h->nc;
  v.cs = (int64_t)l.ntot() * l.B3;
  return v;
}

C2FList c2f_list(Level& l) {
  C2FList g{};
  g.n = (int)l.c2f_dst.size();
  g.dst = l.d_c2f_dst;
  g.J = l.d_c2f_J;
  g.ext = l.d_c2f_ext;
  return g;
}

InjList inj_list(Level& l) {
  InjList g{};
  g.n = (int)l.inj_dst.size();
  g.dst = l.d_inj_dst;
  g.src = l.d_inj_src;
  return g;
}

// ----------------------------------------------------------------------------------
// hierarchy construction
// ----------------------------------------------------------------------------------
void validate_and_build(mg_handle* h) {
  const mg_desc& d = h->d;
  const int B = d.block_size;
  if (!(B == 16 || B == 8)) throw MgError(MG_ERR_ARG, "block_size must be 8 or 16");
  if (d.order != 2 && d.order != 4 && d.order != 6) throw MgError(MG_ERR_ORDER, "order must be 2, 4 or 6");
  if (d.smoother != MG_SMOOTHER_JACOBI && d.smoother != MG_SMOOTHER_RBGS) throw MgError(MG_ERR_ARG, "bad smoother");
  if (d.n_leaf <= 0 || !d.leaves) throw MgError(MG_ERR_ARG, "no leaves");
  if (d.eta1 < 0 || d.eta2 < 0 || !(d.h0 > 0)) throw MgError(MG_ERR_ARG, "bad eta/h0");
  for (int a = 0; a < 3; ++a) {
    if (d.base_blocks[a] <= 0) throw MgError(MG_ERR_ARG, "bad base_blocks");
    if (a == 0 && !(d.pencil_blocks >= 0 && d.pencil_blocks <= 4))
      throw MgError(MG_ERR_ARG, "pencil_blocks must be 0..4");
    if (a == 0 && (d.pencil_order < 0 || d.pencil_order > 2)) throw MgError(MG_ERR_ARG, "pencil_order must be 0..2");
    if (a == 0 && (d.ncomp < 0 || d.ncomp > 8)) throw MgError(MG_ERR_ARG, "ncomp must be 0..8 (0 = 1)");
    if (a == 0 && (d.coarse_pruning < 0 || d.coarse_pruning > 2)) throw MgError(MG_ERR_ARG, "coarse_pruning must be 0..2");
    if (a == 0 && (d.ghost_kernel < 0 || d.ghost_kernel > 2)) throw MgError(MG_ERR_ARG, "ghost_kernel must be 0..2");
    if (a == 0 && (d.zsplit < 0 || d.zsplit > 2 || d.fuse < 0 || d.fuse > 1 || d.staging < 0 || d.staging > 1))
      throw MgError(MG_ERR_ARG, "zsplit must be 0..2, fuse and staging 0..1");
    // face pairs: periodic, unbounded, or semi-unbounded: EVEN/ODD symmetry at
    // the low face with an unbounded high face (reading S1)
    const int lo = d.bc[2 * a], hi = d.bc[2 * a + 1];
    const bool ok = (lo == MG_BC_PERIODIC && hi == MG_BC_PERIODIC) || (lo == MG_BC_UNBOUNDED && hi == MG_BC_UNBOUNDED) ||
                    ((lo == MG_BC_EVEN || lo == MG_BC_ODD) && (hi == MG_BC_UNBOUNDED || hi == MG_BC_ODD)) ||
                    (lo == MG_BC_EVEN && hi == MG_BC_EVEN);
    if (!ok) throw MgError(MG_ERR_BC, "supported face pairs: P/P, U/U, EVEN/U, ODD/U, ODD/ODD, EVEN/ODD, EVEN/EVEN");
    h->per[a] = lo == MG_BC_PERIODIC;
    h->sym[a] = lo == MG_BC_EVEN ? 1 : (lo == MG_BC_ODD ? -1 : 0);
    h->hi_odd[a] = hi == MG_BC_ODD;
    h->hi_even[a] = lo == MG_BC_EVEN && hi == MG_BC_EVEN;
    h->fper[a] = h->per[a] || h->hi_odd[a] || h->hi_even[a];
    if (h->sym[a] && (d.coarse_n > 0 || d.allow_unbounded_refined))
      throw MgError(MG_ERR_BC, "symmetric faces need AMR level 0 as the coarse-solve level and no U1");
  }
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b)
      if (h->hi_even[a] && (d.bc[2 * b] == MG_BC_UNBOUNDED || d.bc[2 * b + 1] == MG_BC_UNBOUNDED))
        throw MgError(MG_ERR_BC, "an EVEN/EVEN axis needs the other axes periodic or symmetric");
  h->nc = d.ncomp > 0 ? d.ncomp : 1;
  h->order = d.order;
  h->I = d.order + 2;
  h->GE = (d.order == 6 && d.allow_unbounded_refined) ? GE_M6U1 : GE_M4;
  h->smoother = d.smoother;
  h->omega = d.omega;
  h->eta1 = d.eta1;
  h->eta2 = d.eta2;

  // ---- AMR tree from the leaves
  int amax = 0;
  for (int64_t i = 0; i < d.n_leaf; ++i) {
    std::array<int, 4> lf = {d.leaves[4 * i], d.leaves[4 * i + 1], d.leaves[4 * i + 2], d.leaves[4 * i + 3]};
    if (lf[0] < 0 || lf[0] > 20) throw MgError(MG_ERR_ARG, "bad leaf level");
    for (int a = 0; a < 3; ++a)
      if (lf[a + 1] < 0 || lf[a + 1] >= (d.base_blocks[a] << lf[0])) throw MgError(MG_ERR_ARG, "leaf out of range");
    amax = std::max(amax, lf[0]);
    h->leaves.push_back(lf);
  }
  std::vector<std::unordered_set<int64_t>> nodes(amax + 1), leafset(amax + 1);
  for (auto& lf : h->leaves) {
    if (!leafset[lf[0]].insert(key3(lf[1], lf[2], lf[3])).second) throw MgError(MG_ERR_LAYOUT_NESTING, "duplicate leaf");
    int x = lf[1], y = lf[2], z = lf[3];
    for (int a = lf[0]; a >= 0; --a) {
      nodes[a].insert(key3(x, y, z));
      x >>= 1; y >>= 1; z >>= 1;
    }
  }
  for (int a = 0; a <= amax; ++a)
    for (int64_t k : leafset[a]) {
      // a leaf may not have descendants
      if (a < amax) {
        const int x = (int)(k & 0xfffff) - 4096, y = (int)((k >> 20) & 0xfffff) - 4096, z = (int)(k >> 40) - 4096;
        if (nodes[a + 1].count(key3(2 * x, 2 * y, 2 * z))) throw MgError(MG_ERR_LAYOUT_NESTING, "leaf is also refined");
      }
    }
  if ((int64_t)nodes[0].size() != (int64_t)d.base_blocks[0] * d.base_blocks[1] * d.base_blocks[2])
    throw MgError(MG_ERR_LAYOUT_NESTING, "level 0 is not fully covered by the leaves");
  for (int a = 0; a < amax; ++a)
    for (int64_t k : nodes[a]) {
      const int x = (int)(k & 0xfffff) - 4096, y = (int)((k >> 20) & 0xfffff) - 4096, z = (int)(k >> 40) - 4096;
      int cnt = 0;
      for (int o = 0; o < 8; ++o) cnt += (int)nodes[a + 1].count(key3(2 * x + (o & 1), 2 * y + ((o >> 1) & 1), 2 * z + (o >> 2)));
      if (cnt != 0 && cnt != 8) throw MgError(MG_ERR_LAYOUT_NESTING, "partially refined block");
    }
  // 26-neighbour 2:1 balance and the unbounded-face rule
  for (auto& lf : h->leaves) {
    const int a = lf[0];
    for (int ax = 0; ax < 3; ++ax)
      if (a > 0 && !h->per[ax] && (lf[ax + 1] == 0 || lf[ax + 1] == (d.base_blocks[ax] << a) - 1) &&
          !d.allow_unbounded_refined)
        throw MgError(MG_ERR_UNBOUNDED_REFINED, "a refined block touches an unbounded face");
    if (a < 2) continue;
    for (int o = 0; o < 27; ++o) {
      if (o == 13) continue;
      int c[3] = {lf[1] + o % 3 - 1, lf[2] + (o / 3) % 3 - 1, lf[3] + o / 9 - 1};
      bool out = false;
      for (int ax = 0; ax < 3; ++ax) {
        const int n = d.base_blocks[ax] << a;
        if (h->per[ax]) c[ax] = ((c[ax] % n) + n) % n;
        else if (c[ax] < 0 || c[ax] >= n) out = true;
      }
      if (out) continue;
      if (!nodes[a - 1].count(key3(c[0] >> 1, c[1] >> 1, c[2] >> 1)))
        throw MgError(MG_ERR_LAYOUT_2TO1, "2:1 constraint violated");
    }
  }

  // ---- multigrid levels: uniform sub-base coarsenings (reading Z5) + AMR levels
  int N0[3];
  for (int a = 0; a < 3; ++a) N0[a] = d.base_blocks[a] * B;
  int nsub = 0;
  if (d.coarse_n > 0) {
    int n = N0[0];
    while (n > d.coarse_n && n % 2 == 0) { n /= 2; ++nsub; }
    if (n != d.coarse_n) throw MgError(MG_ERR_ARG, "coarse_n must be N0 / 2^j");
    for (int a = 0; a < 3; ++a)
      if ((N0[a] >> nsub) << nsub != N0[a]) throw MgError(MG_ERR_ARG, "coarse_n: axes not divisible");
  }
  h->nsub = nsub;
  const int nlev = nsub + amax + 1;
  h->L.resize(nlev);
  for (int m = 0; m < nlev; ++m) {
    Level& l = h->L[m];
    const int a = m - nsub;
    l.amr = a;
    int nmin = 1 << 30;
    for (int ax = 0; ax < 3; ++ax) {
      l.N[ax] = a < 0 ? (N0[ax] >> (-a)) : (N0[ax] << a);
      nmin = std::min(nmin, l.N[ax]);
    }
    l.B = std::min(B, nmin);
    if (!(l.B == 16 || l.B == 8 || l.B == 4)) throw MgError(MG_ERR_ARG, "coarse level too small (block size < 4)");
    for (int ax = 0; ax < 3; ++ax)
      if (l.N[ax] % l.B) throw MgError(MG_ERR_ARG, "level size not divisible by its block size");
    l.B3 = l.B * l.B * l.B;
    l.h = d.h0 * std::pow(2.0, -a);
    std::vector<std::array<int, 3>> cs;
    if (a < 0) {
      for (int z = 0; z < l.N[2] / l.B; ++z)
        for (int y = 0; y < l.N[1] / l.B; ++y)
          for (int x = 0; x < l.N[0] / l.B; ++x) cs.push_back({x, y, z});
    } else {
      for (int64_t k : nodes[a])
        cs.push_back({(int)(k & 0xfffff) - 4096, (int)((k >> 20) & 0xfffff) - 4096, (int)(k >> 40) - 4096});
    }
    std::sort(cs.begin(), cs.end(), [](const std::array<int, 3>& p, const std::array<int, 3>& q) {
      return morton(p[0], p[1], p[2]) < morton(q[0], q[1], q[2]);
    });
    l.coords = cs;
    l.nreal = (int)cs.size();
    for (int i = 0; i < l.nreal; ++i) l.index[key3(cs[i][0], cs[i][1], cs[i][2])] = i;
  }

  // ---- parents (fine block -> covered sub-box of its coarse block) and covered octants
  for (int m = 0; m < nlev; ++m) h->L[m].covmask.assign(h->L[m].nreal, 0);
  for (int m = 1; m < nlev; ++m) {
    Level &F = h->L[m], &C = h->L[m - 1];
    F.parent.assign(4 * F.nreal, 0);
    for (int i = 0; i < F.nreal; ++i) {
      int cb[3], off[3];
      for (int a = 0; a < 3; ++a) {
        const int s = F.B * F.coords[i][a] / 2;
        cb[a] = s / C.B;
        off[a] = s % C.B;
      }
      const int p = C.find(cb[0], cb[1], cb[2]);
      if (p < 0) throw MgError(MG_ERR_LAYOUT_NESTING, "fine block without parent");
      F.parent[4 * i] = p;
      F.parent[4 * i + 1] = off[0];
      F.parent[4 * i + 2] = off[1];
      F.parent[4 * i + 3] = off[2];
      if (F.B / 2 == C.B) C.covmask[p] = 0xff;
      else C.covmask[p] |= (uint8_t)(1u << ((off[0] >= C.B / 2) | ((off[1] >= C.B / 2) << 1) | ((off[2] >= C.B / 2) << 2)));
    }
  }
}

// Mark node (J) of level m as a needed boundary ghost; creates the ghost block.
void need_node(mg_handle* h, Level& l, int Jx, int Jy, int Jz) {
  int J[3] = {Jx, Jy, Jz};
  bool ext = false;
  for (int a = 0; a < 3; ++a) {
    if (h->per[a]) J[a] = ((J[a] % l.N[a]) + l.N[a]) % l.N[a];
    else if (J[a] < 0 || J[a] >= l.N[a]) ext = true;
  }
  const int bx = fdiv(J[0], l.B), by = fdiv(J[1], l.B), bz = fdiv(J[2], l.B);
  int idx = l.find(bx, by, bz);
  if (idx >= 0 && idx < l.nreal) return;  // a real node, not a ghost
  if (idx < 0) {
    idx = l.nreal + l.nghost++;
    l.coords.push_back({bx, by, bz});
    l.index[key3(bx, by, bz)] = idx;
    l.need.emplace_back((l.B3 + 63) / 64, 0ull);
    l.ghost_ext.push_back(ext ? 1 : 0);
  }
  const int g = idx - l.nreal;
  const int loc = ((J[2] - bz * l.B) * l.B + (J[1] - by * l.B)) * l.B + (J[0] - bx * l.B);
  l.need[g][loc >> 6] |= 1ull << (loc & 63);
}

// is_real_node with a one-entry block cache (setup loops walk neighbouring nodes, which
// mostly fall in the block of the previous lookup)
struct RealNodeCache {
  const mg_handle* h;
  const Level* l;
  int bx = INT32_MIN, by = 0, bz = 0, idx = -1;
  bool operator()(int Jx, int Jy, int Jz, int* flat) {
    int J[3] = {Jx, Jy, Jz};
    for (int a = 0; a < 3; ++a) {
      if (h->per[a]) J[a] = ((J[a] % l->N[a]) + l->N[a]) % l->N[a];
      else if (J[a] < 0 || J[a] >= l->N[a]) return false;
    }
    const int cx = J[0] / l->B, cy = J[1] / l->B, cz = J[2] / l->B;
    if (cx != bx || cy != by || cz != bz) {
      bx = cx;
      by = cy;
      bz = cz;
      idx = l->find(cx, cy, cz);
    }
    if (idx < 0 || idx >= l->nreal) return false;
    if (flat) *flat = idx * l->B3 + ((J[2] - cz * l->B) * l->B + (J[1] - cy * l->B)) * l->B + (J[0] - cx * l->B);
    return true;
  }
};

bool is_real_node(const mg_handle* h, const Level& l, int Jx, int Jy, int Jz, int* flat) {
  int J[3] = {Jx, Jy, Jz};
  for (int a = 0; a < 3; ++a) {
    if (h->per[a]) J[a] = ((J[a] % l.N[a]) + l.N[a]) % l.N[a];
    else if (J[a] < 0 || J[a] >= l.N[a]) return false;
  }
  const int bx = J[0] / l.B, by = J[1] / l.B, bz = J[2] / l.B;
  const int idx = l.find(bx, by, bz);
  if (idx < 0 || idx >= l.nreal) return false;
  if (flat) *flat = idx * l.B3 + ((J[2] - bz * l.B) * l.B + (J[1] - by * l.B)) * l.B + (J[0] - bx * l.B);
  return true;
}

void build_ghosts(mg_handle* h) {
  const int nlev = (int)h->L.size();
  // needed halo: every stencil, sweep, residual, transfer and norm evaluates live nodes
  // only, whose operands lie within Chebyshev distance 1 of a real block (the sweeps stage
  // a halo-2 tile, but a ring node at distance 1 is updated only when it is itself real,
  // and then its operands are within distance 1 of its own block); the radius-2 right-hand
  // side of M = 6 needs f at distance 2 (round 1 filled distance 2 for every RB level).
  // tests/test_gpu_edge.py poisons every ghost node outside this set with NaN and checks
  // that nothing reads one.
  const int g = h->order == 6 ? 2 : 1;
  for (int m = nlev - 1; m >= 0; --m) {
    Level& l = h->L[m];
    // halo ghosts: nodes within Chebyshev distance g of a real block, not in one
    for (int i = 0; i < l.nreal; ++i) {
      const auto c = l.coords[i];
      for (int o = 0; o < 27; ++o) {
        if (o == 13) continue;
        const int dx = o % 3 - 1, dy = (o / 3) % 3 - 1, dz = o / 9 - 1;
        int nc[3] = {c[0] + dx, c[1] + dy, c[2] + dz};
        bool ext = false;
        for (int a = 0; a < 3; ++a) {
          const int nb = l.N[a] / l.B;
          if (h->per[a]) nc[a] = ((nc[a] % nb) + nb) % nb;
          else if (nc[a] < 0 || nc[a] >= nb) ext = true;
        }
        (void)ext;
        const int idx = l.find(nc[0], nc[1], nc[2]);
        if (idx >= 0 && idx < l.nreal) continue;
        const int lo[3] = {dx < 0 ? l.B - g : 0, dy < 0 ? l.B - g : 0, dz < 0 ? l.B - g : 0};
        const int hi[3] = {dx > 0 ? g : l.B, dy > 0 ? g : l.B, dz > 0 ? g : l.B};
        // the slab lies in one (ghost) block: mark it there (need_node per node, batched)
        need_node(h, l, (c[0] + dx) * l.B + lo[0], (c[1] + dy) * l.B + lo[1], (c[2] + dz) * l.B + lo[2]);
        const int gidx = l.find(nc[0], nc[1], nc[2]) - l.nreal;
        auto& bits = l.need[gidx];
        for (int z = lo[2]; z < hi[2]; ++z)
          for (int y = lo[1]; y < hi[1]; ++y)
            for (int x = lo[0]; x < hi[0]; ++x) {
              const int loc = (z * l.B + y) * l.B + x;
              bits[loc >> 6] |= 1ull << (loc & 63);
            }
      }
    }
    if (m == 0) {
      // coarsest: every ghost is an exterior node filled from the coarse-solve band
      for (int gi = 0; gi < l.nghost; ++gi)
        if (!l.ghost_ext[gi]) throw MgError(MG_ERR_LAYOUT_NESTING, "coarsest level has interior ghosts");
    }
    // list the needed ghost nodes; for m >= 1 derive the c2f taps on level m-1
    Level* C = m > 0 ? &h->L[m - 1] : nullptr;
    std::vector<uint8_t> injected(m > 0 ? (size_t)C->nreal * C->B3 : 0, 0);  // f2c entries listed
    RealNodeCache ctap{h, C}, cinj{h, C}, finj{h, &l};
    l.n_c2f = 0;
    for (int gi = 0; gi < l.nghost; ++gi) {
      const auto c = l.coords[l.nreal + gi];
      int bb_lo[3] = {1 << 30, 1 << 30, 1 << 30}, bb_hi[3] = {-(1 << 30), -(1 << 30), -(1 << 30)};
      for (int loc = 0; loc < l.B3; ++loc) {
        if (!((l.need[gi][loc >> 6] >> (loc & 63)) & 1)) continue;
        const int J[3] = {c[0] * l.B + loc % l.B, c[1] * l.B + (loc / l.B) % l.B, c[2] * l.B + loc / (l.B * l.B)};
        bool ext = false;
        for (int a = 0; a < 3; ++a)
          if (!h->per[a] && (J[a] < 0 || J[a] >= l.N[a])) ext = true;
        if (ext && m > 0 && !h->d.allow_unbounded_refined)
          throw MgError(MG_ERR_UNBOUNDED_REFINED, "refined level needs exterior ghosts");
        if (ext && m > 0) l.ext_chain = true;
        if (m == 0) {
          for (int a = 0; a < 3; ++a)
            if (!h->per[a] && (J[a] < -h->GE || J[a] >= l.N[a] + h->GE))
              throw MgError(MG_ERR_LAYOUT_GHOST, "exterior ghost beyond the coarse-solve band");
        }
        ++l.n_c2f;
        if (m == 0) {  // the coarse solve scatters its exterior band to these nodes
          l.c2f_dst.push_back((l.nreal + gi) * l.B3 + loc);
          for (int a = 0; a < 3; ++a) l.c2f_J.push_back(J[a]);
          l.c2f_ext.push_back(ext ? 1 : 0);
        }
        for (int a = 0; a < 3; ++a) {
          bb_lo[a] = std::min(bb_lo[a], J[a]);
          bb_hi[a] = std::max(bb_hi[a], J[a]);
        }
        if (m > 0) {
          // coarse tap range per axis (centred I-point rule for odd J)
          int t0[3], t1[3];
          for (int a = 0; a < 3; ++a) {
            if ((J[a] & 1) == 0) { t0[a] = J[a] >> 1; t1[a] = t0[a]; }
            else { t0[a] = ((J[a] - 1) >> 1) - h->I / 2 + 1; t1[a] = t0[a] + h->I - 1; }
          }
          if (ext) {
            for (int z = t0[2]; z <= t1[2]; ++z)
              for (int y = t0[1]; y <= t1[1]; ++y)
                for (int x = t0[0]; x <= t1[0]; ++x)
                  if (!is_real_node(h, *C, x, y, z, nullptr)) need_node(h, *C, x, y, z);
          } else {
            for (int k = 0; k < 8; ++k) {
              const int x = (k & 1) ? t1[0] : t0[0], y = (k & 2) ? t1[1] : t0[1], z = (k & 4) ? t1[2] : t0[2];
              if (!ctap(x, y, z, nullptr))
                throw MgError(MG_ERR_LAYOUT_GHOST, "ghost interpolation stencil leaves the coarse level (2:1?)");
            }
          }
        }
      }
      if (m > 0 && bb_lo[0] <= bb_hi[0]) {
        // f2c injection of every covered coarse node in the tap hull of this ghost block
        for (int z = fdiv(bb_lo[2], 2) - h->I / 2; z <= fdiv(bb_hi[2], 2) + h->I / 2; ++z)
          for (int y = fdiv(bb_lo[1], 2) - h->I / 2; y <= fdiv(bb_hi[1], 2) + h->I / 2; ++y)
            for (int x = fdiv(bb_lo[0], 2) - h->I / 2; x <= fdiv(bb_hi[0], 2) + h->I / 2; ++x) {
              int cflat, fflat;
              if (!cinj(x, y, z, &cflat)) continue;
              if (injected[cflat]) continue;
              if (!finj(2 * x, 2 * y, 2 * z, &fflat)) continue;
              injected[cflat] = 1;
              l.inj_dst.push_back(cflat);
              l.inj_src.push_back(fflat);
            }
      }
    }
  }
  // Exterior chains (reading U1): refreshing level m recomputes the exterior ghosts of
  // every level 1..m, and the oracle's W_{j-1} holds, at EVERY covered node, the value
  // injected from level j (recursively from the finest level).  The per-level f2c lists
  // above only cover the tap hull of level j's own ghosts, so close them: every level-
  // (j-1) node that inj(j-1) reads and that level j covers must first be injected from
  // level j.  (Coarse to fine, so additions to inj(j-1) propagate.)
  for (int j = 2; j < nlev; ++j) {
    if (!h->L[j].ext_chain) continue;
    Level &F = h->L[j], &C = h->L[j - 1];
    std::unordered_set<int32_t> have(F.inj_dst.begin(), F.inj_dst.end());
    for (int32_t src : C.inj_src) {
      const int blk = src / C.B3, loc = src % C.B3;
      const int Jx = C.coords[blk][0] * C.B + loc % C.B, Jy = C.coords[blk][1] * C.B + (loc / C.B) % C.B,
                Jz = C.coords[blk][2] * C.B + loc / (C.B * C.B);
      int fflat;
      if (!is_real_node(h, F, 2 * Jx, 2 * Jy, 2 * Jz, &fflat)) continue;
      if (have.insert(src).second) {
        F.inj_dst.push_back(src);
        F.inj_src.push_back(fflat);
      }
    }
  }

  // f2c lists in ascending destination order (independent copies: any order gives the same
  // values): consecutive threads of k_copy_list then touch neighbouring coarse nodes and the
  // even fine nodes under them, so the 8-byte accesses share 32-byte sectors (cfg5 level-4
  // refresh 76.6 -> 75.3 us)
  for (int j = 1; j < nlev; ++j) {
    Level& F = h->L[j];
    std::vector<size_t> perm(F.inj_dst.size());
    for (size_t e = 0; e < perm.size(); ++e) perm[e] = e;
    std::sort(perm.begin(), perm.end(), [&](size_t a, size_t b) { return F.inj_dst[a] < F.inj_dst[b]; });
    std::vector<int32_t> d2(perm.size()), s2(perm.size());
    for (size_t e = 0; e < perm.size(); ++e) d2[e] = F.inj_dst[perm[e]], s2[e] = F.inj_src[perm[e]];
    F.inj_dst.swap(d2);
    F.inj_src.swap(s2);
  }

  // Composed injection lists of the exterior-chain refresh of level m (reading U1): the
  // lists m, m-1, …, 1 are applied in that order, so a level-j source that list j+1
  // (j+1 <= m) injects from level j+1 is the same value as that level-(j+1) node; follow
  // such sources up to level m and the whole chain becomes one launch of independent
  // copies (identical values).
  for (int m = 2; m < nlev; ++m) {
    Level& T = h->L[m];
    if (!T.ext_chain) continue;
    std::vector<std::unordered_map<int32_t, int32_t>> inj(m + 1);
    for (int j = 1; j <= m; ++j)
      for (size_t e = 0; e < h->L[j].inj_dst.size(); ++e) inj[j][h->L[j].inj_dst[e]] = h->L[j].inj_src[e];
    for (int j = m; j >= 1; --j) {
      const Level& F = h->L[j];
      for (size_t e = 0; e < F.inj_dst.size(); ++e) {
        int lev = j, idx = F.inj_src[e];
        while (lev < m) {
          auto it = inj[lev + 1].find(idx);
          if (it == inj[lev + 1].end()) break;
          idx = it->second;
          ++lev;
        }
        T.chain_lev.push_back((j - 1) | (lev << 4));
        T.chain_dst.push_back(F.inj_dst[e]);
        T.chain_src.push_back(idx);
      }
    }
  }

  // neighbour tables and block maps
  for (int m = 0; m < nlev; ++m) {
    Level& l = h->L[m];
    l.nbr.assign(27 * (size_t)l.nreal, -1);
    l.nbr_real.assign(l.nreal, 0);
    l.nbr_ext.assign(l.nreal, 0);
    for (int i = 0; i < l.nreal; ++i) {
      const auto c = l.coords[i];
      for (int o = 0; o < 27; ++o) {
        int nc[3] = {c[0] + o % 3 - 1, c[1] + (o / 3) % 3 - 1, c[2] + o / 9 - 1};
        for (int a = 0; a < 3; ++a) {
          const int nb = l.N[a] / l.B;
          if (h->per[a]) nc[a] = ((nc[a] % nb) + nb) % nb;
        }
        const int idx = l.find(nc[0], nc[1], nc[2]);
        if (idx < 0) throw MgError(MG_ERR_LAYOUT_GHOST, "missing neighbour block");
        l.nbr[27 * (size_t)i + o] = idx;
        if (idx < l.nreal) l.nbr_real[i] |= 1u << o;
        else if (l.ghost_ext[idx - l.nreal]) {
          l.nbr_ext[i] |= 1u << o;
          l.has_ext_ghosts = true;
        }
      }
    }
    int lo[3], hi[3];
    for (int a = 0; a < 3; ++a) { lo[a] = 0; hi[a] = l.N[a] / l.B - 1; }
    for (auto& c : l.coords)
      for (int a = 0; a < 3; ++a) { lo[a] = std::min(lo[a], c[a]); hi[a] = std::max(hi[a], c[a]); }
    size_t n = 1;
    for (int a = 0; a < 3; ++a) { l.bmap_lo[a] = lo[a]; l.bmap_n[a] = hi[a] - lo[a] + 1; n *= l.bmap_n[a]; }
    l.bmap.assign(n, -1);
    for (int i = 0; i < l.ntot(); ++i) {
      const auto c = l.coords[i];
      l.bmap[((size_t)(c[2] - lo[2]) * l.bmap_n[1] + (c[1] - lo[1])) * l.bmap_n[0] + (c[0] - lo[0])] = i;
    }
  }
}

// Ghost boxes of the c2f kernel (mg_ghost.cu): the needed nodes of every ghost block
// are split into disjoint boxes.  Per axis, the cut points are the planes where the
// need mask changes anywhere; the mask is constant on every cell of that grid, and the
// needed cells are merged greedily (x, then y, then z).  For the usual need mask — a
// union of g-thick halo slabs, one per real neighbour — the boxes are at most g thick
// along some axis, which bounds the kernel's shared memory (~22 KB for I = 6 instead of
// ~48 KB for a 16^3 bounding box, i.e. more resident CTAs) and skips the unneeded
// interior of L-shaped unions.
void build_ghost_boxes(mg_handle* h) {
  const int I = h->I;
  for (size_t m = 1; m < h->L.size(); ++m) {
    Level& l = h->L[m];
    const Level& C = h->L[m - 1];
    l.gbox.clear();
    l.gbox_szA = l.gbox_szB = 0;
    std::vector<int32_t> thin, thick;  // records of boxes <= 2 / > 2 nodes thick along the thinnest axis
    int thin_szA = 0, thin_szB = 0;
    const int B = l.B;
    for (int gi = 0; gi < l.nghost; ++gi) {
      std::vector<uint8_t> nd(l.B3);
      for (int loc = 0; loc < l.B3; ++loc) nd[loc] = (l.need[gi][loc >> 6] >> (loc & 63)) & 1;
      auto at = [&](int x, int y, int z) -> uint8_t& { return nd[(z * B + y) * B + x]; };
      auto emit = [&](const int lo[3], const int hi[3]) {
        const auto c = l.coords[l.nreal + gi];
        int32_t rec[GBOX_REC] = {l.nreal + gi, lo[0], lo[1], lo[2], hi[0], hi[1], hi[2],
                                 c[0] * B, c[1] * B, c[2] * B, 0, 0};
        int nf[3], nc[3], sb[3][3];
        for (int a = 0; a < 3; ++a) {
          const int g0 = rec[7 + a] + lo[a];
          nf[a] = hi[a] - lo[a];
          const int c0 = fdiv(g0, 2) - I / 2 + 1;
          nc[a] = fdiv(g0 + nf[a] - 1, 2) - fdiv(g0, 2) + I;
          // coarse block coordinate of each slot (consecutive blocks met along the taps,
          // periodic wrap included; -1 outside the coarse block map)
          for (int k = 0; k < 3; ++k) sb[a][k] = -1;
          int first = 0;
          for (int q = 0; q < nc[a]; ++q) {
            int ci = c0 + q;
            if (h->per[a]) ci = ((ci % C.N[a]) + C.N[a]) % C.N[a];
            const int cb = fdiv(ci, C.B);
            if (q == 0) first = cb;
            int slot = cb - first;
            if (slot < 0) slot += C.N[a] / C.B;
            if (slot > 2) throw MgError(MG_ERR_LAYOUT_GHOST, "ghost box coarse support spans > 3 blocks");
            const int b = cb - C.bmap_lo[a];
            sb[a][slot] = (b < 0 || b >= C.bmap_n[a]) ? -1 : b;
          }
        }
        for (int k = 0; k < 27; ++k) {
          const int b0 = sb[0][k % 3], b1 = sb[1][(k / 3) % 3], b2 = sb[2][k / 9];
          rec[12 + k] = (b0 < 0 || b1 < 0 || b2 < 0)
                            ? -1
                            : C.bmap[((size_t)b2 * C.bmap_n[1] + b1) * C.bmap_n[0] + b0];
        }
        // thin boxes (<= 2 nodes along some axis: the layers of the distance-1 halo) are
        // candidates for the warp-per-box kernel (decided per level below)
        const bool is_thin = std::min(nf[0], std::min(nf[1], nf[2])) <= 2;
        (is_thin ? thin : thick).insert((is_thin ? thin : thick).end(), rec, rec + GBOX_REC);
        // CTA kernel: region A = max(coarse stage, pass-y output), region B = pass-x output
        int& szA = is_thin ? thin_szA : l.gbox_szA;
        int& szB = is_thin ? thin_szB : l.gbox_szB;
        szA = std::max(szA, std::max(nc[0] * nc[1] * nc[2], nf[0] * nf[1] * nc[2]));
        szB = std::max(szB, nf[0] * nc[1] * nc[2]);
      };
      // cut points per axis: planes k where the need mask differs from plane k-1 anywhere
      std::vector<uint8_t> dif(3 * B, 0);
      for (int z = 0; z < B; ++z)
        for (int y = 0; y < B; ++y) {
          const uint8_t* row = &nd[(z * B + y) * B];
          for (int x = 1; x < B; ++x) dif[x] |= row[x] != row[x - 1];
          if (y > 0) {
            const uint8_t* prev = row - B;
            for (int x = 0; x < B; ++x) dif[B + y] |= row[x] != prev[x];
          }
          if (z > 0) {
            const uint8_t* prev = row - B * B;
            for (int x = 0; x < B; ++x) dif[2 * B + z] |= row[x] != prev[x];
          }
        }
      std::vector<int> cut[3];
      for (int a = 0; a < 3; ++a) {
        cut[a].push_back(0);
        for (int k = 1; k < B; ++k)
          if (dif[a * B + k]) cut[a].push_back(k);
        cut[a].push_back(B);
      }
      const int n0 = (int)cut[0].size() - 1, n1 = (int)cut[1].size() - 1, n2 = (int)cut[2].size() - 1;
      std::vector<uint8_t> cell(n0 * n1 * n2);  // 1 = needed and not yet in a box
      for (int z = 0; z < n2; ++z)
        for (int y = 0; y < n1; ++y)
          for (int x = 0; x < n0; ++x) cell[(z * n1 + y) * n0 + x] = at(cut[0][x], cut[1][y], cut[2][z]);
      auto fr = [&](int x, int y, int z) -> uint8_t& { return cell[(z * n1 + y) * n0 + x]; };
      for (int z = 0; z < n2; ++z)
        for (int y = 0; y < n1; ++y)
          for (int x = 0; x < n0; ++x) {
            if (!fr(x, y, z)) continue;
            int x1 = x, y1 = y, z1 = z;
            while (x1 + 1 < n0 && fr(x1 + 1, y, z)) ++x1;
            for (bool ok = true; ok && y1 + 1 < n1;) {
              for (int xx = x; xx <= x1; ++xx) ok = ok && fr(xx, y1 + 1, z);
              if (ok) ++y1;
            }
            for (bool ok = true; ok && z1 + 1 < n2;) {
              for (int yy = y; yy <= y1; ++yy)
                for (int xx = x; xx <= x1; ++xx) ok = ok && fr(xx, yy, z1 + 1);
              if (ok) ++z1;
            }
            for (int zz = z; zz <= z1; ++zz)
              for (int yy = y; yy <= y1; ++yy)
                for (int xx = x; xx <= x1; ++xx) fr(xx, yy, zz) = 0;
            const int lo[3] = {cut[0][x], cut[1][y], cut[2][z]};
            const int hi[3] = {cut[0][x1 + 1], cut[1][y1 + 1], cut[2][z1 + 1]};
            emit(lo, hi);
          }
    }
    // The warp-per-box kernel (mg_ghost.cu) wins when the level has enough boxes to fill
    // the GPU with warps (cfg5 levels 2-4: 2 000 - 13 000 boxes; with one-warp CTAs also
    // cfg5 level 2, 30.6 -> 23.5 us per refresh, and cfg4 level 2, 22.3 -> 20.0 us); with
    // few boxes (cfg5 level 1, ~800: equal), or the large multi-layer boxes of exterior
    // chains (U1, cfg3: 102 -> 125 us of ghost fill per refresh chain), one CTA per box has
    // more parallelism per box.  mg_desc.ghost_kernel: 1 never, 2 always.
    const int nthin = (int)(thin.size() / GBOX_REC);
    const bool use_thin = h->d.ghost_kernel == 2 || (h->d.ghost_kernel == 0 && !l.ext_chain && nthin >= 1024);
    l.gbox_nthin = use_thin ? nthin : 0;
    if (!use_thin) {
      l.gbox_szA = std::max(l.gbox_szA, thin_szA);
      l.gbox_szB = std::max(l.gbox_szB, thin_szB);
    }
    l.gbox = std::move(thin);
    l.gbox.insert(l.gbox.end(), thick.begin(), thick.end());
    if (sizeof(double) * (size_t)(l.gbox_szA + l.gbox_szB) > c2f_box_smem_max(I))
      throw MgError(MG_ERR_LAYOUT_GHOST, "ghost box exceeds the c2f kernel's shared memory");
  }
}

// Pencils of B = 16 levels: maximal runs of consecutive real blocks along z (same
// bx, by; no periodic wrap inside a run), split into near-equal chunks of at most
// `lmax` blocks, longest first.  The z-marching kernels (mg_pencil.cu) walk one
// pencil per CTA; halos above/below a pencil come through the neighbour tables.
void build_pencils(mg_handle* h) {
  // Pencil length: long pencils amortise the 2+2 halo planes, short ones give more CTAs
  // (rule below).  Ghost-free levels of >= 4 waves whose z-runs average >= 8 blocks use 4
  // — cfg2 256^3 on B200 after the sweep rewrite: sweep 96.9 -> 90.7 us, V-cycle 0.715 ->
  // 0.694 ms.  mg_desc.pencil_blocks forces one length and mg_desc.pencil_order the
  // chunking and launch order (tests), mg_desc.zsplit the z-split of small levels.
  const int lmax_force = h->d.pencil_blocks;
  const int nsm = h->nsm;
  const int S = 4 * nsm;  // CTA slots: the sweep and the fused residual + restriction run 4 CTAs per SM
  // makespan of the list schedule of a launch on S slots (cost of a pencil: 16 len + 4 plane steps)
  auto makespan = [&](const std::vector<int>& lens) {
    std::priority_queue<long, std::vector<long>, std::greater<long>> q;
    for (int i = 0; i < S; ++i) q.push(0);
    long m = 0;
    for (int L : lens) {
      const long t = q.top() + 16 * L + 4;
      q.pop();
      q.push(t);
      m = std::max(m, t);
    }
    return m;
  };
  for (auto& l : h->L) {
    std::vector<std::array<int, 4>> cols;  // (bx, by, bz, idx)
    for (int i = 0; i < l.nreal; ++i) cols.push_back({l.coords[i][0], l.coords[i][1], l.coords[i][2], i});
    std::sort(cols.begin(), cols.end());
    auto run_start = [&](size_t a) {
      return a == 0 || cols[a][0] != cols[a - 1][0] || cols[a][1] != cols[a - 1][1] || cols[a][2] != cols[a - 1][2] + 1;
    };
    int nruns = 0;
    for (size_t a = 0; a < cols.size(); ++a) nruns += run_start(a);
    const bool long_runs = nruns > 0 && l.nreal >= 8 * nruns && l.nghost == 0;
    // automatic length by waves of 1-block pencils (W = nreal / (4 #SM)), measured on cfg5's
    // levels: W <= 1: 1; 1 < W < 8: 2 (below); 8 <= W < 24: 3 (level 3, 6640 blocks:
    // sweep 163.7 -> 154.3 us, residual + restriction 154.8 -> 147.9 us); ghost-free levels
    // of >= 4 waves with long z-runs, and every level of W >= 24: 4.
    // Chunking and order.  "Balanced" (W < 24): a z-run of n blocks is cut into
    // ceil(n / lmax) nearly equal pencils, launched longest first, then by the z of the
    // first block and Morton order of (bx, by).  "Aligned" (W >= 24: cfg5 level 4, 23144
    // blocks): pencils are cut where bz is a multiple of lmax and launched by (bz / lmax,
    // Morton(bx, by)) whatever their length, so that the CTAs resident together cover the
    // same z-slab of neighbouring columns and re-read each other's halos from L2 — with
    // balanced chunks the neighbours of a 4-block pencil start at other z and in other
    // length classes, and 4-block pencils were slower than 2-block ones (554 vs 506 us);
    // aligned, they are faster: cfg5 level-4 sweep 510 -> 492 us, fused residual +
    // restriction 495 -> 472 us (profiles/r02_pencil_aligned_ab.jsonl; lengths 3, 5, 6, 8:
    // 503, 491, 497, 508 us).
    const double W = (double)l.nreal / (4.0 * nsm);
    l.pen_blk.clear();
    l.pen_len.clear();
    if (l.B != 16) {
      l.pen_lmax = lmax_force ? lmax_force : 1;
      continue;
    }
    // the pencil list for one length / order, and its modelled makespan
    auto construct = [&](const int lmax, const bool aligned, std::vector<std::vector<int>>& pens) {
      pens.clear();
      for (size_t a = 0; aligned && a < cols.size(); ++a) {
        if (run_start(a) || cols[a][2] % lmax == 0) pens.emplace_back();
        pens.back().push_back(cols[a][3]);
      }
      for (size_t a = 0; !aligned && a < cols.size();) {
        size_t b = a + 1;
        while (b < cols.size() && !run_start(b)) ++b;
        const int n = (int)(b - a), nchunk = (n + lmax - 1) / lmax;
        for (int c = 0, pos = 0; c < nchunk; ++c) {
          const int len = n / nchunk + (c < n % nchunk ? 1 : 0);
          std::vector<int> p;
          for (int t = 0; t < len; ++t) p.push_back(cols[a + pos + t][3]);
          pos += len;
          pens.push_back(p);
        }
        a = b;
      }
      // launch order (see above): CTAs resident at the same time are spatial neighbours and
      // re-read each other's halos from L2
      auto key = [&](const std::vector<int>& p) {
        const auto& c = l.coords[p[0]];
        return ((uint64_t)(aligned ? c[2] / lmax : c[2]) << 42) | morton(c[0], c[1], 0);
      };
      auto order = [&](std::vector<std::vector<int>>& ps) {
        std::stable_sort(ps.begin(), ps.end(), [&](const std::vector<int>& x, const std::vector<int>& y) {
          if (!aligned && x.size() != y.size()) return x.size() > y.size();
          return key(x) < key(y);
        });
      };
      order(pens);
      std::vector<int> base;
      for (auto& p : pens) base.push_back((int)p.size());
      long best = makespan(base);
      // wave tail: CTAs start in launch order on the S slots; the last wave of long pencils
      // can leave most slots idle.  Split the last k pencils into 1-block pencils, launched
      // last, for the k that minimises the makespan of the list schedule.  cfg5 level 2
      // (2768 blocks, 2.3 waves of 2-block pencils): k = 200, sweep 85.4 -> 76.0 us, fused
      // residual + restriction 77 -> 72 us; level 4 (aligned): k = 96 of 6732, sweep 497 ->
      // 492 us
      if (lmax_force || lmax < 2) return best;
      const int n = (int)pens.size();
      int bestk = 0;
      if (!aligned) {
        int nlong = 0;
        while (nlong < n && (int)pens[nlong].size() == lmax) ++nlong;
        for (int k = 1; k <= std::min(nlong, 2 * S); ++k) {
          std::vector<int> lens(base.begin(), base.begin() + (nlong - k));
          for (int i = 0; i < k * lmax; ++i) lens.push_back(1);
          for (int i = nlong; i < n; ++i) lens.push_back(base[i]);
          std::stable_sort(lens.begin(), lens.end(), std::greater<int>());
          const long m = makespan(lens);
          if (m < best) best = m, bestk = k;
        }
        if (bestk > 0) {
          std::vector<std::vector<int>> out(pens.begin(), pens.begin() + (nlong - bestk));
          for (int i = nlong - bestk; i < n; ++i)
            for (int b : pens[i]) out.push_back({b});
          pens.swap(out);
          order(pens);
        }
      } else {
        for (int k = 8; k <= std::min(n, 2 * S); k += 8) {
          std::vector<int> lens(base.begin(), base.begin() + (n - k));
          for (int i = n - k; i < n; ++i)
            for (int t = 0; t < base[i]; ++t) lens.push_back(1);
          const long m = makespan(lens);
          if (m < best) best = m, bestk = k;
        }
        if (bestk > 0) {
          std::vector<std::vector<int>> out(pens.begin(), pens.begin() + (n - bestk));
          for (int i = n - bestk; i < n; ++i)
            for (int b : pens[i]) out.push_back({b});
          pens.swap(out);
        }
      }
      return best;
    };
    const bool aligned = h->d.pencil_order ? h->d.pencil_order == 2 : W >= 24;
    // W <= 1: one wave of 1-block pencils (20 plane steps); 1 < W < 8: 2 (one wave of 36 steps
    // instead of two of 20 for W <= 2: cfg4 levels 1 and 2, 768 and 936 blocks, sweeps 31.0 ->
    // 27.6 and 36.5 -> 32.0 us, V-cycle 0.710 -> 0.674 ms; cfg5 level 1, 1152 blocks, 38.7 ->
    // 34.3 us).  Choosing among 1, 2, 3 by the makespan model alone picked 3 for cfg3's 4096
    // blocks: 105.7 vs 102.0 us, so the measured thresholds stay.
    const int lmax = lmax_force ? lmax_force
                                : ((W >= 4 && long_runs) || W >= 24 ? 4 : (W >= 8 ? 3 : (W > 1.0 ? 2 : 1)));
    std::vector<std::vector<int>> pens;
    construct(lmax, aligned, pens);
    l.pen_lmax = lmax;
    // every real block in exactly one pencil, each pencil a z-run of one column
    {
      std::vector<char> seen(l.nreal, 0);
      size_t nb = 0;
      for (auto& p : pens) {
        if (p.empty() || (int)p.size() > lmax) throw MgError(MG_ERR_STATE, "pencil list: bad length");
        for (size_t t = 0; t < p.size(); ++t, ++nb) {
          const auto &c = l.coords[p[t]], &c0 = l.coords[p[0]];
          if (seen[p[t]]++ || c[0] != c0[0] || c[1] != c0[1] || c[2] != c0[2] + (int)t)
            throw MgError(MG_ERR_STATE, "pencil list: not a partition into z-runs");
        }
      }
      if (nb != (size_t)l.nreal) throw MgError(MG_ERR_STATE, "pencil list: blocks missing");
    }
    for (auto& p : pens) {
      l.pen_len.push_back((int32_t)p.size());
      for (int t = 0; t < lmax; ++t) l.pen_blk.push_back(t < (int)p.size() ? p[t] : -1);
    }
    // sweep pencils: a level with fewer blocks than SMs splits every block into 2
    // z-parts of 8 planes (twice the CTAs, 12 steps each; cfg2 64^3 level: 58 -> 50 us
    // per 4 sweeps; at 512 blocks the split is slower)
    l.sw_blk.clear();
    l.sw_len.clear();
    l.sw_z.clear();
    const bool zsplit = h->d.zsplit == 2 || (h->d.zsplit == 0 && l.nreal < nsm);
    if (lmax == 1 && zsplit) {
      for (int32_t b : l.pen_blk)
        for (int z0 = 0; z0 < 16; z0 += 8) {
          l.sw_blk.push_back(b);
          l.sw_len.push_back(1);
          l.sw_z.push_back(z0 | (8 << 8));
        }
    }
  }
}

void alloc_device(mg_handle* h) {
  for (auto& l : h->L) {
    const size_t n = (size_t)h->nc * l.ntot() * l.B3;
    for (double** p : {&l.u[0], &l.u[1], &l.f, &l.r, &l.uhat}) {
      CUDA_OK(cudaMalloc(p, n * sizeof(double)));
      CUDA_OK(cudaMemsetAsync(*p, 0, n * sizeof(double), h->s));
    }
    l.d_nbr = dev_upload(l.nbr);
    l.d_nbr_real = dev_upload(l.nbr_real);
    l.d_nbr_ext = dev_upload(l.nbr_ext);
    l.d_covmask = dev_upload(l.covmask);
    l.d_parent = dev_upload(l.parent);
    l.d_bmap = dev_upload(l.bmap);
    l.d_c2f_dst = dev_upload(l.c2f_dst);
    l.d_c2f_J = dev_upload(l.c2f_J);
    l.d_c2f_ext = dev_upload(l.c2f_ext);
    l.d_inj_dst = dev_upload(l.inj_dst);
    l.d_inj_src = dev_upload(l.inj_src);
    l.d_chain_lev = dev_upload(l.chain_lev);
    l.d_chain_dst = dev_upload(l.chain_dst);
    l.d_chain_src = dev_upload(l.chain_src);
    l.d_pen_blk = dev_upload(l.pen_blk);
    l.d_pen_len = dev_upload(l.pen_len);
    l.d_gbox = dev_upload(l.gbox);
    l.d_sw_blk = dev_upload(l.sw_blk);
    l.d_sw_len = dev_upload(l.sw_len);
    l.d_sw_z = dev_upload(l.sw_z);
  }
  // TMA tensor maps of the B = 16 levels (RB sweep plane tiles) when TMA staging is
  // requested (mg_desc.staging = 1; cp.async otherwise, or without a tensor-map encoder)
  for (auto& l : h->L) {
    l.has_tmaps = false;
    if (l.B != 16 || h->d.staging != 1) continue;
    bool ok = true;
    for (int c = 0; c < 2 && ok; ++c)
      ok = encode_tile_maps(l.u[c], h->nc * l.ntot(), l.tmaps[c].u) && encode_tile_maps(l.f, h->nc * l.ntot(), l.tmaps[c].f);
    l.has_tmaps = ok;
  }
  // leaf map: leaf n -> (level, block)
  std::vector<int64_t> map(h->leaves.size());
  for (size_t n = 0; n < h->leaves.size(); ++n) {
    const auto& lf = h->leaves[n];
    const int m = h->nsub + lf[0];
    const int idx = h->L[m].find(lf[1], lf[2], lf[3]);
    map[n] = ((int64_t)m << 32) | (int64_t)idx;
  }
  h->d_leafmap = dev_upload(map);
  h->h_lvl_ptrs.assign(h->L.size(), nullptr);
  CUDA_OK(cudaMalloc(&h->d_lvl_ptrs, h->L.size() * sizeof(double*)));
  CUDA_OK(cudaMalloc(&h->d_norm, 2 * sizeof(unsigned long long)));
  const size_t nl = (size_t)h->nc * h->leaves.size() * h->d.block_size * h->d.block_size * h->d.block_size;
  CUDA_OK(cudaMalloc(&h->d_leafbuf, nl * sizeof(double)));
  CUDA_OK(cudaMalloc(&h->d_leafbuf2, nl * sizeof(double)));
  std::vector<int64_t> lcs;
  for (auto& l : h->L) lcs.push_back((int64_t)l.ntot() * l.B3);
  h->d_lvl_cs = dev_upload(lcs);
}

int smooth7(int n) {
  for (int m = std::max(n, 1);; ++m) {
    int r = m;
    for (int p : {2, 3, 5, 7})
      while (r % p == 0) r /= p;
    if (r == 1) return m;
  }
}

void setup_coarse(mg_handle* h) {
  Level& c = h->L[0];
  int nunb = 0;
  for (int a = 0; a < 3; ++a) {
    // semi-unbounded: the mirror-extended axis of 2N-1 nodes, solved as unbounded;
    // both faces symmetric: the odd (2N) or even-odd (4N) periodic extension (S2)
    const bool semi = h->sym[a] && !h->hi_odd[a] && !h->hi_even[a];
    const int Ne = semi ? 2 * c.N[a] - 1 : c.N[a];
    h->coff[a] = semi ? c.N[a] - 1 : 0;
    if (h->hi_odd[a]) h->P[a] = (h->sym[a] < 0 ? 2 : 4) * c.N[a];
    else if (h->hi_even[a]) h->P[a] = 2 * (c.N[a] - 1);  // even extension about nodes 0 and N-1
    else h->P[a] = h->per[a] ? c.N[a] : smooth7(2 * Ne + 2 * h->GE - 1);
    nunb += !h->fper[a];
  }
  // 0: all periodic (spectral, zero mode -> 0); 1: all unbounded (3D LGF table);
  // 2: any other mix (generalised E14: lower-dimensional LGF on zero periodic
  //    wavenumbers, 1/σ elsewhere; reading Z22)
  h->coarse_kind = nunb == 0 ? 0 : (nunb == 3 ? 1 : 2);
  const int Px = h->P[0], Py = h->P[1], Pz = h->P[2];
  const int64_t nd = (int64_t)Px * Py * Pz, nc = (int64_t)(Px / 2 + 1) * Py * Pz;
  h->pruned = h->coarse_kind == 2 && h->per[0] && !h->per[1] && !h->per[2] && !h->sym[0] && !h->sym[1] &&
               !h->sym[2] && !h->hi_odd[0] && !h->hi_even[0] && h->d.coarse_pruning != 1;
  // one batched transform over the components (dense [ncomp][Pz][Py][Px])
  CUDA_OK(cudaMalloc(&h->d_dense, (size_t)h->nc * nd * sizeof(double)));
  CUDA_OK(cudaMalloc(&h->d_spec, (size_t)h->nc * nc * sizeof(cufftDoubleComplex)));
  {
    int dims[3] = {Pz, Py, Px};
    CUFFT_OK(cufftPlanMany(&h->plan_f, 3, dims, nullptr, 1, (int)nd, nullptr, 1, (int)nc, CUFFT_D2Z, h->nc));
    CUFFT_OK(cufftPlanMany(&h->plan_b, 3, dims, nullptr, 1, (int)nc, nullptr, 1, (int)nd, CUFFT_Z2D, h->nc));
  }
  CUFFT_OK(cufftSetStream(h->plan_f, h->s));
  CUFFT_OK(cufftSetStream(h->plan_b, h->s));
  const double sc = c.h * c.h / (double)nd;
  if (h->coarse_kind == 1) {
    const int R = std::max(Px, std::max(Py, Pz)) / 2 + 8;
    std::vector<double> G = box_lgf(3, h->order, R);
    const int n = 2 * R + 1;
    std::vector<double> T(nd);
    for (int z = 0; z < Pz; ++z)
      for (int y = 0; y < Py; ++y)
        for (int x = 0; x < Px; ++x) {
          const int nx = x <= Px / 2 ? x : x - Px, ny = y <= Py / 2 ? y : y - Py, nz = z <= Pz / 2 ? z : z - Pz;
          T[((size_t)z * Py + y) * Px + x] = G[((size_t)(nz + R) * n + (ny + R)) * n + (nx + R)];
        }
    CUDA_OK(cudaMemcpy(h->d_dense, T.data(), nd * sizeof(double), cudaMemcpyHostToDevice));
    {  // one (unbatched) transform of the LGF table
      cufftHandle p1;
      CUFFT_OK(cufftPlan3d(&p1, Pz, Py, Px, CUFFT_D2Z));
      CUFFT_OK(cufftSetStream(p1, h->s));
      CUFFT_OK(cufftExecD2Z(p1, h->d_dense, (cufftDoubleComplex*)h->d_spec));
      CUDA_OK(cudaStreamSynchronize(h->s));
      cufftDestroy(p1);
    }
    CUDA_OK(cudaMalloc(&h->d_mult, nc * sizeof(double)));
    launch_real_part_scale(h->d_spec, h->d_mult, nc, sc, h->s);
  } else if (h->coarse_kind == 2) {
    int ua = -1, ub = -1;  // the unbounded axes (ub = -1: only one)
    for (int a = 0; a < 3; ++a)
      if (!h->fper[a]) (ua < 0 ? ua : ub) = a;
    double* dLow = nullptr;  // transform of the lower-dimensional LGF, x h^2 / (Px Py Pz)
    if (ub >= 0) {
      const int Pa = h->P[ua], Pb = h->P[ub];
      const int R = std::max(Pa, Pb) / 2 + 8;
      std::vector<double> G = box_lgf(2, h->order, R);
      const int n = 2 * R + 1;
      std::vector<cufftDoubleComplex> T((size_t)Pa * Pb);
      for (int j = 0; j < Pb; ++j)
        for (int i = 0; i < Pa; ++i) {
          const int ni = i <= Pa / 2 ? i : i - Pa, nj = j <= Pb / 2 ? j : j - Pb;
          // G index (first, second) = (axis ua, axis ub), matching the oracle's box layout
          T[(size_t)j * Pa + i] = make_cuDoubleComplex(G[(size_t)(ni + R) * n + (nj + R)], 0.0);
        }
      cufftDoubleComplex* dT = nullptr;
      CUDA_OK(cudaMalloc(&dT, T.size() * sizeof(cufftDoubleComplex)));
      CUDA_OK(cudaMemcpy(dT, T.data(), T.size() * sizeof(cufftDoubleComplex), cudaMemcpyHostToDevice));
      cufftHandle p2;
      CUFFT_OK(cufftPlan2d(&p2, Pb, Pa, CUFFT_Z2Z));
      CUFFT_OK(cufftSetStream(p2, h->s));
      CUFFT_OK(cufftExecZ2Z(p2, dT, dT, CUFFT_FORWARD));
      CUDA_OK(cudaMalloc(&dLow, T.size() * sizeof(double)));
      launch_real_part_scale(dT, dLow, (int64_t)T.size(), sc, h->s);
      CUDA_OK(cudaStreamSynchronize(h->s));
      cufftDestroy(p2);
      cudaFree(dT);
    } else {
      // one unbounded axis: the 1D LGF |n|/2 (δ²(|n|/2) = δ), transformed by a direct DFT
      const int P = h->P[ua];
      std::vector<double> T1(P);
      for (int k = 0; k < P; ++k) {
        double acc = 0.0;
        for (int i = 0; i < P; ++i) {
          const int ni = i <= P / 2 ? i : i - P;
          acc += 0.5 * std::abs(ni) * std::cos(2.0 * M_PI * (double)((int64_t)k * i % P) / P);
        }
        T1[k] = acc * sc;
      }
      dLow = dev_upload(T1);
    }
    CUDA_OK(cudaMalloc(&h->d_mult, nc * sizeof(double)));
    launch_build_mult(h->d_mult, h->P, h->fper, ua, ub, dLow, h->order, c.h * c.h, 1.0 / (double)nd, 0, h->s);
    if (h->pruned) {
      // the same multipliers in the [kz][kx][ky] layout of the pruned transforms
      CUDA_OK(cudaMalloc(&h->pr_mult, nc * sizeof(double)));
      launch_build_mult(h->pr_mult, h->P, h->fper, ua, ub, dLow, h->order, c.h * c.h, 1.0 / (double)nd, 1, h->s);
    }
    CUDA_OK(cudaStreamSynchronize(h->s));
    cudaFree(dLow);
  }
  CUDA_OK(cudaStreamSynchronize(h->s));
  if (h->pruned) {
    const int Nx = c.N[0], Ny = c.N[1], Nz = c.N[2], Hx = Nx / 2 + 1, Py = h->P[1], Pz = h->P[2], GE = h->GE;
    const int Wy = Ny + 2 * GE, Wz = Nz + 2 * GE, nc = h->nc;
    h->pr_W[0] = Nx;
    h->pr_W[1] = Wy;
    h->pr_W[2] = Wz;
    const size_t cz = sizeof(cufftDoubleComplex);
    CUDA_OK(cudaMalloc(&h->pr_X, (size_t)nc * Nz * Ny * Nx * sizeof(double)));
    CUDA_OK(cudaMalloc(&h->pr_C1, (size_t)nc * Nz * Ny * Hx * cz));
    CUDA_OK(cudaMalloc(&h->pr_C2, (size_t)nc * Pz * Hx * Py * cz));
    CUDA_OK(cudaMalloc(&h->pr_C3, (size_t)nc * Wz * Wy * Hx * cz));
    CUDA_OK(cudaMalloc(&h->pr_R, (size_t)nc * Wz * Wy * Nx * sizeof(double)));
    int n1 = Nx;
    CUFFT_OK(cufftPlanMany(&h->pr_xf, 1, &n1, nullptr, 1, Nx, nullptr, 1, Hx, CUFFT_D2Z, nc * Nz * Ny));
    CUFFT_OK(cufftPlanMany(&h->pr_xb, 1, &n1, nullptr, 1, Hx, nullptr, 1, Nx, CUFFT_Z2D, nc * Wz * Wy));
    int ny = Py, nz = Pz, emb = Pz;
    CUFFT_OK(cufftPlanMany(&h->pr_y, 1, &ny, nullptr, 1, Py, nullptr, 1, Py, CUFFT_Z2Z, Nz * Hx));
    CUFFT_OK(cufftPlanMany(&h->pr_y1, 1, &ny, nullptr, 1, Py, nullptr, 1, Py, CUFFT_Z2Z, (Nz + GE) * Hx));
    CUFFT_OK(cufftPlanMany(&h->pr_y2, 1, &ny, nullptr, 1, Py, nullptr, 1, Py, CUFFT_Z2Z, GE * Hx));
    CUFFT_OK(cufftPlanMany(&h->pr_z, 1, &nz, &emb, Hx * Py, 1, &emb, Hx * Py, 1, CUFFT_Z2Z, Hx * Py));
    for (cufftHandle* p : {&h->pr_xf, &h->pr_xb, &h->pr_y, &h->pr_y1, &h->pr_y2, &h->pr_z})
      CUFFT_OK(cufftSetStream(*p, h->s));
    // fused y / z transforms (mg_desc.coarse_pruning 2; measured slower than the cuFFT
    // passes of the default)
    std::vector<double> twy, twz;
    h->fused_fft = h->d.coarse_pruning == 2 && fft_plan(Py, h->fp_y, twy) && fft_plan(Pz, h->fp_z, twz) &&
                   Py <= 880 && Pz <= 880;  // mg_fft.cu FT_MAXN
    if (h->fused_fft) {
      h->d_twy = dev_upload(twy);
      h->d_twz = dev_upload(twz);
    }
  }
  // level-0 exterior f ghosts beyond symmetric low faces: signed mirror copies of real
  // level-0 nodes (f := 0 beyond unbounded faces, Z16; reading S1)
  if (h->sym[0] || h->sym[1] || h->sym[2]) {
    const Level& l = h->L[0];  // f beyond odd / even high faces mirrors too (S2, S3)
    for (size_t e = 0; e < l.c2f_dst.size(); ++e) {
      int J[3] = {l.c2f_J[3 * e], l.c2f_J[3 * e + 1], l.c2f_J[3 * e + 2]};
      int sg = 1;
      bool zero = false;
      for (int a = 0; a < 3 && !zero; ++a) {
        if (h->per[a]) continue;
        if ((J[a] >= l.N[a] && !h->hi_odd[a] && !h->hi_even[a]) || (J[a] < 0 && !h->sym[a]))
          zero = true;  // beyond an unbounded face
        else if (J[a] < 0) {
          J[a] = -J[a];
          sg *= h->sym[a];
        } else if (J[a] >= l.N[a] && h->hi_even[a]) {  // even high face: f(N-1+k) = f(N-1-k)
          J[a] = 2 * (l.N[a] - 1) - J[a];
        } else if (J[a] >= l.N[a]) {   // odd high face: f(N) = 0, f(N + k) = -f(N - k)
          if (J[a] == l.N[a]) zero = true;
          J[a] = 2 * l.N[a] - J[a];
          sg = -sg;
        }
      }
      if (zero) continue;
      int src;
      if (!is_real_node(h, l, J[0], J[1], J[2], &src)) continue;
      h->fm_dst.push_back(l.c2f_dst[e]);
      h->fm_src.push_back(src);
      h->fm_sgn.push_back((int8_t)sg);
    }
    h->d_fm_dst = dev_upload(h->fm_dst);
    h->d_fm_src = dev_upload(h->fm_src);
    h->d_fm_sgn = dev_upload(h->fm_sgn);
    // odd low faces: the wall-plane nodes (u = 0 there; their f is ignored)
    for (int i = 0; i < l.nreal; ++i)
      for (int loc = 0; loc < l.B3; ++loc) {
        const int q[3] = {loc % l.B, (loc / l.B) % l.B, loc / (l.B * l.B)};
        bool wall = false;
        for (int a = 0; a < 3; ++a)
          if (h->sym[a] < 0 && l.coords[i][a] * l.B + q[a] == 0) wall = true;
        if (wall) h->fwall.push_back(i * l.B3 + loc);
      }
    h->d_fwall = dev_upload(h->fwall);
  }
}

// ----------------------------------------------------------------------------------
// V-cycle building blocks
// ----------------------------------------------------------------------------------
void swap_u(Level& l) { l.cur = 1 - l.cur; }

// c2f of every ghost box of level m: thin boxes one warp each, thick boxes one CTA each
void c2f_boxes(mg_handle* h, int m, double* fine_field, const double* coarse_field, bool ext_zero) {
  Level& F = h->L[m];
  const int nbox = (int)F.gbox.size() / GBOX_REC;
  if (nbox == 0) return;
  const LevelView fv = view(h, m), cv = view(h, m - 1);
  launch_c2f_thin(fv, cv, F.d_gbox, F.gbox_nthin, fine_field, coarse_field, h->I, ext_zero, h->s);
  launch_c2f_box(fv, cv, F.d_gbox + (size_t)F.gbox_nthin * GBOX_REC, nbox - F.gbox_nthin, F.gbox_szA, F.gbox_szB,
                 fine_field, coarse_field, h->I, ext_zero, h->s);
}

// boundary-ghost refresh of level m (reading Z9): f2c injection into level m-1,
// then c2f; exterior chains (reading U1) refresh every coarser level first.
void refresh(mg_handle* h, int m) {
  if (m <= 0) return;
  const int lo = h->L[m].ext_chain ? 1 : m;
  bool any = false;
  for (int j = lo; j <= m; ++j) any = any || !h->L[j].inj_dst.empty() || !h->L[j].gbox.empty();
  if (!any) return;  // ghost-free level (no events either: keeps the stage profile honest)
  Prof pr(h, ST_GHOST, m);
  if (lo < m && m < MAX_CHAIN_LEVELS && !h->L[m].chain_dst.empty()) {
    double* fields[MAX_CHAIN_LEVELS] = {};
    int64_t cs[MAX_CHAIN_LEVELS] = {};
    for (int j = 0; j <= m && j < MAX_CHAIN_LEVELS; ++j) {
      fields[j] = h->L[j].u[h->L[j].cur];
      cs[j] = (int64_t)h->L[j].ntot() * h->L[j].B3;
    }
    const Level& T = h->L[m];
    launch_inject_chain((int)T.chain_dst.size(), T.d_chain_lev, T.d_chain_dst, T.d_chain_src, fields, cs, h->nc, h->s);
  } else {
    for (int j = m; j >= lo; --j) {
      Level &F = h->L[j], &C = h->L[j - 1];
      if (!F.inj_dst.empty())
        launch_inject_list(inj_list(F), C.u[C.cur], F.u[F.cur], h->nc, (int64_t)C.ntot() * C.B3, (int64_t)F.ntot() * F.B3,
                           h->s);
    }
  }
  for (int j = lo; j <= m; ++j) c2f_boxes(h, j, h->L[j].u[h->L[j].cur], h->L[j - 1].u[h->L[j - 1].cur], false);
}

bool has_ghosts(mg_handle* h, int m) { return m > 0 && h->L[m].n_c2f > 0; }

// r = f - Δu on all level-m nodes (ghosts already refreshed)
void residual_kernel(mg_handle* h, int m) {
  const LevelView v = view(h, m);
  if (!launch_res_pencil(v, h->order, h->s)) launch_residual(v, h->order, h->s);
}

// fresh: the boundary ghosts of level m are current (refreshed since the last write of
// u on levels m and m-1), so the refresh before the sweep is skipped
void sweep(mg_handle* h, int m, bool with_res, bool fresh = false) {
  if (!fresh) refresh(h, m);
  Level& l = h->L[m];
  const int mode = h->smoother == MG_SMOOTHER_RBGS ? SM_RB : SM_JACOBI;
  // Fuse the residual into the last sweep only on small-block levels: on B = 16
  // levels the halo-3 fused tile is shared-memory-bound, so a
  // halo-2 sweep plus a separate residual pass is faster there.
  const bool fuse = l.B < 16 && h->d.fuse != 1;
  if (with_res && !has_ghosts(h, m) && fuse) {
    Prof pr(h, ST_SMOOTH_RES, m);
    launch_smooth(view(h, m), h->order, mode, h->omega, true, h->s);
    swap_u(l);
    return;
  }
  {
    Prof pr(h, ST_SMOOTH, m);
    const LevelView v = view(h, m);
    if (mode != SM_RB || !launch_rb_pencil(v, h->order, h->omega, l.has_tmaps ? &l.tmaps[l.cur] : nullptr, h->s))
      launch_smooth(v, h->order, mode, h->omega, false, h->s);
    swap_u(l);
  }
  if (with_res) {
    refresh(h, m);
    Prof pr(h, ST_RESIDUAL, m);
    residual_kernel(h, m);
  }
}

// Restriction of level m into m-1 (Alg. 1) starting from refreshed level-m
// ghosts: residual + u injection + full weighting (fused in one pencil kernel on B = 16
// levels; else residual kernel + restriction kernel), then the level-(m-1) refresh,
// FAS right-hand side and the û snapshot.
// Fused residual + restriction (k_rr2_pencil) on B = 16 levels: the fine residual is
// never written to HBM (cfg2 256^3: 127 us instead of 90 + 62 us); mg_desc.fuse = 1
// selects the two-kernel path.
bool fused_res_restrict(mg_handle* h, int m) { return h->d.fuse != 1 && h->L[m].B == 16; }

void restrict_level(mg_handle* h, int m) {
  Level& C = h->L[m - 1];
  bool done = false;
  if (fused_res_restrict(h, m)) {
    Prof pr(h, ST_RESTRICT, m);
    done = launch_res_restrict_pencil(view(h, m), view(h, m - 1), h->order, h->s);
  }
  if (!done) {
    {
      Prof pr(h, ST_RESIDUAL, m);
      residual_kernel(h, m);
    }
    Prof pr(h, ST_RESTRICT, m);
    launch_restrict(view(h, m), view(h, m - 1), h->s);
  }
  refresh(h, m - 1);
  Prof pr(h, ST_FAS, m - 1);  // FAS right-hand side + û of the coarse level (its unknowns)
  if (launch_fas_pencil(view(h, m - 1), h->order, h->s)) {
    // the pencil FAS kernel wrote û on the real blocks; the prolongation also takes ε on
    // the exterior band (reading Z13-W, U1 / level 0), stored in the ghost blocks
    if (C.has_ext_ghosts) {  // the ghost part of every component
      const size_t pitch = (size_t)C.ntot() * C.B3 * sizeof(double);
      CUDA_OK(cudaMemcpy2DAsync(C.uhat + (size_t)C.nreal * C.B3, pitch, C.u[C.cur] + (size_t)C.nreal * C.B3, pitch,
                                (size_t)C.nghost * C.B3 * sizeof(double), h->nc, cudaMemcpyDeviceToDevice, h->s));
    }
  } else {
    launch_fas_rhs(view(h, m), view(h, m - 1), h->order, h->s);
    CUDA_OK(cudaMemcpyAsync(C.uhat, C.u[C.cur], (size_t)h->nc * C.ntot() * C.B3 * sizeof(double),
                            cudaMemcpyDeviceToDevice, h->s));
  }
}

// u_m += P(u - û)_{m-1} (Alg. 1).  Under U1 the exterior band of level m-1
// enters ε (current exterior value minus its snapshot, Z13-W): refresh it first.
void prolong_level(mg_handle* h, int m) {
  if (m - 1 >= 1 && h->L[m - 1].ext_chain) refresh(h, m - 1);
  Prof pr(h, ST_PROLONG, m);
  launch_prolong(view(h, m), view(h, m - 1), h->s);
}

// The x-periodic, y/z-unbounded solve with 1-D transforms (the 3-D R2C factorised, so the
// multiplier and the values are those of the 3-D path up to rounding): R2C along x of
// the N^3 source only; along y (zero-padded to Py) only the Nz source planes; along z
// every line; the multiplier; back along z every line, along y only the planes of the
// output window z in [-GE, N + GE); C2R along x only the (z, y) window lines.  The zero
// half of the padded source and the outputs nobody reads are never transformed.
void coarse_solve_pruned(mg_handle* h) {
  Prof pr(h, ST_COARSE, 0);
  LevelView c = view(h, 0);
  const Level& l0 = h->L[0];
  const int Nx = l0.N[0], Ny = l0.N[1], Nz = l0.N[2], Hx = Nx / 2 + 1, Py = h->P[1], Pz = h->P[2], GE = h->GE;
  const int N[3] = {Nx, Ny, Nz}, zero[3] = {0, 0, 0};
  launch_coarse_gather(c, h->pr_X, N, zero, zero, zero, zero, h->s);
  CUFFT_OK(cufftExecD2Z(h->pr_xf, h->pr_X, (cufftDoubleComplex*)h->pr_C1));
  if (h->fused_fft) {
    // y FFT (zero padding implicit), z FFT x multiplier x inverse z FFT (window rows),
    // inverse y FFT + window, each one kernel (mg_fft.cu)
    launch_fft_y_fwd(h->pr_C1, h->pr_C2, Ny, Nz, Hx, Pz, h->fp_y, h->d_twy, h->nc, h->s);
    launch_fft_z_conv(h->pr_C2, h->pr_mult, Hx * Py, Nz, GE, h->fp_z, h->d_twz, h->nc, h->s);
    launch_fft_y_inv(h->pr_C2, h->pr_C3, Hx, Pz, h->pr_W[1], h->pr_W[2], GE, h->fp_y, h->d_twy, h->nc, h->s);
  } else {
    launch_spec_pad_y(h->pr_C1, h->pr_C2, Nz, Ny, Hx, Py, Pz, h->nc, h->s);
    const size_t plane = (size_t)Hx * Py, comp = (size_t)Pz * plane;
    auto C2 = [&](int cc, int z) { return (cufftDoubleComplex*)h->pr_C2 + cc * comp + (size_t)z * plane; };
    for (int cc = 0; cc < h->nc; ++cc) {
      CUDA_OK(cudaMemsetAsync(C2(cc, Nz), 0, (size_t)(Pz - Nz) * plane * sizeof(cufftDoubleComplex), h->s));
      CUFFT_OK(cufftExecZ2Z(h->pr_y, C2(cc, 0), C2(cc, 0), CUFFT_FORWARD));
      CUFFT_OK(cufftExecZ2Z(h->pr_z, C2(cc, 0), C2(cc, 0), CUFFT_FORWARD));
    }
    launch_coarse_mul_table(h->pr_C2, h->pr_mult, (int64_t)comp, h->nc, h->s);
    for (int cc = 0; cc < h->nc; ++cc) {
      CUFFT_OK(cufftExecZ2Z(h->pr_z, C2(cc, 0), C2(cc, 0), CUFFT_INVERSE));
      CUFFT_OK(cufftExecZ2Z(h->pr_y1, C2(cc, 0), C2(cc, 0), CUFFT_INVERSE));
      CUFFT_OK(cufftExecZ2Z(h->pr_y2, C2(cc, Pz - GE), C2(cc, Pz - GE), CUFFT_INVERSE));
    }
    launch_spec_window(h->pr_C2, h->pr_C3, h->pr_W[2], h->pr_W[1], Hx, Py, Pz, GE, h->nc, h->s);
  }
  CUFFT_OK(cufftExecZ2D(h->pr_xb, (cufftDoubleComplex*)h->pr_C3, h->pr_R));
  const int off[3] = {0, GE, GE};
  launch_coarse_scatter(c, h->pr_R, h->pr_W, off, c2f_list(h->L[0]), h->s);
}

void coarse_solve(mg_handle* h) {
  if (h->pruned) {
    coarse_solve_pruned(h);
    return;
  }
  Prof pr(h, ST_COARSE, 0);
  LevelView c = view(h, 0);
  launch_coarse_gather(c, h->d_dense, h->P, h->sym, h->hi_odd, h->hi_even, h->coff, h->s);
  CUFFT_OK(cufftExecD2Z(h->plan_f, h->d_dense, (cufftDoubleComplex*)h->d_spec));
  if (h->coarse_kind == 0) launch_coarse_mul_periodic(h->d_spec, h->P, h->order, h->L[0].h, h->nc, h->s);
  else launch_coarse_mul_table(h->d_spec, h->d_mult, (int64_t)(h->P[0] / 2 + 1) * h->P[1] * h->P[2], h->nc, h->s);
  CUFFT_OK(cufftExecZ2D(h->plan_b, (cufftDoubleComplex*)h->d_spec, h->d_dense));
  launch_coarse_scatter(c, h->d_dense, h->P, h->coff, c2f_list(h->L[0]), h->s);
}

void inject_up_all(mg_handle* h) {
  Prof pr(h, ST_INJECT_UP, 0);
  for (int m = (int)h->L.size() - 1; m >= 1; --m)
    launch_inject_up(view(h, m), view(h, m - 1), h->L[m - 1].u[h->L[m - 1].cur], h->s);
}

void vcycle_body(mg_handle* h) {
  const int top = (int)h->L.size() - 1;
  for (int m = top; m >= 1; --m) {
    // below the top, restrict_level(m + 1) has just refreshed level m (the FAS kernel
    // after it writes f and û only): the first pre-sweep's refresh would recompute the
    // same ghost values
    bool fresh = m < top;
    for (int k = 1; k <= h->eta1; ++k) {
      sweep(h, m, false, fresh);
      fresh = false;
    }
    if (!fresh) refresh(h, m);
    restrict_level(h, m);
  }
  coarse_solve(h);
  for (int m = 1; m <= top; ++m) {
    prolong_level(h, m);
    for (int k = 0; k < h->eta2; ++k) sweep(h, m, false);
  }
  // Inject-up (a8) is deferred to the next consumer of coarse covered values that is
  // not itself preceded by a re-injection (mg_residual_norm): the next V-cycle
  // overwrites every covered coarse node (f2c lists, restriction) before reading it,
  // so the cycle's results are identical with or without it.
  h->canonical = false;
  if ((h->eta1 + h->eta2) & 1) {
    // keep the buffer parity fixed per cycle (so one captured graph can be replayed)
    for (int m = 1; m <= top; ++m) {
      Level& l = h->L[m];
      CUDA_OK(cudaMemcpyAsync(l.u[1 - l.cur], l.u[l.cur], (size_t)h->nc * l.ntot() * l.B3 * sizeof(double),
                              cudaMemcpyDeviceToDevice, h->s));
      swap_u(l);
    }
  }
}

void run_vcycles(mg_handle* h, int n) {
  if (!h->use_graph) {
    for (int i = 0; i < n; ++i) vcycle_body(h);
    return;
  }
  // the captured graph bakes in the ping-pong parity of every level's u buffers:
  // re-capture if it changed since (debug single sweeps, set_solution)
  int sig = 0;
  for (size_t m = 0; m < h->L.size(); ++m) sig |= h->L[m].cur << (m % 30);
  if (h->gexec && sig != h->graph_cur_sig) {
    cudaGraphExecDestroy(h->gexec);
    h->gexec = nullptr;
  }
  h->graph_cur_sig = sig;
  if (!h->gexec) {
    // capture on a private stream (the caller's may be the legacy default stream,
    // which cannot be captured), replay on the caller's stream
    cudaStream_t orig = h->s, cap = nullptr;
    CUDA_OK(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    const bool prof = h->prof_on;
    cudaGraph_t g = nullptr;
    // restores the handle (stream, cuFFT streams, profiling) and frees the capture
    // objects on every exit path, the exception path included
    auto restore = [&] {
      h->s = orig;
      h->prof_on = prof;
      for (cufftHandle* p : h->plans())
        if (*p) cufftSetStream(*p, orig);
      if (g) cudaGraphDestroy(g);
      g = nullptr;
      if (cap) cudaStreamDestroy(cap);
      cap = nullptr;
    };
    try {
      CUDA_OK(cudaStreamSynchronize(orig));
      h->s = cap;
      h->prof_on = false;
      for (cufftHandle* p : h->plans())
        if (*p) CUFFT_OK(cufftSetStream(*p, cap));
      CUDA_OK(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
      try {
        vcycle_body(h);
      } catch (...) {
        cudaStreamEndCapture(cap, &g);
        throw;
      }
      CUDA_OK(cudaStreamEndCapture(cap, &g));
      CUDA_OK(cudaGraphInstantiate(&h->gexec, g, 0));
    } catch (...) {
      restore();
      h->gexec = nullptr;
      cudaGetLastError();  // clear a sticky capture error
      throw;
    }
    restore();
  }
  for (int i = 0; i < n; ++i) CUDA_OK(cudaGraphLaunch(h->gexec, h->s));
}

double read_norm(mg_handle* h) {
  unsigned long long bits = 0;
  CUDA_OK(cudaMemcpyAsync(&bits, h->d_norm, sizeof(bits), cudaMemcpyDeviceToHost, h->s));
  CUDA_OK(cudaStreamSynchronize(h->s));
  double v;
  std::memcpy(&v, &bits, sizeof(v));
  if (!std::isfinite(v)) throw MgError(MG_ERR_NONFINITE, "non-finite value in norm");
  return v;
}

double residual_abs(mg_handle* h) {
  if (!h->canonical) {
    inject_up_all(h);
    h->canonical = true;
  }
  CUDA_OK(cudaMemsetAsync(h->d_norm, 0, sizeof(unsigned long long), h->s));
  for (int m = 0; m < (int)h->L.size(); ++m) {
    refresh(h, m);
    Prof pr(h, ST_NORM, m);
    const LevelView v = view(h, m);
    if (!launch_norm_pencil(v, h->order, h->d_norm, h->s)) launch_norm(v, h->order, true, h->d_norm, h->s);
  }
  return read_norm(h);
}

void set_level_ptrs(mg_handle* h, int field) {
  for (size_t m = 0; m < h->L.size(); ++m) {
    Level& l = h->L[m];
    h->h_lvl_ptrs[m] = field == MG_FIELD_F ? l.f : l.u[l.cur];
  }
  CUDA_OK(cudaMemcpyAsync(h->d_lvl_ptrs, h->h_lvl_ptrs.data(), h->L.size() * sizeof(double*), cudaMemcpyHostToDevice,
                          h->s));
}

// max|u_new - u_old| / max|u_new| over leaf nodes (E20; zero-norm guard:
// the absolute increment when u_new = 0), u_old in d_leafbuf2 (replaced by u_new)
double cauchy_increment(mg_handle* h) {
  set_level_ptrs(h, MG_FIELD_U);
  CUDA_OK(cudaMemsetAsync(h->d_norm, 0, 2 * sizeof(unsigned long long), h->s));
  launch_leaf_cauchy((int)h->leaves.size(), h->d.block_size * h->d.block_size * h->d.block_size, h->d_leafmap,
                     h->d_leafbuf2, h->d_lvl_ptrs, h->d_lvl_cs, h->nc, h->d_norm, h->s);
  unsigned long long bits[2];
  CUDA_OK(cudaMemcpyAsync(bits, h->d_norm, sizeof(bits), cudaMemcpyDeviceToHost, h->s));
  CUDA_OK(cudaStreamSynchronize(h->s));
  double dm, um;
  std::memcpy(&dm, &bits[0], sizeof(dm));
  std::memcpy(&um, &bits[1], sizeof(um));
  if (!std::isfinite(dm) || !std::isfinite(um)) throw MgError(MG_ERR_NONFINITE, "non-finite value in the Cauchy increment");
  return um > 0 ? dm / um : dm;
}

void leaf_io(mg_handle* h, double* leafbuf, bool to_levels, int field) {
  set_level_ptrs(h, field);
  launch_leaf_scatter((int)h->leaves.size(), h->d.block_size * h->d.block_size * h->d.block_size, h->d_leafmap,
                      leafbuf, h->d_lvl_ptrs, h->d_lvl_cs, h->nc, to_levels, h->s);
  // the pointer table is reused by the next call: order it on the stream
  CUDA_OK(cudaStreamSynchronize(h->s));
}

void set_rhs(mg_handle* h, const double* f_dev) {
  const int nlev = (int)h->L.size();
  // u := 0 (initial solution, Z28), f := 0 (ghost nodes beyond unbounded faces); r is
  // zeroed after the right-hand-side correction, û is written by every restriction
  // before a prolongation reads it
  for (auto& l : h->L) {
    const size_t n = (size_t)h->nc * l.ntot() * l.B3;
    CUDA_OK(cudaMemsetAsync(l.f, 0, n * sizeof(double), h->s));
    CUDA_OK(cudaMemsetAsync(l.u[0], 0, n * sizeof(double), h->s));
    CUDA_OK(cudaMemsetAsync(l.u[1], 0, n * sizeof(double), h->s));
    l.cur = 0;
  }
  leaf_io(h, const_cast<double*>(f_dev), true, MG_FIELD_F);
  // f2c: inject f up the tree (O5)
  for (int m = nlev - 1; m >= 1; --m) {
    LevelView fv = view(h, m), cv = view(h, m - 1);
    fv.u = h->L[m].f;
    launch_inject_up(fv, cv, h->L[m - 1].f, h->s);
  }
  // f ghosts: c2f of f, f := 0 beyond unbounded faces (reading Z16)
  for (int m = 1; m < nlev; ++m) c2f_boxes(h, m, h->L[m].f, h->L[m - 1].f, true);
  const int64_t cs0 = (int64_t)h->L[0].ntot() * h->L[0].B3;
  if (!h->fwall.empty()) launch_fill_list((int)h->fwall.size(), h->d_fwall, h->L[0].f, 0.0, h->nc, cs0, h->s);
  if (!h->fm_dst.empty())
    launch_copy_signed((int)h->fm_dst.size(), h->d_fm_dst, h->d_fm_src, h->d_fm_sgn, h->L[0].f, h->L[0].f, h->nc, cs0,
                       h->s);
  for (int m = 0; m < nlev; ++m) {
    Level& l = h->L[m];
    if (launch_rhs_pencil(view(h, m), h->order, h->s)) {
      // r holds f* (leaves) / f (covered) on the real blocks: copy into f, per component
      const size_t pitch = (size_t)l.ntot() * l.B3 * sizeof(double);
      CUDA_OK(cudaMemcpy2DAsync(l.f, pitch, l.r, pitch, (size_t)l.nreal * l.B3 * sizeof(double), h->nc,
                                cudaMemcpyDeviceToDevice, h->s));
    } else {
      launch_correct_rhs(view(h, m), h->order, l.r, h->s);
    }
  }
  for (auto& l : h->L)
    CUDA_OK(cudaMemsetAsync(l.r, 0, (size_t)h->nc * l.ntot() * l.B3 * sizeof(double), h->s));
  CUDA_OK(cudaMemsetAsync(h->d_norm, 0, sizeof(unsigned long long), h->s));
  for (int m = 0; m < nlev; ++m) launch_norm(view(h, m), h->order, false, h->d_norm, h->s);
  h->fstar_norm = read_norm(h);
  h->rhs_set = true;
}

void destroy(mg_handle* h) {
  if (!h) return;
  cudaStreamSynchronize(h->s);
  prof_flush(h);
  for (auto e : h->evpool) cudaEventDestroy(e);
  for (auto& l : h->L) {
    for (void* p : {(void*)l.u[0], (void*)l.u[1], (void*)l.f, (void*)l.r, (void*)l.uhat, (void*)l.d_nbr,
                    (void*)l.d_nbr_real, (void*)l.d_nbr_ext, (void*)l.d_covmask, (void*)l.d_parent, (void*)l.d_bmap, (void*)l.d_c2f_dst,
                    (void*)l.d_c2f_J, (void*)l.d_c2f_ext, (void*)l.d_inj_dst, (void*)l.d_inj_src, (void*)l.d_pen_blk,
                    (void*)l.d_pen_len, (void*)l.d_gbox, (void*)l.d_sw_blk, (void*)l.d_sw_len, (void*)l.d_sw_z,
                    (void*)l.d_chain_lev, (void*)l.d_chain_dst, (void*)l.d_chain_src})
      if (p) cudaFree(p);
  }
  for (void* p : {(void*)h->d_fm_dst, (void*)h->d_fm_src, (void*)h->d_fm_sgn, (void*)h->d_fwall})
    if (p) cudaFree(p);
  for (void* p : {(void*)h->d_leafmap, (void*)h->d_lvl_ptrs, (void*)h->d_lvl_cs, (void*)h->d_norm, (void*)h->d_leafbuf,
                  (void*)h->d_leafbuf2, (void*)h->d_dense, h->d_spec, (void*)h->d_mult})
    if (p) cudaFree(p);
  for (cufftHandle* p : h->plans())
    if (*p) cufftDestroy(*p);
  for (void* p : {(void*)h->pr_X, (void*)h->pr_R, (void*)h->pr_mult, h->pr_C1, h->pr_C2, h->pr_C3, (void*)h->d_twy,
                  (void*)h->d_twz})
    if (p) cudaFree(p);
  if (h->gexec) cudaGraphExecDestroy(h->gexec);
  delete h;
}

template <class F>
int guard(mg_handle* h, F&& fn) {
  try {
    fn();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw MgError(MG_ERR_CUDA, cudaGetErrorString(e));
    return MG_OK;
  } catch (const MgError& e) {
    g_err = e.what();
    if (h) h->err = g_err;
    return e.code;
  } catch (const std::exception& e) {
    g_err = e.what();
    if (h) h->err = g_err;
    return MG_ERR_CUDA;
  }
}

}  // namespace

// ----------------------------------------------------------------------------------
// C-ABI
// ----------------------------------------------------------------------------------
extern "C" {

int mg_create(const mg_desc* d, void* stream, mg_handle** out) {
  if (!d || !out) {
    g_err = "null argument";
    return MG_ERR_ARG;
  }
  *out = nullptr;
  mg_handle* h = new mg_handle();
  h->d = *d;
  h->s = (cudaStream_t)stream;
  const int rc = guard(h, [&] {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) throw MgError(MG_ERR_CUDA, "no CUDA device");
    prepare_kernels();
    int dev = 0, nsm = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && nsm > 0)
      h->nsm = nsm;
    auto t0 = std::chrono::steady_clock::now();
    auto lap = [&](int i) {
      const auto t1 = std::chrono::steady_clock::now();
      h->setup_ms[i] = std::chrono::duration<double, std::milli>(t1 - t0).count();
      t0 = t1;
    };
    validate_and_build(h);
    lap(0);
    build_ghosts(h);
    lap(1);
    build_ghost_boxes(h);
    lap(2);
    build_pencils(h);
    lap(3);
    alloc_device(h);
    CUDA_OK(cudaStreamSynchronize(h->s));
    lap(4);
    setup_coarse(h);
    CUDA_OK(cudaStreamSynchronize(h->s));
    lap(5);
  });
  if (rc != MG_OK) {
    destroy(h);
    return rc;
  }
  *out = h;
  return MG_OK;
}

void mg_destroy(mg_handle* h) { destroy(h); }

const char* mg_last_error(const mg_handle* h) {
  if (h && !h->err.empty()) return h->err.c_str();
  return g_err.c_str();
}

int mg_set_rhs(mg_handle* h, const double* f_dev) {
  if (!h || !f_dev) return MG_ERR_ARG;
  return guard(h, [&] { set_rhs(h, f_dev); });
}

int mg_set_solution(mg_handle* h, const double* u_dev) {
  if (!h || !u_dev) return MG_ERR_ARG;
  return guard(h, [&] {
    leaf_io(h, const_cast<double*>(u_dev), true, MG_FIELD_U);
    inject_up_all(h);
  });
}

int mg_get_solution(mg_handle* h, double* u_dev) {
  if (!h || !u_dev) return MG_ERR_ARG;
  return guard(h, [&] { leaf_io(h, u_dev, false, MG_FIELD_U); });
}

int mg_vcycle(mg_handle* h, int n) {
  if (!h || n < 0) return MG_ERR_ARG;
  if (!h->rhs_set) {
    h->err = "mg_vcycle before mg_set_rhs";
    return MG_ERR_STATE;
  }
  return guard(h, [&] { run_vcycles(h, n); });
}

int mg_residual_norm(mg_handle* h, double* abs_inf, double* rel_inf) {
  if (!h) return MG_ERR_ARG;
  if (!h->rhs_set) return MG_ERR_STATE;
  return guard(h, [&] {
    const double a = residual_abs(h);
    if (abs_inf) *abs_inf = a;
    if (rel_inf) *rel_inf = h->fstar_norm > 0 ? a / h->fstar_norm : a;
  });
}

int mg_solve(mg_handle* h, double tol, int max_cycles, int criterion, int* cycles_out, double* value_out) {
  if (!h || max_cycles < 0) return MG_ERR_ARG;
  if (criterion != MG_CRIT_RESIDUAL && criterion != MG_CRIT_CAUCHY) {
    h->err = "criterion must be MG_CRIT_RESIDUAL or MG_CRIT_CAUCHY";
    return MG_ERR_ARG;
  }
  if (!h->rhs_set) return MG_ERR_STATE;
  int conv = 0;
  const int rc = guard(h, [&] {
    double val = 0.0;
    int c = 0;
    // Cauchy (E20): the previous iterate stays on the device in leaf layout (d_leafbuf2);
    // each cycle one kernel forms max|u_new - u_old| and max|u_new| and stores u_new
    if (criterion == MG_CRIT_CAUCHY) leaf_io(h, h->d_leafbuf2, false, MG_FIELD_U);
    for (c = 1; c <= max_cycles; ++c) {
      run_vcycles(h, 1);
      if (criterion == MG_CRIT_CAUCHY) {
        val = cauchy_increment(h);
      } else {
        const double a = residual_abs(h);
        val = h->fstar_norm > 0 ? a / h->fstar_norm : a;
      }
      if (val <= tol) {
        conv = 1;
        break;
      }
    }
    if (cycles_out) *cycles_out = std::min(c, max_cycles);
    if (value_out) *value_out = val;
  });
  if (rc != MG_OK) return rc;
  return conv ? MG_OK : MG_WARN_NOT_CONVERGED;
}

int mg_run_host(mg_handle* h, const double* f_host, double* u_host, int ncycles, double* rel_out) {
  if (!h || !f_host || !u_host || ncycles < 0) return MG_ERR_ARG;
  return guard(h, [&] {
    const size_t n = (size_t)h->nc * h->leaves.size() * h->d.block_size * h->d.block_size * h->d.block_size;
    CUDA_OK(cudaMemcpyAsync(h->d_leafbuf, f_host, n * sizeof(double), cudaMemcpyHostToDevice, h->s));
    set_rhs(h, h->d_leafbuf);
    run_vcycles(h, ncycles);
    leaf_io(h, h->d_leafbuf, false, MG_FIELD_U);
    CUDA_OK(cudaMemcpyAsync(u_host, h->d_leafbuf, n * sizeof(double), cudaMemcpyDeviceToHost, h->s));
    const double a = residual_abs(h);
    if (rel_out) *rel_out = h->fstar_norm > 0 ? a / h->fstar_norm : a;
  });
}

int mg_use_graph(mg_handle* h, int enable) {
  if (!h) return MG_ERR_ARG;
  h->use_graph = enable != 0;
  return MG_OK;
}

int mg_profile(mg_handle* h, int enable) {
  if (!h) return MG_ERR_ARG;
  return guard(h, [&] {
    prof_flush(h);
    h->prof_on = enable != 0;
    h->prof_ms.assign((size_t)ST_COUNT * h->L.size(), 0.0);
    h->prof_n.assign((size_t)ST_COUNT * h->L.size(), 0);
  });
}

int mg_profile_read(mg_handle* h, double* ms, int64_t* counts) {
  if (!h) return MG_ERR_ARG;
  return guard(h, [&] {
    prof_flush(h);
    const size_t n = (size_t)ST_COUNT * h->L.size();
    if (h->prof_ms.size() != n) {
      h->prof_ms.assign(n, 0.0);
      h->prof_n.assign(n, 0);
    }
    if (ms) std::memcpy(ms, h->prof_ms.data(), n * sizeof(double));
    if (counts) std::memcpy(counts, h->prof_n.data(), n * sizeof(int64_t));
  });
}

int64_t mg_kernel_launches(void) { return (int64_t)launches_issued(); }

int mg_setup_times(const mg_handle* h, double* ms) {
  if (!h || !ms) return MG_ERR_ARG;
  for (int i = 0; i < 6; ++i) ms[i] = h->setup_ms[i];
  return MG_OK;
}

int mg_num_levels(mg_handle* h) { return h ? (int)h->L.size() : MG_ERR_ARG; }

int mg_level_info(mg_handle* h, int level, int64_t* info) {
  if (!h || !info || level < 0 || level >= (int)h->L.size()) return MG_ERR_ARG;
  Level& l = h->L[level];
  int64_t nleaf_blocks = 0;
  for (int i = 0; i < l.nreal; ++i) nleaf_blocks += l.covmask[i] == 0;
  const int64_t v[10] = {l.B, l.nreal, l.nghost, l.N[0], l.N[1], l.N[2], l.amr,
                         l.n_c2f, (int64_t)l.inj_dst.size(), nleaf_blocks};
  std::memcpy(info, v, sizeof(v));
  return MG_OK;
}

int mg_level_blocks(mg_handle* h, int level, int32_t* coords) {
  const bool all = (level & MG_ALL_BLOCKS) != 0;
  level &= ~MG_ALL_BLOCKS;
  if (!h || !coords || level < 0 || level >= (int)h->L.size()) return MG_ERR_ARG;
  Level& l = h->L[level];
  const int n = all ? l.ntot() : l.nreal;
  for (int i = 0; i < n; ++i)
    for (int a = 0; a < 3; ++a) coords[3 * i + a] = l.coords[i][a];
  return MG_OK;
}

int mg_debug_field(mg_handle* h, int field, int level, int dir, double* dev) {
  if (!h || !dev || level < 0 || level >= (int)h->L.size()) return MG_ERR_ARG;
  const int comp = (field >> 8) & 0xff;
  field &= 0xff;
  if (comp >= h->nc) return MG_ERR_ARG;
  return guard(h, [&] {
    Level& l = h->L[level];
    double* p = field == MG_FIELD_U ? l.u[l.cur] : field == MG_FIELD_F ? l.f : field == MG_FIELD_R ? l.r : l.uhat;
    p += (size_t)comp * l.ntot() * l.B3;
    const size_t n = (size_t)(dir >= 2 ? l.ntot() : l.nreal) * l.B3 * sizeof(double);
    if (dir == 0 || dir == 2) CUDA_OK(cudaMemcpyAsync(dev, p, n, cudaMemcpyDeviceToDevice, h->s));
    else CUDA_OK(cudaMemcpyAsync(p, dev, n, cudaMemcpyDeviceToDevice, h->s));
    CUDA_OK(cudaStreamSynchronize(h->s));
  });
}

static void apply_op(mg_handle* h, int op, int level) {
  const int top = (int)h->L.size() - 1;
  if (level < 0 || level > top) throw MgError(MG_ERR_ARG, "bad level");
  switch (op) {
    case MG_OP_REFRESH: refresh(h, level); break;
    case MG_OP_SMOOTH: sweep(h, level, false); break;
    case MG_OP_SMOOTH_RESIDUAL: sweep(h, level, true); break;
    case MG_OP_RESIDUAL:
      refresh(h, level);
      residual_kernel(h, level);
      break;
    case MG_OP_RESTRICT:
      if (level < 1) throw MgError(MG_ERR_ARG, "restrict needs level >= 1");
      refresh(h, level);
      restrict_level(h, level);
      break;
    case MG_OP_PROLONG:
      if (level < 1) throw MgError(MG_ERR_ARG, "prolong needs level >= 1");
      prolong_level(h, level);
      break;
    case MG_OP_INJECT_UP: inject_up_all(h); break;
    case MG_OP_COARSE_SOLVE: coarse_solve(h); break;
    default: throw MgError(MG_ERR_ARG, "bad op");
  }
}

int mg_transfer(mg_handle* dst, mg_handle* src) {
  if (!dst || !src || dst == src) return MG_ERR_ARG;
  if (!dst->rhs_set) {
    dst->err = "mg_transfer before mg_set_rhs on the destination";
    return MG_ERR_STATE;
  }
  return guard(dst, [&] {
    const mg_desc &a = dst->d, &b = src->d;
    bool same = a.block_size == b.block_size && a.coarse_n == b.coarse_n && dst->nc == src->nc && a.h0 == b.h0;
    for (int i = 0; i < 3; ++i) same = same && a.base_blocks[i] == b.base_blocks[i] && a.origin[i] == b.origin[i];
    for (int i = 0; i < 6; ++i) same = same && a.bc[i] == b.bc[i];
    if (!same) throw MgError(MG_ERR_ARG, "mg_transfer: the grids must share domain, base blocks, B, BC, coarse_n, ncomp");
    // the source's composite solution: canonical coarse values and refreshed ghosts
    CUDA_OK(cudaStreamSynchronize(dst->s));
    if (!src->canonical) {
      inject_up_all(src);
      src->canonical = true;
    }
    for (int m = 1; m < (int)src->L.size(); ++m) refresh(src, m);
    CUDA_OK(cudaStreamSynchronize(src->s));
    const int B = a.block_size;
    std::vector<std::vector<int32_t>> rec(dst->L.size());
    for (const auto& lf : dst->leaves) {
      const int m = dst->nsub + lf[0];
      const int di = dst->L[m].find(lf[1], lf[2], lf[3]);
      const int si = m < (int)src->L.size() ? src->L[m].find(lf[1], lf[2], lf[3]) : -1;
      if (si >= 0 && si < src->L[m].nreal) {
        rec[m].insert(rec[m].end(), {di, si, -1, 0, 0});
        continue;
      }
      const int pi = m >= 1 && m - 1 < (int)src->L.size() ? src->L[m - 1].find(lf[1] >> 1, lf[2] >> 1, lf[3] >> 1) : -1;
      if (pi < 0 || pi >= src->L[m - 1].nreal)
        throw MgError(MG_ERR_LAYOUT_NESTING, "mg_transfer: a leaf more than one level finer than the source grid");
      rec[m].insert(rec[m].end(), {di, pi, (lf[1] & 1) * B / 2, (lf[2] & 1) * B / 2, (lf[3] & 1) * B / 2});
    }
    for (size_t m = 0; m < dst->L.size(); ++m) {
      if (rec[m].empty()) continue;
      Level& D = dst->L[m];
      // copies read the source level m, interpolations level m - 1: one launch each
      std::vector<int32_t> cp, ip;
      for (size_t e = 0; e < rec[m].size(); e += 5) {
        auto& v = rec[m][e + 2] < 0 ? cp : ip;
        v.insert(v.end(), rec[m].begin() + e, rec[m].begin() + e + 5);
      }
      for (int kind = 0; kind < 2; ++kind) {
        const auto& v = kind == 0 ? cp : ip;
        if (v.empty()) continue;
        const Level& S = src->L[kind == 0 ? m : m - 1];
        int32_t* dv = dev_upload(v);
        launch_transfer((int)v.size() / 5, dv, D.u[D.cur], (int64_t)D.ntot() * D.B3, S.u[S.cur], (int64_t)S.ntot() * S.B3,
                        S.d_nbr, B, dst->nc, dst->s);
        CUDA_OK(cudaStreamSynchronize(dst->s));
        cudaFree(dv);
      }
    }
    inject_up_all(dst);
    dst->canonical = true;
    CUDA_OK(cudaStreamSynchronize(dst->s));
  });
}

int mg_debug_poison(mg_handle* h) {
  if (!h) return MG_ERR_ARG;
  return guard(h, [&] {
    // every ghost-block node outside the needed set (the halo the stencils may read,
    // DESIGN.md §5) of every field := NaN; a kernel that reads one spreads it
    const double nan = std::nan("");
    for (auto& l : h->L) {
      std::vector<int32_t> idx;
      for (int gi = 0; gi < l.nghost; ++gi)
        for (int loc = 0; loc < l.B3; ++loc)
          if (!((l.need[gi][loc >> 6] >> (loc & 63)) & 1)) idx.push_back((l.nreal + gi) * l.B3 + loc);
      if (idx.empty()) continue;
      int32_t* d = dev_upload(idx);
      for (double* p : {l.u[0], l.u[1], l.f, l.r, l.uhat})
        launch_fill_list((int)idx.size(), d, p, nan, h->nc, (int64_t)l.ntot() * l.B3, h->s);
      CUDA_OK(cudaStreamSynchronize(h->s));
      cudaFree(d);
    }
  });
}

int mg_debug_apply(mg_handle* h, int op, int level) {
  if (!h) return MG_ERR_ARG;
  return guard(h, [&] {
    apply_op(h, op, level);
    CUDA_OK(cudaStreamSynchronize(h->s));
  });
}

int mg_time_op(mg_handle* h, int op, int level, int reps, double* ms_out) {
  if (!h || reps <= 0) return MG_ERR_ARG;
  return guard(h, [&] {
    cudaEvent_t a, b;
    CUDA_OK(cudaEventCreate(&a));
    CUDA_OK(cudaEventCreate(&b));
    CUDA_OK(cudaEventRecord(a, h->s));
    for (int i = 0; i < reps; ++i) {
      if (op == -1) {
        // the bare fused smoother + residual tile kernel (k_smooth2 with the residual),
        // no ghost refresh (boundary ghosts as they are)
        const int mode = h->smoother == MG_SMOOTHER_RBGS ? SM_RB : SM_JACOBI;
        launch_smooth(view(h, level), h->order, mode, h->omega, true, h->s);
      } else if (op == -2) {
        // the bare production pair: RB pencil sweep, then the residual pencil kernel
        Level& l = h->L[level];
        const LevelView v = view(h, level);
        if (h->smoother != MG_SMOOTHER_RBGS || !launch_rb_pencil(v, h->order, h->omega, nullptr, h->s))
          launch_smooth(v, h->order, h->smoother == MG_SMOOTHER_RBGS ? SM_RB : SM_JACOBI, h->omega, false, h->s);
        swap_u(l);
        residual_kernel(h, level);
      } else if (op < 0) {
        throw MgError(MG_ERR_ARG, "bad op");
      } else if (op == 100) {
        run_vcycles(h, 1);
      } else {
        apply_op(h, op, level);
      }
    }
    CUDA_OK(cudaEventRecord(b, h->s));
    CUDA_OK(cudaEventSynchronize(b));
    float ms = 0;
    CUDA_OK(cudaEventElapsedTime(&ms, a, b));
    if (ms_out) *ms_out = ms / reps;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  });
}

}  // extern "C"
