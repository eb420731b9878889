"""ORACLE — plain, slow, CPU reference of the adaptive FAS V-cycle (test infrastructure).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import or execute this module.  The CUDA product path
(paper_2512_08555_b200) never imports it and shares no code with it: the only
common module is `workloads` (seeded inputs, no method arithmetic).

Representation (independent of the GPU's block layout): every multigrid level k
is a dense lattice N_k^3 (index J = (Jx, Jy, Jz), node at origin + J h_k) with a
boolean mask of the nodes that lie in level-k blocks.  Values are looked up
through ``lookup``: stored value inside level-k blocks (periodic
images by wrap), coarse-to-fine interpolation (c2f) from W_{k-1} at resolution
jumps / exterior nodes, or the last coarse-solve band at the coarsest level.
Extended arrays carry a pad of width E on every axis.  NaN marks "undefined";
a NaN reaching a result means a value outside the method's footprint was used.
A level whose full lattice is large (deep adaptive layouts, > WINDOW_NODES nodes) is
stored on a *window*: the bounding box [lo, lo + n) of its blocks (nodes outside it
are not level-k nodes; the pad beyond the window holds ghost positions like any
other).  Every inter-level map goes through level-global indices J (coarse J <-> fine
2J), so a window only shifts array indices; the arithmetic is the same.

Paper passages (PAPER.md line numbers, P:n):
* Alg. 1 adaptive FAS V(η1,η2)-cycle ............................ P:137-168
* residual r = f - ∇²u ........................................... P:152
* full-weighting restriction ¼[1 2 1] (E6) ....................... P:230-235
* injection of u (E7) ............................................ P:236-241
* block-wise trilinear prolongation ............................... P:228
* smoother: "an iteration of the Gauss-Seidel method" ............ P:227
* 2nd-order cross stencil (E8, E9) ............................... P:252-262
* Mehrstellen Δ_h^M u = R_h^M f, f* = R_h^M f stored once (E10-E12) P:343-354
* ghost interpolation order M+2 (polynomial) ..................... P:63
* coarse FFT direct solve, LGF kernels, Spietz 2-unbounded (E14) .. P:67-100
* zero-average of the coarse solution for periodic problems ...... P:455
* ∞-norm residual convergence / Cauchy criterion (E20) ........... P:170
Readings of silent/garbled passages are listed in DESIGN.md §Readings (Z-codes
from SURVEY.md §8(c)); the ones used here are cited inline.
"""
from __future__ import annotations

import math

import numpy as np

from . import lgf as LGF

PERIODIC, UNBOUNDED, EVEN, ODD = 0, 1, 2, 3


def face_bc(b):
    """(low-face, high-face) condition of one axis: an int means both faces."""
    if isinstance(b, (tuple, list)):
        return int(b[0]), int(b[1])
    return int(b), int(b)
JACOBI, RBGS = 0, 1
E = 8          # pad width of extended arrays (even; > the widest exterior band)
GE = 5         # exterior band width computed by the coarse solve (reading Z21/U1), M <= 4
GE6 = 7        # M = 6: the I = 8 c2f chain of U1 reaches 6 nodes beyond the faces (Z6/U1)
WINDOW_NODES = 1 << 22   # levels with more lattice nodes are stored on their block bounding box


# ----------------------------------------------------------------------------------
# 1D rules
# ----------------------------------------------------------------------------------
def lagrange_midpoint_weights(I: int) -> np.ndarray:
    """Weights of the I-point centred Lagrange interpolant at the midpoint between
    nodes 0 and 1; nodes t = -I/2+1 … I/2 (reading Z7: fixed-weight, always centred)."""
    t = np.arange(-I // 2 + 1, I // 2 + 1, dtype=np.float64)
    w = np.empty(I)
    for a in range(I):
        p = 1.0
        for b in range(I):
            if b != a:
                p *= (0.5 - t[b]) / (t[a] - t[b])
        w[a] = p
    return w


def _shift(A, ax, s):
    """A shifted along axis ax by s (out[i] = A[i+s]); NaN where out of range."""
    out = np.full_like(A, np.nan)
    n = A.shape[ax]
    src = [slice(None)] * A.ndim
    dst = [slice(None)] * A.ndim
    if s >= 0:
        src[ax] = slice(s, n)
        dst[ax] = slice(0, n - s)
    else:
        src[ax] = slice(0, n + s)
        dst[ax] = slice(-s, n)
    out[tuple(dst)] = A[tuple(src)]
    return out


def d2(A, ax):
    """Dimensionless second difference δ² = [1 -2 1] along ax (E9);
    NaN on the two end planes where the stencil leaves the array."""
    out = np.full_like(A, np.nan)
    c = [slice(None)] * A.ndim
    m = [slice(None)] * A.ndim
    p = [slice(None)] * A.ndim
    c[ax], m[ax], p[ax] = slice(1, -1), slice(0, -2), slice(2, None)
    c, m, p = tuple(c), tuple(m), tuple(p)
    out[c] = A[m] - 2.0 * A[c] + A[p]
    return out


def apply_L(X, h, order):
    """Δ_h^M on an extended array (E8 for M=2, E12 for M=4, E13 for M=6)."""
    D = [d2(X, a) for a in range(3)]
    s = D[0] + D[1] + D[2]
    if order >= 4:
        s = s + (d2(D[0], 1) + d2(D[1], 2) + d2(D[2], 0)) / 6.0
    if order == 6:
        s = s + d2(d2(D[0], 1), 2) / 30.0
    return s / (h * h)


def apply_R(X, order):
    """R_h^M f: identity (M=2); f + (1/12)Σδ²f (M=4, right side of E12).
    M=6 (E13 with the δ²_yδ²_z reading Z24): + (1/90)Σδ²δ² - (1/240)Σδ⁴."""
    if order == 2:
        return X.copy()
    D = [d2(X, a) for a in range(3)]
    s = X + (D[0] + D[1] + D[2]) / 12.0
    if order == 6:
        s = s + (d2(D[0], 1) + d2(D[1], 2) + d2(D[2], 0)) / 90.0
        s = s - (d2(D[0], 0) + d2(D[1], 1) + d2(D[2], 2)) / 240.0
    return s


def diag_L(h, order):
    """Centre coefficient of Δ_h^M (fig:stencils P:272-328): -6/h², -24/(6h²), -128/(30h²)."""
    return {2: -6.0, 4: -24.0 / 6.0, 6: -128.0 / 30.0}[order] / (h * h)


def symbol(order, thetas, h):
    """σ_M(θ): eigenvalue of Δ_h^M on e^{iθ·J}; δ² → ŝ = 2cosθ - 2 (P:398 'Fourier symbol')."""
    lams = [2.0 * np.cos(t) - 2.0 for t in thetas]
    return LGF.lattice_symbol_poly(lams, order) / (h * h)


# ----------------------------------------------------------------------------------
# Hierarchy
# ----------------------------------------------------------------------------------
class Level:
    pass


class Oracle:
    """Dense-lattice oracle of the whole solver state.

    desc keys: origin, h0, base_blocks, B, bc (per axis), order, smoother, omega,
    eta1, eta2, coarse_n (0 = AMR level 0 is coarsest), leaves[n,4].
    """

    def __init__(self, desc, leaves):
        self.order = int(desc["order"])
        self.I = self.order + 2                       # interpolation order M+2
        # exterior band of the coarse solve: GE6 only where the I = 8 chain of U1 needs it
        # (the padded LGF sizes then match the GPU's, Z6/U1)
        self.GE = GE6 if (self.order == 6 and int(desc.get("allow_unbounded_refined", 0))) else GE
        self.w_c2f = lagrange_midpoint_weights(self.I)
        self.smoother = int(desc["smoother"])
        self.omega = float(desc["omega"])
        self.eta1, self.eta2 = int(desc["eta1"]), int(desc["eta2"])
        self.B = int(desc["B"])
        # per face: periodic pairs, unbounded pairs, or semi-unbounded = even /
        # odd symmetry at the low face with an unbounded high face (reading S1)
        self.bcf = tuple(face_bc(b) for b in desc["bc"])
        for lo, hi in self.bcf:
            if (lo, hi) not in ((PERIODIC, PERIODIC), (UNBOUNDED, UNBOUNDED), (EVEN, UNBOUNDED), (ODD, UNBOUNDED),
                                (ODD, ODD), (EVEN, ODD), (EVEN, EVEN)):
                raise ValueError(f"unsupported face pair {(lo, hi)}")
        self.per = tuple(lo == PERIODIC for lo, hi in self.bcf)
        self.bc = tuple(PERIODIC if p else UNBOUNDED for p in self.per)   # per-axis kind (legacy use)
        # mirror sign of the low face of each axis: +1 even, -1 odd, 0 none; an odd high
        # face mirrors about the (unstored) node N: u(N) = 0, u(N+k) = -u(N-k) (reading S2)
        self.sym = tuple({EVEN: 1, ODD: -1}.get(lo, 0) for lo, hi in self.bcf)
        self.hi_odd = tuple(hi == ODD for lo, hi in self.bcf)
        # (EVEN, EVEN): homogeneous Neumann on both faces (reading S3): the high wall
        # is the last stored node N-1, u(N-1+k) = u(N-1-k); only with no unbounded axis
        self.hi_even = tuple(lo == EVEN and hi == EVEN for lo, hi in self.bcf)
        if any(self.hi_even) and any(lo == UNBOUNDED or hi == UNBOUNDED for lo, hi in self.bcf):
            raise ValueError("(EVEN, EVEN) axes need the other axes periodic or symmetric")
        self.origin = np.asarray(desc["origin"], dtype=np.float64)
        self.leaves = np.asarray(leaves, dtype=np.int64)
        base = np.asarray(desc["base_blocks"], dtype=np.int64)
        N0 = base * self.B
        amr_max = int(self.leaves[:, 0].max())
        coarse_n = int(desc.get("coarse_n", 0) or 0)
        nsub = 0
        if coarse_n:
            nsub = int(round(math.log2(N0[0] / coarse_n)))
            if not np.all(N0 >> nsub << nsub == N0) or N0[0] >> nsub != coarse_n:
                raise ValueError("coarse_n must be N0 / 2^j on every axis")
        self.nsub = nsub
        self.levels = []
        # MG level m: m < nsub -> sub-base uniform level; m = nsub + a -> AMR level a
        for m in range(nsub + amr_max + 1):
            L = Level()
            a = m - nsub
            L.amr = a
            L.N = (N0 >> (-a)) if a < 0 else (N0 << a)
            L.h = float(desc["h0"]) * (2.0 ** (-a))
            self.levels.append(L)
        # level-k blocks: leaves at k and ancestors of deeper leaves (sub-base: all)
        blocks = [set() for _ in self.levels]
        for lev, bi, bj, bk in self.leaves.tolist():
            c = (bi, bj, bk)
            for a in range(lev, -1, -1):
                blocks[nsub + a].add(c)
                c = (c[0] // 2, c[1] // 2, c[2] // 2)
        for m, L in enumerate(self.levels):
            # storage window [lo, lo + n): the whole lattice, or the block bounding box
            if m < nsub or int(np.prod(L.N)) <= WINDOW_NODES:
                L.lo, L.n = np.zeros(3, dtype=np.int64), L.N.copy()
            else:
                cs = np.array(sorted(blocks[m]), dtype=np.int64)
                L.lo = cs.min(axis=0) * self.B
                L.n = (cs.max(axis=0) + 1) * self.B - L.lo
                for ax in range(3):
                    # a periodic axis is windowed only if the wrap images of the blocks
                    # stay out of the pad (else stored whole, wrap by index)
                    if self.per[ax] and L.n[ax] > L.N[ax] - 2 * E:
                        L.lo[ax], L.n[ax] = 0, L.N[ax]
            L.full = tuple(bool(L.lo[ax] == 0 and L.n[ax] == L.N[ax]) for ax in range(3))
            L.mask = np.zeros(tuple(L.n), dtype=bool)
            if m < nsub:
                L.mask[...] = True
            for c in blocks[m]:
                s0 = np.array(c) * self.B - L.lo
                L.mask[s0[0]:s0[0] + self.B, s0[1]:s0[1] + self.B, s0[2]:s0[2] + self.B] = True
        for m, L in enumerate(self.levels):
            if m + 1 < len(self.levels):
                # coarse J covered iff fine 2J is a level-(m+1) block node
                L.cov = self._down(L, self.levels[m + 1], self.levels[m + 1].mask, False)
            else:
                L.cov = np.zeros(tuple(L.n), dtype=bool)
            L.cov &= L.mask
            L.leaf = L.mask & ~L.cov
            n = tuple(L.n)
            L.u = np.zeros(n)
            L.f = np.zeros(n)
            L.r = np.zeros(n)
            L.uhat = np.zeros(n)
            L.mask_ext = self._pad(L.mask.astype(np.float64), fill=0.0, L=L) > 0.5
            L.parity_ext = self._parity_ext(L)
        c = self.levels[0]
        if not c.mask.all() or not all(c.full):
            raise ValueError("coarsest level must cover the domain")
        c.band = np.zeros(tuple(c.N + 2 * E))        # exterior values of the last coarse solve
        self.fstar_norm = None
        self._coarse_setup()

    # --------------------------------------------------------------- extended arrays
    def _pad(self, A, fill=np.nan, L=None):
        """Extend a level array by E on every axis: periodic axes stored whole by wrap,
        unbounded axes and windowed axes with `fill` (exterior / not a level node)."""
        X = A
        for ax in range(3):
            if self.per[ax] and (L is None or L.full[ax]):
                n = X.shape[ax]
                X = np.take(X, np.arange(-E, n + E) % n, axis=ax)
            else:
                shp = list(X.shape)
                shp[ax] = E
                Z = np.full(shp, fill)
                X = np.concatenate([Z, X, Z], axis=ax)
        return X

    def _parity_ext(self, L):
        idx = [np.arange(-E, n + E) + lo for n, lo in zip(L.n, L.lo)]
        J = np.meshgrid(*idx, indexing="ij")
        return ((J[0] + J[1] + J[2]) % 2 == 0)

    def _interior(self, X, L):
        return X[E:E + L.n[0], E:E + L.n[1], E:E + L.n[2]]

    def _exterior_ext(self, L):
        """True at extended positions outside an unbounded face."""
        ext = np.zeros(tuple(L.n + 2 * E), dtype=bool)
        for ax in range(3):
            if not self.per[ax]:
                J = np.arange(-E, L.n[ax] + E) + L.lo[ax]
                out = (J < 0) | (J >= L.N[ax])
                sh = [1, 1, 1]
                sh[ax] = -1
                ext |= out.reshape(sh)
        return ext

    def _down(self, Lc, Lf, A, fill=np.nan):
        """Coarse-window array of the fine values at the coincident nodes: out(J) =
        A(2J) (injection geometry, E7), `fill` where 2J lies outside the fine window."""
        out = np.full(tuple(Lc.n), fill, dtype=A.dtype)
        idx, ok = [], []
        for ax in range(3):
            i = 2 * (np.arange(Lc.n[ax]) + Lc.lo[ax]) - Lf.lo[ax]
            v = (i >= 0) & (i < Lf.n[ax])
            idx.append(np.where(v, i, 0))
            ok.append(v)
        sub = A[np.ix_(*idx)]
        valid = ok[0][:, None, None] & ok[1][None, :, None] & ok[2][None, None, :]
        out[valid] = sub[valid]
        return out

    # --------------------------------------------------------------- c2f (a1-iii)
    def _c2f_axis(self, W, ax, Lc, Lf):
        """Refine W (extended coarse array of level Lc, along ax) to the extended fine
        array of level Lf: fine J even -> coarse J/2; J odd -> centred I-point
        Lagrange midpoint rule on coarse (J-1)/2 - I/2 + 1 … (J-1)/2 + I/2.
        Extended position p <-> level-global J = p - E + lo (E and lo are even, so p
        has the parity of J)."""
        Wm = np.moveaxis(W, ax, 0)
        nce = Wm.shape[0]
        nf = int(Lf.n[ax])
        lof, loc = int(Lf.lo[ax]), int(Lc.lo[ax])
        out = np.full((nf + 2 * E,) + Wm.shape[1:], np.nan)
        I = self.I
        pe = np.arange(0, nf + 2 * E, 2)                 # J even
        qe = (pe - E + lof) // 2 - loc + E
        ok = (qe >= 0) & (qe < nce)
        out[pe[ok]] = Wm[qe[ok]]
        po = np.arange(1, nf + 2 * E, 2)                 # J odd
        base = (po - E + lof - 1) // 2 - I // 2 + 1 - loc + E
        ok = (base >= 0) & (base + I - 1 < nce)
        po, base = po[ok], base[ok]
        acc = np.zeros((len(po),) + Wm.shape[1:])
        for t in range(I):
            acc += self.w_c2f[t] * Wm[base + t]
        out[po] = acc
        return np.moveaxis(out, 0, ax)

    def c2f(self, W, Lc, Lf):
        """Tensor product of the 1D rule (reading Z7: tensor product at edges/corners)."""
        X = W
        for ax in range(3):
            X = self._c2f_axis(X, ax, Lc, Lf)
        return X

    # --------------------------------------------------------------- value lookup (O2)
    def lookup(self, m, vals, exterior="band"):
        """Extended level-m array of V_m(J): stored values in level-m blocks,
        ghosts from c2f of W_{m-1} (jump and exterior nodes, m >= 1), the last
        coarse-solve band (m = 0, exterior='band') or 0 (exterior='zero', for f)."""
        L = self.levels[m]
        A = self._pad(vals[m], L=L)
        if L.mask_ext.all():
            return A                                  # no ghost nodes on this level
        if m == 0:
            G = np.full(tuple(L.N + 2 * E), np.nan)
            ext = self._exterior_ext(L)
            if exterior == "band":
                G[ext] = L.band[ext]
            else:
                G[ext] = 0.0
                if any(self.sym):
                    # f beyond a symmetric low face is the mirror image (even +, odd -);
                    # beyond unbounded faces it stays 0 (Z16, reading S1)
                    G = np.where(ext, G, A)
                    for ax in range(3):
                        if self.sym[ax]:
                            Gm = np.moveaxis(G, ax, 0)
                            for p in range(E):             # extended p <-> J = p - E < 0
                                Gm[p] = self.sym[ax] * Gm[2 * E - p]
                            if self.hi_odd[ax]:            # J = N + k <-> -(N - k); f(N) = 0
                                n = int(L.N[ax])
                                Gm[E + n] = 0.0
                                for k in range(1, E):
                                    Gm[E + n + k] = -Gm[E + n - k]
                            if self.hi_even[ax]:           # J = N - 1 + k <-> N - 1 - k (S3)
                                n = int(L.N[ax])
                                for k in range(1, E + 1):
                                    Gm[E + n - 1 + k] = Gm[E + n - 1 - k]
                            G = np.moveaxis(Gm, 0, ax)
        else:
            G = self.c2f(self.source_W(m - 1, vals, exterior), self.levels[m - 1], L)
            if exterior == "zero":
                G[self._exterior_ext(L)] = 0.0       # f := 0 beyond unbounded faces (Z16)
        return np.where(L.mask_ext, A, G)

    def source_W(self, m, vals, exterior):
        """W_m: level-m values with every node coinciding with a level-(m+1) block
        node replaced by the fine value (f2c injection, reading Z8), plus exterior
        values; NaN at level-m jump-ghost positions (c2f never reads them, Z7)."""
        L = self.levels[m]
        fine = vals[m + 1]
        Am = vals[m].copy()
        Am[L.cov] = self._down(L, self.levels[m + 1], fine)[L.cov]
        X = np.where(L.mask_ext, self._pad(Am, L=L), np.nan)
        ext = self._exterior_ext(L)
        if ext.any():
            v2 = list(vals)
            v2[m] = Am
            Y = self.lookup(m, v2, exterior)          # exterior values (band / c2f / 0)
            X[ext] = Y[ext]
        return X

    def uvals(self):
        return [L.u for L in self.levels]

    # --------------------------------------------------------------- operators
    def Lu(self, m, vals=None):
        """Δ_h^M u at level m using current ghosts (interior lattice)."""
        vals = self.uvals() if vals is None else vals
        X = self.lookup(m, vals)
        return self._interior(apply_L(X, self.levels[m].h, self.order), self.levels[m])

    def residual(self, m):
        """r_m = f_m - Δ u_m on level-m block nodes (Alg. 1 line P:152)."""
        L = self.levels[m]
        return np.where(L.mask, L.f - self.Lu(m), 0.0)

    def smooth(self, m):
        """One smoothing sweep on all level-m block nodes; boundary ghosts refreshed
        before the sweep and frozen during it (reading Z9).  Jacobi:
        u += ω(f - Δu)/d.  RB (reading Z10): red = even (Jx+Jy+Jz) first, each
        colour updated from a snapshot (Jacobi within colour)."""
        L = self.levels[m]
        vals = self.uvals()
        X = self.lookup(m, vals)
        d = diag_L(L.h, self.order)
        if self.smoother == JACOBI:
            Lx = apply_L(X, L.h, self.order)
            U = X + self.omega * (self._pad(L.f, 0.0, L) - Lx) / d
            L.u = np.where(L.mask, self._interior(U, L), L.u)
            return
        ghosts = np.where(L.mask_ext, np.nan, X)      # frozen boundary ghosts
        Fext = self._pad(L.f, 0.0, L)
        for colour in (True, False):
            Lx = apply_L(X, L.h, self.order)
            U = X + self.omega * (Fext - Lx) / d
            sel = L.mask_ext & (L.parity_ext == colour)
            Unew = np.where(sel, U, X)
            # re-impose periodic images of the updated interior, keep frozen ghosts
            newu = self._interior(Unew, L)
            L.u = np.where(L.mask, newu, L.u)
            X = np.where(L.mask_ext, self._pad(L.u, L=L), ghosts)

    def restrict(self, m):
        """Alg. 1: on the Ω_m-covered nodes of level m-1
        u_{m-1} <- Î u_m (E7), r_{m-1} <- I r_m (E6, r := 0 outside level m, reading Z14),
        then f_{m-1} <- r_{m-1} + Δ u_{m-1} (after the level-(m-1) refresh);
        finally û_{m-1} <- u_{m-1} on every level-(m-1) node (reading Z13-W)."""
        L, C = self.levels[m], self.levels[m - 1]
        r = self.residual(m)
        C.u = np.where(C.cov, self._down(C, L, L.u), C.u)
        R = self._pad(np.where(L.mask, r, 0.0), fill=0.0, L=L)
        for ax in range(3):
            R = 0.25 * _shift(R, ax, -1) + 0.5 * R + 0.25 * _shift(R, ax, 1)
        Rint = self._down(C, L, self._interior(R, L))
        C.r = np.where(C.cov, Rint, 0.0)
        Lc = self.Lu(m - 1)
        C.f = np.where(C.cov, C.r + Lc, C.f)
        C.uhat = np.where(C.mask, C.u, 0.0)
        # "the û snapshot includes the band": the exterior values of
        # level m-1 (c2f chain / coarse-solve band) at this moment (Z13-W)
        if self._exterior_ext(C).any():
            C.uhat_ext = self.lookup(m - 1, self.uvals())

    def prolong(self, m):
        """u_m += I ε_{m-1}, ε = u - û on level-(m-1) nodes (correction sign: reading
        Z12; whole-level snapshot: reading Z13-W); I = trilinear (Alg. 1):
        per axis, fine J even -> coarse J/2, J odd -> mean of (J-1)/2 and (J+1)/2."""
        L, C = self.levels[m], self.levels[m - 1]
        eps = np.where(C.mask, C.u - C.uhat, 0.0)
        X = self._pad(eps, fill=0.0, L=C)
        # exterior band (U1): ε = current exterior value - its snapshot at restriction;
        # jump ghosts keep ε := 0 (Z13-W)
        ext = self._exterior_ext(C)
        if ext.any() and hasattr(C, "uhat_ext"):
            cur = self.lookup(m - 1, self.uvals())
            X = np.where(ext, cur - C.uhat_ext, X)
        for ax in range(3):
            Xm = np.moveaxis(X, ax, 0)
            nce = Xm.shape[0]
            nf = int(L.n[ax])
            lof, loc = int(L.lo[ax]), int(C.lo[ax])       # extended p <-> J = p - E + lo
            out = np.full((nf + 2 * E,) + Xm.shape[1:], np.nan)
            pe = np.arange(0, nf + 2 * E, 2)
            qe = (pe - E + lof) // 2 - loc + E
            ok = (qe >= 0) & (qe < nce)
            out[pe[ok]] = Xm[qe[ok]]
            po = np.arange(1, nf + 2 * E, 2)
            qo = (po - E + lof - 1) // 2 - loc + E
            ok = (qo >= 0) & (qo + 1 < nce)
            out[po[ok]] = 0.5 * (Xm[qo[ok]] + Xm[qo[ok] + 1])
            X = np.moveaxis(out, 0, ax)
        L.u = np.where(L.mask, L.u + self._interior(X, L), L.u)

    def inject_up(self):
        """u_{m-1}[covered] <- u_m(2i), finest to coarsest (E7; canonical state)."""
        for m in range(len(self.levels) - 1, 0, -1):
            L, C = self.levels[m], self.levels[m - 1]
            C.u = np.where(C.cov, self._down(C, L, L.u), C.u)

    # --------------------------------------------------------------- coarse solve (a6)
    def _coarse_setup(self):
        c = self.levels[0]
        # semi-unbounded axes ("adequate symmetries"; reading S1): the source is
        # extended by its mirror image across the symmetric low face to the unbounded
        # domain [-(N-1), N-1] (even: +, odd: - with f(0) := 0) and solved as an
        # unbounded axis of 2N-1 nodes; node J of the level is extended node J + N - 1.
        semi = [self.sym[ax] != 0 and not self.hi_odd[ax] for ax in range(3)]
        N = [2 * int(n) - 1 if semi[ax] else int(n) for ax, n in enumerate(c.N)]
        self.coff = [int(c.N[ax]) - 1 if semi[ax] else 0 for ax in range(3)]
        self.cN = N
        if any(self.hi_odd) or any(self.hi_even):
            self.coarse_kind = "SS"        # a both-sided symmetric axis: _coarse_solve_ss
            return
        self.unb = [ax for ax in range(3) if not self.per[ax]]
        if len(self.unb) == 0:
            self.coarse_kind = "PPP"
            return
        shape = [N[ax] if self.per[ax] else LGF.pad_size(N[ax], self.GE) for ax in range(3)]
        self.coarse_shape = shape
        th = [2 * np.pi * np.fft.fftfreq(s) for s in shape]
        TH = np.meshgrid(*th, indexing="ij")
        if len(self.unb) == 3:
            self.coarse_kind = "UUU"
            R = LGF.box_radius(max(shape))
            G = LGF.box_lgf(3, self.order, R)
            T = LGF.wrapped_table(G, R, shape)
            self.coarse_mult = np.fft.fftn(T).real * c.h * c.h
            return
        # mixed periodic / unbounded (E14, generalised; reading Z22): along the
        # periodic axes the transform is exact, along the unbounded ones zero-padded.  The
        # Fourier modes with zero periodic wavenumber reduce the operator to the unbounded
        # axes alone (their δ² eigenvalues vanish in the symbol): there the multiplier is
        # the transform of that lower-dimensional LGF (2D box LGF, or the 1D LGF |n|/2);
        # every other mode is regular and takes 1/σ_M on the padded lattice.
        sig = symbol(self.order, TH, c.h)
        zero_per = np.ones(tuple(shape), dtype=bool)
        for ax in range(3):
            if self.per[ax]:
                sl = [None, None, None]
                sl[ax] = slice(None)
                zero_per &= (np.arange(shape[ax]) == 0).reshape([-1 if a == ax else 1 for a in range(3)])
        K = 1.0 / np.where(zero_per, 1.0, sig)
        ush = [shape[ax] for ax in self.unb]
        if len(self.unb) == 2:
            self.coarse_kind = "P" + "U" * 2
            R = LGF.box_radius(max(ush))
            G = LGF.box_lgf(2, self.order, R)
            Tl = LGF.wrapped_table(G, R, ush)
            Kl = np.fft.fft2(Tl).real * c.h * c.h
        else:
            self.coarse_kind = "PPU"
            P = ush[0]
            n = np.arange(P)
            n = np.where(n <= P // 2, n, n - P)
            Tl = np.abs(n) / 2.0      # 1D LGF: δ²(|n|/2) = δ[n], G[0] = 0
            Kl = np.fft.fft(Tl).real * c.h * c.h
        shp = [shape[ax] if not self.per[ax] else 1 for ax in range(3)]
        K = np.where(zero_per, Kl.reshape(shp), K)
        self.coarse_mult = K

    def _coarse_solve_ss(self):
        """Coarse solve with a both-sided symmetric axis ("sine or cosine transform
        instead of the standard discrete Fourier transform"; reading S2): ODD/ODD axes
        by the DST-I of the nodes 1..N-1 (u(0) = u(N) = 0, θ_k = πk/N), EVEN/ODD axes by
        the DCT-III of the nodes 0..N-1 (θ_k = π(2k+1)/(2N)), periodic axes by the DFT,
        unbounded (and semi-unbounded, mirror-extended) axes by the zero-padded DFT,
        EVEN/EVEN axes by the DCT-I of the nodes 0..N-1 (walls at nodes 0 and N-1,
        θ_k = πk/(N-1); reading S3).  Every mode takes 1/σ_M(θ) (reading Z22) except the
        one with all-zero wavenumbers (EVEN/EVEN with periodic axes only: the constant),
        set to 0 (zero average of the coarse solution)."""
        import scipy.fft as sf
        c = self.levels[0]
        N = [int(n) for n in c.N]
        X = c.f.astype(np.float64).copy()
        for ax in range(3):               # mirror images across semi-unbounded low faces
            if self.sym[ax] and not self.hi_odd[ax] and not self.hi_even[ax]:
                fm = np.moveaxis(X, ax, 0)
                img = self.sym[ax] * fm[:0:-1]
                mid = fm[:1] if self.sym[ax] > 0 else 0.0 * fm[:1]
                X = np.moveaxis(np.concatenate([img, mid, fm[1:]], axis=0), 0, ax)
        thetas = []
        for ax in range(3):
            n = N[ax]
            if self.hi_odd[ax] and self.sym[ax] < 0:          # ODD / ODD
                X = np.take(X, np.arange(1, n), axis=ax)
                X = sf.dst(X, type=1, axis=ax, norm="ortho")
                thetas.append(np.pi * np.arange(1, n) / n)
            elif self.hi_odd[ax]:                              # EVEN / ODD
                # unnormalised DCT-III = Σ_j w_j f_j cos(θ_k j), w_0 = 1/2: the left
                # eigenvectors of the (non-symmetric) mirrored operator
                X = sf.dct(X, type=3, axis=ax)
                thetas.append(np.pi * (2 * np.arange(n) + 1) / (2 * n))
            elif self.hi_even[ax]:                             # EVEN / EVEN
                # DCT-I = the DFT of the even extension of period 2(N-1)
                X = sf.dct(X, type=1, axis=ax)
                thetas.append(np.pi * np.arange(n) / (n - 1))
            elif self.per[ax]:
                thetas.append(None)
            else:                                              # unbounded / semi-unbounded
                Pp = LGF.pad_size(self.cN[ax], self.GE)
                shp = list(X.shape)
                shp[ax] = Pp - X.shape[ax]
                X = np.concatenate([X, np.zeros(shp)], axis=ax)
                thetas.append(None)
        fft_axes = [ax for ax in range(3) if not self.hi_odd[ax] and not self.hi_even[ax]]
        for ax in fft_axes:
            thetas[ax] = 2 * np.pi * np.fft.fftfreq(X.shape[ax])
        Xc = np.fft.fftn(X, axes=fft_axes) if fft_axes else X
        TH = np.meshgrid(*thetas, indexing="ij")
        sig = symbol(self.order, TH, c.h)
        zero = sig == 0.0                     # the constant mode (only with EVEN/EVEN)
        Xc = np.where(zero, 0.0, Xc / np.where(zero, 1.0, sig))
        X = np.fft.ifftn(Xc, axes=fft_axes).real if fft_axes else Xc
        for ax in range(3):
            if self.hi_odd[ax] and self.sym[ax] < 0:
                X = sf.dst(X, type=1, axis=ax, norm="ortho")
                shp = list(X.shape)
                shp[ax] = 1
                X = np.concatenate([np.zeros(shp), X], axis=ax)   # u(0) = 0
            elif self.hi_odd[ax]:
                X = sf.idct(X, type=3, axis=ax)
            elif self.hi_even[ax]:
                X = sf.idct(X, type=1, axis=ax)
        # interior and exterior band: per axis a source index into X and a sign
        GEb = self.GE
        band = np.full(tuple(c.N + 2 * E), np.nan)
        idx, sgn = [], []
        for ax in range(3):
            n = N[ax]
            J = np.arange(-E, n + E)
            if self.per[ax]:
                i, sg = J % n, np.ones(len(J))
            elif self.hi_odd[ax]:
                i = np.where(J < 0, -J, np.where(J < n, J, 2 * n - J))
                sg = np.where(J < 0, float(self.sym[ax]), np.where(J < n, 1.0, -1.0))
                sg = np.where((J == n) | (J < -(n - 1)) | (J > 2 * n - 1), 0.0, sg)
                i = np.clip(i, 0, n - 1)
            elif self.hi_even[ax]:                 # mirrors about nodes 0 and N-1
                i = np.where(J < 0, -J, np.where(J < n, J, 2 * (n - 1) - J))
                sg = np.where((J < -(n - 1)) | (J > 2 * (n - 1)), np.nan, 1.0)
                i = np.clip(i, 0, n - 1)
            else:
                ok = (J >= -GEb) & (J < n + GEb)
                i = np.where(ok, (J + self.coff[ax]) % X.shape[ax], 0)
                sg = np.where(ok, 1.0, np.nan)
            idx.append(i)
            sgn.append(sg)
        V = X[np.ix_(*idx)] * sgn[0][:, None, None] * sgn[1][None, :, None] * sgn[2][None, None, :]
        o = self.coff
        inner = tuple(slice(E, E + N[ax]) for ax in range(3))
        c.u = V[inner].copy()
        ext = self._exterior_ext(c)
        band[ext] = V[ext]
        c.band = band

    def coarse_solve(self):
        """u_0 <- S_0 f_0 (Alg. 1).  PPP: F^-1[F f / σ_M], zero mode -> 0
        (zero average).  Unbounded: zero-padded convolution with the LGF
        of Δ_h^M, computed on [-GE, N+GE) for the exterior band."""
        c = self.levels[0]
        N = [int(n) for n in c.N]
        if self.coarse_kind == "SS":
            self._coarse_solve_ss()
            return
        if self.coarse_kind == "PPP":
            F = np.fft.fftn(c.f)
            th = [2 * np.pi * np.fft.fftfreq(n) for n in N]
            TH = np.meshgrid(*th, indexing="ij")
            sig = symbol(self.order, TH, c.h)
            sig[0, 0, 0] = 1.0
            U = F / sig
            U[0, 0, 0] = 0.0
            c.u = np.fft.ifftn(U).real
            return
        shape = self.coarse_shape
        Fp = np.zeros(shape)
        fe = c.f
        for ax in range(3):               # mirror images across symmetric low faces
            if self.sym[ax]:
                fm = np.moveaxis(fe, ax, 0)
                img = self.sym[ax] * fm[:0:-1]            # x = -(N-1) … -1  <->  f(N-1) … f(1)
                mid = fm[:1] if self.sym[ax] > 0 else 0.0 * fm[:1]   # odd: f(0) := 0
                fe = np.moveaxis(np.concatenate([img, mid, fm[1:]], axis=0), 0, ax)
        NE = self.cN
        Fp[:NE[0], :NE[1], :NE[2]] = fe
        U = np.fft.ifftn(np.fft.fftn(Fp) * self.coarse_mult).real
        o = self.coff
        c.u = U[o[0]:o[0] + N[0], o[1]:o[1] + N[1], o[2]:o[2] + N[2]].copy()
        # exterior band: outputs at J in [-GE, N+GE) along unbounded axes
        GEb = self.GE
        band = np.full(tuple(c.N + 2 * E), np.nan)
        idx = []
        for ax in range(3):
            if self.per[ax]:
                idx.append(np.arange(-E, N[ax] + E) % N[ax])
            else:
                J = np.arange(-E, N[ax] + E)
                ok = (J >= -GEb) & (J < N[ax] + GEb)
                idx.append(np.where(ok, (J + self.coff[ax]) % shape[ax], -1))
        sub = U[np.ix_(*[np.where(i < 0, 0, i) for i in idx])]
        valid = np.ones(band.shape, dtype=bool)
        for ax in range(3):
            sh = [1, 1, 1]
            sh[ax] = -1
            valid &= (idx[ax] >= 0).reshape(sh)
        band[valid] = sub[valid]
        c.band = band

    # --------------------------------------------------------------- API-level ops
    def _local(self, lev, bi, bj, bk):
        """Array index of node (0,0,0) of leaf block (lev, bi, bj, bk) in its level's window."""
        L = self.levels[self.nsub + lev]
        return tuple(int(c * self.B - L.lo[a]) for a, c in enumerate((bi, bj, bk)))

    def set_rhs(self, f_leaves):
        """O5: place f on leaf nodes, inject up the tree (f2c), f* = R_h^M f on
        leaves via the lookup with f := 0 beyond unbounded faces (Z16)."""
        B = self.B
        fraw = [np.zeros(tuple(L.n)) for L in self.levels]
        for n, (lev, bi, bj, bk) in enumerate(self.leaves.tolist()):
            i, j, k = self._local(lev, bi, bj, bk)
            fraw[self.nsub + lev][i:i + B, j:j + B, k:k + B] = np.asarray(f_leaves[n]).transpose(2, 1, 0)
        for m in range(len(self.levels) - 1, 0, -1):
            C = self.levels[m - 1]
            fraw[m - 1] = np.where(C.cov, self._down(C, self.levels[m], fraw[m]), fraw[m - 1])
        for ax in range(3):
            if self.sym[ax] < 0:          # odd face: the wall plane is u = 0, f there ignored (S1)
                sl = [slice(None)] * 3
                sl[ax] = 0
                fraw[0][tuple(sl)] = 0.0
        for m, L in enumerate(self.levels):
            X = self.lookup(m, fraw, exterior="zero")
            fs = self._interior(apply_R(X, self.order), L)
            L.f = np.where(L.leaf, fs, fraw[m])
        self.fstar_norm = max(float(np.abs(L.f[L.leaf]).max()) if L.leaf.any() else 0.0
                              for L in self.levels)

    def set_solution(self, u_leaves):
        B = self.B
        for n, (lev, bi, bj, bk) in enumerate(self.leaves.tolist()):
            i, j, k = self._local(lev, bi, bj, bk)
            self.levels[self.nsub + lev].u[i:i + B, j:j + B, k:k + B] = np.asarray(u_leaves[n]).transpose(2, 1, 0)
        self.inject_up()

    def get_solution(self):
        B = self.B
        out = np.empty((len(self.leaves), B, B, B))
        for n, (lev, bi, bj, bk) in enumerate(self.leaves.tolist()):
            i, j, k = self._local(lev, bi, bj, bk)
            out[n] = self.levels[self.nsub + lev].u[i:i + B, j:j + B, k:k + B].transpose(2, 1, 0)
        return out

    def transfer_from(self, old):
        """u on this (adapted) grid from the composite solution of `old`, the same domain
        on another leaf set ("refined into 8 finer blocks" / "revert
        back to a single grid block"; reading A3): a level-k block of this grid that is
        also a level-k block of `old` takes its values (a coarsened leaf: the old parent,
        which holds the injected fine values, E7); a block new at level k (a refined leaf)
        takes the trilinear interpolation (the prolongation rule applied to u) of
        the old level k-1, ghosts included (lookup O2 after inject-up).  Then inject-up."""
        old.inject_up()
        B = self.B
        for lev, bi, bj, bk in self.leaves.tolist():
            m = self.nsub + lev
            L, Lo = self.levels[m], old.levels[m] if m < len(old.levels) else None
            i, j, k = self._local(lev, bi, bj, bk)
            J0 = np.array([bi, bj, bk]) * B
            if Lo is not None:
                io = J0 - Lo.lo
                if (io >= 0).all() and (io + B <= Lo.n).all() and Lo.mask[io[0], io[1], io[2]]:
                    L.u[i:i + B, j:j + B, k:k + B] = Lo.u[io[0]:io[0] + B, io[1]:io[1] + B, io[2]:io[2] + B]
                    continue
            C = old.levels[m - 1]
            X = old.lookup(m - 1, old.uvals())            # extended: stored + ghosts
            c0 = J0 // 2 - C.lo + E                          # extended index of coarse node J0/2
            sub = X[c0[0]:c0[0] + B // 2 + 1, c0[1]:c0[1] + B // 2 + 1, c0[2]:c0[2] + B // 2 + 1]
            for ax in range(3):                              # per axis: even -> copy, odd -> mean
                sm = np.moveaxis(sub, ax, 0)
                out = np.empty((B,) + sm.shape[1:])
                out[0::2] = sm[:B // 2]
                out[1::2] = 0.5 * (sm[:B // 2] + sm[1:B // 2 + 1])
                sub = np.moveaxis(out, 0, ax)
            L.u[i:i + B, j:j + B, k:k + B] = sub
        self.inject_up()

    def vcycle(self, n=1):
        """Alg. 1 with readings Z9-Z15, then inject-up."""
        top = len(self.levels) - 1
        for _ in range(n):
            for m in range(top, 0, -1):
                for _ in range(self.eta1):
                    self.smooth(m)
                self.restrict(m)
            self.coarse_solve()
            for m in range(1, top + 1):
                self.prolong(m)
                for _ in range(self.eta2):
                    self.smooth(m)
            self.inject_up()

    def residual_norm(self):
        """a9: max over leaf nodes of all levels of |f - Δu|, and relative to ‖f*‖∞."""
        mx = 0.0
        for m, L in enumerate(self.levels):
            if not L.leaf.any():
                continue
            r = L.f - self.Lu(m)
            mx = max(mx, float(np.abs(r[L.leaf]).max()))
        rel = mx / self.fstar_norm if self.fstar_norm else mx
        return mx, rel

    def solve(self, tol, max_cycles=50, criterion="residual"):
        """Cycle until rel. residual <= tol (configs) or the Cauchy criterion E20."""
        hist = []
        prev = None
        for c in range(1, max_cycles + 1):
            if criterion == "cauchy":
                prev = self.get_solution()
            self.vcycle(1)
            a, r = self.residual_norm()
            if criterion == "cauchy":
                cur = self.get_solution()
                num = np.abs(cur - prev).max()
                den = np.abs(cur).max()
                r = num / den if den > 0 else num
            hist.append(r)
            if r <= tol:
                return c, hist
        return max_cycles, hist
