"""Analytic source terms, sampled at leaf-block nodes (harness; no method arithmetic).

Block arrays are laid out ``[n_leaf][B][B][B]`` with x fastest, i.e. numpy index
``[blk, kz, ky, kx]`` — the layout the C-ABI takes (include/mg.h).
"""
from __future__ import annotations

import math

import numpy as np
from scipy.special import erf

from .layouts import Domain, block_node_coords


def sample_on_leaves(dom: Domain, leaves: np.ndarray, fn, chunk: int = 512) -> np.ndarray:
    """Evaluate fn(x, y, z) (broadcasting) at every node of every leaf block."""
    n = len(leaves)
    B = dom.B
    out = np.empty((n, B, B, B), dtype=np.float64)
    for lev in np.unique(leaves[:, 0]):
        idx = np.nonzero(leaves[:, 0] == lev)[0]
        for s in range(0, len(idx), chunk):
            ii = idx[s:s + chunk]
            x, y, z = block_node_coords(dom, int(lev), leaves[ii, 1:4].astype(np.int64))
            out[ii] = fn(x[:, None, None, :], y[:, None, :, None], z[:, :, None, None])
    return out


def dense_to_blocks(dom: Domain, leaves: np.ndarray, dense_xyz: np.ndarray) -> np.ndarray:
    """Scatter a dense level array indexed [Jx, Jy, Jz] into leaf blocks [b, z, y, x]."""
    B = dom.B
    out = np.empty((len(leaves), B, B, B))
    for n, (lev, i, j, k) in enumerate(leaves.tolist()):
        blk = dense_xyz[i * B:(i + 1) * B, j * B:(j + 1) * B, k * B:(k + 1) * B]
        out[n] = blk.transpose(2, 1, 0)
    return out


# ---- config 1: product of sines (BASELINE configs[0]) ----------------------------
def sines(x, y, z):
    return np.sin(2 * np.pi * x) * np.sin(2 * np.pi * y) * np.sin(2 * np.pi * z)


# ---- config 2: seeded random Fourier modes (BASELINE configs[1]) -----------------
def fourier_modes(seed: int = 2, nmodes: int = 64, kmax: float = 8.0):
    """k_j drawn without replacement, uniformly from {k in Z^3 : 1 <= |k| <= kmax,
    first non-zero component > 0}; a_j ~ N(0,1); phi_j ~ U[0, 2pi); drawn in that
    order from numpy.random.default_rng(seed) (Inputs)."""
    r = int(math.floor(kmax))
    cand = []
    for kx in range(-r, r + 1):
        for ky in range(-r, r + 1):
            for kz in range(-r, r + 1):
                k = (kx, ky, kz)
                n2 = kx * kx + ky * ky + kz * kz
                if n2 < 1 or n2 > kmax * kmax:
                    continue
                first = next(c for c in k if c != 0)
                if first > 0:
                    cand.append(k)
    cand = np.asarray(cand, dtype=np.int64)
    rng = np.random.default_rng(seed)
    sel = rng.choice(len(cand), size=nmodes, replace=False)
    a = rng.normal(0.0, 1.0, size=nmodes)
    phi = rng.uniform(0.0, 2 * np.pi, size=nmodes)
    return cand[sel], a, phi


def fourier_dense(N: int, modes) -> np.ndarray:
    """f(J) = sum_j a_j cos(2 pi k_j . J / N + phi_j) on the periodic N^3 lattice of
    [0,1)^3, synthesised exactly by one inverse FFT; indexed [Jx, Jy, Jz]."""
    k, a, phi = modes
    C = np.zeros((N, N, N), dtype=np.complex128)
    for kk, aa, pp in zip(k.tolist(), a.tolist(), phi.tolist()):
        c = 0.5 * aa * np.exp(1j * pp)
        C[kk[0] % N, kk[1] % N, kk[2] % N] += c
        C[-kk[0] % N, -kk[1] % N, -kk[2] % N] += np.conj(c)
    f = np.fft.ifftn(C).real * (N ** 3)
    return f - f.mean()


def fourier_eval(modes, x, y, z):
    k, a, phi = modes
    out = 0.0
    for kk, aa, pp in zip(k.tolist(), a.tolist(), phi.tolist()):
        out = out + aa * np.cos(2 * np.pi * (kk[0] * x + kk[1] * y + kk[2] * z) + pp)
    return out


# ---- config 3: Gaussian blob, unbounded ---------------------------------------
def gaussian_charge(x, y, z, sigma=0.08, Q=1.0, c=(0.0, 0.0, 0.0)):
    r2 = (x - c[0]) ** 2 + (y - c[1]) ** 2 + (z - c[2]) ** 2
    return Q * (2 * np.pi) ** -1.5 * sigma ** -3 * np.exp(-r2 / (2 * sigma * sigma))


def gaussian_potential(x, y, z, sigma=0.08, Q=1.0, c=(0.0, 0.0, 0.0)):
    """Free-space solution of lap(u) = gaussian_charge: u = -Q erf(r/(sqrt2 sigma))/(4 pi r)."""
    r = np.sqrt((x - c[0]) ** 2 + (y - c[1]) ** 2 + (z - c[2]) ** 2)
    rs = np.where(r > 0, r, 1.0)
    val = -Q * erf(rs / (math.sqrt(2) * sigma)) / (4 * np.pi * rs)
    return np.where(r > 0, val, -Q * math.sqrt(2 / np.pi) / (4 * np.pi * sigma))


# ---- config 4: three seeded blobs, x periodic ------------------------------------
def blobs(seed: int = 4, n: int = 3):
    """Centres x~U[0,1), (y,z)~U[0.3,0.7]; sigma~U[0.02,0.1]; Q~N(0,1); drawn in
    that order from default_rng(seed)."""
    rng = np.random.default_rng(seed)
    cx = rng.uniform(0.0, 1.0, size=n)
    cyz = rng.uniform(0.3, 0.7, size=(n, 2))
    sig = rng.uniform(0.02, 0.1, size=n)
    Q = rng.normal(0.0, 1.0, size=n)
    return np.column_stack([cx, cyz]), sig, Q


def blobs_eval(params, x, y, z, Lx=1.0):
    c, sig, Q = params
    out = 0.0
    for j in range(len(sig)):
        dx = x - c[j, 0]
        dx = dx - Lx * np.round(dx / Lx)  # minimum image along the periodic x axis
        r2 = dx * dx + (y - c[j, 1]) ** 2 + (z - c[j, 2]) ** 2
        out = out + Q[j] * (2 * np.pi * sig[j] ** 2) ** -1.5 * np.exp(-r2 / (2 * sig[j] ** 2))
    return out


# ---- config 5: perturbed torus (vortex-ring-like), x periodic ---------------------
def torus_params(seed: int = 5, nmodes: int = 8, kmax: int = 4):
    rng = np.random.default_rng(seed)
    cand = [(a, b, c) for a in range(-kmax, kmax + 1) for b in range(-kmax, kmax + 1)
            for c in range(-kmax, kmax + 1) if 1 <= a * a + b * b + c * c <= kmax * kmax]
    cand = np.asarray(cand, dtype=np.int64)
    sel = rng.choice(len(cand), size=nmodes, replace=False)
    b = rng.normal(0.0, 1.0, size=nmodes)
    phi = rng.uniform(0.0, 2 * np.pi, size=nmodes)
    b = b / np.abs(b).sum()  # reading: max|xi| <= sum|b_j| = 1
    return cand[sel], b, phi


def torus_eval(params, x, y, z, R=0.5, sigma=0.03, eps=0.05):
    k, b, phi = params
    rho = np.sqrt(y * y + z * z)
    d2 = x * x + (rho - R) ** 2
    A = 1.0 / (4 * np.pi ** 2 * R * sigma ** 2)
    f0 = A * np.exp(-d2 / (2 * sigma * sigma))
    xi = 0.0
    for kk, bb, pp in zip(k.tolist(), b.tolist(), phi.tolist()):
        xi = xi + bb * np.cos(np.pi * (kk[0] * x + kk[1] * y + kk[2] * z) + pp)
    return f0 * (1.0 + eps * xi)


# ---- paper's manufactured product solution (E25-E28) -------------------
def u_per(x):
    return np.exp(np.sin(2 * np.pi * x)) - 1.0


def d2u_per(x):
    s, c = np.sin(2 * np.pi * x), np.cos(2 * np.pi * x)
    return (2 * np.pi) ** 2 * np.exp(s) * (c * c - s)


def u_unb(x):
    t = 2 * x - 1
    inside = np.abs(t) < 1
    ts = np.where(inside, t, 0.0)
    return np.where(inside, np.exp(10 * (1 - 1 / (1 - ts * ts))), 0.0)


def d2u_unb(x):
    # u = exp(g), g = 10(1 - 1/(1-t^2)), t = 2x-1; u'' = (g'^2 + g'') u (in x)
    t = 2 * x - 1
    inside = np.abs(t) < 1
    ts = np.where(inside, t, 0.0)
    q = 1 - ts * ts
    gt = -20 * ts / (q * q)                     # dg/dt
    gtt = -20 / (q * q) - 80 * ts * ts / (q ** 3)  # d2g/dt2
    u = np.exp(10 * (1 - 1 / q))
    return np.where(inside, 4 * (gt * gt + gtt) * u, 0.0)


# ------------------------------------------------------------------ vortex tube (NEXT #4)
# Biot–Savart test of the paper's performance section (E29–E33): a compact
# vortex tube along z, centred in the unit cube (x, y unbounded, z periodic); the
# velocity solves the vector Poisson problem ∇²u = -∇×ω.  R is not given in the
# paper (reading T1: R = 0.25).
def _e2_1():
    from scipy.special import expn
    return float(expn(2, 1.0))


def tube_omega(x, y, z, R=0.25, c=(0.5, 0.5)):
    """ω_z(r) = (1/2π)(2/R²)(1/E₂(1)) exp(-1/(1 - (r/R)²)) for r < R, else 0 (E31)."""
    rho2 = ((x - c[0]) ** 2 + (y - c[1]) ** 2) / (R * R) + 0.0 * z
    inside = rho2 < 1.0
    q = np.where(inside, 1.0 - rho2, 1.0)
    return np.where(inside, (1 / (2 * np.pi)) * (2 / (R * R)) / _e2_1() * np.exp(-1.0 / q), 0.0)


def tube_rhs(x, y, z, comp, R=0.25, c=(0.5, 0.5)):
    """Component comp of f = -∇×ω = (-∂_y ω_z, ∂_x ω_z, 0), with
    ∂_x ω_z = -2 ω_z (x - c_x) / (R² (1 - ρ²)²) (ρ = r/R; smooth, compact)."""
    w = tube_omega(x, y, z, R, c)
    rho2 = ((x - c[0]) ** 2 + (y - c[1]) ** 2) / (R * R) + 0.0 * z
    q = np.where(rho2 < 1.0, 1.0 - rho2, 1.0)
    g = -2.0 * w / (R * R * q * q)
    if comp == 0:
        return -g * (y - c[1])
    if comp == 1:
        return g * (x - c[0])
    return 0.0 * w


def tube_velocity(x, y, z, comp, R=0.25, c=(0.5, 0.5)):
    """Analytic velocity (E32–E33): u = u_θ(r) (-sin θ, cos θ, 0), u_θ = (1/2πr)[1 -
    (1/E₂(1))(1 - ρ²) E₂(1/(1 - ρ²))] for r <= R, 1/(2πr) outside."""
    from scipy.special import expn
    dx, dy = x - c[0] + 0.0 * z, y - c[1] + 0.0 * z
    r2 = dx * dx + dy * dy
    rho2 = r2 / (R * R)
    inside = rho2 < 1.0
    q = np.where(inside, 1.0 - rho2, 1.0)
    frac = np.where(inside, 1.0 - q * expn(2, 1.0 / q) / _e2_1(), 1.0)  # 2π r u_θ
    # u_θ / r = frac / (2π r²), finite at r -> 0 (frac ~ r²)
    with np.errstate(divide="ignore", invalid="ignore"):
        ur = np.where(r2 > 0, frac / (2 * np.pi * np.where(r2 > 0, r2, 1.0)), 0.0)
    if comp == 0:
        return -dy * ur
    if comp == 1:
        return dx * ur
    return 0.0 * ur
