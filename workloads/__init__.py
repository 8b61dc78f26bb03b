"""Seeded synthetic inputs for the five BASELINE.json configurations.

This module is shared by the oracle tests and by the CUDA path (tests,
bench.py, smoke).  It holds NONE of the method's arithmetic: no flux, EOS
closure used by the RHS, differentiation, mortar or transfer operator.  It
only produces the inputs both sides consume bit-identically:

* the leaf list of a 2:1 face-balanced quad/oct-tree forest (level + integer
  anchor per leaf, canonical Morton order, reading R27);
* the hydrostatic background table (rho_bar, Theta_bar, P_bar) for every
  distinct node height, ordered (level, iz, k) (reading R3);
* the initial state [E][F][Np] (readings R21-R26).

To place samples at the LGL nodes it computes the node positions itself, by
Newton iteration in 50-digit decimal arithmetic -- an implementation of its
own, independent of both the oracle's and libdg's basis code.
"""
from __future__ import annotations

import dataclasses
import math
from decimal import Decimal, getcontext
from functools import lru_cache

import numpy as np

# Physical constants (reading R4; BASELINE.json configs[0]; g = 9.81 per SPEC).
GAMMA, R_GAS, CP, P0, GRAV = 1.4, 287.0, 1004.5, 1.0e5, 9.81
THETA0 = 300.0


@dataclasses.dataclass
class Params:
    dim: int
    order: int
    root: tuple
    lo: tuple
    hi: tuple
    periodic: tuple
    max_level: int
    gamma: float = GAMMA
    R: float = R_GAS
    cp: float = CP
    p0: float = P0
    g: float = GRAV

    @property
    def n1(self):
        return self.order + 1

    @property
    def n_nodes(self):
        return self.n1 ** self.dim

    @property
    def n_fields(self):
        return self.dim + 2

    @property
    def vert(self):
        return self.dim - 1

    def padded(self):
        """root/lo/hi/periodic padded to 3 entries (unused axes: 1 / 0 / 1 / 0)."""
        pad = 3 - self.dim
        return (tuple(self.root) + (1,) * pad, tuple(self.lo) + (0.0,) * pad,
                tuple(self.hi) + (1.0,) * pad, tuple(self.periodic) + (0,) * pad)


@dataclasses.dataclass
class Workload:
    name: str
    params: Params
    level: np.ndarray      # int8 [E]
    anchor: np.ndarray     # int32 [E, dim]
    bg: np.ndarray         # float64 [rows, 3] (rho_bar, Theta_bar, P_bar)
    q0: np.ndarray         # float64 [E, F, Np] compact
    dt: float
    note: str = ""

    @property
    def n_elem(self):
        return int(self.level.shape[0])

    @property
    def n_dof(self):
        return self.n_elem * self.params.n_fields * self.params.n_nodes


# --------------------------------------------------------------------------
# LGL node positions (for sampling only), 50-digit Newton
# --------------------------------------------------------------------------
@lru_cache(maxsize=None)
def lgl_nodes(N: int) -> np.ndarray:
    getcontext().prec = 50
    xs = []
    for i in range(N + 1):
        x = Decimal(repr(-math.cos(math.pi * i / N)))
        if i == 0 or i == N:
            xs.append(float(x.to_integral_value()) if abs(x) > 0.5 else 0.0)
            continue
        for _ in range(200):
            p0, p1 = Decimal(1), x
            for k in range(2, N + 1):
                p0, p1 = p1, ((2 * k - 1) * x * p1 - (k - 1) * p0) / k
            # q(x) = x P_N - P_{N-1}; q'(x) = (N+1) P_N
            dx = (x * p1 - p0) / ((N + 1) * p1)
            x -= dx
            if abs(dx) < Decimal("1e-45"):
                break
        xs.append(0.0 if abs(x) < Decimal("1e-30") else float(x))
    xs = np.array(xs)
    xs[0], xs[-1] = -1.0, 1.0
    return xs


# --------------------------------------------------------------------------
# Forests
# --------------------------------------------------------------------------
class Forest:
    """Set of leaves {(level, a0, a1, a2)} over a root grid."""

    def __init__(self, p: Params):
        self.p = p
        self.leaves = set()
        r = p.padded()[0]
        for a2 in range(r[2]):
            for a1 in range(r[1]):
                for a0 in range(r[0]):
                    self.leaves.add((0, a0, a1, a2))

    def children(self, leaf):
        l, a0, a1, a2 = leaf
        out = []
        for b in range(1 << self.p.dim):
            c = [2 * a0 + (b & 1), 2 * a1 + ((b >> 1) & 1), 2 * a2 + ((b >> 2) & 1)]
            for ax in range(self.p.dim, 3):
                c[ax] = 0
            out.append((l + 1, c[0], c[1], c[2]))
        return out

    def split(self, leaf):
        self.leaves.remove(leaf)
        for c in self.children(leaf):
            self.leaves.add(c)

    def containing(self, lev, a):
        """Leaf containing cell (lev, a), or None if that cell is subdivided."""
        for l in range(lev, -1, -1):
            sh = lev - l
            key = (l, a[0] >> sh, a[1] >> sh, a[2] >> sh)
            if key in self.leaves:
                return key
        return None

    def neighbour_cell(self, lev, a, d, s):
        p = self.p
        ext = p.root[d] << lev
        b = list(a)
        b[d] += s
        if b[d] < 0 or b[d] >= ext:
            if not p.periodic[d]:
                return None
            b[d] %= ext
        return b

    def balance(self):
        """Face 2:1 balance including periodic seams (reading R15): ripple from
        the finest level down; the result is the coarsest balanced refinement."""
        p = self.p
        maxl = max(l for l, *_ in self.leaves)
        for lev in range(maxl, 1, -1):
            for leaf in sorted(x for x in self.leaves if x[0] == lev):
                if leaf not in self.leaves:
                    continue
                a = leaf[1:]
                for d in range(p.dim):
                    for s in (-1, 1):
                        nb = self.neighbour_cell(lev, a, d, s)
                        if nb is None:
                            continue
                        while True:
                            c = self.containing(lev, nb)
                            if c is None or c[0] >= lev - 1:
                                break
                            self.split(c)

    def ordered(self):
        """(level int8 [E], anchor int32 [E, dim]) in Morton order (R27)."""
        p = self.p
        L = max(l for l, *_ in self.leaves)
        pad = max(p.root[:p.dim])
        bits = (pad - 1).bit_length() + L
        arr = np.array(sorted(self.leaves), dtype=np.int64)
        lev = arr[:, 0]
        fine = arr[:, 1:4] << (L - lev)[:, None]
        key = np.zeros(len(arr), dtype=np.uint64)
        for bit in range(bits):
            for ax in range(p.dim):
                key |= (((fine[:, ax] >> bit) & 1).astype(np.uint64)
                        << np.uint64(bit * p.dim + ax))
        order = np.argsort(key, kind="stable")
        arr = arr[order]
        return arr[:, 0].astype(np.int8), np.ascontiguousarray(arr[:, 1:1 + p.dim].astype(np.int32))


# --------------------------------------------------------------------------
# Background table and node coordinates
# --------------------------------------------------------------------------
def table_heights(p: Params) -> np.ndarray:
    """Height of every table row (level, iz, k): z = lo_z + (iz + (1+xi_k)/2) h_l,
    h_l = ((hi_z - lo_z)/root_z)/2^l (reading R3)."""
    xi = lgl_nodes(p.order)
    v = p.vert
    zs = []
    for l in range(p.max_level + 1):
        h = ((p.hi[v] - p.lo[v]) / p.root[v]) / (2.0 ** l)
        iz = np.arange(p.root[v] << l, dtype=np.float64)
        zs.append((p.lo[v] + (iz[:, None] + (1.0 + xi[None, :]) / 2.0) * h).ravel())
    return np.concatenate(zs)


def background_table(p: Params, theta0: float = THETA0) -> np.ndarray:
    """Isentropic hydrostatic background: pi = 1 - g z/(cp theta0),
    P_bar = p0 pi^(cp/R), Theta_bar = (p0/R)(P_bar/p0)^(1/gamma), rho_bar = Theta_bar/theta0."""
    z = table_heights(p)
    ex = 1.0 - p.g * z / (p.cp * theta0)
    pbar = p.p0 * ex ** (p.cp / p.R)
    thbar = (p.p0 / p.R) * (pbar / p.p0) ** (1.0 / p.gamma)
    rhobar = thbar / theta0
    return np.ascontiguousarray(np.stack([rhobar, thbar, pbar], axis=1))


def row_offsets(p: Params) -> np.ndarray:
    off = [0]
    for l in range(p.max_level + 1):
        off.append(off[-1] + (p.root[p.vert] << l) * p.n1)
    return np.array(off, dtype=np.int64)


def node_coords(p: Params, level: np.ndarray, anchor: np.ndarray, elems=None):
    """Physical coordinates [E, dim, Np] of every node (x fastest, R28)."""
    xi = lgl_nodes(p.order)
    if elems is None:
        elems = np.arange(level.shape[0])
    lev = level[elems].astype(np.int64)
    n1, Np = p.n1, p.n_nodes
    node = np.arange(Np)
    out = np.empty((len(elems), p.dim, Np))
    for d in range(p.dim):
        i_d = (node // (n1 ** d)) % n1
        h = ((p.hi[d] - p.lo[d]) / p.root[d]) / (2.0 ** lev)
        a = anchor[elems, d].astype(np.float64)
        out[:, d, :] = p.lo[d] + (a[:, None] + (1.0 + xi[i_d][None, :]) / 2.0) * h[:, None]
    return out


def node_background(p: Params, bg: np.ndarray, level, anchor, elems=None):
    """Background rows [E, Np, 3] of every node."""
    if elems is None:
        elems = np.arange(level.shape[0])
    off = row_offsets(p)
    n1 = p.n1
    k = (np.arange(p.n_nodes) // (n1 ** p.vert)) % n1
    rows = off[level[elems].astype(np.int64)][:, None] + anchor[elems, p.vert].astype(np.int64)[:, None] * n1 + k[None, :]
    return bg[rows]


def pressure_balanced_state(p: Params, bgn: np.ndarray, thetap: np.ndarray) -> np.ndarray:
    """Reading R22: Theta = Theta_bar(z), rho = Theta_bar/(theta0 + theta'), U = 0."""
    E = bgn.shape[0]
    q = np.zeros((E, p.n_fields, p.n_nodes))
    q[:, 0, :] = bgn[:, :, 1] / (THETA0 + thetap)
    q[:, p.dim + 1, :] = bgn[:, :, 1]
    return q


def cosine_bubble(r):
    return np.where(r <= 1.0, 0.5 * (1.0 + np.cos(np.pi * np.minimum(r, 1.0))), 0.0)


# --------------------------------------------------------------------------
# Configurations (BASELINE.json configs[0..4]; readings R21-R26)
# --------------------------------------------------------------------------
def c1() -> Workload:
    p = Params(2, 4, (10, 10), (0.0, 0.0), (1000.0, 1000.0), (0, 0), 0)
    f = Forest(p)
    level, anchor = f.ordered()
    bg = background_table(p)
    X = node_coords(p, level, anchor)
    r = np.hypot(X[:, 0] - 500.0, X[:, 1] - 350.0) / 250.0
    q = pressure_balanced_state(p, node_background(p, bg, level, anchor), 0.5 * cosine_bubble(r))
    xi = np.random.default_rng(1).uniform(-1.0, 1.0, size=q.shape)
    q = q * (1.0 + 1e-6 * xi)
    return Workload("c1", p, level, anchor, bg, q, 0.01, "2D 10x10 N=4 warm bubble + 1e-6 noise")


def c2_forest():
    p = Params(2, 4, (32, 8), (0.0, 0.0), (25600.0, 6400.0), (0, 0), 2)
    f = Forest(p)

    def centroid(leaf):
        l = leaf[0]
        return [p.lo[d] + (leaf[1 + d] + 0.5) * ((p.hi[d] - p.lo[d]) / p.root[d]) / 2 ** l for d in range(2)]

    for lev in (0, 1):
        for leaf in sorted(x for x in f.leaves if x[0] == lev):
            cx, cz = centroid(leaf)
            if math.hypot(cx - 0.0, cz - 3000.0) <= 4000.0:
                f.split(leaf)
    f.balance()
    return p, f


def c2() -> Workload:
    p, f = c2_forest()
    level, anchor = f.ordered()
    bg = background_table(p)
    X = node_coords(p, level, anchor)
    r = np.sqrt((X[:, 0] / 4000.0) ** 2 + ((X[:, 1] - 3000.0) / 2000.0) ** 2)
    q = pressure_balanced_state(p, node_background(p, bg, level, anchor), -15.0 * cosine_bubble(r))
    return Workload("c2", p, level, anchor, bg, q, 0.02, "2D quadtree 3 levels, N=4, cold bubble")


def _bubble3d(p, level, anchor, bg, rng):
    X = node_coords(p, level, anchor)
    r = np.sqrt((X[:, 0] - 500.0) ** 2 + (X[:, 1] - 500.0) ** 2 + (X[:, 2] - 350.0) ** 2) / 250.0
    q = pressure_balanced_state(p, node_background(p, bg, level, anchor), 0.5 * cosine_bubble(r))
    u = rng.uniform(-0.01, 0.01, size=(q.shape[0], 3, q.shape[2]))
    q[:, 1:4, :] = q[:, 0:1, :] * u
    return q


def c3() -> Workload:
    p = Params(3, 4, (16, 16, 16), (0.0, 0.0, 0.0), (1000.0, 1000.0, 1000.0), (1, 1, 0), 0)
    level, anchor = Forest(p).ordered()
    bg = background_table(p)
    q = _bubble3d(p, level, anchor, bg, np.random.default_rng(3))
    return Workload("c3", p, level, anchor, bg, q, 0.005, "3D 16^3 N=4 warm bubble + velocity noise")


def c4_forest(rng):
    p = Params(3, 4, (32, 32, 16), (0.0, 0.0, 0.0), (1000.0, 1000.0, 1000.0), (1, 1, 0), 2)
    f = Forest(p)
    ncell = 32 * 32 * 16
    perm = rng.permutation(ncell)
    s1 = perm[: round(0.10 * ncell)]
    s2 = s1[: round(0.02 * ncell)]

    def cell(i):
        return (0, int(i % 32), int((i // 32) % 32), int(i // 1024))

    for i in s1:
        f.split(cell(i))
    for i in s2:
        for ch in f.children(cell(i)):
            f.split(ch)
    f.balance()
    return p, f


def c4() -> Workload:
    rng = np.random.default_rng(4)
    p, f = c4_forest(rng)
    level, anchor = f.ordered()
    bg = background_table(p)
    q = _bubble3d(p, level, anchor, bg, rng)
    return Workload("c4", p, level, anchor, bg, q, 5e-4, "3D octree 32x32x16 + 10%/2% refinement, N=4")


def c4_projection_flags(w: Workload):
    """Refine flags for c4's projection pass: Bernoulli(0.1) per leaf below
    max_level, default_rng(40) (reading R25)."""
    rng = np.random.default_rng(40)
    flags = rng.random(w.n_elem) < 0.1
    flags &= w.level < w.params.max_level
    return np.nonzero(flags)[0].astype(np.int32)


def c5(order: int = 7, root=(64, 64, 32)) -> Workload:
    """BASELINE configs[4].  `root` other than the default gives a smaller box
    with the same element size h = 156.25 m, order and state recipe (used only
    as the bounded CPU-oracle sample of bench.py)."""
    root = tuple(int(r) for r in root)
    p = Params(3, order, root, (0.0, 0.0, 0.0), tuple(156.25 * r for r in root), (1, 1, 0), 0)
    level, anchor = uniform_morton(p)
    bg = background_table(p)
    rng = np.random.default_rng(5)
    centres = rng.uniform(np.array(p.lo), np.array(p.hi), size=(20, 3))
    xi = lgl_nodes(order)
    n1 = p.n1
    # theta' = sum_k exp(-|x-c_k|^2/300^2), written per axis (separable form).
    # Periodic axes use the minimum-image distance with the seam coordinate
    # wrapped exactly (x = hi -> lo), so the field is bitwise continuous across
    # the periodic seams (reading R26).
    g1 = []
    for d in range(3):
        L = p.hi[d] - p.lo[d]
        h = L / p.root[d]
        coord = (p.lo[d] + (np.arange(p.root[d])[:, None] + (1.0 + xi[None, :]) / 2.0) * h)  # [root, n1]
        dx = coord[None, :, :] - centres[:, d][:, None, None]
        if p.periodic[d]:
            coord = np.where(coord >= p.hi[d], coord - L, coord)
            dx = coord[None, :, :] - centres[:, d][:, None, None]
            dx = np.where(dx > 0.5 * L, dx - L, np.where(dx < -0.5 * L, dx + L, dx))
        g1.append(np.exp(-(dx ** 2) / 300.0 ** 2))  # [20, root, n1]
    E = level.shape[0]
    q = np.empty((E, p.n_fields, p.n_nodes))
    bgn_off = row_offsets(p)
    chunk = 8192
    for s in range(0, E, chunk):
        sl = slice(s, min(E, s + chunk))
        ax, ay, az = anchor[sl, 0], anchor[sl, 1], anchor[sl, 2]
        gx, gy, gz = g1[0][:, ax, :], g1[1][:, ay, :], g1[2][:, az, :]   # [20, e, n1]
        th = np.einsum("kex,key,kez->ezyx", gx, gy, gz).reshape(-1, p.n_nodes)
        k = np.arange(p.n_nodes) // (n1 * n1)
        rows = bgn_off[0] + az.astype(np.int64)[:, None] * n1 + k[None, :]
        thbar = bg[rows, 1]
        q[sl, 0, :] = thbar / (THETA0 + th)
        q[sl, 1:4, :] = 0.0
        q[sl, 4, :] = thbar
    return Workload("c5", p, level, anchor, bg, q, 0.005,
                    f"3D 64x64x32 N={order}, 20 Gaussian theta bumps")


def uniform_morton(p: Params):
    """Uniform level-0 forest in Morton order (fast path of Forest.ordered)."""
    r = p.root[: p.dim]
    grids = np.meshgrid(*[np.arange(n) for n in r], indexing="ij")
    a = np.stack([g.ravel() for g in grids], axis=1).astype(np.int64)
    bits = (max(r) - 1).bit_length()
    key = np.zeros(len(a), dtype=np.uint64)
    for bit in range(bits):
        for ax in range(p.dim):
            key |= (((a[:, ax] >> bit) & 1).astype(np.uint64) << np.uint64(bit * p.dim + ax))
    order = np.argsort(key, kind="stable")
    a = a[order]
    return np.zeros(len(a), dtype=np.int8), np.ascontiguousarray(a.astype(np.int32))


# --------------------------------------------------------------------------
# NEXT-2: isentropic vortex (§4.1; reading R36)
# --------------------------------------------------------------------------
VORTEX_BETA, VORTEX_UINF = 5.0, (1.0, 1.0)


def vortex_params(nx: int = 32, order: int = 3) -> Params:
    """[-6, 6]^2, nx x nx level-0 elements, periodic, g = 0."""
    return Params(2, order, (nx, nx), (-6.0, -6.0), (6.0, 6.0), (1, 1), 0, g=0.0)


def vortex_background(p: Params) -> np.ndarray:
    """Constant free-stream background rho = Theta = P = 1 (theta_inf = 1, p_inf = 1)."""
    rows = int(row_offsets(p)[-1])
    return np.ones((rows, 3))


def vortex_state(p: Params, level, anchor, t: float = 0.0, beta: float = VORTEX_BETA,
                 uinf=VORTEX_UINF) -> np.ndarray:
    """Closed-form isentropic vortex at time t: the t = 0 vortex (centre (0, 0),
    P:373) translated by uinf t on the periodic square (minimum image).  In the
    conservative potential-temperature variables of the path (R36): theta = 1
    everywhere (isentropic), T = 1 - (gamma-1) beta^2/(8 gamma pi^2) exp(1 - r^2),
    rho = T^(1/(gamma-1)), so P = Theta^gamma = rho^gamma;
    (u, v) = uinf + beta/(2 pi) exp((1 - r^2)/2) (-(y - yc), x - xc)."""
    X = node_coords(p, level, anchor)
    g = p.gamma
    rel = []
    for d in range(2):
        L = p.hi[d] - p.lo[d]
        c = 0.0 + uinf[d] * t
        dx = X[:, d] - c
        dx = dx - L * np.round(dx / L)
        rel.append(dx)
    r2 = rel[0] ** 2 + rel[1] ** 2
    T = 1.0 - (g - 1.0) * beta ** 2 / (8.0 * g * math.pi ** 2) * np.exp(1.0 - r2)
    rho = T ** (1.0 / (g - 1.0))
    amp = beta / (2.0 * math.pi) * np.exp(0.5 * (1.0 - r2))
    u = uinf[0] - amp * rel[1]
    v = uinf[1] + amp * rel[0]
    q = np.empty((X.shape[0], 4, p.n_nodes))
    q[:, 0] = rho
    q[:, 1] = rho * u
    q[:, 2] = rho * v
    q[:, 3] = rho
    return q


def vortex(nx: int = 32, order: int = 3) -> Workload:
    """NEXT-2 workload: the paper's uniform-grid vortex run (32 x 32, N = 3,
    dt = 2.5e-4 s forward Euler)."""
    p = vortex_params(nx, order)
    level, anchor = uniform_morton(p)
    bg = vortex_background(p)
    return Workload("vortex", p, level, anchor, bg, vortex_state(p, level, anchor), 2.5e-4,
                    f"2D isentropic vortex {nx}x{nx} N={order}, periodic, g = 0")


def lgl_weights(N: int) -> np.ndarray:
    """LGL quadrature weights 2 / (N (N+1) P_N(x_i)^2) at lgl_nodes(N) (diagnostics only)."""
    x = lgl_nodes(N)
    p0, p1 = np.ones_like(x), x.copy()
    for k in range(2, N + 1):
        p0, p1 = p1, ((2 * k - 1) * x * p1 - (k - 1) * p0) / k
    return 2.0 / (N * (N + 1) * p1 ** 2)


def vortex_l2(p: Params, q: np.ndarray, qex: np.ndarray, level=None) -> dict:
    """Error norms of q against the exact state: `paper` is the
    printed formula (1/N_dof) sqrt(sum |q - q_ex|^2) with N_dof = nodes x fields,
    `rms` = sqrt(sum |q - q_ex|^2 / N_dof) (reading R36).  With the leaf levels,
    also `l2` = sqrt(sum_f int |q_f - q_ex,f|^2 dx / (area F)) by LGL quadrature,
    which unlike the node RMS does not depend on where the nodes are (AMR)."""
    d2 = (q - qex) ** 2
    e2 = float(np.sum(d2))
    n = q.size
    out = {"paper": math.sqrt(e2) / n, "rms": math.sqrt(e2 / n), "max": float(np.abs(q - qex).max())}
    if level is not None:
        w1 = lgl_weights(p.order)
        n1 = p.n1
        node = np.arange(p.n_nodes)
        w = np.ones(p.n_nodes)
        for d in range(p.dim):
            w = w * w1[(node // n1 ** d) % n1]
        jac = np.ones(len(level))
        area = 1.0
        for d in range(p.dim):
            jac = jac * 0.5 * (p.hi[d] - p.lo[d]) / p.root[d] / 2.0 ** level.astype(np.float64)
            area *= p.hi[d] - p.lo[d]
        integ = float(np.sum(jac[:, None] * (d2 * w[None, None, :]).sum(axis=1)))
        out["l2"] = math.sqrt(integ / (area * q.shape[1]))
    return out


# --------------------------------------------------------------------------
# NEXT-3 kinematic tracer: the paper's LeVeque swirl (§4.2; R43)
# --------------------------------------------------------------------------
LEVEQUE_T = 5.0


def leveque_params(nx: int = 16, order: int = 4, max_level: int = 2) -> Params:
    """[0,1]^2, nx x nx root elements, walls (the wind has no normal component there)."""
    return Params(2, order, (nx, nx), (0.0, 0.0), (1.0, 1.0), (0, 0), max_level)


def leveque_wind(p: Params, level, anchor, t: float, T: float = LEVEQUE_T) -> np.ndarray:
    """u = sin^2(pi x) sin(2 pi y) g(t), v = -sin^2(pi y) sin(2 pi x) g(t), g = cos(pi t / T)."""
    X = node_coords(p, level, anchor)
    g = math.cos(math.pi * t / T)
    x, y = X[:, 0], X[:, 1]
    return np.stack([np.sin(math.pi * x) ** 2 * np.sin(2 * math.pi * y) * g,
                     -np.sin(math.pi * y) ** 2 * np.sin(2 * math.pi * x) * g], axis=1)


def leveque_state(p: Params, level, anchor, t: float = 0.0, T: float = LEVEQUE_T, hmax: float = 1.0) -> np.ndarray:
    """[E, F, Np]: field 0 = the cosine bell at (0.25, 0.25), r_c = 0.25, exact at
    t = 0 and t = T; fields 1..2 = the wind at time t; field 3 unused (0)."""
    X = node_coords(p, level, anchor)
    r = np.hypot(X[:, 0] - 0.25, X[:, 1] - 0.25) / 0.25
    s = np.zeros((len(level), p.n_fields, p.n_nodes))
    s[:, 0] = hmax * cosine_bubble(r)
    s[:, 1:3] = leveque_wind(p, level, anchor, t, T)
    return s

CONFIGS = {"c1": c1, "c2": c2, "c3": c3, "c4": c4, "c5": c5,
           # extra N=4 HBM point (not in BASELINE): c5's mesh at N=4
           "c5n4": lambda: c5(order=4),
           # NEXT-2: the paper's isentropic vortex
           "vortex": vortex}


def get(name: str) -> Workload:
    return CONFIGS[name]()


def random_forest(seed: int, dim: int, order: int = 2, max_level: int = 3, frac: float = 0.3):
    """Small seeded random balanced forest for connectivity tests: random root
    grid (1-4 cells per axis), random periodicity, random refinement of a
    fraction of leaves level by level, then face balance."""
    rng = np.random.default_rng(1000 + seed)
    root = tuple(int(x) for x in rng.integers(1, 5, size=dim))
    per = tuple(int(x) for x in rng.integers(0, 2, size=dim))
    lo = tuple(0.0 for _ in range(dim))
    hi = tuple(float(100 * r) for r in root)
    p = Params(dim, order, root, lo, hi, per, max_level)
    f = Forest(p)
    for lev in range(max_level):
        cand = sorted(x for x in f.leaves if x[0] == lev)
        pick = rng.random(len(cand)) < frac
        for leaf, k in zip(cand, pick):
            if k:
                f.split(leaf)
    f.balance()
    level, anchor = f.ordered()
    return p, level, anchor
