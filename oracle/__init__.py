"""ctypes binding of the plain CPU oracle (oracle/oracle.cpp).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package.  The product
path (paper_2404_16648_b200) never imports it, and it never imports the
product package.  Inputs come from the shared generator module `workloads`.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "oracle.cpp")
LIB = os.path.join(HERE, "liboracle.so")


def build(force: bool = False) -> str:
    """Compile the oracle: -O2 -ffp-contract=off, no fast-math."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        subprocess.check_call(["g++", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c++17",
                               "-fPIC", "-shared", SRC, "-o", LIB])
    return LIB


class OraParams(C.Structure):
    _fields_ = [("dim", C.c_int32), ("order", C.c_int32), ("root", C.c_int32 * 3),
                ("lo", C.c_double * 3), ("hi", C.c_double * 3), ("periodic", C.c_int32 * 3),
                ("max_level", C.c_int32), ("gamma", C.c_double), ("R", C.c_double),
                ("cp", C.c_double), ("p0", C.c_double), ("g", C.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB)
        dp, ip = C.POINTER(C.c_double), C.POINTER(C.c_int32)
        L.ora_lgl.argtypes = [C.c_int, dp, dp]
        L.ora_dmat.argtypes = [C.c_int, dp]
        L.ora_mortar_ops.argtypes = [C.c_int, dp, dp, dp, dp]
        L.ora_mesh_build.argtypes = [C.POINTER(OraParams), C.c_int64, C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]
        L.ora_mesh_free.argtypes = [C.c_void_p]
        L.ora_mesh_counts.argtypes = [C.c_void_p] + [C.POINTER(C.c_int64)] * 3
        L.ora_mesh_faces.argtypes = [C.c_void_p, ip, ip, ip]
        L.ora_rhs.argtypes = [C.POINTER(OraParams), C.c_void_p, dp, dp, dp, C.c_void_p]
        L.ora_rhs_nc.argtypes = [C.POINTER(OraParams), C.c_void_p, dp, dp, dp, C.c_void_p, C.c_int]
        L.ora_visc.argtypes = [C.POINTER(OraParams), C.c_void_p, dp, dp, C.c_double, dp]
        L.ora_tracer_rhs.argtypes = [C.POINTER(OraParams), C.c_void_p, dp, dp, C.c_int]
        L.ora_passive_rhs.argtypes = [C.POINTER(OraParams), C.c_void_p, dp, dp, dp, dp]
        L.ora_rk_stage.argtypes = [C.POINTER(OraParams), C.c_void_p, dp, C.c_int, C.c_double, dp, dp, dp, C.c_void_p]
        L.ora_refine.argtypes = [C.c_int, C.c_int, C.c_int64, ip, ip, dp, dp]
        L.ora_coarsen.argtypes = [C.c_int, C.c_int, C.c_int64, ip, ip, dp, dp]
        L.ora_integrals.argtypes = [C.POINTER(OraParams), C.c_void_p, dp, dp]
        L.ora_point_flux.argtypes = [C.POINTER(OraParams), C.c_int, dp, dp, dp]
        L.ora_rusanov.argtypes = [C.POINTER(OraParams), C.c_int, C.c_double, dp, dp, dp]
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ip(a):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def params(p) -> OraParams:
    root, lo, hi, per = p.padded()
    o = OraParams()
    o.dim, o.order, o.max_level = p.dim, p.order, p.max_level
    for i in range(3):
        o.root[i], o.lo[i], o.hi[i], o.periodic[i] = root[i], lo[i], hi[i], per[i]
    o.gamma, o.R, o.cp, o.p0, o.g = p.gamma, p.R, p.cp, p.p0, p.g
    return o


def lgl(N):
    x, w = np.zeros(N + 1), np.zeros(N + 1)
    assert lib().ora_lgl(N, _dp(x), _dp(w)) == 0
    return x, w


def dmat(N):
    D = np.zeros((N + 1, N + 1))
    assert lib().ora_dmat(N, _dp(D)) == 0
    return D


def mortar_ops(N):
    n = N + 1
    M, S, P, R = np.zeros((n, n)), np.zeros((2, n, n)), np.zeros((2, n, n)), np.zeros((2, n, n))
    assert lib().ora_mortar_ops(N, _dp(M), _dp(S), _dp(P), _dp(R)) == 0
    return M, S, P, R


class OracleError(RuntimeError):
    def __init__(self, code):
        super().__init__(f"oracle status {code}")
        self.code = code


class Mesh:
    """Oracle connectivity: canonical face lists (reading R29)."""

    def __init__(self, p, level, anchor):
        self.p = p
        self.op = params(p)
        self.level = np.ascontiguousarray(level, dtype=np.int8)
        self.anchor = np.ascontiguousarray(anchor, dtype=np.int32)
        h = C.c_void_p()
        st = lib().ora_mesh_build(C.byref(self.op), len(self.level), self.level.ctypes.data,
                                  self.anchor.ctypes.data, C.byref(h))
        if st != 0:
            raise OracleError(st)
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ora_mesh_free(self.h)
            self.h = None

    def faces(self):
        nc, nn, nb = C.c_int64(), C.c_int64(), C.c_int64()
        lib().ora_mesh_counts(self.h, C.byref(nc), C.byref(nn), C.byref(nb))
        w = 2 + 2 * (1 << (self.p.dim - 1))
        conf = np.zeros((nc.value, 4), np.int32)
        nonc = np.zeros((nn.value, w), np.int32)
        bnd = np.zeros((nb.value, 2), np.int32)
        lib().ora_mesh_faces(self.h, _ip(conf), _ip(nonc), _ip(bnd))
        return conf, nonc, bnd


def _mask(mask, E):
    if mask is None:
        return None
    m = np.zeros(E, np.uint8)
    m[np.asarray(mask)] = 1
    return m


def rhs(mesh: Mesh, bg, q, elems=None, ncmode=0):
    """dq/dt for all elements (or only `elems`; others are left 0).  ncmode 1: the
    pointwise-interpolation baseline on the coarse side of 2:1 faces (NEXT-3, R41)."""
    q = np.ascontiguousarray(q, dtype=np.float64)
    bg = np.ascontiguousarray(bg, dtype=np.float64)
    out = np.zeros(q.shape)  # calloc: pages of unselected elements are never touched
    m = _mask(elems, q.shape[0])
    if ncmode:
        code = lib().ora_rhs_nc(C.byref(mesh.op), mesh.h, _dp(bg), _dp(q), _dp(out),
                                None if m is None else m.ctypes.data, int(ncmode))
        if code != 0:
            raise OracleError(code)
    else:
        lib().ora_rhs(C.byref(mesh.op), mesh.h, _dp(bg), _dp(q), _dp(out),
                      None if m is None else m.ctypes.data)
    return out


def visc(mesh: Mesh, bg, q, mu):
    """NEXT-3 artificial viscosity V = mu div grad u' (reading R42)."""
    q = np.ascontiguousarray(q, dtype=np.float64)
    bg = np.ascontiguousarray(bg, dtype=np.float64)
    out = np.zeros_like(q)
    code = lib().ora_visc(C.byref(mesh.op), mesh.h, _dp(bg), _dp(q), float(mu), _dp(out))
    if code != 0:
        raise OracleError(code)
    return out


def tracer_rhs(mesh: Mesh, s, ncmode=0):
    """Kinematic tracer dC/dt (R43): s [E, F, Np] with field 0 = C, fields 1..dim = wind."""
    s = np.ascontiguousarray(s, dtype=np.float64)
    out = np.zeros_like(s)
    code = lib().ora_tracer_rhs(C.byref(mesh.op), mesh.h, _dp(s), _dp(out), int(ncmode))
    if code != 0:
        raise OracleError(code)
    return out[:, 0]


def passive_rhs(mesh: Mesh, bg, q, c):
    """Passive tracer of the Euler flow (R45): dC/dt for C = rho c, c [E, Np], advected by
    the Euler state q [E, F, Np] with the Euler faces' Rusanov wave speeds (mortars at 2:1 faces)."""
    q = np.ascontiguousarray(q, dtype=np.float64)
    c = np.ascontiguousarray(c, dtype=np.float64)
    bg = np.ascontiguousarray(bg, dtype=np.float64)
    out = np.zeros(c.shape)
    code = lib().ora_passive_rhs(C.byref(mesh.op), mesh.h, _dp(bg), _dp(q), _dp(c), _dp(out))
    if code != 0:
        raise OracleError(code)
    return out


def passive_rk_stage(mesh: Mesh, bg, stage, dt, q_in, c_n, c_in):
    """SSP-RK3 stage (R17, increment form) of the passive tracer with the Euler stage input q_in."""
    L = passive_rhs(mesh, bg, q_in, c_in)
    b = (1.0, 0.25, 2.0 / 3.0)[stage]
    if stage == 0:
        return c_in + dt * L
    return c_n + b * ((c_in - c_n) + dt * L)


def rk_stage_visc(mesh: Mesh, bg, stage, dt, q_n, q_in, mu):
    """SSP-RK3 stage (R17, increment form) of L + V: q_n + b ((q_in - q_n) + dt (L + V))."""
    L = rhs(mesh, bg, q_in) + visc(mesh, bg, q_in, mu)
    b = (1.0, 0.25, 2.0 / 3.0)[stage]
    if stage == 0:
        return q_in + dt * L
    return q_n + b * ((q_in - q_n) + dt * L)


def rk_stage(mesh: Mesh, bg, stage, dt, q_n, q_in, elems=None):
    q_n = np.ascontiguousarray(q_n, dtype=np.float64)
    q_in = np.ascontiguousarray(q_in, dtype=np.float64)
    bg = np.ascontiguousarray(bg, dtype=np.float64)
    out = np.zeros(q_in.shape)  # calloc: pages of unselected elements are never touched
    m = _mask(elems, q_in.shape[0])
    st = lib().ora_rk_stage(C.byref(mesh.op), mesh.h, _dp(bg), stage, dt, _dp(q_n), _dp(q_in), _dp(out),
                            None if m is None else m.ctypes.data)
    if st != 0:
        raise OracleError(st)
    return out


def rk3_step(mesh, bg, dt, q):
    q1 = rk_stage(mesh, bg, 0, dt, q, q)
    q2 = rk_stage(mesh, bg, 1, dt, q, q1)
    return rk_stage(mesh, bg, 2, dt, q, q2)


def refine(dim, N, parent_src, child0_dst, q_src, n_dst):
    parent_src = np.ascontiguousarray(parent_src, np.int32)
    child0_dst = np.ascontiguousarray(child0_dst, np.int32)
    q_src = np.ascontiguousarray(q_src, np.float64)
    q_dst = np.zeros((n_dst,) + q_src.shape[1:])
    lib().ora_refine(dim, N, len(parent_src), _ip(parent_src), _ip(child0_dst), _dp(q_src), _dp(q_dst))
    return q_dst


def coarsen(dim, N, child0_src, parent_dst, q_src, n_dst):
    child0_src = np.ascontiguousarray(child0_src, np.int32)
    parent_dst = np.ascontiguousarray(parent_dst, np.int32)
    q_src = np.ascontiguousarray(q_src, np.float64)
    q_dst = np.zeros((n_dst,) + q_src.shape[1:])
    lib().ora_coarsen(dim, N, len(child0_src), _ip(child0_src), _ip(parent_dst), _dp(q_src), _dp(q_dst))
    return q_dst


def integrals(mesh: Mesh, q):
    q = np.ascontiguousarray(q, np.float64)
    out = np.zeros(mesh.p.n_fields)
    lib().ora_integrals(C.byref(mesh.op), mesh.h, _dp(q), _dp(out))
    return out


def check_state(q):
    """State health scan, written out from its definition (SPEC.md:193-194:
    "rho > 0 at every node (positivity monitored, violation is a diagnostic
    event)"; NaN is a numerical failure).  q: [E][F][Np], fields
    (rho, momenta..., rho*theta).  Returns (number of non-finite values,
    nodes with rho <= 0, nodes with rho*theta <= 0, smallest element index with
    any of these or -1), by plain loops over elements."""
    q = np.asarray(q, np.float64)
    n_nonfinite = n_rho = n_theta = 0
    first = -1
    for e in range(q.shape[0]):
        a = int(np.count_nonzero(~np.isfinite(q[e])))
        b = int(np.count_nonzero(q[e, 0] <= 0.0))
        c = int(np.count_nonzero(q[e, -1] <= 0.0))
        n_nonfinite += a
        n_rho += b
        n_theta += c
        if first < 0 and a + b + c > 0:
            first = e
    return n_nonfinite, n_rho, n_theta, first


def point_flux(p, d, pt):
    """pt = (rho', U..., Theta', rho_bar, Theta_bar, P_bar) -> (F^d, (rho, Th, P', P, a))."""
    pt = np.ascontiguousarray(pt, np.float64)
    F, der = np.zeros(p.n_fields), np.zeros(5)
    op = params(p)
    lib().ora_point_flux(C.byref(op), d, _dp(pt), _dp(F), _dp(der))
    return F, der


def rusanov(p, d, sgn, ptL, ptR):
    ptL = np.ascontiguousarray(ptL, np.float64)
    ptR = np.ascontiguousarray(ptR, np.float64)
    out = np.zeros(p.n_fields)
    op = params(p)
    lib().ora_rusanov(C.byref(op), d, sgn, _dp(ptL), _dp(ptR), _dp(out))
    return out
