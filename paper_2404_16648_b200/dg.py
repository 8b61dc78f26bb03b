"""Thin ctypes binding of libdg (include/dg.h).

Argument marshalling only: every step of the hot path runs in the library's
sm_100a kernels.  Device buffers are torch CUDA tensors (or raw device
addresses); streams are torch.cuda.Stream objects, raw cudaStream_t values,
or None for the current torch stream.  There is no CPU fallback: if
lib/libdg.so is missing or fails to load this module raises ImportError.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# DG_LIB overrides the library path (development: A/B builds of the same sources)
LIB_PATH = os.environ.get("DG_LIB", os.path.join(HERE, "lib", "libdg.so"))

STATUS = {0: "DG_OK", -1: "DG_ERR_ARG", -2: "DG_ERR_UNSUPPORTED", -3: "DG_ERR_MESH",
          -4: "DG_ERR_UNBALANCED", -5: "DG_ERR_STATE", -6: "DG_ERR_CUDA", -7: "DG_ERR_OOM"}

SYMBOLS = ["dg_create", "dg_destroy", "dg_last_error", "dg_mesh_build", "dg_mesh_upload",
           "dg_mesh_face_counts", "dg_mesh_faces", "dg_state_layout", "dg_state_alloc", "dg_state_free",
           "dg_set_background", "dg_rhs", "dg_rk_stage", "dg_amr_project_refine", "dg_amr_project_coarsen",
           "dg_copy_elements", "dg_integrals", "dg_rhs_host", "dg_rk3_step_host", "dg_launch_count",
           "dg_amr_indicator", "dg_regrid_plan_create", "dg_regrid_plan_sizes", "dg_regrid_plan_get",
           "dg_regrid_plan_destroy", "dg_mesh_build_part", "dg_mesh_upload_part", "dg_part_info",
           "dg_part_exchange_lists", "dg_set_nonconforming", "dg_set_viscosity", "dg_tracer_rhs",
           "dg_tracer_rk_stage", "dg_part_face_lists", "dg_pack_faces", "dg_unpack_faces", "dg_check_state", "dg_rhs_elems",
           "dg_rk_stage_elems", "dg_passive_rhs", "dg_passive_rk_stage"]


class DGError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class dg_params(C.Structure):
    _fields_ = [("dim", C.c_int32), ("order", C.c_int32), ("root", C.c_int32 * 3),
                ("lo", C.c_double * 3), ("hi", C.c_double * 3), ("periodic", C.c_int32 * 3),
                ("max_level", C.c_int32), ("gamma", C.c_double), ("R", C.c_double),
                ("cp", C.c_double), ("p0", C.c_double), ("g", C.c_double)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libdg not built: {LIB_PATH} missing (run paper_2404_16648_b200.build.build())")
    lib = C.CDLL(LIB_PATH)
    vp, i64, i32 = C.c_void_p, C.c_int64, C.c_int32
    sig = {
        "dg_create": ([C.POINTER(dg_params), C.POINTER(vp)], C.c_int),
        "dg_destroy": ([vp], None),
        "dg_last_error": ([], C.c_char_p),
        "dg_mesh_build": ([vp, i64, vp, vp], C.c_int),
        "dg_mesh_upload": ([vp, i64, vp, vp, vp], C.c_int),
        "dg_mesh_face_counts": ([vp, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64)], C.c_int),
        "dg_mesh_faces": ([vp, vp, vp, vp], C.c_int),
        "dg_state_layout": ([vp, C.POINTER(i64), C.POINTER(i32), C.POINTER(i32), C.POINTER(i64)], C.c_int),
        "dg_state_alloc": ([vp, C.POINTER(vp), vp], C.c_int),
        "dg_state_free": ([vp, vp], C.c_int),
        "dg_set_background": ([vp, vp, i64, vp], C.c_int),
        "dg_rhs": ([vp, vp, vp, vp], C.c_int),
        "dg_rk_stage": ([vp, i32, C.c_double, vp, vp, vp, vp], C.c_int),
        "dg_rhs_elems": ([vp, vp, vp, i64, vp, vp], C.c_int),
        "dg_passive_rhs": ([vp, vp, vp, vp, vp], C.c_int),
        "dg_passive_rk_stage": ([vp, i32, C.c_double, vp, vp, vp, vp, vp], C.c_int),
        "dg_rk_stage_elems": ([vp, i32, C.c_double, vp, vp, vp, i64, vp, vp], C.c_int),
        "dg_amr_project_refine": ([vp, i64, vp, vp, vp, vp, vp], C.c_int),
        "dg_amr_project_coarsen": ([vp, i64, vp, vp, vp, vp, vp], C.c_int),
        "dg_copy_elements": ([vp, i64, vp, vp, vp, vp, vp], C.c_int),
        "dg_integrals": ([vp, vp, vp, vp], C.c_int),
        "dg_check_state": ([vp, vp, vp, vp], C.c_int),
        "dg_rhs_host": ([vp, vp, vp, vp], C.c_int),
        "dg_rk3_step_host": ([vp, C.c_double, i32, vp, vp], C.c_int),
        "dg_launch_count": ([vp], i64),
        "dg_amr_indicator": ([vp, i32, vp, vp, vp], C.c_int),
        "dg_regrid_plan_create": ([vp, vp, C.c_double, C.c_double, i32, C.POINTER(vp)], C.c_int),
        "dg_regrid_plan_sizes": ([vp, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64), C.POINTER(i64)], C.c_int),
        "dg_regrid_plan_get": ([vp, vp, vp, vp, vp, vp, vp, vp, vp], C.c_int),
        "dg_regrid_plan_destroy": ([vp], None),
        "dg_mesh_build_part": ([vp, i64, vp, vp, i32, i32], C.c_int),
        "dg_mesh_upload_part": ([vp, i64, vp, vp, i32, i32, vp], C.c_int),
        "dg_part_info": ([vp, C.POINTER(i32), C.POINTER(i32), C.POINTER(i64), C.POINTER(i64), C.POINTER(i64)], C.c_int),
        "dg_part_exchange_lists": ([vp, vp, vp, vp], C.c_int),
        "dg_set_nonconforming": ([vp, i32], C.c_int),
        "dg_set_viscosity": ([vp, C.c_double], C.c_int),
        "dg_tracer_rhs": ([vp, vp, vp, vp], C.c_int),
        "dg_tracer_rk_stage": ([vp, i32, C.c_double, vp, vp, vp, vp], C.c_int),
        "dg_part_face_lists": ([vp, vp, vp, vp, vp], C.c_int),
        "dg_pack_faces": ([vp, i64, vp, vp, vp, vp], C.c_int),
        "dg_unpack_faces": ([vp, i64, vp, vp, vp, vp], C.c_int),
    }
    for name, (args, res) in sig.items():
        if "DG_LIB" in os.environ and not hasattr(lib, name):
            continue  # development A/B against an older build: newer entry points absent
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


lib = _load()


def _check(code):
    if code != 0:
        raise DGError(code, lib.dg_last_error().decode())


def _ptr(x):
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    return x.data_ptr()  # torch tensor


def _stream(s):
    if s is None:
        try:
            import torch
            if torch.cuda.is_available():
                return torch.cuda.current_stream().cuda_stream
        except ImportError:
            pass
        return None
    if isinstance(s, int):
        return s
    return s.cuda_stream


def make_params(p) -> dg_params:
    """dg_params from an object with dim/order/root/lo/hi/periodic/max_level and constants."""
    o = dg_params()
    root = (tuple(p.root) + (1, 1, 1))[:3]
    lo = (tuple(p.lo) + (0.0, 0.0, 0.0))[:3]
    hi = (tuple(p.hi) + (1.0, 1.0, 1.0))[:3]
    per = (tuple(p.periodic) + (0, 0, 0))[:3]
    o.dim, o.order, o.max_level = p.dim, p.order, p.max_level
    for i in range(3):
        o.root[i], o.lo[i], o.hi[i], o.periodic[i] = root[i], lo[i], hi[i], per[i]
    o.gamma, o.R, o.cp, o.p0, o.g = p.gamma, p.R, p.cp, p.p0, p.g
    return o


class DG:
    """One libdg context (dg_create ... dg_destroy)."""

    def __init__(self, params):
        self.params = params
        self._p = make_params(params)
        h = C.c_void_p()
        _check(lib.dg_create(C.byref(self._p), C.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None) and lib is not None:
            lib.dg_destroy(self.h)
        self.h = None

    def __del__(self):
        self.close()

    # ---------------------------------------------------------------- mesh
    def mesh_build(self, level, anchor):
        level = np.ascontiguousarray(level, np.int8)
        anchor = np.ascontiguousarray(anchor, np.int32)
        _check(lib.dg_mesh_build(self.h, len(level), level.ctypes.data, anchor.ctypes.data))

    def mesh_upload(self, level, anchor, stream=None):
        level = np.ascontiguousarray(level, np.int8)
        anchor = np.ascontiguousarray(anchor, np.int32)
        _check(lib.dg_mesh_upload(self.h, len(level), level.ctypes.data, anchor.ctypes.data, _stream(stream)))

    def mesh_face_counts(self):
        a, b, c = C.c_int64(), C.c_int64(), C.c_int64()
        _check(lib.dg_mesh_face_counts(self.h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def mesh_faces(self):
        nc, nn, nb = self.mesh_face_counts()
        w = 2 + 2 * (1 << (self.params.dim - 1))
        conf = np.zeros((nc, 4), np.int32)
        nonc = np.zeros((nn, w), np.int32)
        bnd = np.zeros((nb, 2), np.int32)
        _check(lib.dg_mesh_faces(self.h, conf.ctypes.data, nonc.ctypes.data, bnd.ctypes.data))
        return conf, nonc, bnd

    def state_layout(self):
        e, s = C.c_int64(), C.c_int64()
        f, n = C.c_int32(), C.c_int32()
        _check(lib.dg_state_layout(self.h, C.byref(e), C.byref(f), C.byref(n), C.byref(s)))
        return e.value, f.value, n.value, s.value

    # ---------------------------------------------------------------- state
    def set_background(self, table, stream=None):
        _check(lib.dg_set_background(self.h, _ptr(table), int(table.shape[0]), _stream(stream)))

    def rhs(self, q, dqdt, stream=None):
        _check(lib.dg_rhs(self.h, _ptr(q), _ptr(dqdt), _stream(stream)))

    def rk_stage(self, stage, dt, q_n, q_in, q_out, stream=None):
        _check(lib.dg_rk_stage(self.h, int(stage), float(dt), _ptr(q_n), _ptr(q_in), _ptr(q_out), _stream(stream)))

    def rhs_elems(self, q, dqdt, elems, stream=None):
        """dg_rhs on the local elements listed in `elems` (device int32 tensor) only."""
        _check(lib.dg_rhs_elems(self.h, _ptr(q), _ptr(dqdt), int(elems.numel()), _ptr(elems), _stream(stream)))

    def rk_stage_elems(self, stage, dt, q_n, q_in, q_out, elems, stream=None):
        """dg_rk_stage on the local elements listed in `elems` (device int32 tensor) only."""
        _check(lib.dg_rk_stage_elems(self.h, int(stage), float(dt), _ptr(q_n), _ptr(q_in), _ptr(q_out),
                                     int(elems.numel()), _ptr(elems), _stream(stream)))

    def passive_rhs(self, q, c, dcdt, stream=None):
        """Passive tracer of the Euler flow (R45): dcdt field 0 = dC/dt, C = c field 0, Euler state q."""
        _check(lib.dg_passive_rhs(self.h, _ptr(q), _ptr(c), _ptr(dcdt), _stream(stream)))

    def passive_rk_stage(self, stage, dt, q_in, c_n, c_in, c_out, stream=None):
        """SSP-RK3 stage of the passive tracer with the Euler stage input q_in."""
        _check(lib.dg_passive_rk_stage(self.h, int(stage), float(dt), _ptr(q_in), _ptr(c_n), _ptr(c_in),
                                       _ptr(c_out), _stream(stream)))

    def amr_project_refine(self, n, parent_src, child0_dst, q_src, q_dst, stream=None):
        _check(lib.dg_amr_project_refine(self.h, int(n), _ptr(parent_src), _ptr(child0_dst), _ptr(q_src),
                                         _ptr(q_dst), _stream(stream)))

    def amr_project_coarsen(self, n, child0_src, parent_dst, q_src, q_dst, stream=None):
        _check(lib.dg_amr_project_coarsen(self.h, int(n), _ptr(child0_src), _ptr(parent_dst), _ptr(q_src),
                                          _ptr(q_dst), _stream(stream)))

    def copy_elements(self, n, src, dst, q_src, q_dst, stream=None):
        _check(lib.dg_copy_elements(self.h, int(n), _ptr(src), _ptr(dst), _ptr(q_src), _ptr(q_dst),
                                    _stream(stream)))

    def integrals(self, q, stream=None):
        out = np.zeros(self.params.dim + 2)
        _check(lib.dg_integrals(self.h, _ptr(q), out.ctypes.data, _stream(stream)))
        return out

    def check_state(self, q, stream=None):
        """(n_nonfinite, n_rho_nonpos, n_theta_nonpos, first_bad_elem or -1) of device state q."""
        out = np.zeros(4, np.int64)
        _check(lib.dg_check_state(self.h, _ptr(q), out.ctypes.data, _stream(stream)))
        return tuple(int(v) for v in out)

    def rhs_host(self, q_host, dqdt_host, stream=None):
        _check(lib.dg_rhs_host(self.h, _ptr(q_host), _ptr(dqdt_host), _stream(stream)))

    def rk3_step_host(self, dt, n_steps, q_host, stream=None):
        _check(lib.dg_rk3_step_host(self.h, float(dt), int(n_steps), _ptr(q_host), _stream(stream)))

    def launch_count(self):
        return int(lib.dg_launch_count(self.h))

    def set_nonconforming(self, mode):
        """2:1 faces: 0 mortar method (default), 1 pointwise-interpolation baseline (NEXT-3)."""
        _check(lib.dg_set_nonconforming(self.h, int(mode)))

    def set_viscosity(self, mu):
        """NEXT-3 artificial viscosity mu [m^2/s] added to every RHS evaluation (0: off)."""
        _check(lib.dg_set_viscosity(self.h, float(mu)))

    def tracer_rhs(self, s, out, stream=None):
        """Kinematic tracer: out field 0 = dC/dt of s (field 0 = C, fields 1..dim = wind)."""
        _check(lib.dg_tracer_rhs(self.h, _ptr(s), _ptr(out), _stream(stream)))

    def tracer_rk_stage(self, stage, dt, s_n, s_in, s_out, stream=None):
        _check(lib.dg_tracer_rk_stage(self.h, int(stage), float(dt), _ptr(s_n), _ptr(s_in), _ptr(s_out),
                                      _stream(stream)))

    # ---------------------------------------------------------------- NEXT-4 partition
    def mesh_build_part(self, level, anchor, n_parts, part):
        level = np.ascontiguousarray(level, np.int8)
        anchor = np.ascontiguousarray(anchor, np.int32)
        _check(lib.dg_mesh_build_part(self.h, len(level), level.ctypes.data, anchor.ctypes.data, int(n_parts),
                                      int(part)))

    def mesh_upload_part(self, level, anchor, n_parts, part, stream=None):
        level = np.ascontiguousarray(level, np.int8)
        anchor = np.ascontiguousarray(anchor, np.int32)
        _check(lib.dg_mesh_upload_part(self.h, len(level), level.ctypes.data, anchor.ctypes.data, int(n_parts),
                                       int(part), _stream(stream)))

    def part_info(self):
        np_, pt = C.c_int32(), C.c_int32()
        nl, nh, gb = C.c_int64(), C.c_int64(), C.c_int64()
        _check(lib.dg_part_info(self.h, C.byref(np_), C.byref(pt), C.byref(nl), C.byref(nh), C.byref(gb)))
        return {"n_parts": np_.value, "part": pt.value, "n_local": nl.value, "n_halo": nh.value,
                "global_begin": gb.value}

    def part_exchange_lists(self):
        """(send_count [n_parts], recv_count [n_parts], send_idx [sum send_count]) as numpy arrays."""
        n = self.part_info()["n_parts"]
        sc, rc = np.zeros(n, np.int64), np.zeros(n, np.int64)
        _check(lib.dg_part_exchange_lists(self.h, sc.ctypes.data, rc.ctypes.data, None))
        idx = np.zeros(int(sc.sum()), np.int32)
        _check(lib.dg_part_exchange_lists(self.h, sc.ctypes.data, rc.ctypes.data, idx.ctypes.data))
        return sc, rc, idx

    def part_face_lists(self):
        """(send_count, recv_count, send_pairs [n, 2], recv_pairs [n, 2]) of the face-trace exchange."""
        n = self.part_info()["n_parts"]
        sc, rc = np.zeros(n, np.int64), np.zeros(n, np.int64)
        _check(lib.dg_part_face_lists(self.h, sc.ctypes.data, rc.ctypes.data, None, None))
        sp, rp = np.zeros((int(sc.sum()), 2), np.int32), np.zeros((int(rc.sum()), 2), np.int32)
        _check(lib.dg_part_face_lists(self.h, sc.ctypes.data, rc.ctypes.data, sp.ctypes.data, rp.ctypes.data))
        return sc, rc, sp, rp

    def pack_faces(self, n, pairs, q, buf, stream=None):
        _check(lib.dg_pack_faces(self.h, int(n), _ptr(pairs), _ptr(q), _ptr(buf), _stream(stream)))

    def unpack_faces(self, n, pairs, buf, q, stream=None):
        _check(lib.dg_unpack_faces(self.h, int(n), _ptr(pairs), _ptr(buf), _ptr(q), _stream(stream)))

    # ---------------------------------------------------------------- NEXT-1 regrid
    def amr_indicator(self, kind, q, eta, stream=None):
        _check(lib.dg_amr_indicator(self.h, int(kind), _ptr(q), _ptr(eta), _stream(stream)))

    def regrid_plan(self, eta_host, refine_above, coarsen_below, buffer):
        """Host plan (dg_regrid_plan_*) as a dict of numpy arrays."""
        eta_host = np.ascontiguousarray(eta_host, np.float64)
        h = C.c_void_p()
        _check(lib.dg_regrid_plan_create(self.h, eta_host.ctypes.data, float(refine_above), float(coarsen_below),
                                         int(buffer), C.byref(h)))
        try:
            n = [C.c_int64() for _ in range(4)]
            _check(lib.dg_regrid_plan_sizes(h, *[C.byref(x) for x in n]))
            nl, nr, nc, ncp = (x.value for x in n)
            dim = self.params.dim
            out = {"level": np.zeros(nl, np.int8), "anchor": np.zeros((nl, dim), np.int32),
                   "refine_parent": np.zeros(nr, np.int32), "refine_child0": np.zeros(nr, np.int32),
                   "coarsen_child0": np.zeros(nc, np.int32), "coarsen_parent": np.zeros(nc, np.int32),
                   "copy_src": np.zeros(ncp, np.int32), "copy_dst": np.zeros(ncp, np.int32)}
            _check(lib.dg_regrid_plan_get(h, *[out[k].ctypes.data for k in
                                               ("level", "anchor", "refine_parent", "refine_child0",
                                                "coarsen_child0", "coarsen_parent", "copy_src", "copy_dst")]))
        finally:
            lib.dg_regrid_plan_destroy(h)
        return out

    def regrid(self, q, kind, refine_above, coarsen_below, buffer, stream=None):
        """One regrid through the C ABI: indicator (device) -> plan (host) ->
        mesh upload -> transfer kernels.  Returns (new state tensor, plan)."""
        import torch
        E = q.shape[0]
        eta = torch.empty(E, dtype=torch.float64, device=q.device)
        self.amr_indicator(kind, q, eta, stream)
        return self.regrid_eta(q, eta.cpu().numpy(), refine_above, coarsen_below, buffer, stream)

    def regrid_eta(self, q, eta_host, refine_above, coarsen_below, buffer, stream=None):
        """regrid() with a caller-computed indicator eta_host[E] (e.g. a tracer's max |C|)."""
        import torch
        plan = self.regrid_plan(eta_host, refine_above, coarsen_below, buffer)
        self.mesh_upload(plan["level"], plan["anchor"], stream)
        q_new = torch.empty((len(plan["level"]), q.shape[1]), dtype=torch.float64, device=q.device)
        T = lambda a: torch.from_numpy(a).to(q.device)
        if len(plan["copy_src"]):
            self.copy_elements(len(plan["copy_src"]), T(plan["copy_src"]), T(plan["copy_dst"]), q, q_new, stream)
        if len(plan["refine_parent"]):
            self.amr_project_refine(len(plan["refine_parent"]), T(plan["refine_parent"]), T(plan["refine_child0"]),
                                    q, q_new, stream)
        if len(plan["coarsen_parent"]):
            self.amr_project_coarsen(len(plan["coarsen_parent"]), T(plan["coarsen_child0"]),
                                     T(plan["coarsen_parent"]), q, q_new, stream)
        return q_new, plan


# ---------------------------------------------------------------- helpers
def to_device(q_compact, stride, device="cuda"):
    """Compact [E, F, Np] host array -> padded [E, stride] device tensor (layout of dg.h)."""
    import torch
    E = q_compact.shape[0]
    row = q_compact.shape[1] * q_compact.shape[2]
    t = torch.zeros((E, stride), dtype=torch.float64, device=device)
    t[:, :row] = torch.from_numpy(np.ascontiguousarray(q_compact).reshape(E, row)).to(device)
    return t


def from_device(t, F, Np):
    """Padded [E, stride] device tensor -> compact [E, F, Np] numpy array."""
    E = t.shape[0]
    return t[:, :F * Np].cpu().numpy().reshape(E, F, Np)
