#!/usr/bin/env python
"""bench.py -- fp64 dGSEM RHS / SSP-RK3 throughput of libdg on B200.

Workload (N=1): BASELINE.json configs[4] ("c5"): 3D 64x64x32 hexahedra over
10 x 10 x 5 km, LGL order N=7 (512 nodes/element), 5 fields, fp64, periodic
x/y and walls z, hydrostatic background + 20 Gaussian theta bumps (readings
R26/R27 of DESIGN.md).  One "step" = one full SSP-RK3 step = three fused
dg_rk_stage launches (A1-A9 of SURVEY 8(a)).  The c5 mesh is uniform, so the
step exercises no mortar; the secondary object "c4" times BASELINE configs[3]
(oct-tree with 2:1 faces, mortars A7) for one RK3 step and one full
refine->coarsen projection pass (A10/A11); "vortex" is the paper's isentropic
vortex run (NEXT-2) with its error against the closed form.

value = DOF-updates/s summed over ranks, where one DOF-update is one
(node, field) value through one RK stage (reading R18); each state array is
2.68 GB, far larger than the 126 MB L2, so no L2 flush is needed.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--impl reference times the CPU oracle (oracle/, plain fp64 C++, 1 thread) on a
bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "fp64 DG RHS DOF-updates/s per B200 and % of HBM roofline (ncu)"
UNIT = "DOF-updates/s"
SAMPLE_ROOT_REF = (16, 16, 8)      # reference arm: 2048 elements of the c5 element type (all host cores)
SAMPLE_ROOT_CPU = (16, 16, 8)      # cpu_baseline: 2048 elements


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def fp64_row(stage_ms, rhs_ms):
    """FP64 roofline of k_stage_h7: flops per launch counted by ncu (DFMA = 2, DADD/DMUL = 1 per
    thread op, DMMA m8n8k4 = 512 per warp op; profiles/ncu_fp64.json) over the launch times measured
    here, against the measured FP64 peak (DFMA 36.65 / DMMA 37.14 TF/s; they share one datapath,
    profiles/r02_fp64_peaks.json)."""
    path = os.path.join(ROOT, "profiles", "ncu_fp64.json")
    peaks = os.path.join(ROOT, "profiles", "r02_fp64_peaks.json")
    if not (os.path.exists(path) and os.path.exists(peaks)):
        return None
    with open(path) as f:
        d = json.load(f)
    with open(peaks) as f:
        pk = json.load(f)
    peak = float(pk["dmma_tflops"])
    fl = d["flops_per_launch"]
    t = {"stage0": float(np.mean(stage_ms[:, 0])), "stage12": float(np.mean(stage_ms[:, 1:])), "rhs": rhs_ms}
    out = {"unit": "TFLOP/s", "peak": peak, "peak_source": "measured: scripts/fp64_mix.cu, scripts/dmma_peak.cu "
           "(DMMA and DFMA share the FP64 datapath: a mixed kernel takes the sum of the times)",
           "flops_source": d.get("source"), "pipe_util_ncu": d.get("pipe_util")}
    for k, ms in t.items():
        if k in fl:
            a = fl[k] / (ms * 1e-3) / 1e12
            out[k] = {"achieved": a, "frac": a / peak, "flops_per_launch": fl[k]}
    return out


def load_traffic(kernel_key):
    """dram bytes per launch from the committed ncu --set full summary, if any."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        d = json.load(f)
    v = d.get(kernel_key)
    return None if v is None else float(v)


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region (rank 0)."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,utilization.gpu")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], None, set()
        for r in self.rows:
            try:
                s, m, util = float(r[0]), float(r[1]), float(r[6])
            except ValueError:
                continue
            smax = m
            if util > 0:
                sm.append(s)
            for name, v in zip(self.NAMES, r[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- multi-rank aggregation
def reduce_max(x, dist=None, device="cpu"):
    """Max over ranks of a host float (device time of the timed region); identity at N=1."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    import torch
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def whole_job_rate(units_per_rank, seconds_max, world):
    """Whole-job throughput of `world` replicas (weak scaling): all units over the slowest rank's time."""
    return world * float(units_per_rank) / float(seconds_max)


# ----------------------------------------------------------------------------- oracle (CPU) legs
def oracle_steps(root, steps, warmup=0, budget_s=None):
    """Plain CPU oracle SSP-RK3 steps on a c5-type sample; returns (dof_updates_per_s, seconds, steps, E)."""
    import oracle
    import workloads as W
    w = W.c5(root=root)
    m = oracle.Mesh(w.params, w.level, w.anchor)
    q = w.q0
    for _ in range(warmup):
        q = oracle.rk3_step(m, w.bg, w.dt, q)
    t0 = time.perf_counter()
    done = 0
    while True:
        q = oracle.rk3_step(m, w.bg, w.dt, q)
        done += 1
        el = time.perf_counter() - t0
        if budget_s is None and done >= steps:
            break
        if budget_s is not None and (el >= budget_s or done >= steps):
            break
    return 3.0 * w.n_dof * done / el, el, done, w.n_elem


# all-core oracle: fork one worker per host core; each computes the RHS (ora_rhs with an element
# mask) of its static element chunk into a shared buffer -- every element's RHS is the same
# arithmetic as in the 1-thread call, so the result is bitwise identical at any core count -- and
# the parent applies the SSP-RK3 stage formula (R17) elementwise with numpy in the oracle's
# operation order (the oracle is built -ffp-contract=off: no FMA), also bitwise identical.
_PAR = {}


def _par_init(shape, qbuf, lbuf, masks, mesh_args, bg):
    import oracle
    _PAR["q"] = np.frombuffer(qbuf, dtype=np.float64).reshape(shape)
    _PAR["L"] = np.frombuffer(lbuf, dtype=np.float64).reshape(shape)
    _PAR["masks"] = masks
    _PAR["mesh"] = oracle.Mesh(*mesh_args)
    _PAR["bg"] = bg


def _par_rhs(i):
    import ctypes as C
    import oracle
    m = _PAR["mesh"]
    oracle.lib().ora_rhs(C.byref(m.op), m.h, oracle._dp(_PAR["bg"]), oracle._dp(_PAR["q"]), oracle._dp(_PAR["L"]),
                         _PAR["masks"][i].ctypes.data)
    return i


class OracleAllCores:
    """SSP-RK3 steps of the CPU oracle on every host core (fork pool, static element chunks)."""

    def __init__(self, w, workers):
        import multiprocessing as mp
        self.w, self.workers = w, workers
        shape = w.q0.shape
        self.qbuf = mp.RawArray("d", int(np.prod(shape)))
        self.lbuf = mp.RawArray("d", int(np.prod(shape)))
        self.q = np.frombuffer(self.qbuf, dtype=np.float64).reshape(shape)
        self.L = np.frombuffer(self.lbuf, dtype=np.float64).reshape(shape)
        masks = []
        for ch in np.array_split(np.arange(w.n_elem), workers):
            mk = np.zeros(w.n_elem, np.uint8)
            mk[ch] = 1
            masks.append(mk)
        ctx = mp.get_context("fork")
        self.pool = ctx.Pool(workers, initializer=_par_init,
                             initargs=(shape, self.qbuf, self.lbuf, masks, (w.params, w.level, w.anchor),
                                       np.ascontiguousarray(w.bg, np.float64)))

    def rhs(self, q):
        self.q[...] = q
        self.pool.map(_par_rhs, range(self.workers))
        return self.L.copy()

    def step(self, q):
        dt = self.w.dt
        q1 = q + dt * self.rhs(q)
        q2 = q + 0.25 * ((q1 - q) + dt * self.rhs(q1))
        return q + (2.0 / 3.0) * ((q2 - q) + dt * self.rhs(q2))

    def close(self):
        self.pool.close()
        self.pool.join()


def host_cpu():
    """(cores, model name) of this host."""
    n = os.cpu_count() or 1
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return n, model


def oracle_steps_all_cores(root, steps, budget_s, workers):
    import workloads as W
    w = W.c5(root=root)
    par = OracleAllCores(w, workers)
    q = w.q0
    try:
        t0 = time.perf_counter()
        done = 0
        while True:
            q = par.step(q)
            done += 1
            el = time.perf_counter() - t0
            if el >= budget_s or done >= steps:
                break
    finally:
        par.close()
    return 3.0 * w.n_dof * done / el, el, done, w.n_elem, q


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    steps = args.steps
    cores, model = host_cpu()
    v, el, done, E, _ = oracle_steps_all_cores(SAMPLE_ROOT_REF, steps, budget_s=1e9, workers=cores)
    sample = (f"c5 element type (N=7, h=156.25 m, same state recipe) on a {SAMPLE_ROOT_REF[0]}x{SAMPLE_ROOT_REF[1]}x"
              f"{SAMPLE_ROOT_REF[2]} periodic box ({E} elements), {done} SSP-RK3 steps on all {cores} host cores "
              f"({model}; fork pool, static element chunks, bitwise identical to 1 thread)")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": done, "warmup": args.warmup, "ms_per_step": 1e3 * el / done, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "c5 (BASELINE configs[4]) sample", "order": 7, "elements": E},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- GPU leg
def run_ours(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2404_16648_b200 import dg as D
    import workloads as W

    w = W.c5()
    p = w.params
    ctx = D.DG(p)
    ctx.mesh_upload(w.level, w.anchor)
    E, F, Np, stride = ctx.state_layout()
    bg = torch.from_numpy(w.bg).cuda()
    ctx.set_background(bg)
    qn = D.to_device(w.q0, stride)
    qa = torch.empty_like(qn)
    qb = torch.empty_like(qn)
    dof = E * F * Np
    stream = torch.cuda.current_stream()

    bufs = [qn, qa, qb]

    def step(ev=None):
        n, a, b = bufs
        if ev is not None:
            ev[0].record(stream)
        ctx.rk_stage(0, w.dt, n, n, a, stream)
        if ev is not None:
            ev[1].record(stream)
        ctx.rk_stage(1, w.dt, n, a, b, stream)
        if ev is not None:
            ev[2].record(stream)
        ctx.rk_stage(2, w.dt, n, b, a, stream)
        if ev is not None:
            ev[3].record(stream)
        bufs[0], bufs[1] = a, n

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
        time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = ctx.launch_count()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for k in range(args.steps):
        step(evs[k])
    t1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = ctx.launch_count() - launches0
    clocks = sampler.stop() if sampler else None
    ms = t0.elapsed_time(t1)
    st = np.array([[e[i].elapsed_time(e[i + 1]) for i in range(3)] for e in evs])  # ms per stage launch
    ms = reduce_max(ms, dist if world > 1 else None, "cuda")
    ms_per_step = ms / args.steps
    value = whole_job_rate(3.0 * dof * args.steps, ms * 1e-3, world)

    # roofline of the dominant kernel (k_stage<3,7>): algorithmic bytes per launch
    # = 16 (stage 0) / 24 / 24 B per DOF, over its mean launch time
    peak, peak_src = load_peaks()
    bytes_step = 64.0 * dof
    kern_ms = st.sum(axis=1).mean()
    achieved = bytes_step / (kern_ms * 1e-3) / 1e9
    per_stage = {f"stage{i}": {"ms": float(st[:, i].mean()),
                               "GB_per_s": (16.0 if i == 0 else 24.0) * dof / (st[:, i].mean() * 1e-3) / 1e9}
                 for i in range(3)}
    traffic = load_traffic("k_stage_3_7")

    # the RHS alone (dg_rhs, 16 B/DOF: read q, write dq/dt) on the bench workload
    rhs_ms = []
    for _ in range(3):
        ctx.rhs(bufs[0], bufs[1], stream)
    for _ in range(10):
        h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h0.record(stream)
        ctx.rhs(bufs[0], bufs[1], stream)
        h1.record(stream)
        torch.cuda.synchronize()
        rhs_ms.append(h0.elapsed_time(h1))
    rhs_ms = float(np.median(rhs_ms))
    rhs_row = {"kernel": "k_stage_h7<0> (dg_rhs)", "ms": rhs_ms, "dof_updates_per_s": dof / (rhs_ms * 1e-3),
               "GB_per_s": 16.0 * dof / (rhs_ms * 1e-3) / 1e9, "frac": 16.0 * dof / (rhs_ms * 1e-3) / 1e9 / peak,
               "note": "median of 10 dg_rhs launches, CUDA events; 16 B/DOF algorithmic"}
    fp64 = fp64_row(st, rhs_ms)

    # e2e through the C ABI with host buffers: h2d + 1 RK3 step + d2h per call
    e2e = None
    if rank == 0 or world > 1:
        qh = torch.from_numpy(np.ascontiguousarray(w.q0)).pin_memory()
        ctx.rk3_step_host(w.dt, 1, qh, stream)  # warm (scratch alloc)
        n_e2e = max(2, min(5, args.steps))
        if world > 1:
            dist.barrier()
        s0 = time.perf_counter()
        for _ in range(n_e2e):
            ctx.rk3_step_host(w.dt, 1, qh, stream)
        e2e_s = reduce_max(time.perf_counter() - s0, dist if world > 1 else None, "cuda")
        nb = int(qh.numel() * 8)
        e2e = {"value": whole_job_rate(3.0 * dof * n_e2e, e2e_s, world), "unit": UNIT, "h2d_bytes_per_step": nb,
               "d2h_bytes_per_step": nb, "steps": n_e2e,
               "note": "dg_rk3_step_host: pinned host [E][F][Np] -> device, 3 fused stages, device -> host, sync"}
        del qh

    # dg_check_state (SURVEY 5 monitor, not part of the step): one read of the c5 state, 8 B/DOF
    health = None
    if rank == 0:
        res = ctx.check_state(bufs[0], stream)
        hs = []
        for _ in range(10):
            h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            h0.record(stream)
            ctx.check_state(bufs[0], stream)
            h1.record(stream)
            torch.cuda.synchronize()
            hs.append(h0.elapsed_time(h1))
        hms = float(np.median(hs))
        health = {"kernel": "k_check_state", "ms": hms, "GB_per_s": 8.0 * dof / (hms * 1e-3) / 1e9,
                  "frac": 8.0 * dof / (hms * 1e-3) / 1e9 / peak, "result": list(res),
                  "note": "median of 10 calls incl. counter reset and 32-B readback; state healthy after the run"}

    secondary = c4_leg(torch, D, W, stream) if (rank == 0 and not args.skip_c4) else None
    n4u = n4_uniform_leg(torch, D, W) if (rank == 0 and not args.skip_c4) else None
    per_config = (configs_leg(torch, D, W, stream, host_cpu()[0])
                  if (rank == 0 and world == 1 and not args.skip_configs) else None)
    vort = vortex_leg(torch, D, W) if (rank == 0 and not args.skip_vortex) else None

    cpu = None
    if rank == 0 and world == 1 and not args.skip_cpu:
        cores, model = host_cpu()
        v1, el1, done1, Es = oracle_steps(SAMPLE_ROOT_CPU, steps=100, budget_s=10.0)
        va, ela, donea, _, _ = oracle_steps_all_cores(SAMPLE_ROOT_CPU, steps=100, budget_s=10.0, workers=cores)
        sample = (f"c5 element type (N=7, h=156.25 m, same state recipe) on a {SAMPLE_ROOT_CPU[0]}x{SAMPLE_ROOT_CPU[1]}x"
                  f"{SAMPLE_ROOT_CPU[2]} periodic box ({Es} elements)")
        cpu = {"value": va, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu_model": model,
               "sample": f"{sample}: {donea} SSP-RK3 steps in {ela:.1f} s on all {cores} host cores (fork pool, "
                         f"static element chunks, bitwise identical to 1 thread); g++ -O2 -ffp-contract=off",
               "one_thread": {"value": v1, "unit": UNIT, "cores": 1,
                              "sample": f"{sample}: {done1} SSP-RK3 steps in {el1:.1f} s, 1 thread"}}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": "c5 (BASELINE configs[4]): 3D 64x64x32 hex, N=7, 5 fields, fp64, "
                                       "periodic x,y, walls z, 20 Gaussian theta bumps; step = 1 SSP-RK3 step "
                                       "(3 fused dg_rk_stage launches)",
                           "elements": E, "order": 7, "dof": dof, "bytes_per_array": E * stride * 8,
                           "l2": "inputs larger than L2 (2.68 GB per state array vs 126 MB L2); no flush",
                           "parallelism": f"replicas x{world}" if world > 1 else "1 GPU"},
                "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                             "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                             "kernel": "k_stage_h7 (3D N=7 fused RHS + SSP-RK3 stage)",
                             "algorithmic_bytes": "16/24/24 B per DOF for stages 0/1/2 (64 B/DOF per step)",
                             "per_stage": per_stage, "rhs": rhs_row},
                "fp64": fp64,
                "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches), "clocks": clocks}
        if health:
            line["check_state"] = health
        if secondary:
            line["c4"] = secondary
        if n4u:
            line["c5n4"] = n4u
        if per_config:
            line["configs"] = per_config
        if vort:
            line["vortex"] = vort
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def c4_leg(torch, D, W, stream, reps=20):
    """BASELINE configs[3]: RK3 step and refine->coarsen projection pass timings."""
    stream = torch.cuda.Stream()  # graph capture needs a non-default stream
    w = W.c4()
    p = w.params
    ctx = D.DG(p)
    ctx.mesh_upload(w.level, w.anchor)
    E, F, Np, stride = ctx.state_layout()
    nc, nn, nb = ctx.mesh_face_counts()
    bg = torch.from_numpy(w.bg).cuda()
    ctx.set_background(bg)
    dof = E * F * Np
    qn = D.to_device(w.q0, stride)
    qa, qb = torch.empty_like(qn), torch.empty_like(qn)
    ev = lambda: torch.cuda.Event(enable_timing=True)

    def timeit(fn, n=reps):
        # n launches captured in a CUDA graph and replayed: device time per launch, without the
        # Python/ctypes launch overhead (which exceeds the ~30 us transfer kernels' run time)
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for _ in range(n):
                fn()
        g.replay()
        torch.cuda.synchronize()
        a, b = ev(), ev()
        with torch.cuda.stream(stream):
            a.record()
            g.replay()
            b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / n

    rhs_ms = timeit(lambda: ctx.rhs(qn, qa, stream))

    def rk3():
        ctx.rk_stage(0, w.dt, qn, qn, qa, stream)
        ctx.rk_stage(1, w.dt, qn, qa, qb, stream)
        ctx.rk_stage(2, w.dt, qn, qb, qa, stream)
    step_ms = timeit(rk3)

    # projection pass (reading R25): flagged leaves -> 2^3 children, then back
    flags = W.c4_projection_flags(w)
    nch = 8
    isf = np.zeros(E, bool)
    isf[flags] = True
    size = np.where(isf, nch, 1)
    start = np.concatenate([[0], np.cumsum(size)[:-1]]).astype(np.int32)
    E2 = int(size.sum())
    keep = np.nonzero(~isf)[0].astype(np.int32)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.int32)).cuda()
    par, ch0, kp, kd = T(flags), T(start[flags]), T(keep), T(start[keep])
    fine = torch.empty((E2, stride), dtype=torch.float64, device="cuda")
    back = torch.empty_like(qn)

    def proj():
        ctx.amr_project_refine(len(flags), par, ch0, qn, fine, stream)
        ctx.copy_elements(len(keep), kp, kd, qn, fine, stream)
        ctx.amr_project_coarsen(len(flags), ch0, par, fine, back, stream)
        ctx.copy_elements(len(keep), kd, kp, fine, back, stream)
    proj_ms = timeit(proj)
    parts = {"refine": lambda: ctx.amr_project_refine(len(flags), par, ch0, qn, fine, stream),
             "copy": lambda: ctx.copy_elements(len(keep), kp, kd, qn, fine, stream),
             "coarsen": lambda: ctx.amr_project_coarsen(len(flags), ch0, par, fine, back, stream)}
    part_ms = {k: timeit(f) for k, f in parts.items()}
    peak, _ = load_peaks()
    rhs_gbs = 16.0 * dof / (rhs_ms * 1e-3) / 1e9
    step_gbs = 64.0 * dof / (step_ms * 1e-3) / 1e9
    # projection algorithmic bytes: refine reads parent + writes 8 children; copy r+w; coarsen reads 8 children + writes parent
    row = F * Np * 8
    nf, nk = len(flags), len(keep)
    proj_bytes = nf * row * (1 + 8) * 2 + nk * row * 2 * 2
    # per-kernel fractions: refine reads 1 and writes 8 rows per family, coarsen reads 8 and writes 1,
    # copy reads and writes 1 row per unflagged leaf
    part_bytes = {"refine": nf * row * 9, "coarsen": nf * row * 9, "copy": nk * row * 2}
    part_frac = {k: part_bytes[k] / (part_ms[k] * 1e-3) / 1e9 / peak for k in part_ms}
    out = {"workload": "c4 (BASELINE configs[3]): 3D oct-tree 32x32x16 + 10%/2% refinement, N=4",
           "elements": E, "dof": dof, "faces": {"conforming": nc, "nonconforming": nn, "boundary": nb},
           "rhs_ms": rhs_ms, "rhs_dof_updates_per_s": dof / (rhs_ms * 1e-3), "rhs_GB_per_s": rhs_gbs,
           "rhs_frac": rhs_gbs / peak,
           "rk3_step_ms": step_ms, "rk3_dof_updates_per_s": 3.0 * dof / (step_ms * 1e-3), "rk3_GB_per_s": step_gbs,
           "rk3_frac": step_gbs / peak,
           "projection_pass_ms": proj_ms, "projection_parts_ms": part_ms, "projection_parts_frac": part_frac,
           "projection_flagged": nf,
           "projection_GB_per_s":
               proj_bytes / (proj_ms * 1e-3) / 1e9, "projection_frac": proj_bytes / (proj_ms * 1e-3) / 1e9 / peak}
    ctx.close()
    return out


def n4_uniform_leg(torch, D, W, reps=10):
    """3D N = 4 on c5's uniform mesh (64 x 64 x 32 elements, 82 M DOF; the north star's "3D N=4"
    target on a conforming mesh, run by k_stage_h4): dg_rhs and one SSP-RK3 step, CUDA events over
    back-to-back launches, algorithmic 16 / 64 B per DOF against the measured HBM peak."""
    w = W.get("c5n4")
    ctx = D.DG(w.params)
    ctx.mesh_upload(w.level, w.anchor)
    E, F, Np, stride = ctx.state_layout()
    ctx.set_background(torch.from_numpy(w.bg).cuda())
    dof = E * F * Np
    qn = D.to_device(w.q0, stride)
    qa, qb = torch.empty_like(qn), torch.empty_like(qn)
    s = torch.cuda.Stream()

    def timeit(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(reps):
            fn()
        b.record(s)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    rhs_ms = timeit(lambda: ctx.rhs(qn, qa, s))

    def rk3():
        ctx.rk_stage(0, w.dt, qn, qn, qa, s)
        ctx.rk_stage(1, w.dt, qn, qa, qb, s)
        ctx.rk_stage(2, w.dt, qn, qb, qa, s)
    step_ms = timeit(rk3)
    peak, _ = load_peaks()
    ctx.close()
    return {"workload": "c5n4: c5's uniform 64x64x32 mesh at N=4 (k_stage_h4)", "elements": E, "dof": dof,
            "rhs_ms": rhs_ms, "rhs_frac": 16.0 * dof / (rhs_ms * 1e-3) / 1e9 / peak,
            "rk3_step_ms": step_ms, "rk3_frac": 64.0 * dof / (step_ms * 1e-3) / 1e9 / peak,
            "rk3_dof_updates_per_s": 3.0 * dof / (step_ms * 1e-3)}


def configs_leg(torch, D, W, stream, cores):
    """SURVEY 8(d) D.4-D.6 per configuration: GPU RHS and SSP-RK3 step times (c1-c3 replayed from a
    CUDA graph: latency-bound sizes; c4 back-to-back launches), DOF-updates/s, and the oracle timed
    beside them (1 thread and all host cores, bitwise identical) for RHS, step and (c4) the
    refine -> coarsen projection pass.  c5's oracle numbers are the cpu_baseline sample."""
    import oracle
    out = {}
    for name in ("c1", "c2", "c3", "c4"):
        w = W.get(name)
        ctx = D.DG(w.params)
        ctx.mesh_upload(w.level, w.anchor)
        E, F, Np, stride = ctx.state_layout()
        ctx.set_background(torch.from_numpy(w.bg).cuda())
        dof = E * F * Np
        qn = D.to_device(w.q0, stride)
        qa, qb = torch.empty_like(qn), torch.empty_like(qn)
        s = torch.cuda.Stream()
        reps = 200 if name != "c4" else 20

        def timed(fn):
            if name == "c4":
                for _ in range(3):
                    fn(s)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                a.record(s)
                for _ in range(reps):
                    fn(s)
                b.record(s)
                torch.cuda.synchronize()
                return a.elapsed_time(b) * 1e3 / reps
            g = torch.cuda.CUDAGraph()
            fn(s)
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s):
                for _ in range(reps):
                    fn(s)
            g.replay()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                a.record()
                g.replay()
                b.record()
            torch.cuda.synchronize()
            return a.elapsed_time(b) * 1e3 / reps

        def rk3(st):
            ctx.rk_stage(0, w.dt, qn, qn, qa, st)
            ctx.rk_stage(1, w.dt, qn, qa, qb, st)
            ctx.rk_stage(2, w.dt, qn, qb, qa, st)
        rhs_us = timed(lambda st: ctx.rhs(qn, qa, st))
        step_us = timed(rk3)
        m = oracle.Mesh(w.params, w.level, w.anchor)
        t0 = time.perf_counter()
        oracle.rhs(m, w.bg, w.q0)
        o_rhs = time.perf_counter() - t0
        par = OracleAllCores(w, cores)
        try:
            par.rhs(w.q0)
            t0 = time.perf_counter()
            par.rhs(w.q0)
            o_rhs_all = time.perf_counter() - t0
            t0 = time.perf_counter()
            par.step(w.q0)
            o_step_all = time.perf_counter() - t0
        finally:
            par.close()
        row = {"elements": E, "dof": dof, "gpu_rhs_us": rhs_us, "gpu_step_us": step_us,
               "gpu_rhs_dof_updates_per_s": dof / (rhs_us * 1e-6),
               "gpu_step_dof_updates_per_s": 3 * dof / (step_us * 1e-6),
               "timing": "CUDA-graph replay of %d launches" % reps if name != "c4" else "%d back-to-back launches" % reps,
               "oracle_rhs_s_1thread": o_rhs, "oracle_rhs_s_all_cores": o_rhs_all,
               "oracle_step_s_all_cores": o_step_all, "oracle_cores": cores}
        if name != "c4":
            t0 = time.perf_counter()
            oracle.rk3_step(m, w.bg, w.dt, w.q0)
            row["oracle_step_s_1thread"] = time.perf_counter() - t0
        else:
            flags = W.c4_projection_flags(w).astype(np.int32)
            sub = flags[:256]
            ch0 = (8 * np.arange(len(sub))).astype(np.int32)
            t0 = time.perf_counter()
            fine = oracle.refine(3, w.params.order, sub, ch0, w.q0, 8 * len(sub))
            oracle.coarsen(3, w.params.order, ch0, sub, fine, E)
            per = (time.perf_counter() - t0) / len(sub)
            row["oracle_projection_s_1thread"] = per * len(flags)
            row["oracle_projection_note"] = (f"refine + coarsen (Kronecker loops) timed on 256 of the {len(flags)} "
                                             f"flagged families (R25), scaled to all of them; the copy of unflagged "
                                             f"leaves is not oracle arithmetic")
        out[name] = row
        ctx.close()
    return out


def vortex_leg(torch, D, W, k=200):
    """NEXT-2: the paper's isentropic-vortex run --
    32 x 32, N = 3, forward Euler (SSP-RK3 stage 0) with dt = 2.5e-4 s to t = 3 s --
    replayed from a CUDA graph of k launches; error vs the closed form (R36)."""
    w = W.vortex()
    ctx = D.DG(w.params)
    ctx.mesh_upload(w.level, w.anchor)
    E, F, Np, stride = ctx.state_layout()
    ctx.set_background(torch.from_numpy(w.bg).cuda())
    dt, n = w.dt, 12000
    q0 = D.to_device(w.q0, stride)
    q, a = q0.clone(), torch.empty_like(q0)
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        for i in range(k):
            src, dst = (q, a) if i % 2 == 0 else (a, q)
            ctx.rk_stage(0, dt, src, src, dst, s)
    q.copy_(q0)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        ev0.record()
        for _ in range(n // k):
            g.replay()
        ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    qh = D.from_device(q, F, Np)
    err = W.vortex_l2(w.params, qh, W.vortex_state(w.params, w.level, w.anchor, n * dt), w.level)
    ctx.close()
    sys.path.insert(0, os.path.join(ROOT, "scripts"))
    from vortex_amr import run as run_amr  # NEXT-1 regrid loop on the same problem
    amr = run_amr(every=400, refine=0.01, coarsen=0.005, buffer=2)
    return {"workload": "isentropic vortex (P:350-384): [-6,6]^2 periodic, 32x32, N=3, forward Euler, "
                        "dt=2.5e-4 s, 12000 steps to t=3 s, CUDA-graph replay",
            "dof": E * F * Np, "ms_total": ms, "us_per_step": ms * 1e3 / n,
            "l2_rms": err["rms"], "l2_quad": err["l2"], "l2_max": err["max"], "paper_l2": 8.75e-4,
            "note": "paper's value is for its tree-based AMR run; norm read as RMS over nodes x fields (R36)",
            "amr": {k: amr[k] for k in ("workload", "l2_rms", "l2_quad", "elements_min", "elements_max", "regrids",
                                        "regrid_ms_mean", "us_per_step")}}


def run_partitioned(args):
    """NEXT-4 (opt-in, --partition): c5 split over the ranks by the SFC partition
    (dg_mesh_upload_part), halo rows exchanged over NCCL before every stage
    (paper_2404_16648_b200.halo), strong scaling (fixed total c5).  Same timing
    rules as the default path: barrier + synchronize around K timed steps,
    device time, max over ranks."""
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2404_16648_b200 import dg as D
    from paper_2404_16648_b200.halo import HaloExchange
    import workloads as W

    w = W.c5()
    p = w.params
    ctx = D.DG(p)
    ctx.mesh_upload_part(w.level, w.anchor, world, rank)
    info = ctx.part_info()
    rows, F, Np, stride = ctx.state_layout()
    ctx.set_background(torch.from_numpy(w.bg).cuda())
    b, nl = info["global_begin"], info["n_local"]
    q = torch.zeros((rows, stride), dtype=torch.float64, device="cuda")
    q[:nl, :F * Np] = torch.from_numpy(np.ascontiguousarray(w.q0[b:b + nl]).reshape(nl, F * Np)).cuda()
    del w
    a, bb = torch.empty_like(q), torch.empty_like(q)
    hx = HaloExchange(ctx, dist, "cuda") if world > 1 else None
    stream = torch.cuda.current_stream()
    dt = 0.005
    bufs = [q, a, bb]

    def step():
        n, x, y = bufs
        if hx and args.overlap:  # interior elements while the halo is in flight (HaloExchange.rk3_step_overlap)
            hx.rk3_step_overlap(dt, n, x, y, stream)
            bufs[0], bufs[1] = x, n
            return
        if hx:
            hx.exchange(n)
        ctx.rk_stage(0, dt, n, n, x, stream)
        if hx:
            hx.exchange(x)
        ctx.rk_stage(1, dt, n, x, y, stream)
        if hx:
            hx.exchange(y)
        ctx.rk_stage(2, dt, n, y, x, stream)
        bufs[0], bufs[1] = x, n

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = ctx.launch_count()
    t0.record(stream)
    for _ in range(args.steps):
        step()
    t1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = ctx.launch_count() - launches0
    ms = reduce_max(t0.elapsed_time(t1), dist if world > 1 else None, "cuda")
    dof_local = nl * F * Np
    dof = dof_local
    if world > 1:
        t = torch.tensor([float(dof_local)], dtype=torch.float64, device="cuda")
        dist.all_reduce(t)
        dof = int(t.item())
    value = 3.0 * dof * args.steps / (ms * 1e-3)
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": "c5 (BASELINE configs[4]) partitioned over the ranks (SFC ranges + halo "
                                       "exchange per stage, NEXT-4)", "dof": dof, "parallelism": f"sfc{world}",
                           "overlap": bool(args.overlap and hx),
                           "halo_bytes_per_exchange_rank0": hx.bytes_per_exchange if hx else 0},
                "e2e": None, "gpu_launches": int(launches), "roofline": None, "cpu_baseline": None}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--skip-cpu", action="store_true", help="omit the cpu_baseline leg")
    ap.add_argument("--skip-c4", action="store_true", help="omit the secondary c4 leg")
    ap.add_argument("--skip-vortex", action="store_true", help="omit the NEXT-2 isentropic-vortex leg")
    ap.add_argument("--skip-configs", action="store_true", help="omit the per-config (c1-c4) GPU/oracle table")
    ap.add_argument("--overlap", action="store_true",
                    help="with --partition: overlap each stage's halo exchange with the interior elements")
    ap.add_argument("--partition", action="store_true",
                    help="NEXT-4: c5 partitioned over the ranks with halo exchange (strong scaling)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    if args.partition:
        return run_partitioned(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
