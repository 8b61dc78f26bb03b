"""NEXT-4: halo exchange of a partitioned libdg context over torch.distributed.

One process per GPU; rank k holds part k of the SFC partition
(dg_mesh_upload_part).  Before every RHS evaluation the halo of the stage input
is refreshed from its owners with one batched send/recv per peer:

* mode "faces" (default): only the face-node values the kernels read -- for each
  (element, face) pair with a neighbour in the peer's part, F x Nf values,
  gathered by dg_pack_faces and scattered into the receiver's halo rows by
  dg_unpack_faces (Np / Nf = N + 1 times fewer bytes than whole rows per face);
* mode "rows": whole element rows (dg_copy_elements gathers them; the receive
  lands directly in the contiguous halo rows).

Overlap (rk3_step_overlap): the own elements split into interior ones (no face neighbour in
another part: they read no halo row) and boundary ones; each stage computes the interior
elements (dg_rk_stage_elems) on the caller's stream while the exchange runs on a second
stream, then the boundary elements once the halo has landed -- the same arithmetic as the
whole-part call, bit for bit.

Plumbing only: every arithmetic step runs in libdg's kernels.  With CPU tensors
(gloo) the gathers/scatters are torch indexing, so the protocol can be tested
without GPUs.
"""
from __future__ import annotations

import numpy as np


def face_nodes(dim, n1, face):
    """Volume node of each face node of local face `face` (tangential axes ascending, R28)."""
    d, side = face >> 1, (n1 - 1) if (face & 1) else 0
    t = np.arange(n1 ** (dim - 1))
    if dim == 2:
        return side + n1 * t if d == 0 else t + n1 * side
    t1, t2 = t % n1, t // n1
    if d == 0:
        return side + n1 * t1 + n1 * n1 * t2
    if d == 1:
        return t1 + n1 * side + n1 * n1 * t2
    return t1 + n1 * t2 + n1 * n1 * side


class HaloExchange:
    def __init__(self, ctx, dist, device, mode="faces"):
        import torch
        self.torch = torch
        self.ctx, self.dist, self.mode = ctx, dist, mode
        info = ctx.part_info()
        self.n_parts, self.part, self.n_local = info["n_parts"], info["part"], info["n_local"]
        _, F, Np, stride = ctx.state_layout()
        self.F, self.Np, self.stride = F, Np, stride
        p = ctx.params
        self.dim, self.n1 = p.dim, p.order + 1
        if mode == "faces":
            sc, rc, sp, rp = ctx.part_face_lists()
            Nf = Np // self.n1
            self.Nf = Nf
            self.sp = torch.from_numpy(sp).to(device)
            self.rp = torch.from_numpy(rp).to(device)
            self.sendbuf = torch.empty((len(sp), F, Nf), dtype=torch.float64, device=device)
            self.recvbuf = torch.empty((len(rp), F, Nf), dtype=torch.float64, device=device)
            if device == "cpu" or (hasattr(device, "type") and device.type == "cpu"):
                self._cpu_index(sp, "s")
                self._cpu_index(rp, "r")
            self.bytes_per_exchange = 8 * F * Nf * (len(sp) + len(rp))
        else:
            sc, rc, idx = ctx.part_exchange_lists()
            n_send = int(sc.sum())
            self.idx = torch.from_numpy(idx).to(device)
            self.dst = torch.arange(n_send, dtype=torch.int32, device=device)
            self.sendbuf = torch.empty((n_send, stride), dtype=torch.float64, device=device)
            self.bytes_per_exchange = 8 * stride * (n_send + int(rc.sum()))
        self.sc, self.rc = sc.tolist(), rc.tolist()
        self.send_off = np.concatenate([[0], np.cumsum(sc)]).tolist()
        self.recv_off = np.concatenate([[0], np.cumsum(rc)]).tolist()

    def _cpu_index(self, pairs, which):
        """Flat indices into q.view(-1) of every (pair, field, face node) for the CPU path."""
        fn = [face_nodes(self.dim, self.n1, f) for f in range(2 * self.dim)]
        idx = np.empty((len(pairs), self.F, len(fn[0])), np.int64)
        for i, (e, f) in enumerate(pairs):
            idx[i] = e * self.stride + np.arange(self.F)[:, None] * self.Np + fn[f][None, :]
        setattr(self, "flat_" + which, self.torch.from_numpy(idx.reshape(-1)))

    def exchange(self, q, stream=None):
        """Refresh the halo of q ([n_local + n_halo, stride]) from its owners.

        torch's NCCL P2P ops and work.wait() order themselves against torch's CURRENT
        stream only, so the whole exchange (pack kernel, send/recv, unpack kernel) runs
        with `stream` made current: the send cannot read sendbuf before the pack kernel
        has finished, nor the unpack kernel read recvbuf before the receive has landed."""
        if stream is not None and q.is_cuda:
            with self.torch.cuda.stream(stream):
                return self._exchange(q, None)
        return self._exchange(q, None)

    def _exchange(self, q, stream):
        if self.mode == "faces":
            if len(self.sp):
                if q.is_cuda:
                    self.ctx.pack_faces(len(self.sp), self.sp, q, self.sendbuf, stream)
                else:
                    self.sendbuf.view(-1).copy_(q.view(-1)[self.flat_s])
            send = [self.sendbuf[self.send_off[k]:self.send_off[k + 1]] for k in range(self.n_parts)]
            recv = [self.recvbuf[self.recv_off[k]:self.recv_off[k + 1]] for k in range(self.n_parts)]
        else:
            if len(self.idx):
                if q.is_cuda:
                    self.ctx.copy_elements(len(self.idx), self.idx, self.dst, q, self.sendbuf, stream)
                else:
                    self.sendbuf.copy_(q.index_select(0, self.idx.long()))
            send = [self.sendbuf[self.send_off[k]:self.send_off[k + 1]] for k in range(self.n_parts)]
            recv = [q[self.n_local + self.recv_off[k]:self.n_local + self.recv_off[k + 1]] for k in range(self.n_parts)]
        ops = []
        for k in range(self.n_parts):
            if self.sc[k]:
                ops.append(self.dist.P2POp(self.dist.isend, send[k], k))
            if self.rc[k]:
                ops.append(self.dist.P2POp(self.dist.irecv, recv[k], k))
        if ops:
            for r in self.dist.batch_isend_irecv(ops):
                r.wait()
        if self.mode == "faces" and len(self.rp):
            if q.is_cuda:
                self.ctx.unpack_faces(len(self.rp), self.rp, self.recvbuf, q, stream)
            else:
                q.view(-1)[self.flat_r] = self.recvbuf.view(-1)

    def split(self):
        """(interior, boundary): ascending local element rows of this part without / with a face
        neighbour in another part.  Face adjacency is mutual, so the boundary elements are exactly
        the elements this part sends (faces mode: the send pairs' elements; rows mode: the send
        rows)."""
        if self.mode == "faces":
            send = self.ctx.part_face_lists()[2][:, 0]
        else:
            send = self.ctx.part_exchange_lists()[2]
        bnd = np.zeros(self.n_local, bool)
        bnd[np.asarray(send, np.int64)] = True
        return (np.flatnonzero(~bnd).astype(np.int32), np.flatnonzero(bnd).astype(np.int32))

    def rk3_step_overlap(self, dt, q, a, b, stream=None):
        """One SSP-RK3 step (R17) with each stage's halo exchange overlapped with the interior
        elements: exchange on a side stream, interior stage on `stream` (or the current one),
        then the boundary stage after the exchange.  Returns the new state (buffer a)."""
        torch = self.torch
        if not hasattr(self, "_split_dev"):
            inner, bnd = self.split()
            dev = q.device
            self._split_dev = (torch.from_numpy(inner).to(dev), torch.from_numpy(bnd).to(dev))
            self._comm = torch.cuda.Stream(device=dev)
        inner, bnd = self._split_dev
        main = stream if stream is not None else torch.cuda.current_stream()
        comm = self._comm
        for s, (qin, out) in enumerate(((q, a), (a, b), (b, a))):
            ready = torch.cuda.Event()
            ready.record(main)  # qin is complete on the main stream
            comm.wait_event(ready)
            with torch.cuda.stream(comm):
                self._exchange(qin, None)
            self.ctx.rk_stage_elems(s, dt, q, qin, out, inner, main)
            landed = torch.cuda.Event()
            landed.record(comm)
            main.wait_event(landed)
            self.ctx.rk_stage_elems(s, dt, q, qin, out, bnd, main)
        return a

    def allsum(self, local):
        """Whole-mesh sum of per-rank vectors (e.g. the F integrals of dg_integrals on the local
        rows): all-gather, then every rank adds the ranks' values in rank order with Neumaier
        compensation (R20), so the result is identical on all ranks and independent of the
        reduction tree."""
        torch = self.torch
        local = np.asarray(local, dtype=np.float64)
        dev = "cuda" if torch.cuda.is_available() and self.dist.get_backend() == "nccl" else "cpu"
        t = torch.from_numpy(local.copy()).to(dev)
        parts = [torch.empty_like(t) for _ in range(self.n_parts)]
        self.dist.all_gather(parts, t)
        vals = np.stack([x.cpu().numpy() for x in parts])
        out = np.zeros(local.shape)
        comp = np.zeros(local.shape)
        for v in vals:  # Neumaier, rank order
            tot = out + v
            big = np.abs(out) >= np.abs(v)
            comp += np.where(big, (out - tot) + v, (v - tot) + out)
            out = tot
        return out + comp

    def integrals(self, q, stream=None):
        """Integrals of the whole partitioned state (dg_integrals on the local rows, then allsum)."""
        return self.allsum(self.ctx.integrals(q, stream))

    def rk3_step(self, dt, q, a, b, stream=None):
        """One SSP-RK3 step of the partitioned mesh (R17); returns the new state (a or q buffer)."""
        self.exchange(q, stream)
        self.ctx.rk_stage(0, dt, q, q, a, stream)
        self.exchange(a, stream)
        self.ctx.rk_stage(1, dt, q, a, b, stream)
        self.exchange(b, stream)
        self.ctx.rk_stage(2, dt, q, b, a, stream)
        return a
