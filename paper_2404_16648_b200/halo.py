"""NEXT-4: halo exchange of a partitioned libdg context over torch.distributed.

One process per GPU; rank k holds part k of the SFC partition
(dg_mesh_upload_part).  Before every RHS evaluation the halo rows of the stage
input are refreshed from their owners: the rows to send are gathered into one
contiguous buffer by the library's copy kernel (dg_copy_elements), then one
batched NCCL send/recv per peer moves whole element rows straight into the
receiving halo rows (contiguous per peer by construction).  Plumbing only:
every arithmetic step runs in libdg's kernels.  With CPU tensors (gloo) the
gather is a torch index_select, which lets the protocol be tested without GPUs.
"""
from __future__ import annotations

import numpy as np


class HaloExchange:
    def __init__(self, ctx, dist, device):
        import torch
        self.torch = torch
        self.ctx = ctx
        self.dist = dist
        info = ctx.part_info()
        self.n_parts, self.part, self.n_local = info["n_parts"], info["part"], info["n_local"]
        sc, rc, idx = ctx.part_exchange_lists()
        self.sc, self.rc = sc.tolist(), rc.tolist()
        self.send_off = np.concatenate([[0], np.cumsum(sc)]).tolist()
        self.recv_off = (self.n_local + np.concatenate([[0], np.cumsum(rc)])).tolist()
        _, _, _, stride = ctx.state_layout()
        n_send = int(sc.sum())
        self.idx = torch.from_numpy(idx).to(device)
        self.dst = torch.arange(n_send, dtype=torch.int32, device=device)
        self.sendbuf = torch.empty((n_send, stride), dtype=torch.float64, device=device)
        self.bytes_per_exchange = 8 * stride * (n_send + int(rc.sum()))

    def exchange(self, q, stream=None):
        """Refresh the halo rows of q ([n_local + n_halo, stride]) from their owners."""
        if len(self.idx):
            if q.is_cuda:
                self.ctx.copy_elements(len(self.idx), self.idx, self.dst, q, self.sendbuf, stream)
            else:
                self.sendbuf.copy_(q.index_select(0, self.idx.long()))
        ops = []
        for k in range(self.n_parts):
            if self.sc[k]:
                ops.append(self.dist.P2POp(self.dist.isend, self.sendbuf[self.send_off[k]:self.send_off[k + 1]], k))
            if self.rc[k]:
                ops.append(self.dist.P2POp(self.dist.irecv, q[self.recv_off[k]:self.recv_off[k + 1]], k))
        if ops:
            for r in self.dist.batch_isend_irecv(ops):
                r.wait()

    def rk3_step(self, dt, q, a, b, stream=None):
        """One SSP-RK3 step of the partitioned mesh (R17); returns the new state (a or q buffer)."""
        self.exchange(q, stream)
        self.ctx.rk_stage(0, dt, q, q, a, stream)
        self.exchange(a, stream)
        self.ctx.rk_stage(1, dt, q, a, b, stream)
        self.exchange(b, stream)
        self.ctx.rk_stage(2, dt, q, b, a, stream)
        return a
