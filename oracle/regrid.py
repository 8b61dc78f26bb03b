"""NEXT-1 oracle: refinement indicator, regrid plan and state transfer.

TEST INFRASTRUCTURE ONLY (same rule as the rest of oracle/): only tests/,
__graft_entry__.smoke() and bench.py's oracle legs may use it.  Written
directly from the paper's description and the readings of DESIGN.md, with
plain Python sets; it shares no code with libdg's planner (dg_regrid.cpp).

* indicator ("regridding ... based on potential temperature";
  R39): eta_e = max over the element's nodes of |Theta/rho - Theta_bar/rho_bar|
  (kind 0) or |rho - rho_bar| (kind 1).
* plan (§3.2.1; R37, R38): cells with
  eta > refine_above are the feature; B rounds of face-neighbour growth, each
  round along x, then y (then z), give the buffered set T (one cell,
  B = 2 -> its 5x5 block); leaves of T below max_level are split and the 2:1
  balance is restored by splitting coarser neighbours (R15); then, finest level
  first, families of old leaves whose children are all below coarsen_below and
  outside T merge into their parent unless the parent would touch a leaf two
  levels finer.  New leaves are listed in Morton order (R27).
* transfer: the conservative projections of the oracle (oracle.refine /
  oracle.coarsen, R16) and plain copies.
"""
from __future__ import annotations

import numpy as np

import oracle


def indicator(p, level, anchor, bg, q, kind=0):
    """eta [E] (kind 0: |theta'|, kind 1: |rho'|), background row per node (R3)."""
    n1 = p.order + 1
    nv = n1 ** (p.dim - 1)
    off = [0]
    for l in range(p.max_level + 1):
        off.append(off[-1] + (p.root[p.dim - 1] << l) * n1)
    k = np.arange(n1 ** p.dim) // nv
    rows = np.asarray(off)[level.astype(np.int64)][:, None] + anchor[:, p.dim - 1].astype(np.int64)[:, None] * n1 + k
    rb, tb = bg[rows, 0], bg[rows, 1]
    if kind == 0:
        v = np.abs(q[:, p.dim + 1] / q[:, 0] - tb / rb)
    else:
        v = np.abs(q[:, 0] - rb)
    return v.max(axis=1)


class _Forest:
    def __init__(self, p, level, anchor):
        self.p = p
        self.dim = p.dim
        self.leaves = set()
        for l, a in zip(level, anchor):
            self.leaves.add((int(l),) + tuple(int(x) for x in a))

    def cell_across(self, l, a, d, s):
        ext = self.p.root[d] << l
        b = list(a)
        b[d] += s
        if b[d] < 0 or b[d] >= ext:
            if not self.p.periodic[d]:
                return None
            b[d] %= ext
        return tuple(b)

    def neighbours(self, leaf, d, s):
        l, a = leaf[0], leaf[1:]
        c = self.cell_across(l, a, d, s)
        if c is None:
            return []
        if (l,) + c in self.leaves:
            return [(l,) + c]
        if l > 0 and (l - 1,) + tuple(x >> 1 for x in c) in self.leaves:
            return [(l - 1,) + tuple(x >> 1 for x in c)]
        out = []
        tang = [t for t in range(self.dim) if t != d]
        for b in range(1 << (self.dim - 1)):
            f = [2 * x for x in c]
            if s < 0:
                f[d] += 1
            for k, t in enumerate(tang):
                f[t] += (b >> k) & 1
            if (l + 1,) + tuple(f) in self.leaves:
                out.append((l + 1,) + tuple(f))
        return out

    def containing_level(self, l, c):
        for k in range(l, -1, -1):
            if (k,) + tuple(x >> (l - k) for x in c) in self.leaves:
                return k
        return -1

    def children(self, leaf):
        l, a = leaf[0], leaf[1:]
        out = []
        for b in range(1 << self.dim):
            out.append((l + 1,) + tuple(2 * a[t] + ((b >> t) & 1) for t in range(self.dim)))
        return out


def _morton(leaf, dim, max_level):
    l = leaf[0]
    fine = [x << (max_level - l) for x in leaf[1:]]
    key = 0
    for bit in range(20):
        for d in range(dim):
            key |= ((fine[d] >> bit) & 1) << (bit * dim + d)
    return key


def plan(p, level, anchor, eta, refine_above, coarsen_below, buffer):
    dim = p.dim
    F = _Forest(p, level, anchor)
    old = [(int(l),) + tuple(int(x) for x in a) for l, a in zip(level, anchor)]
    old_index = {leaf: i for i, leaf in enumerate(old)}
    # feature set and buffer (R37)
    T = {old[i] for i in range(len(old)) if eta[i] > refine_above}
    for _ in range(buffer):
        for d in range(dim):
            grown = set()
            for leaf in T:
                for s in (-1, 1):
                    grown.update(F.neighbours(leaf, d, s))
            T |= grown
    # refinement and 2:1 ripple (R15)
    refined = set()
    work = []

    def split(leaf):
        F.leaves.remove(leaf)
        refined.add(leaf)
        for c in F.children(leaf):
            F.leaves.add(c)
            work.append(c)

    for leaf in old:
        if leaf in T and leaf[0] < p.max_level:
            split(leaf)
    while work:
        leaf = work.pop()
        if leaf not in F.leaves:
            continue
        l, a = leaf[0], leaf[1:]
        for d in range(dim):
            for s in (-1, 1):
                c = F.cell_across(l, a, d, s)
                if c is None:
                    continue
                while True:
                    k = F.containing_level(l, c)
                    if k < 0 or k >= l - 1:
                        break
                    split((k,) + tuple(x >> (l - k) for x in c))
    # coarsening, finest level first (R38)
    coarsened = set()
    for l in range(p.max_level, 0, -1):
        parents = sorted({(l - 1,) + tuple(x >> 1 for x in leaf[1:]) for leaf in old if leaf[0] == l})
        for par in parents:
            kids = F.children(par)
            if not all(k in F.leaves and k in old_index and k not in T and eta[old_index[k]] < coarsen_below
                       for k in kids):
                continue
            ok = True
            for d in range(dim):
                for s in (-1, 1):
                    c = F.cell_across(l - 1, par[1:], d, s)
                    if c is None or F.containing_level(l - 1, c) >= 0:
                        continue
                    # neighbour cell subdivided: its level-l cells on the shared face must be leaves
                    tang = [t for t in range(dim) if t != d]
                    for b in range(1 << (dim - 1)):
                        f = [2 * x for x in c]
                        if s < 0:
                            f[d] += 1
                        for kk, t in enumerate(tang):
                            f[t] += (b >> kk) & 1
                        if (l,) + tuple(f) not in F.leaves:
                            ok = False
            if not ok:
                continue
            for k in kids:
                F.leaves.remove(k)
                coarsened.add(k)
            F.leaves.add(par)
    new = sorted(F.leaves, key=lambda leaf: _morton(leaf, dim, p.max_level))
    out = {"level": np.array([leaf[0] for leaf in new], np.int8),
           "anchor": np.array([leaf[1:] for leaf in new], np.int32).reshape(len(new), dim)}
    rp, rc, cc, cp, ss, sd = [], [], [], [], [], []
    for i, leaf in enumerate(new):
        if leaf in old_index:
            ss.append(old_index[leaf])
            sd.append(i)
            continue
        par = (leaf[0] - 1,) + tuple(x >> 1 for x in leaf[1:])
        if par in refined and par in old_index:
            if all((x & 1) == 0 for x in leaf[1:]):
                rp.append(old_index[par])
                rc.append(i)
            continue
        kids = F.children(leaf)
        assert all(k in coarsened for k in kids)
        idx = [old_index[k] for k in kids]
        assert idx == list(range(idx[0], idx[0] + len(idx))), "old siblings not consecutive"
        cc.append(idx[0])
        cp.append(i)
    for k, v in (("refine_parent", rp), ("refine_child0", rc), ("coarsen_child0", cc), ("coarsen_parent", cp),
                 ("copy_src", ss), ("copy_dst", sd)):
        out[k] = np.array(v, np.int32)
    return out


def transfer(p, q, pl):
    """New state [E_new, F, Np] from q [E_old, F, Np] through the plan's maps."""
    En = len(pl["level"])
    out = np.zeros((En,) + q.shape[1:])
    out[pl["copy_dst"]] = q[pl["copy_src"]]
    if len(pl["refine_parent"]):
        r = oracle.refine(p.dim, p.order, pl["refine_parent"], pl["refine_child0"], q, En)
        nch = 1 << p.dim
        for c0 in pl["refine_child0"]:
            out[c0:c0 + nch] = r[c0:c0 + nch]
    if len(pl["coarsen_parent"]):
        c = oracle.coarsen(p.dim, p.order, pl["coarsen_child0"], pl["coarsen_parent"], q, En)
        out[pl["coarsen_parent"]] = c[pl["coarsen_parent"]]
    return out
