"""Recognise dense contractions in lifted regions and map them to kernels.

The reference's matmul nests (reference tests/kernels.py:24-38, PAPER.md
143-191) and the contraction nest of the Linear lowering (PAPER.md 443-454)
all have the shape

    for <vars in any order>:            # static bounds
        a = A[fA(m, k)]; b = B[fB(k, n)]; c = C[fC(m, n)]
        C[fC(m, n)] = c + a * b         # f32, each op rounded

with affine index maps.  Every variable plays exactly one role: M (in C and
A), N (in C and B) or K (in A and B only — the reduction, executed in
ascending order per output), or is a trip-1 variable.  Such a region is a
GEMM ``C[m,n] = C[m,n] + sum_k A[m,k] B[k,n]`` over element strides read
off the affine maps, whatever the loop order or parallel/for mix.
"""
from __future__ import annotations

from .analysis import _mixed_radix_injective
from .lift import BINF, LOAD, STORE, PURE_OPS, Aff, Ins


class GemmMatch:
    __slots__ = ("A", "B", "C", "offA", "offB", "offC", "sA", "sB", "sC", "M", "N", "K")

    def __repr__(self):
        return (f"GemmMatch(M={self.M}, N={self.N}, K={self.K}, sA={self.sA}, "
                f"sB={self.sB}, sC={self.sC})")


def _straight_line(nodes):
    return all(isinstance(n, Ins) for n in nodes)


def match_gemm(region, links, remainder, accesses):
    """Return a GemmMatch for a fp32 C += A*B nest, else None."""
    if not links or not _straight_line(remainder):
        return None
    body = [n for n in remainder if n.op not in PURE_OPS or n.op == BINF]
    loads = [n for n in body if n.op == LOAD]
    binf = [n for n in body if n.op == BINF]
    stores = [n for n in body if n.op == STORE]
    if len(loads) != 3 or len(binf) != 2 or len(stores) != 1 or len(body) != 6:
        return None
    st = stores[0]
    add = next((n for n in binf if n.dst == st.a), None)
    if add is None or add.sub != 0 or not add.f32:
        return None
    mul = next((n for n in binf if n is not add), None)
    if mul.sub != 2 or not mul.f32 or mul.dst not in (add.a, add.b):
        return None
    load_of = {n.dst: n for n in loads}
    c_reg = add.b if mul.dst == add.a else add.a
    if c_reg not in load_of or mul.a not in load_of or mul.b not in load_of:
        return None
    lc, la, lb = load_of[c_reg], load_of[mul.a], load_of[mul.b]
    acc = {id(a.node): a for a in accesses}
    aS, aC, aA, aB = acc[id(st)], acc[id(lc)], acc[id(la)], acc[id(lb)]
    bufs = region.buffers
    if aS.slot != aC.slot or aS.offset is None or aS.offset != aC.offset:
        return None
    if aA.offset is None or aB.offset is None:
        return None
    C = bufs[aS.slot]
    A, B = bufs[aA.slot], bufs[aB.slot]
    if any(x.dtype != "f32" for x in (A, B, C)) or aA.slot == aS.slot or aB.slot == aS.slot:
        return None
    vars_ = [v for link in links for v in link.vars]
    roles = {"m": [], "n": [], "k": []}
    for v in vars_:
        lb, step, trip = v.static()
        cc, ca, cb = (aS.offset.t.get(v.id, 0), aA.offset.t.get(v.id, 0),
                      aB.offset.t.get(v.id, 0))
        if trip == 1 and not (cc or ca or cb):
            continue
        if cc and ca and not cb:
            roles["m"].append(v)
        elif cc and cb and not ca:
            roles["n"].append(v)
        elif ca and cb and not cc:
            roles["k"].append(v)
        elif trip == 1:
            continue
        else:
            return None
    # an A-only / B-only operand pairing is symmetric: swap so A carries m
    if any(len(r) != 1 for r in roles.values()):
        return None
    (vm,), (vn,), (vk,) = roles["m"], roles["n"], roles["k"]
    g = GemmMatch()

    def stride(off, v):
        return off.t.get(v.id, 0) * v.static()[1]

    def base(off):
        b = off.c
        for vid, c in off.t.items():
            b += c * region.vars[vid].static()[0]
        return b

    g.A, g.B, g.C = A, B, C
    g.sA = (stride(aA.offset, vm), stride(aA.offset, vk))
    g.sB = (stride(aB.offset, vk), stride(aB.offset, vn))
    g.sC = (stride(aS.offset, vm), stride(aS.offset, vn))
    g.M, g.N, g.K = vm.static()[2], vn.static()[2], vk.static()[2]
    g.offA, g.offB, g.offC = base(aA.offset), base(aB.offset), base(aS.offset)
    if not _mixed_radix_injective([(abs(g.sC[0]), g.M), (abs(g.sC[1]), g.N)], 0):
        return None
    return g


__all__ = ["match_gemm", "GemmMatch"]
