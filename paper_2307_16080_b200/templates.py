"""Recognise dense contractions in lifted regions and map them to kernels.

The reference's matmul nests (reference tests/kernels.py:24-38, PAPER.md
143-191), the contraction nest of the Linear lowering (PAPER.md 443-454) and
the NCHW/FCHW convolution (tests/kernels.py:50-64, PAPER.md 1048-1068) all
have the shape

    for <vars, any nesting / parallel / launch mix, static bounds>:
        a = A[fA(vars)]; b = B[fB(vars)]; c = C[fC(vars)]
        C[fC(vars)] = c + a * b            # f32 or f64, each op rounded

with affine index maps.  Every variable with trip > 1 must play exactly one
role: M (appears in C and A), N (C and B) or K (A and B only — a reduction,
executed per output in nest order, i.e. lexicographically over the K
variables in nesting order).  Trip-1 variables are constants.  Then

    C[cM(m) + cN(n)] = C[..] + sum_k A[aM(m) + aK(k)] * B[bK(k) + bN(n)]

where each offset function is a per-group table (mixed-radix enumeration of
that group's variables).  A contraction whose every group walks one
arithmetic progression in its operands — a single variable, or the origin +
offset pair of a tiled nest (passes/tiling.py:56-80) — is a plain strided
GEMM (and can use the tensor-core path; the tile sizes are kept to choose
the CTA tile); anything else (conv = implicit GEMM with M = (n, ho, wo),
N = co, K = (ci, ki, kj), ...) uses offset tables or the conv kernels.
"""
from __future__ import annotations

import numpy as np

from .analysis import _mixed_radix_injective
from .lift import BINF, LOAD, PURE_OPS, RETURN_GPU, STORE, Ins

_IGNORED = PURE_OPS | {RETURN_GPU}


class ContractMatch:
    """A recognised contraction: operands, groups and addressing."""

    __slots__ = ("A", "B", "C", "dtype", "M", "N", "K", "m_vars", "n_vars", "k_vars",
                 "_tables", "_make_tables", "origins", "strided", "offA", "offB", "offC",
                 "sA", "sB", "sC", "offsets", "stat", "tiles")

    def __repr__(self):
        return (f"ContractMatch({self.dtype}, M={self.M}, N={self.N}, K={self.K}, "
                f"strided={self.strided})")

    @property
    def tables(self):
        """(a_m, a_k, b_k, b_n, c_m, c_n) int64 element-offset tables, built on
        first use: only the table-addressed kernel needs them, and for large
        conv / tiled nests they cost milliseconds of host time per plan."""
        if self._tables is None:
            self._tables = self._make_tables()
        return self._tables


def _straight_line(nodes):
    return all(isinstance(n, Ins) for n in nodes)



def _table(region, vars_, off, stat):
    """Element offsets of one operand over the mixed-radix enumeration of vars_."""
    t = np.zeros(1, dtype=np.int64)
    for v in vars_:
        lb, st, trip = stat(v)
        vals = off.t.get(v.id, 0) * (lb + st * np.arange(trip, dtype=np.int64))
        t = (t[:, None] + vals[None, :]).reshape(-1)
    return t


def _statement(ops, acc):
    """Match one `C[f] = C[f] + A[a] * B[b]` statement: (aS, aA, aB, f32)."""
    loads = [n for n in ops if n.op == LOAD]
    binf = [n for n in ops if n.op == BINF]
    stores = [n for n in ops if n.op == STORE]
    if len(loads) != 3 or len(binf) != 2 or len(stores) != 1 or len(ops) != 6:
        return None
    st = stores[0]
    add = next((n for n in binf if n.dst == st.a), None)
    if add is None or add.sub != 0:
        return None
    mul = next((n for n in binf if n is not add), None)
    if mul.sub != 2 or mul.f32 != add.f32 or mul.dst not in (add.a, add.b):
        return None
    load_of = {n.dst: n for n in loads}
    c_reg = add.b if mul.dst == add.a else add.a
    if c_reg not in load_of or mul.a not in load_of or mul.b not in load_of:
        return None
    lc, la, lb = load_of[c_reg], load_of[mul.a], load_of[mul.b]
    aS, aC, aA, aB = acc[id(st)], acc[id(lc)], acc[id(la)], acc[id(lb)]
    if aS.slot != aC.slot or aS.offset is None or aS.offset != aC.offset:
        return None
    if aA.offset is None or aB.offset is None or aA.slot == aS.slot or aB.slot == aS.slot:
        return None
    return aS, aA, aB, add.f32


def _reroll(stmts, vars_):
    """U unrolled clones of one contraction statement -> the rolled loop.

    loop-unroll (reference passes/unroll.py:42-56) multiplies the innermost
    step by U and clones the body with iv + u*step: clone u reads A/B at a
    constant offset u*delta from clone 0 and accumulates into the same C
    element, so the clones are exactly the next U iterations of the
    reduction.  Returns {var id: (lb, step, trip)} overriding the unrolled
    variable, or None if the clones are not such a progression.
    """
    s0 = stmts[0]
    U = len(stmts)
    dS = [s[0].offset.c - s0[0].offset.c for s in stmts]
    dA = [s[1].offset.c - s0[1].offset.c for s in stmts]
    dB = [s[2].offset.c - s0[2].offset.c for s in stmts]
    for s in stmts:
        if (s[0].slot, s[1].slot, s[2].slot) != (s0[0].slot, s0[1].slot, s0[2].slot) or \
                s[0].offset.t != s0[0].offset.t or s[1].offset.t != s0[1].offset.t or \
                s[2].offset.t != s0[2].offset.t or s[3] != s0[3]:
            return None
    # the unrolled variable may be a reduction (same C, shifted A/B: the next
    # U steps of each chain) or an output dimension (shifted C: U distinct
    # outputs whose chains are interleaved but individually unchanged)
    for v in vars_:
        lb, step, trip = v.static()
        cs, ca, cb = (s0[0].offset.t.get(v.id, 0), s0[1].offset.t.get(v.id, 0),
                      s0[2].offset.t.get(v.id, 0))
        if not (cs or ca or cb) or step % U:
            continue
        sub = step // U
        if all(dS[u] == u * cs * sub and dA[u] == u * ca * sub and dB[u] == u * cb * sub
               for u in range(U)):
            return {v.id: (lb, sub, trip * U)}
    return None


def match_contraction(region, links, remainder, accesses):
    """Return a ContractMatch for a C (+)= A*B nest (possibly unrolled), else None."""
    if not links or not _straight_line(remainder):
        return None
    body = [n for n in remainder if n.op not in _IGNORED or n.op == BINF]
    acc = {id(a.node): a for a in accesses}
    stmts, cur = [], []
    for n in body:
        cur.append(n)
        if n.op == STORE:
            s = _statement(cur, acc)
            if s is None:
                return None
            stmts.append(s)
            cur = []
    if cur or not stmts:
        return None
    vars_ = [v for link in links for v in link.vars]
    ovr = {}
    if len(stmts) > 1:
        ovr = _reroll(stmts, vars_)
        if ovr is None:
            return None
    aS, aA, aB, f32 = stmts[0]
    bufs = region.buffers
    C, A, B = bufs[aS.slot], bufs[aA.slot], bufs[aB.slot]
    dtype = C.dtype
    if dtype not in ("f32", "f64") or A.dtype != dtype or B.dtype != dtype:
        return None
    if f32 != (dtype == "f32"):
        return None

    def stat(v):
        return ovr.get(v.id) or v.static()

    groups = {"m": [], "n": [], "k": []}
    for v in vars_:
        lb_, step, trip = stat(v)
        cc, ca, cb = (aS.offset.t.get(v.id, 0), aA.offset.t.get(v.id, 0),
                      aB.offset.t.get(v.id, 0))
        if trip == 1:
            continue   # a constant: folded into the tables below
        if cc and ca and not cb:
            groups["m"].append(v)
        elif cc and cb and not ca:
            groups["n"].append(v)
        elif ca and cb and not cc:
            groups["k"].append(v)
        else:
            return None   # batch dims, reductions into C, or unused loop vars
    if not groups["k"]:
        return None
    # M / N: order by decreasing |C stride| so the last (fastest) index is the
    # most contiguous in C; K: nest order (the reference's reduction order).
    for key in ("m", "n"):
        groups[key].sort(key=lambda v: -abs(aS.offset.t.get(v.id, 0) * stat(v)[1]))

    g = ContractMatch()
    g.stat = stat   # (lb, step, trip) per variable, unrolled ones re-rolled
    g.A, g.B, g.C, g.dtype = A, B, C, dtype
    g.offsets = (aA.offset, aB.offset, aS.offset)
    g.m_vars, g.n_vars, g.k_vars = groups["m"], groups["n"], groups["k"]
    prod = lambda vs: int(np.prod([stat(v)[2] for v in vs])) if vs else 1  # noqa: E731
    g.M, g.N, g.K = prod(g.m_vars), prod(g.n_vars), prod(g.k_vars)

    def const(off, used):
        c = off.c
        for vid, coef in off.t.items():
            if vid not in used:
                c += coef * region.vars[vid].static()[0]   # trip-1 vars
        return c

    used = {v.id for v in vars_ if stat(v)[2] > 1}
    cA, cB, cC = const(aA.offset, used), const(aB.offset, used), const(aS.offset, used)

    def make_tables():
        return (_table(region, g.m_vars, aA.offset, stat) + cA,
                _table(region, g.k_vars, aA.offset, stat),
                _table(region, g.k_vars, aB.offset, stat) + cB,
                _table(region, g.n_vars, aB.offset, stat),
                _table(region, g.m_vars, aS.offset, stat) + cC,
                _table(region, g.n_vars, aS.offset, stat))

    g._tables, g._make_tables = None, make_tables

    def first(off, vs):   # the tables' first entries: every variable at its lb
        return sum(off.t.get(v.id, 0) * stat(v)[0] for v in vs)

    g.origins = (cA + first(aA.offset, g.m_vars) + first(aA.offset, g.k_vars),
                 cB + first(aB.offset, g.k_vars) + first(aB.offset, g.n_vars),
                 cC + first(aS.offset, g.m_vars) + first(aS.offset, g.n_vars))
    # outputs must be distinct (writes of different (m, n) never collide)
    terms = [(abs(aS.offset.t.get(v.id, 0) * stat(v)[1]), stat(v)[2])
             for v in g.m_vars + g.n_vars]
    if not _mixed_radix_injective(terms, 0):
        return None
    # one strided dimension per group: a single variable, or the origin and
    # offset loops of a tiled nest (passes/tiling.py:56-80: index = origin +
    # offset) that together walk one arithmetic progression in every operand
    mS = _progression(reversed(g.m_vars), (aS.offset, aA.offset), stat)
    nS = _progression(reversed(g.n_vars), (aS.offset, aB.offset), stat)
    # K: the progression must also be the nest order (outer = larger stride),
    # the order every output's chain is rounded in
    kS = _progression(reversed(g.k_vars), (aA.offset, aB.offset), stat)
    g.strided = mS is not None and nS is not None and kS is not None
    g.tiles = (_tile(g.m_vars, stat), _tile(g.n_vars, stat)) if g.strided else (None, None)
    if g.strided:
        g.sA = (mS[1], kS[0])
        g.sB = (kS[1], nS[1])
        g.sC = (mS[0], nS[0])
        g.offA, g.offB, g.offC = (int(o) for o in g.origins)
    return g


def _progression(vars_, offs, stat):
    """Element strides, one per form in ``offs``, of the variables ``vars_``
    (innermost = smallest stride first) merged into one loop — or None.

    They merge when each variable's stride is the previous one's times its
    trip count in every operand (a mixed-radix enumeration with one radix
    chain: 0 .. trip-1 of the merged loop, each point once, in order).  An
    empty group is a stride-0 dimension of extent 1."""
    vs = list(vars_)
    if not vs:
        return tuple(0 for _ in offs)
    base = [off.t.get(vs[0].id, 0) * stat(vs[0])[1] for off in offs]
    expect = list(base)
    for v in vs:
        _, step, trip = stat(v)
        for i, off in enumerate(offs):
            if off.t.get(v.id, 0) * step != expect[i]:
                return None
            expect[i] *= trip
    return tuple(base)


def _tile(vars_, stat):
    """The tile extent of a tiled group (the innermost, offset loop's trip),
    or None when the group is a single loop."""
    return stat(vars_[-1])[2] if len(vars_) > 1 else None



class ConvView:
    """A contraction that is exactly conv_2d_nchw_fchw (valid, stride 1)."""

    __slots__ = ("nb", "c", "hp", "wp", "f", "ho", "wo", "kh", "kw", "inp", "ker", "out",
                 "k_order",   # k_order: the reduction variables' roles in nest order
                 "n0")        # first image (a batch shard's range starts there)

    def __repr__(self):
        return (f"ConvView(nb={self.nb}, c={self.c}, {self.hp}x{self.wp} -> f={self.f}, "
                f"{self.ho}x{self.wo}, {self.kh}x{self.kw})")


def conv_view(region, g, dtypes=("f32",)):
    """Recognise out[n,f,h,w] += in[n,c,h+i,w+j] * w[f,c,i,j] (reference
    tests/kernels.py:50-64) from a ContractMatch's index maps.  Every variable
    starts at 0 and carries exactly one role's coefficients; an output role
    may be carried by several variables — the origin and offset loops of a
    tiled nest (passes/tiling.py: index = origin + offset) — when together
    they enumerate 0 .. extent-1 exactly once (mixed radix: steps 1, t0,
    t0 t1, ...).  Reduction roles take one variable each; ``k_order`` lists
    them in nest (= rounding) order."""
    if g is None or g.dtype not in dtypes:
        return None
    A, B, C = g.A, g.B, g.C
    if len(A.shape) != 4 or len(B.shape) != 4 or len(C.shape) != 4:
        return None
    sa, sb, sc = A.strides, B.strides, C.strides
    offA, offB, offC = _offsets(region, g)
    # every loop starts at 0, except that a single batch loop may start at
    # n0 (a batch shard, shard.py): the operands' base offsets are then
    # n0 whole images of the input and the output
    n0 = g.origins[0] // sa[0] if sa[0] > 0 else 0
    if n0 < 0 or tuple(g.origins) != (n0 * sa[0], 0, n0 * sc[0]):
        return None
    for v in g.m_vars + g.n_vars + g.k_vars:
        lb, st, t = g.stat(v)
        if st < 1:
            return None
        if lb != 0 and ((offC.t.get(v.id, 0), offA.t.get(v.id, 0)) != (sc[0], sa[0]) or
                        st != 1 or lb != n0):
            return None
    # classify each variable by its coefficient signature.  Size-1
    # dimensions make signatures coincide (e.g. a 1x1 filter over one output
    # row: the input's channel and row strides are both W), so a variable
    # takes the first role, in nest order, whose signature matches and whose
    # dimension its index range fits (the shape checks below confirm it)
    def fits(v, extent):
        lb, st, t = g.stat(v)
        return lb + st * (t - 1) < extent

    roles = {}
    m_roles = (((sc[0], sa[0]), "n", C.shape[0]), ((sc[2], sa[2]), "ho", C.shape[2]),
               ((sc[3], sa[3]), "wo", C.shape[3]))
    for v in g.m_vars:
        sig = (offC.t.get(v.id, 0), offA.t.get(v.id, 0))
        role = next((r for sg, r, ext in m_roles if sg == sig and fits(v, ext)), None)
        if role is None:
            return None
        roles.setdefault(role, []).append(v)
    for v in g.n_vars:
        if (offC.t.get(v.id, 0), offB.t.get(v.id, 0)) != (sc[1], sb[0]):
            return None
        roles.setdefault("co", []).append(v)
    k_roles = (((sa[1], sb[1]), "ci", B.shape[1]), ((sa[2], sb[2]), "ki", B.shape[2]),
               ((sa[3], sb[3]), "kj", B.shape[3]))
    for v in g.k_vars:
        sig = (offA.t.get(v.id, 0), offB.t.get(v.id, 0))
        role = next((r for sg, r, ext in k_roles
                     if sg == sig and r not in roles and fits(v, ext)), None)
        if role is None:
            return None
        if g.stat(v)[1] != 1:
            return None
        roles[role] = [v]
    # a role without a variable has extent 1 (trip-1 loops are folded into
    # the constants); the shape checks below confirm every extent

    def extent(name):
        if name not in roles:
            return 1
        step = 1
        for v in sorted(roles[name], key=lambda v: g.stat(v)[1]):
            _, st, t = g.stat(v)
            if st != step:
                return None   # not an exact mixed-radix cover of 0 .. extent-1
            step *= t
        return step

    cv = ConvView()
    cv.nb, cv.f, cv.ho, cv.wo = extent("n"), extent("co"), extent("ho"), extent("wo")
    cv.c, cv.kh, cv.kw = extent("ci"), extent("ki"), extent("kj")
    if None in (cv.nb, cv.f, cv.ho, cv.wo):
        return None
    if n0 and len(roles.get("n", ())) > 1:
        return None
    if n0 + cv.nb > A.shape[0] or n0 + cv.nb > C.shape[0]:
        return None
    if A.shape[1] != cv.c or C.shape[1:] != (cv.f, cv.ho, cv.wo) or \
            B.shape != (cv.f, cv.c, cv.kh, cv.kw):
        return None
    cv.n0 = n0
    cv.hp, cv.wp = A.shape[2], A.shape[3]
    if cv.hp < cv.ho + cv.kh - 1 or cv.wp < cv.wo + cv.kw - 1:
        return None
    cv.inp, cv.ker, cv.out = A, B, C
    by_id = {vs[0].id: name for name, vs in roles.items() if name in ("ci", "ki", "kj")}
    cv.k_order = tuple(by_id[v.id] for v in g.k_vars)
    return cv


def _offsets(region, g):
    """The element-offset affine forms of C, A, B recorded for g."""
    return g.offsets


class MapMatch:
    """A pointwise f32 nest: box dims, operands, straight-line program."""

    __slots__ = ("trips", "buffers", "bases", "coefs", "prog", "consts", "vector", "kind",
                 "nload")

    def __repr__(self):
        return f"MapMatch({self.kind}, trips={self.trips}, ops={len(self.buffers)})"


M_LD, M_CF, M_BF, M_ST = 0, 1, 2, 3


def match_map(region, links, remainder, accesses, band):
    """Straight-line f32 body over a fully distributed static box."""
    from .lift import CONST

    if not links or not _straight_line(remainder):
        return None
    box = [v for link in links for v in link.vars]
    if set(band) != {v.id for v in box}:
        return None
    dims = [v for v in box if v.static()[2] > 1]
    if not dims or len(dims) > 8:
        return None
    acc_of = {id(a.node): a for a in accesses}
    m = MapMatch()
    m.trips = [v.static()[2] for v in dims]
    m.buffers, m.bases, m.coefs, m.prog, m.consts = [], [], [], [], []
    regs = {}

    def reg_of(v):
        return regs.get(v)

    def new_reg(v):
        if len(regs) >= 32:
            raise ValueError
        regs[v] = len(regs)
        return regs[v]

    def operand(a):
        buf = region.buffers[a.slot]
        if buf.dtype != "f32" or a.offset is None or len(m.buffers) >= 16:
            raise ValueError
        base = a.offset.c
        for vid, c in a.offset.t.items():
            base += c * region.vars[vid].static()[0]
        m.buffers.append(buf)
        m.bases.append(base)
        m.coefs.append([a.offset.t.get(v.id, 0) * v.static()[1] for v in dims])
        return len(m.buffers) - 1

    n_mem = 0
    try:
        for n in remainder:
            if n.op == LOAD:
                k = operand(acc_of[id(n)])
                m.prog.append(M_LD | (new_reg(n.dst) << 8) | (k << 16))
                n_mem += 1
            elif n.op == STORE:
                k = operand(acc_of[id(n)])
                r = reg_of(n.a)
                if r is None:
                    return None
                m.prog.append(M_ST | (r << 8) | (k << 16))
                n_mem += 1
            elif n.op == CONST and isinstance(n.value, float):
                if len(m.consts) >= 32:
                    return None
                m.consts.append(n.value)
                m.prog.append(M_CF | (new_reg(n.dst) << 8) | ((len(m.consts) - 1) << 16))
            elif n.op == BINF:
                a, b = reg_of(n.a), reg_of(n.b)
                if a is None or b is None or not n.f32:
                    return None
                m.prog.append(M_BF | (new_reg(n.dst) << 8) | (a << 16) | (b << 24))
                m.prog.append(n.sub)
            elif n.op in _IGNORED:
                continue   # index arithmetic: folded into the affine operands
            else:
                return None
    except ValueError:
        return None
    _merge_dims(m)
    _hoist_loads(m)
    ops_seq, pc = [], 0
    while pc < len(m.prog):
        op = m.prog[pc] & 0xFF
        ops_seq.append(op)
        pc += 2 if op == M_BF else 1
    if M_ST not in ops_seq or len(m.prog) > 256:
        return None
    inner = len(m.trips) - 1
    m.vector = m.trips[inner] % 4 == 0 and all(
        c[inner] in (0, 1) and (c[inner] == 0 or (b % 4 == 0 and all(x % 4 == 0 for x in c[:inner])))
        for b, c in zip(m.bases, m.coefs))
    m.kind = ("fill" if ops_seq == [M_CF, M_ST] else
              "copy" if ops_seq == [M_LD, M_ST] else "ewise")
    return m


def _hoist_loads(m):
    """Move every load to the front of the program (loads only depend on
    affine addresses) unless a load follows a store — then a read-after-
    write through memory inside one point could exist and order is kept.
    m.nload = number of leading loads (the kernel issues them together)."""
    words, pc, seen_store = [], 0, False
    loads, rest = [], []
    hoistable = True
    while pc < len(m.prog):
        w = m.prog[pc]
        op = w & 0xFF
        if op == M_BF:
            rest.append([w, m.prog[pc + 1]])
            pc += 2
            continue
        if op == M_ST:
            seen_store = True
        if op == M_LD:
            if seen_store:
                hoistable = False
            loads.append([w])
        else:
            rest.append([w])
        pc += 1
    if hoistable and len(loads) <= 4:
        m.prog = [x for ins in loads + rest for x in ins]
        m.nload = len(loads)
    else:
        m.nload = 0


def _merge_dims(m):
    """Collapse adjacent box dims that every operand walks contiguously
    (coef[d] == coef[d+1] * trip[d+1]); a dense row-major box becomes 1-D."""
    d = len(m.trips) - 2
    while d >= 0:
        t_in = m.trips[d + 1]
        if all(c[d] == c[d + 1] * t_in for c in m.coefs):
            m.trips[d] = m.trips[d] * t_in
            del m.trips[d + 1]
            for c in m.coefs:
                del c[d]          # the merged dim keeps coef[d+1]
        d -= 1


def match_gemm(region, links, remainder, accesses):
    """Back-compat: a strided fp32 contraction only."""
    g = match_contraction(region, links, remainder, accesses)
    if g is None or not g.strided or g.dtype != "f32":
        return None
    return g


__all__ = ["match_contraction", "match_gemm", "match_map", "ContractMatch", "MapMatch"]
