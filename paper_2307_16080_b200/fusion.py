"""Cross-region fusion of queued kernel plans (the Linear lowering and friends).

The Linear(32,32) lowering is four top-level nests:

    fill  tmp[i,j] = 0.0                          (map, kind "fill")
    copy  out[i,j] = tmp[i,j]                      (map, kind "copy")
    mm    out[i,j] = out[i,j] + x[i,k] * wt[k,j]   (contraction)
    bias  out[i,j] = out[i,j] + bias[j]            (map, kind "ewise")

Executed naively that is four launches and three extra passes over `out`.
Because each of these nests is race-free and fully covers its output, their
composition is exactly

    tmp = fill(0.0);  out[i,j] = ((0.0 + x.w chain in k order) + bias[j])

so the copy disappears, the fill value becomes the contraction's initial
value and the bias becomes its epilogue — every f32 op still individually
rounded in reference order (init -> k-ascending chain -> + bias), hence
bit-identical on the exact path.  `tmp` is still filled because it is a
live (observable) buffer.  A fill immediately overwritten by a covering
contraction (fill(out); mm(out)) is dropped entirely.
"""
from __future__ import annotations

import math


class MapItem:
    __slots__ = ("m", "tally")

    def __init__(self, m):
        self.m = m


class ContractItem:
    __slots__ = ("g", "init", "init_value", "bias", "bias_base", "bias_stride", "fused",
                 "shadow_out", "shadow_in")

    def __init__(self, g):
        self.g = g
        self.init = 0
        self.init_value = 0.0
        self.bias = None
        self.bias_base = 0
        self.bias_stride = 0
        self.fused = []
        self.shadow_out = False   # also write C as the next contraction's packed A
        self.shadow_in = False    # A is the previous contraction's shadow of its C


def _size(buf):
    return math.prod(buf.shape)


def _map_span(m, k):
    """The element range [lo, hi) operand k of a map touches, when it is a
    dense range walked once (one progression of unit stride over the box,
    e.g. a whole buffer, a batch shard's rows or a tiled nest's origin +
    offset loops), else None."""
    w = _walk([(c, 0, t) for c, t in zip(m.coefs[k], m.trips) if t > 1])
    if w is None or w[0] not in (0, 1):
        return None
    return m.bases[k], m.bases[k] + w[2]


def _contract_span(g):
    """The element range of C a contraction writes, when dense (rows of a
    row-major C: the whole buffer or a batch shard's rows), else None."""
    if g.strided and tuple(g.sC) == (g.N, 1):
        return g.offC, g.offC + g.M * g.N
    if g.M * g.N == _size(g.C):
        # distinct outputs (match_contraction proves injectivity) as many as
        # the buffer's elements: every element, whatever the index maps
        return 0, _size(g.C)
    return None


def _fill(item):
    """(buffer, value, span) if item is a dense constant fill."""
    if isinstance(item, MapItem) and item.m.kind == "fill" and len(item.m.buffers) == 1:
        span = _map_span(item.m, 0)
        if span is not None:
            return item.m.buffers[0], item.m.consts[0], span
    return None


def _copy(item):
    """(dst, dst span, src, src span) if item is a dense copy."""
    if isinstance(item, MapItem) and item.m.kind == "copy" and len(item.m.buffers) == 2:
        src, dst = item.m.buffers
        ss, ds = _map_span(item.m, 0), _map_span(item.m, 1)
        if ss is not None and ds is not None and src is not dst:
            return dst, ds, src, ss
    return None


def _contract_covers(item, buf, span):
    g = item.g
    return g.C is buf and _contract_span(g) == span


def _walk(dims):
    """(C stride, bias stride, trip) of map dims [(c coef, b coef, trip)] that
    walk one arithmetic progression (a 2-D nest's single loop, or the origin
    and offset loops of a tiled one: passes/tiling.py:56-80), else None."""
    dims = sorted(dims, key=lambda d: abs(d[0]))
    if not dims:
        return 0, 0, 1
    c0, b0, _ = dims[0]
    ec, eb, trip = c0, b0, 1
    for c, b, t in dims:
        if c != ec or b != eb:
            return None
        ec, eb, trip = ec * t, eb * t, trip * t
    return c0, b0, trip


def _bias(citem, item):
    """(bias buffer, base, stride) if item adds a per-column vector to the
    strided GEMM output of citem over the whole output."""
    g = citem.g
    if not isinstance(item, MapItem) or item.m.kind != "ewise" or not g.strided:
        return None
    m = item.m
    if len(m.buffers) != 3:
        return None
    o_ld, b_ld, o_st = m.buffers
    prog = m.prog
    # LD r0<-op0 ; LD r1<-op1 ; BF add r2 = r0+r1 | r1+r0 ; ST op2<-r2
    if len(prog) != 5 or prog[0] & 0xFF != 0 or prog[1] & 0xFF != 0 or \
            prog[2] & 0xFF != 2 or prog[3] != 0 or prog[4] & 0xFF != 3:
        return None
    if o_ld is not g.C or o_st is not g.C or b_ld is g.C:
        return None
    if m.bases[0] != m.bases[2] or m.coefs[0] != m.coefs[2]:
        return None
    if _contract_span(g) is None or _map_span(m, 2) != _contract_span(g):
        return None
    if b_ld.dtype != g.C.dtype or m.bases[0] != g.offC:
        return None
    # the map dims the bias does not move along are the GEMM's m, the others
    # its n; each side must be one progression with the GEMM's C stride
    dims = list(zip(m.coefs[0], m.coefs[1], m.trips))
    mw = _walk([d for d in dims if d[1] == 0])
    nw = _walk([d for d in dims if d[1] != 0])
    if mw is None or nw is None:
        return None
    if (mw[0], mw[2]) != (g.sC[0], g.M) and not (g.M == 1 and mw[2] == 1):
        return None
    if (nw[0], nw[2]) != (g.sC[1], g.N):
        return None
    return b_ld, m.bases[1], nw[1]


def fuse(items):
    """Peephole-fuse a queue of MapItem / ContractItem in program order."""
    out = []
    i = 0
    n = len(items)
    while i < n:
        it = items[i]
        f = _fill(it)
        # fill(T); copy(O <- T); contract(O)  ->  fill(T); contract(O, init)
        # (the copy reads only filled elements of T and writes exactly the
        # contraction's output range)
        if f is not None and i + 2 < n:
            c = _copy(items[i + 1])
            nxt = items[i + 2]
            if c is not None and c[2] is f[0] and f[2][0] <= c[3][0] and c[3][1] <= f[2][1] \
                    and isinstance(nxt, ContractItem) and _contract_covers(nxt, c[0], c[1]) \
                    and nxt.g.dtype == "f32":
                out.append(it)
                nxt.init, nxt.init_value = 1, f[1]
                nxt.fused += ["copy", "init"]
                items[i + 2] = nxt
                i += 2
                continue
        # fill(O); contract(O)  ->  contract(O, init)
        if f is not None and i + 1 < n and isinstance(items[i + 1], ContractItem) and \
                _contract_covers(items[i + 1], f[0], f[2]) and items[i + 1].g.dtype == "f32":
            nxt = items[i + 1]
            nxt.init, nxt.init_value = 1, f[1]
            nxt.fused += ["fill"]
            i += 1
            continue
        # contract(O); bias(O)  ->  contract(O, bias)
        if isinstance(it, ContractItem) and it.bias is None and i + 1 < n:
            b = _bias(it, items[i + 1])
            if b is not None:
                it.bias, it.bias_base, it.bias_stride = b
                it.fused += ["bias"]
                out.append(it)
                i += 2
                continue
        out.append(it)
        i += 1
    return out


def _dense_rows(buf, off, s, rows, cols):
    """The operand is whole rows of a row-major buffer (rows x cols): all of
    it, or a batch shard's rows."""
    return tuple(s) == (cols, 1) and off % cols == 0 and off + rows * cols <= _size(buf) \
        and cols > 0


def plan_shadows(items):
    """Mark producer/consumer pairs for the bf16 shadow of a contraction's C.

    Chained Linear layers read one contraction's output C as the next one's
    A operand.  On the tensor-core path that A is packed to bf16 K-major
    first (a full extra pass over C); instead the producer's epilogue can
    write the bf16 copy while it writes C (b200_gemm_tc_shadow).  A pair
    qualifies when both are strided GEMMs, C is the whole buffer row-major
    and is read as the whole of A row-major with the same M (K = producer
    N), and no item in between touches that buffer — so the shadow is
    exactly the pack of the consumer's A.  Whether the tensor-core path runs
    at all is the backend's decision; an unused mark costs nothing.
    """
    for i, p in enumerate(items):
        if not isinstance(p, ContractItem) or not p.g.strided:
            continue
        pg = p.g
        if not _dense_rows(pg.C, pg.offC, pg.sC, pg.M, pg.N):
            continue
        for c in items[i + 1:]:
            if isinstance(c, ContractItem):
                cg = c.g
                if cg.A is pg.C and cg.strided and cg.C is not pg.C and cg.B is not pg.C and \
                        cg.M == pg.M and cg.K == pg.N and cg.offA == pg.offC and \
                        _dense_rows(cg.A, cg.offA, cg.sA, cg.M, cg.K):
                    p.shadow_out = c.shadow_in = True
                    break
                if cg.C is pg.C:      # overwritten before a qualifying reader
                    break
            elif any(b is pg.C for b in c.m.buffers):   # maps: conservatively
                break
    return items


__all__ = ["MapItem", "ContractItem", "fuse", "plan_shadows"]
