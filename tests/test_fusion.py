"""Plan-level rules of fusion.plan_shadows (CPU, no device).

A contraction's C may be handed to the next contraction as its packed bf16
A operand only when that consumer reads the whole buffer row-major with
matching shape and nothing writes the buffer in between.
"""
from paper_2307_16080_b200 import fusion


class Buf:
    def __init__(self, *shape):
        self.shape = shape


class G:
    """The ContractMatch fields plan_shadows looks at."""

    def __init__(self, A, B, C, M, N, K, sA=None, sC=None, offA=0, offC=0, strided=True):
        self.A, self.B, self.C = A, B, C
        self.M, self.N, self.K = M, N, K
        self.sA = sA or (K, 1)
        self.sC = sC or (N, 1)
        self.offA, self.offC = offA, offC
        self.strided = strided


class M:
    def __init__(self, *buffers):
        self.buffers = list(buffers)


def chain(*middle, consumer_kw=None):
    x, w1, h, w2, y = Buf(64, 32), Buf(32, 128), Buf(64, 128), Buf(128, 16), Buf(64, 16)
    p = fusion.ContractItem(G(x, w1, h, 64, 128, 32))
    c = fusion.ContractItem(G(h, w2, y, 64, 16, 128, **(consumer_kw or {})))
    items = [p] + [m(h, y) if callable(m) else m for m in middle] + [c]
    fusion.plan_shadows(items)
    return p, c


def test_linear_chain_is_shadowed():
    p, c = chain()
    assert p.shadow_out and c.shadow_in


def test_unrelated_map_in_between_keeps_the_shadow():
    p, c = chain(fusion.MapItem(M(Buf(4, 4))))
    assert p.shadow_out and c.shadow_in


def test_map_touching_c_in_between_drops_it():
    p, c = chain(lambda h, y: fusion.MapItem(M(h)))
    assert not p.shadow_out and not c.shadow_in


def test_contraction_overwriting_c_in_between_takes_over():
    made = []

    def writer(h, y):
        made.append(fusion.ContractItem(G(Buf(64, 8), Buf(8, 128), h, 64, 128, 8)))
        return made[0]

    p, c = chain(writer)
    # the consumer reads the in-between writer's output, not p's
    assert not p.shadow_out
    assert made[0].shadow_out and c.shadow_in


def test_transposed_or_partial_reads_are_not_shadowed():
    p, c = chain(consumer_kw={"sA": (1, 64)})
    assert not p.shadow_out
    p, c = chain(consumer_kw={"offA": 128})
    assert not p.shadow_out
