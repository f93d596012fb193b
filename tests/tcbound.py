"""The tensor-core parity bound (tests only).

Operands are rounded to the kernel's input type (bf16 / tf32) exactly as the
pack kernels round them, so every product is exact in fp32 and the only
difference from the reference's f32 chain (interp/_evalpy.py:115-127) is the
accumulation: fp32 sums in another order.  Per output

    |got - want| <= 8 sqrt(K) 2^-24 sum_k |a_k b_k| + 4 2^-24 |want|

with ``want`` the float64 sum of the same rounded products (plus the initial
C and bias).  The probabilistic sqrt(K) form is ~ sqrt(K)/16 times tighter
than the worst-case 2 K 2^-24 bound of round 1, and catches one lost or
duplicated average product: |a_k b_k| ~ sum / K exceeds 8 sqrt(K) 2^-24 sum
whenever K^1.5 < 2^21, i.e. K < 16384.  The observed maximum of
|got - want| / (2^-24 sqrt(K) sum|ab|) is recorded (conftest.TC_ERRORS) and
printed in the session summary.
"""
import numpy as np

U = 2.0 ** -24


def bf16(x):
    import torch

    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(
        torch.bfloat16).float().numpy()


def tf32(x):
    """Round to nearest even at 10 mantissa bits (b200_pack_operand kind 1)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.int32).astype(np.int64)
    u = (u + 0xFFF + ((u >> 13) & 1)) & ~0x1FFF
    return u.astype(np.uint32).view(np.float32).reshape(np.shape(x))


def rounder(precision):
    return {"bf16": bf16, "tf32": tf32}[precision]


def check(got, want, mag, K, label):
    """Assert the bound; record and return the max normalised error."""
    import conftest

    got = np.asarray(got, dtype=np.float64)
    err = np.abs(got - want)
    scale = U * np.sqrt(K) * mag + 1e-300
    norm = float((np.maximum(err - 4 * U * np.abs(want), 0) / scale).max())
    conftest.TC_ERRORS.append((label, K, norm))
    bad = err > 8 * U * np.sqrt(K) * mag + 4 * U * np.abs(want) + 1e-30
    assert not bad.any(), (f"{label}: {bad.sum()} of {bad.size} outputs outside the bound; "
                           f"max_norm_err {norm:.3f}")
    return norm
