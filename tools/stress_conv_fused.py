"""Dev stress: random shapes for the bf16 conv with the input converted in
the kernel (b200_conv2d_tc_fused) against pack + conv (b200_pack_conv_input
+ b200_conv2d_tc): the patches hold the same bf16 values, so the outputs
must be bit-identical.  Shapes the fused kernel declines (EUNSUPPORTED) are
counted, not failed.

    python tools/stress_conv_fused.py [cases] [seed]
"""
import ctypes
import os
import random
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2307_16080_b200 import runtime  # noqa: E402


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    rnd = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
    lib = runtime.load_library()
    P = ctypes.c_void_p
    I64 = ctypes.c_int64 * 4
    s = P(torch.cuda.current_stream().cuda_stream)
    bad = declined = 0
    for case in range(cases):
        nb = rnd.randint(1, 8)
        c = rnd.choice([3, 8, 16, 32, 48, 64])
        f = rnd.choice([32, 64])
        ho = 2 * rnd.randint(2, 28)
        wo = 2 * rnd.randint(2, 28)
        init = rnd.randint(0, 1)
        kh = kw = 3
        hp, wp = ho + 2, wo + 2
        cp = 64
        g = torch.Generator(device="cuda").manual_seed(case)
        x = torch.rand(nb, c, hp, wp, device="cuda", generator=g) * 2 - 1
        w = torch.rand(f, c, kh, kw, device="cuda", generator=g) * 2 - 1
        o0 = torch.rand(nb, f, ho, wo, device="cuda", generator=g) * 2 - 1
        xp = torch.empty(nb, hp, wp, cp, device="cuda", dtype=torch.bfloat16)
        wt = torch.empty(f, kh * kw * cp, device="cuda", dtype=torch.bfloat16)
        xs, ws, os_ = I64(*x.stride()), I64(*w.stride()), I64(*o0.stride())
        runtime.check(lib.b200_pack_conv_weight(P(w.data_ptr()), ws, P(wt.data_ptr()), f, c, kh,
                                                kw, cp, s), "wpack")
        a, b = o0.clone(), o0.clone()
        runtime.check(lib.b200_pack_conv_input(P(x.data_ptr()), xs, P(xp.data_ptr()), nb, c, hp,
                                               wp, cp, s), "pack")
        rc = lib.b200_conv2d_tc(P(xp.data_ptr()), P(wt.data_ptr()), P(a.data_ptr()), os_, nb, cp,
                                hp, wp, f, ho, wo, kh, kw, init, ctypes.c_float(0.5), s)
        assert rc == 0, rc
        rc = lib.b200_conv2d_tc_fused(P(x.data_ptr()), xs, P(wt.data_ptr()), P(b.data_ptr()),
                                      os_, nb, c, hp, wp, f, ho, wo, kh, kw, init,
                                      ctypes.c_float(0.5), s)
        torch.cuda.synchronize()
        tag = f"case {case}: nb {nb} C {c} F {f} {ho}x{wo} init {init}"
        if rc != 0:
            declined += 1
            print(f"{tag}: fused declined ({rc})", flush=True)
            continue
        same = torch.equal(a, b)
        bad += not same
        print(f"{tag}: {'ok' if same else 'MISMATCH'}", flush=True)
    print(f"{cases - bad - declined}/{cases} bit-identical, {declined} declined, {bad} mismatched")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
