"""Dev stress: the tcgen05 GEMMs (b200_gemm_tc variants 1/2/3 = single CTA,
CTA pair, SOLO clusters; b200_gemm_tc_kn) over random shapes, CTA counts
(persistent loops, split tail waves), init / bias, bf16 and tf32, against a
float64 product of the same rounded operands within the tensor-core bound
(tests/test_gpu_tc.py's).

    python tools/stress_tc.py [cases] [seed]
"""
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import test_gpu_tc as tt

    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    rnd = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 0)
    bad = 0
    for c in range(cases):
        kind = rnd.choice([0, 1])
        variant = rnd.choice([1, 2, 3])
        M = rnd.choice([64, 128, 200, 256, 384, 512, 1000, 1024, 1536, 2048, 3000])
        N = rnd.choice([16, 64, 128, 200, 256, 520, 768, 1024, 2048, 2304])
        K = 8 * rnd.randint(1, 160) if kind == 0 else 4 * rnd.randint(1, 320)
        init, bias, trans_b = rnd.randint(0, 1), rnd.randint(0, 1) == 1, rnd.randint(0, 1) == 1
        max_ctas = rnd.choice([0, 0, 2, 4, 8, 30, 100])
        err, bound, *_ = tt._run(kind, M, N, K, init=init, bias=bias, trans_b=trans_b, seed=c,
                                 max_ctas=max_ctas, variant=variant)
        nbad = int((err > bound).sum().item())
        bad += nbad > 0
        print(f"case {c}: kind {kind} variant {variant} {M}x{N}x{K} init {init} bias {bias} "
              f"transB {trans_b} ctas {max_ctas}: {'ok' if nbad == 0 else f'{nbad} OUT OF BOUND'}",
              flush=True)
    print(f"{cases - bad}/{cases} within the bound")
    sys.exit(1 if bad else 0)


if __name__ == "__main__":
    main()
