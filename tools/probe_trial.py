"""Dev probe: where one sweep trial's wall time goes on the B200 engine
(pass pipeline / run / guard), with explicit syncs so device time is
attributed to the phase that launched it.

    python tools/probe_trial.py [trials]
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2307_16080_b200.host import ensure_staircase  # noqa: E402

ensure_staircase()

import bench_kernels as bk  # noqa: E402


def main():
    import itertools

    import torch

    from paper_2307_16080_b200 import sweep
    from staircase.passes import run_pipeline
    from staircase.tuner import ParamSpace

    n = int(sys.argv[1]) if len(sys.argv) > 1 else 40
    torch.zeros(1, device="cuda")
    space = ParamSpace(tile_sizes=([1, 2, 4, 8, 16, 32, 64, 128],) * 2, unroll_factors=[1, 2, 4, 8])
    for fn in (bk.mm_par1024, bk.conv_paper):
        import paper_2307_16080_b200 as b2

        Session, ref = sweep._session_class()
        t0 = time.perf_counter()
        s = Session(fn.module, b2.engine)
        torch.cuda.synchronize()
        t_setup = time.perf_counter() - t0
        pts = list(itertools.product(*space.tile_sizes, space.unroll_factors))[:n]
        tp = tr = tg = 0.0
        for idx, pt in enumerate(pts):
            tiles, unroll = list(pt[:-1]), pt[-1]
            t0 = time.perf_counter()
            work, _ = run_pipeline(fn.module, s.template(tiles, unroll)) \
                if True else (None, None)
            fn.module.ctx.modules.remove(work)
            t1 = time.perf_counter()
            s.trial(idx + 1, tiles, unroll)
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            tp += t1 - t0
            tr += t2 - t1
        print(f"{fn.__name__}: setup {t_setup * 1e3:.1f} ms; per trial: pipeline "
              f"{tp / n * 1e3:.2f} ms, whole trial (incl. its own pipeline) {tr / n * 1e3:.2f} ms")
        # the trial's parts on one representative point
        for pt in pts[:3] + pts[-3:]:
            tiles, unroll = list(pt[:-1]), pt[-1]
            work, _ = run_pipeline(fn.module, s.template(tiles, unroll))
            sess, args = s._resident_args()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            results, stats = sess.run(work, s.func, args)
            t1 = time.perf_counter()
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            stage = sess.be.stage
            ok = True
            for a, w in zip(args, s.want_args):
                if hasattr(w, "data"):
                    ent = stage.dev.get(id(a))
                    ok &= sweep._fast_buffers_close(a, w, lambda b, e=ent: e[1])
            t3 = time.perf_counter()
            fn.module.ctx.modules.remove(work)
            print(f"  tiles {tiles} unroll {unroll}: run host {1e3 * (t1 - t0):.2f} ms, "
                  f"device tail {1e3 * (t2 - t1):.2f} ms, guard {1e3 * (t3 - t2):.2f} ms, ok {ok}, "
                  f"plan {b2.engine.last_plan[:1] or sess.plan[:1]}")


if __name__ == "__main__":
    main()
