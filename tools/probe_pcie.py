"""Dev probe: pinned host<->device copy bandwidth, each direction alone and
both at once on two streams (is the link full duplex for the staging?)."""
import time

import torch


def main():
    n = 256 << 20
    h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
    d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
    d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / reps

    def h2d():
        with torch.cuda.stream(s1):
            d_a.copy_(h_in, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            h_out.copy_(d_b, non_blocking=True)

    def both():
        h2d()
        d2h()

    t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
    print(f"H2D {n / t1 / 1e9:.1f} GB/s  D2H {n / t2 / 1e9:.1f} GB/s  "
          f"both {2 * n / t3 / 1e9:.1f} GB/s aggregate ({t3 * 1e3:.2f} ms vs {1e3 * (t1 + t2):.2f} serial)")
    # pageable source for comparison
    p_in = torch.empty(n, dtype=torch.uint8)
    t4 = timed(lambda: d_a.copy_(p_in))
    print(f"H2D pageable {n / t4 / 1e9:.1f} GB/s")


if __name__ == "__main__":
    main()
