"""Dev probe: D2H / H2D rates into array.array storage registered by
runtime.pin_host (the engine's path for Buffers), by size."""
import array
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2307_16080_b200 import runtime

    for mib in (64, 256, 1024):
        n = mib << 18
        arr = array.array("f", bytes(4 * n))
        host = torch.frombuffer(arr, dtype=torch.float32)
        runtime.pin_host(arr, host)
        runtime.pin_host(arr, host)
        pinned = id(arr) in runtime._PINNED
        dev = torch.empty(n, device="cuda")
        for name, fn in (("d2h", lambda: host.copy_(dev, non_blocking=True)),
                         ("h2d", lambda: dev.copy_(host, non_blocking=True))):
            fn()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            ms = (time.perf_counter() - t0) / 3 * 1e3
            print(f"{mib} MiB pinned={pinned} {name}: {ms:.2f} ms, {4 * n / ms / 1e6:.1f} GB/s",
                  flush=True)


if __name__ == "__main__":
    main()
