"""bench.py end to end with two ranks on the one B200 of a gpurun box.

The driver's scaling runs launch bench.py under torch.distributed.run with
NCCL, one rank per GPU; a 1-GPU box cannot host two NCCL ranks, so the same
launch runs here with B200_BENCH_BACKEND=gloo (host-side collectives; both
ranks' kernels share the GPU).  The JSON line must report both ranks' work
(n_gpus 2, the batch-sharded conv's flops over the whole batch, each rank on
its own half of the images) with the checksums of both ranks, and the
outputs' all-gather timed separately.
"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("workload", ["linear32", "conv"])
def test_bench_two_ranks_gloo(workload):
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, B200_BENCH_BACKEND="gloo")
    out = subprocess.run(
        [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
         "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2",
         "--steps", "3", "--warmup", "3", "--workload", workload, "--min-seconds", "0.2"],
        cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout          # rank 0 prints the one line
    line = lines[0]
    assert line["n_gpus"] == 2 and len(line["checksums"]) == 2
    assert line["value"] > 0 and line["gpu_launches"] > 0
    if workload == "conv":
        assert line["scaling"] == "strong"
        assert "batch shard x2 (rows 0..127 on rank 0)" == line["config"]["parallelism"]
        assert line["gather"]["bytes_received_per_rank"] == 128 * 64 * 56 * 56 * 4
        assert line["e2e"]["h2d_bytes_per_step"] < 256 * 64 * 58 * 58 * 4
