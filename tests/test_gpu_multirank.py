"""bench.py's multi-GPU rank path on real kernels, on a one-GPU box: two
ranks launched by torch.distributed.run, both on cuda:0, gloo for the
barrier and the max-over-ranks timing reduction (PPFG_BENCH_BACKEND /
PPFG_BENCH_SAME_DEVICE). Each rank synthesises its own contiguous segment of
one stream plus its (T-1)-spectrum halo and runs the fused
kernel on it; every rank's whole output is checked against the reference
(--parity-all-ranks), so the shard / halo arithmetic is verified end to end.
The driver's SCALE run measures real multi-GPU scaling; this covers the
code path."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("config,extra", [("ska", ["--spectra", "30001"]),
                                          ("long16", ["--spectra", "60000"])])
def test_two_ranks_on_one_device(config, extra):
    env = dict(os.environ, PPFG_BENCH_BACKEND="gloo", PPFG_BENCH_SAME_DEVICE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "3", "--warmup", "3",
           "--config", config, "--no-e2e", "--no-cpu-baseline", "--no-configs", "--no-exact",
           "--parity-all-ranks", *extra]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]   # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["gpu_launches"] == 3
    p = d["parity"]
    assert p["ranks"] == 2 and p["pass"], p
    if config == "long16":    # strong scaling: the two shards tile the stream's outputs
        assert p["n_outputs"] == (60000 - 16 + 1) * 1024
    else:                      # weak: every rank a full segment
        assert p["n_outputs"] == 2 * 30001 * 1024
