"""The N>1 path on CPU: world_size-2 gloo ranks each take their contiguous
output range plus the (T-1)-spectrum halo (ppfg_shard_range), compute it (with
the oracle here, since this host has no GPU), and the gathered shards equal the
one-shot result bit for bit. Also exercises bench.py's max-over-ranks timing
reduction on the same process group. No data-path collective is involved."""
import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port_no, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port_no)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle
    from paper_1411_3656_b200 import ppf
    import bench
    C, T, S = 256, 8, 403
    x = ppf.synth(C, S * C, seed=77).reshape(S, C)
    coeffs = oracle.port().generate_prototype(C, T, 9.0)
    ib, ic, ob, oc = ppf.shard_range(S, T, rank, world)
    part = oracle.port().fir_fft(x[ib:ib + ic], C, T, coeffs)
    parts = [None] * world
    dist.all_gather_object(parts, (ob, oc, part))
    t = bench.max_over_ranks(0.5 + rank)
    if rank == 0:
        parts.sort(key=lambda p: p[0])
        got = np.concatenate([p[2] for p in parts])
        want = oracle.port().fir_fft(x, C, T, coeffs)
        q.put((bool(np.array_equal(got.view(np.uint32), want.view(np.uint32))),
               [p[:2] for p in parts], t))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shards_reassemble():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_no = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port_no, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok, ranges, t = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ok
    assert ranges == [(0, 198), (198, 198)]
    assert t == 1.5
