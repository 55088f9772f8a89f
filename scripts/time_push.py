"""Throughput of the incremental stream API (ppfg_stream_push) with 32 MiB pushes
from pageable numpy buffers (C=1024, T=8, EXACT), 2 GiB total."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1411_3656_b200 import ppf
C, T = 1024, 8
blk = 4096 * C * 8
x = ppf.synth(C, (2 << 30) // 8, seed=1).view(np.uint8)
with ppf.Plan(C, T, ppf.generate_prototype(C, T)) as p:
    for rep in range(2):
        s = ppf.Stream(p, block_spectra=4096)
        t0 = time.perf_counter()
        n = 0
        for o in range(0, x.size, blk):
            n += len(s.push(memoryview(x[o:o + blk])))
        s.close()
        t = time.perf_counter() - t0
    print({"push_gb_per_s_in": round(x.size / t / 1e9, 2), "out_bytes": n})
