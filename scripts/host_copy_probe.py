"""Single-thread host memcpy rate on the GPU box (the bound for process_stream's
reader/writer threads, which copy istream -> pinned slot and pinned slot -> ostream)."""
import time, json
import numpy as np
import torch
n = 1 << 30
src = np.ones(n, dtype=np.uint8)
pin = torch.empty(n, dtype=torch.uint8, pin_memory=True).numpy()
dst = np.empty(n, dtype=np.uint8)
r = {}
for name, a, b in (("pageable->pinned", src, pin), ("pinned->pageable", pin, dst), ("pageable->pageable", src, dst)):
    np.copyto(b, a)
    t = time.perf_counter()
    for _ in range(3):
        np.copyto(b, a)
    r[name] = round(3 * n / (time.perf_counter() - t) / 1e9, 2)
print(json.dumps({"single_thread_memcpy_GBps": r}))
