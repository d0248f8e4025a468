"""H2D DMA time of a 16 MB pinned buffer: right after the CPU wrote it, after
an idle gap, and back to back (is a staged chunk's DMA slower than a DMA of an
untouched pinned buffer?)."""
import time
import numpy as np
import torch

n = 16 << 20
src = np.random.default_rng(0).random(n // 4, dtype=np.float32)
pin = torch.empty(n // 4, dtype=torch.float32, pin_memory=True)
dst = torch.empty(n // 4, dtype=torch.float32, device="cuda")
s = torch.cuda.Stream()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def dma():
    with torch.cuda.stream(s):
        e0.record(s); dst.copy_(pin, non_blocking=True); e1.record(s)
    s.synchronize()
    return e0.elapsed_time(e1)


for _ in range(3):
    dma()
print("back to back    ", ["%.3f" % dma() for _ in range(5)])
out = []
for _ in range(5):
    time.sleep(0.01); out.append(dma())
print("after 10 ms idle", ["%.3f" % x for x in out])
out = []
for _ in range(5):
    pin.numpy()[:] = src; out.append(dma())
print("after CPU write ", ["%.3f" % x for x in out])
out = []
for _ in range(5):
    time.sleep(0.005); pin.numpy()[:] = src; out.append(dma())
print("idle + CPU write", ["%.3f" % x for x in out])
