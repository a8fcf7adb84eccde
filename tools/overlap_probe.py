"""How much do two independent config-4 step-1 chains overlap on one GPU?  Runs the same short
step 1 (1 sweep x `inner` updates) on two contexts, first one after the other, then concurrently on
two streams from two host threads.  Usage: python tools/overlap_probe.py [inner]"""
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2602_17494_b200 as pkg  # noqa: E402
from tvs_synth import CONFIGS  # noqa: E402

inner = int(sys.argv[1]) if len(sys.argv) > 1 else 4
c = CONFIGS["c4"]
img = c.image()
L = (c.m2, c.m1, c.overlap, c.overlap)
cx = [pkg.Context(0), pkg.Context(0)]
d0 = torch.from_numpy(img).cuda()
st = [torch.cuda.Stream(), torch.cuda.Stream()]
for k in range(2):
    cx[k].tv_stokes_step1(d0, c.delta, L, (1, 1, c.t), stream=st[k])
torch.cuda.synchronize()


def one(k):
    with torch.cuda.stream(st[k]):
        cx[k].tv_stokes_step1(d0, c.delta, L, (1, inner, c.t), stream=st[k])


t0 = time.time()
one(0)
one(1)
torch.cuda.synchronize()
seq = time.time() - t0
t0 = time.time()
th = [threading.Thread(target=one, args=(k,)) for k in range(2)]
for t in th:
    t.start()
for t in th:
    t.join()
torch.cuda.synchronize()
par = time.time() - t0
print(f"inner {inner}: sequential {seq * 1e3:.1f} ms, concurrent {par * 1e3:.1f} ms, ratio {par / seq:.3f}")
