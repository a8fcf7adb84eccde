"""Config 5 at full size (32768^2, 16 x 16 subdomains, overlap 32) step 1 on ONE GPU: one outer
sweep with `inner` Alg. 5 updates (subdomain groups sized to the free HBM), device memory and
time.  Usage: python tools/c5_step1_probe.py [inner]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2602_17494_b200 as pkg  # noqa: E402
from tvs_synth import CONFIGS  # noqa: E402

inner = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c = CONFIGS["c5"]
t0 = time.time()
img = c.image()
print(f"image {time.time() - t0:.1f} s", flush=True)
ctx = pkg.Context(0)
d0 = torch.from_numpy(img).cuda()
del img
L = (c.m2, c.m1, c.overlap, c.overlap)
free0, tot = torch.cuda.mem_get_info()
t0 = time.time()
tau, p, st = ctx.tv_stokes_step1(d0, c.delta, L, (1, inner, c.t))
torch.cuda.synchronize()
wall = time.time() - t0
free1, _ = torch.cuda.mem_get_info()
ctx.set_profiling(True)
ctx.reset_kernel_times()
tau, p, st2 = ctx.tv_stokes_step1(d0, c.delta, L, (1, inner, c.t))
ctx.set_profiling(False)
kt = ctx.kernel_times()
fam = {nm: [kt.counts[i], round(kt.ms[i], 1)] for i, nm in enumerate(pkg.KERNEL_FAMILIES) if kt.counts[i]}
print(json.dumps({"inner": inner, "first_call_wall_s": round(wall, 1), "seconds": st2.seconds,
                  "pixel_updates": st2.pixel_updates, "launches": st2.launches,
                  "free_before_GB": free0 / 1e9, "free_after_GB": free1 / 1e9, "total_GB": tot / 1e9,
                  "E1": st2.primal_energy, "gap": st2.gap, "families_ms": fam,
                  "tau_finite": bool(torch.isfinite(tau).all())}), flush=True)
