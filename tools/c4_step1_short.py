"""Config 4 step 1 (8192^2, 8 strips, overlap 32), one outer sweep x `inner` Alg. 5 updates after
a warm-up call: per-family device times.  Used for A/B runs and ncu captures of the chirp-z
kernels.  Usage: python tools/c4_step1_short.py [inner] [config, default c4] [step1|step2]
(step2: one sweep of `inner` Alg. 3 updates on tau = P tau_0)"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2602_17494_b200 as pkg  # noqa: E402
from tvs_synth import CONFIGS  # noqa: E402

inner = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c = CONFIGS[sys.argv[2] if len(sys.argv) > 2 else "c4"]
img = c.image()
ctx = pkg.Context(0)
d0 = torch.from_numpy(img).cuda()
L = (c.m2, c.m1, c.overlap, c.overlap)
step = sys.argv[3] if len(sys.argv) > 3 else "step1"
if step == "step2":
    tau1, _, _ = ctx.tv_stokes_step1(d0, c.delta, L, (1, 0, c.t))
    run = lambda it: ctx.tv_stokes_step2(tau1, d0, c.lam, L, (1, it, c.t))
else:
    run = lambda it: ctx.tv_stokes_step1(d0, c.delta, L, (1, it, c.t))
run(1)
torch.cuda.synchronize()
_, _, st0 = run(inner)   # unprofiled (device time)
ctx.set_profiling(True)
ctx.reset_kernel_times()
tau, _, st = run(inner)
ctx.set_profiling(False)
kt = ctx.kernel_times()
fam = {nm: {"n": kt.counts[i], "avg_us": round(kt.ms[i] / kt.counts[i] * 1e3, 1),
            **({"tflops": round(kt.flops[i] / (kt.ms[i] / 1e3) / 1e12, 2)} if kt.flops[i] else {})}
       for i, nm in enumerate(pkg.KERNEL_FAMILIES) if kt.counts[i]}
tau_hash = int(tau.contiguous().view(torch.int32).to(torch.int64).sum())   # bitwise A/B check
print(json.dumps({"inner": inner, "seconds": st0.seconds, "seconds_profiled": st.seconds, "E1": st.primal_energy,
                  "tau_hash": tau_hash,
                  "env": {k: v for k, v in os.environ.items() if k.startswith("TVS_")}, "families": fam}))
