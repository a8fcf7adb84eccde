"""The paper's DD-vs-non-DD energy protocol (section 6.3, Fig. 7) on the GPU, with the
synthetic stand-in for Image 10 (tvs_synth.ellipses_rect: 270 x 480, sigma = 0.1).

* reference (non-DD): one subdomain (layout 1 x 1, Schwarz 1 x 1 = Chambolle, C-8), 1e6 iterations
  per step: TFS (delta 0.15), then IRV1 (mu 0.1, eps 1e-3) and IRV2 (alpha 10) on its tau;
* DD: 3 x 3 subdomains, overlaps 4 (y) / 3 (x) (alpha_hat = 1/4), 10 inner x at most 5000 outer
  sweeps, stopping when |D(p^n)^2 - D(p^{n+1})^2| / |Gamma| < 1e-10 (criterion 2, tvs_set_stopping);
  step 2 fed the DD tau (solid curves of Fig. 7 b/c) and the reference tau (dashed);
* every DD iterate's energy from the library's per-sweep trace (tvs_set_trace).
Writes a JSON with the reference energies and E_DD(n) - E_ref at log-spaced n.
Usage: python tools/fig7_protocol.py out.json [ref_iters]"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2602_17494_b200 as pkg  # noqa: E402
from tvs_synth import ellipses_rect  # noqa: E402

out_path = sys.argv[1] if len(sys.argv) > 1 else "fig7.json"
ref_iters = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
img = ellipses_rect()
n2, n1 = img.shape
d0 = torch.from_numpy(img).cuda()
delta, mu, alpha, eps, t = 0.15, 0.1, 10.0, 1e-3, 0.125
ONE = (1, 1, 0, 0)
DD = (3, 3, 4, 3)
ctx = pkg.Context(0)
res = {"image": "tvs_synth.ellipses_rect(270, 480, seed 1010, sigma 0.1)", "layout_dd": DD,
       "delta": delta, "mu": mu, "alpha": alpha, "epsilon": eps, "t": t, "ref_iters": ref_iters}

t0 = time.time()
tau_ref, _, s = ctx.tv_stokes_step1(d0, delta, ONE, (1, ref_iters, t))
res["ref"] = {"tfs": {"E": s.primal_energy, "gap": s.gap, "D": s.dual_energy}}
_, _, s = ctx.tv_stokes_step2(tau_ref, d0, mu, ONE, (1, ref_iters, t), variant="irv1", eps=eps)
res["ref"]["irv1"] = {"E": s.primal_energy, "gap": s.gap, "D": s.dual_energy}
_, _, s = ctx.tv_stokes_step2(tau_ref, d0, 1.0 / alpha, ONE, (1, ref_iters, t))
res["ref"]["irv2"] = {"E": s.primal_energy, "gap": s.gap, "D": s.dual_energy}
res["ref_seconds"] = time.time() - t0


def curve(trace, e_ref):
    n = trace.shape[0]
    idx = sorted(set([0, 1, 2, 5, n - 1] + [int(round(x)) for x in np.geomspace(1, max(n - 1, 1), 60)]))
    return {"n": idx, "E": [float(trace[k, 0]) for k in idx],
            "E_minus_Eref": [float(trace[k, 0] - e_ref) for k in idx],
            "gap": [float(trace[k, 2]) for k in idx], "sweeps_run": n - 1}


ctx.set_stopping(2, 1e-10)
ctx.set_trace(5001)
tau_dd, _, s = ctx.tv_stokes_step1(d0, delta, DD, (5000, 10, t))
res["dd_tfs"] = curve(ctx.trace(), res["ref"]["tfs"]["E"])
for name, tau, tag in (("dd_tau", tau_dd, "solid"), ("ref_tau", tau_ref, "dashed")):
    _, _, s = ctx.tv_stokes_step2(tau, d0, mu, DD, (5000, 10, t), variant="irv1", eps=eps)
    res[f"irv1_{name}"] = curve(ctx.trace(), res["ref"]["irv1"]["E"]) | {"fig7_line": tag}
    _, _, s = ctx.tv_stokes_step2(tau, d0, 1.0 / alpha, DD, (5000, 10, t))
    res[f"irv2_{name}"] = curve(ctx.trace(), res["ref"]["irv2"]["E"]) | {"fig7_line": tag}
ctx.set_trace(0)
ctx.set_stopping(0, 0.0)
res["tau_dd_vs_ref_maxabs"] = float((tau_dd - tau_ref).abs().max())
res["seconds"] = time.time() - t0
summary = {k: {"sweeps": v["sweeps_run"], "final_rel": v["E_minus_Eref"][-1] / abs(res["ref"][k.split("_")[0].replace("dd", "tfs")]["E"])}
           for k, v in res.items() if isinstance(v, dict) and "E_minus_Eref" in v}
res["summary"] = summary
json.dump(res, open(out_path, "w"), indent=1)
print(json.dumps(summary, indent=1))
