#!/usr/bin/env python3
"""Benchmark of the TV-Stokes overlapping-Schwarz dual iteration on B200.

One *step* = one full pass of the hot path: tv_stokes_denoise =
step 1 (TFS, Alg. 2 + Alg. 5) then step 2 (IRV2, Alg. 2 + Alg. 3) on BASELINE config 4 by
default (8192 x 8192 Voronoi-1024 image, 8 horizontal strips, overlap 32, 30 sweeps x 20 inner per
step): the largest BASELINE configuration that runs on one GPU and the one the north star's HBM
and 8-GPU strong-scaling targets are quoted on.

metric: dual pixel-updates/s (sum over subdomains of |Gamma_m| per inner update, overlap counted
per subdomain, both steps), whole job over all ranks.  `value` is device-timed with the input
resident in HBM; `e2e` is the same metric through the host-buffer C-ABI call
tv_stokes_denoise_host (H2D of d0 and D2H of d inside the timed region).

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
       [--workload c1|c2|c3|c4|c5w1]
With --gpus N > 1 and no WORLD_SIZE in the environment, bench.py launches itself under
torch.distributed.run (one process per GPU, NCCL); under torchrun it runs as one rank.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from tvs_synth import CONFIGS  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
# FP32 SIMT peak: 148 SMs x 128 FP32 lanes x 2 flop x 1.965 GHz
FP32_SIMT_PEAK_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12
FALLBACK_HBM_GBS = 6650.0


def measured_peaks():
    try:
        with open(PEAKS_PATH) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": FALLBACK_HBM_GBS}, "fallback"


def workload(name):
    c = CONFIGS[name]
    return c, (c.m2, c.m1, c.overlap, c.overlap), (c.sweeps, c.inner, c.t)


def sum_sub(n, L, extended):
    from paper_2602_17494_b200 import layout_range
    m2, m1, sy, sx = L
    ys = [layout_range(n + 1, m2, sy, k) for k in range(m2)]
    xs = [layout_range(n + 1, m1, sx, k) for k in range(m1)]
    lim = n if extended else n - 1
    return sum((min(b, lim) - a + 1) for a, b in ys) * sum((min(b, lim) - a + 1) for a, b in xs)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region (B200_PROFILING.md)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4)
                          if len(r) > 5 + k and r[5 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def flush_l2(buf):
    buf.add_(1.0)   # 256 MB write > 126 MB L2


# ----------------------------------------------------------------------------- our arm

def run_ours(args, rank, world, local_rank):
    import torch
    import paper_2602_17494_b200 as pkg

    c, L, it = workload(args.workload)
    img = c.image()
    aux = (not args.no_aux) and world == 1
    aux_c3_img = CONFIGS["c3"].image() if aux and c.name != "c3" else None   # before CUDA init
    aux5_img = CONFIGS["c5w1"].image() if aux else None
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        # one process per GPU: the library owns an NCCL communicator (band send/recv per sweep,
        # all-gathers of partial x-DCT rows and of the outputs); rank 0 creates the unique id
        obj = [pkg.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctx = pkg.Context(local_rank, rank, world, obj[0])
    else:
        ctx = pkg.Context(local_rank)
    stream = torch.cuda.current_stream()
    d0 = torch.from_numpy(img).cuda()
    out = torch.empty_like(d0)
    flush = torch.empty(64 * 1024 * 1024, device="cuda", dtype=torch.float32)
    n = c.n
    upd_step = (sum_sub(n, L, True) + sum_sub(n, L, False)) * it[0] * it[1]

    def step():
        return ctx.tv_stokes_denoise(d0, c.delta, c.lam, L, it, it, out=out)

    for _ in range(args.warmup):
        flush_l2(flush)
        step()
    torch.cuda.synchronize()
    # ---- timed region: K steps, device events on the launching stream, L2 flushed between steps
    # per-kernel CUDA events (the roofline's per-launch times) on the first timed step only
    ctx.reset_kernel_times()
    launches = 0
    step_ms = []
    stats = None
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local_rank) as clk:
        for k in range(args.steps):
            ctx.set_profiling(k == 0)
            flush_l2(flush)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            _, _, s1, s2 = step()
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            launches += s1.launches + s2.launches
            stats = (s1, s2)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ctx.set_profiling(False)
    kt = ctx.kernel_times()
    profiled_ms = step_ms[0]
    total_ms = sum(step_ms)
    if dist:
        t = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = upd_step * args.steps / (total_ms / 1e3)      # strong scaling: the job's updates

    # ---- e2e: same metric through the host-buffer C-ABI call (H2D of d0 + D2H of d inside)
    h_in = torch.from_numpy(img).pin_memory()
    h_out = torch.empty_like(h_in).pin_memory()
    e2e_ms = []
    for _ in range(max(1, min(args.steps, 3))):
        flush_l2(flush)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        ctx.tv_stokes_denoise_host(h_in.numpy(), c.delta, c.lam, L, it, it, out=h_out.numpy())
        e1.record(stream)
        e1.synchronize()
        e2e_ms.append(e0.elapsed_time(e1))
    e2e_t = statistics.median(e2e_ms)
    if dist:
        t = torch.tensor([e2e_t], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_t = float(t.item())

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    peaks, peak_src = measured_peaks()
    names = pkg.KERNEL_FAMILIES
    kern = {}
    for i, nm in enumerate(names):
        if kt.counts[i] == 0:
            continue
        avg = kt.ms[i] / kt.counts[i]
        entry = {"launches": kt.counts[i], "avg_us": round(avg * 1e3, 3),
                 "share": round(kt.ms[i] / max(profiled_ms, 1e-9), 4)}
        if kt.flops[i] > 0:
            entry["tflops"] = round(kt.flops[i] / (kt.ms[i] / 1e3) / 1e12, 3)
        if kt.bytes[i] > 0:
            entry["gbs"] = round(kt.bytes[i] / (kt.ms[i] / 1e3) / 1e9, 1)
        kern[nm] = entry
    roof = roofline(kt, names, peaks, peak_src, c.name)
    s1, s2 = stats
    line = {
        "metric": "dual pixel-updates/s (step 1 + step 2, overlap counted per subdomain)",
        "value": value, "unit": "pixel-updates/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None, "dtype": "f32 (fp64 y-solves and reductions)", "data": "synthetic",
        "config": bench_config(c, world, upd_step),
        "gpu_launches": launches,
        "e2e": {"value": upd_step / (e2e_t / 1e3), "unit": "pixel-updates/s",
                "h2d_bytes_per_step": int(img.nbytes), "d2h_bytes_per_step": int(img.nbytes),
                "ms_per_step": e2e_t},
        "roofline": roof,
        "kernels": kern,
        "step_seconds": {"step1": round(s1.seconds, 4), "step2": round(s2.seconds, 4)},
        "energies": {"E1": s1.primal_energy, "gap1": s1.gap, "D1": s1.dual_energy,
                     "E2": s2.primal_energy, "gap2": s2.gap, "D2": s2.dual_energy},
        "clocks": clk.summary(),
    }
    if aux:
        line["aux_kernel_a_c4"] = aux_kernel_a(ctx, pkg, img if c.name == "c4" else CONFIGS["c4"].image(),
                                               peaks, peak_src, flush)
        if aux_c3_img is not None:
            line["aux_c3"] = aux_c3(ctx, pkg, aux_c3_img, flush)
        line["aux_c5w1"] = aux_c5w1(ctx, pkg, aux5_img, flush)
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(c, L, it)
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def roofline(kt, names, peaks, peak_src, workload_name):
    """Roofline of the dominant kernel family (largest share of the profiled step's device time):
    chirp-z FFT pairs against the FP32 SIMT peak (method flops 2 x 5 M log2 M per FFT pair),
    the tcgen05 3xTF32 GEMMs against the tf32 tensor peak / 3, stencils against measured HBM."""
    dom = max(range(len(kt.ms)), key=lambda i: kt.ms[i])
    nm = names[dom]
    sec = kt.ms[dom] / 1e3
    if nm.endswith("_czt"):
        ach = kt.flops[dom] / sec / 1e12
        roof = {"bound": "alu", "achieved": round(ach, 3), "peak": round(FP32_SIMT_PEAK_TFLOPS, 1),
                "unit": "TFLOP/s", "frac": round(ach / FP32_SIMT_PEAK_TFLOPS, 4),
                "peak_source": "FP32 SIMT: 148 SM x 128 FP32 lanes x 2 flop x 1.965 GHz "
                               "(B200_PROFILING.md SM count and clocks.max.sm; DESIGN.md section 5)",
                "work": "FFT flops of the chirp-z form: 2 x 5 M log2 M per (row, pass, chunk), "
                        "M = 16384 at config 4"}
    elif kt.flops[dom] > 0:
        tf32 = peaks.get("bf16_tflops", 1590.0) * (1.1 / 2.25)
        pk = tf32 / 3.0
        ach = kt.flops[dom] / sec / 1e12
        roof = {"bound": "tensor", "achieved": round(ach, 3), "peak": round(pk, 1),
                "unit": "TFLOP/s", "frac": round(ach / pk, 4),
                "peak_source": f"tf32 = bf16_tflops ({peak_src}) x 1.1/2.25 = {tf32:.0f}; fp32-equivalent "
                               "of 3xTF32 = tf32/3; achieved counts algorithmic fp32 flops 2MNK"}
    else:
        ach = kt.bytes[dom] / sec / 1e9
        roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": round(ach / peaks["hbm_gbs"], 4),
                "peak_source": f"hbm_gbs ({peak_src}) MEASURED_PEAKS.json"}
    roof["kernel"] = nm
    roof["avg_us"] = round(kt.ms[dom] / kt.counts[dom] * 1e3, 2)
    roof["traffic"], roof["traffic_source"] = ncu_traffic(workload_name, nm)
    return roof


def ncu_traffic(workload, family):
    """DRAM bytes (read + write) per launch of the dominant kernel family, from the committed
    `ncu --set full` capture summarised in profiles/ncu_traffic.json (one launch of the local
    projection batch of this workload); None when no capture of that family exists."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f)[workload][family]
        return t["dram_bytes"], t["source"]
    except Exception:
        return None, None


def aux_kernel_a(ctx, pkg, img, peaks, peak_src, flush):
    """Kernel (a) in the HBM-bound regime the north-star's >=70 % target refers to: config-4
    step 2 (8192^2, 8 horizontal strips, overlap 32, 30 x 20), tau = 0 (the sweep's work and
    traffic are data-independent).  Algorithmic traffic: 20 B per point per pass (v read 8,
    omega0 4, v write 8).  Reported twice: the default two-updates-per-pass kernel (temporal
    blocking, 10 B per update) and the single-update kernel (TVS_SWEEP2X2=0, 20 B per update)."""
    import torch
    c4 = CONFIGS["c4"]
    L4, it4 = (c4.m2, c4.m1, c4.overlap, c4.overlap), (c4.sweeps, c4.inner, c4.t)
    d0 = torch.from_numpy(img).cuda()
    tau = torch.zeros((2, c4.n + 1, c4.n + 1), device="cuda", dtype=torch.float32)

    def measure(cx):
        cx.tv_stokes_step2(tau, d0, c4.lam, L4, it4)          # warm-up (plan build)
        flush_l2(flush)
        torch.cuda.synchronize()
        cx.reset_kernel_times()
        cx.set_profiling(True)
        _, _, st = cx.tv_stokes_step2(tau, d0, c4.lam, L4, it4)
        cx.set_profiling(False)
        kt = cx.kernel_times()
        i = pkg.KERNEL_FAMILIES.index("sweep2")
        gbs = kt.bytes[i] / (kt.ms[i] / 1e3) / 1e9
        per_pass = st.pixel_updates / max(1, kt.counts[i] * sum_sub(c4.n, L4, False))   # 1 or 2
        return {"achieved": round(gbs, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": round(gbs / peaks["hbm_gbs"], 4), "frac_of_8TBs": round(gbs / 8000.0, 4),
                "avg_us": round(kt.ms[i] / kt.counts[i] * 1e3, 2), "launches": kt.counts[i],
                "updates_per_pass": round(per_pass, 3), "bytes_per_update": round(20 / per_pass, 2),
                "step2_pixel_updates_per_s": st.pixel_updates / st.seconds}

    out = {"workload": "c4 step 2: 8192x8192, 8 strips, overlap 32, 30x20, tau = 0",
           "kernel": "sweep2 (kernel a)", "bound": "hbm", "peak_source": f"hbm_gbs ({peak_src})"}
    out.update(measure(ctx))
    old = os.environ.get("TVS_SWEEP2X2")
    os.environ["TVS_SWEEP2X2"] = "0"
    try:
        single = pkg.Context(torch.cuda.current_device())
    finally:
        if old is None:
            del os.environ["TVS_SWEEP2X2"]
        else:
            os.environ["TVS_SWEEP2X2"] = old
    out["single_update_per_pass"] = measure(single)
    single.close()
    return out


def aux_c3(ctx, pkg, img, flush):
    """Config 3 (2048^2 Voronoi-64, 8 x 8 subdomains, overlap 16, 50 x 10 per step, both steps):
    the round-1 headline, now auxiliary -- its tiles are short, so the dense tcgen05 GEMM form of
    the partial x-DCTs runs there.  Device time of two denoise calls after
    a warm-up, L2 flushed before each; rate in dual pixel-updates/s."""
    import torch
    c, L, it = workload("c3")
    d0 = torch.from_numpy(img).cuda()
    upd = (sum_sub(c.n, L, True) + sum_sub(c.n, L, False)) * it[0] * it[1]
    ctx.tv_stokes_denoise(d0, c.delta, c.lam, L, it, it)
    secs = []
    for _ in range(2):
        flush_l2(flush)
        torch.cuda.synchronize()
        _, _, s1, s2 = ctx.tv_stokes_denoise(d0, c.delta, c.lam, L, it, it)
        secs.append(s1.seconds + s2.seconds)
    t = min(secs)
    return {"workload": "c3: 2048x2048 Voronoi-64, 8x8 subdomains, overlap 16, 50x10 per step",
            "ms_per_step": round(t * 1e3, 2), "pixel_updates_per_s": upd / t,
            "dct": "dense tcgen05 3xTF32 GEMM (local tiles), chirp-z (global projection)"}


def aux_c5w1(ctx, pkg, img, flush):
    """Config 5 at its one-GPU weak-scaling size (11585^2, 16 x 16 subdomains, s = 32): step 2
    over the full 20 x 10 schedule and one outer sweep of step 1 (10 Alg. 5 updates, chirp-z
    x-DCTs), each after a warm-up call; rates in dual pixel-updates/s."""
    import torch
    c = CONFIGS["c5w1"]
    L = (c.m2, c.m1, c.overlap, c.overlap)
    d0 = torch.from_numpy(img).cuda()
    tau = torch.zeros((2, c.n + 1, c.n + 1), device="cuda", dtype=torch.float32)
    ctx.tv_stokes_step2(tau, d0, c.lam, L, (1, 2, c.t))
    flush_l2(flush)
    _, _, s2 = ctx.tv_stokes_step2(tau, d0, c.lam, L, (c.sweeps, c.inner, c.t))
    ctx.tv_stokes_step1(d0, c.delta, L, (1, 1, c.t))
    flush_l2(flush)
    _, _, s1 = ctx.tv_stokes_step1(d0, c.delta, L, (1, c.inner, c.t))
    return {"workload": "c5 weak-scaling base: 11585x11585, 16x16 subdomains, overlap 32",
            "step2_20x10": {"seconds": round(s2.seconds, 3), "pixel_updates": s2.pixel_updates,
                            "pixel_updates_per_s": s2.pixel_updates / s2.seconds},
            "step1_1x10": {"seconds": round(s1.seconds, 3), "pixel_updates": s1.pixel_updates,
                           "pixel_updates_per_s": s1.pixel_updates / s1.seconds},
            "dct": "chirp-z (N = 11586 > 4096)"}


# ----------------------------------------------------------------------------- oracle (CPU)

def _blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max([p.get("num_threads", 1) for p in threadpool_info()] + [1])
    except Exception:
        return os.cpu_count() or 1


def oracle_sample(c, L, it):
    """Time the fp64 oracle (as it stands) on a bounded sample of the workload and extrapolate the
    full step by operation counts.  Pieces (each an oracle call on the real sizes):
      (1) step 2: one inner update of Alg. 3 on every subdomain (irv2_local_iterations), one task
          per subdomain on the oracle's threads (solvers.map_subdomains) -- the wall time;
      (2) step 1, local: one literal local projection R_{S+} P E_{S+} w of subdomain 0
          (solvers.local_projection: the block-DCT sum of Eq. invLaplLowCapLong); an Alg. 5 update
          applies it once, omega0 once per sweep (the update's stencils are not counted);
      (3) step 1, global: one of the four N~ x N~ x N~ DCT products of the global Delta^dagger
          (spectral.lap_pinv) on a 1/8 row slab; one global projection = 4 x 8 x that.
    Full step = step 2: sweeps x inner x (1); step 1: sweeps x (inner + 1) x M x (2) +
    (sweeps + 2) x (3), where (2) ran on all cores (BLAS threads), i.e. the same throughput as the
    threaded sweep with one core per subdomain.  Returns (rate, description, sample seconds, threads, step s)."""
    from oracle import layout as olayout, solvers as S, spectral
    img = c.image().astype(np.float64)
    n = c.n
    lay = olayout.Layout(n, n, *L)
    subs = lay.subdomains()
    M = len(subs)
    workers = min(M, os.cpu_count() or 1)
    sweeps, inner, t = it
    # (1) step 2, one inner update on every subdomain (f from tau = 0: the work is data-independent)
    _, _, f = S.irv2_data(img, np.zeros((2, n + 1, n + 1)), c.lam)

    def upd2(m):
        s = lay.rect(m, extended=False)
        omega0 = S.restrict(f, S.full_rect(n, n), S.rect_plus(s, n, n))
        return S.irv2_local_iterations(lay, m, omega0, np.zeros((2,) + S.rect_shape(s)), 1, t)

    t0 = time.perf_counter()
    S.map_subdomains(upd2, subs, workers)
    t_upd2 = time.perf_counter() - t0
    del f
    # (2) step 1: one literal local projection R_{S+} P E_{S+} w of subdomain 0 (the operator an
    # Alg. 5 update applies once; the DCT matrices are built and cached by the oracle first)
    n2t = n1t = n + 1
    cy, cx = spectral.cut_points(n2t, lay.m2), spectral.cut_points(n1t, lay.m1)
    spectral.dct_matrix(n2t), spectral.dct_matrix(n1t)
    sp0 = S.rect_plus(lay.rect(subs[0], True), n2t, n1t)
    w = np.random.default_rng(5).standard_normal((2,) + S.rect_shape(sp0))
    t0 = time.perf_counter()
    S.local_projection(w, sp0, n2t, n1t, cy, cx)
    t_lp = time.perf_counter() - t0
    del w
    # (3) step 1, global: one DCT product on a 1/8 row slab
    cmat = spectral.dct_matrix(n1t)
    slab = np.random.default_rng(6).standard_normal((max(1, n2t // 8), n1t))
    t0 = time.perf_counter()
    slab @ cmat.T
    t_prod = time.perf_counter() - t0
    t_global = 4 * 8 * t_prod
    del cmat, slab
    spectral._DCT_CACHE.clear()
    step2_s = sweeps * inner * t_upd2
    step1_s = sweeps * (inner + 1) * M * t_lp + (sweeps + 2) * t_global
    u1 = sum((b - a + 1) for a, b in lay.ry) * sum((b - a + 1) for a, b in lay.rx) * sweeps * inner
    u2 = (sum((min(b, n - 1) - a + 1) for a, b in lay.ry) *
          sum((min(b, n - 1) - a + 1) for a, b in lay.rx) * sweeps * inner)
    rate = (u1 + u2) / (step1_s + step2_s)
    secs = t_upd2 + t_lp + t_prod
    desc = (f"{c.name}: (1) one Alg.3 inner update on all {M} subdomains, {workers} threads "
            f"({t_upd2:.2f} s); (2) one literal block-DCT local projection of subdomain 0 "
            f"({t_lp:.2f} s); (3) one 1/8-slab DCT product of the global "
            f"projection ({t_prod:.2f} s); extrapolated by operation count to the full "
            f"{sweeps}x{inner} schedule of both steps: step 1 {step1_s:.0f} s, step 2 {step2_s:.0f} s")
    threads = {"subdomain_threads": workers, "blas_threads": _blas_threads()}
    return rate, desc, secs, threads, step1_s + step2_s


def cpu_baseline(c, L, it):
    rate, desc, secs, threads, step_s = oracle_sample(c, L, it)
    return {"value": rate, "unit": "pixel-updates/s", "cores": max(threads.values()),
            "threads": threads, "kind": "oracle", "sample": desc, "sample_seconds": round(secs, 1),
            "extrapolated_step_seconds": round(step_s, 1), "cpu": _cpu_model(),
            "nproc": os.cpu_count()}


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def bench_config(c, world, upd_step):
    """The `config` object of both arms (same workload description)."""
    return {"workload": f"{c.name}: {c.n}x{c.n} Voronoi-{c.cells}, {c.m2}x{c.m1} subdomains, "
                        f"overlap {c.overlap}, {c.sweeps}x{c.inner} per step, delta {c.delta}, "
                        f"lambda {c.lam}, t {c.t}",
            "pixel_updates_per_step": upd_step,
            "l2": ("inputs larger than L2 (config-4 working set about 3 GB) and L2 flushed (256 MB "
                   "write) between steps" if c.n >= 8192 else "flushed (256 MB write) between steps"),
            "parallelism": f"slab decomposition over {world} GPUs (NCCL)" if world > 1 else "1 GPU"}


def _oracle_updates(c):
    """Dual pixel-updates per step counted with the oracle's layout (reference arm only)."""
    from oracle.layout import ranges_1d
    ys, xs = ranges_1d(c.n + 1, c.m2, c.overlap), ranges_1d(c.n + 1, c.m1, c.overlap)
    tot = 0
    for lim in (c.n, c.n - 1):   # Omega~ (step 1), Omega (step 2)
        tot += sum(min(b, lim) - a + 1 for a, b in ys) * sum(min(b, lim) - a + 1 for a, b in xs)
    return tot * c.sweeps * c.inner


def run_reference(args, rank, world):
    """Reference arm: the fp64 oracle (there is no installable reference implementation --
    /root/reference is a paper), timed as it stands on the host cores on a bounded sample of the
    same workload per step (oracle_sample); ms_per_step is the extrapolated full step."""
    if rank != 0:
        return
    c, L, it = workload(args.workload)
    for _ in range(args.warmup):
        oracle_sample(c, L, it)
    steps_s, secs = [], 0.0
    for _ in range(args.steps):
        r, desc, s, threads, step_s = oracle_sample(c, L, it)
        steps_s.append(step_s)
        secs += s
    step_s = statistics.median(steps_s)
    upd = _oracle_updates(c)
    value = upd / step_s
    line = {
        "impl": "reference", "metric": "dual pixel-updates/s (step 1 + step 2, overlap counted per subdomain)",
        "value": value, "unit": "pixel-updates/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * step_s, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(c, world, upd),
        "cpu_baseline": {"value": value, "unit": "pixel-updates/s", "cores": max(threads.values()),
                         "threads": threads, "kind": "oracle", "sample": desc,
                         "sample_seconds_per_step": round(secs / args.steps, 1),
                         "cpu": _cpu_model(), "nproc": os.cpu_count()},
        "e2e": {"value": value, "unit": "pixel-updates/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def launch_self(args):
    """--gpus N > 1 outside torchrun: relaunch this script under torch.distributed.run, one process
    per GPU (rendezvous on 127.0.0.1), and pass its output through."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c4", choices=["c1", "c2", "c3", "c4", "c5w1"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-aux", action="store_true", help="skip the auxiliary measurements")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(launch_self(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
