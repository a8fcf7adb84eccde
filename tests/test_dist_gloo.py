"""Multi-rank host logic of the slab decomposition on CPU with gloo.

Each rank takes its rows from the library's own plan (tvs_dist_rows, host-only C-ABI), keeps
p valid only on its rows V (everything else is NaN-poisoned, so reading outside V fails the
test), runs the fp64 oracle's local solves for its own subdomains, exchanges the band partial
sums with its slab neighbours by send/recv, combines them in the same grouping as the CUDA
kernel (sum_ky of sum_kx), and -- for step 1 -- computes the global residual from its core rows'
partial x-DCT plus an all-gather.  The result must equal the single-process oracle.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import layout as olayout, ops, solvers as S, spectral
from tvs_synth import random_image


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _partial(lay, qhat, rows, k0, k1, n1, planes_shape, extended):
    """sum over local ky covering each row of sum_kx E qhat (rows [a, b))."""
    a, b = rows
    out = np.zeros(planes_shape + (max(b - a, 0), n1))
    for i in range(a, b):
        for ky in range(k0, k1):
            (y0, y1), _ = lay.rect((ky, 0), extended)
            if not (y0 <= i <= y1):
                continue
            part = np.zeros(planes_shape + (n1,))
            for kx in range(lay.m1):
                (y0, y1), (x0, x1) = lay.rect((ky, kx), extended)
                part[..., x0:x1 + 1] += qhat[(ky, kx)][..., i - y0, :]
            out[..., i - a, :] += part
    return out


def _exchange(pl, rank, world, send_up, send_dn, shape_up, shape_dn):
    recv_up = np.zeros(shape_up)
    recv_dn = np.zeros(shape_dn)
    ops_ = []
    if rank > 0:
        if send_up.size:
            ops_.append(dist.P2POp(dist.isend, torch.from_numpy(np.ascontiguousarray(send_up)), rank - 1))
        t_up = torch.zeros(shape_up, dtype=torch.float64)
        if t_up.numel():
            ops_.append(dist.P2POp(dist.irecv, t_up, rank - 1))
    if rank < world - 1:
        if send_dn.size:
            ops_.append(dist.P2POp(dist.isend, torch.from_numpy(np.ascontiguousarray(send_dn)), rank + 1))
        t_dn = torch.zeros(shape_dn, dtype=torch.float64)
        if t_dn.numel():
            ops_.append(dist.P2POp(dist.irecv, t_dn, rank + 1))
    if ops_:
        for r in dist.batch_isend_irecv(ops_):
            r.wait()
    if rank > 0 and np.prod(shape_up):
        recv_up = t_up.numpy()
    if rank < world - 1 and np.prod(shape_dn):
        recv_dn = t_dn.numpy()
    return recv_up, recv_dn


def _combine(lay, p, qhat, D, recv_up, recv_dn, extended, n1):
    """p^{n+1} on rows [V0, V1) with the remote parts, grouped sum_ky (sum_kx)."""
    out = p.copy()
    for i in range(D["V0"], D["V1"]):
        acc = np.zeros(p.shape[:-2] + (n1,))
        for ky in range(lay.m2):
            (y0, y1), _ = lay.rect((ky, 0), extended)
            if not (y0 <= i <= y1):
                continue
            if ky < D["k0"]:
                assert D["ur0"] <= i < D["ur1"]
                acc = acc + recv_up[..., i - D["ur0"], :]
            elif ky >= D["k1"]:
                assert D["dr0"] <= i < D["dr1"]
                acc = acc + recv_dn[..., i - D["dr0"], :]
            else:
                part = np.zeros(p.shape[:-2] + (n1,))
                for kx in range(lay.m1):
                    (yy0, yy1), (x0, x1) = lay.rect((ky, kx), extended)
                    part[..., x0:x1 + 1] += qhat[(ky, kx)][..., i - yy0, :]
                acc = acc + part
        out[..., i, :] = (1 - lay.alpha_hat) * p[..., i, :] + lay.alpha_hat * acc
    return out


def _poison(a, V0, V1):
    a = a.copy()
    a[..., :V0, :] = np.nan
    a[..., V1:, :] = np.nan
    return a


def _worker(rank, world, port, case, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2602_17494_b200 as pkg
        n2, n1, L, sweeps, inner = case
        img = random_image(n2, n1, 77).astype(np.float64)
        lay = olayout.Layout(n2, n1, *L)
        # ---------------- step 2 (IRV2) on Omega
        D = pkg.dist_rows(n2, n1, L, 2, rank, world)
        tau = S.chambolle_tfs(img, 0.05, 10)[0]
        alpha, g, f = S.irv2_data(img, tau, 0.1)
        p = np.zeros((2, n2, n1))
        qhat = {}
        for ky in range(D["k0"], D["k1"]):
            for kx in range(lay.m1):
                qhat[(ky, kx)] = np.zeros((2,) + S.rect_shape(lay.rect((ky, kx), False)))
        for _ in range(sweeps):
            pp = _poison(p, D["V0"], D["V1"])
            for m in list(qhat):
                qhat[m] = S._irv2_inner_local(m, lay, pp, f, qhat[m], inner, 0.125)
            assert all(np.isfinite(v).all() for v in qhat.values())
            su = _partial(lay, qhat, (D["us0"], D["us1"]), D["k0"], D["k1"], n1, (2,), False)
            sd = _partial(lay, qhat, (D["ds0"], D["ds1"]), D["k0"], D["k1"], n1, (2,), False)
            ru, rd = _exchange(None, rank, world, su, sd, (2, D["ur1"] - D["ur0"], n1),
                               (2, D["dr1"] - D["dr0"], n1))
            p = _combine(lay, pp, qhat, D, ru, rd, False, n1)
        d_ref, p_ref, _ = S.dd_step2(img, tau, 0.1, lay, sweeps, inner)
        core = slice(D["R0"], D["R1"])
        err2 = float(np.abs(p[:, core] - p_ref[:, core]).max())
        # ---------------- step 1 (TFS) on Omega~, global residual from core rows + all-gather
        n2t, n1t = n2 + 1, n1 + 1
        D1 = pkg.dist_rows(n2, n1, L, 1, rank, world)
        c1 = spectral.dct_matrix(n1t)

        def global_residual(p_valid, fpart):
            # w on [E0, V1) from p on [V0, V1); q on the core rows; partial x-DCT of the core rows
            w = ops.multidiv(np.nan_to_num(p_valid, nan=0.0))
            w_ok = np.full_like(w, np.nan)
            w_ok[..., D1["E0"]:D1["V1"], :] = w[..., D1["E0"]:D1["V1"], :]
            q = ops.div(np.nan_to_num(w_ok, nan=0.0))
            qc = q[D1["R0"]:D1["R1"]] @ c1.T
            parts = [None] * world
            dist.all_gather_object(parts, (D1["R0"], qc))
            qhat_full = np.zeros((n2t, n1t))
            for r0, blk in parts:
                qhat_full[r0:r0 + blk.shape[0]] = blk
            # the rest of Delta^dagger from the gathered partial x-DCT (same operator as P)
            c2 = spectral.dct_matrix(n2t)
            y = spectral.spectral_inverse(n2t, n1t) * (c2 @ qhat_full)
            phi = c2.T @ y @ c1
            rr = fpart - (w - ops.grad(phi))
            out = np.full_like(rr, np.nan)
            out[..., D1["E0"]:D1["V1"], :] = rr[..., D1["E0"]:D1["V1"], :]
            return out

        fglob = spectral.project(S.tau0(img)) / 0.05
        p1 = np.zeros((2, 2, n2t, n1t))
        qh1 = {}
        for ky in range(D1["k0"], D1["k1"]):
            for kx in range(lay.m1):
                qh1[(ky, kx)] = np.zeros((2, 2) + S.rect_shape(lay.rect((ky, kx), True)))
        for _ in range(sweeps):
            pp = _poison(p1, D1["V0"], D1["V1"])
            r = global_residual(pp, fglob)
            for m in list(qh1):
                qh1[m] = S._tfs_inner_local(m, lay, pp, r, qh1[m], inner, 0.125)
            assert all(np.isfinite(v).all() for v in qh1.values())
            su = _partial(lay, qh1, (D1["us0"], D1["us1"]), D1["k0"], D1["k1"], n1t, (2, 2), True)
            sd = _partial(lay, qh1, (D1["ds0"], D1["ds1"]), D1["k0"], D1["k1"], n1t, (2, 2), True)
            ru, rd = _exchange(None, rank, world, su, sd, (2, 2, D1["ur1"] - D1["ur0"], n1t),
                               (2, 2, D1["dr1"] - D1["dr0"], n1t))
            p1 = _combine(lay, pp, qh1, D1, ru, rd, True, n1t)
        _, p1_ref, _ = S.dd_step1(img, 0.05, lay, sweeps, inner)
        core1 = slice(D1["R0"], D1["R1"])
        err1 = float(np.abs(p1[..., core1, :] - p1_ref[..., core1, :]).max())
        q.put((rank, err2, err1, D, D1))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,case", [
    (2, (24, 20, (2, 2, 4, 4), 3, 3)),
    (2, (30, 18, (4, 1, 4, 0), 2, 3)),
    (3, (36, 22, (3, 2, 2, 4), 2, 2)),
])
def test_distributed_schwarz_matches_single_process(world, case):
    import paper_2602_17494_b200 as pkg
    from paper_2602_17494_b200 import build as pbuild
    pbuild.build()
    pkg.load_library()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    res.sort()
    # core rows tile the grid
    assert res[0][3]["R0"] == 0 and res[-1][3]["R1"] == case[0]
    assert res[0][4]["R0"] == 0 and res[-1][4]["R1"] == case[0] + 1
    for rank, err2, err1, D, D1 in res:
        assert err2 < 1e-12, (rank, err2)
        assert err1 < 1e-11, (rank, err1)


def test_dist_rows_plan_properties():
    """Host-only plan checks: sends match the neighbour's receives; core rows tile the grid."""
    import paper_2602_17494_b200 as pkg
    from paper_2602_17494_b200 import build as pbuild
    pbuild.build()
    for (n, L) in [(2048, (8, 8, 16, 16)), (8192, (8, 1, 32, 32)), (500, (5, 3, 6, 6))]:
        for step in (1, 2):
            for world in (1, 2, 4, 8):
                if L[0] < world:
                    continue
                plans = [pkg.dist_rows(n, n, L, step, r, world) for r in range(world)]
                G2 = n + 1 if step == 1 else n
                assert plans[0]["R0"] == 0 and plans[-1]["R1"] == G2
                for r in range(world - 1):
                    a, b = plans[r], plans[r + 1]
                    assert a["R1"] == b["R0"]
                    assert (a["ds0"], a["ds1"]) == (b["ur0"], b["ur1"])
                    assert (b["us0"], b["us1"]) == (a["dr0"], a["dr1"])
                if world == 1:
                    assert (plans[0]["V0"], plans[0]["V1"]) == (0, G2)
    with pytest.raises(pkg.TvsError):
        pkg.dist_rows(100, 100, (2, 2, 4, 4), 1, 0, 4)     # m2 < world
