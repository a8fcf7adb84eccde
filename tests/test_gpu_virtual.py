"""Multi-GPU data path on ONE GPU: a virtual slab group (tvs_create_virtual_group) runs W ranks of
the slab decomposition as W host threads on one device, each with its own stream;
their exchanges -- the partial band sums (k_partial), the band send/recv, the remote-band branches
of the combine, the row all-gathers of the partial x-DCT and of the outputs, the energy
all-reduces -- are device-to-device copies instead of NCCL calls.  Everything else is the code
that runs with one process per GPU.  The Schwarz iteration is additive with a fixed combine
order, so tau / d / p must be BITWISE those of world = 1 ("GPU-count invariance")."""
import threading

import numpy as np
import pytest

from tvs_synth import random_image, voronoi

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2602_17494_b200 as pkg
    c = pkg.Context(0)
    yield c
    c.close()


def _dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def run_group(world, fn):
    """fn(ctx_r, stream_r) on `world` threads of a fresh virtual group; returns the results."""
    import paper_2602_17494_b200 as pkg
    ctxs = pkg.Context.virtual_group(world, 0)
    streams = [torch.cuda.Stream() for _ in range(world)]
    out, err = [None] * world, [None] * world

    def body(r):
        try:
            with torch.cuda.stream(streams[r]):
                out[r] = fn(ctxs[r], streams[r])
                streams[r].synchronize()
        except Exception as e:   # noqa: BLE001 -- re-raised below
            err[r] = e

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=900)
    for c in ctxs:
        c.close()
    return out, err


CASES = [
    # (shape, layout, worlds): even and uneven splits of the layout rows, ragged tiles
    ((96, 80), (4, 3, 6, 5), (2, 4)),
    ((131, 77), (5, 2, 4, 3), (2, 3, 5)),
    ((256, 256), (8, 8, 16, 16), (2, 4, 8)),
]


@pytest.mark.parametrize("shape,L,worlds", CASES)
def test_virtual_step2_bitwise(ctx, shape, L, worlds):
    img = random_image(*shape, seed=shape[0] + 7)
    d0 = _dev(img)
    tau_ref, _, _ = ctx.tv_stokes_step1(d0, 0.05, L, (2, 3, 0.125))
    it = (4, 5, 0.125)
    d1, p1, s1 = ctx.tv_stokes_step2(tau_ref, d0, 0.1, L, it, want_p=True)
    torch.cuda.synchronize()
    for w in worlds:
        res, err = run_group(w, lambda c, s: c.tv_stokes_step2(tau_ref, d0, 0.1, L, it, want_p=True,
                                                              stream=s))
        assert not any(err), err
        for r, (d, p, st) in enumerate(res):
            assert torch.equal(d, d1), (w, r, float((d - d1).abs().max()))
            assert torch.equal(p, p1), (w, r)
            assert abs(st.primal_energy - s1.primal_energy) <= 1e-9 * abs(s1.primal_energy)
            assert abs(st.dual_energy - s1.dual_energy) <= 1e-9 * abs(s1.dual_energy)


@pytest.mark.parametrize("shape,L,worlds", CASES)
def test_virtual_step1_bitwise(ctx, shape, L, worlds):
    img = random_image(*shape, seed=shape[1] + 3)
    d0 = _dev(img)
    it = (3, 4, 0.125)
    t1, p1, s1 = ctx.tv_stokes_step1(d0, 0.05, L, it, want_p=True)
    torch.cuda.synchronize()
    for w in worlds:
        res, err = run_group(w, lambda c, s: c.tv_stokes_step1(d0, 0.05, L, it, want_p=True,
                                                              stream=s))
        assert not any(err), err
        for r, (t, p, st) in enumerate(res):
            assert torch.equal(t, t1), (w, r, float((t - t1).abs().max()))
            assert torch.equal(p, p1), (w, r)
            assert abs(st.primal_energy - s1.primal_energy) <= 1e-9 * abs(s1.primal_energy)
            assert abs(st.gap - s1.gap) <= 1e-9 * abs(s1.primal_energy)


def test_virtual_denoise_config3_layout_bitwise(ctx):
    """The config-3 layout (8 x 8 subdomains, overlap 16) on a 1024^2 Voronoi image, 4 and 8
    virtual ranks, full denoise (step 1 with the global all-gathered projection, then step 2)."""
    img = voronoi(1024, 64, 1003)
    d0 = _dev(img)
    L = (8, 8, 16, 16)
    it = (2, 3, 0.125)
    d1, t1, _, _ = ctx.tv_stokes_denoise(d0, 0.05, 0.1, L, it, it, want_tau=True)
    torch.cuda.synchronize()
    for w in (4, 8):
        res, err = run_group(w, lambda c, s: c.tv_stokes_denoise(d0, 0.05, 0.1, L, it, it,
                                                                 want_tau=True, stream=s))
        assert not any(err), err
        for r, (d, t, _, _) in enumerate(res):
            assert torch.equal(t, t1) and torch.equal(d, d1), (w, r)


def test_virtual_group_rank_failure_aborts_the_others(ctx):
    """A rank that fails (here: an invalid delta on rank 1) aborts the group's rendezvous: the other
    ranks return an error instead of waiting forever."""
    import paper_2602_17494_b200 as pkg
    d0 = _dev(random_image(40, 40, 5))
    L = (4, 2, 4, 4)
    _, err = run_group(2, lambda c, s: c.tv_stokes_step1(d0, -1.0 if c.vrank == 1 else 0.05, L,
                                                         (2, 2, 0.125), stream=s))
    assert isinstance(err[1], pkg.TvsError) and err[1].code == 1      # TVS_EINVAL
    assert isinstance(err[0], pkg.TvsError) and err[0].code == 6      # aborted rendezvous
