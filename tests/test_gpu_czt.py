"""Chirp-z form of the partial x-DCTs (tvs_czt.cu) forced on every projection
batch (TVS_DCT=czt) and compared with the fp64 oracle at the north-star tolerances, on ragged
layouts (several chunk / pass geometries), config 2 in full and config 3 at full size."""
import os

import numpy as np
import pytest

from oracle import solvers as S
from tvs_synth import CONFIGS, random_image

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from test_gpu_parity import check_step1, check_step2   # noqa: E402


def _context(**env):
    import paper_2602_17494_b200 as pkg
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return pkg.Context(0)
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    c = _context(TVS_DCT="czt")
    yield c
    c.close()


@pytest.fixture(scope="module")
def ctx_chunked():
    """FFT size capped at 64 points: every small case runs several input chunks / output passes."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    c = _context(TVS_DCT="czt", TVS_CZT_MAXM="64")
    yield c
    c.close()


@pytest.mark.parametrize("shape,L", [((16, 16), (1, 1, 0, 0)), ((24, 20), (2, 2, 4, 4)),
                                     ((37, 53), (3, 2, 3, 5)), ((40, 18), (4, 1, 4, 0)),
                                     ((18, 40), (1, 4, 0, 3)), ((2, 2), (1, 1, 0, 0)),
                                     ((63, 63), (1, 1, 0, 0)), ((127, 127), (4, 1, 6, 0))])
def test_step1_czt_small(ctx, ctx_chunked, shape, L):
    img = random_image(*shape, seed=shape[0] * 7 + shape[1] + 1)
    check_step1(ctx, img, 0.05, L, 3, 4)
    check_step1(ctx_chunked, img, 0.05, L, 3, 4)


@pytest.mark.parametrize("shape,L", [((20, 150), (1, 16, 0, 2)), ((20, 300), (1, 24, 0, 2)),
                                     ((24, 600), (2, 24, 2, 2))])
def test_step1_czt_narrow_tiles(ctx, shape, L):
    """Tiles at most M/16 wide (M = 256, 1024): the forward transform takes the pruned first FFT
    pass (input read straight from global memory) and the inverse the pruned last pass (outputs
    written straight through the post-chirp), as config 5's 16 x 16 layout does at full size."""
    img = random_image(*shape, seed=shape[0] * 5 + shape[1])
    check_step1(ctx, img, 0.05, L, 3, 4)


def test_config2_czt(ctx):
    c = CONFIGS["c2"]
    img = c.image()
    L = (c.m2, c.m1, c.overlap, c.overlap)
    tau_ref, _ = check_step1(ctx, img, c.delta, L, c.sweeps, c.inner)
    check_step2(ctx, img, tau_ref, c.lam, L, c.sweeps, c.inner)


def test_config3_czt_full_size(ctx):
    c = CONFIGS["c3"]
    img = c.image()
    L = (c.m2, c.m1, c.overlap, c.overlap)
    check_step1(ctx, img, c.delta, L, 1, 2)


@pytest.fixture(scope="module")
def ctx_grouped():
    """Tile groups of at most 3 tiles sharing one projection scratch (TVS_PROJ_GROUP=3): the path
    config 5 takes at full size, where the whole local batch's scratch would exceed HBM."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    c = _context(TVS_DCT="czt", TVS_PROJ_GROUP="3")
    yield c
    c.close()


@pytest.mark.parametrize("shape,L", [((37, 53), (3, 2, 3, 5)), ((64, 64), (4, 4, 4, 4)),
                                     ((40, 18), (4, 1, 4, 0)), ((300, 90), (2, 2, 8, 4)),
                                     ((1400, 40), (1, 4, 0, 4))])
def test_step1_czt_tile_groups(ctx, ctx_grouped, shape, L):
    """Groups of 3 consecutive tiles (ragged last group; groups spanning several layout rows, so
    solve4's per-group launch order and solve3's tile offsets are both exercised -- the 300-row
    case has tiles taller than solve4's shared-memory limit): parity with the oracle, and bitwise
    equality with the ungrouped batch (same kernels, same per-tile arithmetic).  The 1400-row
    tiles are taller than solve4's shared-memory limit and than solve3's shared z (global z
    scratch, shared by the group), as config 5's 2083-row tiles."""
    img = random_image(*shape, seed=shape[0] * 11 + shape[1])
    check_step1(ctx_grouped, img, 0.05, L, 3, 4)
    d0 = torch.from_numpy(img).cuda()
    t1, p1, _ = ctx.tv_stokes_step1(d0, 0.05, L, (3, 4, 0.125), want_p=True)
    t2, p2, _ = ctx_grouped.tv_stokes_step1(d0, 0.05, L, (3, 4, 0.125), want_p=True)
    torch.cuda.synchronize()
    assert torch.equal(t1, t2) and torch.equal(p1, p2)


@pytest.fixture(scope="module")
def ctx_general():
    """The general chirp-z form everywhere (TVS_CZT_MAKHOUL=0), for A/B against the Makhoul form."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    c = _context(TVS_DCT="czt", TVS_CZT_MAKHOUL="0")
    yield c
    c.close()


@pytest.mark.parametrize("shape,L", [((40, 32), (2, 2, 4, 4)), ((20, 128), (1, 3, 0, 6)),
                                     ((33, 128), (3, 1, 4, 0)), ((8, 8), (1, 1, 0, 0)),
                                     ((129, 512), (2, 4, 6, 8))])
def test_step1_makhoul_form(ctx, ctx_general, shape, L):
    """Axes with N~1 = n1 + 1 in {9, 33, 129, 513}, where M = 2N - 2 is a power of 4: the partial
    x-DCTs run in the Makhoul form (forward: two rows per DFT_N; inverse: the DCT-III pair and the
    shifted sine transform as two packed DCT-IIIs).  Parity with the oracle on full-width, narrow
    and ragged tiles (odd and even row counts: the row pairs of the forward and y-inverse jobs),
    and agreement with the general chirp-z form to fp32 rounding."""
    img = random_image(*shape, seed=shape[0] * 3 + shape[1] + 5)
    check_step1(ctx, img, 0.05, L, 3, 4)
    d0 = torch.from_numpy(img).cuda()
    t1, _, _ = ctx.tv_stokes_step1(d0, 0.05, L, (3, 4, 0.125))
    t2, _, _ = ctx_general.tv_stokes_step1(d0, 0.05, L, (3, 4, 0.125))
    torch.cuda.synchronize()
    assert float((t1 - t2).abs().max()) < 2e-5


@pytest.fixture(scope="module")
def ctx_nox6():
    """The sine form (kind 5) for every Makhoul inverse-x job (TVS_CZT_X6=0)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    c = _context(TVS_DCT="czt", TVS_CZT_X6="0")
    yield c
    c.close()


@pytest.mark.parametrize("shape,L", [((40, 32), (2, 2, 4, 4)), ((33, 128), (3, 1, 4, 0)),
                                     ((129, 512), (2, 4, 6, 8)), ((65, 512), (1, 1, 0, 0))])
def test_step1_makhoul_x6_ab(ctx, ctx_nox6, shape, L):
    """The local projections' x-gradient by differencing phi (kind 6, row pairs) against the sine
    form (kind 5): both match the oracle, and agree with each other to fp32 rounding, on even and
    odd row counts and single-domain layouts."""
    img = random_image(*shape, seed=shape[0] * 7 + shape[1] + 11)
    check_step1(ctx, img, 0.05, L, 3, 4)
    check_step1(ctx_nox6, img, 0.05, L, 3, 4)
    d0 = torch.from_numpy(img).cuda()
    t1, _, _ = ctx.tv_stokes_step1(d0, 0.05, L, (3, 4, 0.125))
    t2, _, _ = ctx_nox6.tv_stokes_step1(d0, 0.05, L, (3, 4, 0.125))
    torch.cuda.synchronize()
    assert float((t1 - t2).abs().max()) < 2e-5


def test_pipelined_groups_bitwise(ctx):
    """Two subdomain groups in flight on two streams with separate scratch (TVS_PIPE=1) give
    bitwise the serial schedule's tau and p, also with more than two groups (TVS_PROJ_GROUP) and
    odd inner counts."""
    serial = _context(TVS_DCT="czt", TVS_PIPE="1")
    grouped = _context(TVS_DCT="czt", TVS_PIPE="1", TVS_PROJ_GROUP="2")
    try:
        for shape, L, it in (((40, 32), (4, 2, 4, 4), (3, 4)), ((64, 64), (4, 4, 4, 4), (2, 3)),
                             ((37, 53), (3, 2, 3, 5), (3, 3))):
            img = random_image(*shape, seed=shape[0] + 2 * shape[1])
            d0 = torch.from_numpy(img).cuda()
            sch = (it[0], it[1], 0.125)
            t0, p0, _ = serial.tv_stokes_step1(d0, 0.05, L, sch, want_p=True)
            t1, p1, _ = ctx.tv_stokes_step1(d0, 0.05, L, sch, want_p=True)
            t2, p2, _ = grouped.tv_stokes_step1(d0, 0.05, L, sch, want_p=True)
            torch.cuda.synchronize()
            assert torch.equal(t0, t1) and torch.equal(p0, p1), shape
            assert torch.equal(t0, t2) and torch.equal(p0, p2), shape
    finally:
        serial.close()
        grouped.close()
