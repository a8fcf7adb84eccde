"""fp64 CPU ORACLE for the TV-Stokes overlapping-Schwarz dual iteration (arXiv 2602.17494).

TEST INFRASTRUCTURE ONLY.  Nothing in the product path (``paper_2602_17494_b200``) may import,
call or link anything under ``oracle/``; only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs use it.  The oracle shares no code,
tables or constants with the CUDA path; the only common module is ``tvs_synth`` (seeded inputs,
none of the method's arithmetic).

Plain, slow, obviously-correct NumPy in float64, written from PAPER.md (``P:<line>``):

* ``ops``       finite differences, grad/div, multigrad/multidiv, Neumann D^{neum-}
* ``spectral``  DCT-II matrix, sigma, Moore-Penrose Delta^dagger, projection P_K
* ``layout``    overlapping layout, partition of unity, alpha-hat  (readings A6-A8)
* ``solvers``   tau_0, g, Chambolle (Alg. 1), Schwarz Alg. 2 with Alg. 3 (IRV2) and Alg. 4/5
                (TFS), the literal block-DCT local projection (Eq. invLaplLowCapLong), energies.

Readings of ambiguous passages (A1..A21) are the ones listed in DESIGN.md / SURVEY.md 8(c).
Parity status: every function is pinned by ``tests/test_oracle_*.py`` except the finite-schedule
Schwarz trajectory itself, which is pinned only transitively (its unit steps are pinned, and it
converges to the pinned single-domain solution) -- "parity unpinned" beyond that, see DESIGN.md.
"""
from . import ops, spectral, layout, solvers  # noqa: F401
