"""CPU oracle for the ADER-DG element update of arXiv:1903.11521 (Uphoff & Bader), Sec. 5.1.

TEST INFRASTRUCTURE ONLY.  Nothing in the product path (``paper_1903_11521_b200``) may
import, call, link or execute anything under ``oracle/``; only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference``
legs do.  The oracle shares no code with the CUDA path: it builds its own basis, its
own global matrices (exact rational arithmetic), its own geometry, physics, Riemann
solver and face matching.

Citations: ``P:n`` = line n of the paper's LaTeX source.  Where the paper is
silent or garbled the reading taken is the one recorded in DESIGN.md §3 ("Readings").

Modules
-------
basis     Dubiner basis on the reference tetrahedron and face basis, as exact integer
          polynomials ("Dubiner's basis functions"; reading R6).
matrices  Global matrices by exact integration: M, K^c, Ktilde^c, Khat^c, face matrices
          F^-, F^+ and (for pins / literal mode) R^i, f^h.
physics   Jacobians, star matrices, Godunov flux solvers, viscoelastic source
          (readings R5, R8, R14).
mesh      Geometry, face matching, neighbour relation (P:1342 Neigh/Face/Rot).
step      One ADER-DG step, plain dense evaluation; literal einsum mode.

Pinned by ``tests/test_oracle_*.py`` (``-m "not gpu"``).  Parity status of each function is
listed in DESIGN.md §4.
"""
