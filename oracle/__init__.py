"""CPU ORACLE — test infrastructure, NOT part of the product path.

A plain, slow, obviously-correct FP64 numpy implementation of the nodal DG
semi-discrete Maxwell operator and its LSERK4 time integration, written from
Klöckner–Warburton–Hesthaven, arXiv:1211.0582 and the
textbook it follows for the strong form, nodes and operators (Hesthaven &
Warburton, "Nodal Discontinuous Galerkin Methods", 2008 — "HW").

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` leg may import anything from here.  The product package
`paper_1211_0582_b200` never imports it, and this package never imports the
product package: the two share no code, headers, tables or constants.  Inputs
come from `dg_inputs` (which holds none of the method's arithmetic).

Modules
  refelem  reference element: warp&blend nodes, Dubiner Vandermonde, Dr/Ds/Dt,
           mass and face-mass matrices, LIFT (eqs. 3, 6; HW ch. 6/10)
  mesh     affine geometry, normals/Fscale, face connectivity, vmapM/vmapP by
           coordinate matching
  maxwell  Maxwell RHS with upwind flux + PEC walls, LSERK4, energy
           
  acoustics  second linear system: linear acoustics with upwind
           flux + rigid walls through the same four stages

Parity pins: every function is pinned by a `-m "not gpu"` test in
tests/test_oracle_*.py against closed forms, invariants, brute force or
golden values (see DESIGN.md §"Oracle and its pins").  Functions whose result is
pinned only by invariants (the interior warp&blend node positions for N >= 4)
say so in their docstring: "parity unpinned beyond invariants".
"""
from . import refelem, mesh, maxwell, acoustics  # noqa: F401
from .refelem import RefElement, build_reference  # noqa: F401
from .mesh import Setup  # noqa: F401
from .maxwell import rhs, lserk4, lserk4_coefficients, energy  # noqa: F401
