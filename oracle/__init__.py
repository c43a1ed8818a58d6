"""CPU ORACLE for the PODP on-line stage -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may
import or execute anything under ``oracle/``.  The product path (``paper_2307_05590_b200``) never imports it and
fails loudly if its CUDA library is missing.  The oracle shares no code with the CUDA path; the only common
dependency is the seeded input generator package ``podp_inputs`` (which holds no on-line arithmetic).

It is a plain, slow, obviously-correct NumPy complex128 evaluation of the paper's formulas, written out in the
paper's order (PAPER.md = /root/reference/PAPER.md; "P:<line>"):
  * reduced shifted solve                      P:593-596  eqn:ReducedA  (LAPACK zgesv via numpy.linalg.solve)
  * MM real part R                             P:600-604  eqn:podprealmpt
  * MM imaginary part I                        P:606-620  eqn:podpimagmpt (shared-basis form)
  * Lemma 4.1 certificate Delta via w^H G w    P:632-661  lemma:certificate
  * Algorithm 1 interval maxima / selection    P:677-682  alg:adapt lines 10-15
  * full-order FMM formulas (pins only)        P:506-553  eqn:Rmatrixmeth, eqn:I_tensor_coeffs

Pinned by ``tests/test_oracle_pins.py`` (pins C1-C12 of SURVEY.md 8(c)).  Parity unpinned: the Lemma 4.1
*inequality* |R - R^PODP| <= Delta itself (needs Wilson2021's Y^(hp) norm and alpha_LB) -- the oracle
evaluates the formula only.
"""
from .podp_oracle import (  # noqa: F401
    ENTRY_ORDER, solve_reduced, mpt_R, mpt_I, residual_coeffs, certificate, evaluate_one, evaluate, select,
    to6, from6, invariants, coil_voltage,
)
