"""CPU oracle for the Polya/SDP hot path of Kamyar, Peet & Peet (arxiv 1411.3769).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_1411_3769_b200``) never imports it and
shares no code, table or constant generator with it; only the seeded input
generator ``synth`` serves both sides.

The oracle is plain, slow and follows PAPER.md step by step (line numbers are
PAPER.md lines, "S:n" SPEC.md lines; the readings R1..R16 are listed in
DESIGN.md "Readings of the paper"):

* ``monomials``  -- W_d, Eq. (1)/(2), reading R1;
* ``polya``      -- beta and H by explicit polynomial multiplication of
                    (sum alpha)^d * P(alpha) and (sum alpha)^d * A(alpha) P(alpha)
                    (Eqs. LMI_1-LMI_4) plus the literal
                    recursions Eqs. (19)-(22), C by Eq. (27);
                    homogenisation and the simplex maps g of
                    Examples 1-2 (reading R17);
* ``sdp``        -- the basis E_k (Eqs. 4-5, reading R2), the V-map (Eq. 30),
                    dense F_i blocks (Eq. 31), B(X) and B^T(y) (Eqs. 14, 16),
                    and the Schur complement lambda_{k,l} = sum_b tr(B_k Z^-1 B_l X)
                    (Eq. T2) by literal traces;
* ``ipm``        -- one predictor-corrector iteration of Algorithm 2 on dense
                    block matrices, readings R3-R6;
                    the iteration to the stopping rule and the
                    grid-checked verdict (O8).

Every function is pinned by ``tests/test_oracle_*.py`` against values the paper
prints, closed forms, invariants and brute force.
"""
from . import monomials, polya, sdp  # noqa: F401
