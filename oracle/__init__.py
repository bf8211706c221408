"""FS-1 ORACLE — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU fp64 implementation of what the FS-1 hot
path computes (Liao et al., arXiv 2202.10042; /root/reference/PAPER.md).
It exists to prove the CUDA path right.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The product package
``paper_2202_10042_b200`` never imports it, shares no code with it, and fails
loudly when its CUDA library is missing.

Contents (each function cites the passage it follows):

* ``dense``    — the Gibbs kernel K_ij = lambda^|i-j| (PAPER.md:80-89, 112-122,
                 powers by stepwise multiplication, Remark 3.3 PAPER.md:236-238),
                 dense applies in the scaling and log domains, the 2D block
                 kernel, the distance-weighted kernel of the
                 return line.
* ``recur``    — the paper's O(N) forward/backward recursion written out
                 literally in plain C (Eq. ``recursion`` PAPER.md:129-137,
                 Algorithm 1 lines 3-6 / 8-11 PAPER.md:149-158) and its
                 log-sum-exp form (BASELINE.json north_star); used where dense
                 is infeasible (N = 2^24, 2048^2).
* ``sinkhorn`` — Algorithm 1 / Algorithm 2 loops:
                 initialisation, psi-first update order, marginal-error
                 termination, non-finite detection, the return-line cost.
* ``w1``       — exact W1 closed form and the N=2 entropic closed form (pins).

Parity status: every function is pinned by ``tests/test_oracle_*.py`` against
closed forms, brute force, library routines or invariants.
No function is "parity unpinned".
"""
