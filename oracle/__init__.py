"""oracle/ -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously correct CPU implementation of what the Atlas hot path
computes (PAPER.md, arXiv 2408.09055), written from the paper and independent
of the CUDA product path:

  * sim.py        O1: gate-at-a-time complex128 simulator (C, sv_oracle.c)
  * einsum_sim.py O1': an independent NumPy tensor-contraction simulator (n <= 16)
  * gates.py      the oracle's own textbook gate table + insularity by definition
  * planner.py    O2: brute-force staging (ILP optimum by enumeration), the
                  contiguous-segmentation optimum (OrderedKernelize target),
                  Constraint 1 / extensible-qubit definitions, plan checker
  * remap.py      O3: the remap as a pure index permutation

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import anything from here.  The product package
(paper_2408_09055_b200/) never imports it, and it never imports the product.
Parity status of each function is stated in its docstring ("pinned by ..."
or "parity unpinned").
"""
