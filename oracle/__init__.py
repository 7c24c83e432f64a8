"""oracle/ -- TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation (plain C, liboracle.so)
of Batch-BFS + BCTS, written from PAPER.md. Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference`
leg may import this package. It shares no code with the CUDA path in
paper_2107_01715_b200/ and never imports it.

Parity-pin status of every function: DESIGN.md §2 ("Oracle pins").
"""
from .oracle import (Oracle, build, bf16_round, penalty_eq5, bias_gap_eq4, inv_norm_cdf, B_n, bias_exact,  # noqa: F401
                     LIB_PATH)
