"""CPU oracle for arXiv 2110.04493's filtered PIM matrix exponential.

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / `--impl reference` legs may import this package.  The product
(paper_2110_04493_b200) never imports it and shares no code with it.
"""
from .oracle import (  # noqa: F401
    build,
    r0,
    plan,
    alg41,
    expm,
    spgemm,
    spmm,
    rcm,
    add,
    norm_one,
    norm_fro,
    norm_fro_I_plus,
    bandwidth,
    Options,
)
