"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This package holds NO arithmetic of the method (no products, no filter, no
plan): it only builds the matrices H of the paper's workload classes as
canonical CSR (int64 rowptr, int32 sorted columns, float64 values, no
explicit zeros).  Both `oracle/` and `paper_2110_04493_b200/` consume it;
neither imports the other.
"""
from .configs import (  # noqa: F401
    CSR,
    CONFIGS,
    make_config,
    tridiag,
    laplacian_2d,
    laplacian_3d,
    structural_state_space,
    neumann_laplacian_2d,
    random_banded,
    random_skew,
    diagonal,
    geometric_graph,
    dense_to_csr,
    csr_to_dense,
)
