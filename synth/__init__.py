"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This package holds NO arithmetic of the SymNMF method: it only draws the
input matrices of the five BASELINE.json configurations, the paper's random
initial factor and the hyperparameter alpha = max(A)
(P:1103-1105).  Both sides (oracle/ and paper_2402_08134_b200/) receive the
identical fp32 arrays produced here.
"""
from .configs import (  # noqa: F401
    CONFIGS,
    Config,
    CsrMatrix,
    make_input,
    init_factor,
    alpha_of,
    planted_dense,
    sbm_csr,
    powerlaw_csr,
    gaussian_points,
    gaussian_kernel_rows,
    gaussian_kernel_dense,
    random_factor,
)
