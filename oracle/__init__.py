"""fp64 CPU oracle of randomized SymNMF (arXiv 2402.08134) -- TEST INFRASTRUCTURE.

This package is NOT part of the product path.  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import it.  It shares no code with paper_2402_08134_b200/ (the CUDA
library and its binding): neither imports the other; both consume inputs from
synth/ only.

Every function cites the PAPER.md passage (P:<line>) it follows and, where the
paper is silent or ambiguous, the DESIGN.md reading (Z<n>) it implements.

Parity unpinned (no pin independent of the oracle exists):
  * lvs_iterate trajectories vs an independent RNG run (statistical only),
  * the synthetic generator choices Z22-Z24 (synth/, no paper values).
"""
from .symnmf import *  # noqa: F401,F403
from .philox import philox4x32_10, philox_u64, mulhi64  # noqa: F401
