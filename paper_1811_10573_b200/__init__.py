"""paper_1811_10573_b200 — B200 (sm_100a) hot path of CP-ALS with pairwise perturbation.

The product is libcppp.so (csrc/, C ABI in include/cppp.h); ``cppp`` is its thin ctypes
binding.  Importing the package does not load the library; the first binding call does, and
raises if it is missing (no CPU fallback).
"""
from . import cppp  # noqa: F401
from .cppp import (  # noqa: F401
    als_sweep, cp_destroy, cp_get_factors, cp_init, cp_set_factors, cp_set_phase_override,
    cppp_generate, fitness, mttkrp_dt, pp_build_operators, pp_get_operator, pp_get_single,
    pp_update,
)

__version__ = "0.1.0"
