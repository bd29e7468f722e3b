"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This package holds NONE of the method's arithmetic (no filter, no orthonormalisation,
no Rayleigh-Ritz, no spectral operator, no proximal/DRS update).  It only builds the
problem data that BASELINE.json's configs describe.
Both `oracle/` and `paper_1904_10585_b200/` import it; it imports neither.
"""
from .generators import (  # noqa: F401
    Config, CONFIGS, config, reduced,
    initial_block, lanczos_start, cfg1_problem, cfg1_noise,
    pfpg_problem, pfam_problem, sym_bernoulli_bitmask, unpack_bitmask,
    bitmask_words, cfg5_spectrum, cfg5_reflectors, cfg5_basis_columns, Cfg5Matrix, cfg5_problem,
    hash_gauss, cfg5_noise_rows, cfg5_perturb, NEXT_CONFIGS, nce_problem,
    svt_problem, svt_guard_block, BENCH_METHOD, bench_config,
)
