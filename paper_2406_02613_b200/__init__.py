"""B200-native ACCO (Accumulate While Communicate, arXiv 2406.02613).

Drop-in for the ACCO round of the reference simulator `accosim`: the C-ABI in
include/acco.h (library ``_acco_b200.so``) plus the Python host mirror in
:mod:`paper_2406_02613_b200.api` of the reference's ``run_protocol`` /
``OptimizerConfig`` / ``SimConfig`` / JSON config.
"""
