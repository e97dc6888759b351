"""B200-native (sm_100a) hot path of arXiv 2409.17688: (min,+) powers of the 2-domination
transfer matrix until quasi-periodicity, and gamma_2(P_n x C_m) read off from them.

The computation lives in ``libminplus.so`` (CUDA kernels behind the C ABI of
``include/minplus.h``); this package is its argument-marshalling binding.
"""
from ._native import (  # noqa: F401
    MP_FINITE_MAX, MP_INF, MP_MAX_K, MP_MAX_N, MinplusError, PeriodicResult, PowerStats,
    build_transition_matrix, count_words, dist_set, dist_set_allgather, dist_set_torch, fingerprint_unit,
    gamma2_cylinder, gamma2_record, kernel_launches, last_error, last_profile, minplus_closure, minplus_mul,
    minplus_mul_batched_device, minplus_mul_device,
    minplus_power_rows, minplus_power_until_periodic, minplus_power_until_periodic_device,
    repeat_candidate, set_grouping, set_power_observer, set_small_path, set_transfer_hint, set_row_reuse, set_spmm_width, set_options, set_stream, set_symmetry, set_word_symmetry,
    word_reversal, shard_range, shutdown, version, column_plan,
)
