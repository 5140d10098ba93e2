"""B200-native HPL hot path (arXiv 2304.10397): blocked right-looking LU with
partial pivoting — device panel FACT, LASWP gather/scatter, DTRSM and the
TMA-fed DMMA trailing DGEMM with look-ahead — behind the C ABI in
include/hpl.h.  Importing this package loads libhpl.so and fails loudly if it
is missing (no CPU fallback)."""
from .hpl import (  # noqa: F401
    Ctx, HplError, HplSingular, hpl_factor, hpl_free, hpl_get_ipiv, hpl_get_local,
    hpl_get_timeline, hpl_get_fact_detail, hpl_get_unique_id, hpl_init, hpl_init_dist,
    hpl_init_loopback, hpl_last_timing, hpl_launch_count, hpl_phase_stats, hpl_pin_host,
    hpl_plan_iteration, hpl_plan_fact, hpl_load_local, hpl_load_factor, hpl_regenerate, hpl_residual,
    hpl_set_option, hpl_set_timing, hpl_solve, run_ranks,
    hplk_back_solve, hplk_dgemm_bench, hplk_dgemm_update, hplk_dmma_peak, hplk_panel_bench,
    hplk_generate, hplk_laswp, hplk_panel_fact, hplk_residual, hplk_rs_exchange, hplk_trsm,
)
