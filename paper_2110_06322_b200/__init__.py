"""B200-native closest point method (CPM) hot path: band build, matrix-free
stabilised operator apply, CGS2-GMRES and RAS, behind the C ABI of include/cpm.h.

The compute runs in libcpm.so (hand-written sm_100a CUDA, built in-tree by
paper_2110_06322_b200._build).  This package is the thin binding; it never
imports the CPU oracle (oracle/), which is test infrastructure only.
"""
from .cpm import (  # noqa: F401
    Band,
    CpmError,
    cpm_apply,
    cpm_apply_async,
    cpm_apply_sync,
    cpm_band_active_coords,
    cpm_band_eval_order,
    cpm_band_item_rounds,
    cpm_band_ghost_coords,
    cpm_build_band,
    cpm_comm_init,
    cpm_comm_init_host,
    cpm_comm_unique_id,
    cpm_eval_sph,
    cpm_eval_torus_rhs,
    cpm_kernel_launches,
    cpm_part_apply,
    cpm_part_apply_local,
    cpm_part_create,
    cpm_part_halo_nodes,
    cpm_part_ras_apply,
    cpm_part_ras_setup,
    cpm_part_rd_step,
    cpm_part_set_send,
    cpm_part_solve,
    cpm_profile_enable,
    cpm_profile_read,
    cpm_profile_reset,
    cpm_ras_apply,
    cpm_ras_setup,
    cpm_rd_step,
    cpm_solve,
    cpm_version,
    load_library,
)
