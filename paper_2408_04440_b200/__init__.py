"""B200-native drop-in for the BLAS3 hot path of sphemu (arXiv 2408.04440).

Mirrors the reference's Python module (proj/python/sphemu/__init__.py,
proj/bindings/module.cpp): forward_sht / inverse_sht / tiled_cholesky /
make_spd_matrix / max_band_limit / resolution_summary, backed by hand-written
sm_100a kernels in lib/libsphemu_gpu.so (see include/sphemu_gpu.h).
"""
from ._sphemu import (  # noqa: F401
    Cholesky,
    ForcingTrajectory,
    NotPositiveDefiniteError,
    ShtPlan,
    __version__,
    assign_precisions,
    detrend,
    emulate,
    emulate_model,
    estimate_innovation_covariance,
    fit_var,
    forward_sht,
    inverse_sht,
    make_spd_matrix,
    mean_table,
    nccl_unique_id,
    max_band_limit,
    resolution_summary,
    retrend,
    synth_bandlimited,
    tiled_cholesky,
    tile_norm_precisions,
    wigner_d_half_pi,
)
from .emulator import Emulator, read_sphf, write_sphf  # noqa: F401

__all__ = [
    "Cholesky", "ForcingTrajectory", "NotPositiveDefiniteError", "ShtPlan", "__version__", "assign_precisions", "emulate", "emulate_model",
    "estimate_innovation_covariance", "fit_var", "forward_sht", "inverse_sht", "make_spd_matrix", "nccl_unique_id", "max_band_limit", "resolution_summary",
    "synth_bandlimited", "tiled_cholesky", "wigner_d_half_pi", "mean_table", "detrend", "retrend",
    "Emulator", "read_sphf", "write_sphf", "tile_norm_precisions",
]
