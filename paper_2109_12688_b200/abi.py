"""ctypes mirror of include/dreg_cuda.h (struct layouts and status codes).

Every struct here is a field-for-field copy of the C declaration; the C header cites
the reference type each one mirrors (proj/core/include/dreg/*.hpp).
"""
from __future__ import annotations

import ctypes as C

DREG_OK = 0
DREG_INVALID_ARGUMENT = 2
DREG_IO_ERROR = 3
DREG_NUMERIC = 4
DREG_RUNTIME = 5

DREG_MAX_LEVELS = 10
DREG_MAX_WARPS = 256

DREG_KIND_SCALAR = 0
DREG_KIND_VECTOR = 1
DREG_KIND_LABEL = 2

DREG_PROFILE_CAPPED = 0
DREG_PROFILE_CONVERGED = 1


class Dims3(C.Structure):
    """dreg::Dims3 (volume.hpp:11-21): x fastest."""

    _fields_ = [("x", C.c_int), ("y", C.c_int), ("z", C.c_int)]

    def voxels(self) -> int:
        return self.x * self.y * self.z

    def shape(self) -> tuple[int, int, int]:
        """numpy shape (z, y, x) of an x-fastest buffer."""
        return (self.z, self.y, self.x)

    def __repr__(self) -> str:
        return f"Dims3({self.x},{self.y},{self.z})"


class Spacing3(C.Structure):
    _fields_ = [("x", C.c_double), ("y", C.c_double), ("z", C.c_double)]


class SolverCfg(C.Structure):
    """dreg::SolverConfig (admm.hpp:13-23)."""

    _fields_ = [
        ("data_term", C.c_int),
        ("order", C.c_int),
        ("lambda_", C.c_double),
        ("theta", C.c_double),
        ("epsilon", C.c_double),
        ("max_iters", C.c_int),
        ("tol", C.c_double),
        ("accelerate", C.c_int),
        ("log_objective", C.c_int),
    ]


class RegCfg(C.Structure):
    """dreg::RegistrationConfig (registration.hpp:16-24)."""

    _fields_ = [
        ("solver", SolverCfg),
        ("levels", C.c_int),
        ("max_warps_per_level", C.c_int * DREG_MAX_LEVELS),
        ("max_admm_iters_per_level", C.c_int * DREG_MAX_LEVELS),
        ("warp_improvement_threshold", C.c_double),
        ("profile", C.c_int),
        ("smooth_levels", C.c_int),
    ]


class SolverDiag(C.Structure):
    """dreg::SolverDiagnostics (admm.hpp:28-34)."""

    _fields_ = [
        ("iterations", C.c_int),
        ("final_change", C.c_double),
        ("converged", C.c_int),
        ("objective", C.POINTER(C.c_double)),
        ("constraint_residual", C.POINTER(C.c_double)),
    ]


class LevelLog(C.Structure):
    """dreg::LevelLog (registration.hpp:32-37)."""

    _fields_ = [
        ("dims", Dims3),
        ("warps", C.c_int),
        ("mean_sad", C.c_double * (DREG_MAX_WARPS + 1)),
        ("solver_iterations", C.c_int * DREG_MAX_WARPS),
    ]


class PairResult(C.Structure):
    """dreg::RegistrationResult scalars (registration.hpp:39-45)."""

    _fields_ = [
        ("status", C.c_int),
        ("velocity_count", C.c_int),
        ("solves", C.c_int),
        ("levels", C.c_int),
        ("per_level", LevelLog * DREG_MAX_LEVELS),
        ("elapsed_seconds", C.c_double),
        ("folding_voxels", C.c_int64),  # jacobian_stats of the returned phi, computed on device
        ("min_det", C.c_double),
    ]


class PairRecord(C.Structure):
    """dreg_pair_record: the per-pair record of the multi-device all-gather (64 bytes)."""

    _fields_ = [
        ("pair", C.c_int32),
        ("device", C.c_int32),
        ("status", C.c_int32),
        ("velocity_count", C.c_int32),
        ("solves", C.c_int32),
        ("levels", C.c_int32),
        ("folding_voxels", C.c_int64),
        ("admm_iterations", C.c_int64),
        ("final_mean_sad", C.c_double),
        ("min_det", C.c_double),
        ("reserved", C.c_int64),
    ]


class JacobianStats(C.Structure):
    """dreg::JacobianStats (metrics.hpp:44-48) plus raw counts."""

    _fields_ = [
        ("pct_nonpositive", C.c_double),
        ("min_det", C.c_double),
        ("nonpositive", C.c_int64),
        ("interior", C.c_int64),
    ]


class VolumeInfo(C.Structure):
    """DREG container header (io.hpp:15-22): kind, dims, spacing."""

    _fields_ = [("kind", C.c_int), ("dims", Dims3), ("spacing", Spacing3)]


class ReportConfig(C.Structure):
    """dreg::ReportConfig (io.hpp:43-54)."""

    _fields_ = [
        ("data_term", C.c_char_p),
        ("order", C.c_int),
        ("lambda_", C.c_double),
        ("theta", C.c_double),
        ("levels", C.c_int),
        ("profile", C.c_char_p),
        ("tol", C.c_double),
        ("warp_improvement_threshold", C.c_double),
        ("epsilon", C.c_double),
        ("threads", C.c_int),
    ]


class RunReport(C.Structure):
    """dreg::RunReport (io.hpp:56-62); label maps as parallel arrays."""

    _fields_ = [
        ("n_dice", C.c_int),
        ("dice_labels", C.POINTER(C.c_int)),
        ("dice", C.POINTER(C.c_double)),
        ("n_hausdorff", C.c_int),
        ("hausdorff_labels", C.POINTER(C.c_int)),
        ("hausdorff_mm", C.POINTER(C.c_double)),
        ("jacobian_pct_nonpositive", C.c_double),
        ("runtime_seconds", C.c_double),
        ("velocity_count", C.c_int),
        ("config", ReportConfig),
    ]


def dims3(d) -> Dims3:
    """Accept Dims3, an (x, y, z) tuple (reference Dims3 order, NOT a numpy shape),
    or a numpy array of shape (z, y, x) / (z, y, x, 3)."""
    if isinstance(d, Dims3):
        return d
    if hasattr(d, "shape"):
        shp = d.shape
        if len(shp) == 4:  # (z, y, x, 3) AoS vector field
            shp = shp[:3]
        z, y, x = shp
        return Dims3(x, y, z)
    x, y, z = d
    return Dims3(int(x), int(y), int(z))


def solver_cfg(
    data_term: int = 1,
    order: int = 2,
    lambda_: float = 0.0,
    theta: float = 0.1,
    epsilon: float = 1e-6,
    max_iters: int = 100,
    tol: float = 0.0,
    accelerate: bool = True,
    log_objective: bool = True,
) -> SolverCfg:
    """SolverConfig with the reference defaults (admm.hpp:14-22)."""
    return SolverCfg(
        data_term, order, lambda_, theta, epsilon, max_iters, tol, int(accelerate), int(log_objective)
    )


def reg_cfg(
    solver: SolverCfg,
    levels: int = 1,
    max_warps=(5,),
    max_admm_iters=(50,),
    warp_improvement_threshold: float = 0.02,
    profile: int = DREG_PROFILE_CAPPED,
    smooth_levels: bool = True,
) -> RegCfg:
    c = RegCfg()
    c.solver = solver
    c.levels = levels
    for i, v in enumerate(max_warps):
        c.max_warps_per_level[i] = v
    for i, v in enumerate(max_admm_iters):
        c.max_admm_iters_per_level[i] = v
    c.warp_improvement_threshold = warp_improvement_threshold
    c.profile = profile
    c.smooth_levels = int(smooth_levels)
    return c


def level_logs(res: PairResult) -> list[dict]:
    out = []
    for l in range(res.levels):
        lg = res.per_level[l]
        out.append(
            {
                "dims": (lg.dims.x, lg.dims.y, lg.dims.z),
                "warps": lg.warps,
                "mean_sad": [lg.mean_sad[i] for i in range(min(lg.warps, DREG_MAX_WARPS) + 1)],
                "solver_iterations": [lg.solver_iterations[i] for i in range(min(lg.warps, DREG_MAX_WARPS))],
            }
        )
    return out
