"""Python mirror of the reference `dreg` hot-path API over the C ABI (include/dreg_cuda.h).

Same function names, argument meaning and error behaviour as the reference C++
library (proj/core/include/dreg/*.hpp):

  ValueError    <- std::invalid_argument   (status DREG_INVALID_ARGUMENT)
  NumericError  <- dreg::numeric_error     (status DREG_NUMERIC, errors.hpp:15-17)
  IoError       <- dreg::io_error          (status DREG_IO_ERROR; file I/O only)
  RuntimeError  <- CUDA / allocation       (status DREG_RUNTIME)

Volumes are numpy float32 arrays shaped (z, y, x) (x fastest, volume.hpp:10) and
vector fields (z, y, x, 3) interleaved like the reference VectorField.  Every compute
call runs sm_100a kernels from paper_2109_12688_b200/lib/libdreg_cuda.so; there is no
CPU fallback -- a missing library or GPU raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import abi
from .abi import (  # noqa: F401  (re-exported config helpers)
    DREG_PROFILE_CAPPED,
    DREG_PROFILE_CONVERGED,
    Dims3,
    JacobianStats,
    PairResult,
    RegCfg,
    SolverCfg,
    Spacing3,
    level_logs,
    reg_cfg,
    solver_cfg,
)

_LIB_PATH = os.environ.get("DREG_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libdreg_cuda.so")
_F = C.POINTER(C.c_float)
_D = C.POINTER(C.c_double)
_lib = None


class NumericError(RuntimeError):
    """dreg::numeric_error: non-finite values produced or encountered."""


class IoError(RuntimeError):
    """dreg::io_error: unreadable / malformed / unwritable DREG files."""


def lib_path() -> str:
    return _LIB_PATH


def load_library() -> C.CDLL:
    """Load libdreg_cuda.so (built by __graft_entry__.build()); raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"{_LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = C.CDLL(_LIB_PATH)
    P, V = C.c_void_p, C.c_void_p
    L.dreg_cuda_ctx_create.argtypes = [C.c_int, C.POINTER(P)]
    L.dreg_cuda_ctx_destroy.argtypes = [P]
    L.dreg_cuda_ctx_destroy.restype = None
    L.dreg_cuda_last_error.argtypes = [P]
    L.dreg_cuda_last_error.restype = C.c_char_p
    L.dreg_cuda_set_stream.argtypes = [P, V]
    L.dreg_cuda_kernel_launches.argtypes = [P]
    L.dreg_cuda_kernel_launches.restype = C.c_int64
    L.dreg_cuda_set_batch_chunk.argtypes = [P, C.c_int]
    L.dreg_cuda_set_use_graphs.argtypes = [P, C.c_int]
    L.dreg_cuda_set_precision.argtypes = [P, C.c_int]
    L.dreg_nesterov_next_alpha.argtypes = [C.c_double]
    L.dreg_nesterov_next_alpha.restype = C.c_double
    L.dreg_validate_solver_cfg.argtypes = [C.POINTER(SolverCfg)]
    L.dreg_make_registration_config.argtypes = [C.c_int, C.POINTER(SolverCfg), C.c_int, C.POINTER(RegCfg)]
    L.dreg_laplacian_symbol.argtypes = [C.c_int, Dims3, _D]
    L.dreg_cuda_register_pair.argtypes = [P, _F, _F, Dims3, Spacing3, C.POINTER(RegCfg), _F, _F, C.POINTER(PairResult)]
    L.dreg_cuda_register_batch.argtypes = [
        P, C.c_int, C.POINTER(_F), C.POINTER(_F), Dims3, Spacing3, C.POINTER(RegCfg),
        C.POINTER(_F), C.POINTER(_F), C.POINTER(PairResult),
    ]
    L.dreg_cuda_register_batch_device.argtypes = [
        P, C.c_int, V, V, Dims3, Spacing3, C.POINTER(RegCfg), V, V, C.POINTER(PairResult),
    ]
    L.dreg_cuda_solve_velocity.argtypes = [P, _F, _F, Dims3, C.POINTER(SolverCfg), _F, C.POINTER(abi.SolverDiag)]
    L.dreg_cuda_time_kernels.argtypes = [P, C.c_int, _D]
    L.dreg_cuda_time_iteration.argtypes = [P, C.POINTER(SolverCfg), C.c_int, _D]
    L.dreg_cuda_v_update.argtypes = [P, _F, _F, _F, _F, _F, Dims3, C.POINTER(SolverCfg), _F]
    L.dreg_cuda_w_update.argtypes = [P, _F, _F, Dims3, C.POINTER(SolverCfg), _F]
    L.dreg_cuda_regulariser_energy.argtypes = [P, _F, Dims3, C.c_int, _D]
    L.dreg_cuda_data_term_value.argtypes = [P, _F, _F, _F, _F, Dims3, C.c_int, _D]
    L.dreg_cuda_trilinear_sample.argtypes = [P, _F, C.c_int, Dims3, _D, C.c_int64, _D]
    L.dreg_cuda_warp_image.argtypes = [P, _F, _F, Dims3, _F]
    L.dreg_cuda_image_gradient.argtypes = [P, _F, Dims3, _F]
    L.dreg_cuda_compose_deformation.argtypes = [P, _F, _F, Dims3, _F]
    L.dreg_cuda_jacobian.argtypes = [P, _F, Dims3, _F, C.POINTER(JacobianStats)]
    L.dreg_cuda_jacobian_device.argtypes = [P, V, Dims3, V, C.POINTER(JacobianStats)]
    L.dreg_cuda_normalize_intensity_pair.argtypes = [P, _F, _F, Dims3, _F, _F]
    L.dreg_cuda_binomial_smooth.argtypes = [P, _F, Dims3, _F]
    L.dreg_cuda_mean_sad.argtypes = [P, _F, _F, Dims3, _D]
    L.dreg_cuda_downsample.argtypes = [P, _F, Dims3, _F]
    L.dreg_cuda_upsample_velocity.argtypes = [P, _F, Dims3, Dims3, _F]
    CP, SZ = C.c_char_p, C.c_size_t
    L.dreg_volume_info_read.argtypes = [CP, C.POINTER(abi.VolumeInfo), CP, SZ]
    L.dreg_volume_read.argtypes = [CP, C.c_int, C.POINTER(abi.VolumeInfo), V, SZ, CP, SZ]
    L.dreg_volume_write.argtypes = [CP, C.c_int, Dims3, Spacing3, V, CP, SZ]
    L.dreg_report_write.argtypes = [CP, C.POINTER(abi.RunReport), CP, SZ]
    L.dreg_cuda_warp_labels.argtypes = [P, V, _F, Dims3, V]
    L.dreg_cuda_dice.argtypes = [P, V, V, Dims3, C.c_int, _D]
    L.dreg_cuda_hausdorff_slice_avg.argtypes = [P, V, V, Dims3, Spacing3, C.c_int, _D]
    L.dreg_cuda_label_metrics.argtypes = [P, V, V, Dims3, Spacing3, C.c_int, V, V, V, V]
    PR = C.POINTER(abi.PairRecord)
    L.dreg_cuda_multi_create.argtypes = [C.POINTER(C.c_int), C.c_int, C.POINTER(P)]
    L.dreg_cuda_multi_destroy.argtypes = [P]
    L.dreg_cuda_multi_destroy.restype = None
    L.dreg_cuda_multi_last_error.argtypes = [P]
    L.dreg_cuda_multi_last_error.restype = C.c_char_p
    L.dreg_cuda_multi_device_count.argtypes = [P]
    L.dreg_cuda_multi_register_batch.argtypes = [
        P, C.c_int, C.POINTER(_F), C.POINTER(_F), Dims3, Spacing3, C.POINTER(RegCfg),
        C.POINTER(_F), C.POINTER(_F), C.POINTER(PairResult), PR,
    ]
    L.dreg_shard_range.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]
    L.dreg_records_unpack.argtypes = [PR, C.c_int, C.c_int, C.c_int, PR]
    _lib = L
    return L


def _fp(a: np.ndarray):
    return a.ctypes.data_as(_F)


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def _raise(status: int, msg: str, results=None):
    """Map a status to the reference's exception types.  Batch calls attach every
    pair's result (per-pair `status`) to a NumericError as `.results`, so one bad pair
    does not lose the other pairs' outputs."""
    if status == abi.DREG_INVALID_ARGUMENT:
        raise ValueError(msg)
    if status == abi.DREG_NUMERIC:
        e = NumericError(msg)
        e.results = results
        raise e
    raise RuntimeError(msg or f"dreg_cuda status {status}")


# ---- pure host helpers (no device work) --------------------------------------------
def nesterov_next_alpha(alpha: float) -> float:
    """admm.cpp:198-200."""
    return load_library().dreg_nesterov_next_alpha(alpha)


def validate(cfg: SolverCfg) -> None:
    """admm.cpp:174-196: raises ValueError when a field is out of range."""
    if load_library().dreg_validate_solver_cfg(C.byref(cfg)) != abi.DREG_OK:
        raise ValueError("solver: invalid configuration")


def make_registration_config(profile: int, solver: SolverCfg, levels: int = 3) -> RegCfg:
    """registration.cpp:62-83."""
    out = RegCfg()
    if load_library().dreg_make_registration_config(profile, C.byref(solver), levels, C.byref(out)):
        raise ValueError("registration: levels must be in [1, 8]")
    return out


def laplacian_symbol(order: int, dims) -> np.ndarray:
    """regularizer.cpp:51-79 (full grid, fp64)."""
    d = abi.dims3(dims)
    out = np.zeros(d.shape(), np.float64)
    if load_library().dreg_laplacian_symbol(order, d, out.ctypes.data_as(_D)):
        raise ValueError("laplacian_symbol: order must be in [1, 6] and every axis >= 2")
    return out


# ---- DREG files and run reports (io.hpp; host only) ---------------------------------
_KIND_DTYPE = {abi.DREG_KIND_SCALAR: np.float32, abi.DREG_KIND_VECTOR: np.float32, abi.DREG_KIND_LABEL: np.uint16}
_KIND_OF = {"scalar": abi.DREG_KIND_SCALAR, "vector": abi.DREG_KIND_VECTOR, "label": abi.DREG_KIND_LABEL}


def _io_check(st: int, err) -> None:
    if st == abi.DREG_OK:
        return
    msg = err.value.decode(errors="replace")
    if st == abi.DREG_IO_ERROR:
        raise IoError(msg)
    _raise(st, msg)


def read_volume(path, expected_kind: int = -1):
    """read_volume / read_scalar / read_vector / read_label (io.hpp:27-35).

    Returns (kind, array, spacing): float32 (z, y, x) for scalars, float32 (z, y, x, 3)
    for vector fields, uint16 (z, y, x) for labels; spacing = (sx, sy, sz)."""
    L = load_library()
    err = C.create_string_buffer(1024)
    info = abi.VolumeInfo()
    p = os.fsencode(str(path))
    _io_check(L.dreg_volume_read(p, int(expected_kind), C.byref(info), None, 0, err, 1024), err)
    shape = info.dims.shape() + ((3,) if info.kind == abi.DREG_KIND_VECTOR else ())
    out = np.empty(shape, _KIND_DTYPE[info.kind])
    _io_check(L.dreg_volume_read(p, int(expected_kind), C.byref(info), out.ctypes.data, out.nbytes, err, 1024), err)
    return info.kind, out, (info.spacing.x, info.spacing.y, info.spacing.z)


def read_scalar(path):
    return read_volume(path, abi.DREG_KIND_SCALAR)[1:]


def read_vector(path):
    return read_volume(path, abi.DREG_KIND_VECTOR)[1:]


read_deformation = read_vector


def read_label(path):
    return read_volume(path, abi.DREG_KIND_LABEL)[1:]


def write_volume(path, data, spacing=(1.0, 1.0, 1.0), kind: str | None = None) -> None:
    """write_volume (io.hpp:37-40).  kind defaults from the array: uint16 -> label,
    (z, y, x, 3) float -> vector, (z, y, x) float -> scalar."""
    if kind is None:
        a = np.asarray(data)
        kind = "label" if a.dtype == np.uint16 else ("vector" if a.ndim == 4 else "scalar")
    k = _KIND_OF[kind]
    a = np.ascontiguousarray(data, dtype=_KIND_DTYPE[k])
    err = C.create_string_buffer(1024)
    st = load_library().dreg_volume_write(os.fsencode(str(path)), k, abi.dims3(a), Spacing3(*spacing),
                                          a.ctypes.data, err, 1024)
    _io_check(st, err)


def write_report(path, *, dice=None, hausdorff_mm=None, jacobian_pct_nonpositive=0.0, runtime_seconds=0.0,
                 velocity_count=0, data_term="l1", order=0, lambda_=0.0, theta=0.0, levels=0, profile="capped",
                 tol=0.0, warp_improvement_threshold=0.0, epsilon=0.0, threads=1) -> None:
    """write_report (io.hpp:64-66); dice / hausdorff_mm map label -> value."""
    dice = dict(dice or {})
    hd = dict(hausdorff_mm or {})
    dl = (C.c_int * max(len(dice), 1))(*dice.keys())
    dv = (C.c_double * max(len(dice), 1))(*dice.values())
    hl = (C.c_int * max(len(hd), 1))(*hd.keys())
    hv = (C.c_double * max(len(hd), 1))(*hd.values())
    cfg = abi.ReportConfig(data_term.encode(), order, lambda_, theta, levels, profile.encode(), tol,
                           warp_improvement_threshold, epsilon, threads)
    rep = abi.RunReport(len(dice), dl, dv, len(hd), hl, hv, jacobian_pct_nonpositive, runtime_seconds,
                        velocity_count, cfg)
    err = C.create_string_buffer(1024)
    _io_check(load_library().dreg_report_write(os.fsencode(str(path)), C.byref(rep), err, 1024), err)


def shard_range(n_pairs: int, n_shards: int, shard: int) -> tuple[int, int]:
    """[begin, end) of a shard's contiguous pair block (dreg_shard_range)."""
    b, e = C.c_int(), C.c_int()
    st = load_library().dreg_shard_range(n_pairs, n_shards, shard, C.byref(b), C.byref(e))
    if st != abi.DREG_OK:
        raise ValueError("dreg_shard_range: bad arguments")
    return b.value, e.value


class MultiContext:
    """Pairs sharded over several GPUs (dreg_cuda_multi): one host thread + context per
    device inside the library, one NCCL all-gather of the per-pair records."""

    def __init__(self, devices):
        self.lib = load_library()
        devs = (C.c_int * len(devices))(*devices)
        h = C.c_void_p()
        st = self.lib.dreg_cuda_multi_create(devs, len(devices), C.byref(h))
        if st != abi.DREG_OK:
            raise RuntimeError(f"dreg_cuda_multi_create({list(devices)}) failed with status {st}")
        self.h = h
        self.devices = list(devices)

    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.dreg_cuda_multi_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def register_batch(self, targets, sources, cfg: RegCfg, spacing=(1.0, 1.0, 1.0)):
        """-> (phis, warped, results, records), records in pair order."""
        targets = [_f32(t) for t in targets]
        sources = [_f32(s) for s in sources]
        n = len(targets)
        shape = targets[0].shape
        phis = [np.zeros(shape + (3,), np.float32) for _ in range(n)]
        warps = [np.zeros(shape, np.float32) for _ in range(n)]
        T = (_F * n)(*[_fp(t) for t in targets])
        S = (_F * n)(*[_fp(s) for s in sources])
        PO = (_F * n)(*[_fp(p) for p in phis])
        WO = (_F * n)(*[_fp(w) for w in warps])
        res = (PairResult * n)()
        rec = (abi.PairRecord * n)()
        st = self.lib.dreg_cuda_multi_register_batch(self.h, n, T, S, abi.dims3(targets[0]), Spacing3(*spacing),
                                                     C.byref(cfg), PO, WO, res, rec)
        if st != abi.DREG_OK:
            _raise(st, self.lib.dreg_cuda_multi_last_error(self.h).decode(),
                   (phis, warps, list(res), list(rec)) if st == abi.DREG_NUMERIC else None)
        return phis, warps, list(res), list(rec)


class Context:
    """One CUDA device context (dreg_cuda_ctx).  Not thread-safe; one per thread/GPU."""

    def __init__(self, device: int = 0):
        self.lib = load_library()
        h = C.c_void_p()
        st = self.lib.dreg_cuda_ctx_create(int(device), C.byref(h))
        if st != abi.DREG_OK:
            raise RuntimeError(f"dreg_cuda_ctx_create(device={device}) failed with status {st} (no sm_100 GPU?)")
        self.h = h
        self.device = device

    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.dreg_cuda_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _check(self, st: int) -> None:
        if st != abi.DREG_OK:
            _raise(st, self.lib.dreg_cuda_last_error(self.h).decode())

    # ---- host helpers (same names as the module functions / reference API) --------
    nesterov_next_alpha = staticmethod(nesterov_next_alpha)
    validate = staticmethod(validate)
    make_registration_config = staticmethod(make_registration_config)
    laplacian_symbol = staticmethod(laplacian_symbol)

    # ---- context knobs ---------------------------------------------------------
    def kernel_launches(self) -> int:
        return int(self.lib.dreg_cuda_kernel_launches(self.h))

    def set_stream(self, stream_ptr: int | None) -> None:
        self._check(self.lib.dreg_cuda_set_stream(self.h, C.c_void_p(stream_ptr or 0)))

    def set_batch_chunk(self, pairs: int) -> None:
        self._check(self.lib.dreg_cuda_set_batch_chunk(self.h, pairs))

    def set_precision(self, mode: int) -> None:
        """0 auto (fp64 spectral arithmetic for solves > 100 iterations), 1 fp32, 2 fp64."""
        self._check(self.lib.dreg_cuda_set_precision(self.h, int(mode)))

    def set_use_graphs(self, enable: bool) -> None:
        self._check(self.lib.dreg_cuda_set_use_graphs(self.h, int(enable)))

    # ---- hot path ----------------------------------------------------------------
    def register_pair(self, target, source, cfg: RegCfg, spacing=(1.0, 1.0, 1.0)):
        """registration.hpp:74-75 -> (phi (z,y,x,3), warped (z,y,x), PairResult)."""
        target, source = _f32(target), _f32(source)
        if target.shape != source.shape:
            raise ValueError("register_pair: dimension mismatch")
        phi = np.zeros(target.shape + (3,), np.float32)
        warped = np.zeros_like(target)
        res = PairResult()
        self._check(
            self.lib.dreg_cuda_register_pair(
                self.h, _fp(target), _fp(source), abi.dims3(target), Spacing3(*spacing), C.byref(cfg),
                _fp(phi), _fp(warped), C.byref(res),
            )
        )
        return phi, warped, res

    def register_batch(self, targets, sources, cfg: RegCfg, want_phi=True, want_warped=True, spacing=(1.0, 1.0, 1.0)):
        """n independent registrations (same dims/cfg) from host buffers."""
        targets = [_f32(t) for t in targets]
        sources = [_f32(s) for s in sources]
        n = len(targets)
        if n == 0:
            return [], [], []
        shape = targets[0].shape
        if any(t.shape != shape for t in targets) or any(s.shape != shape for s in sources):
            raise ValueError("register_batch: dimension mismatch")
        phis = [np.zeros(shape + (3,), np.float32) for _ in range(n)] if want_phi else None
        warps = [np.zeros(shape, np.float32) for _ in range(n)] if want_warped else None
        T = (_F * n)(*[_fp(t) for t in targets])
        S = (_F * n)(*[_fp(s) for s in sources])
        PO = (_F * n)(*[_fp(p) for p in phis]) if phis else None
        WO = (_F * n)(*[_fp(w) for w in warps]) if warps else None
        res = (PairResult * n)()
        st = self.lib.dreg_cuda_register_batch(self.h, n, T, S, abi.dims3(targets[0]), Spacing3(*spacing),
                                               C.byref(cfg), PO, WO, res)
        if st != abi.DREG_OK:
            _raise(st, self.lib.dreg_cuda_last_error(self.h).decode(),
                   (phis, warps, list(res)) if st == abi.DREG_NUMERIC else None)
        return phis, warps, list(res)

    def register_batch_device(self, n: int, targets_ptr: int, sources_ptr: int, dims, cfg: RegCfg,
                              phi_ptr: int = 0, warped_ptr: int = 0):
        """Device-resident batch: [n][voxels] inputs, [n][3][voxels] SoA phi output."""
        res = (PairResult * n)()
        st = self.lib.dreg_cuda_register_batch_device(
            self.h, n, C.c_void_p(targets_ptr), C.c_void_p(sources_ptr), abi.dims3(dims), Spacing3(1, 1, 1),
            C.byref(cfg), C.c_void_p(phi_ptr or 0), C.c_void_p(warped_ptr or 0), res,
        )
        if st != abi.DREG_OK:
            _raise(st, self.lib.dreg_cuda_last_error(self.h).decode(), list(res) if st == abi.DREG_NUMERIC else None)
        return list(res)

    def solve_velocity(self, target, warped_source, cfg: SolverCfg):
        """admm.hpp:76-77 -> (velocity (z,y,x,3), diagnostics dict)."""
        target, warped_source = _f32(target), _f32(warped_source)
        if target.shape != warped_source.shape:
            raise ValueError("solve_velocity: dimension mismatch")
        v = np.zeros(target.shape + (3,), np.float32)
        n = max(cfg.max_iters, 1)
        obj = np.zeros(n, np.float64)
        res = np.zeros(n, np.float64)
        diag = abi.SolverDiag(0, 0.0, 0, obj.ctypes.data_as(_D), res.ctypes.data_as(_D))
        self._check(
            self.lib.dreg_cuda_solve_velocity(
                self.h, _fp(target), _fp(warped_source), abi.dims3(target), C.byref(cfg), _fp(v), C.byref(diag)
            )
        )
        it = diag.iterations
        return v, {
            "iterations": it,
            "final_change": diag.final_change,
            "converged": bool(diag.converged),
            "objective": obj[:it].copy() if cfg.log_objective else np.zeros(0),
            "constraint_residual": res[:it].copy(),
        }

    def time_kernels(self, reps: int = 20, solver: SolverCfg | None = None) -> dict:
        """CUDA-event timing of the per-iteration kernels on the current workspace
        (with `solver`'s parameters and precision policy when given)."""
        out = np.zeros(7, np.float64)
        if solver is None:
            self._check(self.lib.dreg_cuda_time_kernels(self.h, reps, out.ctypes.data_as(_D)))
        else:
            self._check(self.lib.dreg_cuda_time_iteration(self.h, C.byref(solver), reps, out.ctypes.data_as(_D)))
        return {"xpass_ms": out[0], "plane_ms": out[1], "xpass_bytes": out[2], "plane_bytes": out[3],
                "pairs": int(out[4]), "precise": int(out[5]), "spectral_state": int(out[6])}

    # ---- building blocks ---------------------------------------------------------
    def v_update(self, target, warped, grad, w_hat, b_hat, cfg: SolverCfg) -> np.ndarray:
        target, warped, grad, w_hat, b_hat = map(_f32, (target, warped, grad, w_hat, b_hat))
        out = np.zeros_like(grad)
        self._check(
            self.lib.dreg_cuda_v_update(
                self.h, _fp(target), _fp(warped), _fp(grad), _fp(w_hat), _fp(b_hat), abi.dims3(target),
                C.byref(cfg), _fp(out),
            )
        )
        return out

    def v_update_l1(self, target, warped, grad, w_hat, b_hat, cfg: SolverCfg) -> np.ndarray:
        c = SolverCfg.from_buffer_copy(cfg)
        c.data_term = 1
        return self.v_update(target, warped, grad, w_hat, b_hat, c)

    def v_update_l2(self, target, warped, grad, w_hat, b_hat, cfg: SolverCfg) -> np.ndarray:
        c = SolverCfg.from_buffer_copy(cfg)
        c.data_term = 2
        return self.v_update(target, warped, grad, w_hat, b_hat, c)

    def w_update(self, v, b_hat, cfg: SolverCfg) -> np.ndarray:
        v, b_hat = _f32(v), _f32(b_hat)
        out = np.zeros_like(v)
        self._check(self.lib.dreg_cuda_w_update(self.h, _fp(v), _fp(b_hat), abi.dims3(v), C.byref(cfg), _fp(out)))
        return out

    def data_term_value(self, target, warped, grad, v, s: int) -> float:
        """admm.hpp:68 / admm.cpp:239-250."""
        target, warped, grad, v = map(_f32, (target, warped, grad, v))
        out = C.c_double()
        self._check(self.lib.dreg_cuda_data_term_value(self.h, _fp(target), _fp(warped), _fp(grad), _fp(v),
                                                       abi.dims3(target), int(s), C.byref(out)))
        return out.value

    def trilinear_sample(self, field, points) -> np.ndarray:
        """volume.hpp:107,110 at points [n, 3] (x, y, z): scalar field (z,y,x) -> [n];
        vector field (z,y,x,3) -> [n, 3]."""
        field = _f32(field)
        pts = np.ascontiguousarray(points, np.float64).reshape(-1, 3)
        ncomp = 3 if field.ndim == 4 else 1
        out = np.zeros((pts.shape[0], 3) if ncomp == 3 else pts.shape[0], np.float64)
        dims = abi.dims3(field[..., 0] if ncomp == 3 else field)
        self._check(self.lib.dreg_cuda_trilinear_sample(self.h, _fp(field), ncomp, dims, pts.ctypes.data_as(_D),
                                                        pts.shape[0], out.ctypes.data_as(_D)))
        return out

    def regulariser_energy(self, w, order: int) -> float:
        w = _f32(w)
        out = C.c_double()
        self._check(self.lib.dreg_cuda_regulariser_energy(self.h, _fp(w), abi.dims3(w), order, C.byref(out)))
        return out.value

    def warp_image(self, img, disp) -> np.ndarray:
        img, disp = _f32(img), _f32(disp)
        if disp.shape[:3] != img.shape:
            raise ValueError("warp_image: dimension mismatch")
        out = np.zeros_like(img)
        self._check(self.lib.dreg_cuda_warp_image(self.h, _fp(img), _fp(disp), abi.dims3(img), _fp(out)))
        return out

    def image_gradient(self, img) -> np.ndarray:
        img = _f32(img)
        out = np.zeros(img.shape + (3,), np.float32)
        self._check(self.lib.dreg_cuda_image_gradient(self.h, _fp(img), abi.dims3(img), _fp(out)))
        return out

    def compose_deformation(self, disp, v) -> np.ndarray:
        disp, v = _f32(disp), _f32(v)
        if disp.shape != v.shape:
            raise ValueError("compose_deformation: dimension mismatch")
        out = np.zeros_like(disp)
        self._check(self.lib.dreg_cuda_compose_deformation(self.h, _fp(disp), _fp(v), abi.dims3(disp), _fp(out)))
        return out

    def jacobian_determinant(self, disp) -> np.ndarray:
        disp = _f32(disp)
        out = np.zeros(disp.shape[:3], np.float32)
        self._check(self.lib.dreg_cuda_jacobian(self.h, _fp(disp), abi.dims3(disp), _fp(out), None))
        return out

    def jacobian_stats(self, disp) -> JacobianStats:
        disp = _f32(disp)
        st = JacobianStats()
        self._check(self.lib.dreg_cuda_jacobian(self.h, _fp(disp), abi.dims3(disp), None, C.byref(st)))
        return st

    def jacobian_stats_device(self, disp_soa_ptr: int, dims) -> JacobianStats:
        """Folding statistics of a device-resident SoA displacement [3][voxels]."""
        st = JacobianStats()
        self._check(self.lib.dreg_cuda_jacobian_device(self.h, C.c_void_p(disp_soa_ptr), abi.dims3(dims), None, C.byref(st)))
        return st

    def normalize_intensity_pair(self, a, b):
        a, b = _f32(a), _f32(b)
        if a.shape != b.shape:
            raise ValueError("normalize_intensity_pair: dimension mismatch")
        oa, ob = np.zeros_like(a), np.zeros_like(b)
        self._check(self.lib.dreg_cuda_normalize_intensity_pair(self.h, _fp(a), _fp(b), abi.dims3(a), _fp(oa), _fp(ob)))
        return oa, ob

    def binomial_smooth(self, img) -> np.ndarray:
        img = _f32(img)
        out = np.zeros_like(img)
        self._check(self.lib.dreg_cuda_binomial_smooth(self.h, _fp(img), abi.dims3(img), _fp(out)))
        return out

    def mean_sad(self, a, b) -> float:
        a, b = _f32(a), _f32(b)
        if a.shape != b.shape:
            raise ValueError("mean_sad: dimension mismatch")
        out = C.c_double()
        self._check(self.lib.dreg_cuda_mean_sad(self.h, _fp(a), _fp(b), abi.dims3(a), C.byref(out)))
        return out.value

    def downsample(self, img) -> np.ndarray:
        img = _f32(img)
        z, y, x = img.shape
        out = np.zeros(((z + 1) // 2, (y + 1) // 2, (x + 1) // 2), np.float32)
        self._check(self.lib.dreg_cuda_downsample(self.h, _fp(img), abi.dims3(img), _fp(out)))
        return out

    def upsample_velocity(self, v, dst_dims) -> np.ndarray:
        v = _f32(v)
        dd = abi.dims3(dst_dims)
        out = np.zeros(dd.shape() + (3,), np.float32)
        self._check(self.lib.dreg_cuda_upsample_velocity(self.h, _fp(v), abi.dims3(v), dd, _fp(out)))
        return out

    # ---- label metrics (metrics.hpp:31-42) ----------------------------------------
    def warp_labels(self, labels, disp) -> np.ndarray:
        """Nearest-neighbour label warp at x + disp(x) (metrics.cpp:182-204)."""
        lbl = np.ascontiguousarray(labels, dtype=np.uint16)
        disp = _f32(disp)
        if disp.shape != lbl.shape + (3,):
            raise ValueError("warp_labels: dimension mismatch")
        out = np.empty_like(lbl)
        self._check(self.lib.dreg_cuda_warp_labels(self.h, lbl.ctypes.data, _fp(disp), abi.dims3(lbl), out.ctypes.data))
        return out

    def label_metrics(self, a, b, labels, spacing=(1.0, 1.0, 1.0)):
        """Dice and slice-averaged Hausdorff for every label in one upload.
        Returns (dice[list], hausdorff[list], valid[list])."""
        a = np.ascontiguousarray(a, dtype=np.uint16)
        b = np.ascontiguousarray(b, dtype=np.uint16)
        if a.shape != b.shape:
            raise ValueError("label metrics: dimension mismatch")
        lab = np.ascontiguousarray(list(labels), dtype=np.int32)
        n = len(lab)
        dice = np.zeros(max(n, 1), np.float64)
        hd = np.zeros(max(n, 1), np.float64)
        ok = np.zeros(max(n, 1), np.int32)
        self._check(self.lib.dreg_cuda_label_metrics(self.h, a.ctypes.data, b.ctypes.data, abi.dims3(a),
                                                     Spacing3(*spacing), n, lab.ctypes.data, dice.ctypes.data,
                                                     hd.ctypes.data, ok.ctypes.data))
        return dice[:n].tolist(), hd[:n].tolist(), [bool(v) for v in ok[:n]]

    def dice(self, a, b, label: int) -> float:
        """2|A n B| / (|A| + |B|); 1 when both masks are empty (metrics.cpp:131-147)."""
        a = np.ascontiguousarray(a, dtype=np.uint16)
        b = np.ascontiguousarray(b, dtype=np.uint16)
        if a.shape != b.shape:
            raise ValueError("dice: dimension mismatch")
        out = C.c_double()
        self._check(self.lib.dreg_cuda_dice(self.h, a.ctypes.data, b.ctypes.data, abi.dims3(a), int(label),
                                            C.byref(out)))
        return out.value

    def hausdorff_slice_avg(self, a, b, label: int, spacing=(1.0, 1.0, 1.0)) -> float:
        """Per-z-slice symmetric Hausdorff (mm, in-plane spacing), averaged over slices
        where both masks are non-empty; ValueError when none is (metrics.cpp:149-180)."""
        a = np.ascontiguousarray(a, dtype=np.uint16)
        b = np.ascontiguousarray(b, dtype=np.uint16)
        if a.shape != b.shape:
            raise ValueError("hausdorff_slice_avg: dimension mismatch")
        out = C.c_double()
        self._check(self.lib.dreg_cuda_hausdorff_slice_avg(self.h, a.ctypes.data, b.ctypes.data, abi.dims3(a),
                                                           Spacing3(*spacing), int(label), C.byref(out)))
        return out.value
