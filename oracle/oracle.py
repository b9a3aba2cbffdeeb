"""TEST INFRASTRUCTURE ONLY -- Python loader for the CPU oracle libraries.

  CpuLib("oracle")    -> oracle/lib/libdreg_oracle.so  (plain-C restatement, dro_*)
  CpuLib("reference") -> oracle/_ref/libdreg_ref.so    (unmodified reference, ref_*)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this module, and only as the checker or the CPU baseline.  Both
libraries expose the same signatures; volumes are numpy float32 arrays shaped
(z, y, x) and vector fields (z, y, x, 3) (AoS, like the reference VectorField).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import sys

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_HERE)
if _ROOT not in sys.path:
    sys.path.insert(0, _ROOT)

from paper_2109_12688_b200 import abi  # noqa: E402

_PATHS = {
    "oracle": (os.path.join(_HERE, "lib", "libdreg_oracle.so"), "dro_"),
    "reference": (os.path.join(_HERE, "_ref", "libdreg_ref.so"), "ref_"),
    # same reference objects over MKL DFTI (timing only; see fftw_shim/fftw_mkl.c)
    "reference_mkl": (os.path.join(_HERE, "_ref", "libdreg_ref_mkl.so"), "ref_"),
}

_F = C.POINTER(C.c_float)
_D = C.POINTER(C.c_double)


class OracleError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"status {status}: {msg}")
        self.status = status


def build(reference: bool = True) -> None:
    """make -C oracle (and `ref` when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    if reference and os.path.isdir("/root/reference/proj/core/src"):
        subprocess.run(["make", "-s", "-C", _HERE, "ref"], check=True)


def available(kind: str) -> bool:
    return os.path.exists(_PATHS[kind][0])


def _fp(a: np.ndarray):
    return a.ctypes.data_as(_F)


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


class CpuLib:
    def __init__(self, kind: str = "oracle"):
        path, prefix = _PATHS[kind]
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing; run `make -C oracle{' ref' if kind == 'reference' else ''}`")
        self.kind = kind
        self.lib = C.CDLL(path)
        self.p = prefix
        L = self.lib
        g = lambda n: getattr(L, prefix + n)  # noqa: E731
        self._g = g
        g("last_error").restype = C.c_char_p
        g("nesterov_next_alpha").restype = C.c_double
        g("nesterov_next_alpha").argtypes = [C.c_double]
        for n in [
            "validate",
            "make_registration_config",
            "laplacian_symbol",
            "regulariser_energy",
            "v_update",
            "w_update",
            "data_term_value",
            "trilinear_sample",
            "solve_velocity",
            "warp_image",
            "image_gradient",
            "compose_deformation",
            "jacobian",
            "normalize_intensity_pair",
            "binomial_smooth",
            "mean_sad",
            "downsample",
            "upsample_velocity",
            "register_pair",
        ]:
            g(n).restype = C.c_int
        if kind in ("reference", "reference_mkl"):
            L.ref_set_thread_count.argtypes = [C.c_int]
            L.ref_hardware_threads.restype = C.c_int

    # -- helpers ---------------------------------------------------------------
    def _check(self, st: int) -> None:
        if st != abi.DREG_OK:
            raise OracleError(st, self._g("last_error")().decode())

    def set_threads(self, n: int) -> None:
        if self.kind in ("reference", "reference_mkl"):
            self.lib.ref_set_thread_count(int(n))

    # -- API mirror ------------------------------------------------------------
    def nesterov_next_alpha(self, a: float) -> float:
        return self._g("nesterov_next_alpha")(a)

    def validate(self, cfg: abi.SolverCfg) -> None:
        self._check(self._g("validate")(C.byref(cfg)))

    def make_registration_config(self, profile: int, solver: abi.SolverCfg, levels: int = 3) -> abi.RegCfg:
        out = abi.RegCfg()
        self._check(self._g("make_registration_config")(profile, C.byref(solver), levels, C.byref(out)))
        return out

    def laplacian_symbol(self, order: int, dims) -> np.ndarray:
        d = abi.dims3(dims)
        out = np.zeros(d.shape(), np.float64)
        self._check(self._g("laplacian_symbol")(order, d, out.ctypes.data_as(_D)))
        return out

    def regulariser_energy(self, w: np.ndarray, order: int) -> float:
        w = _f32(w)
        out = C.c_double()
        self._check(self._g("regulariser_energy")(_fp(w), abi.dims3(w), order, C.byref(out)))
        return out.value

    def v_update(self, target, warped, grad, w_hat, b_hat, cfg: abi.SolverCfg) -> np.ndarray:
        target, warped, grad, w_hat, b_hat = map(_f32, (target, warped, grad, w_hat, b_hat))
        out = np.zeros_like(grad)
        self._check(
            self._g("v_update")(
                _fp(target), _fp(warped), _fp(grad), _fp(w_hat), _fp(b_hat), abi.dims3(target), C.byref(cfg), _fp(out)
            )
        )
        return out

    def w_update(self, v, b_hat, cfg: abi.SolverCfg) -> np.ndarray:
        v, b_hat = _f32(v), _f32(b_hat)
        out = np.zeros_like(v)
        self._check(self._g("w_update")(_fp(v), _fp(b_hat), abi.dims3(v), C.byref(cfg), _fp(out)))
        return out

    def data_term_value(self, target, warped, grad, v, s: int) -> float:
        target, warped, grad, v = map(_f32, (target, warped, grad, v))
        out = C.c_double()
        self._check(
            self._g("data_term_value")(_fp(target), _fp(warped), _fp(grad), _fp(v), abi.dims3(target), s, C.byref(out))
        )
        return out.value

    def trilinear_sample(self, field, points) -> np.ndarray:
        field = _f32(field)
        pts = np.ascontiguousarray(points, np.float64).reshape(-1, 3)
        ncomp = 3 if field.ndim == 4 else 1
        out = np.zeros((pts.shape[0], 3) if ncomp == 3 else pts.shape[0], np.float64)
        dims = abi.dims3(field[..., 0] if ncomp == 3 else field)
        self._check(self._g("trilinear_sample")(_fp(field), ncomp, dims, pts.ctypes.data_as(_D), C.c_int64(pts.shape[0]),
                                                out.ctypes.data_as(_D)))
        return out

    def solve_velocity(self, target, warped, cfg: abi.SolverCfg):
        target, warped = _f32(target), _f32(warped)
        out = np.zeros(target.shape + (3,), np.float32)
        obj = np.zeros(max(cfg.max_iters, 1), np.float64)
        res = np.zeros(max(cfg.max_iters, 1), np.float64)
        diag = abi.SolverDiag(0, 0.0, 0, obj.ctypes.data_as(_D), res.ctypes.data_as(_D))
        self._check(
            self._g("solve_velocity")(_fp(target), _fp(warped), abi.dims3(target), C.byref(cfg), _fp(out), C.byref(diag))
        )
        it = diag.iterations
        return out, {
            "iterations": it,
            "final_change": diag.final_change,
            "converged": bool(diag.converged),
            "objective": obj[:it].copy() if cfg.log_objective else np.zeros(0),
            "constraint_residual": res[:it].copy(),
        }

    def warp_image(self, img, disp) -> np.ndarray:
        img, disp = _f32(img), _f32(disp)
        out = np.zeros_like(img)
        self._check(self._g("warp_image")(_fp(img), _fp(disp), abi.dims3(img), _fp(out)))
        return out

    def image_gradient(self, img) -> np.ndarray:
        img = _f32(img)
        out = np.zeros(img.shape + (3,), np.float32)
        self._check(self._g("image_gradient")(_fp(img), abi.dims3(img), _fp(out)))
        return out

    def compose_deformation(self, disp, v) -> np.ndarray:
        disp, v = _f32(disp), _f32(v)
        out = np.zeros_like(disp)
        self._check(self._g("compose_deformation")(_fp(disp), _fp(v), abi.dims3(disp), _fp(out)))
        return out

    def jacobian_determinant(self, disp) -> np.ndarray:
        disp = _f32(disp)
        out = np.zeros(disp.shape[:3], np.float32)
        self._check(self._g("jacobian")(_fp(disp), abi.dims3(disp), _fp(out), None))
        return out

    def jacobian_stats(self, disp) -> abi.JacobianStats:
        disp = _f32(disp)
        st = abi.JacobianStats()
        self._check(self._g("jacobian")(_fp(disp), abi.dims3(disp), None, C.byref(st)))
        return st

    def normalize_intensity_pair(self, a, b):
        a, b = _f32(a), _f32(b)
        oa, ob = np.zeros_like(a), np.zeros_like(b)
        self._check(self._g("normalize_intensity_pair")(_fp(a), _fp(b), abi.dims3(a), _fp(oa), _fp(ob)))
        return oa, ob

    def binomial_smooth(self, img) -> np.ndarray:
        img = _f32(img)
        out = np.zeros_like(img)
        self._check(self._g("binomial_smooth")(_fp(img), abi.dims3(img), _fp(out)))
        return out

    def mean_sad(self, a, b) -> float:
        a, b = _f32(a), _f32(b)
        out = C.c_double()
        self._check(self._g("mean_sad")(_fp(a), _fp(b), abi.dims3(a), C.byref(out)))
        return out.value

    def downsample(self, img) -> np.ndarray:
        img = _f32(img)
        z, y, x = img.shape
        out = np.zeros(((z + 1) // 2, (y + 1) // 2, (x + 1) // 2), np.float32)
        self._check(self._g("downsample")(_fp(img), abi.dims3(img), _fp(out)))
        return out

    def upsample_velocity(self, v, dst_dims) -> np.ndarray:
        v = _f32(v)
        dd = abi.dims3(dst_dims)
        out = np.zeros(dd.shape() + (3,), np.float32)
        self._check(self._g("upsample_velocity")(_fp(v), abi.dims3(v), dd, _fp(out)))
        return out

    # ---- reference-only helpers (oracle/_ref): the reference's synthetic cases ----
    def make_case(self, kind: str, shape, shift=(0.0, 0.0, 0.0), seed: int = 0):
        """synth.hpp make_translate_case / make_sphere_ellipsoid_case / make_random_smooth_case
        -> (target, source, target_labels, source_labels), arrays (z, y, x)."""
        if self.kind != "reference":
            raise RuntimeError("make_case needs the reference library")
        k = {"translate": 0, "sphere_ellipsoid": 1, "random_smooth": 2}[kind]
        t, s = np.zeros(shape, np.float32), np.zeros(shape, np.float32)
        tl, sl = np.zeros(shape, np.uint16), np.zeros(shape, np.uint16)
        sh = (C.c_double * 3)(*shift)
        u16 = C.POINTER(C.c_ushort)
        f = self.lib.ref_make_case
        f.argtypes = [C.c_int, abi.Dims3, C.POINTER(C.c_double), C.c_uint, _F, _F, u16, u16]
        self._check(f(k, abi.dims3(t), sh, seed, _fp(t), _fp(s), tl.ctypes.data_as(u16), sl.ctypes.data_as(u16)))
        return t, s, tl, sl

    def warped_label_dice(self, moving_labels, disp, fixed_labels, label: int = 1) -> float:
        """metrics.hpp:31,39: dice(warp_labels(moving, phi), fixed, label)."""
        u16 = C.POINTER(C.c_ushort)
        m = np.ascontiguousarray(moving_labels, np.uint16)
        fx = np.ascontiguousarray(fixed_labels, np.uint16)
        disp = _f32(disp)
        out = C.c_double()
        f = self.lib.ref_warped_label_dice
        f.argtypes = [u16, _F, u16, abi.Dims3, C.c_int, C.POINTER(C.c_double)]
        self._check(f(m.ctypes.data_as(u16), _fp(disp), fx.ctypes.data_as(u16), abi.dims3(m), label, C.byref(out)))
        return out.value

    # ---- reference-only: label metrics, DREG files, reports, salt-and-pepper ------
    def _ref(self):
        if self.kind != "reference":
            raise RuntimeError("needs the reference library (oracle/_ref)")
        return self.lib

    def add_salt_pepper(self, vol, fraction: float, seed: int) -> np.ndarray:
        """synth.hpp add_salt_pepper on a copy of vol."""
        v = _f32(vol).copy()
        f = self._ref().ref_add_salt_pepper
        f.argtypes = [_F, abi.Dims3, C.c_double, C.c_uint]
        self._check(f(_fp(v), abi.dims3(v), fraction, seed))
        return v

    def dice(self, a, b, label: int) -> float:
        a, b = np.ascontiguousarray(a, np.uint16), np.ascontiguousarray(b, np.uint16)
        f = self._ref().ref_dice
        f.argtypes = [C.c_void_p, C.c_void_p, abi.Dims3, C.c_int, _D]
        out = C.c_double()
        self._check(f(a.ctypes.data, b.ctypes.data, abi.dims3(a), label, C.byref(out)))
        return out.value

    def hausdorff_slice_avg(self, a, b, label: int, spacing=(1.0, 1.0, 1.0)) -> float:
        a, b = np.ascontiguousarray(a, np.uint16), np.ascontiguousarray(b, np.uint16)
        f = self._ref().ref_hausdorff_slice_avg
        f.argtypes = [C.c_void_p, C.c_void_p, abi.Dims3, abi.Spacing3, C.c_int, _D]
        out = C.c_double()
        self._check(f(a.ctypes.data, b.ctypes.data, abi.dims3(a), abi.Spacing3(*spacing), label, C.byref(out)))
        return out.value

    def warp_labels(self, labels, disp) -> np.ndarray:
        lbl = np.ascontiguousarray(labels, np.uint16)
        disp = _f32(disp)
        out = np.empty_like(lbl)
        f = self._ref().ref_warp_labels
        f.argtypes = [C.c_void_p, _F, abi.Dims3, C.c_void_p]
        self._check(f(lbl.ctypes.data, _fp(disp), abi.dims3(lbl), out.ctypes.data))
        return out

    def write_volume(self, path, data, spacing=(1.0, 1.0, 1.0), kind: str | None = None) -> None:
        a = np.asarray(data)
        if kind is None:
            kind = "label" if a.dtype == np.uint16 else ("vector" if a.ndim == 4 else "scalar")
        k = {"scalar": 0, "vector": 1, "label": 2}[kind]
        a = np.ascontiguousarray(a, np.uint16 if k == 2 else np.float32)
        f = self._ref().ref_write_volume
        f.argtypes = [C.c_char_p, C.c_int, abi.Dims3, abi.Spacing3, C.c_void_p]
        self._check(f(os.fsencode(str(path)), k, abi.dims3(a), abi.Spacing3(*spacing), a.ctypes.data))

    def read_volume(self, path, expected_kind: int = -1):
        """(kind, array, spacing) like paper_2109_12688_b200.dreg.read_volume."""
        L = self._ref()
        f = L.ref_read_volume
        f.argtypes = [C.c_char_p, C.c_int, C.POINTER(abi.VolumeInfo), C.c_void_p, C.c_size_t]
        info = abi.VolumeInfo()
        p = os.fsencode(str(path))
        self._check(f(p, expected_kind, C.byref(info), None, 0))
        shape = info.dims.shape() + ((3,) if info.kind == 1 else ())
        out = np.empty(shape, np.uint16 if info.kind == 2 else np.float32)
        self._check(f(p, expected_kind, C.byref(info), out.ctypes.data, out.nbytes))
        return info.kind, out, (info.spacing.x, info.spacing.y, info.spacing.z)

    def write_report(self, path, report: abi.RunReport) -> None:
        f = self._ref().ref_write_report
        f.argtypes = [C.c_char_p, C.POINTER(abi.RunReport)]
        self._check(f(os.fsencode(str(path)), C.byref(report)))

    def register_pair(self, target, source, cfg: abi.RegCfg, spacing=(1.0, 1.0, 1.0)):
        target, source = _f32(target), _f32(source)
        phi = np.zeros(target.shape + (3,), np.float32)
        warped = np.zeros_like(target)
        res = abi.PairResult()
        self._check(
            self._g("register_pair")(
                _fp(target),
                _fp(source),
                abi.dims3(target),
                abi.Spacing3(*spacing),
                C.byref(cfg),
                _fp(phi),
                _fp(warped),
                C.byref(res),
            )
        )
        return phi, warped, res
