"""C ABI checks without a GPU: the product library loads, exports every function that
include/dreg_cuda.h declares, the ctypes mirror (paper_2109_12688_b200/abi.py) has
the C compiler's struct layout, and pure host entry points behave like the reference.
"""
import ctypes as C
import os
import re
import subprocess
import tempfile

import pytest

from paper_2109_12688_b200 import abi, dreg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dreg_cuda.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dreg_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_hot_path():
    fns = declared_functions()
    for f in ["dreg_cuda_register_pair", "dreg_cuda_register_batch", "dreg_cuda_register_batch_device",
              "dreg_cuda_solve_velocity", "dreg_cuda_w_update", "dreg_cuda_v_update", "dreg_cuda_jacobian"]:
        assert f in fns


def test_library_exports_every_declared_symbol():
    lib = dreg.load_library()  # raises if the sm_100a library was not built
    missing = [f for f in declared_functions() if not hasattr(lib, f)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", dreg.lib_path()], capture_output=True, text=True).stdout
    for f in declared_functions():
        assert re.search(rf"\bT {f}\b", out), f


def test_synth_library_exports_dreg_synth_h():
    hdr = open(os.path.join(ROOT, "include", "dreg_synth.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    fns = sorted(set(re.findall(r"\b(dreg_[a-z0-9_]+)\s*\(", hdr)))
    assert "dreg_synth_case" in fns and "dreg_synth_pair" in fns
    path = os.path.join(ROOT, "paper_2109_12688_b200", "lib", "libdreg_synth.so")
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True).stdout
    for f in fns:
        assert re.search(rf"\bT {f}\b", out), f


def test_cli_binary_links_the_product_library():
    exe = os.path.join(ROOT, "paper_2109_12688_b200", "lib", "dreg")
    out = subprocess.run(["ldd", exe], capture_output=True, text=True).stdout
    assert "libdreg_cuda.so" in out and "libdreg_synth.so" in out
    assert "not found" not in out.split("libdreg_cuda.so")[1].splitlines()[0]


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", dreg.lib_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in out


STRUCTS = {
    "dreg_dims3": abi.Dims3,
    "dreg_spacing3": abi.Spacing3,
    "dreg_solver_cfg": abi.SolverCfg,
    "dreg_reg_cfg": abi.RegCfg,
    "dreg_solver_diag": abi.SolverDiag,
    "dreg_level_log": abi.LevelLog,
    "dreg_pair_result": abi.PairResult,
    "dreg_jacobian_stats": abi.JacobianStats,
    "dreg_pair_record": abi.PairRecord,
    "dreg_volume_info": abi.VolumeInfo,
    "dreg_report_config": abi.ReportConfig,
    "dreg_run_report": abi.RunReport,
}


def test_struct_layouts_match_c_compiler():
    lines = ["#include <stdio.h>", "#include <stddef.h>", '#include "dreg_cuda.h"', "int main(void) {"]
    for cname, py in STRUCTS.items():
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            cf = "lambda" if fname == "lambda_" else fname
            lines.append(f'printf("{cname}.{fname} %zu\\n", offsetof({cname}, {cf}));')
    lines.append("return 0; }")
    with tempfile.TemporaryDirectory() as td:
        src = os.path.join(td, "l.c")
        exe = os.path.join(td, "l")
        open(src, "w").write("\n".join(lines))
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), src, "-o", exe], check=True)
        out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout
    got = dict(line.rsplit(" ", 1) for line in out.strip().splitlines())
    for cname, py in STRUCTS.items():
        assert int(got[f"{cname} size"]) == C.sizeof(py), cname
        for fname, _ in py._fields_:
            assert int(got[f"{cname}.{fname}"]) == getattr(py, fname).offset, (cname, fname)


def test_host_helpers_match_reference_semantics(oracle):
    # nesterov_next_alpha (admm.cpp:198-200)
    a = 1.0
    for _ in range(20):
        assert dreg.nesterov_next_alpha(a) == oracle.nesterov_next_alpha(a)
        a = dreg.nesterov_next_alpha(a)
    # make_registration_config (registration.cpp:62-83)
    s = abi.solver_cfg(tol=0.0)
    for prof in (abi.DREG_PROFILE_CAPPED, abi.DREG_PROFILE_CONVERGED):
        for L in (1, 2, 3):
            ours = dreg.make_registration_config(prof, s, L)
            ref = oracle.make_registration_config(prof, s, L)
            assert list(ours.max_warps_per_level) == list(ref.max_warps_per_level)
            assert list(ours.max_admm_iters_per_level) == list(ref.max_admm_iters_per_level)
            assert ours.solver.tol == ref.solver.tol
    # capped caps {10,5,5}/{10,10,5}; converged tol 0.01 (test_registration.cpp:183-195)
    c = dreg.make_registration_config(abi.DREG_PROFILE_CAPPED, s, 3)
    assert list(c.max_admm_iters_per_level)[:3] == [10, 5, 5] and list(c.max_warps_per_level)[:3] == [10, 10, 5]
    assert dreg.make_registration_config(abi.DREG_PROFILE_CONVERGED, s, 3).solver.tol == 0.01


@pytest.mark.parametrize("field,value", [("data_term", 3), ("order", 0), ("order", 7), ("lambda_", -1.0),
                                         ("theta", 0.0), ("epsilon", 0.0), ("max_iters", 0), ("tol", -1.0)])
def test_validate_rejects(oracle, field, value):
    """admm.cpp:174-196 -> std::invalid_argument (ValueError here)."""
    cfg = abi.solver_cfg()
    setattr(cfg, field, value)
    with pytest.raises(ValueError):
        dreg.validate(cfg)
    with pytest.raises(Exception):
        oracle.validate(cfg)
    dreg.validate(abi.solver_cfg())


def test_context_without_gpu_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(RuntimeError):
        dreg.Context(0)
