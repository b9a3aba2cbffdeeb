"""The `dreg` command-line drop-in (paper_2109_12688_b200/lib/dreg) against the
reference tool's surface (proj/tools/dreg.cpp, proj/tests/test_cli.cpp; SURVEY.md
§8(f) item 4).

CPU: exit codes for argument and I/O errors, and `synth` outputs byte-identical to the
reference's synthetic cases (compiled reference in oracle/_ref).  GPU (-m gpu): the
register -> warp -> jacobian / evaluate flow of test_cli.cpp, the translation-overlap
criterion, thread-count invariance, and parity of every CLI product with the library
API and the reference's metrics.
"""
import json
import os
import subprocess

import numpy as np
import pytest

from paper_2109_12688_b200 import dreg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_2109_12688_b200", "lib", "dreg")


def run(*args):
    p = subprocess.run([BIN, *[str(a) for a in args]], capture_output=True, text=True, timeout=600)
    return p.returncode, p.stdout + p.stderr


@pytest.fixture(scope="module", autouse=True)
def _binary():
    if not os.path.exists(BIN):
        pytest.fail(f"{BIN} missing: run __graft_entry__.build()")


def test_missing_subcommand_and_unknown_flags_exit_2(tmp_path):
    """test_cli.cpp:67-71."""
    assert run()[0] == 2
    assert run("register", "--bogus", "1")[0] == 2
    assert run("synth", "--case", "nosuch", "--dims", "8,8,8", "--out-prefix", tmp_path / "x")[0] == 2
    assert run("frobnicate")[0] == 2
    rc, out = run("register", "--target", "a")
    assert rc == 2 and out.startswith("dreg: argument-error: ")


def test_range_validation_exits_2(tmp_path):
    """test_cli.cpp:73-80."""
    pre = tmp_path / "pair"
    assert run("synth", "--case", "translate", "--dims", "16,16,16", "--out-prefix", pre)[0] == 0
    io = ["--target", f"{pre}_target.dreg", "--source", f"{pre}_source.dreg", "--out", tmp_path / "phi.dreg"]
    assert run("register", *io, "--lambda", "-1", "--theta", "0.05")[0] == 2
    assert run("register", *io, "--lambda", "1", "--theta", "0")[0] == 2
    assert run("register", *io, "--lambda", "1", "--theta", "0.05", "--order", "5")[0] == 2
    assert run("register", *io, "--lambda", "1", "--theta", "0.05", "--levels", "7")[0] == 2
    assert run("register", *io, "--lambda", "1", "--theta", "0.05", "--data-term", "l3")[0] == 2
    assert run("register", *io, "--lambda", "1", "--theta", "0.05", "--tol", "-1")[0] == 2
    assert run("--threads", "0", "jacobian", "--phi", "x")[0] == 2
    assert run("synth", "--case", "blob", "--dims", "8,8", "--out-prefix", pre)[0] == 2
    assert run("synth", "--case", "blob", "--dims", "8,8,8", "--noise", "2", "--out-prefix", pre)[0] == 2


def test_missing_inputs_exit_3(tmp_path):
    """test_cli.cpp:82-86."""
    assert run("register", "--target", "/nonexistent.dreg", "--source", "/nonexistent.dreg", "--out",
               tmp_path / "x.dreg", "--lambda", "1", "--theta", "0.05")[0] == 3
    rc, out = run("jacobian", "--phi", "/nonexistent.dreg")
    assert rc == 3 and out.startswith("dreg: io-error: cannot open")


def test_kind_mismatch_exits_3(tmp_path):
    """test_cli.cpp:88-93: a scalar volume is not a deformation field."""
    pre = tmp_path / "pair"
    assert run("synth", "--case", "translate", "--dims", "16,16,16", "--out-prefix", pre)[0] == 0
    assert run("jacobian", "--phi", f"{pre}_target.dreg")[0] == 3
    assert run("warp", "--in", f"{pre}_target.dreg", "--phi", f"{pre}_target.dreg", "--out", tmp_path / "o")[0] == 3


@pytest.mark.parametrize("case,extra,shape,ref_kind,shift,seed,noise", [
    ("translate", [], (16, 16, 16), "translate", (3.0, 0.0, 0.0), 1, 0.0),
    ("translate", ["--shift", "1.5,-2,0.25"], (12, 20, 16), "translate", (1.5, -2.0, 0.25), 1, 0.0),
    ("sphere-ellipsoid", [], (24, 20, 16), "sphere_ellipsoid", (0, 0, 0), 1, 0.0),
    ("blob", ["--seed", "9"], (16, 24, 32), "random_smooth", (0, 0, 0), 9, 0.0),
    ("blob", ["--seed", "5", "--noise", "0.05"], (16, 16, 16), "random_smooth", (0, 0, 0), 5, 0.05),
])
def test_synth_byte_identical_to_reference(tmp_path, reference, case, extra, shape, ref_kind, shift, seed, noise):
    """dreg.cpp:207-226 on the reference's own generators (synth.cpp): the four files
    equal the reference's volumes written by the reference's writer."""
    pre = tmp_path / "c"
    z, y, x = shape
    assert run("synth", "--case", case, "--dims", f"{x},{y},{z}", "--out-prefix", pre, *extra)[0] == 0
    t, s, tl, sl = reference.make_case(ref_kind, shape, shift, seed)
    if noise > 0:
        s = reference.add_salt_pepper(s, noise, seed + 17)
    for name, vol in (("target", t), ("source", s), ("target_labels", tl), ("source_labels", sl)):
        ref_path = tmp_path / f"ref_{name}.dreg"
        reference.write_volume(ref_path, vol)
        with open(f"{pre}_{name}.dreg", "rb") as a, open(ref_path, "rb") as b:
            assert a.read() == b.read(), name


# ---- GPU ------------------------------------------------------------------------------
@pytest.mark.gpu
def test_evaluate_identical_labels(tmp_path):
    """test_cli.cpp:95-104."""
    pre = tmp_path / "pair"
    assert run("synth", "--case", "sphere-ellipsoid", "--dims", "16,16,16", "--out-prefix", pre)[0] == 0
    rc, out = run("evaluate", "--a", f"{pre}_target_labels.dreg", "--b", f"{pre}_target_labels.dreg", "--labels", "1")
    assert rc == 0, out
    assert "label 1 dice 1 hausdorff_mm 0" in out


@pytest.mark.gpu
def test_evaluate_every_requested_label(tmp_path, reference):
    """test_cli.cpp:106-119, plus an absent label (hausdorff nan) and values vs the
    reference's metrics."""
    lbl = np.zeros((2, 8, 8), np.uint16)
    lbl[0, 2, 2] = 1
    lbl[0, 5, 5] = 2
    lbl[1, 2, 2] = 1
    p = tmp_path / "two_labels.dreg"
    dreg.write_volume(p, lbl)
    rc, out = run("evaluate", "--a", p, "--b", p, "--labels", "1,2")
    assert rc == 0, out
    assert "label 1 dice 1 hausdorff_mm 0" in out and "label 2 dice 1 hausdorff_mm 0" in out
    t, s, tl, sl = reference.make_case("sphere_ellipsoid", (20, 24, 28))
    pa, pb = tmp_path / "a.dreg", tmp_path / "b.dreg"
    dreg.write_volume(pa, tl, (0.8, 1.1, 2.0))
    dreg.write_volume(pb, sl, (0.8, 1.1, 2.0))
    rc, out = run("evaluate", "--a", pa, "--b", pb, "--labels", "1,3")
    assert rc == 0, out
    d = reference.dice(tl, sl, 1)
    h = reference.hausdorff_slice_avg(tl, sl, 1, (0.8, 1.1, 2.0))
    assert f"label 1 dice {d:.6g} hausdorff_mm {h:.6g}" in out
    assert "label 3 dice 1 hausdorff_mm nan" in out


@pytest.mark.gpu
def test_register_warp_jacobian_end_to_end(tmp_path, ctx):
    """test_cli.cpp:121-151; the CLI's phi equals the library API's register_pair."""
    pre = tmp_path / "pair"
    assert run("synth", "--case", "translate", "--dims", "16,16,16", "--shift", "1,0,0", "--out-prefix", pre)[0] == 0
    phi, warped, report = tmp_path / "phi.dreg", tmp_path / "warped.dreg", tmp_path / "report.json"
    rc, out = run("register", "--target", f"{pre}_target.dreg", "--source", f"{pre}_source.dreg", "--out", phi,
                  "--warped", warped, "--data-term", "l1", "--order", "2", "--lambda", "8", "--theta", "0.05",
                  "--levels", "2", "--seed-report", report)
    assert rc == 0, out
    assert phi.exists() and warped.exists() and report.exists()
    rc, out = run("jacobian", "--phi", phi)
    assert rc == 0 and "pct_nonpositive 0 " in out, out

    rewarped = tmp_path / "rewarped.dreg"
    assert run("warp", "--in", f"{pre}_source.dreg", "--phi", phi, "--out", rewarped)[0] == 0
    assert dreg.read_scalar(warped)[0].tobytes() == dreg.read_scalar(rewarped)[0].tobytes()
    wl = tmp_path / "warped_labels.dreg"
    assert run("warp", "--in", f"{pre}_source_labels.dreg", "--phi", phi, "--out", wl, "--labels")[0] == 0
    assert wl.exists()

    # same library, same inputs: the API gives the same field bit for bit
    tgt = dreg.read_scalar(f"{pre}_target.dreg")[0]
    src = dreg.read_scalar(f"{pre}_source.dreg")[0]
    solver = dreg.solver_cfg(data_term=1, order=2, lambda_=8.0, theta=0.05)
    cfg = dreg.make_registration_config(dreg.DREG_PROFILE_CAPPED, solver, 2)
    api_phi, api_warped, res = ctx.register_pair(tgt, src, cfg)
    assert dreg.read_deformation(phi)[0].tobytes() == api_phi.tobytes()
    j = json.loads(report.read_text())
    assert j["velocity_count"] == res.velocity_count
    assert j["config"] == {"data_term": "l1", "order": 2, "lambda": 8.0, "theta": 0.05, "levels": 2,
                           "profile": "capped", "tol": cfg.solver.tol,
                           "warp_improvement_threshold": cfg.warp_improvement_threshold,
                           "epsilon": 1e-06, "threads": 1}


@pytest.mark.gpu
def test_translation_registers_to_high_overlap(tmp_path, reference):
    """test_cli.cpp:153-167: dice >= 0.95 in the report; the report's dice and
    Hausdorff equal the reference's metrics on the CLI's own phi."""
    pre = tmp_path / "pair"
    assert run("synth", "--case", "translate", "--dims", "32,32,32", "--shift", "2,0,0", "--out-prefix", pre)[0] == 0
    report, phi = tmp_path / "t_report.json", tmp_path / "t_phi.dreg"
    rc, out = run("register", "--target", f"{pre}_target.dreg", "--source", f"{pre}_source.dreg", "--out", phi,
                  "--data-term", "l1", "--order", "2", "--lambda", "5", "--theta", "0.1", "--seed-report", report,
                  "--target-labels", f"{pre}_target_labels.dreg", "--source-labels", f"{pre}_source_labels.dreg")
    assert rc == 0, out
    j = json.loads(report.read_text())
    assert j["dice"]["1"] >= 0.95
    disp = dreg.read_deformation(phi)[0]
    tl = dreg.read_label(f"{pre}_target_labels.dreg")[0]
    sl = dreg.read_label(f"{pre}_source_labels.dreg")[0]
    w = reference.warp_labels(sl, disp)
    assert j["dice"]["1"] == float(f"{reference.dice(w, tl, 1):.6g}")
    assert j["hausdorff_mm"]["1"] == float(f"{reference.hausdorff_slice_avg(w, tl, 1):.6g}")


@pytest.mark.gpu
def test_worker_threads_do_not_change_the_result(tmp_path):
    """test_cli.cpp:169-176."""
    pre = tmp_path / "pair"
    assert run("synth", "--case", "translate", "--dims", "16,16,16", "--shift", "1,0,0", "--out-prefix", pre)[0] == 0
    common = ["register", "--target", f"{pre}_target.dreg", "--source", f"{pre}_source.dreg", "--data-term", "l1",
              "--order", "2", "--lambda", "5", "--theta", "0.1", "--levels", "2", "--out"]
    p1, p2 = tmp_path / "phi_t1.dreg", tmp_path / "phi_t2.dreg"
    assert run(*common, p1, "--threads", "1")[0] == 0
    assert run("--threads", "2", *common, p2)[0] == 0
    with open(p1, "rb") as a, open(p2, "rb") as b:
        assert a.read() == b.read()


# ---- the reference's CLI-driven acceptance criteria (acceptance_main.cpp) ----------
@pytest.mark.gpu
def test_acceptance_pipeline_through_cli(tmp_path):
    """Criterion 4 (acceptance_main.cpp:215-258): a 3-voxel translation of a 64^3 case is
    recovered end to end through the CLI: mean displacement inside the target label
    within 0.5 voxel of (-3, 0, 0), dice >= 0.95, Hausdorff <= 2 x spacing, < 60 s."""
    import time

    pre = tmp_path / "c4"
    assert run("synth", "--case", "translate", "--dims", "64,64,64", "--shift", "3,0,0", "--out-prefix", pre)[0] == 0
    t0 = time.time()
    rc, out = run("register", "--threads", "1", "--target", f"{pre}_target.dreg", "--source", f"{pre}_source.dreg",
                  "--out", f"{pre}_phi.dreg", "--warped", f"{pre}_warped.dreg", "--data-term", "l1", "--order", "2",
                  "--lambda", "5", "--theta", "0.1", "--profile", "capped", "--seed-report", f"{pre}_report.json",
                  "--target-labels", f"{pre}_target_labels.dreg", "--source-labels", f"{pre}_source_labels.dreg")
    elapsed = time.time() - t0
    assert rc == 0, out
    phi = dreg.read_deformation(f"{pre}_phi.dreg")[0].astype(np.float64)
    lbl, sp = dreg.read_label(f"{pre}_target_labels.dreg")
    mean = phi[lbl == 1].mean(axis=0)
    err = float(np.linalg.norm(mean - np.array([-3.0, 0.0, 0.0])))
    rep = json.loads(open(f"{pre}_report.json").read())
    print(f"criterion 4: mean disp err {err:.3f} vox, dice {rep['dice']['1']}, "
          f"hausdorff {rep['hausdorff_mm']['1']} mm, {elapsed:.2f} s")
    assert err <= 0.5
    assert rep["dice"]["1"] >= 0.95
    assert rep["hausdorff_mm"]["1"] <= 2.0 * max(sp)
    assert elapsed < 60.0


@pytest.mark.gpu
def test_acceptance_sweep_through_cli(tmp_path):
    """Criterion 6 (acceptance_main.cpp:296-355): every data term x order in
    {l1, l2} x {1, 2, 3} reaches dice >= 0.85 on the sphere->ellipsoid case, and with 5%
    salt-and-pepper on the source the robust l1 term is at least as good as l2."""
    pre = tmp_path / "c6"
    assert run("synth", "--case", "sphere-ellipsoid", "--dims", "32,32,32", "--out-prefix", pre)[0] == 0

    def reg(tag, dt, order, lam, src):
        out = tmp_path / f"c6_{tag}"
        rc, msg = run("register", "--threads", "1", "--target", f"{src}_target.dreg", "--source",
                      f"{src}_source.dreg", "--out", f"{out}_phi.dreg", "--data-term", dt, "--order", order,
                      "--lambda", lam, "--theta", "0.05", "--profile", "capped", "--seed-report",
                      f"{out}_report.json", "--target-labels", f"{src}_target_labels.dreg", "--source-labels",
                      f"{src}_source_labels.dreg")
        assert rc == 0, msg
        return json.loads(open(f"{out}_report.json").read())["dice"]["1"]

    lam_for = {1: 1.0, 2: 5.0, 3: 5.0}
    dices = {}
    for dt in ("l1", "l2"):
        for order in (1, 2, 3):
            dices[f"{dt}{order}"] = reg(f"{dt}{order}", dt, order, lam_for[order], pre)
    noisy = tmp_path / "c6_noisy"
    assert run("synth", "--case", "sphere-ellipsoid", "--dims", "32,32,32", "--noise", "0.05", "--seed", "5",
               "--out-prefix", noisy)[0] == 0
    d1 = reg("noisy_l1", "l1", 2, 10.0, noisy)
    d2 = reg("noisy_l2", "l2", 2, 10.0, noisy)
    print("criterion 6:", dices, f"noisy l1={d1} l2={d2}")
    assert all(d >= 0.85 for d in dices.values()), dices
    assert d1 >= d2


@pytest.mark.gpu
def test_acceptance_reproducibility_through_cli(tmp_path):
    """Criterion 7 (acceptance_main.cpp:358-395): identical invocations produce
    byte-identical deformation files and reports identical modulo runtime."""
    pre = tmp_path / "c7"
    assert run("synth", "--case", "translate", "--dims", "32,32,32", "--shift", "2,0,0", "--out-prefix", pre)[0] == 0
    common = ["register", "--threads", "1", "--target", f"{pre}_target.dreg", "--source", f"{pre}_source.dreg",
              "--data-term", "l1", "--order", "2", "--lambda", "10", "--theta", "0.05", "--profile", "capped"]
    assert run(*common, "--out", f"{pre}_phi_a.dreg", "--seed-report", f"{pre}_report_a.json")[0] == 0
    assert run(*common, "--out", f"{pre}_phi_b.dreg", "--seed-report", f"{pre}_report_b.json")[0] == 0
    with open(f"{pre}_phi_a.dreg", "rb") as a, open(f"{pre}_phi_b.dreg", "rb") as b:
        assert a.read() == b.read()
    ra = json.loads(open(f"{pre}_report_a.json").read())
    rb = json.loads(open(f"{pre}_report_b.json").read())
    ra.pop("runtime_seconds")
    rb.pop("runtime_seconds")
    assert ra == rb
