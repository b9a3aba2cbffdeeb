"""DREG volume container and JSON run report (reference io.hpp / io.cpp; SURVEY.md §8(f)
item 3).  Host-only: runs without a GPU.

Parity is byte-for-byte against the UNMODIFIED reference io.cpp compiled into
oracle/_ref (the `reference` fixture): files written by either side are identical and
readable by the other, and every rejection the reference's test_io.cpp checks
(bad magic / version / kind, truncated / trailing payloads, non-finite values, missing
files, absurd dims) fails on both sides with the same message.
"""
import os
import struct

import numpy as np
import pytest

from conftest import Rng, random_field, random_volume
from oracle.oracle import OracleError
from paper_2109_12688_b200 import abi, dreg


def _bytes(p):
    with open(p, "rb") as f:
        return f.read()


def _labels(shape, seed, top=5):
    return (Rng(seed).uniform(int(np.prod(shape))) * top).astype(np.uint16).reshape(shape)


CASES = [
    ("scalar", lambda: random_volume((5, 4, 3), 11, -2.0, 2.0), (1.0, 1.0, 1.0)),
    ("scalar", lambda: random_volume((7, 9, 11), 12), (0.7, 1.9, 2.5)),
    ("vector", lambda: random_field((6, 5, 4), 13, 3.0), (1.25, 1.0, 0.5)),
    ("label", lambda: _labels((8, 6, 4), 14), (1.5, 1.5, 3.0)),
    ("label", lambda: _labels((1, 1, 1), 15), (1.0, 2.0, 3.0)),
]


@pytest.mark.parametrize("kind,make,spacing", CASES)
def test_round_trip_bit_for_bit(tmp_path, kind, make, spacing):
    """test_io.cpp:41-77: every kind round-trips dims, spacing and payload exactly."""
    data = make()
    p = tmp_path / "v.dreg"
    dreg.write_volume(p, data, spacing)
    k, back, sp = dreg.read_volume(p)
    assert k == {"scalar": 0, "vector": 1, "label": 2}[kind]
    assert sp == spacing
    assert back.dtype == data.dtype and back.shape == data.shape
    assert back.tobytes() == data.tobytes()


@pytest.mark.parametrize("kind,make,spacing", CASES)
def test_files_byte_identical_to_reference(tmp_path, reference, kind, make, spacing):
    data = make()
    ours, theirs = tmp_path / "ours.dreg", tmp_path / "ref.dreg"
    dreg.write_volume(ours, data, spacing)
    reference.write_volume(theirs, data, spacing)
    assert _bytes(ours) == _bytes(theirs)
    # and each side reads the other's file
    k1, a1, s1 = dreg.read_volume(theirs)
    k2, a2, s2 = reference.read_volume(ours)
    assert (k1, s1) == (k2, s2)
    assert a1.tobytes() == a2.tobytes() == data.tobytes()


def test_header_layout(tmp_path):
    """README.md:99-114: offsets of magic, version, kind, dims, spacing, payload."""
    v = random_volume((2, 3, 4), 3)
    p = tmp_path / "h.dreg"
    dreg.write_volume(p, v, (0.5, 1.5, 2.5))
    b = _bytes(p)
    assert b[:4] == b"DREG"
    assert struct.unpack("<I", b[4:8])[0] == 1
    assert b[8] == 0
    assert struct.unpack("<3I", b[9:21]) == (4, 3, 2)
    assert struct.unpack("<3d", b[21:45]) == (0.5, 1.5, 2.5)
    assert len(b) == 45 + 4 * v.size
    assert np.frombuffer(b[45:], "<f4").tobytes() == v.tobytes()


def test_deformations_are_vector_fields(tmp_path, reference):
    """test_io.cpp:70-77: a deformation is stored as a vector field; reading it as a
    scalar is a kind mismatch."""
    phi = random_field((4, 4, 4), 5, 1.0)
    p = tmp_path / "phi.dreg"
    dreg.write_volume(p, phi)
    assert dreg.read_deformation(p)[0].tobytes() == phi.tobytes()
    with pytest.raises(dreg.IoError) as ours:
        dreg.read_scalar(p)
    with pytest.raises(OracleError) as theirs:
        reference.read_volume(p, 0)
    assert theirs.value.status == abi.DREG_IO_ERROR
    assert str(ours.value) in str(theirs.value)


def _corrupt(tmp_path, name, mutate):
    v = random_volume((3, 3, 3), 7)
    p = tmp_path / name
    dreg.write_volume(p, v)
    b = bytearray(_bytes(p))
    b = mutate(b)
    with open(p, "wb") as f:
        f.write(bytes(b))
    return p


def _set(off, raw):
    def f(b):
        b[off:off + len(raw)] = raw
        return b
    return f


REJECTIONS = [
    ("bad_magic", _set(0, b"XREG")),                                  # test_io.cpp:79-87
    ("bad_version", _set(4, struct.pack("<I", 2))),                   # :89-96
    ("bad_kind", _set(8, b"\x07")),                                   # :98-105
    ("truncated", lambda b: b[:-3]),                                  # :107-115
    ("trailing", lambda b: b + b"\x00"),                              # :117-124
    ("nonfinite", _set(45 + 4 * 5, struct.pack("<f", float("nan")))),  # :126-138
    ("inf", _set(45, struct.pack("<f", float("inf")))),
    ("absurd_dims", _set(9, struct.pack("<3I", 100000, 1, 1))),       # :144-155
    ("too_large", _set(9, struct.pack("<3I", 65536, 65536, 2))),
    ("zero_dim", _set(13, struct.pack("<I", 0))),
    ("zero_spacing", _set(21, struct.pack("<d", 0.0))),
    ("neg_spacing", _set(29, struct.pack("<d", -1.0))),
    ("nan_spacing", _set(37, struct.pack("<d", float("nan")))),
    ("short_header", lambda b: b[:30]),
    ("empty", lambda b: b[:0]),
]


@pytest.mark.parametrize("name,mutate", REJECTIONS, ids=[r[0] for r in REJECTIONS])
def test_rejections_match_reference(tmp_path, reference, name, mutate):
    p = _corrupt(tmp_path, name + ".dreg", mutate)
    with pytest.raises(dreg.IoError) as ours:
        dreg.read_volume(p)
    with pytest.raises(OracleError) as theirs:
        reference.read_volume(p)
    assert theirs.value.status == abi.DREG_IO_ERROR
    assert str(theirs.value).endswith(str(ours.value)), (str(ours.value), str(theirs.value))


def test_missing_file(tmp_path, reference):
    """test_io.cpp:140-142."""
    p = tmp_path / "does_not_exist.dreg"
    with pytest.raises(dreg.IoError, match="cannot open"):
        dreg.read_volume(p)
    with pytest.raises(OracleError):
        reference.read_volume(p)


def test_unwritable_path(tmp_path):
    with pytest.raises(dreg.IoError, match="cannot open for writing"):
        dreg.write_volume(tmp_path / "no" / "such" / "dir.dreg", random_volume((2, 2, 2), 1))


# ---- run report ------------------------------------------------------------------------
def _report(**kw):
    dice = kw.pop("dice", {})
    hd = kw.pop("hausdorff_mm", {})
    cfg = dict(data_term="l1", order=0, lambda_=0.0, theta=0.0, levels=0, profile="capped", tol=0.0,
               warp_improvement_threshold=0.0, epsilon=0.0, threads=1)
    top = dict(jacobian_pct_nonpositive=0.0, runtime_seconds=0.0, velocity_count=0)
    for k, v in kw.items():
        (cfg if k in cfg else top)[k] = v
    return dice, hd, cfg, top


def _write_both(tmp_path, reference, dice, hd, cfg, top):
    ours, theirs = tmp_path / "ours.json", tmp_path / "ref.json"
    dreg.write_report(ours, dice=dice, hausdorff_mm=hd, **cfg, **top)
    dl = (np.ctypeslib.ctypes.c_int * max(len(dice), 1))(*dice.keys())
    dv = (np.ctypeslib.ctypes.c_double * max(len(dice), 1))(*dice.values())
    hl = (np.ctypeslib.ctypes.c_int * max(len(hd), 1))(*hd.keys())
    hv = (np.ctypeslib.ctypes.c_double * max(len(hd), 1))(*hd.values())
    rc = abi.ReportConfig(cfg["data_term"].encode(), cfg["order"], cfg["lambda_"], cfg["theta"], cfg["levels"],
                          cfg["profile"].encode(), cfg["tol"], cfg["warp_improvement_threshold"], cfg["epsilon"],
                          cfg["threads"])
    rep = abi.RunReport(len(dice), dl, dv, len(hd), hl, hv, top["jacobian_pct_nonpositive"],
                        top["runtime_seconds"], top["velocity_count"], rc)
    reference.write_report(theirs, rep)
    return _bytes(ours).decode(), _bytes(theirs).decode()


def test_report_identity_registration(tmp_path, reference):
    """test_io.cpp:157-182: the contract fields of an identity registration's report."""
    import json

    case = _report(dice={1: 1.0}, hausdorff_mm={1: 0.0}, runtime_seconds=0.125, velocity_count=3, data_term="l1",
                   order=2, lambda_=10.0, theta=0.05, levels=3, profile="capped", tol=1e-3,
                   warp_improvement_threshold=0.02, epsilon=1e-6, threads=1)
    ours, theirs = _write_both(tmp_path, reference, *case)
    assert ours == theirs
    j = json.loads(ours)
    assert list(j) == ["dice", "hausdorff_mm", "jacobian_pct_nonpositive", "runtime_seconds", "velocity_count",
                       "config"]
    assert j["dice"]["1"] == 1.0 and j["velocity_count"] == 3 and j["config"]["lambda"] == 10.0


def test_report_six_significant_digits(tmp_path, reference):
    """test_io.cpp:184-198."""
    case = _report(dice={2: 0.123456789}, runtime_seconds=0.00123456789, lambda_=1.0 / 3.0)
    ours, theirs = _write_both(tmp_path, reference, *case)
    assert ours == theirs
    assert '"2": 0.123457' in ours and "0.00123457" in ours and "0.333333" in ours


def test_report_number_layout_fuzz(tmp_path, reference):
    """Random magnitudes (tiny, huge, negative, integral, zero) and label maps:
    the JSON text is byte-identical to the reference's serialiser."""
    r = Rng(77)
    for trial in range(40):
        u = r.uniform(40)
        mags = 10.0 ** (np.floor(u[:20] * 44) - 22)
        vals = (u[20:40] - 0.3) * mags
        vals[trial % 20] = float(np.round(vals[trial % 20]))  # an integral value
        if trial % 7 == 0:
            vals[3] = 0.0
        nl = trial % 5
        labels = [int(x) for x in (r.uniform(nl) * 300)]
        dice = {lab: float(vals[i]) for i, lab in enumerate(labels)}
        hd = {lab: float(vals[10 + i]) for i, lab in enumerate(labels[::-1])}
        case = _report(dice=dice, hausdorff_mm=hd, jacobian_pct_nonpositive=float(vals[5]),
                       runtime_seconds=float(vals[6]), velocity_count=trial, data_term="l2", order=1 + trial % 3,
                       lambda_=float(vals[7]), theta=float(vals[8]), levels=1 + trial % 6,
                       profile="converged" if trial % 2 else "capped", tol=float(vals[9]),
                       warp_improvement_threshold=float(vals[15]), epsilon=float(vals[16]), threads=1 + trial)
        ours, theirs = _write_both(tmp_path, reference, *case)
        assert ours == theirs, (trial, ours, theirs)
