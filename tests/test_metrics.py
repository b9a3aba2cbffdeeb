"""Label metrics: warp_labels, dice, hausdorff_slice_avg (reference metrics.hpp:31-42,
metrics.cpp:23-204).

The reference's own metric tests (proj/tests/test_metrics.cpp) are restated and run on
the compiled reference (CPU, always) and on the sm_100a kernels (-m gpu).  GPU parity
is bit-exact: Dice counts are integers, the Hausdorff distance transform issues the
reference's fp64 operations in the reference's order, and the label warp is a
nearest-neighbour gather.
"""
import numpy as np
import pytest

from conftest import Rng, random_field


def random_labels(shape, seed, fill_prob):
    """test_metrics.cpp:14-21."""
    return (Rng(seed).uniform(int(np.prod(shape))) < fill_prob).astype(np.uint16).reshape(shape)


def brute_force_hausdorff(a, b, label, spacing):
    """oracles.cpp brute_force_hausdorff: all-pairs per-slice symmetric Hausdorff."""
    sx, sy = spacing[0], spacing[1]
    total, n = 0.0, 0
    for z in range(a.shape[0]):
        pa = np.argwhere(a[z] == label)
        pb = np.argwhere(b[z] == label)
        if len(pa) == 0 or len(pb) == 0:
            continue
        d = (((pa[:, None, 1] - pb[None, :, 1]) * sx) ** 2 + ((pa[:, None, 0] - pb[None, :, 0]) * sy) ** 2)
        total += np.sqrt(max(d.min(axis=1).max(), d.min(axis=0).max()))
        n += 1
    return total / n if n else -1.0


class _Ref:
    """The reference's metrics with the GPU context's call signatures."""

    def __init__(self, lib):
        self.lib = lib

    def dice(self, a, b, label):
        return self.lib.dice(a, b, label)

    def hausdorff_slice_avg(self, a, b, label, spacing=(1.0, 1.0, 1.0)):
        from oracle.oracle import OracleError

        try:
            return self.lib.hausdorff_slice_avg(a, b, label, spacing)
        except OracleError as e:
            raise ValueError(str(e)) from e

    def warp_labels(self, labels, disp):
        return self.lib.warp_labels(labels, disp)


@pytest.fixture(params=["reference", pytest.param("gpu", marks=pytest.mark.gpu)])
def lib(request, reference):
    if request.param == "reference":
        return _Ref(reference)
    return request.getfixturevalue("ctx")


def test_dice_basics(lib):
    """test_metrics.cpp:27-53."""
    a = np.zeros((1, 4, 4), np.uint16)
    b = np.zeros_like(a)
    assert lib.dice(a, b, 1) == 1.0  # both empty
    a[0, 1, 1] = a[0, 2, 2] = 1
    assert lib.dice(a, a.copy(), 1) == 1.0
    a[:] = 0
    a[0, 0, 0] = 1
    b[0, 3, 3] = 1
    assert lib.dice(a, b, 1) == 0.0
    a[:] = 0
    b[:] = 0
    a[0, 0, 0] = a[0, 0, 1] = 1
    b[0, 0, 1] = b[0, 0, 2] = 1
    assert lib.dice(a, b, 1) == 0.5


def test_dice_symmetric_bounded(lib):
    """test_metrics.cpp:55-61."""
    a = random_labels((4, 8, 8), 3, 0.3)
    b = random_labels((4, 8, 8), 4, 0.3)
    d = lib.dice(a, b, 1)
    assert d == lib.dice(b, a, 1)
    assert 0.0 <= d <= 1.0


def test_hausdorff_identical_is_zero(lib):
    """test_metrics.cpp:63-66."""
    a = random_labels((3, 8, 8), 9, 0.4)
    assert lib.hausdorff_slice_avg(a, a, 1) == 0.0


def test_hausdorff_two_voxels(lib):
    """test_metrics.cpp:68-75: three voxels apart at 1.2 mm -> 3.6."""
    a = np.zeros((1, 8, 8), np.uint16)
    b = np.zeros_like(a)
    a[0, 4, 2] = 1
    b[0, 4, 5] = 1
    assert lib.hausdorff_slice_avg(a, b, 1, (1.2, 1.2, 1.0)) == pytest.approx(3.6, rel=1e-12)


def test_hausdorff_matches_all_pairs(lib):
    """test_metrics.cpp:77-85 (epsilon 1e-9)."""
    a = random_labels((4, 16, 16), 21, 0.15)
    b = random_labels((4, 16, 16), 22, 0.15)
    expected = brute_force_hausdorff(a, b, 1, (1.0, 1.0))
    assert expected >= 0.0
    assert lib.hausdorff_slice_avg(a, b, 1) == pytest.approx(expected, rel=1e-9)
    assert lib.hausdorff_slice_avg(b, a, 1) == pytest.approx(expected, rel=1e-9)


def test_hausdorff_anisotropic(lib):
    """test_metrics.cpp:87-98: spacing (0.7, 1.9) in plane."""
    r = Rng(31)
    u = r.uniform(2 * 12 * 10 * 3)
    a = (u[0::2] < 0.2).astype(np.uint16).reshape(3, 10, 12)
    b = (u[1::2] < 0.2).astype(np.uint16).reshape(3, 10, 12)
    expected = brute_force_hausdorff(a, b, 1, (0.7, 1.9))
    assert lib.hausdorff_slice_avg(a, b, 1, (0.7, 1.9, 2.0)) == pytest.approx(expected, rel=1e-9)


def test_hausdorff_needs_a_shared_slice(lib):
    """test_metrics.cpp:100-106."""
    a = np.zeros((2, 4, 4), np.uint16)
    b = np.zeros_like(a)
    a[0, 0, 0] = 1
    b[1, 0, 0] = 1
    with pytest.raises(ValueError):
        lib.hausdorff_slice_avg(a, b, 1)


def test_warp_labels_identity(lib):
    """test_metrics.cpp:108-112."""
    lbl = random_labels((6, 6, 6), 41, 0.3)
    assert np.array_equal(lib.warp_labels(lbl, np.zeros(lbl.shape + (3,), np.float32)), lbl)


def test_warp_labels_integer_translation(lib):
    """test_metrics.cpp:114-127: out(x) samples lbl at x+1, clamped at the edge."""
    lbl = np.zeros((3, 3, 5), np.uint16)
    lbl[1, 1, 2] = 7
    disp = np.zeros(lbl.shape + (3,), np.float32)
    disp[..., 0] = 1.0
    out = lib.warp_labels(lbl, disp)
    assert out[1, 1, 1] == 7 and out[1, 1, 2] == 0 and out[1, 1, 4] == lbl[1, 1, 4]


def test_warp_labels_per_voxel_loop(lib):
    """test_metrics.cpp:129-150: bit for bit against the lround/clamp loop."""
    lbl = random_labels((8, 8, 8), 51, 0.4)
    disp = random_field((8, 8, 8), 52, 2.0)
    out = lib.warp_labels(lbl, disp)
    z, y, x = np.meshgrid(np.arange(8), np.arange(8), np.arange(8), indexing="ij")

    def near(v, n):  # std::lround: half away from zero
        return np.clip((np.sign(v) * np.floor(np.abs(v) + 0.5)).astype(np.int64), 0, n - 1)

    d = disp.astype(np.float64)
    exp = lbl[near(z + d[..., 2], 8), near(y + d[..., 1], 8), near(x + d[..., 0], 8)]
    assert np.array_equal(out, exp)


def test_warped_label_set_is_subset(lib):
    """test_metrics.cpp:152-163."""
    lbl = (Rng(61).uniform(216) * 4.0).astype(np.uint16).reshape(6, 6, 6)
    out = lib.warp_labels(lbl, random_field((6, 6, 6), 62, 3.0))
    assert out.max() <= 3


# ---- GPU vs reference, bit-exact -----------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("shape,spacing,nl", [
    ((5, 17, 23), (1.0, 1.0, 1.0), 1),
    ((6, 31, 29), (0.7, 1.9, 2.0), 3),
    ((4, 64, 48), (1.3, 0.9, 2.5), 4),
    ((64, 128, 128), (1.25, 1.25, 8.0), 3),
])
def test_gpu_metrics_bit_exact_vs_reference(ctx, reference, shape, spacing, nl):
    r = Rng(sum(shape) + nl)
    a = (r.uniform(int(np.prod(shape))) * (nl + 1)).astype(np.uint16).reshape(shape)
    # b: a smoothly warped copy of a (realistic overlap) with some random flips
    disp = random_field(shape, 7, 1.6)
    b = reference.warp_labels(a, disp)
    flip = r.uniform(b.size).reshape(shape) < 0.05
    b = np.where(flip, (r.uniform(b.size).reshape(shape) * (nl + 1)).astype(np.uint16), b).astype(np.uint16)
    labels = list(range(1, nl + 1)) + [nl + 7]  # the last label is absent from both
    dice, hd, ok = ctx.label_metrics(a, b, labels, spacing)
    for j, lab in enumerate(labels):
        assert dice[j] == reference.dice(a, b, lab)
        assert ctx.dice(a, b, lab) == dice[j]
        if lab > nl:
            assert not ok[j] and dice[j] == 1.0
            continue
        assert ok[j]
        ref_hd = reference.hausdorff_slice_avg(a, b, lab, spacing)
        assert hd[j] == ref_hd, (lab, hd[j], ref_hd)
        assert ctx.hausdorff_slice_avg(a, b, lab, spacing) == ref_hd
    assert np.array_equal(ctx.warp_labels(a, disp), reference.warp_labels(a, disp))


@pytest.mark.gpu
def test_gpu_warped_synth_labels_vs_reference(ctx, reference):
    """The reference's sphere->ellipsoid labels through a smooth random deformation:
    warp + dice + hausdorff identical to the reference."""
    t, s, tl, sl = reference.make_case("sphere_ellipsoid", (32, 32, 32))
    disp = random_field((32, 32, 32), 99, 2.5)
    w_gpu = ctx.warp_labels(sl, disp)
    w_ref = reference.warp_labels(sl, disp)
    assert np.array_equal(w_gpu, w_ref)
    assert ctx.dice(w_gpu, tl, 1) == reference.dice(w_ref, tl, 1)
    assert ctx.hausdorff_slice_avg(w_gpu, tl, 1) == reference.hausdorff_slice_avg(w_ref, tl, 1)


@pytest.mark.gpu
def test_gpu_metrics_errors(ctx):
    a = np.zeros((2, 4, 4), np.uint16)
    with pytest.raises(ValueError):
        ctx.dice(a, np.zeros((2, 4, 5), np.uint16), 1)
    with pytest.raises(ValueError):
        ctx.hausdorff_slice_avg(a, a, 1, (0.0, 1.0, 1.0))
    with pytest.raises(ValueError):
        ctx.warp_labels(a, np.zeros((2, 4, 5, 3), np.float32))
