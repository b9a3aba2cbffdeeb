"""The reference's own hot-path test pins (proj/tests/test_{admm,volume,regularizer,
registration}.cpp and acceptance_main.cpp), restated with numpy and run against the
CPU oracle (always) and the sm_100a path (-m gpu).  Cited per test; parameters and
tolerances follow the reference unless noted (the GPU spectral solve is fp32, held
to the reference's own 1e-5 * max|ref| w-update tolerance).
"""
import numpy as np
import pytest

from conftest import Rng, max_abs, random_field, random_volume, rel_l2, smooth_random_field
from paper_2109_12688_b200 import abi


@pytest.fixture(params=["oracle", pytest.param("gpu", marks=pytest.mark.gpu)])
def lib(request, oracle):
    if request.param == "oracle":
        return oracle
    return request.getfixturevalue("ctx")


def dense_neg_laplacian(shape):
    """oracles.cpp:111-131: periodic 7-point negative Laplacian, voxels x voxels."""
    z, y, x = shape
    n = x * y * z
    m = np.zeros((n, n))
    idx = lambda xx, yy, zz: (xx % x) + x * ((yy % y) + y * (zz % z))  # noqa: E731
    for k in range(z):
        for j in range(y):
            for i in range(x):
                r = idx(i, j, k)
                m[r, r] += 6.0
                for d in ((-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0), (0, 0, -1), (0, 0, 1)):
                    m[r, idx(i + d[0], j + d[1], k + d[2])] -= 1.0
    return m


def dense_w_solve(rhs, order, lam, theta):
    """oracles.cpp:141-164: (lambda K^n + theta I) w = theta rhs per component."""
    shp = rhs.shape[:3]
    K = np.linalg.matrix_power(dense_neg_laplacian(shp), order)
    A = lam * K + theta * np.eye(K.shape[0])
    out = np.zeros_like(rhs, dtype=np.float64)
    for c in range(3):
        out[..., c] = np.linalg.solve(A, theta * rhs[..., c].reshape(-1).astype(np.float64)).reshape(shp)
    return out


# ---- test_admm.cpp ---------------------------------------------------------------
def test_alpha_sequence(lib):
    """test_admm.cpp:53-64: alpha_1 = 1.618034, first coefficient 0, increasing."""
    a = 1.0
    nxt = lib.nesterov_next_alpha(a)
    assert abs(nxt - 1.618034) < 1e-6
    assert (a - 1.0) / nxt == 0.0
    prev = nxt
    for _ in range(50):
        cur = lib.nesterov_next_alpha(prev)
        assert cur > prev
        prev = cur


def _one_voxel(vals):
    return np.array(vals, np.float32).reshape(1, 1, 1, 3)


def test_l1_zero_residual_returns_u(lib):
    """test_admm.cpp:66-89: rho(w_hat - b_hat) = 0 -> v = w_hat - b_hat (theta 0.07)."""
    g = _one_voxel([0.5, -0.25, 1.0])
    wh, bh = _one_voxel([0.3, 0.1, -0.2]), _one_voxel([0.1, -0.1, 0.05])
    u = (wh.astype(np.float64) - bh)
    # choose warped - target so that g.u + d = 0
    d = -float((g.astype(np.float64) * u).sum())
    t = np.zeros((1, 1, 1), np.float32)
    w = np.array(d, np.float32).reshape(1, 1, 1)
    out = lib.v_update(t, w, g, wh, bh, abi.solver_cfg(data_term=1, theta=0.07))
    assert np.allclose(out, u, atol=1e-6)


@pytest.mark.parametrize("dt", [1, 2])
def test_zero_gradient_returns_u(lib, dt):
    """test_admm.cpp:91-109 (l1, theta 0.1) and :136-153 (l2, 2^3, seeds 9/10, theta 0.05)."""
    shp = (2, 2, 2)
    wh, bh = random_field(shp, 9, 1.0), random_field(shp, 10, 1.0)
    g = np.zeros_like(wh)
    t, w = random_volume(shp, 11), random_volume(shp, 12)
    out = lib.v_update(t, w, g, wh, bh, abi.solver_cfg(data_term=dt, theta=0.1 if dt == 1 else 0.05))
    assert np.allclose(out, wh.astype(np.float64) - bh, atol=1e-6)


def test_l2_normal_equation(lib):
    """test_admm.cpp:155-182: (g g^T + theta I) v = theta u - d g; 8^3 seed 900, theta 0.09."""
    shp = (8, 8, 8)
    g, wh, bh = random_field(shp, 900, 1.0), random_field(shp, 901, 1.0), random_field(shp, 902, 1.0)
    t, w = random_volume(shp, 903), random_volume(shp, 904)
    theta = 0.09
    v = lib.v_update(t, w, g, wh, bh, abi.solver_cfg(data_term=2, theta=theta)).astype(np.float64)
    g64 = g.astype(np.float64)
    u = wh.astype(np.float64) - bh
    d = (w.astype(np.float64) - t)[..., None]
    rhs = theta * u - d * g64
    lhs = g64 * (g64 * v).sum(-1, keepdims=True) + theta * v
    scale = 1.0 + np.abs(rhs).max()
    assert np.abs(lhs - rhs).max() <= 1e-5 * scale * 10  # fp32 storage of v


def test_l1_matches_line_search(lib):
    """test_admm.cpp:111-134: closed-form l1 vs a dense sweep of t in u + t g (theta 0.08)."""
    shp = (4, 4, 4)
    theta = 0.08
    for seed in range(500, 503):
        g, wh, bh = random_field(shp, seed, 1.0), random_field(shp, seed + 10, 1.0), random_field(shp, seed + 20, 1.0)
        t, w = random_volume(shp, seed + 30), random_volume(shp, seed + 40)
        v = lib.v_update(t, w, g, wh, bh, abi.solver_cfg(data_term=1, theta=theta)).astype(np.float64)
        g64 = g.astype(np.float64).reshape(-1, 3)
        u = (wh.astype(np.float64) - bh).reshape(-1, 3)
        d = (w.astype(np.float64) - t).reshape(-1)
        gg = (g64 * g64).sum(1)
        rho_u = (g64 * u).sum(1) + d
        # objective along the gradient direction: |rho(u) + t gg| + theta/2 t^2 gg
        ts = np.linspace(-40, 40, 160001)
        for i in range(0, u.shape[0], 7):
            f = np.abs(rho_u[i] + ts * gg[i]) + 0.5 * theta * ts * ts * gg[i]
            tb = ts[np.argmin(f)]
            assert np.allclose(v.reshape(-1, 3)[i], u[i] + tb * g64[i], atol=2e-3)


@pytest.mark.parametrize("shape", [(4, 4, 4), (4, 6, 4), (4, 4, 5)])
@pytest.mark.parametrize("order", [1, 2])
def test_w_update_dense_solve(lib, shape, order):
    """test_admm.cpp:184-211: w_update == dense periodic solve, lambda 2, theta 0.1."""
    v, bh = random_field(shape, 40 + order, 1.0), random_field(shape, 50 + order, 1.0)
    out = lib.w_update(v, bh, abi.solver_cfg(order=order, lambda_=2.0, theta=0.1))
    ref = dense_w_solve(v.astype(np.float64) + bh, order, 2.0, 0.1)
    assert np.abs(out - ref).max() <= 1e-5 * np.abs(ref).max()


def test_w_update_lambda_zero_and_constant(lib):
    """test_admm.cpp:213-248: lambda 0 -> v + b_hat; constant field passes through."""
    v, bh = random_field((6, 6, 6), 60, 1.0), random_field((6, 6, 6), 61, 1.0)
    out = lib.w_update(v, bh, abi.solver_cfg(order=2, lambda_=0.0, theta=0.1))
    assert np.abs(out - (v.astype(np.float64) + bh)).max() <= 1e-5
    c = np.full((4, 4, 4, 3), 0.75, np.float32)
    out = lib.w_update(c, np.zeros_like(c), abi.solver_cfg(order=2, lambda_=3.0, theta=0.1))
    assert np.abs(out - 0.75).max() <= 1e-6


def test_identical_images_give_zero_velocity(lib):
    """test_admm.cpp:250-266: I0 == I1 -> mean |v| <= 1e-4."""
    blob = gaussian_blob((12, 12, 12), (5.5, 5.5, 5.5), 3.0)
    v, d = lib.solve_velocity(blob, blob,
                              abi.solver_cfg(data_term=1, order=1, lambda_=1.0, theta=0.1, max_iters=50, tol=1e-7))
    assert np.abs(v).mean() <= 1e-4


def test_constraint_residual_shrinks(lib):
    """test_admm.cpp:268-284: l2, n 1, lambda 2, theta 0.05, tol 1e-4 on 16^3."""
    zz, yy, xx = np.mgrid[0:16, 0:16, 0:16]
    a = np.exp(-((xx - 7.5) ** 2 + (yy - 8) ** 2 + (zz - 8) ** 2) / 18.0).astype(np.float32)
    b = np.exp(-((xx - 8.5) ** 2 + (yy - 8) ** 2 + (zz - 8) ** 2) / 18.0).astype(np.float32)
    v, d = lib.solve_velocity(a, b, abi.solver_cfg(data_term=2, order=1, lambda_=2.0, theta=0.05, max_iters=400,
                                                   tol=1e-4, log_objective=False))
    r = d["constraint_residual"]
    assert r[-1] < r[0]


def gaussian_blob(shape, centre, sigma):
    """test_admm.cpp:35-47."""
    z, y, x = shape
    zz, yy, xx = np.mgrid[0:z, 0:y, 0:x].astype(np.float64)
    d2 = (xx - centre[0]) ** 2 + (yy - centre[1]) ** 2 + (zz - centre[2]) ** 2
    return np.exp(-d2 / (2.0 * sigma * sigma)).astype(np.float32)


def test_objective_matches_direct_solve(lib, oracle):
    """test_admm.cpp:286-360: 16^3 blobs, l2 data term, n = 1, lambda 1.5, theta 0.05,
    400 iterations, tol 1e-6: the final ADMM objective is within 1% of the objective of
    the direct solve of (blockdiag(g g^T) + lambda K per component) v = -g diff
    (periodic 7-point K; scipy sparse LU in place of Eigen's SimplicialLDLT)."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla

    shape = (16, 16, 16)
    target = gaussian_blob(shape, (7.5, 7.5, 7.5), 3.5)
    source = gaussian_blob(shape, (8.5, 7.5, 7.5), 3.5)
    lam = 1.5
    cfg = abi.solver_cfg(data_term=2, order=1, lambda_=lam, theta=0.05, max_iters=400, tol=1e-6, log_objective=True)
    v, d = lib.solve_velocity(target, source, cfg)
    assert d["objective"].size > 0
    admm_obj = d["objective"][-1]

    g = oracle.image_gradient(source).astype(np.float64).reshape(-1, 3)  # voxel-major, x fastest
    n = g.shape[0]
    K = sp.csr_matrix(dense_neg_laplacian(shape))
    A = sp.kron(K, sp.identity(3), format="csr") * lam  # unknown 3 i + c
    rows = np.repeat(np.arange(n) * 3, 9) + np.tile(np.repeat(np.arange(3), 3), n)
    cols = np.repeat(np.arange(n) * 3, 9) + np.tile(np.tile(np.arange(3), 3), n)
    A = A + sp.csr_matrix((np.einsum("ic,id->icd", g, g).reshape(-1), (rows, cols)), shape=A.shape)
    diff = source.astype(np.float64).reshape(-1) - target.astype(np.float64).reshape(-1)
    x = spla.spsolve(A.tocsc(), (-g * diff[:, None]).reshape(-1))
    direct = x.reshape(shape + (3,)).astype(np.float32)
    grad = oracle.image_gradient(source)
    direct_obj = oracle.data_term_value(target, source, grad, direct, 2) + lam * oracle.regulariser_energy(direct, 1)
    assert abs(admm_obj - direct_obj) <= 0.01 * abs(direct_obj), (admm_obj, direct_obj)


def test_accelerate_on_off_same_objective(lib):
    """test_admm.cpp:362-382: accelerated and plain both converge to objectives within 1%."""
    t = gaussian_blob((12, 12, 12), (5.5, 5.5, 5.5), 2.5)
    s = gaussian_blob((12, 12, 12), (6.3, 5.5, 5.5), 2.5)
    objs = []
    for acc in (True, False):
        v, d = lib.solve_velocity(t, s, abi.solver_cfg(data_term=2, order=2, lambda_=3.0, theta=0.05, max_iters=400,
                                                       tol=1e-5, accelerate=acc, log_objective=True))
        assert d["converged"]
        objs.append(d["objective"][-1])
    assert abs(objs[0] - objs[1]) <= 0.01 * abs(objs[1])


def test_acceptance_acceleration_criterion(lib):
    """acceptance_main.cpp:164-210 (criterion 3): 32^3 sinusoid shifted by 4 voxels,
    accelerated needs <= the plain iterations and objectives agree within 1%."""
    r = Rng(11)
    ph = r.uniform(3, 0.0, 6.28)
    zz, yy, xx = np.mgrid[0:32, 0:32, 0:32].astype(np.float64)
    img = lambda x, y, z: 0.5 + 0.4 * np.sin(2 * 3.14159265358979 * x / 16 + ph[0]) * \
        np.sin(2 * 3.14159265358979 * y / 16 + ph[1]) * np.sin(2 * 3.14159265358979 * z / 16 + ph[2])  # noqa: E731
    t = img(xx, yy, zz).astype(np.float32)
    s = img(xx + 4.0, yy, zz).astype(np.float32)
    res = []
    for acc in (True, False):
        v, d = lib.solve_velocity(t, s, abi.solver_cfg(data_term=2, order=2, lambda_=1.0, theta=0.02, max_iters=2000,
                                                       tol=0.01, accelerate=acc, log_objective=True))
        assert d["converged"]
        res.append((d["iterations"], d["objective"][-1]))
    assert res[0][0] <= res[1][0]
    assert abs(res[0][1] - res[1][1]) <= 0.01 * abs(res[1][1])


# ---- test_regularizer.cpp ---------------------------------------------------------
@pytest.mark.parametrize("n", [1, 2, 3])
def test_symbol_identities(oracle, n):
    """test_regularizer.cpp:66-101: zero at DC, 4^n at pure-x Nyquist, <= 12^n."""
    k = oracle.laplacian_symbol(n, (8, 6, 4))
    assert k[0, 0, 0] == 0.0
    assert abs(k[0, 0, 4] - 4.0 ** n) <= 1e-9 * 4.0 ** n
    assert k.max() <= 12.0 ** n + 1e-9


@pytest.mark.parametrize("n", [1, 2])
def test_energy_dense_form_and_homogeneity(lib, n):
    """test_regularizer.cpp:114-154: energy == 0.5 sum w^T K^n w; quadratic in w."""
    w = random_field((4, 5, 4), 70 + n, 1.0)
    K = np.linalg.matrix_power(dense_neg_laplacian(w.shape[:3]), n)
    ref = 0.5 * sum(w[..., c].reshape(-1).astype(np.float64) @ K @ w[..., c].reshape(-1).astype(np.float64)
                    for c in range(3))
    e = lib.regulariser_energy(w, n)
    assert abs(e - ref) <= (1e-9 if lib.__class__.__name__ == "CpuLib" else 2e-6) * abs(ref)
    e2 = lib.regulariser_energy(w * np.float32(2.0), n)
    assert abs(e2 - 4 * e) <= 1e-5 * abs(e2)


# ---- test_volume.cpp --------------------------------------------------------------
def test_trilinear_lattice_and_clamp(lib):
    """test_volume.cpp:39-70: lattice points exact; clamped outside; affine images exact."""
    shp = (8, 8, 8)
    zz, yy, xx = np.mgrid[0:8, 0:8, 0:8].astype(np.float32)
    affine = (0.5 * xx + 0.25 * yy - 0.125 * zz + 1.0).astype(np.float32)
    disp = np.zeros(shp + (3,), np.float32)
    disp[..., 0] = 0.5
    out = lib.warp_image(affine, disp)
    expect = 0.5 * np.minimum(xx + 0.5, 7) + 0.25 * yy - 0.125 * zz + 1.0
    assert np.allclose(out, expect, atol=1e-6)
    disp[..., 0] = -20.0
    out = lib.warp_image(affine, disp)
    assert np.allclose(out, 0.25 * yy - 0.125 * zz + 1.0, atol=1e-6)


def test_warp_matches_naive(lib):
    """test_volume.cpp:79-97: warp == naive trilinear oracle (1e-6), 8^3 seeds 21/22, amplitude 1.5."""
    img, disp = random_volume((8, 8, 8), 21), random_field((8, 8, 8), 22, 1.5)
    out = lib.warp_image(img, disp)
    z, y, x = img.shape
    ref = np.zeros_like(out, dtype=np.float64)
    for k in range(z):
        for j in range(y):
            for i in range(x):
                p = np.array([i, j, k], np.float64) + disp[k, j, i].astype(np.float64)
                c = np.clip(p, 0, np.array([x - 1, y - 1, z - 1], np.float64))
                lo = np.floor(c).astype(int)
                hi = np.minimum(lo + 1, [x - 1, y - 1, z - 1])
                f = c - lo
                acc = 0.0
                for dz in (0, 1):
                    for dy in (0, 1):
                        for dx in (0, 1):
                            wgt = (f[0] if dx else 1 - f[0]) * (f[1] if dy else 1 - f[1]) * (f[2] if dz else 1 - f[2])
                            acc += wgt * img[hi[2] if dz else lo[2], hi[1] if dy else lo[1], hi[0] if dx else lo[0]]
                ref[k, j, i] = acc
    assert np.abs(out - ref).max() <= 1e-6


def test_gradient_exact_cases(lib):
    """test_volume.cpp:105-141: ramp, constant and quadratic profiles."""
    zz, yy, xx = np.mgrid[0:6, 0:7, 0:8].astype(np.float32)
    g = lib.image_gradient((2 * xx - 3 * yy + 0.5 * zz).astype(np.float32))
    assert np.allclose(g[..., 0], 2) and np.allclose(g[..., 1], -3) and np.allclose(g[..., 2], 0.5)
    assert np.array_equal(lib.image_gradient(np.full((4, 4, 4), 3.0, np.float32)), np.zeros((4, 4, 4, 3), np.float32))
    q = (xx * xx).astype(np.float32)
    g = lib.image_gradient(q)
    assert np.allclose(g[:, :, 1:-1, 0], 2 * xx[:, :, 1:-1])  # central difference exact on quadratics
    assert np.allclose(g[:, :, 0, 0], 1.0) and np.allclose(g[:, :, -1, 0], 49 - 36)


def test_compose_translations_add(lib, oracle):
    """test_volume.cpp:148-190: v = 0 bit-exact; translations add."""
    a = smooth_random_field((8, 8, 8), 51, 0.4, oracle)
    assert np.array_equal(lib.compose_deformation(a, np.zeros_like(a)), a)
    t1 = np.zeros((8, 8, 8, 3), np.float32)
    t1[..., 0] = 0.5
    t2 = np.zeros_like(t1)
    t2[..., 1] = -0.25
    out = lib.compose_deformation(t1, t2)
    interior = out[1:-1, 1:-1, 1:-1]
    assert np.allclose(interior[..., 0], 0.5) and np.allclose(interior[..., 1], -0.25)


def test_jacobian_identities(lib):
    """test_volume.cpp:214-248: det 1 for identity/translation; (1+a)(1+b)(1+c) for linear maps."""
    u = np.zeros((6, 7, 8, 3), np.float32)
    assert np.allclose(lib.jacobian_determinant(u), 1.0)
    u[..., 0] = 1.25
    assert np.allclose(lib.jacobian_determinant(u), 1.0)
    zz, yy, xx = np.mgrid[0:6, 0:7, 0:8].astype(np.float32)
    u = np.stack([0.1 * xx, -0.2 * yy, 0.3 * zz], -1).astype(np.float32)
    assert np.allclose(lib.jacobian_determinant(u), 1.1 * 0.8 * 1.3, atol=1e-5)


# ---- test_registration.cpp -----------------------------------------------------------
def test_register_identity_pair(lib):
    """test_registration.cpp:197-210: identity pair -> mean |u| <= 0.05."""
    from paper_2109_12688_b200 import synth

    f, _ = synth.make_pair(1, 9, (16, 16, 16))
    s = abi.solver_cfg(data_term=1, order=2, lambda_=5.0, theta=0.05, max_iters=10, log_objective=False)
    phi, warped, res = lib.register_pair(f, f, abi.reg_cfg(s, 1, (5,), (10,)))
    assert np.abs(phi).mean() <= 0.05


def test_register_translation_recovery(lib):
    """test_registration.cpp:211-230: a translated blob is recovered (interior mean error)."""
    zz, yy, xx = np.mgrid[0:24, 0:24, 0:24].astype(np.float64)
    t = np.exp(-((xx - 12) ** 2 + (yy - 12) ** 2 + (zz - 12) ** 2) / (2 * 16.0)).astype(np.float32)
    s = np.exp(-((xx - 13) ** 2 + (yy - 12) ** 2 + (zz - 12) ** 2) / (2 * 16.0)).astype(np.float32)
    cfg = abi.reg_cfg(abi.solver_cfg(data_term=2, order=2, lambda_=0.05, theta=0.5, max_iters=50,
                                     log_objective=False), 1, (10,), (50,))
    phi, warped, res = lib.register_pair(t, s, cfg)
    core = phi[8:16, 8:16, 8:16]
    assert abs(core[..., 0].mean() - 1.0) <= 0.5
    assert res.velocity_count >= 1
    # accepted mean SAD is monotone (test_registration.cpp:263-284)
    ms = abi.level_logs(res)[0]["mean_sad"]
    assert all(b <= a for a, b in zip(ms, ms[1:]))


def test_register_rejects_bad_input(lib):
    """test_registration.cpp:304-349: NaN -> numeric_error; invalid configs -> invalid_argument."""
    f = random_volume((8, 8, 8), 5)
    m = f.copy()
    m[1, 2, 3] = np.nan
    ok = abi.reg_cfg(abi.solver_cfg(max_iters=2), 1, (1,), (2,))
    with pytest.raises(Exception) as e:
        lib.register_pair(f, m, ok)
    assert "non-finite" in str(e.value)
    bad = abi.reg_cfg(abi.solver_cfg(order=7), 1, (1,), (2,))
    with pytest.raises(Exception):
        lib.register_pair(f, f, bad)


# ---- the reference's own synthetic cases (synth.cpp via oracle/_ref) -------------------
def _capped(data_term, lam, levels, theta=0.05):
    from paper_2109_12688_b200 import dreg

    s = abi.solver_cfg(data_term=data_term, order=2, lambda_=lam, theta=theta, log_objective=False)
    return dreg.make_registration_config(abi.DREG_PROFILE_CAPPED, s, levels)


def test_register_identical_sphere_case(lib, reference):
    """test_registration.cpp:197-215: sphere case 16^3 registered to itself (l1, n 2,
    lambda 10, capped, 2 levels) stays near the identity: mean |u| <= 0.05 and the
    warped target labels keep Dice >= 0.99."""
    t, _, tl, _ = reference.make_case("sphere_ellipsoid", (16, 16, 16))
    phi, warped, res = lib.register_pair(t, t, _capped(1, 10.0, 2))
    assert np.abs(phi.astype(np.float64)).mean() <= 0.05
    assert reference.warped_label_dice(tl, phi, tl) >= 0.99


def test_register_translate_case_recovery(lib, reference):
    """test_registration.cpp:217-245: 32^3 blob shifted by (2, 0, 0) (l1, n 2, lambda 10,
    capped, 3 levels): mean displacement over label 1 within 0.5 voxel of -shift, and
    the result's warped image is warp_image(source, phi) bit for bit."""
    t, s, tl, _ = reference.make_case("translate", (32, 32, 32), shift=(2.0, 0.0, 0.0))
    phi, warped, res = lib.register_pair(t, s, _capped(1, 10.0, 3))
    mean = phi[tl == 1].astype(np.float64).mean(0)
    assert np.linalg.norm(mean - np.array([-2.0, 0.0, 0.0])) <= 0.5, mean
    assert np.array_equal(lib.warp_image(s, phi), warped)


def test_register_sphere_to_ellipsoid(lib, reference):
    """test_registration.cpp:247-261: 32^3 sphere -> ellipsoid (l1, n 2, lambda 5, capped,
    3 levels): Dice(warp_labels(source labels, phi), target labels) >= 0.90 and no
    non-positive Jacobian."""
    t, s, tl, sl = reference.make_case("sphere_ellipsoid", (32, 32, 32))
    phi, warped, res = lib.register_pair(t, s, _capped(1, 5.0, 3))
    assert reference.warped_label_dice(sl, phi, tl) >= 0.90
    assert lib.jacobian_stats(phi).nonpositive == 0


def test_acceptance_diffeomorphism(lib, reference, oracle):
    """acceptance_main.cpp:261-291 (criterion 5): 13 registrations at 32^3 -- translate
    (3, 0, 0), sphere -> ellipsoid, random smooth seeds 3 and 100..109 (l1, n 2,
    lambda 10, theta 0.05, capped, 3 levels) -- all with 0% non-positive Jacobians.

    The GPU additionally matches the oracle's velocity count and phi within the contract
    (max-abs 1e-3, rel-L2 1e-4).  The l1 pyramid is chaotic (the shrinkage
    z / max(|z|, 1) switches branch on rounding-level changes: the oracle itself moves
    phi by up to 0.27 voxel under a 1-ulp change of the target), so the
    l1 path runs the precise mode, which repeats the reference's arithmetic (fp64
    spectrum, the reference's multiplier expression, unfused fp64 point-wise updates):
    on all 13 cases phi is bit-identical to the oracle (tools/l1_parity_table.py)."""
    cases = [("translate", dict(shift=(3.0, 0.0, 0.0))), ("sphere_ellipsoid", {})]
    cases += [("random_smooth", dict(seed=sd)) for sd in [3] + list(range(100, 110))]
    cfg = _capped(1, 10.0, 3)
    identical = 0
    for kind, kw in cases:
        t, s, _, _ = reference.make_case(kind, (32, 32, 32), **kw)
        phi, warped, res = lib.register_pair(t, s, cfg)
        st = lib.jacobian_stats(phi)
        assert st.nonpositive == 0 and st.pct_nonpositive == 0.0, (kind, kw, st.nonpositive)
        if lib is not oracle:
            phi_o, _, res_o = oracle.register_pair(t, s, cfg)
            assert res.velocity_count == res_o.velocity_count, (kind, kw)
            err, rel = max_abs(phi, phi_o), rel_l2(phi, phi_o)
            assert err <= 1e-3 and rel <= 1e-4, (kind, kw, err, rel)
            identical += int(np.array_equal(phi, phi_o))
    if lib is not oracle:
        print(f"criterion 5: {identical}/13 phi bit-identical to the oracle")


def test_accepted_sad_monotone_and_velocity_bound(lib, reference):
    """test_registration.cpp:263-284: per level the accepted mean SAD is monotone
    non-increasing and velocity_count <= the sum of the per-level warp caps."""
    t, s, _, _ = reference.make_case("random_smooth", (32, 32, 32), seed=7)
    cfg = _capped(1, 10.0, 3)
    phi, warped, res = lib.register_pair(t, s, cfg)
    assert res.velocity_count <= sum(cfg.max_warps_per_level[l] for l in range(cfg.levels))
    for l in range(res.levels):
        lg = res.per_level[l]
        sad = [lg.mean_sad[i] for i in range(lg.warps + 1)]
        assert all(b <= a for a, b in zip(sad, sad[1:])), (l, sad)


# ---- argument checks and identities (test_volume.cpp, test_registration.cpp) ----------
def _expect_invalid(fn):
    """std::invalid_argument in the reference: status 2 through the C ABI (ValueError on
    the sm_100a path, OracleError(status=2) on the oracle)."""
    with pytest.raises(Exception) as e:
        fn()
    assert isinstance(e.value, ValueError) or getattr(e.value, "status", None) == 2, repr(e.value)


def test_gradient_rejects_short_axes(lib):
    """test_volume.cpp:143-146: an axis shorter than 2 is invalid."""
    _expect_invalid(lambda: lib.image_gradient(np.zeros((4, 4, 1), np.float32)))


def test_jacobian_rejects_short_axes(lib):
    """test_volume.cpp:250-253: an axis shorter than 3 is invalid."""
    _expect_invalid(lambda: lib.jacobian_determinant(np.zeros((5, 5, 2, 3), np.float32)))


def test_upsample_rejects_shrinking_target(lib):
    """test_registration.cpp:121-124: a target smaller than the source is invalid."""
    _expect_invalid(lambda: lib.upsample_velocity(np.zeros((4, 4, 4, 3), np.float32), (3, 4, 4)))


def test_upsample_zero_and_uniform(lib):
    """test_registration.cpp:101-119: zero stays zero, a uniform field doubles."""
    assert not lib.upsample_velocity(np.zeros((4, 4, 4, 3), np.float32), (8, 8, 8)).any()
    u = np.zeros((4, 4, 4, 3), np.float32)
    u[..., 0] = 1.0
    up = lib.upsample_velocity(u, (8, 8, 8))
    assert np.allclose(up[..., 0], 2.0) and not up[..., 1:].any()


def test_downsample_odd_axis_edge_replication(lib):
    """test_registration.cpp:93-99: {3,2,2} of ones -> {2,1,1} of ones."""
    out = lib.downsample(np.ones((2, 2, 3), np.float32))
    assert out.shape == (1, 1, 2) and np.allclose(out, 1.0)


def test_composition_agrees_with_warping_twice(lib, oracle):
    """test_volume.cpp:171-212: warp(I, compose(phi, v)) ~ warp(warp(I, phi), v) two
    voxels in from the faces, within 1e-3 of the image range."""
    zz, yy, xx = np.mgrid[0:8, 0:8, 0:8].astype(np.float64)
    bump = np.exp(-((xx - 3.5) ** 2 + (yy - 3.5) ** 2 + (zz - 3.5) ** 2) / 16.0)
    img = (xx + 0.5 * yy + 0.25 * zz + 0.05 * bump).astype(np.float32)
    phi = smooth_random_field((8, 8, 8), 51, 0.4, oracle)
    v = smooth_random_field((8, 8, 8), 52, 0.4, oracle)
    composed = lib.warp_image(img, lib.compose_deformation(phi, v))
    twice = lib.warp_image(lib.warp_image(img, phi), v)
    tol = 1e-3 * float(img.max() - img.min())
    assert np.abs(composed - twice)[2:-2, 2:-2, 2:-2].max() <= tol


def test_operations_deterministic(lib):
    """test_volume.cpp:255-264: warp and gradient are bit-reproducible."""
    img = random_volume((8, 8, 8), 77)
    phi = random_field((8, 8, 8), 78, 1.0)
    assert np.array_equal(lib.warp_image(img, phi), lib.warp_image(img, phi))
    assert np.array_equal(lib.image_gradient(img), lib.image_gradient(img))


def test_downsample_identities(lib):
    """test_registration.cpp:60-91: constant kept, 2x2x2 block -> its mean, ramp slope doubles."""
    out = lib.downsample(np.full((8, 8, 8), 2.5, np.float32))
    assert out.shape == (4, 4, 4) and np.allclose(out, 2.5)
    assert np.allclose(lib.downsample(np.arange(8, dtype=np.float32).reshape(2, 2, 2)), 3.5)
    ramp = np.broadcast_to(np.arange(8, dtype=np.float32), (4, 4, 8)).copy()
    out = lib.downsample(ramp)
    assert np.allclose(out[0, 0, :], 2.0 * np.arange(4) + 0.5)


# ---- test_metrics.cpp (jacobian_stats) ---------------------------------------------
def test_jacobian_stats_identity_translation_and_folding(lib):
    """test_metrics.cpp:160-187: identity and translations give 0% / min det 1; the
    field u_x = -2x folds every interior voxel (100%, min det -1)."""
    u = np.zeros((6, 6, 6, 3), np.float32)
    st = lib.jacobian_stats(u)
    assert st.pct_nonpositive == 0.0 and abs(st.min_det - 1.0) < 1e-9 and st.interior == 64
    u[...] = (2.0, -1.0, 0.5)
    st = lib.jacobian_stats(u)
    assert st.pct_nonpositive == 0.0 and abs(st.min_det - 1.0) < 1e-9
    u = np.zeros((6, 6, 6, 3), np.float32)
    u[..., 0] = -2.0 * np.arange(6, dtype=np.float32)[None, None, :]
    st = lib.jacobian_stats(u)
    assert abs(st.pct_nonpositive - 100.0) < 1e-9 and abs(st.min_det + 1.0) < 1e-9 and st.nonpositive == 64
