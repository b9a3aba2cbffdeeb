import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import CpuLib

    return CpuLib("oracle")


@pytest.fixture(scope="session")
def reference():
    from oracle.oracle import CpuLib, available

    if not available("reference"):
        pytest.skip("oracle/_ref/libdreg_ref.so not built (needs /root/reference at build time)")
    return CpuLib("reference")


@pytest.fixture(scope="session")
def ctx():
    from paper_2109_12688_b200 import dreg

    c = dreg.Context(0)
    yield c
    c.close()


class Rng:
    """std::mt19937 + gen()/2^32, like the reference tests (tests/oracles.hpp:19-27)."""

    def __init__(self, seed: int):
        self.bg = np.random.MT19937(0)
        self.bg._legacy_seeding(seed)

    def uniform(self, n, lo=0.0, hi=1.0):
        raw = self.bg.random_raw(n).astype(np.float64)
        return lo + (hi - lo) * (raw * (1.0 / 4294967296.0))


@pytest.fixture
def mt():
    return Rng


def random_volume(shape, seed, lo=0.0, hi=1.0):
    """oracles.cpp:23-30 (random_volume)."""
    return Rng(seed).uniform(int(np.prod(shape)), lo, hi).astype(np.float32).reshape(shape)


def random_field(shape, seed, amplitude):
    """oracles.cpp:32-39 (random_field)."""
    n = int(np.prod(shape)) * 3
    return Rng(seed).uniform(n, -amplitude, amplitude).astype(np.float32).reshape(tuple(shape) + (3,))


def smooth_random_field(shape, seed, amplitude, oracle_lib):
    """oracles.cpp:41-64: coarse random lattice, corner-aligned trilinear upsample."""
    z, y, x = shape
    coarse = (max(2, z // 4), max(2, y // 4), max(2, x // 4))
    lat = random_field(coarse, seed, amplitude)
    # upsample_velocity doubles the field; the oracle helper does not -> halve.
    return oracle_lib.upsample_velocity(lat, (x, y, z)) * np.float32(0.5)


def max_abs(a, b):
    return float(np.max(np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64))))


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
