"""Synthetic BASELINE inputs: determinism, sizes, and the device density recipe."""

import numpy as np
import pytest

from paper_1401_6961_b200 import configs


def test_sizes_match_survey_appendix_b():
    c1 = configs.config1()
    assert (c1.n_shells, c1.n_functions) == (32, 32)
    c2 = configs.config2()
    assert (c2.n_shells, c2.n_functions) == (512, 768)
    c3 = configs.config3(host_density=False)
    assert (c3.n_shells, c3.n_functions) == (1280, 1792)


def test_density_is_symmetric_with_unit_diagonal():
    cfg = configs.cube_cluster(3, 9, "tiny")
    P = cfg.P
    assert np.array_equal(P, P.T)
    assert np.all(np.diag(P) == 1.0)
    off = np.abs(P[~np.eye(len(P), dtype=bool)])
    assert off.max() <= 1.0 and off.min() > 0.0


def test_device_density_recipe_matches_host():
    torch = pytest.importorskip("torch")
    cfg = configs.cube_cluster(4, 11, "tiny")
    Pd = configs.decay_density_device(cfg.system, cfg.density_seed, "cpu").numpy()
    assert np.array_equal(np.sign(Pd), np.sign(cfg.P))
    assert np.allclose(Pd, cfg.P, rtol=2e-15, atol=0)  # exp/sqrt last-ulp differences
    assert np.array_equal(Pd, Pd.T)
    del torch


def test_generation_is_deterministic():
    a = configs.config2(n_centers=12)
    b = configs.config2(n_centers=12)
    assert np.array_equal(a.P, b.P)
    assert np.array_equal(np.array([s.center for s in a.system.shells]),
                          np.array([s.center for s in b.system.shells]))
