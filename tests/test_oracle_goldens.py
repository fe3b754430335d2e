"""Pin the CPU oracle to the reference itself.

tests/golden/ref_goldens.json is produced by oracle/ref_goldens.cpp compiled
against the reference's OWN Eigen-free headers (tensor.hpp, selector.hpp;
`make -C oracle goldens`).  The oracle's restatements must reproduce them
bit-for-bit (integers / RNG streams) or to the last ulp (doubles)."""
import json
from pathlib import Path

import numpy as np
import pytest

G = json.loads((Path(__file__).parent / "golden" / "ref_goldens.json").read_text())


def test_mix_seed_matches_reference(oracle):
    for seed, salt, want in G["mix_seed"]:
        assert oracle.mix_seed(seed, salt) == int(want)


def test_random_tensor_uniform_stream(oracle):
    x = oracle.random_tensor([3, 3], 42, "uniform01")
    assert x.ravel(order="F").tolist() == G["uniform_3x3_seed42"]


def test_random_tensor_normal_stream(oracle):
    x = oracle.random_tensor([3, 4, 5], 42, "normal")
    assert x.ravel(order="F").tolist() == G["normal_3x4x5_seed42"]
    assert oracle.frobenius_norm(x) == pytest.approx(G["normal_3x4x5_seed42_norm"], rel=1e-15)


def test_c1_input_matches_reference(oracle):
    """The C1 BASELINE input: random_tensor({200,200,200}, 1, StandardNormal)."""
    x = oracle.random_tensor([200, 200, 200], 1, "normal")
    flat = x.ravel(order="F")
    assert flat[:8].tolist() == G["c1_head"]
    assert flat[-4:].tolist() == G["c1_tail"]
    assert oracle.frobenius_norm(x) == pytest.approx(G["c1_norm"], rel=1e-14)


def test_als_initial_guess_stream(oracle):
    l0 = oracle.als_initial_guess(16, 1, 0, 0)
    assert l0.ravel(order="F").tolist() == G["als_l0_seed0_mode0"]
    l1 = oracle.als_initial_guess(4, 4, 3, 2)
    assert l1.ravel(order="F").tolist() == G["als_l0_seed3_mode2"]


def test_cost_model_matches_reference(oracle):
    cases = [(10, 2, 100), (200, 20, 40000), (1024, 32, 1048576), (2048, 64, 4194304), (48, 8, 5308416)]
    for (i, r, j), ce, ca in zip(cases, G["cost_eig"], G["cost_als"]):
        assert oracle.cost_eig(i, r, j) == ce
        assert oracle.cost_als(i, r, j) == pytest.approx(ca, rel=1e-15)


def test_cost_model_kats(oracle):
    """test_selector.cpp:65-81 / SPEC.md:435,444."""
    assert oracle.cost_eig(10, 2, 100) == 23000.0
    assert oracle.cost_als(10, 2, 100) == pytest.approx(49834.66667, abs=1e-5)


def test_hash_uniform_grid(oracle):
    v = oracle.hash_uniform(7, 100000)
    assert v.min() >= -1.0 and v.max() < 1.0
    k = v.astype(np.float64) * 2.0**23
    assert np.all(k == np.round(k))  # exact 2^-23 grid => exact in fp32
    assert abs(float(v.mean())) < 0.01
    np.testing.assert_array_equal(oracle.hash_uniform(7, 10, start=5), v[5:15])
