"""Pins for the seeded input generators (datagen/), CPU only."""
import json
import os

import numpy as np

import datagen

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold():
    with open(os.path.join(GOLD, "spec_examples.json")) as fh:
        return json.load(fh)


def test_closed_forms_root_and_two_dups():
    """P:351 / P:353: the shuffled arrays hold exactly the multiset
    of the closed forms; exhaustive at n <= 10^4."""
    g = gold()
    for name, key in (("rootdups", "root_dups_formula"), ("twodups", "two_dups_formula")):
        n = g[key]["n"]
        got = datagen.generate_host(name, n, 1)
        assert sorted(got.tolist()) == sorted(g[key]["expect_unshuffled"])
    for n in (10, 97, 1000, 10_000):
        i = np.arange(n, dtype=np.uint64)
        r = int(np.floor(np.sqrt(n)))
        while r * r > n:
            r -= 1
        assert np.array_equal(np.sort(datagen.generate_host("rootdups", n, 1)), np.sort(i % np.uint64(r)))
        two = (i * i + np.uint64(n // 2)) % np.uint64(n)
        assert np.array_equal(np.sort(datagen.generate_host("twodups", n, 1)), np.sort(two))
        # the shuffle is a permutation of positions: not the identity
        assert not np.array_equal(datagen.generate_host("rootdups", n, 1), i % np.uint64(r))


def test_duplicate_ratio_examples():
    for keys, expect in gold()["duplicate_ratio"]["cases"]:
        assert abs(datagen.duplicate_ratio(np.array(keys, dtype=np.uint64)) - expect) < 1e-12


def test_zipf_paper_anchor():
    """"Zipfian distribution with skew 0.9, which corresponds to 72%
    duplicates" (universe unstated; S:297 band 0.72 +- 0.08, universe = n)."""
    x = datagen.generate_host("zipf", 10_000_000, 0, zipf_s=0.9, zipf_V=10_000_000)
    assert abs(datagen.duplicate_ratio(x) - 0.72) <= 0.08


def test_twodups_ratio_survey_appendix():
    """TwoDups dup ratio at n = 10^6 is 0.9219 (number theoretic)."""
    assert abs(datagen.duplicate_ratio(datagen.generate_host("twodups", 1_000_000, 1)) - 0.9219) < 1e-4


def test_continuous_families_no_duplicates_and_determinism():
    for d in ("uniform01", "normal", "lognormal", "exponential", "mixgauss", "chisq4", "uniform_u64"):
        a = datagen.generate_host(d, 200_000, 3)
        assert datagen.duplicate_ratio(a) < 0.001
        assert np.array_equal(a.view(np.uint64), datagen.generate_host(d, 200_000, 3).view(np.uint64))
        if a.dtype == np.float64:
            assert not np.any(np.isnan(a))
            assert not np.any(np.signbit(a) & (a == 0))  # no -0.0
    # slices are position-addressed
    p = datagen.Plan("normal", 1000, 9)
    assert np.array_equal(p.host(100, 50), p.host()[100:150])


def test_distribution_moments():
    n = 400_000
    x = datagen.generate_host("normal", n, 0)
    assert abs(x.mean()) < 0.01 and abs(x.std() - 1) < 0.01
    x = datagen.generate_host("lognormal", n, 0)
    assert abs(np.log(x).std() - 0.5) < 0.01
    x = datagen.generate_host("exponential", n, 0)
    assert abs(x.mean() - 0.5) < 0.01 and x.min() >= 0
    x = datagen.generate_host("chisq4", n, 0)
    assert abs(x.mean() - 4) < 0.05
    x = datagen.generate_host("uniform01", n, 0)
    assert x.min() >= 0 and x.max() < 1 and abs(x.mean() - 0.5) < 0.01
    pl = datagen.Plan("mixgauss", n, 0)
    mu, sig = pl.mix_params()
    assert all(-100 <= m <= 100 for m in mu) and all(1 <= s <= 10 for s in sig)
    x = datagen.generate_host("cfg5mix", n, 1000)
    assert np.mean(x >= 1.0) > 0.5 and np.mean(x == 1.0) > 0.02
