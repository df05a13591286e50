"""Pins for the LearnedSort 1.0 oracle variant (oracle/ls1_oracle.c, SURVEY
§8(f) f4: context only). CPU only.

  * hand trace of the fixed-capacity partition with its spill bucket
    (tests/golden/ls1_hand_trace.json, P:49/P:58/P:263)
  * the exception table: an all-equal input never reaches the buckets;
    a value that repeats in the sample is counted, not partitioned
  * the level-0 spill equals the overflow counted by brute force over the
    bucket ids of the LS 2.0 oracle's routines; capacities that can hold
    every key leave the spill bucket empty
  * the result is the plain definition (numpy sort on totalOrder) on every
    generator and on brute-force short sequences
"""
import itertools
import json
import os

import numpy as np
import pytest

import datagen
import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def ref_sorted(keys):
    u = keys.view(np.uint64)
    if keys.dtype == np.float64:
        o = np.where(u >> np.uint64(63) == 1, ~u, u | np.uint64(1 << 63))
    else:
        o = u
    return keys[np.argsort(o, kind="stable")]


def test_ls1_hand_trace():
    g = json.load(open(os.path.join(GOLD, "ls1_hand_trace.json")))
    keys = np.array(g["input"], dtype=np.uint64)
    cfg = O.ls1_config(fanout=g["fanout"], leaf_count=g["leaf_count"],
                       sample_stride=g["sample_stride"], cap0=g["cap0"], cap1=g["cap1"],
                       exc_min=g["exc_min"])
    out, st = O.ls1_sort(keys, cfg)
    assert out.tolist() == g["output"]
    assert st["spill_l0"] == g["spill_l0"]
    assert st["spill_keys"] == g["spill_keys"]
    assert st["exception_values"] == g["exception_values"]


def test_ls1_all_equal_goes_through_the_exception_table():
    keys = np.full(10_000, 77, dtype=np.uint64)
    out, st = O.ls1_sort(keys)
    assert (out == 77).all()
    assert st["exception_values"] == 1 and st["exception_keys"] == 10_000
    assert st["spill_keys"] == 0


def test_ls1_problematic_value_counted_not_partitioned():
    rng = np.random.default_rng(3)
    n = 200_000
    keys = rng.random(n)
    heavy = rng.random(n) < 0.30          # 30 % copies of one value: ~600 of a 2000-key sample
    keys[heavy] = 0.25
    out, st = O.ls1_sort(keys)
    assert np.array_equal(out.view(np.uint64), ref_sorted(keys).view(np.uint64))
    assert st["exception_values"] == 1
    assert st["exception_keys"] == int(heavy.sum())


def test_ls1_spill_counts_by_brute_force():
    """Level-0 spill = sum over buckets of max(0, count - cap0), counted from
    the bucket ids of the LS 2.0 oracle's routines (no exception keys)."""
    keys = datagen.generate_host("normal", 50_000, 5)
    f, cap0 = 100, 400                   # expected 500 per bucket: most overflow
    cfg = O.ls1_config(fanout=f, leaf_count=100, cap0=cap0, cap1=10_000, exc_min=10**9)
    out, st = O.ls1_sort(keys, cfg)
    m = O.train(keys, 100, 100)
    L = O.lib()
    b0 = np.array([L.lso_bucket_l0(p, f) for p in O.predict(m, keys)])
    cnt = np.bincount(b0, minlength=f)
    assert st["spill_l0"] == int(np.maximum(cnt - cap0, 0).sum())
    assert st["spill_keys"] == st["spill_l0"]          # cap1 never reached
    assert np.array_equal(out.view(np.uint64), ref_sorted(keys).view(np.uint64))


def test_ls1_no_spill_with_room():
    keys = datagen.generate_host("uniform01", 100_000, 2)
    n = len(keys)                       # every bucket can hold every key
    out, st = O.ls1_sort(keys, O.ls1_config(fanout=10, leaf_count=100, cap0=n, cap1=n))
    assert st["spill_keys"] == 0 and st["exception_values"] == 0
    assert np.array_equal(out.view(np.uint64), ref_sorted(keys).view(np.uint64))


@pytest.mark.parametrize("dist", ["uniform01", "normal", "lognormal", "exponential", "mixgauss",
                                  "zipf", "rootdups", "twodups", "telemetry", "cfg5mix", "uniform_u64", "chisq4"])
def test_ls1_sorts_every_generator(dist):
    keys = datagen.generate_host(dist, 300_000, 1)
    out, st = O.ls1_sort(keys)
    assert np.array_equal(out.view(np.uint64), ref_sorted(keys).view(np.uint64))


def test_ls1_brute_force_short_sequences():
    cfg = O.ls1_config(fanout=2, leaf_count=4, sample_stride=1, cap0=2, cap1=1)
    for n in range(0, 7):
        for seq in itertools.product([0, 1, 2, 3], repeat=n) if n <= 5 else [tuple(range(6))]:
            keys = np.array(seq, dtype=np.uint64)
            out, _ = O.ls1_sort(keys, cfg)
            assert out.tolist() == sorted(seq)


def test_ls1_rejects_nan():
    keys = np.array([1.0, np.nan, 0.5])
    with pytest.raises(O.OracleError):
        O.ls1_sort(keys)
