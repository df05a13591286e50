"""Pins for the CPU oracle (oracle/ls2_oracle.c) against what the paper and the
mathematics fix -- never against the oracle itself. CPU only.

Pins, and the mistake each one catches:
  * SPEC hand trace of Alg. 1 + Defragment (fragment order, write head, S_F)
  * closed forms of the chord model on linear / gapped / duplicate samples
    (root routing, eCDF targets with ties, chord slope/offset, empty leaves)
  * SPEC arithmetic examples for bucket ids and the counting sort (indices, adj)
  * the plain definition of the result (sort by IEEE totalOrder via numpy) on
    every generator, brute force on all short sequences, fault-injected models
"""
import ctypes as C
import itertools
import json
import os

import numpy as np
import pytest

import datagen
import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")
PMAX = 1.0 - 2.0 ** -52


def gold(name):
    with open(os.path.join(GOLD, name)) as fh:
        return json.load(fh)


def ref_sorted(keys):
    """np.sort on the totalOrder key: a library routine, independent of the oracle."""
    u = keys.view(np.uint64)
    if keys.dtype == np.float64:
        o = np.where(u >> np.uint64(63) == 1, ~u, u | np.uint64(1 << 63))
    else:
        o = u
    return keys[np.argsort(o, kind="stable")]


def exact_model(a=1.0, lo=0.0, hi=PMAX, xmin=0.0, xmax=1.0):
    """A one-leaf model p(x) = clamp(a*x, lo, hi) for arithmetic pins."""
    m = O.Model()
    m.leaf_count = 1
    m.n_sample = 1
    m.xmin, m.xmax, m.root_scale = xmin, xmax, 0.0
    m.leaf[0].a, m.leaf[0].c, m.leaf[0].b = a, 0.0, 0.0
    m.leaf[0].lo, m.leaf[0].hi = lo, hi
    return m


# ---------------------------------------------------------------- Alg. 1 ----

def test_alg1_hand_trace():
    g = gold("alg1_hand_trace.json")
    a = np.array(g["input"], dtype=np.float64)
    m = O.train(a, stride=g["sample_stride"], leaf_count=g["leaf_count"])
    np.testing.assert_array_equal(O.predict(m, a), np.array(g["p"]))
    L = O.lib()
    b0 = [L.lso_bucket_l0(p, g["fanout"]) for p in O.predict(m, a)]
    assert b0 == g["b0"]
    A = a.copy()
    u = A.view(np.uint64)
    SB = np.zeros(g["fanout"], np.uint64)
    SF = (O.Frag * 16)()
    nf = L.lso_partition(u.ctypes.data, len(A), C.byref(m), O.F64, 0, 0, g["fanout"],
                         g["frag_capacity"], SB.ctypes.data, C.addressof(SF))
    assert A.tolist() == g["after_partition"]
    assert SB.tolist() == g["S_B"]
    assert [[SF[i].bucket, SF[i].size] for i in range(nf)] == g["S_F"]
    scratch = np.zeros(len(A), np.uint64)
    assert L.lso_defragment(u.ctypes.data, len(A), g["fanout"], SB.ctypes.data,
                            C.addressof(SF), nf, scratch.ctypes.data) == O.OK
    assert A.tolist() == g["after_defragment"]


def test_defragment_rejects_corrupt_state():
    """inconsistent S_B / S_F -> 'corrupt partition state'."""
    L = O.lib()
    A = np.arange(4, dtype=np.uint64)
    SB = np.array([2, 2], np.uint64)
    SF = (O.Frag * 2)()
    SF[0].bucket, SF[0].size = 0, 3
    SF[1].bucket, SF[1].size = 1, 1
    assert L.lso_defragment(A.ctypes.data, 4, 2, SB.ctypes.data, C.addressof(SF), 2,
                            np.zeros(4, np.uint64).ctypes.data) == O.E_INTERNAL


def test_partition_all_equal_one_bucket():
    """all-equal keys -> one non-empty bucket, multiset unchanged."""
    a = np.full(1000, 7.25)
    m = O.train(a, stride=1, leaf_count=1000)
    A = a.copy()
    SB = np.zeros(10, np.uint64)
    SF = (O.Frag * 200)()
    nf = O.lib().lso_partition(A.view(np.uint64).ctypes.data, 1000, C.byref(m), O.F64, 0, 0, 10,
                               100, SB.ctypes.data, C.addressof(SF))
    assert nf == 10 and SB[0] == 1000 and SB.sum() == 1000
    assert np.array_equal(A, a)


def test_quasi_sortedness_after_level0():
    """after level-0 partition + defragment, max(bucket b) <=
    min(bucket b+1), and every key re-predicts to its bucket."""
    for dist in ("normal", "lognormal", "zipf", "telemetry", "twodups"):
        a = datagen.generate_host(dist, 200_000, 3)
        m = O.train(a)
        A = a.copy()
        u = A.view(np.uint64)
        f = 1000
        SB = np.zeros(f, np.uint64)
        SF = (O.Frag * (len(A) // 100 + f + 1))()
        L = O.lib()
        nf = L.lso_partition(u.ctypes.data, len(A), C.byref(m), O.dtype_code(a), 0, 0, f, 100,
                             SB.ctypes.data, C.addressof(SF))
        assert L.lso_defragment(u.ctypes.data, len(A), f, SB.ctypes.data, C.addressof(SF), nf,
                                np.zeros(len(A), np.uint64).ctypes.data) == O.OK
        o = O.ord_key(A)
        starts = np.concatenate([[0], np.cumsum(SB)]).astype(np.int64)
        prev_max = None
        for b in range(f):
            s, e = starts[b], starts[b + 1]
            if e == s:
                continue
            if prev_max is not None:
                assert prev_max <= o[s:e].min()
            prev_max = o[s:e].max()
        p = O.predict(m, A[:: 997])
        b0 = np.minimum((p * 1000).astype(np.int64), 999)
        owner = np.searchsorted(starts, np.arange(len(A))[:: 997], side="right") - 1
        assert np.array_equal(b0, owner)


# ----------------------------------------------------------------- model ----

def test_chord_linear_sample_closed_form():
    """Sample 0..9999 (stride 1), L = 10: the sample eCDF is y = x/10^4 at every
    key, so the chord interpolant is p(x) = x/10^4 below the last leaf's first
    key; in the last leaf it runs to (xmax, PMAX)."""
    keys = np.arange(10_000, dtype=np.float64)
    m = O.train(keys, stride=1, leaf_count=10)
    assert m.xmin == 0.0 and m.xmax == 9999.0 and m.root_scale == 10 / 9999
    k = np.arange(9000, dtype=np.float64)
    assert np.max(np.abs(O.predict(m, k) - k / 10_000)) < 1e-15
    # between keys: leaf l = floor(x*10/9999) starts at its first key
    # c_l = ceil(l*999.9); below c_l the line is clamped at lo = c_l/10^4
    x = np.linspace(0, 8999, 5001)
    c = np.ceil(np.floor(x * 10 / 9999) * 999.9)
    expect = np.where(x >= c, x, c) / 10_000
    assert np.max(np.abs(O.predict(m, x) - expect)) < 1e-15
    lv = m.leaves()
    x9 = lv[9, 1]  # first key of the last leaf
    assert x9 == np.ceil(9 * 9999 / 10)
    xs = np.linspace(x9, 9999, 101)
    expect = x9 / 10_000 + (PMAX - x9 / 10_000) * (xs - x9) / (9999 - x9)
    assert np.max(np.abs(O.predict(m, xs) - expect)) < 1e-15
    assert np.all(np.diff(O.predict(m, np.linspace(-5, 2e4, 20001))) >= 0)


def test_chord_gap_sample_empty_leaves():
    """Sample {0..99} u {900..999}, L = 10: leaves 1..8 are empty and predict the
    next knot's eCDF (1/2); leaf 0's chord runs to the next leaf's first key."""
    keys = np.concatenate([np.arange(100), np.arange(900, 1000)]).astype(np.float64)
    m = O.train(keys, stride=1, leaf_count=10)
    assert O.predict(m, np.array([500.0]))[0] == 0.5
    assert O.predict(m, np.array([120.0]))[0] == 0.5
    x = np.arange(0, 100, 0.5)
    assert np.max(np.abs(O.predict(m, x) - 0.5 * x / 900)) < 1e-15
    xs = np.arange(900, 999.5, 0.5)
    expect = 0.5 + (PMAX - 0.5) * (xs - 900) / 99
    assert np.max(np.abs(O.predict(m, xs) - expect)) < 1e-15


def test_chord_duplicate_sample_strict_ecdf():
    """Ties: the model "returns the count of keys in the input that are less than
    x". Values 0..499 with multiplicities 1..500 (stride 1, L = 1000):
    every value sits alone at the head of its leaf, so p(v) = #{keys < v}/m exactly."""
    vals = np.arange(500)
    mult = np.arange(1, 501)
    keys = np.repeat(vals, mult).astype(np.uint64)
    np.random.default_rng(1).shuffle(keys)
    m = O.train(keys, stride=1, leaf_count=1000)
    mtot = len(keys)
    less = np.concatenate([[0], np.cumsum(mult)[:-1]])
    np.testing.assert_array_equal(O.predict(m, vals.astype(np.uint64)), less / mtot)


def test_spec_model_examples():
    # 1000 evenly spaced keys, 4 leaves -> |p(x) - x/1000| <= 0.01
    keys = np.arange(1000, dtype=np.float64)
    m = O.train(keys, stride=1, leaf_count=4)
    x = np.linspace(0, 999, 4000)
    assert np.max(np.abs(O.predict(m, x) - x / 1000)) <= 0.01
    # all-equal sample -> predicts 0 (degenerate model)
    m = O.train(np.full(4, 7.0), stride=1, leaf_count=1000)
    assert m.degenerate == 1 and O.predict(m, np.array([7.0, -3.0, 1e9])).tolist() == [0, 0, 0]
    # 10^4 N(0,1) keys, 1000 leaves -> mean |p - sample eCDF| < 0.005
    s = np.random.default_rng(0).standard_normal(10_000)
    m = O.train(s, stride=1, leaf_count=1000)
    ecdf = np.searchsorted(np.sort(s), s, side="left") / len(s)
    assert np.mean(np.abs(O.predict(m, s) - ecdf)) < 0.005
    # below the minimum -> 0; above the maximum -> < 1
    assert O.predict(m, np.array([-1e300]))[0] == 0.0
    assert O.predict(m, np.array([1e300]))[0] < 1.0
    assert O.predict(m, np.array([np.inf]))[0] == O.predict(m, np.array([s.max()]))[0]


@pytest.mark.parametrize("n", [1_000_000, 10_000_000])
def test_sorted_input_bucket_counts(n):
    """SURVEY §8(c) chord-leaf pin: A[i] = i, n = 100·m, stride 100. The sample
    eCDF is exactly linear, so at every sampled key below the last leaf
    p(100k) = 100k/n. Exact level-0 counts: bucket 999 = n/f + 99 (the 99 keys
    above the last sample key clamp to PMAX), bucket 998 = n/f, buckets 0..997
    hold n/f or n/f - 1 keys (a boundary key may round down one bucket), and
    sum S_B = n (so exactly 99 of them hold n/f - 1); b0 is non-decreasing and
    key i lies in bucket floor(i·f/n) or, when its p rounds up across the
    boundary, the one above it."""
    f = 1000
    q = n // f
    a = np.arange(n, dtype=np.float64)
    m = O.train(a)
    idx = np.arange(0, (n * 999) // 1000 - 100, 100)  # (below the last leaf)
    assert np.max(np.abs(O.predict(m, a[idx]) - idx / n)) < 1e-15
    _, _, _, d = O.sort(a, dumps=True)
    b0 = d["b0"].astype(np.int64)
    assert np.all(np.diff(b0) >= 0)
    S = d["S_B"].astype(np.int64)
    assert S.sum() == n and np.array_equal(np.bincount(b0, minlength=f), S)
    assert S[999] == q + 99 and S[998] == q
    assert set(np.unique(S[:998]).tolist()) <= {q - 1, q}
    assert int(np.sum(S[:998] == q - 1)) == 99
    i = np.arange((n * 998) // 1000, dtype=np.int64)
    ideal = (i * f) // n
    assert np.all((b0[i] == ideal) | (b0[i] == ideal + 1))


# -------------------------------------------------------- ids / counting ----

def test_bucket_index_examples():
    g = gold("spec_examples.json")
    L = O.lib()
    for c in g["bucket_index"]["cases"]:
        got = (L.lso_bucket_l0(c["p"], c["f"]) if c["level"] == 0
               else L.lso_bucket_l1(c["p"], c["f"], c["parent"]))
        assert got == c["expect"], c
    c = g["bucket_clamp"]
    assert L.lso_bucket_l0(c["p"], c["f"]) == c["b0"]
    assert L.lso_bucket_l1(c["p"], c["f"], c["b0"]) == c["b1"]
    assert L.lso_bucket_l0(PMAX, 1000) == 999 and L.lso_bucket_l1(PMAX, 1000, 999) == 999


def test_counting_sort_example():
    g = gold("spec_examples.json")["counting_sort"]
    L = O.lib()
    m = exact_model()
    a = np.array(g["input"])
    pos = [L.lso_cs_pos(x, g["i"], g["j"], g["f"], g["n_total"], len(a)) for x in a]
    assert pos == g["pos"]
    u = a.copy().view(np.uint64)
    K = np.zeros(3, np.uint64)
    T = np.zeros(3, np.uint64)
    L.lso_counting_sort(u.ctypes.data, 3, C.byref(m), O.F64, g["i"], g["j"], g["f"],
                        g["n_total"], K.ctypes.data, T.ctypes.data)
    assert u.view(np.float64).tolist() == g["expect"]


def test_counting_sort_is_a_permutation_and_groups_ordered():
    """After the counting sort, keys with different pos are in order; only runs of
    equal pos can be out of order (the invariant behind the touch-up, R15)."""
    L = O.lib()
    m = exact_model()
    rng = np.random.default_rng(5)
    a = 0.25 + rng.random(997) * 0.01  # sub-bucket (i, j) = (2, 500) of f = 1000
    u = a.copy().view(np.uint64)
    K = np.zeros(997, np.uint64)
    T = np.zeros(997, np.uint64)
    L.lso_counting_sort(u.ctypes.data, 997, C.byref(m), O.F64, 250, 0, 1000, 100_000,
                        K.ctypes.data, T.ctypes.data)
    out = u.view(np.float64)
    assert np.array_equal(np.sort(out), np.sort(a))
    pos = np.array([L.lso_cs_pos(x, 250, 0, 1000, 100_000, 997) for x in out])
    assert np.all(np.diff(pos.astype(np.int64)) >= 0)


def test_is_homogeneous_and_insertion_sort_examples():
    g = gold("spec_examples.json")
    L = O.lib()
    for keys, expect in g["is_homogeneous"]["cases"]:
        a = np.array(keys, dtype=np.uint64)
        assert bool(L.lso_is_homogeneous(a.ctypes.data, len(a), O.U64)) == expect
    for keys, expect, disp in g["insertion_sort"]["cases"]:
        a = np.array(keys, dtype=np.uint64)
        fired = C.c_int(0)
        shifts = L.lso_insertion_sort(a.ctypes.data, len(a), O.U64, 0, C.byref(fired))
        assert a.tolist() == expect and shifts == disp
    # bit equality under ord: -0.0 and +0.0 are different keys (R11/R12)
    z = np.array([0.0, -0.0])
    assert not L.lso_is_homogeneous(z.ctypes.data, 2, O.F64)


def test_insertion_sort_guard_same_result():
    L = O.lib()
    a = np.random.default_rng(2).integers(0, 1 << 62, 5000).astype(np.uint64)
    b = a.copy()
    fired = C.c_int(0)
    L.lso_insertion_sort(a.ctypes.data, len(a), O.U64, 100, C.byref(fired))
    assert fired.value == 1 and np.array_equal(a, np.sort(b))


# ------------------------------------------------------- whole algorithm ----

def test_two_dups_example():
    g = gold("spec_examples.json")["two_dups_sort"]
    out, _, _, _ = O.sort(np.array(g["input"], dtype=np.uint64))
    assert out.tolist() == g["expect"]


@pytest.mark.parametrize("dist", sorted(datagen.DISTS))
@pytest.mark.parametrize("n", [1000, 100_000])
def test_sort_equals_reference_all_generators(dist, n):
    """output == comparison sort, every generator, 5 seeds."""
    for seed in range(5):
        a = datagen.generate_host(dist, n, seed)
        out, _, st, _ = O.sort(a)
        assert np.array_equal(out.view(np.uint64), ref_sorted(a).view(np.uint64)), (dist, seed)


@pytest.mark.parametrize("dist", ["normal", "exponential", "zipf", "rootdups", "twodups", "telemetry"])
def test_sort_equals_reference_1e6_and_invariants(dist):
    a = datagen.generate_host(dist, 1_000_000, 7)
    out, model, st, d = O.sort(a, dumps=True)
    assert np.array_equal(out.view(np.uint64), ref_sorted(a).view(np.uint64))
    f = 1000
    # S_B / S'_B are the run lengths of b0 / (b0, b1) along the sorted output
    p = O.predict(model, out[:: 1])
    b0 = np.minimum((p * f).astype(np.int64), f - 1)
    b1 = np.clip((p * 1e6).astype(np.int64) - b0 * f, 0, f - 1)
    assert np.array_equal(np.bincount(b0, minlength=f), d["S_B"].astype(np.int64))
    raw = np.bincount(b0 * f + b1, minlength=f * f)
    assert np.array_equal(raw, d["hist1_raw"].astype(np.int64))
    rows = d["H0"].astype(bool)
    s1 = d["S_B1"].reshape(f, f).astype(np.int64)
    assert np.array_equal(s1[~rows], raw.reshape(f, f)[~rows]) and s1[rows].sum() == 0
    # homogeneous flags: H0 bucket <=> all its keys equal
    starts = np.concatenate([[0], np.cumsum(d["S_B"])]).astype(np.int64)
    ou = out.view(np.uint64)
    for b in range(f):
        seg = ou[starts[b]:starts[b + 1]]
        assert bool(d["H0"][b]) == (len(seg) <= 1 or bool(np.all(seg == seg[0])))
    # H1 (Alg. 2, R11): for a bucket that is not homogeneous, sub-bucket
    # (i, j) is flagged exactly when its range of the sorted output holds <= 1
    # key or one value (sorted: first == last); rows of H0 buckets are zero
    H1 = d["H1"].reshape(f, f).astype(bool)
    assert not H1[rows].any()
    sub_end = np.cumsum(raw).astype(np.int64)
    sub_beg = sub_end - raw
    nz = raw > 0
    want = np.ones(f * f, bool)
    first, last = ou[sub_beg[nz]], ou[sub_end[nz] - 1]
    want[nz] = (raw[nz] <= 1) | (first == last)
    want = want.reshape(f, f)
    want[rows] = False
    assert np.array_equal(H1, want)
    assert int(H1.sum()) >= st["h1_subbuckets"]  # (stats count only sub-buckets of >= 2 keys)
    hk = raw.reshape(f, f)[H1 & (raw.reshape(f, f) >= 2)]
    assert st["h1_subbuckets"] == len(hk) and st["h1_keys"] == int(hk.sum())
    if dist == "rootdups":  # S:414 acceptance 7
        assert st["h1_subbuckets"] >= 1


def test_fault_injection_constant_and_foreign_models():
    """a constant model, zero-slope leaves, a model fitted on another
    distribution -- the output is still the sorted permutation."""
    a = datagen.generate_host("lognormal", 50_000, 11)
    want = ref_sorted(a).view(np.uint64)
    const = exact_model(a=0.0, lo=0.3, hi=0.3)
    out, _, st, _ = O.sort(a, model=const)
    assert np.array_equal(out.view(np.uint64), want) and st["guard_fired"] >= 1
    foreign = O.train(datagen.generate_host("normal", 50_000, 1))
    out, _, _, _ = O.sort(a, model=foreign)
    assert np.array_equal(out.view(np.uint64), want)
    flat = O.train(a)
    for l in range(flat.leaf_count):
        flat.leaf[l].a = 0.0
    out, _, _, _ = O.sort(a, model=flat)
    assert np.array_equal(out.view(np.uint64), want)


def _brute(values, length, f, stride, dtype):
    cfg = O.config(fanout=f, leaf_count=1000, sample_stride=stride, frag_capacity=100)
    for seq in itertools.product(values, repeat=length):
        a = np.array(seq, dtype=dtype)
        out, _, _, _ = O.sort(a, cfg=cfg)
        assert np.array_equal(out, np.sort(a)), (seq, f, stride)


@pytest.mark.parametrize("f,stride", [(2, 1), (3, 2)])
def test_brute_force_all_4pow8(f, stride):
    """Every sequence of length 8 over {0,1,2,3} (SURVEY §8(c) pins)."""
    _brute([0, 1, 2, 3], 8, f, stride, np.uint64)


@pytest.mark.parametrize("f", [2, 3, 1000])
@pytest.mark.parametrize("stride", [1, 2, 100])
def test_brute_force_short(f, stride):
    for length in range(0, 6):
        _brute([0.0, 1.5, -2.0, 3.0], length, f, stride, np.float64)


def test_edge_cases():
    # NaN -> E_NAN, input untouched
    a = np.array([3.0, np.nan, 1.0])
    b = a.copy()
    with pytest.raises(O.OracleError) as e:
        O.lib()  # ensure loaded
        u = b.view(np.uint64)
        rc = O.lib().lso_sort(u.ctypes.data, 3, O.F64, None, None, None, None, None)
        raise O.OracleError(rc)
    assert e.value.rc == O.E_NAN and np.array_equal(b.view(np.uint64), a.view(np.uint64))
    # 0 / 1 elements -> no-op
    for a in (np.array([], np.float64), np.array([4.0])):
        out, _, _, _ = O.sort(a)
        assert np.array_equal(out, a)
    # infinities, denormals, signed zero, extreme u64 and fp64-colliding u64 keys
    cases = [
        np.array([np.inf, -np.inf, 1.0, -1.0, 0.0, 5e-324, -5e-324, 1e308, -1e308] * 30),
        np.array([-0.0, 0.0] * 50 + [1.0]),
        np.array([np.inf] * 20 + [-np.inf] * 20),
        np.array([2 ** 64 - 1, 2 ** 64 - 2, 0, 1, 2 ** 63] * 40, dtype=np.uint64),
        np.array([2 ** 60 + k for k in range(300)][::-1], dtype=np.uint64),
        np.array([2 ** 53 + k for k in range(0, 400, 3)] * 3, dtype=np.uint64),
    ]
    for a in cases:
        for stride in (1, 100):
            out, _, _, _ = O.sort(a, cfg=O.config(sample_stride=stride))
            assert np.array_equal(out.view(np.uint64), ref_sorted(a).view(np.uint64))
    for n in (2, 3, 99, 100, 101, 8191, 8192, 8193):
        a = datagen.generate_host("normal", n, n)
        out, _, _, _ = O.sort(a)
        assert np.array_equal(out, np.sort(a))
        r = np.sort(a)[::-1].copy()
        out, _, _, _ = O.sort(r)
        assert np.array_equal(out, np.sort(a))


def test_host_sort_baselines_equal_reference():
    """bench.py's CPU context baselines (oracle/host_sorts.cpp: std::sort(≺)
    on one core, __gnu_parallel::sort(≺) on all cores) give the plain
    definition of the result, including -0.0 before +0.0 and ±inf."""
    rng = np.random.default_rng(3)
    a = rng.standard_normal(200_000)
    a[:6] = [-0.0, 0.0, np.inf, -np.inf, 5e-324, -5e-324]
    rng.shuffle(a)
    want = ref_sorted(a).view(np.uint64)
    assert np.array_equal(O.std_sort(a).view(np.uint64), want)
    p, threads = O.parallel_sort(a)
    assert np.array_equal(p.view(np.uint64), want) and threads >= 1
    u = rng.integers(0, 2 ** 64 - 1, 100_000, dtype=np.uint64)
    assert np.array_equal(O.std_sort(u), np.sort(u))
    assert np.array_equal(O.parallel_sort(u)[0], np.sort(u))
