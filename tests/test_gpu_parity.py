"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bar (north_star): sorted output bit-exact; with identical model parameters,
p / b0 / b1 / pos / S_B / S'_B / H0 / H1 bit-exact; independently fitted RMI
parameters bit-identical (the chord fit has no floating-point reductions, so
the 1e-9 relative allowance is not needed). Inputs are generated on the device
and the same bytes are handed to the oracle.
"""
import ctypes as C

import numpy as np
import pytest

import datagen
import oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2107_03290_b200 as ls  # noqa: E402

DEV = torch.device("cuda:0")
DISTS_F64 = ["uniform01", "normal", "lognormal", "exponential", "mixgauss", "chisq4"]
DISTS_U64 = ["zipf", "rootdups", "twodups", "telemetry", "uniform_u64"]


def gen(dist, n, seed):
    plan = datagen.Plan(dist, n, seed)
    t = torch.empty(n, dtype=torch.float64 if plan.dtype == np.float64 else torch.uint64, device=DEV)
    if n:
        plan.device(t)
    torch.cuda.synchronize()
    return t


def to_np(t):
    a = t.view(torch.int64).cpu().numpy().view(np.uint64)
    return a.view(np.float64) if t.dtype == torch.float64 else a


def from_np(a):
    t = torch.from_numpy(a.view(np.int64).copy()).to(DEV)
    return t.view(torch.float64) if a.dtype == np.float64 else t.view(torch.uint64)


def bits(x):
    return np.ascontiguousarray(x).view(np.uint64)


def oracle_model_to_ls(m: O.Model) -> ls.Model:
    out = ls.Model()
    out.leaf_count, out.n_sample, out.degenerate = m.leaf_count, m.n_sample, m.degenerate
    out.xmin, out.xmax, out.root_scale = m.xmin, m.xmax, m.root_scale
    C.memmove(C.addressof(out.leaf), C.addressof(m.leaf), 40 * m.leaf_count)
    return out


def ls_leaves(m: ls.Model) -> np.ndarray:
    arr = np.ctypeslib.as_array(m.leaf).view(np.float64).reshape(-1, 5)
    return arr[: m.leaf_count].copy()


def assert_models_identical(g: ls.Model, o: O.Model):
    assert g.leaf_count == o.leaf_count and g.degenerate == o.degenerate
    assert g.n_sample == o.n_sample
    for k in ("xmin", "xmax", "root_scale"):
        assert bits(np.float64(getattr(g, k))) == bits(np.float64(getattr(o, k))), k
    assert np.array_equal(bits(ls_leaves(g)), bits(o.leaves()))


def dumps_for(f):
    d = dict(S_B=torch.zeros(f, dtype=torch.int64, device=DEV),
             S_B1=torch.zeros(f * f, dtype=torch.int32, device=DEV),
             H0=torch.zeros(f, dtype=torch.uint8, device=DEV),
             H1=torch.zeros(f * f, dtype=torch.uint8, device=DEV))
    model = ls.Model()
    dd = ls.Dumps(d["S_B"].data_ptr(), d["S_B1"].data_ptr(), d["H0"].data_ptr(),
                  d["H1"].data_ptr(), C.pointer(model))
    return d, dd, model


# ------------------------------------------------------------------ model ---

@pytest.mark.parametrize("dist", DISTS_F64 + DISTS_U64)
def test_train_rmi_bit_identical(dist):
    keys = gen(dist, 1_000_000, 3)
    sample = keys[::100].contiguous()
    g = ls.ls_train_rmi(sample)
    o = O.train(to_np(sample), stride=1)
    assert_models_identical(g, o)
    # the fit inside ls_sort (strided sample of the whole input) == oracle's O1-O5
    d, dd, model = dumps_for(1000)
    ls.ls_sort(keys.clone(), dumps=dd)
    assert_models_identical(model, O.train(to_np(keys)))


# -------------------------------------------------------- ids / histograms --

@pytest.mark.parametrize("dist", ["normal", "exponential", "mixgauss", "zipf", "twodups", "telemetry"])
def test_bucket_ids_bit_exact(dist):
    keys = gen(dist, 1_000_000, 5)
    h = to_np(keys)
    _, om, _, od = O.sort(h, dumps=True)
    out = ls.ls_bucket_ids(keys, oracle_model_to_ls(om))
    assert np.array_equal(bits(out["p"].cpu().numpy()), bits(od["p"]))
    for k in ("b0", "b1", "pos"):
        assert np.array_equal(out[k].cpu().numpy().astype(np.uint32), od[k]), k
    assert np.array_equal(out["hist1"].cpu().numpy().astype(np.uint64), od["hist1_raw"])
    assert np.array_equal(out["hist0"].cpu().numpy().astype(np.uint64), od["S_B"])


# ------------------------------------------------------------- whole sort ---

def check_sort(keys, cfg=None, model=None, ocfg=None, f=1000):
    h = to_np(keys)
    osorted, om, ost, od = O.sort(h, cfg=ocfg, dumps=True,
                                  model=None if model is None else model)
    d, dd, gm = dumps_for(f)
    t = keys.clone()
    st = ls.ls_sort(t, cfg=cfg, dumps=dd,
                    model=None if model is None else oracle_model_to_ls(model))
    got = to_np(t)
    assert np.array_equal(bits(got), bits(osorted)), "sorted output differs from the oracle"
    assert np.array_equal(d["S_B"].cpu().numpy().astype(np.uint64), od["S_B"])
    assert np.array_equal(d["H0"].cpu().numpy(), od["H0"])
    assert np.array_equal(d["S_B1"].cpu().numpy().astype(np.uint64), od["S_B1"])
    assert np.array_equal(d["H1"].cpu().numpy(), od["H1"])
    assert st["h0_buckets"] == ost["h0_buckets"] and st["h0_keys"] == ost["h0_keys"]
    assert st["h1_subbuckets"] == ost["h1_subbuckets"] and st["h1_keys"] == ost["h1_keys"]
    return st, ost


@pytest.mark.parametrize("dist", DISTS_F64 + DISTS_U64)
def test_sort_bit_exact_1e6(dist):
    st, ost = check_sort(gen(dist, 1_000_000, 7))
    assert st["small_keys"] + st["big_keys"] + st["h1_keys"] + st["h0_keys"] <= 1_000_000


@pytest.mark.parametrize("dist", ["normal", "lognormal", "zipf", "rootdups", "twodups", "telemetry",
                                  "cfg5mix"])
def test_sort_bit_exact_1e7(dist):
    """(cfg5mix: the Zipf head packs hundreds of b0 thresholds into a few grid
    cells, so the refined sub-grids of the b0 search are in use; S_B parity
    checks every key's b0.)"""
    check_sort(gen(dist, 10_000_000, 11))


@pytest.mark.parametrize("dist,seed", [("twodups", 13), ("twodups", 5), ("zipf", 13), ("zipf", 5)])
def test_sort_bit_exact_3e6_dups(dist, seed):
    """Regression: at 3M duplicate-heavy keys the warp sort meets several
    all-equal collision groups > 8 keys in one sub-bucket (skipping one must
    not end the sub-bucket's touch-up)."""
    check_sort(gen(dist, 3_000_000, seed))


# ------------------------------------------ cluster-resident round 1 (f2) --

FUSED = dict(flags=ls.LS_FLAG_FUSED_ROUND1)


@pytest.mark.parametrize("dist", ["normal", "uniform01", "mixgauss", "zipf", "rootdups", "twodups",
                                  "telemetry"])
def test_fused_round1_bit_exact(dist, monkeypatch):
    """SURVEY §8(f) f2 (LS_FLAG_FUSED_ROUND1): level-0 buckets partitioned by
    one 8-CTA cluster each (forced down to small buckets with LS_FR_MIN;
    Zipf's and config 4's largest buckets exceed the cluster and take the
    separate path in the same call) give the oracle's output, S_B, S'_B, H0
    and H1, as the default separate count/scatter path does."""
    monkeypatch.setenv("LS_FR_MIN", "256")
    keys = gen(dist, 3_000_000, 13)
    st, _ = check_sort(keys, cfg=ls.config(**FUSED))
    assert st["fused_buckets"] > 0
    st2, _ = check_sort(keys)
    assert st2["fused_buckets"] == 0
    # P5 (the in-bucket sort inside k_round1) accounts for the same sub-buckets
    for k in ("small_subbuckets", "small_keys", "h1_subbuckets", "h1_keys", "big_keys"):
        assert st[k] == st2[k], k


def test_fused_round1_default_threshold():
    """At 70M keys the level-0 buckets (~70K keys) take the cluster path, and
    their ~70-key sub-buckets are sorted inside it (P5)."""
    st, _ = check_sort(gen("normal", 70_000_000, 17), cfg=ls.config(**FUSED))
    assert st["fused_buckets"] >= 990
    assert st["small_keys"] > 60_000_000


@pytest.mark.parametrize("n", [0, 1, 2, 3, 31, 99, 100, 101, 2047, 2048, 2049, 4097, 8191, 8192,
                               8193, 65535, 65536, 65537, 131073, 300_001])
def test_sort_sizes(n):
    for dist in ("normal", "twodups"):
        keys = gen(dist, n, n)
        h = to_np(keys)
        t = keys.clone()
        ls.ls_sort(t)
        want = O.sort(h)[0] if n else h
        assert np.array_equal(bits(to_np(t)), bits(want))


EDGE = {
    "inf_denormal_zero": np.array([np.inf, -np.inf, 1.0, -1.0, 0.0, 5e-324, -5e-324, 1e308,
                                   -1e308, 2.5] * 3000),
    "signed_zero": np.array([-0.0, 0.0] * 5000 + [1.0]),
    "all_inf": np.array([np.inf] * 500 + [-np.inf] * 500),
    "all_equal": np.full(100_000, 3.25),
    "two_values": np.array([1.0, 2.0] * 60_000),
    "sorted": np.arange(200_000, dtype=np.float64),
    "reverse": np.arange(200_000, dtype=np.float64)[::-1].copy(),
    "u64_extremes": np.array([2 ** 64 - 1, 2 ** 64 - 2, 0, 1, 2 ** 63] * 4000, dtype=np.uint64),
    "u64_fp64_collisions": np.array([2 ** 60 + k for k in range(50_000)][::-1], dtype=np.uint64),
    "u64_collide_dups": np.array([2 ** 53 + k for k in range(0, 30_000, 3)] * 7, dtype=np.uint64),
    "huge_range": np.array([-1.7e308, 1.7e308, 0.0, 1.0] * 10_000),
}


@pytest.mark.parametrize("name", sorted(EDGE))
def test_sort_edge_cases(name):
    a = EDGE[name].copy()
    np.random.default_rng(0).shuffle(a)
    for stride in (1, 100):
        cfg = ls.config(sample_stride=stride)
        ocfg = O.config(sample_stride=stride)
        keys = from_np(a)
        h = to_np(keys)
        t = keys.clone()
        ls.ls_sort(t, cfg=cfg)
        assert np.array_equal(bits(to_np(t)), bits(O.sort(h, cfg=ocfg)[0]))


@pytest.mark.parametrize("dist,n,seed,kw", [
    ("telemetry", 235_725, 439_674_140, dict(big_threshold=64)),
    ("chisq4", 1_179_994, 516_369_813, dict(fanout=100, big_threshold=100)),
    ("twodups", 992_914, 52_170_342, dict(fanout=100, big_threshold=64)),
])
def test_many_big_items(dist, n, seed, kw):
    """Regressions from scripts/stress.py: with a small big threshold more
    than n/257 sub-buckets become big items; the item lists are sized from the
    threshold (n / (T + 1)), so no capacity error and the oracle's output."""
    cfg = ls.config(**kw)
    ocfg = O.config(fanout=kw.get("fanout", 1000))
    check_sort(gen(dist, n, seed), cfg=cfg, ocfg=ocfg, f=kw.get("fanout", 1000))


def test_misaligned_keys_rejected():
    """Keys at an odd 8-byte offset (a tensor slice) are rejected before any
    work, as include/ls.h states: the TMA stages address aligned key pairs."""
    keys = gen("normal", 10_001, 5)
    view = keys[1:]
    before = to_np(view).copy()
    with pytest.raises(ls.LSError) as e:
        ls.ls_sort(view)
    assert e.value.status == ls.LS_E_INVALID
    assert np.array_equal(bits(to_np(view)), bits(before))


def test_nan_rejected_input_untouched():
    a = np.random.default_rng(1).standard_normal(100_000)
    a[54_321] = np.nan
    t = from_np(a)
    with pytest.raises(ls.LSError) as e:
        ls.ls_sort(t)
    assert e.value.status == ls.LS_E_NAN
    assert np.array_equal(bits(to_np(t)), bits(a))


def test_fault_injection_models():
    """constant model / zero slopes / foreign model still sort exactly."""
    keys = gen("lognormal", 300_000, 13)
    h = to_np(keys)
    const = O.Model()
    const.leaf_count, const.n_sample = 1, 1
    const.leaf[0].a, const.leaf[0].b, const.leaf[0].lo, const.leaf[0].hi = 0.0, 0.3, 0.3, 0.3
    foreign = O.train(datagen.generate_host("normal", 300_000, 1))
    flat = O.train(h)
    for l in range(flat.leaf_count):
        flat.leaf[l].a = 0.0
    for m in (const, foreign, flat):
        check_sort(keys, model=m)


def test_injected_model_validation():
    keys = gen("normal", 10_000, 1)
    m = oracle_model_to_ls(O.train(to_np(keys)))
    m.leaf[3].a = -1.0
    with pytest.raises(ls.LSError) as e:
        ls.ls_sort(keys.clone(), model=m)
    assert e.value.status == ls.LS_E_INVALID


@pytest.mark.parametrize("f,L,stride,n", [(2, 1000, 1, 5000), (3, 7, 2, 20_000), (10, 50, 5, 100_000),
                                          (64, 1000, 100, 500_000), (1024, 1024, 100, 2_000_000)])
def test_other_fanouts(f, L, stride, n):
    keys = gen("exponential", n, f)
    check_sort(keys, cfg=ls.config(fanout=f, leaf_count=L, sample_stride=stride),
               ocfg=O.config(fanout=f, leaf_count=L, sample_stride=stride), f=f)


@pytest.mark.parametrize("thr", [64, 512, 1024, 4096])
def test_big_threshold(thr):
    """Small thresholds push sub-buckets through the exact big path."""
    for dist in ("telemetry", "normal"):
        keys = gen(dist, 1_000_000, 17)
        h = to_np(keys)
        t = keys.clone()
        st = ls.ls_sort(t, cfg=ls.config(big_threshold=thr))
        assert np.array_equal(bits(to_np(t)), bits(O.sort(h)[0]))
        if thr == 64:
            assert st["big_subbuckets"] > 0


def test_sort_host_end_to_end():
    keys = gen("mixgauss", 2_000_000, 23)
    h = to_np(keys)
    host = torch.from_numpy(h.copy()).pin_memory()
    buf = torch.empty_like(keys)
    ls.ls_sort_host(host, buf)
    assert np.array_equal(bits(host.numpy()), bits(np.sort(h)))


def test_determinism():
    keys = gen("twodups", 3_000_000, 29)
    outs = []
    for _ in range(2):
        d, dd, _ = dumps_for(1000)
        t = keys.clone()
        ls.ls_sort(t, dumps=dd)
        outs.append((to_np(t), {k: v.cpu().numpy() for k, v in d.items()}))
    assert np.array_equal(bits(outs[0][0]), bits(outs[1][0]))
    for k in outs[0][1]:
        assert np.array_equal(outs[0][1][k], outs[1][1][k])


# --------------------------------------------------------- full size (200M) -

@pytest.mark.slow
@pytest.mark.parametrize("dist", ["normal", "zipf", "telemetry", "twodups", "lognormal", "exponential",
                                  "mixgauss", "rootdups", "uniform01", "uniform_u64"])
def test_full_size_200m(dist):
    """BASELINE configs 2-4 and both reference rows (every 200M line bench.py
    reports) at full size, in the bench launch configuration
    (same workspace, same default config, CUDA Graph replay on the second
    call): the sorted output equals the oracle's (Alg. 2 run on the same 200M
    bytes) element by element, and so do S_B, S'_B, H0, H1 and the
    homogeneous-class counts; the fitted model is bit-identical; p and b0 on
    10^5 sampled keys are bit-exact against the oracle's predict."""
    n = 200_000_000
    keys = gen(dist, n, 0 if dist != "zipf" else 1)
    h = to_np(keys)
    d, dd, gm = dumps_for(1000)
    t = keys.clone()
    cfg = ls.config(flags=ls.LS_FLAG_PHASE_TIMING)  # (bench.py's config)
    ws = ls.workspace(n, ls.dtype_code(t), cfg)
    ls.ls_sort(t, cfg=cfg, ws=ws)              # first call (direct launches)
    t.copy_(keys)
    st = ls.ls_sort(t, cfg=cfg, ws=ws, dumps=dd)
    got = to_np(t)
    osorted, om, ost, od = O.sort(h, dumps="tables")
    assert np.array_equal(bits(got), bits(osorted)), "sorted output differs from the oracle"
    del got, osorted
    assert_models_identical(gm, om)
    assert np.array_equal(d["S_B"].cpu().numpy().astype(np.uint64), od["S_B"])
    assert np.array_equal(d["H0"].cpu().numpy(), od["H0"])
    assert np.array_equal(d["S_B1"].cpu().numpy().astype(np.uint64), od["S_B1"])
    assert np.array_equal(d["H1"].cpu().numpy(), od["H1"])
    for k in ("h0_buckets", "h0_keys", "h1_subbuckets", "h1_keys"):
        assert st[k] == ost[k], k
    idx = np.random.default_rng(0).choice(n, 100_000, replace=False)
    sub = from_np(h[idx])
    ids = ls.ls_bucket_ids(sub, oracle_model_to_ls(om), want=("p", "b0", "b1"))
    p = O.predict(om, h[idx])
    assert np.array_equal(bits(ids["p"].cpu().numpy()), bits(p))
    L = O.lib()
    b0 = np.array([L.lso_bucket_l0(float(x), 1000) for x in p[:20_000]], np.uint64)
    assert np.array_equal(ids["b0"].cpu().numpy()[:20_000].astype(np.uint64), b0)
    b1 = np.array([L.lso_bucket_l1(float(x), 1000, int(q)) for x, q in zip(p[:20_000], b0)], np.uint64)
    assert np.array_equal(ids["b1"].cpu().numpy()[:20_000].astype(np.uint64), b1)


# ------------------------------------------------------------- multi-GPU ---

def test_sort_multi_single_rank():
    """ls_sort_multi with a one-rank NCCL communicator: split sample, splitters,
    destination count/scatter, NCCL send/recv to self, local sort. (N > 1 host
    logic: tests/test_multi_gloo.py; this box has one GPU.)"""
    comm = ls.Comm(0, 1, ls.Comm.unique_id())
    try:
        for dist, n in (("cfg5mix", 2_000_000), ("twodups", 300_001)):
            keys = gen(dist, n, 1000)
            h = to_np(keys)
            out = torch.empty(n + 1000, dtype=keys.dtype, device=DEV)
            n_out, st = ls.ls_sort_multi(comm, keys, out)
            assert n_out == n
            assert np.array_equal(bits(to_np(out[:n_out])), bits(O.sort(h)[0]))
        small = torch.empty(10, dtype=keys.dtype, device=DEV)
        with pytest.raises(ls.LSError) as e:
            ls.ls_sort_multi(comm, keys, small)
        assert e.value.status == ls.LS_E_CAPACITY
    finally:
        comm.close()


def ord_np(a):
    """IEEE totalOrder key (R12) of fp64 / identity for u64, as uint64."""
    b = bits(a).astype(np.uint64)
    if a.dtype == np.float64:
        neg = (b >> np.uint64(63)) == 1
        return np.where(neg, ~b, b | np.uint64(1 << 63))
    return b


@pytest.mark.parametrize("world,dist", [(2, "normal"), (3, "zipf"), (4, "twodups"),
                                        (8, "cfg5mix"), (5, "telemetry")])
def test_multi_route_world_gt1(world, dist):
    """§8(e) for R > 1 ranks on one GPU, without a communicator (nothing waits
    on another rank): each virtual rank's split sample (ls_multi_sample), the
    splitters of the gathered samples, and each rank's destination counts and
    send buffer (ls_multi_route: k_dest_count + k_dest_scatter, steps 3 and 5
    of ls_sort_multi). Checked: every key's destination equals the
    lexicographic (ord, rank, index) rule recomputed on the host, each
    destination receives exactly that multiset, and sorting the destinations
    one by one (the local ls_sort of step 7) and concatenating them gives the
    oracle's global order."""
    rng = np.random.default_rng(world)
    n = 1_500_007
    keys = gen(dist, n, 31)
    h = to_np(keys)
    cuts = np.concatenate([[0], np.sort(rng.choice(np.arange(1, n), world - 1, replace=False)), [n]])
    shards = [keys[cuts[r]:cuts[r + 1]].clone() for r in range(world)]  # (aligned copies)
    gathered = np.concatenate([ls.multi_sample(sh, r) for r, sh in enumerate(shards)])
    spl = ls.multi_splitters(gathered.copy(), world)
    recv = [[] for _ in range(world)]
    for r, sh in enumerate(shards):
        send = torch.empty_like(sh)
        counts = ls.multi_route(sh, r, world, spl, send)
        assert int(counts.sum()) == sh.numel()
        # host rule: dest = #splitters below (ord, r, i)
        o = ord_np(to_np(sh))
        idx = np.arange(sh.numel(), dtype=np.uint64)
        dest = np.zeros(sh.numel(), np.int64)
        for s_ in spl:
            so, sr, si = np.uint64(s_["ord"]), np.uint32(s_["rank"]), np.uint64(s_["index"])
            below = (so < o) | ((so == o) & ((sr < np.uint32(r)) | ((sr == np.uint32(r)) & (si < idx))))
            dest += below
        assert np.array_equal(np.bincount(dest, minlength=world).astype(np.uint64), counts)
        sent = to_np(send)
        sd = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        for p in range(world):
            part = sent[sd[p]:sd[p + 1]]
            want = to_np(sh)[dest == p]
            assert np.array_equal(np.sort(ord_np(part)), np.sort(ord_np(want)))
            recv[p].append(part)
    out = []
    for p in range(world):
        rp = np.concatenate(recv[p]) if recv[p] else np.zeros(0, h.dtype)
        t = from_np(rp)
        if t.numel():
            ls.ls_sort(t)
        out.append(to_np(t))
    assert np.array_equal(bits(np.concatenate(out)), bits(O.sort(h)[0]))


@pytest.mark.parametrize("world,dist", [(2, "normal"), (3, "zipf"), (8, "cfg5mix"), (5, "telemetry"),
                                        (4, "twodups")])
def test_multi_route_peer_world_gt1(world, dist):
    """SURVEY f1 (LS_FLAG_PEER_SCATTER's fused scatter) for R > 1 virtual ranks
    on one GPU: each rank's destination scatter stores its runs straight into
    the R receive buffers (separate allocations standing for the peers' d_out)
    at its own slice (after the lower ranks', as ls_sort_multi places them).
    Checked: the counts equal the send-buffer path's, every slice holds exactly
    the keys the host rule sends there, no slice spills into another (the
    buffers start filled with a sentinel and every key is accounted for), the
    split is balanced (R = 8: within 10 % of n/R), and sorting the receive
    buffers one by one reproduces the oracle's global order."""
    rng = np.random.default_rng(world + 100)
    n = 1_500_007
    keys = gen(dist, n, 37)
    h = to_np(keys)
    cuts = np.concatenate([[0], np.sort(rng.choice(np.arange(1, n), world - 1, replace=False)), [n]])
    shards = [keys[cuts[r]:cuts[r + 1]].clone() for r in range(world)]
    gathered = np.concatenate([ls.multi_sample(sh, r) for r, sh in enumerate(shards)])
    spl = ls.multi_splitters(gathered.copy(), world)
    sends, mat = [], []
    for r, sh in enumerate(shards):
        send = torch.empty_like(sh)
        mat.append(ls.multi_route(sh, r, world, spl, send))
        sends.append(to_np(send))
    mat = np.stack(mat).astype(np.int64)          # mat[r][p]: keys rank r sends to p
    sizes = mat.sum(0)
    assert sizes.sum() == n
    assert sizes.max() <= 1.10 * n / world, f"imbalanced split: {sizes}"
    sent_bits = np.uint64(0x7ff4dead0000beef)    # (a NaN pattern: never a generated key)
    recv = [torch.full((int(sizes[p]) + 8,), 0, dtype=torch.int64, device=DEV) for p in range(world)]
    for t in recv:
        t.fill_(int(sent_bits.astype(np.int64)))
    recv = [t.view(keys.dtype) for t in recv]
    for r, sh in enumerate(shards):
        off = mat[:r].sum(0).astype(np.uint64)
        got = ls.multi_route_peer(sh, r, world, spl, recv, off)
        assert np.array_equal(got.astype(np.int64), mat[r])
    for p in range(world):
        rp = to_np(recv[p])
        assert np.all(bits(rp[sizes[p]:]) == sent_bits)      # nothing past the slices
        o = 0
        for r in range(world):
            sd = np.concatenate([[0], np.cumsum(mat[r])])
            want = sends[r][sd[p]:sd[p + 1]]
            part = rp[o:o + mat[r][p]]
            assert np.array_equal(np.sort(ord_np(part)), np.sort(ord_np(want)))
            o += mat[r][p]
    out = []
    for p in range(world):
        t = recv[p][:sizes[p]].clone()
        if t.numel():
            ls.ls_sort(t)
        out.append(to_np(t))
    assert np.array_equal(bits(np.concatenate(out)), bits(O.sort(h)[0]))


def test_sort_multi_single_rank_peer_scatter():
    """ls_sort_multi with LS_FLAG_PEER_SCATTER on a one-rank communicator: the
    fused scatter writes straight into d_out (the rank's own slice), one NCCL
    all-reduce, the local sort -- the oracle's output."""
    comm = ls.Comm(0, 1, ls.Comm.unique_id())
    try:
        cfg = ls.config(flags=ls.LS_FLAG_PEER_SCATTER)
        for dist, n in (("cfg5mix", 2_000_000), ("twodups", 300_001), ("normal", 1)):
            keys = gen(dist, n, 1001)
            h = to_np(keys)
            out = torch.empty(n + 1000, dtype=keys.dtype, device=DEV)
            n_out, st = ls.ls_sort_multi(comm, keys, out, cfg=cfg)
            assert n_out == n and st["peer_scatter"] == 1
            assert np.array_equal(bits(to_np(out[:n_out])), bits(O.sort(h)[0]))
    finally:
        comm.close()


# -------------------------------------------------- large big sub-buckets --

def _clusters(dtype, seed):
    """Three tight clusters of 400K keys each (the model cannot separate them:
    large BIG sub-buckets) plus a uniform background."""
    rng = np.random.default_rng(seed)
    if dtype == np.uint64:
        parts = [np.uint64(c) + rng.integers(0, 5000, 400_000).astype(np.uint64)
                 for c in (10 ** 15, 2 ** 62, 2 ** 63 + 12345)]
        parts.append(rng.integers(0, 2 ** 64 - 1, 200_000, dtype=np.uint64))
    else:
        parts = [c + rng.integers(0, 5000, 400_000) * 1e-9 for c in (-3.0, 0.25, 7e3)]
        parts.append(rng.uniform(-1e4, 1e4, 200_000))
        parts.append(np.array([np.inf, -np.inf, 0.0] * 100))
    a = np.concatenate(parts).astype(dtype)
    rng.shuffle(a)
    return a


@pytest.mark.parametrize("case", ["cfg5mix", "clusters_u64", "clusters_f64", "twovalue"])
def test_large_big_items(case):
    """Sub-buckets > 64K keys take the grid-parallel path (ls_bigpath.cu):
    homogeneous digit pieces filled by value, the rest scattered and sorted."""
    if case == "cfg5mix":
        keys = gen("cfg5mix", 6_000_000, 1000)
    elif case == "twovalue":
        rng = np.random.default_rng(3)
        a = np.where(rng.random(2_000_000) < 0.5, 1.0, 2.0)
        a[:1000] = rng.uniform(0, 1e6, 1000)
        keys = from_np(a)
    else:
        keys = from_np(_clusters(np.uint64 if case.endswith("u64") else np.float64, 7))
    h = to_np(keys)
    t = keys.clone()
    st = ls.ls_sort(t)
    assert np.array_equal(bits(to_np(t)), bits(O.sort(h)[0]))
    if case.startswith("clusters"):
        assert st["big_keys"] >= 800_000


def _dense_clusters(case, seed):
    """20 clusters of 30K keys (BIG sub-buckets of 8K..256K keys: the per-CTA
    big path) plus a uniform background. The cluster values decide whether the
    counting sort by value (k_big's dense path: keys = mn + s * 2^tz with
    fewer than 16K slots) or the MSD radix path sorts them."""
    rng = np.random.default_rng(seed)
    if case == "f64":                 # 6000 consecutive doubles per cluster (ord stride 1)
        parts = [c + rng.integers(0, 6000, 30_000) * np.spacing(abs(c))
                 for c in rng.uniform(-1e6, 1e6, 20)]
        parts.append(rng.uniform(-1e6, 1e6, 200_001))
        a = np.concatenate(parts)
        rng.shuffle(a)
        return a
    centres = rng.integers(2 ** 40, 2 ** 62, 20)
    parts = []
    for j, c in enumerate(centres):
        if case == "stride1024":      # config 4's fp64-built IDs: multiples of 2^10, ~8K slots
            k = np.clip(np.rint(rng.normal(0, 1024, 30_000)), -4000, 4000).astype(np.int64)
            v = np.uint64(c & ~1023) + (k * 1024).astype(np.uint64)
        elif case == "stride1":       # consecutive integers, 10K slots
            v = np.uint64(c) + rng.integers(0, 10_000, 30_000).astype(np.uint64)
        elif case == "wide":          # 50K slots: radix path
            v = np.uint64(c) + rng.integers(0, 50_000, 30_000).astype(np.uint64)
        elif case == "mixed":         # one cluster in two breaks the stride with a single odd key
            v = np.uint64(c & ~1023) + (rng.integers(0, 8000, 30_000) * 1024).astype(np.uint64)
            if j % 2:
                v[7] += np.uint64(1)
        parts.append(v.astype(np.uint64))
    parts.append(rng.integers(0, 2 ** 63, 200_001, dtype=np.uint64))
    a = np.concatenate(parts)
    rng.shuffle(a)
    return a


@pytest.mark.parametrize("case", ["stride1024", "stride1", "wide", "mixed", "f64"])
def test_dense_big_items(case):
    """k_big's counting sort by value (dense slots) and its radix fallback:
    the oracle's output, S_B/S'_B/H0/H1 and the class counts."""
    keys = from_np(_dense_clusters(case, 11))
    st, ost = check_sort(keys)
    assert st["big_keys"] >= 400_000


# ------------------------------------------- the paper's second workloads --

@pytest.mark.parametrize("s", [0.5, 0.9, 0.99])
def test_zipf_skew_sweep_bit_exact(s):
    """Fig. 6: Zipf skews 0.5 .. 0.99 (V = 10^5 values)."""
    plan = datagen.Plan("zipf", 2_000_000, 1, zipf_s=s, zipf_V=100_000)
    keys = torch.empty(2_000_000, dtype=torch.uint64, device=DEV)
    plan.device(keys)
    torch.cuda.synchronize()
    check_sort(keys)


@pytest.mark.parametrize("n", [1_000_000, 4_000_000, 16_000_000])
def test_size_sweep_bit_exact(n):
    """Fig. 5: Normal(0,1) and TwoDups across sizes."""
    for dist in ("normal", "twodups"):
        keys = gen(dist, n, 0)
        h = to_np(keys)
        t = keys.clone()
        ls.ls_sort(t)
        assert np.array_equal(bits(to_np(t)), bits(O.sort(h)[0]))


# ------------------------------------------------ CUDA Graph replay (f2) --

@pytest.mark.parametrize("n", [1_000_000, 3_000_001])
def test_graph_replay_bit_exact(n, monkeypatch):
    """the launch sequence is captured into a CUDA Graph the
    second time the same (keys, n, dtype, config, workspace) comes back and
    replayed afterwards. Different inputs through the same buffers must each
    come out bit-exact (LS_GRAPH=2: a failed capture is an error, not a silent
    direct launch); LS_GRAPH=0 (direct launches) gives the same bytes."""
    monkeypatch.setenv("LS_GRAPH", "2")
    t = torch.empty(n, dtype=torch.float64, device=DEV)
    ws = ls.workspace(n, ls.LS_F64)
    inputs = [("normal", 1), ("lognormal", 2), ("mixgauss", 3), ("normal", 4), ("uniform01", 5)]
    for i, (dist, seed) in enumerate(inputs):
        src = gen(dist, n, seed)
        if i == 4:  # few distinct values and an all-equal run through the replayed graph
            src[: n // 2] = 0.25
        h = to_np(src)
        t.copy_(src)
        st = ls.ls_sort(t, ws=ws)
        assert np.array_equal(bits(to_np(t)), bits(O.sort(h)[0])), (i, dist)
        assert st["kernel_launches"] > 10
        if i == 3:
            monkeypatch.setenv("LS_GRAPH", "0")
            t.copy_(src)
            ls.ls_sort(t, ws=ws)
            assert np.array_equal(bits(to_np(t)), bits(O.sort(h)[0]))
            monkeypatch.setenv("LS_GRAPH", "2")


def test_graph_replay_phase_timing(monkeypatch):
    """With LS_FLAG_PHASE_TIMING the phase events are event-record nodes of the
    captured graph: the replayed sorts still report every phase's time."""
    monkeypatch.setenv("LS_GRAPH", "2")
    n = 2_000_000
    t = torch.empty(n, dtype=torch.float64, device=DEV)
    cfg = ls.config(flags=ls.LS_FLAG_PHASE_TIMING)
    ws = ls.workspace(n, ls.LS_F64, cfg)
    for seed in (1, 2, 3):
        src = gen("normal", n, seed)
        h = to_np(src)
        t.copy_(src)
        st = ls.ls_sort(t, cfg=cfg, ws=ws)
        assert np.array_equal(bits(to_np(t)), bits(O.sort(h)[0]))
        ph = st["phase_ms"]
        for k in ("fit", "count0", "scatter0", "count1", "scatter1", "bucketsort"):
            assert ph[k] > 0, (seed, k, ph)
        assert sum(ph.values()) < 1000


def test_graph_cache_eviction(monkeypatch):
    """More distinct (buffer, size) keys than the 16-entry graph cache holds:
    entries are evicted (their graphs destroyed) and re-captured, and every
    sort stays bit-exact."""
    monkeypatch.setenv("LS_GRAPH", "2")
    bufs = []
    for i in range(20):
        n = 50_000 + 1_000 * i
        bufs.append((torch.empty(n, dtype=torch.float64, device=DEV), ls.workspace(n, ls.LS_F64),
                     gen("mixgauss", n, 100 + i)))
    for rnd in range(2):
        for t, ws, src in bufs:
            for rep in range(3):  # seen, captured + replayed, replayed
                t.copy_(src)
                ls.ls_sort(t, ws=ws)
                assert np.array_equal(bits(to_np(t)), bits(np.sort(to_np(src)))), (rnd, rep)


def test_graph_replay_launch_failure_falls_back(monkeypatch):
    """A failed replay launch (forced by LS_TEST_GRAPH_LAUNCH_FAIL; in the
    field: a graph whose context was reset) drops every cached graph and the
    capture streams, clears the error and launches the sequence directly; the
    sort is still bit-exact, reports no CUDA error, and the next calls capture
    and replay again."""
    monkeypatch.setenv("LS_GRAPH", "1")
    n = 500_000
    t = torch.empty(n, dtype=torch.float64, device=DEV)
    ws = ls.workspace(n, ls.LS_F64)
    src = gen("normal", n, 77)
    want = O.sort(to_np(src))[0]
    for i in range(6):
        if i == 3:
            monkeypatch.setenv("LS_TEST_GRAPH_LAUNCH_FAIL", "1")
        elif i == 4:
            monkeypatch.delenv("LS_TEST_GRAPH_LAUNCH_FAIL")
        t.copy_(src)
        ls.ls_sort(t, ws=ws)
        assert np.array_equal(bits(to_np(t)), bits(want)), i


def test_round0_exact_fallback(monkeypatch):
    """Round 0 by reservation (k_cap0 + k_scatter0r): bucket capacities come
    from the 1 % strided sample. An input whose sample misrepresents it (every
    100th key spread over [0, 1), the other 99 % inside [0, 0.001)) overflows
    bucket 0's capacity; the call then takes the exact count pass (k_count0 +
    k_scatter0) and is still bit-exact with the oracle, S_B / S'_B / H0 / H1
    included. LS_EXACT0=1 forces the exact pass on a smooth input (same bytes
    as the reservation path)."""
    n = 1_000_000
    rng = np.random.default_rng(9)
    a = rng.random(n) * 1e-3
    a[::100] = rng.random(len(a[::100]))
    st, _ = check_sort(from_np(a))
    assert st["round0_exact"] == 1
    keys = gen("normal", 2_000_000, 4)
    st, _ = check_sort(keys)
    assert st["round0_exact"] == 0
    monkeypatch.setenv("LS_EXACT0", "1")
    st, _ = check_sort(keys)
    assert st["round0_exact"] == 1
