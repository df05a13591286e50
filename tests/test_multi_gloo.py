"""N > 1 path of ls_sort_multi on CPU: world_size-2 (and 3) gloo process groups.

ls_sort_multi = split sample -> all-gather -> R-1 splitters on
(ord, rank, index) -> destination per key -> count matrix -> all-to-all ->
local LearnedSort 2.0. The device kernels need a GPU, so here every rank runs
the library's own HOST planning entry points (ls_multi_splitters,
ls_multi_dest, ls_multi_plan -- the same functions ls_sort_multi calls), the
exchange goes over gloo, and the local sort is the oracle. Checked: every rank
derives identical splitters, rank r receives a contiguous slice of the global
order (the concatenation over ranks equals the sorted union bit for bit), the
plan's counts/displacements match what arrived, and heavy duplicates (config 5's
Zipf(1.0) half) are spread across ranks by the (rank, index)
tie-break instead of overloading one rank.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

SPLIT_K = 16384  # sample entries per rank (ls_multi.cu SPLIT_K = LS_MULTI_SAMPLE)
TAGGED = np.dtype([("ord", "<u8"), ("rank", "<u4"), ("pad", "<u4"), ("index", "<u8")])


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def split_sample(keys_ord, rank):
    """Host restatement of k_split_sample: k < SPLIT_K, idx = k*n/SPLIT_K."""
    n = len(keys_ord)
    out = np.zeros(SPLIT_K, TAGGED)
    out["ord"], out["rank"], out["index"] = ~np.uint64(0), 0xFFFFFFFF, ~np.uint64(0)
    valid = min(n, SPLIT_K)
    idx = np.arange(valid, dtype=np.uint64)
    if n > SPLIT_K:
        idx = (idx * np.uint64(n)) // np.uint64(SPLIT_K)
    out["ord"][:valid] = keys_ord[idx.astype(np.int64)]
    out["rank"][:valid] = rank
    out["index"][:valid] = idx
    return out


def worker(rank, world, port, dist_name, n, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import datagen
        import oracle as O
        import paper_2107_03290_b200 as ls

        keys = datagen.generate_host(dist_name, n + 37 * rank, 1000 + rank)  # unequal shards
        o = O.ord_key(keys)
        # 1. split sample + all-gather
        samp = split_sample(o, rank)
        gathered = [torch.zeros(SPLIT_K * TAGGED.itemsize, dtype=torch.uint8) for _ in range(world)]
        dist.all_gather(gathered, torch.from_numpy(samp.view(np.uint8).copy()))
        entries = np.concatenate([g.numpy().view(TAGGED) for g in gathered])
        # 2. splitters (library host code), identical on every rank
        spl = ls.multi_splitters(entries, world)
        allspl = [None] * world
        dist.all_gather_object(allspl, spl.tobytes())
        assert all(s == allspl[0] for s in allspl)
        # 3. destination per key (library rule), monotone in (ord, rank, index)
        dest = np.array([ls.multi_dest(spl, world, int(o[i]), rank, i) for i in range(len(o))])
        order = np.lexsort((np.arange(len(o)), o))
        assert np.all(np.diff(dest[order]) >= 0)
        counts = np.bincount(dest, minlength=world).astype(np.int64)
        # 4. count matrix -> plan
        cm = [torch.zeros(world, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(cm, torch.from_numpy(counts))
        mat = torch.stack(cm).numpy().astype(np.uint64)
        sd, rc, rd, n_out = ls.multi_plan(mat, world, rank)
        assert np.array_equal(sd, np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.uint64))
        # 5. scatter by destination (stable) + 6. all-to-all
        send = keys.view(np.uint64)[np.argsort(dest, kind="stable")]
        recv = torch.zeros(int(n_out), dtype=torch.int64)
        dist.all_to_all_single(recv, torch.from_numpy(send.view(np.int64).copy()),
                               output_split_sizes=[int(c) for c in rc],
                               input_split_sizes=[int(c) for c in counts])
        got = recv.numpy().view(np.uint64)
        # receive displacements: block p of recv came from rank p
        for p in range(world):
            blk = got[int(rd[p]): int(rd[p]) + int(rc[p])]
            assert len(blk) == int(mat[p, rank])
        # 7. local LearnedSort 2.0 (oracle here; ls_sort on the GPU)
        mine = got.view(keys.dtype)
        local = O.sort(mine)[0] if len(mine) > 1 else mine
        parts = [None] * world
        dist.all_gather_object(parts, (local.view(np.uint64).tobytes(), keys.view(np.uint64).tobytes()))
        if rank == 0:
            results.put([(np.frombuffer(a, np.uint64), np.frombuffer(b, np.uint64)) for a, b in parts])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,dist_name,n", [(2, "cfg5mix", 30_000), (3, "cfg5mix", 20_000),
                                               (2, "normal", 25_000), (2, "rootdups", 20_000)])
def test_multi_rank_range_split_gloo(world, dist_name, n):
    import datagen
    import oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, dist_name, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    dt = datagen.np_dtype(dist_name)
    slices = [a.view(dt) for a, _ in parts]
    union = np.concatenate([b.view(dt) for _, b in parts])
    want = O.sort(union)[0]
    got = np.concatenate(slices)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    # balance: the (ord, rank, index) tie-break spreads equal keys across ranks
    sizes = np.array([len(s) for s in slices])
    assert sizes.min() > 0
    assert sizes.max() <= 1.25 * len(union) / world
