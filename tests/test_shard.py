"""The Morton-range sharded path (paper_2103_05162_b200/shard.py)
with world size 2 over gloo.

CPU tests run the distributed protocol with the oracle as the local engine
(test infrastructure: O(n^2) numpy neighbourhoods, the C restatement's
Morton codes); the gpu-marked tests run the same protocol with the product
DeviceEngine (C-ABI device stages), two processes sharing cuda:0. In both,
the union of the shards' results must equal the single-process reference
result: core flags and noise exact, core labels equal (global minimum core
id), every border label valid."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle


class OracleEngine:
    """Test-only local engine on CPU tensors (exact fp64 predicates)."""

    def morton(self, x, lo, hi):
        c = oracle.morton_codes(x.numpy(), lo.numpy(), hi.numpy())
        return torch.from_numpy(c.astype(np.int64))

    @staticmethod
    def _d2(a, b):
        a = a.astype(np.float64)
        b = b.astype(np.float64)
        d = a[:, None, 0] - b[None, :, 0]
        s = d * d
        for k in range(1, a.shape[1]):
            d = a[:, None, k] - b[None, :, k]
            s = s + d * d
        return s

    def near_boxes(self, x, eps, blo, bhi):
        p = x.numpy().astype(np.float64)
        lo = blo.numpy().astype(np.float64)
        hi = bhi.numpy().astype(np.float64)
        s = np.zeros((p.shape[0], lo.shape[0]))
        for k in range(p.shape[1]):
            d = np.maximum(np.maximum(lo[None, :, k] - p[:, None, k], p[:, None, k] - hi[None, :, k]), 0)
            s = s + d * d
        e2 = np.float64(np.float32(eps)) ** 2
        return torch.from_numpy((s <= e2).any(1).astype(np.uint8))

    def core_flags(self, x, eps, minpts):
        e2 = np.float64(np.float32(eps)) ** 2
        cnt = (self._d2(x.numpy(), x.numpy()) <= e2).sum(1)
        return torch.from_numpy((cnt >= minpts).astype(np.uint8))

    def cluster_keyed(self, x, keys, eps, minpts):
        """Labels = key of the cluster's minimum-key core (FoF when minpts == 2)."""
        r = oracle.dbscan(x.numpy(), eps, minpts, 0)
        lab = r["labels"].astype(np.int64)
        core = r["core"].astype(bool)
        k = keys.numpy().astype(np.int64)
        big = np.iinfo(np.int64).max
        best = np.full(len(lab), big, np.int64)
        cm = core & (lab >= 0)
        np.minimum.at(best, lab[cm], k[cm])
        out = np.where(lab >= 0, best[np.maximum(lab, 0)], -1)
        return torch.from_numpy(out.astype(np.int32)), torch.from_numpy(r["core"].astype(np.uint8))

    def local(self, x, keys, eps):
        """Test double of tcg_local_*: core flags, then the main pass with the
        given flags, labels = key of the cluster's minimum-key core."""
        eng = self

        class Local:
            def core_flags(self, minpts):
                return eng.core_flags(x, eps, minpts)

            def cluster(self, core):
                lab = eng.cluster_given_core(x, eps, core).numpy().astype(np.int64)
                k = keys.numpy().astype(np.int64)
                c = core.numpy().astype(bool)
                big = np.iinfo(np.int64).max
                best = np.full(len(lab), big, np.int64)
                cm = c & (lab >= 0)
                np.minimum.at(best, lab[cm], k[cm])
                out = np.where(lab >= 0, best[np.maximum(lab, 0)], -1)
                return torch.from_numpy(out.astype(np.int32))

            def close(self):
                pass

        return Local()

    def cluster_given_core(self, x, eps, core):
        e2 = np.float64(np.float32(eps)) ** 2
        adj = self._d2(x.numpy(), x.numpy()) <= e2
        c = core.numpy().astype(bool)
        n = len(c)
        parent = np.arange(n)

        def find(i):
            while parent[i] != i:
                parent[i] = parent[parent[i]]
                i = parent[i]
            return i

        for i, j in zip(*np.nonzero(np.triu(adj & c[:, None] & c[None, :], 1))):
            a, b = find(i), find(j)
            if a != b:
                parent[max(a, b)] = min(a, b)
        lab = np.full(n, -1, np.int64)
        for i in range(n):
            if c[i]:
                lab[i] = find(i)
        for i in range(n):
            if not c[i]:
                nb = np.nonzero(adj[i] & c)[0]
                if len(nb):
                    lab[i] = lab[nb].min()
        return torch.from_numpy(lab.astype(np.int32))

    def union_edges(self, edges, n):
        parent = np.arange(n)

        def find(i):
            while parent[i] != i:
                parent[i] = parent[parent[i]]
                i = parent[i]
            return i

        for a, b in edges.numpy():
            ra, rb = find(a), find(b)
            if ra != rb:
                parent[max(ra, rb)] = min(ra, rb)
        return torch.from_numpy(np.array([find(i) for i in range(n)], np.int32))


class OracleEngineFused(OracleEngine):
    """OracleEngine plus numpy doubles of the fused device stages
    (tcg_shard_route_device, tcg_shard_region_boxes_device,
    tcg_near_peers_device), so the CPU tests drive the same protocol branch
    as the DeviceEngine."""

    def route(self, x, gid, codes, splitters):
        c = codes.numpy()
        owner = np.searchsorted(splitters.numpy(), c, side="right")
        order = np.argsort(owner, kind="stable")
        d = x.shape[1]
        rows = np.concatenate([x.numpy()[order].view(np.int32),
                               gid.numpy()[order].view(np.int32).reshape(-1, 2),
                               c[order].view(np.int32).reshape(-1, 2)], 1).reshape(-1, d + 4)
        counts = np.bincount(owner, minlength=splitters.shape[0] + 1)
        return torch.from_numpy(np.ascontiguousarray(rows)), [int(v) for v in counts]

    def region_boxes(self, x, codes):
        c = codes.numpy().astype(np.uint64)
        lo, hi = int(c.min()), int(c.max())
        shift = 0
        while (hi >> shift) - (lo >> shift) >= (1 << 12):
            shift += 1
        cell = (c >> np.uint64(shift)) - np.uint64(lo >> shift)
        uniq, inv = np.unique(cell, return_inverse=True)
        p = x.numpy()
        blo = np.full((len(uniq), p.shape[1]), np.inf, np.float32)
        bhi = np.full((len(uniq), p.shape[1]), -np.inf, np.float32)
        np.minimum.at(blo, inv, p)
        np.maximum.at(bhi, inv, p)
        return torch.from_numpy(np.concatenate([blo, bhi], 1))

    def near_peers(self, x, eps, blo, bhi, owner):
        mask = np.zeros(x.shape[0], np.int64)
        own = owner.numpy()
        for j in np.unique(own):
            sel = own == j
            m = self.near_boxes(x, eps, blo[torch.from_numpy(sel)], bhi[torch.from_numpy(sel)])
            mask |= m.numpy().astype(np.int64) << int(j)
        return torch.from_numpy(mask)


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, coords, eps, minpts, use_gpu, out_q, backend="gloo",
            force_exchange=False, fused=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    if backend == "nccl":
        import torch as _t
        _t.cuda.set_device(0)
        dist.init_process_group("nccl", rank=rank, world_size=world,
                                device_id=_t.device("cuda", 0))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2103_05162_b200.shard import DeviceEngine, cluster_sharded

    n = coords.shape[0]
    # input partition: interleaved slices (deliberately not spatial)
    idx = np.arange(rank, n, world)
    x = torch.from_numpy(coords[idx])
    gid = torch.from_numpy(idx.astype(np.int64))
    if use_gpu:
        engine = DeviceEngine("cuda:0")
        x = x.cuda()
        gid = gid.cuda()
    else:
        engine = OracleEngineFused() if fused else OracleEngine()
    g, lab, core = cluster_sharded(x, gid, eps, minpts, engine, block=64, samples=256,
                                   force_exchange=force_exchange)
    out_q.put((rank, g.cpu().numpy(), lab.cpu().numpy(), core.cpu().numpy()))
    dist.barrier()
    dist.destroy_process_group()


def run_sharded(coords, eps, minpts, world=2, use_gpu=False, backend="gloo",
                force_exchange=False, fused=False):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, coords, eps, minpts, use_gpu, q,
                                               backend, force_exchange, fused))
             for r in range(world)]
    for p in procs:
        p.start()
    import queue
    import time
    res, deadline = [], time.time() + 600
    while len(res) < world:  # fail fast when a rank dies instead of waiting out the timeout
        try:
            res.append(q.get(timeout=2))
        except queue.Empty:
            dead = [p.exitcode for p in procs if p.exitcode not in (None, 0)]
            assert not dead, f"a rank exited with {dead}"
            assert time.time() < deadline, "sharded run timed out"
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    n = coords.shape[0]
    labels = np.full(n, -2, np.int64)
    core = np.zeros(n, np.uint8)
    owned = 0
    for _, g, lab, c in res:
        labels[g] = lab
        core[g] = c
        owned += len(g)
    assert owned == n and (labels != -2).all(), "every point owned exactly once"
    return labels, core


def check_against_oracle(coords, eps, minpts, labels, core):
    want = oracle.dbscan(coords, eps, minpts, 0)
    assert np.array_equal(core, want["core"]), "core flags differ"
    assert np.array_equal(labels == -1, want["labels"] == -1), "noise differs"
    cm = want["core"] == 1
    assert np.array_equal(labels[cm], want["labels"][cm]), "core labels differ"
    ok, msg = oracle.check_equivalence(coords, eps, labels.astype(np.int32), core,
                                       want["labels"], want["core"])
    assert ok, msg


def blob_mix(seed, n, dim):
    rng = np.random.default_rng(seed)
    k = 6
    centers = rng.uniform(0, 10, (k, dim))
    pts = [rng.normal(centers[rng.integers(k)], 0.35, (n // (2 * k), dim)) for _ in range(2 * k)]
    pts.append(rng.uniform(0, 10, (n // 4, dim)))
    return np.concatenate(pts).astype(np.float32)


@pytest.mark.parametrize("dim,eps,minpts", [(3, 0.3, 2), (3, 0.45, 5), (2, 0.2, 4), (2, 0.15, 2)])
def test_sharded_world2_matches_single_process(dim, eps, minpts):
    coords = blob_mix(10 + dim + minpts, 1800, dim)
    labels, core = run_sharded(coords, eps, minpts, world=2)
    check_against_oracle(coords, eps, minpts, labels, core)


@pytest.mark.parametrize("world,minpts", [(2, 2), (3, 5)])
def test_sharded_fused_stages(world, minpts):
    """The protocol branch of the fused device stages (route, region boxes,
    one-pass peer halo), with their numpy doubles."""
    coords = blob_mix(31 + world, 1500, 3)
    labels, core = run_sharded(coords, 0.4, minpts, world=world, fused=True)
    check_against_oracle(coords, 0.4, minpts, labels, core)


def test_sharded_world3_uneven():
    coords = blob_mix(5, 1500, 3)[:1237]
    labels, core = run_sharded(coords, 0.4, 4, world=3)
    check_against_oracle(coords, 0.4, 4, labels, core)


@pytest.mark.gpu
@pytest.mark.parametrize("dim,eps,minpts", [(3, 0.3, 2), (2, 0.2, 5)])
def test_sharded_device_engine_world2(dim, eps, minpts):
    coords = blob_mix(40 + dim, 6000, dim)
    labels, core = run_sharded(coords, eps, minpts, world=2, use_gpu=True)
    check_against_oracle(coords, eps, minpts, labels, core)


@pytest.mark.parametrize("minpts", [2, 4])
def test_sharded_world1(minpts):
    """A single rank: no exchange at all, the local run is the whole result."""
    coords = blob_mix(21, 1200, 3)
    labels, core = run_sharded(coords, 0.35, minpts, world=1)
    check_against_oracle(coords, 0.35, minpts, labels, core)


@pytest.mark.gpu
@pytest.mark.parametrize("minpts", [2, 6])
def test_sharded_device_engine_world1(minpts):
    coords = blob_mix(44, 8000, 3)
    labels, core = run_sharded(coords, 0.3, minpts, world=1, use_gpu=True)
    check_against_oracle(coords, 0.3, minpts, labels, core)


@pytest.mark.parametrize("minpts", [2, 4])
def test_sharded_world1_forced_exchange(minpts):
    """One rank running the whole multi-rank protocol (redistribution to
    itself, halo exchange with no peers, edge merge)."""
    coords = blob_mix(23, 1200, 3)
    labels, core = run_sharded(coords, 0.35, minpts, world=1, force_exchange=True)
    check_against_oracle(coords, 0.35, minpts, labels, core)


@pytest.mark.gpu
@pytest.mark.parametrize("minpts", [2, 6])
def test_sharded_nccl_world1_forced_exchange(minpts):
    """The NCCL branch of every collective (device tensors in all_reduce,
    padded all_gather, variable all_to_all_single incl. empty sends) on the
    one GPU of the box: the multi-rank protocol forced on a single rank, with
    the product engine, against the oracle."""
    coords = blob_mix(45, 8000, 3)
    labels, core = run_sharded(coords, 0.3, minpts, world=1, use_gpu=True, backend="nccl",
                               force_exchange=True)
    check_against_oracle(coords, 0.3, minpts, labels, core)


@pytest.mark.parametrize("minpts", [2, 3, 5])
def test_sharded_rank_without_points(minpts):
    """All points at one coordinate: every Morton code is equal, the splitters
    coincide and one rank owns nothing. That rank must still take part in every
    collective of the chosen path (divergent collectives would
    hang), and the result must equal the single-process one."""
    coords = np.tile(np.array([[1.5, -2.0, 0.25]], np.float32), (40, 1))
    labels, core = run_sharded(coords, 0.1, minpts, world=2)
    check_against_oracle(coords, 0.1, minpts, labels, core)


def test_sharded_world3_two_clumps_one_empty_rank():
    """Two coincident clumps and world 3: at least one rank owns no points."""
    a = np.tile(np.array([[0.0, 0.0, 0.0]], np.float32), (30, 1))
    b = np.tile(np.array([[5.0, 5.0, 5.0]], np.float32), (30, 1))
    coords = np.concatenate([a, b])
    labels, core = run_sharded(coords, 0.2, 4, world=3)
    check_against_oracle(coords, 0.2, 4, labels, core)


# ---------------- tcg_cluster_multi: the sharded path behind the C ABI ----------------
@pytest.mark.gpu
@pytest.mark.parametrize("shards", [1, 2, 3, 5])
@pytest.mark.parametrize("case", ["blobs3d-2", "blobs3d-5", "blobs2d-4", "hacc-2", "hacc-20"])
def test_cluster_multi_matches_single_gpu(shards, case):
    """tcg_cluster_multi with `shards` shards on cuda:0 (the
    same device listed repeatedly: the full partition / halo / merge protocol
    through peer copies) equals tc_cluster: core flags, noise, core labels,
    counts; every border label valid (device border check)."""
    import torch

    import paper_2103_05162_b200 as tb
    from paper_2103_05162_b200 import Algorithm, Dataset

    if case.startswith("blobs3d"):
        ds, eps = Dataset.blobs(12, 4000, 3, 1.0, 0.12, 17), 0.09
    elif case.startswith("blobs2d"):
        ds, eps = Dataset.blobs(10, 5000, 2, 1.0, 0.1, 5), 0.03
    else:
        ds, eps = Dataset.hacc_like(400_000, seed=7), 0.042
    minpts = int(case.split("-")[1])
    want = tb.cluster(ds, eps, minpts, Algorithm.FDBSCAN)
    got = tb.cluster_multi(ds, eps, minpts, [0] * shards)
    assert np.array_equal(got.core_flags, want.core_flags)
    assert np.array_equal(got.labels == -1, want.labels == -1)
    cm = want.core_flags == 1
    assert np.array_equal(got.labels[cm], want.labels[cm])
    for k in ("cluster_count", "core_count", "noise_count"):
        assert got.stats[k] == want.stats[k], k
    x = torch.from_numpy(ds.coords()).cuda()
    bad = tb.api.first_bad_border(x, eps, torch.from_numpy(got.labels).cuda(),
                                  torch.from_numpy(got.core_flags).cuda())
    assert bad < 0


@pytest.mark.gpu
def test_cluster_multi_argument_errors():
    import paper_2103_05162_b200 as tb
    from paper_2103_05162_b200 import Algorithm, Dataset, Status, TreeclustError

    ds = Dataset.blobs(2, 100, 2, 1.0, 0.1, 1)
    for args in ((0.0, 5, [0]), (0.1, 1, [0]), (0.1, 5, [99]), (0.1, 5, [])):
        with pytest.raises(TreeclustError) as e:
            tb.cluster_multi(ds, *args)
        assert e.value.status == Status.INVALID_ARGUMENT, args
    with pytest.raises(TreeclustError) as e:
        tb.cluster_multi(ds, 0.1, 5, [0], Algorithm.BRUTEFORCE)
    assert e.value.status == Status.INVALID_ARGUMENT


# ---------------- the fused shard stages, directly ----------------
@pytest.mark.gpu
@pytest.mark.parametrize("dim", [2, 3])
def test_route_rows_and_counts(dim):
    """tcg_shard_route_device: every point lands in its owner's group exactly
    once (owner = bucketize(code, splitters, right=True)), rows carry the
    coordinates' bits, the global id and the code."""
    from paper_2103_05162_b200.shard import DeviceEngine

    rng = np.random.default_rng(dim)
    n = 50_000
    x = torch.from_numpy(rng.uniform(-3, 3, (n, dim)).astype(np.float32)).cuda()
    gid = torch.from_numpy(rng.permutation(n).astype(np.int64) + 10**9).cuda()
    eng = DeviceEngine("cuda:0")
    codes = eng.morton(x, x.min(0).values, x.max(0).values)
    splitters = torch.sort(codes[torch.randint(0, n, (5,), device="cuda")]).values
    rows, counts = eng.route(x, gid, codes, splitters)
    owner = torch.bucketize(codes, splitters, right=True)
    assert counts == torch.bincount(owner, minlength=6).tolist()
    rows = rows.cpu()
    start = 0
    for o, c in enumerate(counts):
        grp = rows[start:start + c]
        start += c
        g = grp[:, dim:dim + 2].contiguous().view(torch.int64).view(-1)
        sel = (owner == o).cpu()
        assert torch.equal(torch.sort(g).values, torch.sort(gid.cpu()[sel]).values)
        want = dict(zip(gid.cpu()[sel].tolist(), codes.cpu()[sel].tolist()))
        got_codes = grp[:, dim + 2:].contiguous().view(torch.int64).view(-1).tolist()
        assert all(want[a] == b for a, b in zip(g.tolist(), got_codes))
        pos = {v: i for i, v in enumerate(gid.cpu().tolist())}
        xs = x.cpu()[[pos[v] for v in g.tolist()]]
        assert torch.equal(grp[:, :dim].contiguous().view(torch.float32), xs)


@pytest.mark.gpu
def test_region_boxes_cover_and_near_peers():
    """tcg_shard_region_boxes_device covers every point with tight cell boxes;
    tcg_near_peers_device flags exactly the points within eps of a peer's
    boxes (against a brute-force fp64 check)."""
    from paper_2103_05162_b200.shard import DeviceEngine

    rng = np.random.default_rng(7)
    pts = np.concatenate([rng.normal(0, 0.3, (20_000, 3)), rng.uniform(-2, 2, (20_000, 3))])
    x = torch.from_numpy(pts.astype(np.float32)).cuda()
    eng = DeviceEngine("cuda:0")
    codes = eng.morton(x, x.min(0).values, x.max(0).values)
    boxes = eng.region_boxes(x, codes).cpu().numpy()
    assert 0 < len(boxes) <= 1 << 12
    p = x.cpu().numpy()
    inside = np.zeros(len(p), bool)
    for b in boxes:
        inside |= np.all((p >= b[:3]) & (p <= b[3:]), axis=1)
    assert inside.all()
    # two "peers": the boxes of two halves of another cloud
    q = rng.uniform(-2.5, 2.5, (3000, 3)).astype(np.float32)
    qx = torch.from_numpy(q).cuda()
    qc = eng.morton(qx, qx.min(0).values, qx.max(0).values)
    half = len(q) // 2
    b0 = eng.region_boxes(qx[:half].contiguous(), qc[:half].contiguous())
    b1 = eng.region_boxes(qx[half:].contiguous(), qc[half:].contiguous())
    ball = torch.cat([b0, b1])
    own = torch.cat([torch.full((b0.shape[0],), 2, dtype=torch.int32),
                     torch.full((b1.shape[0],), 5, dtype=torch.int32)]).cuda()
    eps = 0.05
    mask = eng.near_peers(x, eps, ball[:, :3], ball[:, 3:], own).cpu().numpy()
    e2 = np.float64(np.float32(eps)) ** 2
    pd = p.astype(np.float64)
    for bit, bx in ((2, b0.cpu().numpy()), (5, b1.cpu().numpy())):
        lo, hi = bx[None, :, :3].astype(np.float64), bx[None, :, 3:].astype(np.float64)
        want = np.zeros(len(p), bool)
        for c0 in range(0, len(p), 1000):
            pc = pd[c0:c0 + 1000, None, :]
            d = np.maximum(np.maximum(lo - pc, pc - hi), 0)
            want[c0:c0 + 1000] = ((d * d).sum(2) <= e2).any(1)
        assert np.array_equal(((mask >> bit) & 1).astype(bool), want)
    assert ((mask & ~((1 << 2) | (1 << 5))) == 0).all()


@pytest.mark.parametrize("fused", [False, True])
def test_sharded_all_ranks_empty(fused):
    """No points anywhere: no samples, no splitters; every rank still takes
    part in every collective and returns empty results."""
    coords = np.zeros((0, 3), np.float32)
    labels, core = run_sharded(coords, 0.1, 2, world=2, fused=fused)
    assert labels.shape == (0,) and core.shape == (0,)
