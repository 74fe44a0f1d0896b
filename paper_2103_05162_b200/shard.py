"""Morton-range sharded DBSCAN across GPUs.

One process per GPU; the collectives go through torch.distributed (NCCL on
GPUs, gloo in the CPU tests); every data-path stage runs in the C-ABI library
(`DeviceEngine`, tcg_*_device). Protocol, for eps and minpts:

1. global scene box: all-reduce MIN / MAX of the local bounds;
2. Morton codes against the global box; every rank all-gathers a sorted
   sample of its codes, the world picks world-1 splitters;
3. all-to-all: each point (coords + global id) moves to the rank owning its
   Morton range;
4. each rank describes its region by the boxes of runs of `block`
   consecutive own points in Morton order and all-gathers them; every rank
   sends each peer the own points within eps of one of that peer's boxes
   (all-to-all). Every point within eps of a peer-owned point is within eps of
   a box holding it, so the ghosts a rank receives contain every neighbour of
   its own points;
5. local set = own + ghosts, ordered by global id (so local minimum index ==
   global minimum id). Core flags of own points are exact (complete
   neighbourhoods); ghosts take their owner's flags (all-to-all of the flags of
   the points sent in step 4, same order);
6. local main pass with those flags (tcg_cluster_given_core_device);
7. every core point that is a ghost here or was exported as a ghost yields an
   edge (global id, global id of its local root); the edges are all-gathered
   and merged by a device union-find (min-index hooking, so representatives
   are global minimum ids) — the cluster representative is then the global
   minimum core id, exactly the 1-GPU label; own points are relabelled.

Steps 5-6 run on one local context (tcg_local_*: own + ghost points keyed by
global id, one tree for both passes, labels in global ids). minpts == 2
skips steps 5-6: every within-eps pair is a core-core union and
"core" is "has a neighbour", exact for own points, so one keyed local run
(tcg_cluster_keyed_device: own + ghost points, labels = global id of the
cluster's minimum-id point) replaces the flag exchange, the global-id sort and
the second tree build; step 7 takes its labels as they are.

Result per rank: (global ids, labels, core flags) of the points it owns.
"""
from __future__ import annotations

import ctypes as C

import torch
import torch.distributed as dist

from ._lib import TcClusterStats, lib
from .api import Status, TreeclustError


def _check(st, where):
    if st != 0:
        raise TreeclustError(st, where)


class DeviceEngine:
    """The product engine: device stages of the C ABI on CUDA tensors."""

    def __init__(self, device):
        self.device = torch.device(device)
        self.launches = 0  # kernels of this library launched through the engine
        self.record_stages = False  # keep the local run's stage times (last_stages)
        self.last_stages = None
        self.last_local_n = 0

    def _s(self):
        return C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def _count(self):
        self.launches += int(lib.tcg_last_launch_count())

    def morton(self, x, lo, hi):
        n, d = x.shape
        out = torch.empty(n, dtype=torch.int64, device=x.device)
        lo_h = (C.c_float * 3)(*[float(v) for v in lo.tolist()] + [0.0] * (3 - d))
        hi_h = (C.c_float * 3)(*[float(v) for v in hi.tolist()] + [0.0] * (3 - d))
        _check(lib.tcg_morton_codes_device(C.c_void_p(x.data_ptr()), n, d, lo_h, hi_h,
                                           C.c_void_p(out.data_ptr()), self._s()),
               "tcg_morton_codes_device")
        self._count()
        return out

    def near_boxes(self, x, eps, blo, bhi):
        n, d = x.shape
        mask = torch.empty(n, dtype=torch.uint8, device=x.device)
        if n == 0:
            return mask
        blo = blo.contiguous()
        bhi = bhi.contiguous()
        _check(lib.tcg_near_boxes_device(C.c_void_p(x.data_ptr()), n, d, C.c_float(eps),
                                         C.c_void_p(blo.data_ptr()), C.c_void_p(bhi.data_ptr()),
                                         blo.shape[0], C.c_void_p(mask.data_ptr()), self._s()),
               "tcg_near_boxes_device")
        self._count()
        return mask

    def core_flags(self, x, eps, minpts):
        n, d = x.shape
        core = torch.empty(n, dtype=torch.uint8, device=x.device)
        _check(lib.tcg_core_flags_device(C.c_void_p(x.data_ptr()), n, d, C.c_float(eps),
                                         int(minpts), C.c_void_p(core.data_ptr()), self._s()),
               "tcg_core_flags_device")
        self._count()
        return core

    def cluster_given_core(self, x, eps, core):
        n, d = x.shape
        labels = torch.empty(n, dtype=torch.int32, device=x.device)
        core_out = torch.empty(n, dtype=torch.uint8, device=x.device)
        core = core.contiguous()
        _check(lib.tcg_cluster_given_core_device(C.c_void_p(x.data_ptr()), n, d, C.c_float(eps),
                                                 C.c_void_p(core.data_ptr()),
                                                 C.c_void_p(labels.data_ptr()),
                                                 C.c_void_p(core_out.data_ptr()), self._s(),
                                                 None),
               "tcg_cluster_given_core_device")
        self._count()
        return labels

    def cluster_keyed(self, x, keys, eps, minpts):
        """FDBSCAN of x with labels = key of the cluster's minimum-key core."""
        n, d = x.shape
        labels = torch.empty(n, dtype=torch.int32, device=x.device)
        core = torch.empty(n, dtype=torch.uint8, device=x.device)
        keys = keys.contiguous()
        st = TcClusterStats() if self.record_stages else None  # stats: stage events kept
        _check(lib.tcg_cluster_keyed_device(C.c_void_p(x.data_ptr()), C.c_void_p(keys.data_ptr()),
                                            n, d, C.c_float(eps), int(minpts),
                                            C.c_void_p(labels.data_ptr()),
                                            C.c_void_p(core.data_ptr()), self._s(),
                                            C.byref(st) if st is not None else None),
               "tcg_cluster_keyed_device")
        self._count()
        if self.record_stages:  # (reading the stage events waits for the run)
            from .api import last_stage_ms
            self.last_stages = last_stage_ms()
            self.last_local_n = n
        return labels, core

    def local(self, x, keys, eps):
        """A LocalContext over (x, keys): one tree for the core and main passes."""
        return LocalContext(self, x, keys, eps)

    def route(self, x, gid, codes, splitters):
        """Rows (dim + 4 int32 words: coords, gid, code) grouped by owner, and
        the per-owner counts (host list)."""
        n, d = x.shape
        world = splitters.shape[0] + 1
        rows = torch.empty((n, d + 4), dtype=torch.int32, device=x.device)
        counts = torch.empty(world, dtype=torch.int64, device=x.device)
        sp = splitters.contiguous()
        _check(lib.tcg_shard_route_device(C.c_void_p(x.data_ptr()), C.c_void_p(gid.data_ptr()),
                                          C.c_void_p(codes.data_ptr()), n, d,
                                          C.c_void_p(sp.data_ptr()), sp.shape[0],
                                          C.c_void_p(rows.data_ptr()),
                                          C.c_void_p(counts.data_ptr()), self._s()),
               "tcg_shard_route_device")
        self._count()
        return rows, counts.tolist()

    def unpack(self, rows, dim, with_codes):
        """(coords [n, dim] f32, gid [n] i64, codes [n] i64 or None) from rows."""
        n = rows.shape[0]
        x = torch.empty((n, dim), dtype=torch.float32, device=rows.device)
        g = torch.empty(n, dtype=torch.int64, device=rows.device)
        c = torch.empty(n, dtype=torch.int64, device=rows.device) if with_codes else None
        rows = rows.contiguous()
        _check(lib.tcg_shard_unpack_rows_device(C.c_void_p(rows.data_ptr()), n, dim,
                                                C.c_void_p(x.data_ptr()), C.c_void_p(g.data_ptr()),
                                                C.c_void_p(c.data_ptr()) if c is not None else None,
                                                self._s()),
               "tcg_shard_unpack_rows_device")
        self._count()
        return x, g, c

    def region_boxes(self, x, codes):
        """(k, 2*dim) float32 boxes covering the points (Morton-prefix cells)."""
        n, d = x.shape
        cap = 1 << 12
        lo = torch.empty((cap, d), dtype=torch.float32, device=x.device)
        hi = torch.empty((cap, d), dtype=torch.float32, device=x.device)
        cnt = torch.zeros(1, dtype=torch.int64, device=x.device)
        _check(lib.tcg_shard_region_boxes_device(C.c_void_p(x.data_ptr()),
                                                 C.c_void_p(codes.data_ptr()), n, d,
                                                 C.c_void_p(lo.data_ptr()), C.c_void_p(hi.data_ptr()),
                                                 C.c_void_p(cnt.data_ptr()), self._s()),
               "tcg_shard_region_boxes_device")
        self._count()
        k = int(cnt.item())
        return torch.cat([lo[:k], hi[:k]], 1)

    def near_peers(self, x, eps, blo, bhi, owner):
        """Bit j of mask[i]: point i lies within eps of a box of peer j."""
        n, d = x.shape
        mask = torch.zeros(n, dtype=torch.int64, device=x.device)
        if n == 0:
            return mask
        blo, bhi = blo.contiguous(), bhi.contiguous()
        owner = owner.to(device=x.device, dtype=torch.int32).contiguous()
        _check(lib.tcg_near_peers_device(C.c_void_p(x.data_ptr()), n, d, C.c_float(eps),
                                         C.c_void_p(blo.data_ptr()), C.c_void_p(bhi.data_ptr()),
                                         C.c_void_p(owner.data_ptr()), blo.shape[0],
                                         C.c_void_p(mask.data_ptr()), self._s()),
               "tcg_near_peers_device")
        self._count()
        return mask

    def union_edges(self, edges, n):
        root = torch.empty(n, dtype=torch.int32, device=self.device)
        edges = edges.to(device=self.device, dtype=torch.int32).contiguous()
        _check(lib.tcg_union_edges_device(C.c_void_p(edges.data_ptr()), edges.shape[0], int(n),
                                          C.c_void_p(root.data_ptr()), self._s()),
               "tcg_union_edges_device")
        self._count()
        return root


class LocalContext:
    """tcg_local_*: the local (own + ghost) point set of a shard, its BVH built
    once; core_flags() then cluster() with the owners' ghost flags. Labels
    are keys (global ids)."""

    def __init__(self, engine, x, keys, eps):
        self.engine = engine
        self.x = x.contiguous()
        self.keys = keys.contiguous()
        self.n = x.shape[0]
        h = C.c_void_p()
        _check(lib.tcg_local_create(C.c_void_p(self.x.data_ptr()), C.c_void_p(self.keys.data_ptr()),
                                    self.n, x.shape[1], C.c_float(eps), engine._s(), C.byref(h)),
               "tcg_local_create")
        engine._count()
        self.h = h

    def core_flags(self, minpts):
        core = torch.empty(self.n, dtype=torch.uint8, device=self.x.device)
        _check(lib.tcg_local_core_flags(self.h, int(minpts), C.c_void_p(core.data_ptr())),
               "tcg_local_core_flags")
        self.engine._count()
        return core

    def cluster(self, core):
        core = core.contiguous()
        labels = torch.empty(self.n, dtype=torch.int32, device=self.x.device)
        core_out = torch.empty(self.n, dtype=torch.uint8, device=self.x.device)
        _check(lib.tcg_local_cluster(self.h, C.c_void_p(core.data_ptr()),
                                     C.c_void_p(labels.data_ptr()), C.c_void_p(core_out.data_ptr())),
               "tcg_local_cluster")
        self.engine._count()
        return labels

    def close(self):
        if self.h is not None and self.h.value:
            lib.tcg_local_free(self.h)
        self.h = None

    def __del__(self):
        self.close()


# ---------------------------------------------------------------------------
# collectives (moved through host memory when the backend is gloo)
# ---------------------------------------------------------------------------
def _host_collectives(group):
    return dist.get_backend(group) == "gloo"


def _to_comm(t, group):
    return t.cpu() if _host_collectives(group) else t


def _all_reduce(t, op, group):
    c = _to_comm(t, group)
    dist.all_reduce(c, op=op, group=group)
    return c.to(t.device)


def _all_gather_var(t, group):
    """All-gather tensors whose first dimension differs per rank."""
    world = dist.get_world_size(group)
    dev = t.device
    c = _to_comm(t.contiguous(), group)
    n = torch.tensor([c.shape[0]], dtype=torch.int64, device=c.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    mx = max(sizes) if sizes else 0
    pad = torch.zeros((mx,) + tuple(c.shape[1:]), dtype=c.dtype, device=c.device)
    pad[: c.shape[0]] = c
    outs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(outs, pad, group=group)
    return [o[:s].to(dev) for o, s in zip(outs, sizes)]


def _all_to_all(t, send_counts, group):
    """Variable all-to-all along dim 0; send_counts[j] rows go to rank j."""
    world = dist.get_world_size(group)
    dev = t.device
    sc = torch.tensor(send_counts, dtype=torch.int64)
    rc = torch.empty(world, dtype=torch.int64)
    if _host_collectives(group):
        dist.all_to_all_single(rc, sc, group=group)
    else:
        rcd = torch.empty(world, dtype=torch.int64, device=dev)
        dist.all_to_all_single(rcd, sc.to(dev), group=group)
        rc = rcd.cpu()
    recv = [int(v) for v in rc.tolist()]
    c = _to_comm(t.contiguous(), group)
    out = torch.empty((sum(recv),) + tuple(c.shape[1:]), dtype=c.dtype, device=c.device)
    dist.all_to_all_single(out, c, recv, list(send_counts), group=group)
    return out.to(dev), recv


def _merge_edges(edges, root_gid, engine, group):
    """Global merge: all-gather the (global id, local root id) edges, union
    them (min-id hooking, so the global representative is the minimum id),
    and map this rank's local roots to global representatives."""
    all_edges = torch.cat(_all_gather_var(edges, group))
    if all_edges.shape[0]:
        uniq, comp = torch.unique(all_edges.view(-1), return_inverse=True)
        root = engine.union_edges(comp.view(-1, 2), uniq.shape[0]).to(torch.int64)
        rep = uniq[root]  # compact ids are ordered like global ids: min id wins
        last = uniq.shape[0] - 1
        pos = torch.searchsorted(uniq, root_gid.clamp(min=0))
        hit = (root_gid >= 0) & (pos <= last) & (uniq[pos.clamp(max=last)] == root_gid)
        root_gid = torch.where(hit, rep[pos.clamp(max=last)], root_gid)
    return root_gid


def _unpack(rows, dim):
    """(coords f32 [n, dim], gid i64 [n]) from int32 rows [n, dim + 2]. Copies
    the column slices (an empty slice keeps a storage offset that a dtype view
    rejects)."""
    x = rows[:, :dim].clone(memory_format=torch.contiguous_format).view(torch.float32)
    g = rows[:, dim:].clone(memory_format=torch.contiguous_format).view(torch.int64).view(-1)
    return x, g


class _StageMarks:
    """Per-stage CUDA-event times of cluster_sharded (TCB_SHARD_TIMING=1)."""

    def __init__(self, dev):
        import os
        self.on = os.environ.get("TCB_SHARD_TIMING") == "1" and dev.type == "cuda"
        self.ev = []
        if self.on:
            self.mark("1")

    def mark(self, name):
        if self.on:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            self.ev.append((name, e))

    def report(self, rank):
        if not self.on:
            return
        torch.cuda.synchronize()
        parts = [f"{a}:{ea.elapsed_time(eb):.2f}" for (a, ea), (_, eb) in zip(self.ev, self.ev[1:])]
        print(f"[shard rank {rank}] stage ms " + " ".join(parts), flush=True)


# ---------------------------------------------------------------------------
def cluster_sharded(x, gid, eps, minpts, engine, group=None, block=2048, samples=4096,
                    force_exchange=None):
    """Clusters the union of every rank's (x, gid) points.

    x: (n_local, dim) float32 tensor on the engine's device; gid: (n_local,)
    int64 global ids (unique across ranks). Returns (own_gid, labels, core)
    for the points this rank owns after the Morton-range redistribution;
    labels are global ids of the cluster representative (minimum core id), -1
    for noise. Identical to the single-GPU result on the concatenated input.

    force_exchange (default: TCB_SHARD_FORCE_EXCHANGE=1): run the
    multi-rank protocol even on a single rank (sampling, the all-to-all
    redistribution to itself, the halo exchange with no peers), so that one
    GPU exercises the backend's collectives exactly as N ranks issue them.
    """
    if force_exchange is None:
        import os
        force_exchange = os.environ.get("TCB_SHARD_FORCE_EXCHANGE") == "1"
    if not (eps > 0) or minpts < 2:
        raise TreeclustError(Status.INVALID_ARGUMENT, "cluster_sharded")
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = x.device
    n, dim = x.shape
    marks = _StageMarks(dev)
    single = world == 1 and not force_exchange  # no exchange at all

    # 1. global scene box
    if n:
        lo = x.min(0).values
        hi = x.max(0).values
    else:
        lo = torch.full((dim,), float("inf"), device=dev)
        hi = torch.full((dim,), float("-inf"), device=dev)
    lo = _all_reduce(lo.clone(), dist.ReduceOp.MIN, group)
    hi = _all_reduce(hi.clone(), dist.ReduceOp.MAX, group)

    marks.mark("2")
    # 2. codes and splitters
    codes = engine.morton(x, lo, hi) if n else torch.empty(0, dtype=torch.int64, device=dev)
    k = min(n, samples)
    if k and not single:
        # a pseudo-random subsample (fixed seed) stands in for the local
        # distribution; only load balance depends on it, never correctness
        g = torch.Generator(device=dev)
        g.manual_seed(1234 + rank)
        sample = codes[torch.randint(0, n, (k,), device=dev, generator=g)]
    else:
        sample = codes[:0]
    allsamp = torch.sort(torch.cat(_all_gather_var(sample, group))).values
    m = allsamp.shape[0]
    if not single and m:
        q = torch.tensor([(j * m) // world for j in range(1, world)], dtype=torch.int64, device=dev)
        splitters = allsamp[q.clamp(max=m - 1)]
    else:
        splitters = torch.empty(0, dtype=torch.int64, device=dev)
    owner = None if hasattr(engine, "route") else torch.bucketize(codes, splitters, right=True)

    marks.mark("3")
    # 3. redistribution by Morton range (the codes travel along: step 4
    #    orders the own points by them)
    if single:
        own_x, own_gid, own_codes = x.contiguous(), gid, codes
    else:
        if hasattr(engine, "route"):  # one device pass: owners + packed rows in owner order
            payload, counts = engine.route(x.contiguous(), gid.contiguous(), codes, splitters)
            counts = counts + [0] * (world - len(counts))  # (no splitters: all to rank 0)
        else:
            order = torch.argsort(owner, stable=True)
            counts = torch.bincount(owner, minlength=world).tolist() if n else [0] * world
            payload = torch.cat([x[order].view(torch.int32),
                                 gid[order].view(torch.int32).view(-1, 2),
                                 codes[order].view(torch.int32).view(-1, 2)], 1)
        recv, _ = _all_to_all(payload, counts, group)
        if hasattr(engine, "unpack"):
            own_x, own_gid, own_codes = engine.unpack(recv, dim, True)
        else:
            own_x, own_gid = _unpack(recv[:, :dim + 2], dim)
            own_codes = recv[:, dim + 2:].clone(memory_format=torch.contiguous_format).view(
                torch.int64).view(-1)
    n_own = own_x.shape[0]

    marks.mark("4")
    # 4. region boxes and the eps halo (a single rank has no peers)
    if single:
        ghost_x = own_x[:0]
        ghost_gid = own_gid[:0]
        send_idx = torch.empty(0, dtype=torch.int64, device=dev)
        send_counts = [0]
    elif n_own and hasattr(engine, "region_boxes"):  # Morton-prefix cell boxes, no sort
        boxes = engine.region_boxes(own_x, own_codes)
    elif n_own:
        perm = torch.argsort(own_codes)
        xs = own_x[perm]
        nb = (n_own + block - 1) // block
        padn = nb * block - n_own
        big = torch.full((padn, dim), float("inf"), device=dev)
        blo = torch.cat([xs, big]).view(nb, block, dim).min(1).values
        bhi = torch.cat([xs, -big]).view(nb, block, dim).max(1).values
        boxes = torch.cat([blo, bhi], 1)
    else:
        boxes = torch.empty((0, 2 * dim), dtype=torch.float32, device=dev)
    if not single:
        peer_boxes = _all_gather_var(boxes, group)
        send_idx, send_counts = [], []
        if hasattr(engine, "near_peers") and world <= 64:
            # one traversal per own point over every peer's boxes (bit j = peer j)
            others = [j for j in range(world) if j != rank and peer_boxes[j].shape[0]]
            if n_own and others:
                ball = torch.cat([peer_boxes[j] for j in others])
                bown = torch.cat([torch.full((peer_boxes[j].shape[0],), j, dtype=torch.int32,
                                             device=dev) for j in others])
                pmask = engine.near_peers(own_x, eps, ball[:, :dim], ball[:, dim:], bown)
            for j in range(world):
                if j not in others or n_own == 0:
                    send_counts.append(0)
                    continue
                idx = torch.nonzero((pmask >> j) & 1, as_tuple=False).view(-1)
                send_idx.append(idx)
                send_counts.append(int(idx.shape[0]))
        else:
            for j in range(world):
                if j == rank or n_own == 0 or peer_boxes[j].shape[0] == 0:
                    send_counts.append(0)
                    continue
                pb = peer_boxes[j]
                mask = engine.near_boxes(own_x, eps, pb[:, :dim], pb[:, dim:])
                idx = torch.nonzero(mask, as_tuple=False).view(-1)
                send_idx.append(idx)
                send_counts.append(int(idx.shape[0]))
        send_idx = torch.cat(send_idx) if send_idx else torch.empty(0, dtype=torch.int64, device=dev)
        halo_payload = torch.cat([own_x[send_idx].view(torch.int32),
                                  own_gid[send_idx].view(torch.int32).view(-1, 2)], 1)
        ghost, _ = _all_to_all(halo_payload, send_counts, group)
        ghost_x, ghost_gid = _unpack(ghost, dim)

    marks.mark("5")
    lgid = torch.cat([own_gid, ghost_gid])
    # The path below must be the same on every rank (each issues a different
    # sequence of collectives): decide it from all-reduced facts only.
    gmax = torch.tensor([int(lgid.max().item()) if lgid.numel() else -1], dtype=torch.int64,
                        device=dev)
    fits = int(_all_reduce(gmax, dist.ReduceOp.MAX, group).item()) < 2**31
    e64 = torch.empty(0, dtype=torch.int64, device=dev)
    no_edges = torch.empty((0, 2), dtype=torch.int64, device=dev)
    if minpts == 2 and hasattr(engine, "cluster_keyed") and fits:
        # minpts == 2 (friends-of-friends): every within-eps pair is a
        # core-core union and core == "has a neighbour", exact for own points
        # (complete neighbourhoods); no flag exchange is needed. One local run
        # keyed by global id labels the own + ghost set in global ids.
        lx = torch.cat([own_x, ghost_x]).contiguous()
        if lx.shape[0] == 0:
            _merge_edges(no_edges, e64, engine, group)
            return e64, e64.to(torch.int32), e64.to(torch.uint8)
        lab, lcore = engine.cluster_keyed(lx, lgid.to(torch.int32), eps, 2)
        lab = lab.to(torch.int64)
        marks.mark("7")
        own_lab, own_core = lab[:n_own], lcore[:n_own]
        g_lab = lab[n_own:]
        e_lab = own_lab[send_idx]
        gsel, esel = g_lab >= 0, e_lab >= 0
        edges = torch.cat([torch.stack([ghost_gid[gsel], g_lab[gsel]], 1),
                           torch.stack([own_gid[send_idx][esel], e_lab[esel]], 1)])
        root_gid = _merge_edges(edges, own_lab, engine, group)
        marks.mark("end")
        marks.report(rank)
        return own_gid, root_gid, own_core

    if hasattr(engine, "local") and fits:
        # 5. one local context (own + ghost points, keyed by global id): exact
        #    own flags, owners' flags for the ghosts, then the main pass on the
        #    same tree; labels come out as global ids
        lx = torch.cat([own_x, ghost_x]).contiguous()
        nl = lx.shape[0]
        if nl == 0:  # still part of the ghost-flag exchange and the merge
            _all_to_all(torch.empty((0, 1), dtype=torch.uint8, device=dev), [0] * world, group)
            _merge_edges(no_edges, e64, engine, group)
            return e64, e64.to(torch.int32), e64.to(torch.uint8)
        ctx = engine.local(lx, lgid.to(torch.int32), eps)
        local_core = ctx.core_flags(minpts)
        own_core = local_core[:n_own]
        ghost_core, _ = _all_to_all(own_core[send_idx].view(-1, 1), send_counts, group)
        core = local_core.clone()
        core[n_own:] = ghost_core.view(-1)
        marks.mark("6")
        lab = ctx.cluster(core).to(torch.int64)
        ctx.close()
        marks.mark("7")
        # 7. cross-shard edges: every core that is a ghost here or was sent
        #    away as one, with its local label (a global id)
        touched = torch.zeros(nl, dtype=torch.bool, device=dev)
        touched[n_own:] = True
        touched[send_idx] = True
        sel = (core.bool() & touched).nonzero(as_tuple=False).view(-1)
        edges = torch.stack([lgid[sel], lab[sel]], 1)
        root_gid = _merge_edges(edges, lab[:n_own], engine, group)
        marks.mark("end")
        marks.report(rank)
        return own_gid, root_gid, own_core

    # 5. local set ordered by global id; exact own flags; owners' ghost flags
    lx = torch.cat([own_x, ghost_x])
    nl = lx.shape[0]
    if nl == 0:  # still part of the ghost-flag exchange and the merge
        _all_to_all(torch.empty((0, 1), dtype=torch.uint8, device=dev), [0] * world, group)
        _merge_edges(no_edges, e64, engine, group)
        return e64, e64.to(torch.int32), e64.to(torch.uint8)
    lorder = torch.argsort(lgid)
    lx = lx[lorder].contiguous()
    lgid = lgid[lorder]
    inv = torch.empty_like(lorder)
    inv[lorder] = torch.arange(lorder.shape[0], device=dev)
    own_pos = inv[:n_own]
    ghost_pos = inv[n_own:]
    local_core = engine.core_flags(lx, eps, minpts)
    own_core = local_core[own_pos]
    ghost_core, _ = _all_to_all(own_core[send_idx].view(-1, 1), send_counts, group)
    core = local_core.clone()
    core[ghost_pos] = ghost_core.view(-1)

    marks.mark("6")
    # 6. local main pass with the true flags
    lab = engine.cluster_given_core(lx, eps, core).to(torch.int64)

    marks.mark("7")
    # 7. cross-shard edges (global ids) and the global merge
    exported = torch.zeros(nl, dtype=torch.bool, device=dev)
    exported[own_pos[send_idx]] = True
    is_ghost = torch.zeros(nl, dtype=torch.bool, device=dev)
    is_ghost[ghost_pos] = True
    sel = (core.bool() & (is_ghost | exported)).nonzero(as_tuple=False).view(-1)
    edges = torch.stack([lgid[sel], lgid[lab[sel]]], 1)
    own_lab = lab[own_pos]
    root_gid = torch.where(own_lab >= 0, lgid[own_lab.clamp(min=0)], torch.full_like(own_lab, -1))
    root_gid = _merge_edges(edges, root_gid, engine, group)
    marks.mark("end")
    marks.report(rank)
    return own_gid, root_gid, own_core
