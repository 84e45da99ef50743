"""Multi-GPU AMS-sort: one process per GPU over torch.distributed.

PE layout: logical PEs are fixed; PE i lives on rank
``i * G // p``.  The first level's single group spans every rank:

    sample positions    every rank computes the whole group's draw
                        (C++ restatement of draw_sample, ams.py:157-175), so
                        every rank also knows how many sample elements each
                        rank holds
    sample all-gather   local sample elements -> full sample on every rank
                        (the all-gather of fastsort.py:84-93 / gossip_merge)
    splitters           replicated, identical on every rank
    classify            local PEs; one all-gather of the histograms and the
                        key range (the allreduce of ams.py:236-237, which
                        deliver_simple also needs)
    plan                replicated (optimal_group_plan, ams.py:238)
    scatter = exchange  every rank writes its PEs' pieces straight into the
                        receive buffers of the groups' owner GPUs (peer
                        pointers over NVLink, mapped with CUDA IPC), at the
                        offsets of Network.exchange (simnet.py:294-335):
                        group g's buffer is its source PEs' pieces in PE order
                        (ams.py:252-256) — no send buffer, no copy kernel

Groups of the first level must not straddle ranks (``group_counts[0] % G
== 0``), so every later level and the final sort are rank-local.

The device work goes through an ``ops`` object (:class:`CudaOps` on GPUs);
the collectives are torch.distributed calls on the ops' tensors, so the same
orchestration runs over NCCL with CUDA tensors and over gloo with CPU
tensors (tests/test_dist_gloo.py drives it with oracle-backed test ops).
"""

from __future__ import annotations

import math

import numpy as np
import torch
import torch.distributed as dist

from . import _lib as L
from .engine import (SCHEMES, LevelRecord, check_out, key_kind_of, level_targets, load_budget,
                     native_params, run_records)
from .params import as_params, as_seed


class _DeviceView:
    """A library-owned device buffer exposed to torch without a copy."""

    def __init__(self, addr: int, n: int, device_index: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i8", "data": (addr, False),
                                         "version": 3}
        self.device_index = device_index


class CudaOps:
    """Device work of one rank: the C ABI on this rank's GPU."""

    def __init__(self, sorter):
        self.sorter = sorter
        self.ctx = sorter.ctx
        self.device = sorter.device
        self._caps = None     # replicated receive-buffer capacity (keys) of every rank
        self._peers = None    # per rank: (keys address, values address) as mapped here
        self._vals = None

    # buffers -------------------------------------------------------------
    def empty(self, n, dtype=torch.int64):
        # +2: bulk tile loads cover whole 16-byte units past a segment end
        return torch.empty(max(n, 1) + 2, dtype=dtype, device=self.device)

    def workspace(self, n, with_vals):
        return self.sorter.workspace(n, with_vals)

    # steps ---------------------------------------------------------------
    def sample(self, src, kind, idx, gpos, out_keys, out_pos):
        self.ctx.level_sample(src, kind, idx, gpos, out_keys, out_pos)

    def splitters(self, s_keys, s_pos, soff, nb):
        self.ctx.level_splitters(s_keys, s_pos, soff, nb)

    def classify(self, src, kind, offs, sizes, seg_group, posbase, nb_stride, track_minmax, stable):
        return self.ctx.level_classify(src, kind, offs, sizes, seg_group, posbase, nb_stride,
                                       track_minmax, stable)

    def get_minmax(self):
        return self.ctx.get_minmax()

    def set_minmax(self, lo, hi):
        self.ctx.set_minmax(lo, hi)

    def scatter(self, src, src_v, kind, dst, dst_v, r, bnd, dst_start, child_first, child_count,
                bucket_major=False):
        self.ctx.level_scatter(src, src_v, kind, dst, dst_v, r, bnd, dst_start, child_first,
                               child_count, bucket_major=bucket_major)

    def exchange(self, src, src_v, kind, need, cell_base, bucket_dst, r, bnd, child_first,
                 child_count, group=None):
        """Level 1 across the GPUs: make every rank's receive buffer hold at
        least need[rank] keys, map the peers' buffers, and scatter this
        rank's pieces straight into them (ams_level_scatter_peers).  Returns
        this rank's receive buffers (keys, values) as tensors."""
        world = len(need)
        rank = dist.get_rank(group) if world > 1 else 0
        with_vals = src_v is not None
        # Capacities follow one deterministic rule on every rank, so a rank
        # knows without asking whether any peer re-allocated.
        caps = [max(int(x), 1) for x in need]
        grow = self._caps is None or self._vals != with_vals or any(
            c > old for c, old in zip(caps, self._caps))
        if grow:
            caps = [max(c + c // 4, old) if self._caps else c + c // 4
                    for c, old in zip(caps, self._caps or caps)]
        cap = (self._caps if not grow else caps)[rank]
        kp, kh, _ = self.ctx.peer_buffer(0, 8 * (cap + 2))
        vp, vh = 0, b""
        if with_vals:
            vp, vh, _ = self.ctx.peer_buffer(1, 8 * (cap + 2))
        if grow:
            if world > 1:
                torch.cuda.current_stream(self.device).synchronize()
                got = [None] * world
                dist.all_gather_object(got, (kh, vh), group=group)
                self.ctx.peer_close_all()
                self._peers = [(kp, vp) if k == rank else
                               (self.ctx.peer_open(h[0]), self.ctx.peer_open(h[1]) if with_vals else 0)
                               for k, h in enumerate(got)]
            else:
                self._peers = [(kp, vp)]
            self._caps, self._vals = caps, with_vals
        if world > 1:  # receivers are done with their buffers (previous sort's later levels)
            torch.cuda.current_stream(self.device).synchronize()
            dist.barrier(group=group)
        self.ctx.level_scatter_peers(src, src_v, kind, [q[0] for q in self._peers],
                                     [q[1] for q in self._peers] if with_vals else None,
                                     bucket_dst, cell_base, r, bnd, child_first, child_count)
        if world > 1:  # every piece has landed before anyone reads
            torch.cuda.current_stream(self.device).synchronize()
            dist.barrier(group=group)
        n = int(need[rank])
        recv = torch.as_tensor(_DeviceView(kp, cap + 2, self.device.index), device=self.device)
        recv_v = (torch.as_tensor(_DeviceView(vp, cap + 2, self.device.index), device=self.device)
                  if with_vals else None)
        return recv, recv_v

    def final_sort(self, src, src_v, tmp, tmp_v, out, out_v, kind, offs, sizes):
        self.ctx.final_sort(src, src_v, tmp, tmp_v, out, out_v, kind, offs, sizes)

    def iota(self, dst, n, start):
        self.ctx.fill_iota(dst, n, start)

    def copy_ranges(self, ranges, src, dst, src_v, dst_v):
        self.ctx.copy_ranges(ranges, src, dst, src_v, dst_v)

    def run_from(self, src, src_v, params, a, master, stream_id, kind, scheme, level_base,
                 init_groups, pe_base, local_sizes, out, out_vals):
        """The levels from `level_base` on and the final sort of this rank's
        PEs: ams_sort_run continuing on the context that ran level 1 (it
        holds the groups' key bounds).  Returns (final PE sizes, records)."""
        prm = native_params(params, master, stream_id, kind, True, SCHEMES[scheme], False,
                            oversampling=a, level_base=level_base, init_groups=init_groups,
                            pe_base=pe_base)
        n = int(np.asarray(local_sizes, dtype=np.uint64).sum())
        final_sizes, _ = self.ctx.sort_run(prm, local_sizes, src if n else None,
                                           src_v if n else None, out if n else None,
                                           out_vals if (n and out_vals is not None) else None)
        return final_sizes, run_records(self.ctx, self.ctx.run_id(), tuple(params.group_counts),
                                        params.per_level_imbalance(), first_level=level_base)

    def final_sort_buckets(self, src, tmp, out, kind, bk_off, bk_len, bk_group, bk_bucket):
        self.ctx.final_sort_buckets(src, tmp, out, kind, bk_off, bk_len, bk_group, bk_bucket)


def _u64_to_i64(x: int) -> int:
    return x - (1 << 64) if x >= (1 << 63) else x


def level1_cell_base(hist: np.ndarray, bnd: np.ndarray, rank: int, world: int, pl: int,
                     bucket_major: bool):
    """Destination of every (local source PE, bucket) run of level 1.

    ``hist`` is the (p, nb) histogram of all PEs, ``bnd`` the plan's group
    boundaries; group g lives on rank g // (r / world) and its buffer there
    starts after the rank's earlier groups.  In the (g(b), j, b) order of
    deliver_simple (SURVEY §8 layout contract step 5) run (j, b) starts at
    start(g) + sum_{j' < j} piece(j', g) + sum_{b' in [B_g, b)} H[j][b'];
    bucket-major (keys-only last level) at start(g) + sum_{b' in [B_g, b)}
    total(b') + sum_{j' < j} H[j'][b].  Returns (cell_base[pl, nb] for this
    rank's PEs, bucket -> owner rank, keys each rank receives)."""
    p, nb = hist.shape
    r = len(bnd) - 1
    gpr = r // world
    H = hist.astype(np.int64)
    g_of_b = np.searchsorted(bnd, np.arange(nb), side="right") - 1
    owner = (g_of_b // gpr).astype(np.int32)
    tot_b = H.sum(axis=0)
    m_g = np.array([tot_b[bnd[g]:bnd[g + 1]].sum() for g in range(r)], np.int64)
    g_start = np.zeros(r, np.int64)          # start of group g in its owner's buffer
    for k in range(world):
        gs = np.arange(k * gpr, (k + 1) * gpr)
        g_start[gs] = np.concatenate([[0], np.cumsum(m_g[gs])[:-1]])
    need = np.array([m_g[k * gpr:(k + 1) * gpr].sum() for k in range(world)], np.int64)
    base = np.zeros((pl, nb), np.int64)
    mine = slice(rank * pl, (rank + 1) * pl)
    for g in range(r):
        b0, b1 = int(bnd[g]), int(bnd[g + 1])
        if b1 == b0:
            continue
        blk = H[:, b0:b1]                                   # (p, buckets of g)
        if bucket_major:
            col = np.concatenate([[0], np.cumsum(blk.sum(axis=0))[:-1]])       # earlier buckets
            above = np.cumsum(blk, axis=0) - blk                                # earlier PEs, same bucket
            base[:, b0:b1] = g_start[g] + col[None, :] + above[mine]
        else:
            piece = blk.sum(axis=1)
            before_j = np.concatenate([[0], np.cumsum(piece)[:-1]])             # earlier source PEs
            within = np.cumsum(blk, axis=1) - blk                               # earlier buckets of j
            base[:, b0:b1] = g_start[g] + before_j[mine][:, None] + within[mine]
    return base.astype(np.uint64), owner, need


def sort_distributed(keys: torch.Tensor, pe_sizes_local, params, seed, ops, vals=None, out=None,
                     out_vals=None, key_kind=None, group=None, scheme: str = "simple"):
    """Sort this rank's PEs as part of one global ams_sort(scheme).

    Level 1 (the group of all PEs) runs here across the ranks; under a
    non-simple scheme (delivery.py:188-455) its delivery is the simple
    exchange followed by a rank-local relayout (the members of a subgroup
    live on one rank), with origin tags travelling as the values to break
    key ties from level 2 on.  The later levels and the final sort are
    rank-local: one ``ops.run_from`` call (``ams_sort_run`` continuing at
    level 2 on the GPU).  User payloads are carried under the simple scheme
    only.

    ``keys`` holds this rank's PEs (PE-major), ``pe_sizes_local`` their
    sizes; PE ids are rank-major (rank k owns PEs [k*p/G, (k+1)*p/G)).
    Returns (sorted local keys, vals, local per-PE sizes, level records); the
    rank-ordered concatenation of the outputs is the global sort."""
    if scheme not in SCHEMES:
        raise ValueError(f"unknown delivery scheme {scheme!r}; supported: {tuple(SCHEMES)}")
    det = scheme != "simple"
    if det and vals is not None:
        raise ValueError("the multi-GPU driver carries payloads under the simple delivery scheme only "
                         f"(origin tags travel as the values under {scheme!r})")
    params = as_params(params)
    master, stream_id = as_seed(seed)
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    kind = key_kind_of(keys, key_kind)
    local_sizes = np.asarray(pe_sizes_local, dtype=np.uint64)
    pl = len(local_sizes)
    p = pl * world
    params.validate_for(p)                                           # ams.py:276
    r1 = params.group_counts[0]
    if r1 % world:
        raise ValueError(f"first-level group count {r1} must be a multiple of the {world} ranks")
    dev = keys.device
    # Global PE sizes (every rank learns all of them).
    ls = torch.tensor(local_sizes.astype(np.int64), device=dev)
    gsz = [torch.zeros_like(ls) for _ in range(world)]
    dist.all_gather(gsz, ls, group=group)
    sizes = np.concatenate([g.cpu().numpy() for g in gsz]).astype(np.uint64)
    n = int(sizes.sum())
    n_local = int(local_sizes.sum())
    pe_lo = rank * pl
    a = params.oversampling_for(n)                                   # ams.py:278-280
    eps_l = params.per_level_imbalance()
    b = params.overpartition
    k_levels = len(params.group_counts)
    levels = []

    # ---------------- level 1: one group over all ranks --------------------
    lv, r = 0, r1
    goffs = np.zeros(p + 1, np.uint64)
    np.cumsum(sizes, out=goffs[1:])
    rank_offs = goffs[np.arange(world + 1) * pl]                     # first key of every rank
    rank_off = int(rank_offs[rank])
    n_g = np.array([n], np.uint64)
    br, target = level_targets(n_g, r, b, a)
    gf, gn = np.zeros(1, np.int32), np.array([p], np.int32)
    idx, gpos, drawn = L.draw_sample_positions(master, stream_id, lv, gf, gn, target, sizes,
                                               goffs[:-1])
    # The draw is replicated, so every rank knows every rank's share of the
    # sample: one fixed-size all-gather of (key, position) pairs.
    owner_of = np.searchsorted(rank_offs, idx, side="right") - 1
    counts = np.bincount(owner_of, minlength=world) if len(idx) else np.zeros(world, np.int64)
    mine = owner_of == rank
    l_idx, l_gpos = idx[mine] - np.uint64(rank_off), gpos[mine]
    cnt = int(counts[rank])
    width = max(int(counts.max()), 1)
    s_keys, s_pos = ops.empty(cnt, torch.int64), ops.empty(cnt, torch.int32)
    ops.sample(keys, kind, l_idx, l_gpos, s_keys, s_pos)
    pack = torch.zeros(2 * width, dtype=torch.int64, device=dev)
    pack[:cnt] = s_keys[:cnt]
    pack[width:width + cnt] = s_pos[:cnt].to(torch.int64)
    packs = [torch.zeros_like(pack) for _ in range(world)]
    dist.all_gather(packs, pack, group=group)
    all_keys = torch.cat([q[:int(c)] for q, c in zip(packs, counts)])
    all_pos = torch.cat([q[width:width + int(c)] for q, c in zip(packs, counts)]).to(torch.int32)
    S = int(drawn.sum())
    assert all_keys.numel() == S
    nb = np.minimum(br, drawn.astype(np.int64) + 1)                    # ams.py:228
    soff = np.array([0, S], np.uint64)
    ops.splitters(all_keys, all_pos, soff, nb)
    loffs = np.zeros(pl + 1, np.uint64)
    np.cumsum(local_sizes, out=loffs[1:])
    nb_stride = int(nb.max())
    hist_l = ops.classify(keys, kind, loffs[:-1], local_sizes, np.zeros(pl, np.int32),
                          np.array([rank_off], np.int64), nb_stride, True, True)
    # Histograms and key range (ordered encoding) of every rank: one all-gather.
    lo, hi = ops.get_minmax()
    ht = torch.from_numpy(np.concatenate([hist_l.astype(np.int64).ravel(),
                                          [_u64_to_i64(lo), _u64_to_i64(hi)]])).to(dev)
    hts = [torch.zeros_like(ht) for _ in range(world)]
    dist.all_gather(hts, ht, group=group)
    got = [h.cpu().numpy() for h in hts]
    hist = np.concatenate([x[:-2].reshape(pl, nb_stride) for x in got]).astype(np.uint32)
    los = [int(x[-2]) & ((1 << 64) - 1) for x in got if x[-2] != -1 or x[-1] != 0]
    his = [int(x[-1]) & ((1 << 64) - 1) for x in got if x[-2] != -1 or x[-1] != 0]
    if los:
        ops.set_minmax(min(los), max(his))
    bnd, loads, mx, new_sizes, stats = L.plan_level(gn, nb, r, hist)
    # Keys-only single level: buckets contiguous for the final sort (F7).
    bucket_major = k_levels == 1 and vals is None and not det
    cell_base, bucket_dst, need = level1_cell_base(hist, bnd[0].astype(np.int64), rank, world,
                                                    pl, bucket_major)
    gpr = r // world                                               # groups per rank
    # Non-simple schemes: origin tags (index in the global input) travel as the values.
    src_v = vals
    if det:
        src_v = ops.empty(n_local, torch.int64)
        ops.iota(src_v, n_local, rank_off)
    recv, recv_v = ops.exchange(keys, src_v, kind, need, cell_base, bucket_dst, r, bnd[0],
                                rank * gpr, gpr, group=group)
    n_recv = int(need[rank])
    step = p // r                                                  # members of a subgroup
    if det:
        # Member assignment of the scheme from the replicated piece matrix;
        # subgroup g's members all live on g's owner rank, so the relayout
        # of the simple layout into the member arrays is rank-local.
        bd = bnd[0].astype(np.int64)
        pieces = np.stack([hist[:, bd[g]:bd[g + 1]].sum(axis=1, dtype=np.uint64) for g in range(r)],
                          axis=1)
        ls_name = f"{stream_id}/L0-g0"
        if scheme == "deterministic":
            new_sizes, slices, st4 = L.deliver_deterministic(pieces, 0)
        elif scheme == "permuted":
            new_sizes, slices, st4 = L.deliver_permuted(pieces, master, ls_name)
        else:
            new_sizes, slices, st4 = L.deliver_randomized(pieces, master, ls_name)
        stats = st4.reshape(1, 4)
        if step > 1:
            m_g = pieces.sum(axis=0)
            e0 = int(m_g[:rank * gpr].sum())                        # this rank's part of the simple layout
            d0 = int(new_sizes[:pe_lo].sum())                       # ... and of the member arrays
            sel = (slices[:, 0] >= e0) & (slices[:, 0] < e0 + n_recv) & (slices[:, 2] > 0)
            loc = slices[sel].copy()
            loc[:, 0] -= np.uint64(e0)
            loc[:, 1] -= np.uint64(d0)
            relaid, relaid_v = ops.empty(n_recv, torch.int64), ops.empty(n_recv, torch.int64)
            ops.copy_ranges(loc, recv, relaid, recv_v, relaid_v)
            recv, recv_v = relaid, relaid_v
    rec = LevelRecord(lv, r, gf, gn, sizes.copy(), drawn, nb, hist, bnd, loads, mx,
                      load_budget(n_g, r, eps_l), new_sizes, stats)
    levels.append(rec)
    my_groups = np.arange(rank * gpr, (rank + 1) * gpr)
    local_next = np.asarray(new_sizes, dtype=np.uint64)[pe_lo:pe_lo + pl]
    n_out = int(local_next.sum())
    if isinstance(out, torch.Tensor) and out.is_cuda:
        check_out(out, n_out, dev, "out")
        check_out(out_vals, n_out, dev, "out_vals")
    if out is None:
        out = torch.empty(max(n_out, 1), dtype=keys.dtype, device=dev)
    if vals is not None and out_vals is None:
        out_vals = torch.empty(max(n_out, 1), dtype=vals.dtype, device=dev)

    if k_levels == 1:
        # Single level: the received groups are the final PEs.
        offs = np.zeros(pl + 1, np.uint64)
        np.cumsum(local_next, out=offs[1:])
        work, work_v = ops.workspace(max(n_recv, 1), recv_v is not None)
        if bucket_major:  # this rank's buckets in output order (level1_cell_base's layout)
            tot = hist.astype(np.int64).sum(axis=0)
            bk = np.arange(int(bnd[0][my_groups[0]]), int(bnd[0][my_groups[-1] + 1]), dtype=np.int32)
            ln = tot[bk].astype(np.uint64)
            off = np.concatenate([[0], np.cumsum(ln)[:-1]]).astype(np.uint64)
            ops.final_sort_buckets(recv, work[0], out, kind, off, ln, np.zeros(len(bk), np.int32), bk)
        elif det:
            # keys only (equal keys are indistinguishable): a key sort of every PE
            ops.final_sort(recv, None, work[0], None, out, None, kind, offs[:-1], local_next)
        else:
            ops.final_sort(recv, recv_v, work[0], work_v[0], out, out_vals, kind, offs[:-1], local_next)
        return out[:n_out], (out_vals[:n_out] if out_vals is not None else None), local_next, levels

    # ---------------- later levels and the final sort: rank-local -----------
    final_sizes, later = ops.run_from(recv, recv_v, params, a, master, stream_id, kind, scheme,
                                      level_base=1, init_groups=gpr, pe_base=pe_lo,
                                      local_sizes=local_next, out=out, out_vals=out_vals)
    return (out[:n_out], (out_vals[:n_out] if out_vals is not None else None),
            np.asarray(final_sizes, dtype=np.uint64), _Levels(levels, later))


class _Levels(list):
    """Level 1's record followed by the continuation's records, which are
    read from the context on first use."""

    def __init__(self, first, later):
        super().__init__(first)
        self._later = later

    def _fill(self):
        if self._later is not None:
            later, self._later = self._later, None
            self.extend(later() if callable(later) else later)

    def __iter__(self):
        self._fill()
        return super().__iter__()

    def __len__(self):
        self._fill()
        return super().__len__()

    def __getitem__(self, i):
        self._fill()
        return super().__getitem__(i)
