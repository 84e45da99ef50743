"""Multi-GPU AMS-sort: one process per GPU over torch.distributed.

PE layout: logical PEs are fixed; PE i lives on rank
``i * G // p``.  The first level's single group spans every rank:

    sample positions    every rank computes the whole group's draw
                        (C++ restatement of draw_sample, ams.py:157-175)
    sample all-gather   local sample elements -> full sample on every rank
                        (the all-gather of fastsort.py:84-93 / gossip_merge)
    splitters           replicated, identical on every rank
    classify            local PEs; histogram all-gather (the allreduce of
                        ams.py:236-237, which deliver_simple also needs)
    plan                replicated (optimal_group_plan, ams.py:238)
    scatter + exchange  local scatter in (group, PE, bucket) order, then one
                        point-to-point chunk per (source rank, group)
                        (Network.exchange, simnet.py:294-335; receive
                        order = source order, ams.py:252-256)

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
from .engine import LevelRecord, bucket_table, check_out, load_budget, level_targets, key_kind_of
from .params import as_params, as_seed


class CudaOps:
    """Device work of one rank: the C ABI on this rank's GPU."""

    def __init__(self, sorter):
        self.sorter = sorter
        self.ctx = sorter.ctx
        self.device = sorter.device

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

    def final_sort(self, src, src_v, tmp, tmp_v, out, out_v, kind, offs, sizes):
        self.ctx.final_sort(src, src_v, tmp, tmp_v, out, out_v, kind, offs, sizes)

    def final_sort_buckets(self, src, tmp, out, kind, bk_off, bk_len, bk_group, bk_bucket):
        self.ctx.final_sort_buckets(src, tmp, out, kind, bk_off, bk_len, bk_group, bk_bucket)


def _u64_to_i64(x: int) -> int:
    return x - (1 << 64) if x >= (1 << 63) else x


def _allgather_var(t: torch.Tensor, count: int, world: int, group=None):
    """All-gather variable-length 1-D tensors; returns the rank-ordered
    concatenation and the per-rank counts."""
    counts = torch.tensor([count], dtype=torch.int64, device=t.device)
    all_counts = [torch.zeros_like(counts) for _ in range(world)]
    dist.all_gather(all_counts, counts, group=group)
    cs = [int(c.item()) for c in all_counts]
    mx = max(max(cs), 1)
    pad = torch.zeros(mx, dtype=t.dtype, device=t.device)
    pad[:count] = t[:count]
    outs = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(outs, pad, group=group)
    return torch.cat([o[:c] for o, c in zip(outs, cs)]), cs


def sort_distributed(keys: torch.Tensor, pe_sizes_local, params, seed, ops, vals=None, out=None,
                     out_vals=None, key_kind=None, group=None, scheme: str = "simple"):
    """Sort this rank's PEs as part of one global ams_sort(scheme="simple").
    The multi-GPU driver implements the simple delivery scheme only; any
    other ``scheme`` raises ValueError (single-GPU ``ams_sort_tensors``
    implements all four).

    ``keys`` holds this rank's PEs (PE-major), ``pe_sizes_local`` their
    sizes; PE ids are rank-major (rank k owns PEs [k*p/G, (k+1)*p/G)).
    Returns (sorted local keys, vals, local per-PE sizes, level records); the
    rank-ordered concatenation of the outputs is the global sort."""
    if scheme != "simple":
        raise ValueError(f"the multi-GPU driver implements the simple delivery scheme only, "
                         f"not {scheme!r}")
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
    levels = []

    # ---------------- level 1: one group over all ranks --------------------
    lv, r = 0, r1
    goffs = np.zeros(p + 1, np.uint64)
    np.cumsum(sizes, out=goffs[1:])
    rank_off = int(goffs[pe_lo])
    n_g = np.array([n], np.uint64)
    br, target = level_targets(n_g, r, b, a)
    gf, gn = np.zeros(1, np.int32), np.array([p], np.int32)
    idx, gpos, drawn = L.draw_sample_positions(master, stream_id, lv, gf, gn, target, sizes,
                                               goffs[:-1])
    mine = (idx >= rank_off) & (idx < rank_off + n_local)
    l_idx, l_gpos = idx[mine] - np.uint64(rank_off), gpos[mine]
    cnt = len(l_idx)
    s_keys, s_pos = ops.empty(cnt, torch.int64), ops.empty(cnt, torch.int32)
    ops.sample(keys, kind, l_idx, l_gpos, s_keys, s_pos)
    all_keys, _ = _allgather_var(s_keys, cnt, world, group)
    all_pos, _ = _allgather_var(s_pos, cnt, world, group)
    S = int(drawn.sum())
    assert all_keys.numel() == S
    nb = np.minimum(br, drawn.astype(np.int64) + 1)                    # ams.py:228
    soff = np.array([0, S], np.uint64)
    ops.splitters(all_keys, all_pos, soff, nb)
    loffs = np.zeros(pl + 1, np.uint64)
    np.cumsum(local_sizes, out=loffs[1:])
    nb_stride = int(nb.max())
    last_level = len(params.group_counts) == 1
    hist_l = ops.classify(keys, kind, loffs[:-1], local_sizes, np.zeros(pl, np.int32),
                          np.array([rank_off], np.int64), nb_stride, True,
                          not (last_level and vals is None))
    # Global key range (ordered encoding) and histograms.
    lo, hi = ops.get_minmax()
    mm = torch.tensor([_u64_to_i64(lo) ^ -(1 << 63), _u64_to_i64(hi) ^ -(1 << 63)],
                      dtype=torch.int64, device=dev)
    mins = mm[:1].clone()
    maxs = mm[1:].clone()
    dist.all_reduce(mins, op=dist.ReduceOp.MIN, group=group)
    dist.all_reduce(maxs, op=dist.ReduceOp.MAX, group=group)
    glo = (int(mins.item()) ^ -(1 << 63)) & ((1 << 64) - 1)
    ghi = (int(maxs.item()) ^ -(1 << 63)) & ((1 << 64) - 1)
    ops.set_minmax(glo, ghi)
    ht = torch.from_numpy(hist_l.astype(np.int64)).to(dev)
    hts = [torch.zeros_like(ht) for _ in range(world)]
    dist.all_gather(hts, ht, group=group)
    hist = np.concatenate([h.cpu().numpy() for h in hts]).astype(np.uint32)
    bnd, loads, mx, new_sizes, stats = L.plan_level(gn, nb, r, hist)
    # Local scatter into (group, local PE, bucket) order.
    work, work_v = ops.workspace(max(n_local, int(new_sizes.reshape(world, -1).sum(1).max())),
                                 vals is not None)
    send, send_v = ops.empty(n_local), (ops.empty(n_local) if vals is not None else None)
    gpr = r // world                                               # groups per rank
    ops.scatter(keys, vals, kind, send, send_v, r, bnd, np.zeros(1, np.uint64),
                rank * gpr, gpr)
    # Pieces: elements of (source PE j, destination group g).
    pieces = np.zeros((p, r), np.int64)
    for g in range(r):
        pieces[:, g] = hist[:, int(bnd[0, g]):int(bnd[0, g + 1])].sum(axis=1)
    per_rank = pieces.reshape(world, pl, r).sum(axis=1)            # [src rank, g]
    m_g = per_rank.sum(axis=0)
    # Send my chunk of group g to its owner; receive (source s, my group g)
    # at E_g offset sum_{s' < s} per_rank[s', g] (source order).
    recv = work[0]
    recv_v = work_v[0]
    my_groups = range(rank * gpr, (rank + 1) * gpr)
    g_start = np.concatenate([[0], np.cumsum([m_g[g] for g in my_groups])])
    send_off = np.concatenate([[0], np.cumsum(per_rank[rank])])
    ops_list, copies = [], []
    for g in range(r):
        owner = g // gpr
        c0, c1 = int(send_off[g]), int(send_off[g + 1])
        if c1 == c0:
            continue
        if owner == rank:
            continue
        ops_list.append(dist.P2POp(dist.isend, send[c0:c1], owner, group))
        if send_v is not None:
            ops_list.append(dist.P2POp(dist.isend, send_v[c0:c1], owner, group))
    for li, g in enumerate(my_groups):
        for s in range(world):
            c = int(per_rank[s, g])
            if c == 0:
                continue
            o = int(g_start[li]) + int(per_rank[:s, g].sum())
            if s == rank:
                c0 = int(send_off[g])
                copies.append((recv[o:o + c], send[c0:c0 + c]))
                if send_v is not None:
                    copies.append((recv_v[o:o + c], send_v[c0:c0 + c]))
                continue
            ops_list.append(dist.P2POp(dist.irecv, recv[o:o + c], s, group))
            if send_v is not None:
                ops_list.append(dist.P2POp(dist.irecv, recv_v[o:o + c], s, group))
    for dst_t, src_t in copies:
        dst_t.copy_(src_t)
    if ops_list:
        for req in dist.batch_isend_irecv(ops_list):
            req.wait()
    rec = LevelRecord(lv, r, gf, gn, sizes.copy(), drawn, nb, hist, bnd, loads, mx,
                      load_budget(n_g, r, eps_l), new_sizes, stats)
    levels.append(rec)

    # ---------------- later levels: rank-local ------------------------------
    sizes = new_sizes.astype(np.uint64)           # global-length; local entries used
    src, src_v, src_kind = recv, recv_v, L.KEY_U64
    step = p // r
    gf = (pe_lo + np.arange(gpr, dtype=np.int64) * step).astype(np.int32)
    gn = np.full(gpr, step, np.int32)
    buf = 1
    final_buckets = None
    for lv in range(1, len(params.group_counts)):
        r = params.group_counts[lv]
        offs = np.zeros(p + 1, np.uint64)          # positions in the local buffer
        np.cumsum(np.where((np.arange(p) >= pe_lo) & (np.arange(p) < pe_lo + pl), sizes, 0),
                  out=offs[1:])
        G = len(gf)
        n_g = np.array([int(sizes[f:f + c].sum()) for f, c in zip(gf, gn)], np.uint64)
        br, target = level_targets(n_g, r, b, a)
        idx, gpos, drawn = L.draw_sample_positions(master, stream_id, lv, gf, gn, target, sizes,
                                                   offs[:-1])
        nb = np.minimum(br, drawn.astype(np.int64) + 1)
        soff = np.zeros(G + 1, np.uint64)
        np.cumsum(drawn, out=soff[1:])
        S = int(soff[-1])
        s_keys, s_pos = ops.empty(S, torch.int64), ops.empty(S, torch.int32)
        ops.sample(src, src_kind, idx, gpos, s_keys, s_pos)
        ops.splitters(s_keys, s_pos, soff, nb)
        loc = slice(pe_lo, pe_lo + pl)
        seg_group = np.repeat(np.arange(G, dtype=np.int32), gn)
        posbase = -offs[gf].astype(np.int64)
        nb_stride = int(nb.max())
        last_level = lv == len(params.group_counts) - 1
        hist = ops.classify(src, src_kind, offs[loc], sizes[loc], seg_group, posbase, nb_stride,
                            False, not (last_level and vals is None))
        bnd, loads, mx, new_local, stats = L.plan_level(gn, nb, r, hist)
        dst, dst_v = work[buf], work_v[buf]
        # Keys-only last level: bucket-major groups for the fixed-capacity final sort.
        bucket_major = last_level and vals is None
        ops.scatter(src, src_v, src_kind, dst, dst_v, r, bnd, offs[gf], 0, G * r,
                    bucket_major=bucket_major)
        if bucket_major:
            final_buckets = bucket_table(hist, gf - pe_lo, gn, nb, offs[gf])
        rec = LevelRecord(lv, r, gf.copy(), gn.copy(), sizes[loc].copy(), drawn, nb, hist, bnd,
                          loads, mx, load_budget(n_g, r, eps_l), new_local, stats)
        levels.append(rec)
        sizes = sizes.copy()
        sizes[loc] = new_local
        src, src_v = dst, dst_v
        buf = 1 - buf
        step = gn // r
        gf = (gf[:, None] + np.arange(r, dtype=np.int32)[None, :] * step[:, None]).reshape(-1)
        gf = gf.astype(np.int32)
        gn = np.repeat(step, r).astype(np.int32)
    local_final = sizes[pe_lo:pe_lo + pl].astype(np.uint64)
    n_out = int(local_final.sum())
    if isinstance(out, torch.Tensor) and out.is_cuda:
        check_out(out, n_out, dev, "out")
        check_out(out_vals, n_out, dev, "out_vals")
    if out is None:
        out = torch.empty(max(n_out, 1), dtype=keys.dtype, device=dev)
    if vals is not None and out_vals is None:
        out_vals = torch.empty(max(n_out, 1), dtype=vals.dtype, device=dev)
    offs = np.zeros(pl + 1, np.uint64)
    np.cumsum(local_final, out=offs[1:])
    tmp, tmp_v = work[buf], work_v[buf]
    if final_buckets is not None:
        ops.final_sort_buckets(src, tmp, out, kind, *final_buckets)
    else:
        ops.final_sort(src, src_v, tmp, tmp_v, out, out_vals, kind, offs[:-1], local_final)
    return out[:n_out], (out_vals[:n_out] if out_vals is not None else None), local_final, levels
