"""CPU stand-in for CudaOps used ONLY by tests/test_dist_gloo.py: the
device steps restated with the numpy oracle so the multi-rank orchestration
in paper_1410_6754_b200/dist.py (sample all-gather, histogram all-gather,
replicated plan, exchange offsets) can run over gloo without a GPU.  The
product path never uses this (it raises without CUDA)."""

import numpy as np
import torch

from oracle import ams_oracle as O

U64 = np.uint64
SIGN = np.uint64(1 << 63)


def _u(t: torch.Tensor) -> np.ndarray:
    return t.numpy().view(np.uint64)


def _ordered(x: np.ndarray, kind: int) -> np.ndarray:
    if kind == 1:  # int64
        return x ^ SIGN
    if kind == 2:  # float64 bits
        neg = (x >> np.uint64(63)).astype(bool)
        return np.where(neg, ~x, x | SIGN)
    return x


def _from_ordered(x: np.ndarray, kind: int) -> np.ndarray:
    if kind == 1:
        return x ^ SIGN
    if kind == 2:
        top = (x >> np.uint64(63)).astype(bool)
        return np.where(top, x & ~SIGN, ~x)
    return x


class NumpyOps:
    def __init__(self):
        self.spl = []
        self.lvl = None
        self.mm = (0, 0)

    def empty(self, n, dtype=torch.int64):
        return torch.zeros(max(n, 1), dtype=dtype)

    def workspace(self, n, with_vals):
        mk = lambda: torch.zeros(max(n, 1), dtype=torch.int64)
        return [mk(), mk()], ([mk(), mk()] if with_vals else [None, None])

    def sample(self, src, kind, idx, gpos, out_keys, out_pos):
        idx = np.asarray(idx, np.int64)
        if len(idx):
            _u(out_keys)[:len(idx)] = _ordered(_u(src)[idx], kind)
            out_pos.numpy()[:len(idx)] = np.asarray(gpos, np.int64).astype(np.int32)

    def splitters(self, s_keys, s_pos, soff, nb):
        keys, pos = _u(s_keys), s_pos.numpy().astype(np.int64)
        self.spl = []
        for g in range(len(nb)):
            a, b = int(soff[g]), int(soff[g + 1])
            self.spl.append(O.select_splitters(keys[a:b].copy(), pos[a:b].copy(), int(nb[g])))

    def classify(self, src, kind, offs, sizes, seg_group, posbase, nb_stride, track_minmax, stable):
        x = _u(src)
        hist = np.zeros((len(sizes), nb_stride), np.uint32)
        self.lvl = []
        lo, hi = ~np.uint64(0), np.uint64(0)
        for s in range(len(sizes)):
            o, n = int(offs[s]), int(sizes[s])
            k = _ordered(x[o:o + n], kind)
            g = int(seg_group[s])
            pos = np.arange(o, o + n, dtype=np.int64) + int(posbase[g])
            b = O.classify(k, pos, *self.spl[g])
            np.add.at(hist[s], b, 1)
            self.lvl.append((o, n, g, k, b))
            if n:
                lo, hi = min(lo, k.min()), max(hi, k.max())
        if track_minmax:
            self.mm = (int(lo), int(hi))
        return hist

    def get_minmax(self):
        return self.mm

    def set_minmax(self, lo, hi):
        self.mm = (lo, hi)

    def scatter(self, src, src_v, kind, dst, dst_v, r, bnd, dst_start, child_first, child_count,
                bucket_major=False):
        d = _u(dst)
        vs = src_v.numpy() if src_v is not None else None
        groups = sorted({g for _, _, g, _, _ in self.lvl})
        for g in groups:
            segs = [t for t in self.lvl if t[2] == g]
            keys = np.concatenate([t[3] for t in segs]) if segs else np.zeros(0, U64)
            bk = np.concatenate([t[4] for t in segs]) if segs else np.zeros(0, np.int64)
            j = np.concatenate([np.full(t[1], i) for i, t in enumerate(segs)]) if segs else bk
            gid = np.searchsorted(np.asarray(bnd[g], np.int64), bk, side="right") - 1
            if bucket_major:  # (bucket, source) order: buckets contiguous (keys-only last level)
                order = np.argsort(bk * len(segs) + j, kind="stable")
            else:
                order = np.argsort((gid * len(segs) + j) * (1 << 20) + bk, kind="stable")
            st = int(dst_start[g])
            d[st:st + len(keys)] = keys[order]
            if vs is not None:
                v = np.concatenate([vs[t[0]:t[0] + t[1]] for t in segs])
                dst_v.numpy()[st:st + len(keys)] = v[order]

    def exchange(self, src, src_v, kind, need, cell_base, bucket_dst, r, bnd, child_first,
                 child_count, group=None):
        """The peer scatter's semantics over gloo: every local key goes to
        rank bucket_dst[b] at index cell_base[s][b] + its rank among the
        earlier keys of (segment s, bucket b)."""
        import torch.distributed as dist
        world = len(need)
        rank = dist.get_rank(group)
        vs = src_v.numpy() if src_v is not None else None
        parts = [[] for _ in range(world)]
        for s, (o, n, g, k, b) in enumerate(self.lvl):
            b = np.asarray(b, np.int64)
            order = np.argsort(b, kind="stable")
            bs = b[order]
            first = np.searchsorted(bs, bs, side="left")
            rank_in = np.empty(n, np.int64)
            rank_in[order] = np.arange(n) - first
            dest = np.asarray(bucket_dst, np.int64)[b]
            idx = np.asarray(cell_base, np.int64)[s][b] + rank_in
            v = vs[o:o + n] if vs is not None else None
            for d in range(world):
                sel = dest == d
                parts[d].append((idx[sel], k[sel], None if v is None else v[sel]))
        got = [None] * world
        dist.all_gather_object(got, parts, group=group)
        recv = torch.zeros(max(int(need[rank]), 1), dtype=torch.int64)
        recv_v = torch.zeros_like(recv) if src_v is not None else None
        for q in got:
            for idx, k, v in q[rank]:
                recv.numpy().view(np.uint64)[idx] = k
                if recv_v is not None:
                    recv_v.numpy()[idx] = v
        self.mm_children = None
        return recv, recv_v

    def final_sort_buckets(self, src, tmp, out, kind, bk_off, bk_len, bk_group, bk_bucket):
        x = _u(src)
        o_ = _u(out)
        for o, n in zip(bk_off, bk_len):
            o, n = int(o), int(n)
            o_[o:o + n] = _from_ordered(np.sort(x[o:o + n]), kind)

    def final_sort(self, src, src_v, tmp, tmp_v, out, out_v, kind, offs, sizes):
        x = _u(src)
        o_ = _u(out)
        for s in range(len(sizes)):
            o, n = int(offs[s]), int(sizes[s])
            order = np.argsort(x[o:o + n], kind="stable")
            o_[o:o + n] = _from_ordered(x[o:o + n][order], kind)
            if src_v is not None:
                out_v.numpy()[o:o + n] = src_v.numpy()[o:o + n][order]

    def iota(self, dst, n, start):
        dst.numpy()[:n] = np.arange(start, start + n, dtype=np.int64)

    def copy_ranges(self, ranges, src, dst, src_v, dst_v):
        for s0, d0, ln in np.asarray(ranges, np.int64).reshape(-1, 3):
            dst.numpy()[d0:d0 + ln] = src.numpy()[s0:s0 + ln]
            if src_v is not None:
                dst_v.numpy()[d0:d0 + ln] = src_v.numpy()[s0:s0 + ln]

    def run_from(self, src, src_v, params, a, master, stream_id, kind, scheme, level_base,
                 init_groups, pe_base, local_sizes, out, out_vals):
        """The oracle's level loop (ams_oracle.ams_sort) from `level_base` on
        for this rank's PEs [pe_base, pe_base + len(local_sizes))."""
        from types import SimpleNamespace
        sizes = [int(x) for x in local_sizes]
        pl = len(sizes)
        n = sum(sizes)
        buf = _u(src)[:n].copy()
        det = scheme != "simple"
        org = src_v.numpy()[:n].astype(np.int64).copy() if det else np.arange(n, dtype=np.int64)
        vbuf = src_v.numpy()[:n].copy() if (src_v is not None and not det) else None
        groups = [(i * (pl // init_groups), pl // init_groups) for i in range(init_groups)]
        recs = []
        for lv in range(level_base, len(params.group_counts)):
            r = params.group_counts[lv]
            offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
            nbuf, norg = np.empty_like(buf), np.empty_like(org)
            nv = None if vbuf is None else np.empty_like(vbuf)
            nsz = list(sizes)
            nxt, bnds = [], []
            for lo, cnt in groups:
                gs, ge = int(offs[lo]), int(offs[lo + cnt])
                o, ov, ns, info, oo = O.ams_level(
                    buf[gs:ge], sizes[lo:lo + cnt], r, params.overpartition, a, master, stream_id, lv,
                    pe_base + lo, None if vbuf is None else vbuf[gs:ge], False, scheme,
                    org[gs:ge] if det else None)
                nbuf[gs:ge], norg[gs:ge] = o, (oo if det else org[gs:ge])
                if nv is not None:
                    nv[gs:ge] = ov
                nsz[lo:lo + cnt] = ns
                bnds.append(list(info.plan.boundaries))
                stp = cnt // r
                nxt.extend((lo + i * stp, stp) for i in range(r))
            buf, org, vbuf, sizes, groups = nbuf, norg, nv, nsz, nxt
            recs.append(SimpleNamespace(level=lv, boundaries=np.asarray(bnds, np.uint64)))
        offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        o_ = _u(out)
        for pe in range(pl):
            s_, e_ = int(offs[pe]), int(offs[pe + 1])
            order = np.lexsort((org[s_:e_], buf[s_:e_])) if det else np.argsort(buf[s_:e_], kind="stable")
            o_[s_:e_] = _from_ordered(buf[s_:e_][order], kind)
            if vbuf is not None:
                out_vals.numpy()[s_:e_] = vbuf[s_:e_][order]
        return np.asarray(sizes, np.uint64), recs
