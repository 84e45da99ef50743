"""Level orchestration of AMS-sort on one B200 (host side, Python).

One call of :meth:`AmsSorter.sort` runs the reference's ``ams_sort``
(ams.py:271-313) with ``scheme="simple"`` over device-resident keys:

    for each level lv, r in group_counts:                       ams.py:285
        sample positions (C++ restatement of SeedSpec + random.sample)
        K1 gather + K2 rank-by-counting splitters            ams.py:223-229
        K3 classify + histograms  -> host (the level's one sync)  231-237
        plan (C++ optimal_group_plan) + next member sizes        238, 78-80
        K4 offsets + K6 stable scatter into (g, j, b) order      240-256
    K7-K9 final per-PE stable sort                               310-312

Positions are implicit (index in the group buffer): the tie-broken order
(key, origin_pe, origin_pos) equals (key, position) inside every group
(SURVEY F6), so no origin tags are stored on the device.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib as L
from .params import AmsParams, as_params, as_seed

_KIND_OF_DTYPE = {torch.uint64: L.KEY_U64, torch.int64: L.KEY_I64, torch.float64: L.KEY_F64}
_KIND_NAMES = {"u64": L.KEY_U64, "uint64": L.KEY_U64, "i64": L.KEY_I64, "int64": L.KEY_I64,
               "f64": L.KEY_F64, "float64": L.KEY_F64}


def check_out(t, n: int, device, name: str) -> None:
    """A caller-supplied output buffer must hold n contiguous 8-byte
    elements on the sort's device: the native driver writes n keys there and
    also uses ``out`` as relayout scratch."""
    if t is None:
        return
    if not isinstance(t, torch.Tensor) or t.device != device:
        raise ValueError(f"{name} must be a tensor on {device}")
    if t.element_size() != 8 or not t.is_contiguous() or t.numel() < n:
        raise ValueError(f"{name} must be a contiguous tensor of at least {n} 8-byte elements")


def key_kind_of(t: torch.Tensor, key_kind=None) -> int:
    if key_kind is not None:
        return _KIND_NAMES[key_kind] if isinstance(key_kind, str) else int(key_kind)
    if t.dtype not in _KIND_OF_DTYPE:
        raise ValueError(f"keys must be uint64, int64 or float64, got {t.dtype}")
    return _KIND_OF_DTYPE[t.dtype]


# Delivery schemes (delivery.py:439-455 SCHEMES) the device path implements.
SCHEMES = {"simple": 0, "deterministic": 1, "permuted": 2, "randomized": 3}  # AMS_SCHEME_*
# Where sample positions come from: the reference's seeded streams (bucket
# boundaries equal the reference's) or stratified positions drawn on the
# device (no host draw; same quota split, different boundaries).
SAMPLE_MODES = {"parity": 0, "device": 1}  # AMS_SAMPLE_*


@dataclass
class LevelRecord:
    """Host-side facts of one level (all groups), for reports and parity."""

    level: int
    r: int
    group_first: np.ndarray
    group_npe: np.ndarray
    sizes_before: np.ndarray
    sample_size: np.ndarray       # per group: drawn
    bucket_count: np.ndarray      # per group: br after shrinking (ams.py:228)
    seg_hist: np.ndarray          # (P_total, nb_stride)
    boundaries: np.ndarray        # (G, r+1)
    loads: np.ndarray             # (G, r)
    max_load: np.ndarray          # (G,)
    load_budget: np.ndarray       # (G,)
    new_sizes: np.ndarray         # (P_total,)
    stats: np.ndarray | None      # (G, 4) exchange stats
    splitters: list = field(default_factory=list)  # per group (keys, pos) if recorded
    holders: np.ndarray | None = None  # per PE: splitters drawn from it (record_holders)

    def report(self) -> dict:
        """The per-level dict ams_sort returns (ams.py:296-308)."""
        rep = {
            "level": self.level + 1,
            "r": self.r,
            "max_load": int(self.new_sizes.max()),
            "min_load": int(self.new_sizes.min()),
            "sample_size": int(self.sample_size.max()),
            "plan_load": int(self.max_load.max()),
            "over_budget": int((self.max_load > self.load_budget).sum()),
        }
        if self.stats is not None:
            for i, k in enumerate(("max_words", "max_msgs", "max_sent_msgs", "max_recv_msgs")):
                rep[k] = int(self.stats[:, i].max())
        return rep


@dataclass
class SortOutput:
    keys: torch.Tensor
    vals: torch.Tensor | None
    pe_sizes: np.ndarray
    _levels: object  # list of LevelRecord, or a callable building it on first use
    launches: int

    @property
    def levels(self) -> list:
        """Per-level records; the one-call driver's are read from the context on
        first use (it keeps the last 8 runs), off the sort's critical path."""
        if callable(self._levels):
            self._levels = self._levels()
        return self._levels

    @property
    def reports(self) -> list:
        return [lv.report() for lv in self.levels]


def bucket_table(seg_hist: np.ndarray, group_first, group_npe, nb, group_start):
    """Buckets of a bucket-major (keys-only) last level in output order:
    (offset, length, group, bucket) arrays for ams_final_sort_buckets.  Group
    g starts at group_start[g]; its bucket b holds the sum over the group's
    members of seg_hist[member][b]."""
    off, ln, grp, bkt = [], [], [], []
    for g, (f, c) in enumerate(zip(group_first, group_npe)):
        tot = seg_hist[int(f):int(f) + int(c), :int(nb[g])].astype(np.uint64).sum(axis=0)
        starts = int(group_start[g]) + np.concatenate([[0], np.cumsum(tot)[:-1]]).astype(np.uint64)
        off.append(starts)
        ln.append(tot)
        grp.append(np.full(len(tot), g, np.int32))
        bkt.append(np.arange(len(tot), dtype=np.int32))
    cat = lambda xs, dt: np.concatenate(xs).astype(dt) if xs else np.zeros(0, dt)
    return cat(off, np.uint64), cat(ln, np.uint64), cat(grp, np.int32), cat(bkt, np.int32)


def level_targets(n_g: np.ndarray, r: int, b: int, a: float):
    """br and sample target per group (ams.py:224-225)."""
    br = np.minimum(b * r, n_g + 1).astype(np.int64)
    target = np.array([min(int(n), max(int(x) - 1, math.ceil(a * int(x))))
                       for n, x in zip(n_g, br)], dtype=np.int64)
    return br, target


def load_budget(n_g: np.ndarray, r: int, eps_level: float) -> np.ndarray:
    """ams.py:258."""
    return np.array([math.ceil((1.0 + eps_level) * int(n) / r) for n in n_g], dtype=np.int64)


def run_records(ctx, run: int, group_counts, eps_l: float, first_level: int = 0,
                record_holders: bool = False):
    """Callable that reads the level records of ams_sort_run `run` from the
    context on first use (levels first_level..; the context keeps 8 runs)."""

    def levels():
        recs = []
        for lv in range(first_level, len(group_counts)):
            r = group_counts[lv]
            d = ctx.run_level(lv, run)
            n_g = np.add.reduceat(d["sizes_before"], d["group_first"]) if len(d["sizes_before"]) \
                else np.zeros(len(d["group_first"]), np.uint64)
            recs.append(LevelRecord(lv, r, d["group_first"], d["group_npe"], d["sizes_before"],
                                    d["drawn"], d["nb"].astype(np.int64), d["seg_hist"],
                                    d["boundaries"], d["loads"], d["max_load"],
                                    load_budget(n_g, r, eps_l), d["new_sizes"], d["stats"]))
            if record_holders:
                recs[-1].holders = ctx.run_level_holders(lv, len(d["sizes_before"]), run)
        return recs
    return levels


def native_params(params, master, stream_id, kind, with_stats=True, scheme=0, record_holders=False,
                  oversampling=None, level_base=0, init_groups=0, pe_base=0, sample_mode=0):
    """ams_params_t for ams_sort_run (include/ams_b200.h)."""
    prm = L.ParamsT()
    gc = tuple(params.group_counts)
    if len(gc) > L.MAX_LEVELS:
        raise ValueError(f"at most {L.MAX_LEVELS} levels are supported")
    prm.levels = len(gc)
    for i, r in enumerate(gc):
        prm.group_counts[i] = int(r)
    a = oversampling if oversampling is not None else params.oversampling
    prm.oversampling = float(a) if a is not None else 0.0
    prm.overpartition = int(params.overpartition)
    prm.imbalance = float(params.imbalance)
    prm.master_seed = int(master)
    prm.stream_id = stream_id.encode()
    prm.key_kind = int(kind)
    prm.with_stats = int(bool(with_stats))
    prm.scheme = int(scheme)
    prm.record_holders = int(bool(record_holders))
    prm.level_base = int(level_base)
    prm.init_groups = int(init_groups)
    prm.pe_base = int(pe_base)
    prm.sample_mode = int(sample_mode)
    return prm


class AmsSorter:
    """Device-resident AMS-sort on one GPU (one process per GPU)."""

    def __init__(self, device: int | torch.device | None = None):
        if not torch.cuda.is_available():
            raise RuntimeError("AmsSorter needs a CUDA device (B200, sm_100a); there is no CPU path")
        dev = torch.device("cuda", torch.cuda.current_device() if device is None else
                           (device.index if isinstance(device, torch.device) else int(device)))
        self.device = dev
        self.ctx = L.Context(dev.index)
        self._work: dict = {}

    def close(self):
        self.ctx.close()

    # -- workspace ----------------------------------------------------------
    def workspace(self, n: int, with_vals: bool):
        key = (n, with_vals)
        if key not in self._work:
            self._work.clear()
            # +2 keys: the fixed-capacity partition's bulk loads cover whole
            # 16-byte units past a bucket's end (k_scatter_fixed).
            mk = lambda: torch.empty(max(n, 1) + 2, dtype=torch.int64, device=self.device)
            self._work[key] = ([mk(), mk()], [mk(), mk()] if with_vals else [None, None])
        return self._work[key]

    # -- main entry ---------------------------------------------------------
    def sort(self, keys: torch.Tensor, pe_sizes, params: AmsParams, seed, vals=None, out=None,
             out_vals=None, key_kind=None, record_splitters: bool = False,
             with_stats: bool = True, scheme: str = "simple",
             record_holders: bool = False, sample_mode: str = "parity") -> SortOutput:
        """Sort ``keys`` (1-D, PE-major: PE i owns the next ``pe_sizes[i]``
        keys) exactly as ams_sort(scheme) orders them (every scheme of the
        reference's SCHEMES registry; the per-level host driver,
        ``record_splitters=True``, runs "simple" only); returns the sorted
        keys (concatenation of per-PE outputs), per-PE sizes and per-level
        records."""
        if scheme not in SCHEMES:
            raise ValueError(f"unknown delivery scheme {scheme!r}; supported: {tuple(SCHEMES)}")
        if sample_mode not in SAMPLE_MODES:
            raise ValueError(f"unknown sample mode {sample_mode!r}; supported: {tuple(SAMPLE_MODES)}")
        if sample_mode != "parity" and (record_splitters or record_holders):
            raise ValueError("splitter records need sample_mode='parity'")
        if record_splitters and scheme != "simple":
            raise ValueError("record_splitters runs the per-level host driver, which implements "
                             "the simple scheme only")
        params = as_params(params)
        master, stream_id = as_seed(seed)
        if keys.dim() != 1 or not keys.is_cuda:
            raise ValueError("keys must be a 1-D CUDA tensor")
        kind = key_kind_of(keys, key_kind)
        sizes = np.asarray(pe_sizes, dtype=np.uint64)
        p = len(sizes)
        params.validate_for(p)                                       # ams.py:276
        n = int(sizes.sum())
        if n != keys.numel():
            raise ValueError(f"pe_sizes sum to {n}, keys has {keys.numel()} elements")
        if vals is not None and (vals.numel() != n or vals.element_size() != 8 or not vals.is_cuda
                                 or vals.device != keys.device):
            raise ValueError("vals must be a CUDA tensor of n 8-byte values on the keys' device")
        check_out(out, n, keys.device, "out")
        if out_vals is not None and vals is None:
            raise ValueError("out_vals given without vals")
        check_out(out_vals, n, keys.device, "out_vals")
        keys = keys.contiguous()
        if vals is not None:
            vals = vals.contiguous()
        if out is None:
            out = torch.empty_like(keys)
        if vals is not None and out_vals is None:
            out_vals = torch.empty_like(vals)
        ret_out, ret_vals = out, out_vals
        if n == 0:
            # Empty tensors have no storage; every segment is empty, so the
            # kernels never touch these one-element stand-ins.
            keys = torch.zeros(1, dtype=keys.dtype, device=keys.device)
            out = torch.zeros_like(keys)
            if vals is not None:
                vals = torch.zeros(1, dtype=vals.dtype, device=vals.device)
                out_vals = torch.zeros_like(vals)
        stream = torch.cuda.current_stream(self.device)
        self.ctx.set_stream(stream.cuda_stream)
        launches0 = self.ctx.launches
        if not record_splitters:
            # The whole level loop in C++ (ams_sort_run); same steps as below.
            return self._sort_native(keys, vals, ret_out, ret_vals, out, out_vals, sizes, params,
                                     master, stream_id, kind, with_stats, launches0, n,
                                     SCHEMES[scheme], record_holders, SAMPLE_MODES[sample_mode])
        a = params.oversampling_for(n)                               # ams.py:278-280
        eps_l = params.per_level_imbalance()
        b = params.overpartition
        work, work_v = self.workspace(n, vals is not None)
        src, src_v, src_kind = keys, vals, kind
        gf = np.zeros(1, np.int32)
        gn = np.array([p], np.int32)
        levels = []
        for lv, r in enumerate(params.group_counts):
            offs = np.zeros(p + 1, np.uint64)
            np.cumsum(sizes, out=offs[1:])
            G = len(gf)
            n_g = np.add.reduceat(sizes, gf) if p else np.zeros(G, np.uint64)
            br, target = level_targets(n_g, r, b, a)
            idx, gpos, drawn = L.draw_sample_positions(master, stream_id, lv, gf, gn, target,
                                                       sizes, offs[:-1])
            nb = np.minimum(br, drawn.astype(np.int64) + 1)             # ams.py:228
            if nb.max() > L.MAX_BUCKETS:
                raise ValueError(f"{int(nb.max())} buckets exceed the supported {L.MAX_BUCKETS}")
            soff = np.zeros(G + 1, np.uint64)
            np.cumsum(drawn, out=soff[1:])
            S = int(soff[-1])
            s_keys = torch.empty(max(S, 1), dtype=torch.int64, device=self.device)
            s_pos = torch.empty(max(S, 1), dtype=torch.int32, device=self.device)
            self.ctx.level_sample(src, src_kind, idx, gpos, s_keys, s_pos)
            self.ctx.level_splitters(s_keys, s_pos, soff, nb)
            seg_group = np.repeat(np.arange(G, dtype=np.int32), gn)
            posbase = -offs[gf].astype(np.int64)
            nb_stride = int(nb.max())
            # Only PE membership matters at the last level (F7): keys-only
            # runs may drop in-tile order there.
            last_level = lv == len(params.group_counts) - 1
            hist = self.ctx.level_classify(src, src_kind, offs[:-1], sizes, seg_group, posbase,
                                           nb_stride, track_minmax=(lv == 0),
                                           stable=not (last_level and vals is None))
            bnd, loads, mx, new_sizes, stats = L.plan_level(gn, nb, r, hist, with_stats)
            dst, dst_v = work[lv % 2], work_v[lv % 2]
            # Keys-only last level: bucket-major groups for the fixed-capacity final sort.
            bucket_major = last_level and vals is None
            self.ctx.level_scatter(src, src_v, src_kind, dst, dst_v, r, bnd, offs[gf],
                                   bucket_major=bucket_major)
            if bucket_major:
                final_buckets = bucket_table(hist, gf, gn, nb, offs[gf])
            rec = LevelRecord(lv, r, gf.copy(), gn.copy(), sizes.copy(), drawn, nb, hist, bnd,
                              loads, mx, load_budget(n_g, r, eps_l), new_sizes, stats)
            if record_splitters:
                rec.splitters = [self.ctx.read_splitters(g) for g in range(G)]
            levels.append(rec)
            src, src_v, src_kind = dst, dst_v, L.KEY_U64
            sizes = new_sizes
            step = gn // r
            gf = (gf[:, None] + np.arange(r, dtype=np.int32)[None, :] * step[:, None]).reshape(-1)
            gf = gf.astype(np.int32)
            gn = np.repeat(step, r).astype(np.int32)
        # Final local sort (ams.py:310-312): final PE s = child s of the
        # last level; its key bounds were derived by the last scatter.
        k = len(params.group_counts)
        offs = np.zeros(p + 1, np.uint64)
        np.cumsum(sizes, out=offs[1:])
        tmp, tmp_v = work[k % 2], work_v[k % 2]
        if vals is None:
            self.ctx.final_sort_buckets(src, tmp, out, kind, *final_buckets)
        else:
            self.ctx.final_sort(src, src_v, tmp, tmp_v, out, out_vals, kind, offs[:-1], sizes)
        return SortOutput(ret_out, ret_vals, sizes, levels, self.ctx.launches - launches0)

    def _sort_native(self, keys, vals, ret_out, ret_vals, out, out_vals, sizes, params, master,
                     stream_id, kind, with_stats, launches0, n, scheme=0, record_holders=False,
                     sample_mode=0):
        gc = tuple(params.group_counts)
        prm = native_params(params, master, stream_id, kind, with_stats, scheme, record_holders,
                            sample_mode=sample_mode)
        final_sizes, _ = self.ctx.sort_run(prm, sizes, keys if n else None,
                                           vals if n else None, out if n else None,
                                           out_vals if n else None)
        levels = run_records(self.ctx, self.ctx.run_id(), gc, params.per_level_imbalance(),
                             record_holders=record_holders)
        return SortOutput(ret_out, ret_vals, final_sizes, levels, self.ctx.launches - launches0)
