"""ctypes binding of ``libams_b200.so`` (the C ABI in include/ams_b200.h).

The library is the only compute path: there is no CPU fallback.  If it is
missing, importing this module raises — build it with
``python -m paper_1410_6754_b200.build`` (``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .build import LIB

AMS_OK, AMS_EINVAL, AMS_ECUDA, AMS_ENOMEM, AMS_EINTERNAL = 0, 1, 2, 3, 4
KEY_U64, KEY_I64, KEY_F64 = 0, 1, 2
TILE = 4096
SMEM_SORT_CAP = 4096
MAX_BUCKETS = 4096
KCAT_NAMES = ("sample_gather", "sample_rank", "build_classifier", "level_hist", "chunk_scan",
              "cell_base", "level_scatter", "final_ranges", "final_hist", "final_scatter",
              "smem_sort", "map_keys", "level_scatter_unstable")

_P = C.c_void_p
_I = C.c_int
_I64 = C.c_int64
_U64 = C.c_uint64

# name -> (restype, argtypes); every array argument is passed as a pointer.
_SIGNATURES = {
    "ams_last_error": (C.c_char_p, []),
    "ams_version": (_I, []),
    "ams_stream_seed": (_I, [_I64, C.c_char_p, _P, _P]),
    "ams_blake2b_128": (_I, [_P, _U64, _P]),
    "ams_sample_indices": (_I, [_P, _I, _U64, _U64, _P]),
    "ams_mt_getrandbits": (_I, [_P, _I, _I, _U64, _P]),
    "ams_draw_sample_positions": (_I, [_I64, C.c_char_p, _I, _I, _P, _P, _P, _P, _P, _U64,
                                       _P, _P, _P]),
    "ams_scan_groups": (_I, [_P, _I, _I, _U64, _P, _P, _P]),
    "ams_group_plan": (_I, [_P, _I, _I, _P, _P, _P]),
    "ams_plan_level": (_I, [_I, _P, _P, _I, _P, _I, _P, _P, _P, _P, _P]),
    "ams_deliver_deterministic": (_I, [_I, _I, _I, _P, _P, _P, _I, _P, _P]),
    "ams_deliver_permuted": (_I, [_I, _I, _I64, C.c_char_p, _P, _P, _P, _I, _P, _P]),
    "ams_deliver_randomized": (_I, [_I, _I, _I64, C.c_char_p, _P, _P, _P, _I, _P, _P]),
    "ams_ctx_create": (_I, [_I, _P, C.POINTER(_P)]),
    "ams_ctx_destroy": (_I, [_P]),
    "ams_ctx_set_stream": (_I, [_P, _P]),
    "ams_ctx_launches": (_U64, [_P]),
    "ams_ctx_sync": (_I, [_P]),
    "ams_ctx_set_timing": (_I, [_P, _I]),
    "ams_ctx_kernel_stats": (_I, [_P, _P, _P, _P, _I]),
    "ams_ctx_reset_stats": (_I, [_P]),
    "ams_ctx_timeline": (_I, [_P, _P, _P, _P, _I, C.POINTER(_I)]),
    "ams_level_sample": (_I, [_P, _P, _I, _U64, _P, _P, _P, _P]),
    "ams_level_splitters": (_I, [_P, _I, _P, _P, _P, _P]),
    "ams_read_splitters": (_I, [_P, _I, _P, _P, C.POINTER(_I)]),
    "ams_level_classify": (_I, [_P, _P, _I, _I, _P, _P, _P, _I, _P, _I, _I, _I, _P]),
    "ams_level_scatter": (_I, [_P, _P, _P, _I, _P, _P, _I, _P, _P, _I, _I]),
    "ams_final_sort_stats": (_I, [_P, _P]),
    "ams_final_sort_fixed_stats": (_I, [_P, _P]),
    "ams_run_id": (C.c_uint64, [_P]),
    "ams_run_level_dims_at": (_I, [_P, C.c_uint64, _I, _P, _P, _P, _P, _P]),
    "ams_run_level_at": (_I, [_P, C.c_uint64, _I] + [_P] * 11),
    "ams_run_level_holders_at": (_I, [_P, C.c_uint64, _I, _P]),
    "ams_level_scatter_ex": (_I, [_P, _P, _P, _I, _P, _P, _I, _P, _P, _I, _I, _I]),
    "ams_final_sort_buckets": (_I, [_P, _P, _P, _P, _I, _I, _P, _P, _P, _P]),
    "ams_get_minmax": (_I, [_P, _P]),
    "ams_peer_buffer": (_I, [_P, _I, C.c_uint64, _P, _P, _P]),
    "ams_peer_open": (_I, [_P, _P, _P]),
    "ams_peer_close_all": (_I, [_P]),
    "ams_level_scatter_peers": (_I, [_P, _P, _P, _I, _I, _P, _P, _P, _P, _I, _P, _I, _I]),
    "ams_set_minmax": (_I, [_P, _P]),
    "ams_final_sort": (_I, [_P, _P, _P, _P, _P, _P, _P, _I, _I, _P, _P]),
    "ams_map_keys": (_I, [_P, _P, _P, _U64, _I, _I]),
    "ams_sort_run": (_I, [_P, _P, _I, _P, _P, _P, _P, _P, _P, _P]),
    "ams_run_level_dims": (_I, [_P, _I, _P, _P, _P, _P, _P]),
    "ams_run_level": (_I, [_P, _I] + [_P] * 11),
    "ams_deliver_simple": (_I, [_I, _I, _P, _P, _P]),
    "ams_mg_create": (_I, [_P, _I, C.POINTER(_P)]),
    "ams_mg_destroy": (_I, [_P]),
    "ams_mg_size": (_I, [_P]),
    "ams_mg_ctx": (_I, [_P, _I, C.POINTER(_P)]),
    "ams_mg_sort_run": (_I, [_P, _P, _I, _P, _P, _P, _P, _P, _P, _P]),
    "ams_mg_level1_dims": (_I, [_P, _P, _P, _P]),
    "ams_mg_level1": (_I, [_P] * 10),
    "ams_copy_ranges": (_I, [_P, _P, _I, _P, _P, _P, _P]),
    "ams_fill_iota": (_I, [_P, _P, _U64, _U64]),
    "ams_rlm_sort_run": (_I, [_P, _I, _P, _I, _I64, C.c_char_p, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P]),
    "ams_rlm_level_dims": (_I, [_P, _I, _P, _P, _P]),
    "ams_rlm_level": (_I, [_P, _I] + [_P] * 6),
}

MAX_LEVELS = 8


class ParamsT(C.Structure):
    """ams_params_t (include/ams_b200.h)."""

    _fields_ = [("levels", C.c_int), ("group_counts", C.c_int * MAX_LEVELS),
                ("oversampling", C.c_double), ("overpartition", C.c_int),
                ("imbalance", C.c_double), ("master_seed", C.c_int64),
                ("stream_id", C.c_char_p), ("key_kind", C.c_int), ("with_stats", C.c_int),
                ("scheme", C.c_int), ("record_holders", C.c_int), ("level_base", C.c_int),
                ("init_groups", C.c_int), ("pe_base", C.c_int), ("sample_mode", C.c_int)]


class LevelReportT(C.Structure):
    """ams_level_report_t (include/ams_b200.h)."""

    _fields_ = [("level", C.c_int), ("r", C.c_int)] + [
        (f, C.c_uint64) for f in ("max_load", "min_load", "sample_size", "plan_load",
                                  "over_budget", "max_words", "max_msgs", "max_sent_msgs",
                                  "max_recv_msgs")]

class RlmReportT(C.Structure):
    """ams_rlm_report_t (include/ams_b200.h)."""

    _fields_ = [("level", C.c_int), ("r", C.c_int)] + [
        (f, C.c_uint64) for f in ("max_load", "min_load", "max_words", "max_msgs",
                                  "max_sent_msgs", "max_recv_msgs")]


EXPORTED = tuple(_SIGNATURES)
BUCKET_MAJOR = 1  # AMS_SCATTER_BUCKET_MAJOR


def _load():
    path = os.environ.get("AMS_LIB", LIB)  # alternative build (experiments)
    if not os.path.exists(path):
        raise ImportError(
            f"{LIB} is missing: build it with `python -m paper_1410_6754_b200.build` "
            "(there is no CPU fallback for the AMS-sort hot path)")
    lib = C.CDLL(path)
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


class AmsError(RuntimeError):
    pass


def check(rc: int) -> int:
    if rc == AMS_OK:
        return rc
    msg = lib.ams_last_error().decode(errors="replace")
    if rc == AMS_EINVAL:
        raise ValueError(msg)
    raise AmsError(f"libams_b200 error {rc}: {msg}")


def ptr(a) -> int | None:
    """Address of a numpy array or torch tensor (None for None)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()


def u64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint64)


def i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


# ---------------------------------------------------------------- host helpers

def stream_seed_words(master_seed: int, stream_id: str) -> np.ndarray:
    words = np.zeros(4, dtype=np.uint32)
    n = C.c_int(0)
    check(lib.ams_stream_seed(int(master_seed), stream_id.encode(), words.ctypes.data,
                              C.addressof(n)))
    return words[: n.value].copy()


def blake2b_128(msg: bytes) -> bytes:
    buf = np.frombuffer(msg, dtype=np.uint8) if msg else np.zeros(1, np.uint8)
    out = np.zeros(16, dtype=np.uint8)
    check(lib.ams_blake2b_128(buf.ctypes.data, len(msg), out.ctypes.data))
    return out.tobytes()


def sample_indices(seed_words: np.ndarray, n: int, k: int) -> np.ndarray:
    w = np.ascontiguousarray(seed_words, dtype=np.uint32)
    out = np.zeros(max(k, 1), dtype=np.uint64)
    check(lib.ams_sample_indices(w.ctypes.data, len(w), n, k, out.ctypes.data))
    return out[:k]


def getrandbits(seed_words: np.ndarray, k: int, count: int) -> np.ndarray:
    w = np.ascontiguousarray(seed_words, dtype=np.uint32)
    out = np.zeros(max(count, 1), dtype=np.uint64)
    check(lib.ams_mt_getrandbits(w.ctypes.data, len(w), k, count, out.ctypes.data))
    return out[:count]


def draw_sample_positions(master_seed, stream, level, group_first, group_npe, targets, sizes,
                          offs):
    gf, gn = i32(group_first), i32(group_npe)
    tg, sz, of = u64(targets), u64(sizes), u64(offs)
    cap = int(tg.sum())
    idx = np.zeros(max(cap, 1), np.uint64)
    gpos = np.zeros(max(cap, 1), np.uint64)
    cnt = np.zeros(len(gf), np.uint64)
    check(lib.ams_draw_sample_positions(int(master_seed), stream.encode(), level, len(gf),
                                        gf.ctypes.data, gn.ctypes.data, tg.ctypes.data,
                                        sz.ctypes.data, of.ctypes.data, cap, idx.ctypes.data,
                                        gpos.ctypes.data, cnt.ctypes.data))
    total = int(cnt.sum())
    return idx[:total], gpos[:total], cnt


def scan_groups(sizes, r: int, limit: int):
    s = u64(sizes)
    bnd = np.zeros(r + 1, np.uint64)
    loads = np.zeros(r, np.uint64)
    mx = np.zeros(1, np.uint64)
    rc = lib.ams_scan_groups(s.ctypes.data, len(s), r, limit, bnd.ctypes.data, loads.ctypes.data,
                             mx.ctypes.data)
    if rc == 1:
        return None
    check(rc)
    return tuple(int(x) for x in bnd), tuple(int(x) for x in loads), int(mx[0])


def group_plan(sizes, r: int):
    s = u64(sizes)
    bnd = np.zeros(r + 1, np.uint64)
    loads = np.zeros(r, np.uint64)
    mx = np.zeros(1, np.uint64)
    check(lib.ams_group_plan(s.ctypes.data, len(s), r, bnd.ctypes.data, loads.ctypes.data,
                             mx.ctypes.data))
    return tuple(int(x) for x in bnd), tuple(int(x) for x in loads), int(mx[0])


def plan_level(group_npe, group_nb, r: int, seg_hist: np.ndarray, with_stats: bool = True):
    gn, gb = i32(group_npe), i32(group_nb)
    G = len(gn)
    hist = np.ascontiguousarray(seg_hist, dtype=np.uint32)
    nb_stride = hist.shape[1]
    bnd = np.zeros((G, r + 1), np.uint64)
    loads = np.zeros((G, r), np.uint64)
    mx = np.zeros(G, np.uint64)
    new_sizes = np.zeros(int(gn.sum()), np.uint64)
    stats = np.zeros((G, 4), np.uint64) if with_stats else None
    check(lib.ams_plan_level(G, gn.ctypes.data, gb.ctypes.data, r, hist.ctypes.data, nb_stride,
                             bnd.ctypes.data, loads.ctypes.data, mx.ctypes.data,
                             new_sizes.ctypes.data, ptr(stats)))
    return bnd, loads, mx, new_sizes, stats


def deliver_deterministic(pieces: np.ndarray, pe0: int = 0, with_stats: bool = True):
    """Host restatement of deliver_deterministic's member assignment
    (delivery.py:188-306) for one group: pieces [P][r] -> (new member sizes,
    slices [k][3] = (src, dst, len) relative to the group's simple layout /
    new member arrays, stats[4] or None)."""
    pc = np.ascontiguousarray(pieces, dtype=np.uint64)
    P, r = pc.shape
    ns = np.zeros(P, np.uint64)
    slices = np.zeros((P * (r + 1), 3), np.uint64)
    cnt = C.c_int(0)
    stats = np.zeros(4, np.uint64) if with_stats else None
    check(lib.ams_deliver_deterministic(P, r, int(pe0), pc.ctypes.data, ns.ctypes.data,
                                        slices.ctypes.data, P * (r + 1), C.byref(cnt), ptr(stats)))
    return ns, slices[:cnt.value].copy(), stats


def _deliver_seeded(fn, pieces, master_seed, level_stream, with_stats):
    pc = np.ascontiguousarray(pieces, dtype=np.uint64)
    P, r = pc.shape
    cap = P * (2 * r + 2) + 16
    ns = np.zeros(P, np.uint64)
    slices = np.zeros((cap, 3), np.uint64)
    cnt = C.c_int(0)
    stats = np.zeros(4, np.uint64) if with_stats else None
    check(fn(P, r, int(master_seed), level_stream.encode(), pc.ctypes.data, ns.ctypes.data,
             slices.ctypes.data, cap, C.byref(cnt), ptr(stats)))
    return ns, slices[:cnt.value].copy(), stats


def deliver_permuted(pieces: np.ndarray, master_seed: int, level_stream: str,
                     with_stats: bool = True):
    """Host restatement of deliver_simple_permuted's slices
    (delivery.py:151-185): as :func:`deliver_deterministic`."""
    return _deliver_seeded(lib.ams_deliver_permuted, pieces, master_seed, level_stream, with_stats)


def deliver_randomized(pieces: np.ndarray, master_seed: int, level_stream: str,
                       with_stats: bool = True):
    """Host restatement of deliver_randomized's slices (delivery.py:318-436):
    as :func:`deliver_deterministic`."""
    return _deliver_seeded(lib.ams_deliver_randomized, pieces, master_seed, level_stream, with_stats)


# ---------------------------------------------------------------- device context

class Context:
    """One ``ams_ctx_t`` bound to a CUDA device and stream."""

    def __init__(self, device: int, stream: int | None = None):
        h = C.c_void_p()
        check(lib.ams_ctx_create(int(device), stream, C.byref(h)))
        self.h = h
        self.device = int(device)

    def close(self):
        if self.h:
            lib.ams_ctx_destroy(self.h)
            self.h = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream: int | None):
        check(lib.ams_ctx_set_stream(self.h, stream))

    @property
    def launches(self) -> int:
        return int(lib.ams_ctx_launches(self.h))

    def sync(self):
        check(lib.ams_ctx_sync(self.h))

    def set_timing(self, enable: bool):
        check(lib.ams_ctx_set_timing(self.h, int(bool(enable))))

    def reset_stats(self):
        check(lib.ams_ctx_reset_stats(self.h))

    def kernel_stats(self) -> dict:
        """{category: (device ms, algorithmic bytes, launches)} since reset."""
        n = len(KCAT_NAMES)
        ms = np.zeros(n, np.float64)
        by = np.zeros(n, np.float64)
        la = np.zeros(n, np.uint64)
        check(lib.ams_ctx_kernel_stats(self.h, ms.ctypes.data, by.ctypes.data, la.ctypes.data, n))
        return {name: (float(ms[i]), float(by[i]), int(la[i])) for i, name in enumerate(KCAT_NAMES)}

    def timeline(self):
        """[(category, start ms, end ms)] of the timed launches since the last
        call, in launch order (times from the first launch of each batch)."""
        cap = 1 << 16
        cat = np.zeros(cap, np.int32)
        t0 = np.zeros(cap, np.float32)
        t1 = np.zeros(cap, np.float32)
        cnt = C.c_int(0)
        check(lib.ams_ctx_timeline(self.h, cat.ctypes.data, t0.ctypes.data, t1.ctypes.data, cap,
                                   C.byref(cnt)))
        n = min(cnt.value, cap)
        return [(KCAT_NAMES[int(cat[i])], float(t0[i]), float(t1[i])) for i in range(n)]

    def level_sample(self, src, kind, idx, gpos, out_keys, out_pos):
        idx, gpos = u64(idx), u64(gpos)
        check(lib.ams_level_sample(self.h, ptr(src), kind, len(idx), idx.ctypes.data,
                                   gpos.ctypes.data, ptr(out_keys), ptr(out_pos)))

    def level_splitters(self, sample_keys, sample_pos, soff, nb):
        soff, nb = u64(soff), i32(nb)
        check(lib.ams_level_splitters(self.h, len(nb), ptr(sample_keys), ptr(sample_pos),
                                      soff.ctypes.data, nb.ctypes.data))

    def read_splitters(self, group: int):
        keys = np.zeros(MAX_BUCKETS, np.uint64)
        pos = np.zeros(MAX_BUCKETS, np.uint32)
        n = C.c_int(0)
        check(lib.ams_read_splitters(self.h, group, keys.ctypes.data, pos.ctypes.data, C.byref(n)))
        return keys[: n.value].copy(), pos[: n.value].copy()

    def level_classify(self, src, kind, seg_off, seg_len, seg_group, group_posbase, nb_stride,
                       track_minmax, stable=True):
        so, sl, sg, pb = u64(seg_off), u64(seg_len), i32(seg_group), i64(group_posbase)
        out = np.zeros((len(so), nb_stride), np.uint32)
        check(lib.ams_level_classify(self.h, ptr(src), kind, len(so), so.ctypes.data,
                                     sl.ctypes.data, sg.ctypes.data, len(pb), pb.ctypes.data,
                                     nb_stride, int(bool(track_minmax)), int(bool(stable)),
                                     out.ctypes.data))
        return out

    def level_scatter(self, src, src_vals, kind, dst, dst_vals, r, boundaries, group_dst_start,
                      child_first=0, child_count=None, bucket_major=False):
        b, d = u64(boundaries), u64(group_dst_start)
        if child_count is None:
            child_count = len(d) * r
        check(lib.ams_level_scatter_ex(self.h, ptr(src), ptr(src_vals), kind, ptr(dst), ptr(dst_vals),
                                       r, b.ctypes.data, d.ctypes.data, int(child_first),
                                       int(child_count), BUCKET_MAJOR if bucket_major else 0))

    def final_sort_buckets(self, src, tmp, out, key_kind, bk_off, bk_len, bk_group, bk_bucket):
        bo, bl, bg, bb = u64(bk_off), u64(bk_len), i32(bk_group), i32(bk_bucket)
        check(lib.ams_final_sort_buckets(self.h, ptr(src), ptr(tmp), ptr(out), key_kind, len(bo),
                                         bo.ctypes.data, bl.ctypes.data, bg.ctypes.data, bb.ctypes.data))

    def final_sort_stats(self):
        out = np.zeros(2, np.uint64)
        check(lib.ams_final_sort_stats(self.h, out.ctypes.data))
        fx = np.zeros(2, np.uint64)
        check(lib.ams_final_sort_fixed_stats(self.h, fx.ctypes.data))
        return {"overflow_cells": int(out[0]), "fallback_cells": int(out[1]),
                "fixed_buckets": int(fx[0]), "fixed_overflow_buckets": int(fx[1])}

    # -- multi-GPU level 1 (peer buffers over NVLink) --------------------------
    def peer_buffer(self, slot: int, nbytes: int):
        """(device address, 64-byte IPC handle, grown) of library buffer `slot`."""
        p = C.c_void_p()
        h = (C.c_ubyte * 64)()
        g = C.c_int()
        check(lib.ams_peer_buffer(self.h, int(slot), int(nbytes), C.byref(p), h, C.byref(g)))
        return int(p.value), bytes(h), bool(g.value)

    def peer_open(self, handle: bytes) -> int:
        p = C.c_void_p()
        hb = (C.c_ubyte * 64).from_buffer_copy(handle)
        check(lib.ams_peer_open(self.h, hb, C.byref(p)))
        return int(p.value)

    def peer_close_all(self):
        check(lib.ams_peer_close_all(self.h))

    def level_scatter_peers(self, src, src_vals, kind, dst_ptrs, dst_vals_ptrs, bucket_dst, cell_base,
                            r, boundaries, child_first, child_count):
        nd = len(dst_ptrs)
        dp = (C.c_void_p * nd)(*dst_ptrs)
        dv = (C.c_void_p * nd)(*dst_vals_ptrs) if dst_vals_ptrs is not None else None
        bd, cb, bnd = i32(bucket_dst), u64(cell_base), u64(boundaries)
        check(lib.ams_level_scatter_peers(self.h, ptr(src), ptr(src_vals), kind, nd, dp, dv, bd.ctypes.data,
                                          cb.ctypes.data, int(r), bnd.ctypes.data, int(child_first),
                                          int(child_count)))

    def get_minmax(self):
        out = np.zeros(2, np.uint64)
        check(lib.ams_get_minmax(self.h, out.ctypes.data))
        return int(out[0]), int(out[1])

    def set_minmax(self, lo: int, hi: int):
        a = np.array([lo, hi], np.uint64)
        check(lib.ams_set_minmax(self.h, a.ctypes.data))

    def final_sort(self, src, src_vals, tmp, tmp_vals, out, out_vals, key_kind, seg_off, seg_len):
        so, sl = u64(seg_off), u64(seg_len)
        check(lib.ams_final_sort(self.h, ptr(src), ptr(src_vals), ptr(tmp), ptr(tmp_vals), ptr(out),
                                 ptr(out_vals), key_kind, len(so), so.ctypes.data, sl.ctypes.data))

    def sort_run(self, params: ParamsT, pe_sizes, keys, vals, out, out_vals):
        """ams_sort_run: returns (final PE sizes, [LevelReportT])."""
        sz = u64(pe_sizes)
        out_sizes = np.zeros(max(len(sz), 1), np.uint64)
        reps = (LevelReportT * params.levels)()
        check(lib.ams_sort_run(self.h, C.byref(params), len(sz), sz.ctypes.data, ptr(keys),
                               ptr(vals), ptr(out), ptr(out_vals), out_sizes.ctypes.data, reps))
        return out_sizes[: len(sz)], list(reps)

    def copy_ranges(self, ranges, src, dst, src_vals=None, dst_vals=None):
        """dst[d + i] = src[s + i] for every (s, d, len) row of ``ranges``."""
        rg = np.ascontiguousarray(ranges, dtype=np.uint64).reshape(-1, 3)
        check(lib.ams_copy_ranges(self.h, rg.ctypes.data, len(rg), ptr(src), ptr(dst), ptr(src_vals),
                                  ptr(dst_vals)))

    def fill_iota(self, dst, n: int, start: int = 0):
        check(lib.ams_fill_iota(self.h, ptr(dst), int(n), int(start)))

    def rlm_sort_run(self, group_counts, scheme: int, master_seed: int, stream_id: str, key_kind: int,
                     pe_sizes, keys, vals, out, out_origin, out_vals):
        """ams_rlm_sort_run: returns (final PE sizes, [RlmReportT])."""
        sz = u64(pe_sizes)
        gc = np.ascontiguousarray(group_counts, dtype=np.int32)
        out_sizes = np.zeros(max(len(sz), 1), np.uint64)
        reps = (RlmReportT * max(len(gc), 1))()
        check(lib.ams_rlm_sort_run(self.h, len(gc), gc.ctypes.data, int(scheme), int(master_seed),
                                   stream_id.encode(), int(key_kind), len(sz), sz.ctypes.data, ptr(keys),
                                   ptr(vals), ptr(out), ptr(out_origin), ptr(out_vals),
                                   out_sizes.ctypes.data, reps))
        return out_sizes[: len(sz)], list(reps)[: len(gc)]

    def rlm_level(self, level: int) -> dict:
        """Host records of one level of the last rlm_sort_run."""
        r, G, P = (C.c_int() for _ in range(3))
        check(lib.ams_rlm_level_dims(self.h, level, C.byref(r), C.byref(G), C.byref(P)))
        r, G, P = r.value, G.value, P.value
        d = {"r": r, "group_first": np.zeros(G, np.int32), "group_npe": np.zeros(G, np.int32),
             "sizes_before": np.zeros(P, np.uint64), "cuts": np.zeros((P, r + 1), np.uint64),
             "new_sizes": np.zeros(P, np.uint64), "stats": np.zeros((G, 4), np.uint64)}
        order = ("group_first", "group_npe", "sizes_before", "cuts", "new_sizes", "stats")
        check(lib.ams_rlm_level(self.h, level, *[d[k].ctypes.data for k in order]))
        return d

    def run_id(self) -> int:
        """Id of the last sort_run (its records stay readable for 8 runs)."""
        return int(lib.ams_run_id(self.h))

    def run_level(self, level: int, run: int = 0) -> dict:
        """Host records of one level of sort_run `run` (0 = the last)."""
        r, G, P, nbs, hs = (C.c_int() for _ in range(5))
        check(lib.ams_run_level_dims_at(self.h, int(run), level, C.byref(r), C.byref(G), C.byref(P),
                                        C.byref(nbs), C.byref(hs)))
        r, G, P, nbs = r.value, G.value, P.value, nbs.value
        d = {"r": r, "group_first": np.zeros(G, np.int32), "group_npe": np.zeros(G, np.int32),
             "sizes_before": np.zeros(P, np.uint64), "drawn": np.zeros(G, np.uint64),
             "nb": np.zeros(G, np.int32), "seg_hist": np.zeros((P, nbs), np.uint32),
             "boundaries": np.zeros((G, r + 1), np.uint64), "loads": np.zeros((G, r), np.uint64),
             "max_load": np.zeros(G, np.uint64), "new_sizes": np.zeros(P, np.uint64),
             "stats": np.zeros((G, 4), np.uint64) if hs.value else None}
        order = ("group_first", "group_npe", "sizes_before", "drawn", "nb", "seg_hist",
                 "boundaries", "loads", "max_load", "new_sizes", "stats")
        check(lib.ams_run_level_at(self.h, int(run), level, *[ptr(d[k]) for k in order]))
        return d

    def run_level_holders(self, level: int, npe: int, run: int = 0) -> np.ndarray:
        """Per PE: splitters of that level drawn from the PE (record_holders runs)."""
        out = np.zeros(max(npe, 1), np.uint32)
        check(lib.ams_run_level_holders_at(self.h, int(run), level, out.ctypes.data))
        return out[:npe]

    def map_keys(self, src, dst, n, from_kind, to_kind):
        check(lib.ams_map_keys(self.h, ptr(src), ptr(dst), n, from_kind, to_kind))
