"""Single-process multi-device AMS-sort: one host
process drives G device contexts through ``ams_mg_sort_run``.

PE i lives on context ``i * G // p``; ``group_counts[0]`` must be a multiple
of G.  Level 1 crosses the devices by peer-pointer stores
(``ams_level_scatter_peers``); everything after it is device-local.  The
one-process-per-GPU form of the same algorithm is
:func:`paper_1410_6754_b200.dist.sort_distributed`.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib as L
from .engine import SCHEMES, key_kind_of, native_params
from .params import as_params, as_seed


class MultiDeviceSorter:
    """``devices`` lists the CUDA device of every context; entries may repeat
    (several contexts on one GPU run the same code path)."""

    def __init__(self, devices):
        if not torch.cuda.is_available():
            raise RuntimeError("MultiDeviceSorter needs CUDA devices (B200, sm_100a); there is no CPU path")
        self.devices = [int(d) for d in devices]
        dv = np.asarray(self.devices, dtype=np.int32)
        h = C.c_void_p()
        L.check(L.lib.ams_mg_create(dv.ctypes.data, len(dv), C.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            L.lib.ams_mg_destroy(self.h)
            self.h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def sort(self, keys, pe_sizes, params, seed, vals=None, scheme: str = "simple", key_kind=None):
        """keys[i]: device tensor of context i's PEs (PE-major).  Returns
        (per-context sorted keys, per-context values or None, final PE sizes,
        level reports as dicts, level-1 record)."""
        if scheme not in SCHEMES:
            raise ValueError(f"unknown delivery scheme {scheme!r}; supported: {tuple(SCHEMES)}")
        G = len(self.devices)
        if len(keys) != G or (vals is not None and len(vals) != G):
            raise ValueError(f"one key (and value) tensor per context is needed ({G})")
        params = as_params(params)
        master, stream_id = as_seed(seed)
        sizes = np.asarray(pe_sizes, dtype=np.uint64)
        p = len(sizes)
        params.validate_for(p)
        if p % G:
            raise ValueError(f"{p} PEs do not divide over {G} contexts")
        pl = p // G
        kind = key_kind_of(keys[0], key_kind)
        for i, t in enumerate(keys):
            want = int(sizes[i * pl:(i + 1) * pl].sum())
            if t.dim() != 1 or not t.is_cuda or t.device.index != self.devices[i] or t.numel() != want \
                    or t.element_size() != 8 or not t.is_contiguous():
                raise ValueError(f"keys[{i}] must be a contiguous CUDA tensor of {want} 8-byte keys on "
                                 f"device {self.devices[i]}")
            if vals is not None and (vals[i].numel() != want or vals[i].device != t.device
                                     or vals[i].element_size() != 8 or not vals[i].is_contiguous()):
                raise ValueError(f"vals[{i}] must match keys[{i}]")
        n = int(sizes.sum())
        # Every device ends with at most r1/G groups of at most (1 + eps') n / r1 keys (ams.py:258).
        r1 = params.group_counts[0]
        eps_l = params.per_level_imbalance()
        cap = int(np.ceil((1.0 + eps_l) * n / r1)) * max(r1 // G, 1) + 16 if n else 1
        outs = [torch.empty(cap, dtype=keys[i].dtype, device=keys[i].device) for i in range(G)]
        outs_v = [torch.empty(cap, dtype=vals[i].dtype, device=vals[i].device) for i in range(G)] \
            if vals is not None else None
        for d in set(self.devices):
            torch.cuda.synchronize(d)  # the contexts run on their own streams
        prm = native_params(params, master, stream_id, kind, True, SCHEMES[scheme], False)
        arr = lambda ts: (C.c_void_p * G)(*[L.ptr(t) if t.numel() else None for t in ts])
        out_sizes = np.zeros(p, np.uint64)
        reps = (L.LevelReportT * prm.levels)()
        L.check(L.lib.ams_mg_sort_run(self.h, C.byref(prm), p, sizes.ctypes.data, arr(keys),
                                      arr(vals) if vals is not None else None, arr(outs),
                                      arr(outs_v) if outs_v is not None else None,
                                      out_sizes.ctypes.data, reps))
        res_k, res_v = [], ([] if outs_v is not None else None)
        for i in range(G):
            cnt = int(out_sizes[i * pl:(i + 1) * pl].sum())
            if cnt > cap:
                raise RuntimeError("a device received more keys than the level-1 load budget allows")
            res_k.append(outs[i][:cnt])
            if res_v is not None:
                res_v.append(outs_v[i][:cnt])
        reports = [{f: int(getattr(r, f)) for f, _ in L.LevelReportT._fields_} for r in reps]
        return res_k, res_v, out_sizes, reports, self.level1()

    def level1(self) -> dict:
        r, p, nbs = C.c_int(), C.c_int(), C.c_int()
        L.check(L.lib.ams_mg_level1_dims(self.h, C.byref(r), C.byref(p), C.byref(nbs)))
        r, p, nbs = r.value, p.value, nbs.value
        d = {"sizes_before": np.zeros(p, np.uint64), "drawn": np.zeros(1, np.uint64),
             "nb": np.zeros(1, np.int32), "seg_hist": np.zeros((p, nbs), np.uint32),
             "boundaries": np.zeros(r + 1, np.uint64), "loads": np.zeros(r, np.uint64),
             "max_load": np.zeros(1, np.uint64), "new_sizes": np.zeros(p, np.uint64),
             "stats": np.zeros(4, np.uint64)}
        order = ("sizes_before", "drawn", "nb", "seg_hist", "boundaries", "loads", "max_load",
                 "new_sizes", "stats")
        L.check(L.lib.ams_mg_level1(self.h, *[d[k].ctypes.data for k in order]))
        d["r"] = r
        return d

    def context(self, i: int) -> L.Context:
        """A non-owning view of the i-th context (records of the later levels)."""
        h = C.c_void_p()
        L.check(L.lib.ams_mg_ctx(self.h, int(i), C.byref(h)))
        c = L.Context.__new__(L.Context)
        c.h, c.device = h, self.devices[i]
        c.close = lambda: None
        return c
