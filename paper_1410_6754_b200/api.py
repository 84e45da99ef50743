"""Public entry points.

* :func:`ams_sort` — drop-in for the reference's
  ``mlpsort.ams.ams_sort(net, data, params, scheme, seed)``
  (ams.py:271-313): same arguments, same return structure
  ``(dict[pe] -> sorted list of Elements, level_reports)``.
* :func:`ams_sort_tensors` — the same sort over a device tensor of keys
  (optionally with 8-byte payloads), no Python objects per element.
* :func:`ams_sort_host` — host (numpy) buffers in, host buffers out; the
  end-to-end path (H2D, sort, D2H) a user without device buffers calls.
* :class:`HostSortPipeline` — a stream of host batches sorted with the
  copies overlapped: the H2D of batch i+1 and the D2H of batch i-1 run on
  their own CUDA streams while batch i sorts.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib as L
from . import ledger
from .engine import AmsSorter, SortOutput
from .params import Element, as_params, as_seed

_SORTERS: dict = {}

SUPPORTED_SCHEMES = ("simple", "deterministic", "permuted", "randomized")


def get_sorter(device=None) -> AmsSorter:
    idx = torch.cuda.current_device() if device is None else (
        device.index if isinstance(device, torch.device) else int(device))
    s = _SORTERS.get(idx)
    if s is None:
        s = _SORTERS[idx] = AmsSorter(idx)
    return s


def _check_scheme(scheme: str):
    if scheme not in SUPPORTED_SCHEMES:
        raise ValueError(
            f"delivery scheme {scheme!r} is not implemented on the B200 path; "
            f"supported: {SUPPORTED_SCHEMES} (delivery.py:151-455)")


def ams_sort_tensors(keys: torch.Tensor, pe_sizes, params, seed, vals: torch.Tensor | None = None,
                     scheme: str = "simple", key_kind=None, out=None, out_vals=None,
                     record_splitters: bool = False, record_holders: bool = False,
                     sample_mode: str = "parity") -> SortOutput:
    """Sort device keys laid out PE-major (``pe_sizes``); returns a
    :class:`~paper_1410_6754_b200.engine.SortOutput`.  ``sample_mode``:
    "parity" draws the sample positions from the reference's seeded streams
    (bucket boundaries equal the reference's); "device" draws stratified
    positions on the GPU (same quota split, ams.py:166-171; no host draw —
    the output and the (1 + eps) bound are unchanged, the boundaries are not
    the reference's)."""
    _check_scheme(scheme)
    return get_sorter(keys.device).sort(keys, pe_sizes, params, seed, vals=vals, out=out,
                                        out_vals=out_vals, key_kind=key_kind,
                                        record_splitters=record_splitters, scheme=scheme,
                                        record_holders=record_holders, sample_mode=sample_mode)


def ams_sort_host(keys: np.ndarray, pe_sizes, params, seed, vals: np.ndarray | None = None,
                  device=None, key_kind=None):
    """Host buffers in and out: pinned H2D copy, device sort, D2H copy.
    Returns (sorted keys ndarray, sorted vals ndarray or None, pe_sizes,
    reports)."""
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else int(device))
    kt = torch.from_numpy(np.ascontiguousarray(keys))
    d_keys = kt.pin_memory().to(dev, non_blocking=True)
    d_vals = None
    if vals is not None:
        d_vals = torch.from_numpy(np.ascontiguousarray(vals)).pin_memory().to(dev, non_blocking=True)
    res = ams_sort_tensors(d_keys, pe_sizes, params, seed, vals=d_vals, key_kind=key_kind)
    out_k = res.keys.cpu().numpy()
    out_v = res.vals.cpu().numpy() if res.vals is not None else None
    return out_k, out_v, res.pe_sizes, res.reports


class HostSortPipeline:
    """Sort many same-shaped host batches (pinned CPU tensors of n 8-byte
    keys, PE-major ``pe_sizes``) end to end with copy/compute overlap.

    Two device input and two output buffers alternate: while batch i sorts
    on the compute stream, batch i+1 is copied in on a copy stream and batch
    i-1 is copied out on another (PCIe is full duplex, so both directions run
    at once).  Every batch still makes the full trip host -> device -> host.
    """

    def __init__(self, n: int, pe_sizes, params, seed, key_kind="u64", device=None):
        self.dev = torch.device("cuda", torch.cuda.current_device() if device is None else int(device))
        self.n = int(n)
        self.pe_sizes = np.asarray(pe_sizes, dtype=np.uint64)
        if int(self.pe_sizes.sum()) != self.n:
            raise ValueError("pe_sizes must sum to n")
        self.params, self.seed, self.key_kind = params, seed, key_kind
        mk = lambda: torch.empty(max(self.n, 1), dtype=torch.int64, device=self.dev)
        self.d_in = [mk(), mk()]
        self.d_out = [mk(), mk()]
        self.s_in = torch.cuda.Stream(self.dev)
        self.s_out = torch.cuda.Stream(self.dev)
        self.ev_in = [torch.cuda.Event(), torch.cuda.Event()]      # H2D into d_in[j] done
        self.ev_sorted = [torch.cuda.Event(), torch.cuda.Event()]  # sort reading d_in[j] done
        self.ev_out = [torch.cuda.Event(), torch.cuda.Event()]     # D2H from d_out[j] done
        self.sorter = get_sorter(self.dev)

    def _h2d(self, j, host):
        with torch.cuda.stream(self.s_in):
            self.d_in[j][: self.n].copy_(host.view(torch.int64), non_blocking=True)
            self.ev_in[j].record(self.s_in)

    def run(self, inputs, outputs, done_events=None):
        """Sort inputs[i] into outputs[i] (pinned CPU tensors); returns the
        final per-PE sizes of every batch.  Blocks until the last D2H ends.
        ``done_events`` (optional list) receives one timing event per batch,
        recorded when its D2H has completed."""
        if len(inputs) != len(outputs):
            raise ValueError("one output per input")
        for t in list(inputs) + list(outputs):
            if t.device.type != "cpu" or t.numel() != self.n or t.element_size() != 8:
                raise ValueError("inputs/outputs must be CPU tensors of n 8-byte keys")
        comp = torch.cuda.current_stream(self.dev)
        sizes = []
        if inputs:
            self._h2d(0, inputs[0])
        for i, (hin, hout) in enumerate(zip(inputs, outputs)):
            j = i % 2
            if i + 1 < len(inputs):
                # d_in[1 - j] was last read by sort(i - 1).
                self.s_in.wait_event(self.ev_sorted[1 - j])
                self._h2d(1 - j, inputs[i + 1])
            comp.wait_event(self.ev_in[j])
            comp.wait_event(self.ev_out[j])  # d_out[j] was last read by D2H(i - 2)
            res = self.sorter.sort(self.d_in[j][: self.n], self.pe_sizes, self.params, self.seed,
                                   out=self.d_out[j][: self.n], key_kind=self.key_kind,
                                   with_stats=False)
            self.ev_sorted[j].record(comp)
            sizes.append(res.pe_sizes)
            with torch.cuda.stream(self.s_out):
                self.s_out.wait_event(self.ev_sorted[j])
                hout.view(torch.int64).copy_(self.d_out[j][: self.n], non_blocking=True)
                self.ev_out[j].record(self.s_out)
                if done_events is not None:
                    ev = torch.cuda.Event(enable_timing=True)
                    ev.record(self.s_out)
                    done_events.append(ev)
        self.s_out.synchronize()
        return sizes


def _flatten(data, p):
    keys, tags = [], []
    sizes = np.zeros(p, dtype=np.uint64)
    flat = []
    for pe in range(p):
        seq = data[pe]
        sizes[pe] = len(seq)
        flat.extend(seq)
    return flat, sizes


def ams_sort(net, data, params, scheme: str, seed):
    """Drop-in for ``mlpsort.ams.ams_sort`` (ams.py:271-313).

    ``net`` needs ``.p`` (the reference's ``Network``).  When it also has a
    ``ledger``, the ledger is charged exactly as
    the reference charges it (phases, per-PE words/messages, modeled time;
    ``ledger.charge_sort`` from the device run's level records), for every
    scheme of the reference's ``SCHEMES`` registry.
    Elements keep their identity: the returned lists hold the caller's own
    Element objects.  Requires origin tags that increase along the PE-major
    concatenation (as ``generate_input`` produces, bench.py:176), which makes
    the reference's (key, origin_pe, origin_pos) order equal to the
    (key, position) order the device uses.
    """
    _check_scheme(scheme)
    params = as_params(params)
    p = int(net.p)
    params.validate_for(p)
    flat, sizes = _flatten(data, p)
    n = len(flat)
    if n:
        tags = np.array([(e.origin_pe, e.origin_pos) for e in flat], dtype=np.int64)
        if n > 1:
            d0 = np.diff(tags[:, 0])
            d1 = np.diff(tags[:, 1])
            if np.any((d0 < 0) | ((d0 == 0) & (d1 <= 0))):
                raise ValueError("element origin tags must increase along the PE-major input "
                                 "order for the B200 path (tie-break by position)")
        ks = [int(e.key) for e in flat]
        lo, hi = min(ks), max(ks)
        if lo < 0:
            if lo < -(1 << 63) or hi >= (1 << 63):
                raise ValueError("keys must fit in 64 bits")
            keys = np.array(ks, dtype=np.int64)
            kind = "i64"
        else:
            if hi >= (1 << 64):
                raise ValueError("keys must fit in 64 bits")
            keys = np.array(ks, dtype=np.uint64)
            kind = "u64"
    else:
        keys = np.zeros(0, dtype=np.uint64)
        kind = "u64"
    dev = torch.device("cuda", torch.cuda.current_device())
    d_keys = torch.from_numpy(keys.view(np.int64)).to(dev)
    d_vals = torch.arange(n, dtype=torch.int64, device=dev)
    charge = scheme in ledger.CHARGED_SCHEMES and getattr(net, "ledger", None) is not None
    res = ams_sort_tensors(d_keys, sizes, params, seed, vals=d_vals, key_kind=kind, scheme=scheme,
                           record_holders=charge)
    if charge:
        ledger.charge_sort(net, res.levels, params, params.oversampling_for(n), scheme,
                           *as_seed(seed))
    order = res.vals.cpu().numpy()
    out, start = {}, 0
    for pe in range(p):
        cnt = int(res.pe_sizes[pe])
        out[pe] = [flat[i] for i in order[start:start + cnt]]
        start += cnt
    return out, res.reports
