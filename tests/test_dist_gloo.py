"""Multi-rank orchestration (paper_1410_6754_b200/dist.py) over gloo on CPU,
world_size 2 and 4, with oracle-backed device ops: the rank-ordered
concatenation of outputs, per-PE sizes, plans and the payload permutation
must equal the single-process oracle (itself pinned to the reference)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import ams_oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, keys, pe_sizes, groups, vals, q, scheme="simple"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1410_6754_b200.dist import sort_distributed
        from paper_1410_6754_b200 import AmsParams, SeedSpec
        from tests.dist_ops import NumpyOps
        p = len(pe_sizes)
        pl = p // world
        offs = np.concatenate([[0], np.cumsum(pe_sizes)]).astype(np.int64)
        a, b = offs[rank * pl], offs[(rank + 1) * pl]
        k = torch.from_numpy(keys[a:b].view(np.int64).copy())
        v = torch.from_numpy(vals[a:b].copy()) if vals is not None else None
        out, ov, sizes, levels = sort_distributed(
            k, pe_sizes[rank * pl:(rank + 1) * pl], AmsParams(tuple(groups), None, 16, 0.1),
            SeedSpec(5, "algo/rep0"), NumpyOps(), vals=v, key_kind="u64", scheme=scheme)
        q.put((rank, out.numpy().view(np.uint64).copy(),
               None if ov is None else ov.numpy().copy(), [int(x) for x in sizes],
               [lv.boundaries.tolist() for lv in levels]))
    except Exception as e:  # reported to the parent instead of hanging it
        q.put((rank, "error", repr(e), None, None))
    finally:
        dist.destroy_process_group()


def run_world(world, keys, pe_sizes, groups, vals=None, scheme="simple"):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, keys, pe_sizes, groups, vals, q, scheme))
             for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    errors = [r for r in res if isinstance(r[1], str)]
    if errors:
        raise RuntimeError(f"rank errors: {errors}")
    return sorted(res, key=lambda t: t[0])


@pytest.mark.parametrize("world,groups,npe,dist_kind", [
    (2, (8, 8), 600, "uniform"),
    (2, (2, 4), 1000, "zipf"),
    (4, (8, 2), 500, "uniform"),
    (2, (4, 2, 2), 400, "equal"),
])
def test_distributed_matches_oracle(world, groups, npe, dist_kind):
    p = int(np.prod(groups))
    n = p * npe
    rng = np.random.default_rng(world * 100 + npe)
    if dist_kind == "uniform":
        keys = rng.integers(0, 2**64, n, dtype=np.uint64)
    elif dist_kind == "zipf":
        keys = O.zipf_keys(n, 3)
    else:
        keys = np.full(n, 7, dtype=np.uint64)
    pe_sizes = [npe] * p
    vals = np.arange(n, dtype=np.int64)
    ref = O.ams_sort(keys, pe_sizes, groups, None, 16, 0.1, 5, "algo/rep0", vals=vals)
    res = run_world(world, keys, pe_sizes, groups, vals)
    out = np.concatenate([r[1] for r in res])
    ov = np.concatenate([r[2] for r in res])
    sizes = sum((r[3] for r in res), [])
    assert np.array_equal(out, ref.keys)
    assert np.array_equal(ov, ref.vals)
    assert sizes == list(ref.pe_sizes)
    # Level-1 plan replicated on every rank and equal to the oracle's.
    for r in res:
        assert [int(x) for x in r[4][0][0]] == list(ref.levels[0][0].plan.boundaries)


def test_rejects_groups_straddling_ranks():
    keys = np.arange(64, dtype=np.uint64)
    with pytest.raises(RuntimeError, match="multiple of the 4 ranks"):
        run_world(4, keys, [8] * 8, (2, 4))


@pytest.mark.parametrize("scheme", ["deterministic", "permuted", "randomized"])
@pytest.mark.parametrize("world,groups,npe,dist_kind", [
    (2, (4, 4), 250, "sorted"),
    (2, (2, 2, 4), 250, "equal"),
    (4, (8, 2), 300, "zipf"),
    (2, (8,), 400, "uniform"),
])
def test_distributed_other_schemes_match_oracle(scheme, world, groups, npe, dist_kind):
    """Non-simple deliveries (delivery.py:188-455) across ranks: level 1's
    relayout is rank-local, origin tags break ties from level 2 on; keys
    only.  Sorted / equal inputs place members differently from "simple"."""
    p = int(np.prod(groups))
    n = p * npe
    rng = np.random.default_rng(world * 7 + npe)
    keys = {"uniform": lambda: rng.integers(0, 2**64, n, dtype=np.uint64),
            "zipf": lambda: O.zipf_keys(n, 3), "equal": lambda: np.full(n, 7, dtype=np.uint64),
            "sorted": lambda: np.arange(n, dtype=np.uint64)}[dist_kind]()
    pe_sizes = [npe] * p
    ref = O.ams_sort(keys, pe_sizes, groups, None, 16, 0.1, 5, "algo/rep0", scheme=scheme)
    res = run_world(world, keys, pe_sizes, groups, None, scheme)
    assert np.array_equal(np.concatenate([r[1] for r in res]), ref.keys)
    assert sum((r[3] for r in res), []) == list(ref.pe_sizes)
    for r in res:
        assert [int(x) for x in r[4][0][0]] == list(ref.levels[0][0].plan.boundaries)


def test_other_schemes_reject_payloads():
    from paper_1410_6754_b200 import dist as D
    with pytest.raises(ValueError, match="simple delivery scheme only"):
        D.sort_distributed(torch.zeros(8, dtype=torch.int64), [4, 4], (2,), 1, ops=None,
                           vals=torch.zeros(8, dtype=torch.int64), scheme="deterministic")
    with pytest.raises(ValueError, match="unknown delivery scheme"):
        D.sort_distributed(torch.zeros(8, dtype=torch.int64), [4, 4], (2,), 1, ops=None, scheme="x")


@pytest.mark.parametrize("world,groups,npe,dist_kind", [
    (2, (8, 8), 600, "uniform"),
    (4, (8, 2), 500, "zipf"),
    (2, (8,), 900, "uniform"),
    (4, (4, 2, 2), 300, "equal"),
    (2, (16,), 700, "sorted"),
])
def test_distributed_keys_only_matches_oracle(world, groups, npe, dist_kind):
    """Keys only: the last level goes bucket-major into the fixed-capacity
    final sort, single-level runs straight from the level-1 exchange."""
    p = int(np.prod(groups))
    n = p * npe
    rng = np.random.default_rng(world * 10 + npe)
    keys = {"uniform": lambda: rng.integers(0, 2**64, n, dtype=np.uint64),
            "zipf": lambda: O.zipf_keys(n, 3), "equal": lambda: np.full(n, 7, dtype=np.uint64),
            "sorted": lambda: np.arange(n, dtype=np.uint64)}[dist_kind]()
    pe_sizes = [npe] * p
    ref = O.ams_sort(keys, pe_sizes, groups, None, 16, 0.1, 5, "algo/rep0")
    res = run_world(world, keys, pe_sizes, groups, None)
    assert np.array_equal(np.concatenate([r[1] for r in res]), ref.keys)
    assert sum((r[3] for r in res), []) == list(ref.pe_sizes)
    for r in res:
        assert [int(x) for x in r[4][0][0]] == list(ref.levels[0][0].plan.boundaries)
