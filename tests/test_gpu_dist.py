"""Multi-GPU level 1 on the B200 (dist.py + ams_level_scatter_peers).

* world 1 over NCCL: the peer scatter writes into this GPU's own receive
  buffer;
* world 2 as two processes on ONE GPU over gloo: each process maps the
  other's receive buffer with CUDA IPC and its level-1 scatter stores into it
  (the same peer-pointer path as across GPUs; no kernel waits on another —
  the ranks synchronise on the host).
Both must equal the oracle (output, payload permutation, per-PE sizes, plan)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import ams_oracle as O

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _case(groups, npe, dist_kind, seed=4):
    p = int(np.prod(groups))
    n = p * npe
    rng = np.random.default_rng(seed)
    keys = {"uniform": lambda: rng.integers(0, 2**64, n, dtype=np.uint64),
            "zipf": lambda: O.zipf_keys(n, 3), "sorted": lambda: np.arange(n, dtype=np.uint64)}[dist_kind]()
    return keys, [npe] * p


def _run_rank(rank, world, port, keys, sizes, groups, with_vals, backend, q, scheme="simple"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        torch.cuda.set_device(0)
        dist.init_process_group(backend, rank=rank, world_size=world)
        from paper_1410_6754_b200 import AmsParams, SeedSpec
        from paper_1410_6754_b200.api import get_sorter
        from paper_1410_6754_b200.dist import CudaOps, sort_distributed
        p = len(sizes)
        pl = p // world
        offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        a, b = offs[rank * pl], offs[(rank + 1) * pl]
        k = torch.from_numpy(keys[a:b].view(np.int64).copy()).cuda()
        v = torch.arange(a, b, dtype=torch.int64, device="cuda") if with_vals else None
        ops = CudaOps(get_sorter(0))
        outs = []
        for _ in range(2):  # twice: the second reuses the mapped peer buffers
            out, ov, sz, levels = sort_distributed(k, sizes[rank * pl:(rank + 1) * pl],
                                                   AmsParams(groups, None, 16, 0.1),
                                                   SeedSpec(5, "algo/rep0"), ops, vals=v, key_kind="u64",
                                                   scheme=scheme)
            torch.cuda.synchronize()
            outs.append((out.cpu().numpy().view(np.uint64).copy(),
                         None if ov is None else ov.cpu().numpy().copy(), [int(x) for x in sz],
                         [int(x) for x in levels[0].boundaries[0]],
                         [[[int(x) for x in row] for row in lv.boundaries] for lv in levels]))
        q.put((rank, outs))
    except Exception as e:  # reported to the parent instead of hanging it
        q.put((rank, repr(e)))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def _spawn(world, keys, sizes, groups, with_vals, backend, scheme="simple"):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_run_rank,
                         args=(r, world, port, keys, sizes, groups, with_vals, backend, q, scheme))
             for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
    bad = [r for r in res if isinstance(r[1], str)]
    assert not bad, bad
    return sorted(res, key=lambda t: t[0])


@pytest.mark.parametrize("world,backend", [(1, "nccl"), (2, "gloo")], ids=["world1-nccl", "world2-ipc"])
@pytest.mark.parametrize("groups,npe,dist_kind,with_vals", [
    ((8, 8), 3000, "uniform", True), ((8, 8), 3000, "uniform", False),
    ((4, 4), 5000, "zipf", True), ((8,), 9000, "sorted", False), ((2, 4, 2), 2000, "uniform", False),
])
def test_level1_peer_exchange_matches_oracle(world, backend, groups, npe, dist_kind, with_vals):
    keys, sizes = _case(groups, npe, dist_kind)
    n = len(keys)
    ref = O.ams_sort(keys, sizes, groups, None, 16, 0.1, 5, "algo/rep0",
                     vals=np.arange(n, dtype=np.int64) if with_vals else None)
    res = _spawn(world, keys, sizes, groups, with_vals, backend)
    for it in range(2):
        out = np.concatenate([r[1][it][0] for r in res])
        assert np.array_equal(out, ref.keys)
        if with_vals:
            assert np.array_equal(np.concatenate([r[1][it][1] for r in res]), ref.vals)
        assert sum((r[1][it][2] for r in res), []) == list(ref.pe_sizes)
        for r in res:
            assert r[1][it][3] == list(ref.levels[0][0].plan.boundaries)



def _later_boundaries(ref, world, rank):
    """The oracle's plan boundaries of levels >= 2 for the groups a rank owns."""
    out = []
    for infos in ref.levels[1:]:
        per = len(infos) // world
        out.append([list(i.plan.boundaries) for i in infos[rank * per:(rank + 1) * per]])
    return out


@pytest.mark.parametrize("world,backend", [(1, "nccl"), (2, "gloo")], ids=["world1-nccl", "world2-ipc"])
@pytest.mark.parametrize("scheme", ["deterministic", "permuted", "randomized"])
@pytest.mark.parametrize("groups,npe,dist_kind", [
    ((4, 4), 3000, "sorted"), ((8, 8), 2000, "uniform"), ((2, 2, 4), 2500, "zipf"), ((16,), 4000, "uniform"),
])
def test_other_schemes_across_ranks_match_oracle(world, backend, scheme, groups, npe, dist_kind):
    """Non-simple deliveries on the multi-GPU path (rank-local level-1
    relayout, origin tags from level 2 on, ams_sort_run continuation)."""
    keys, sizes = _case(groups, npe, dist_kind)
    ref = O.ams_sort(keys, sizes, groups, None, 16, 0.1, 5, "algo/rep0", scheme=scheme)
    res = _spawn(world, keys, sizes, groups, False, backend, scheme)
    for it in range(2):
        assert np.array_equal(np.concatenate([r[1][it][0] for r in res]), ref.keys)
        assert sum((r[1][it][2] for r in res), []) == list(ref.pe_sizes)
        for rank, r in enumerate(res):
            assert r[1][it][3] == list(ref.levels[0][0].plan.boundaries)
            assert r[1][it][4][1:] == _later_boundaries(ref, world, rank)


def test_later_levels_records_simple_world2():
    """The continuation's level records (levels >= 2) equal the oracle's."""
    groups = (4, 2, 2)
    keys, sizes = _case(groups, 3000, "uniform")
    ref = O.ams_sort(keys, sizes, groups, None, 16, 0.1, 5, "algo/rep0")
    res = _spawn(2, keys, sizes, groups, False, "gloo")
    for rank, r in enumerate(res):
        assert r[1][0][4][1:] == _later_boundaries(ref, 2, rank)
