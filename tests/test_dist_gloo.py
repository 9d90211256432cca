"""Multi-process (world_size 2, gloo, CPU) coverage of the series-sharded
path: shard plan per rank, per-rank transform, ordered all-gather equals
the single-process result (reference engine.py:336-364; the GPU transform
is stood in for by the pinned oracle, which is test infrastructure)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import sys

    import torch
    import torch.distributed as dist

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.dirname(here))
    sys.path.insert(0, here)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import golden_cases as gc
        from oracle.oracle import oracle_transform
        from paper_2601_17091_b200.distributed import gather_rows, shard_of, sharded_transform

        case = gc.CASES["rc11"]
        values = gc.case_values(case)
        bank = gc.make_bank(gc.BANKS[case["bank"]])
        start, feats = sharded_transform(values, bank, lambda rows: oracle_transform(rows, bank, nthreads=1))
        assert (start, feats.shape[0]) == shard_of(values.shape[0], world, rank)
        full = gather_rows(torch.from_numpy(feats), values.shape[0])
        q.put((rank, full.numpy().tobytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_shard_and_gather_equals_single(golden_transforms):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    expected = golden_transforms["rc11/single"].tobytes()
    assert results[0] == expected and results[1] == expected


def _ridge_worker(rank, world, port, q, name):
    import sys

    import torch.distributed as dist

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, os.path.dirname(here))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2601_17091_b200 import ridge
        from paper_2601_17091_b200.distributed import shard_of

        with np.load(os.path.join(here, "golden", "ridge.npz")) as z:
            feats, labels = z[f"{name}/features"], [str(v) for v in z["labels"]]
        start, count = shard_of(feats.shape[0], world, rank)
        m = ridge.fit_sharded(feats[start : start + count], labels[start : start + count], alpha=1.0,
                              device="cpu")
        q.put((rank, m.weights, m.feature_means, m.feature_scales))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("name", ["primal", "dual"])
def test_two_rank_sharded_ridge_equals_reference(name):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ridge_worker, args=(r, world, port, q, name)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    here = os.path.dirname(os.path.abspath(__file__))
    with np.load(os.path.join(here, "golden", "ridge.npz")) as z:
        for _, w, mu, sd in results:
            np.testing.assert_allclose(w, z[f"{name}/weights"], rtol=1e-8, atol=1e-11)
            np.testing.assert_allclose(mu, z[f"{name}/means"], rtol=1e-12, atol=1e-14)
            np.testing.assert_allclose(sd, z[f"{name}/scales"], rtol=1e-12, atol=1e-14)
