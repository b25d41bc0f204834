"""Multi-rank host logic of the field-partitioned solve with world_size 2 over gloo
on the CPU: source shards replicated by all-gather (the library does it with NCCL inside
cylfmm_fmm_solve_dist), the cost-weighted Morton field partition (cylfmm_partition_fields,
host-only, identical on every rank), per-rank solves over the rank's own field points and the
output gather.  There is no GPU here, so the per-rank solve is the oracle FMM (test
infrastructure) standing in for the device solve; the device side of the same claim -- each
part solved through libcylfmm equals the one-solve result bit for bit -- is
tests/test_gpu_parity.py::test_partitioned_solve_bitwise, and the library's NCCL path is
test_dist_solve_single_rank_bitwise."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from tests.inputs import uniform_rings


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem():
    rng = np.random.default_rng(31)
    sr, sz, S = uniform_rings(rng, 1500, 4)
    fr, fz, _ = uniform_rings(rng, 700, 1)
    return sr, sz, S, fr, fz


def _worker(rank, world, port, outdir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2301_01179_b200 import FMMConfig
        from paper_2301_01179_b200 import distributed as dd
        sr, sz, S, fr, fz = _problem()
        cfg = FMMConfig(n_modes=4, order=6, depth=4)
        # 1. sources: each rank owns a shard, replicated by all-gather
        sl = dd.source_shard(len(sr), rank, world)
        r, z, Sf = dd.allgather_sources((torch.as_tensor(sr[sl]), torch.as_tensor(sz[sl]),
                                         torch.as_tensor(S[sl])))
        assert np.array_equal(r.numpy(), sr) and np.array_equal(Sf.numpy(), S)
        # 2. identical partition on every rank
        part, cost = dd.field_partition(r.numpy(), z.numpy(), fr, fz, cfg, world)
        allp = [torch.zeros(len(fr), dtype=torch.int32) for _ in range(world)]
        dist.all_gather(allp, torch.as_tensor(part))
        assert all(np.array_equal(a.numpy(), part) for a in allp)
        # 3. per-rank solve over its own field points (oracle stands in for the device solve)
        idx = dd.my_fields(part, rank)
        loc, _ = oracle.fmm(r.numpy(), z.numpy(), Sf.numpy(), fr[idx], fz[idx], cfg.order,
                            cfg.depth, cfg.L, cfg.z0)
        # 4. gather
        full = dd.gather_outputs(torch.as_tensor(loc), idx, len(fr))
        if rank == 0:
            np.save(os.path.join(outdir, "full.npy"), full.numpy())
            np.save(os.path.join(outdir, "part.npy"), part)
            np.save(os.path.join(outdir, "cost.npy"), cost)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_two_rank_field_partition_matches_single_process(tmp_path, orc):
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    full = np.load(tmp_path / "full.npy")
    part = np.load(tmp_path / "part.npy")
    cost = np.load(tmp_path / "cost.npy")
    sr, sz, S, fr, fz = _problem()
    ref, _ = orc.fmm(sr, sz, S, fr, fz, 6, 4, 1.0, 0.0)
    assert np.array_equal(full, ref)
    assert set(np.unique(part)) == {0, 1}
    assert cost.max() / cost.mean() < 1.25


def test_partition_is_contiguous_in_morton_order_and_balanced(orc):
    from paper_2301_01179_b200 import FMMConfig, partition_fields
    from tests.inputs import config_c4
    pr = config_c4(n=65536)
    cfg = FMMConfig(n_modes=pr.K, order=pr.p, depth=6, L=pr.L)
    for world in (1, 2, 4, 8):
        part, cost = partition_fields(pr.sr, pr.sz, pr.fr, pr.fz, cfg, world)
        key, _ = orc.tree_keys(pr.fr, pr.fz, 6, pr.L, 0.0)
        order = np.argsort(key, kind="stable")
        assert np.all(np.diff(part[order]) >= 0)          # contiguous Morton ranges
        assert part.min() == 0 and part.max() == world - 1
        assert abs(cost.sum() / cost.mean() - world) < 1e-9
        assert cost.max() / cost.mean() < 1.3


def test_partition_rejects_points_outside_domain():
    from paper_2301_01179_b200 import CylFMMError, FMMConfig, partition_fields
    cfg = FMMConfig(n_modes=2, order=4, depth=3)
    with pytest.raises(CylFMMError) as ei:
        partition_fields(np.array([0.5]), np.array([0.5]), np.array([1.5]), np.array([0.5]), cfg, 2)
    assert ei.value.status == 2
