"""Multi-GPU host helpers (BASELINE north_star): one process per GPU, field points
partitioned across ranks by cost-weighted contiguous Morton ranges (cylfmm_partition_fields),
the rank's contiguous source shard, and the optional gather of the per-rank outputs.  The
device solve replicates the sources and the leaf moments itself (cylfmm_fmm_solve_dist, a
library-owned NCCL communicator: Plan(cfg, dist=(nranks, rank, comm_unique_id()))); the
torch.distributed all-gather helpers below serve the output gather and the gloo CPU tests.

The FMM result at a field point depends only on the sources and on its own box chain, so each
rank's solve over its own field points reproduces the single-GPU values bitwise."""
from __future__ import annotations

import numpy as np

from .cylfmm import FMMConfig, partition_fields


def source_shard(n_src: int, rank: int, world: int) -> slice:
    """Contiguous block of the source list owned by `rank` before the all-gather."""
    return slice(rank * n_src // world, (rank + 1) * n_src // world)


def _allgather_rows(t, group=None):
    """All-gather row blocks of possibly different lengths (padded to the longest block: NCCL
    and gloo all-gather equal-sized buffers); complex tensors travel as real views."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    n_loc = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
    sizes = [torch.zeros_like(n_loc) for _ in range(world)]
    dist.all_gather(sizes, n_loc, group=group)
    sizes = [int(s.item()) for s in sizes]
    nmax = max(sizes)
    x = torch.view_as_real(t.contiguous()) if t.is_complex() else t.contiguous()
    pad = torch.zeros((nmax,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
    pad[: x.shape[0]] = x
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    out = torch.cat([b[:n] for b, n in zip(bufs, sizes)], dim=0)
    return torch.view_as_complex(out) if t.is_complex() else out


def allgather_sources(parts, group=None):
    """Replicate the sources: all-gather the per-rank shards [(r, z, S), ...] (torch tensors on
    the rank's device) into the full (r, z, S) on every rank, in rank order."""
    return tuple(_allgather_rows(t, group) for t in parts)


def field_partition(src_r, src_z, fld_r, fld_z, cfg: FMMConfig, world: int):
    """Identical on every rank: (part of each field point, estimated cost per part)."""
    return partition_fields(np.asarray(src_r), np.asarray(src_z), np.asarray(fld_r),
                            np.asarray(fld_z), cfg, world)


def my_fields(part: np.ndarray, rank: int) -> np.ndarray:
    """Input-order indices of the field points this rank evaluates."""
    return np.flatnonzero(part == rank)


def gather_outputs(local_out, idx_local: np.ndarray, n_fld: int, group=None):
    """Assemble the full [n_fld, K] output on every rank from the per-rank rows (all-gather of
    the row blocks and of their input-order indices)."""
    import torch
    rows = _allgather_rows(local_out, group)
    idx = _allgather_rows(torch.as_tensor(idx_local, dtype=torch.int64, device=local_out.device),
                          group)
    full = torch.empty((n_fld, local_out.shape[1]), dtype=local_out.dtype, device=local_out.device)
    full[idx] = rows
    return full
