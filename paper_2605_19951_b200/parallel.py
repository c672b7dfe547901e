"""Pole sharding across GPUs (one process per GPU) and the ordered exchange.

Mirrors PoleWorkerPool (/root/reference/pkg/src/rbainv/shifted.py:129-155):
rank r owns poles {i : i mod G == r}.  After each action (forward, J v,
J^T w) every rank holds per-pole partials for its own poles; they are
all-gathered (NCCL over NVLink on GPUs, gloo on CPU) into a
[rank][local slot] array and summed on every rank in ascending *global* pole
order by the combine kernels, so the result is bitwise independent of G --
the reference's worker-count invariance (SPEC.md:220,
pkg/tests/test_acceptance.py:212-234).
"""

from __future__ import annotations

import math

import numpy as np
import torch
import torch.distributed as dist

__all__ = ["PoleComm", "ShardComm", "owned_poles", "gathered_slot_of_pole"]


def owned_poles(m: int, world: int, rank: int) -> list[int]:
    return [i for i in range(m) if i % world == rank]


def gathered_slot_of_pole(m: int, world: int) -> np.ndarray:
    """Row of pole i in the all-gathered [world * n_max] partial array."""
    n_max = math.ceil(m / world)
    return np.array([(i % world) * n_max + i // world for i in range(m)], dtype=np.int32)


class PoleComm:
    def __init__(self, world: int = 1, rank: int = 0, group=None):
        self.world = int(world)
        self.rank = int(rank)
        self.group = group

    @classmethod
    def current(cls) -> "PoleComm":
        if dist.is_available() and dist.is_initialized():
            return cls(dist.get_world_size(), dist.get_rank())
        return cls(1, 0)

    def local_poles(self, m: int) -> list[int]:
        return owned_poles(m, self.world, self.rank)

    def slot_of_pole(self, m: int) -> np.ndarray:
        if self.world == 1:
            return np.arange(m, dtype=np.int32)
        return gathered_slot_of_pole(m, self.world)

    def gather_partials(self, part: torch.Tensor) -> torch.Tensor:
        """[n_local, ...] -> [world * n_max, ...] (rank-major), padded rows zero."""
        if self.world == 1:
            return part
        # every rank allocates n_max = ceil(m / G) rows, so sizes agree
        src = part.contiguous()
        if src.is_complex():
            src = torch.view_as_real(src)
        out = torch.empty((self.world * src.shape[0],) + tuple(src.shape[1:]),
                          dtype=src.dtype, device=src.device)
        dist.all_gather_into_tensor(out, src, group=self.group)
        return torch.view_as_complex(out) if part.is_complex() else out

    def agree_min(self, value: int) -> int:
        """Minimum of an integer over the ranks (mode decisions all ranks share)."""
        if self.world == 1:
            return int(value)
        t = torch.tensor([int(value)], dtype=torch.int64,
                         device="cuda" if dist.get_backend(self.group) == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=self.group)
        return int(t.item())

    def n_max(self, m: int) -> int:
        return math.ceil(m / self.world)

    def barrier(self):
        if self.world > 1:
            dist.barrier(group=self.group)


class ShardComm(PoleComm):
    """Rank `rank` of a G-rank pole sharding run inside ONE process (no
    collective): used to time or check each rank's share on one device --
    scaling_benchmark's per-shard timings, the bitwise multi-GPU tests.  The
    caller concatenates the shards' partials rank-major itself."""

    def agree_min(self, value: int) -> int:
        return int(value)

    def gather_partials(self, part):
        raise RuntimeError("ShardComm has no collective: concatenate the shards' partials")

    def barrier(self):
        pass
