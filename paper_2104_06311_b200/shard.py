"""Multi-GPU host logic: contiguous frame-range shards with halos and the counter reduction.

SURVEY §8(e) / BASELINE.json north_star: "The stream is sharded across 1/2/4/8 GPUs of one box as contiguous
frame ranges with overlap halos. Only the error/Q counters are combined, by an NCCL allreduce over NVLink."
Every grid of the chain is anchored at global sample 0, so a shard's decisions are bit-identical to the
same frames processed by one GPU (tests/test_gpu_parity.py::test_chunk_and_shard_invariance).
There is no data-path collective: a rank reads its core samples plus `halo` samples on each side.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List

FRAME_SAMPLES = 16384
HALO = 16640            # kk_halo(): one neighbour frame + half a Hilbert block
HALO_UP = 16656         # kk_halo() with upsample = 2 (+16 for the half-band interpolator)


@dataclass(frozen=True)
class Shard:
    rank: int
    first: int          # global index of the first core sample (multiple of FRAME_SAMPLES)
    n: int              # core samples (multiple of FRAME_SAMPLES)
    halo: int = HALO    # kk_halo() of the receiver configuration

    @property
    def read_first(self) -> int:   # first global sample the rank must hold
        return self.first - self.halo

    @property
    def read_count(self) -> int:
        return self.n + 2 * self.halo

    @property
    def frames(self) -> range:
        return range(self.first // FRAME_SAMPLES, (self.first + self.n) // FRAME_SAMPLES)


def plan_strong(total_samples: int, world: int, stream_first: int = 0, halo: int = HALO) -> List[Shard]:
    """Split one stream of `total_samples` into `world` contiguous frame ranges (sizes differ by ≤ 1 frame)."""
    assert total_samples % FRAME_SAMPLES == 0 and stream_first % FRAME_SAMPLES == 0 and world >= 1
    nf = total_samples // FRAME_SAMPLES
    out = []
    for r in range(world):
        f0 = (r * nf) // world
        f1 = ((r + 1) * nf) // world
        out.append(Shard(r, stream_first + f0 * FRAME_SAMPLES, (f1 - f0) * FRAME_SAMPLES, halo))
    return out


def plan_weak(samples_per_rank: int, world: int, stream_first: int = 0, halo: int = HALO) -> List[Shard]:
    """Each rank owns `samples_per_rank` consecutive samples of one global stream (fixed per-GPU work)."""
    assert samples_per_rank % FRAME_SAMPLES == 0 and stream_first % FRAME_SAMPLES == 0
    return [Shard(r, stream_first + r * samples_per_rank, samples_per_rank, halo) for r in range(world)]


def allreduce_counters(counters, group=None):
    """Sum the 24 int64 counter words of all ranks in place (the only cross-GPU data movement).
    Integer sums: the result is independent of the reduction order."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(counters, op=dist.ReduceOp.SUM, group=group)
    return counters


def max_over_ranks(value: float, device="cpu", group=None) -> float:
    """Max of a per-rank float (e.g. elapsed time) — the contract's max-over-ranks timing."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
