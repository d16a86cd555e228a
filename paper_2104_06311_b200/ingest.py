"""Single-ingest distribution: one rank owns the ADC stream and feeds every rank.

PAPER.md:82: "Buffers containing 2^22 samples are transferred using DMA from the 4 GS/s ADC to the GPU" —
the paper has one ADC and one GPU. With several GPUs in one box the ADC still lands in ONE host/GPU; this
module carries it from there to the others: the source rank copies each rank's read window (its core
chunk plus the kk_halo() samples on both sides, shard.Shard) from pinned host memory to its device and
sends it point-to-point (NCCL over NVLink on GPUs, gloo on CPU tests); every rank receives its window into
one of two buffers and hands it to `process` while the next window is in flight. The per-rank data path
is unchanged (kk_process_frames on the window), so decisions and counters are bit-identical to local
ingest — only the bytes move differently. No collective besides these sends; halos are sent twice (to
the two ranks that share them), ≈ 2·halo/chunk extra bytes.

Plumbing only (marshalling + torch.distributed); the receive chain itself is the C ABI.
"""
from __future__ import annotations

from typing import Callable, List, Optional

import torch
import torch.distributed as dist

from .shard import Shard


def window_bounds(shard: Shard, c0: int, nc: int):
    """Global [start, stop) of the samples rank `shard.rank` needs for its core chunk [first + c0, + nc)."""
    s = shard.first + c0 - shard.halo
    return s, s + nc + 2 * shard.halo


def distribute(shards: List[Shard], chunk: int, process: Callable[[torch.Tensor, int, int], None],
               host_stream: Optional[torch.Tensor] = None, stream_first: int = 0, src: int = 0,
               device: Optional[torch.device] = None, dtype=torch.int16, group=None) -> int:
    """Feed every rank its windows from the source rank and call `process(window, first_sample, n)` on each.

    shards:      the plan (shard.plan_weak / plan_strong with the receiver's halo), same on every rank.
    host_stream: on the source rank only — the samples of global [stream_first, …) covering every window
                 (pinned host memory for the GPU path); None elsewhere.
    window:      a tensor of n + 2·halo samples on `device`; element halo is global sample first_sample.
    Returns the number of samples this rank received (core + halos).
    """
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    assert len(shards) == world
    dev = device if device is not None else torch.device("cpu")
    if dev.type == "cuda":
        return _distribute_cuda(shards, chunk, process, host_stream, stream_first, src, dev, dtype, group,
                                rank, world)
    me = shards[rank]
    halo = me.halo
    n_max = max(s.n for s in shards)
    bufs = [torch.empty(chunk + 2 * halo, dtype=dtype, device=dev) for _ in range(2)]
    received = 0
    k = 0
    for c0 in range(0, n_max, chunk):
        buf = bufs[k & 1]
        if rank == src:
            assert host_stream is not None
            for r, sh in enumerate(shards):
                if c0 >= sh.n:
                    continue
                a, b = window_bounds(sh, c0, min(chunk, sh.n - c0))
                view = host_stream[a - stream_first:b - stream_first]
                assert view.numel() == b - a, "host stream does not cover the window"
                if r == rank:
                    buf[:b - a].copy_(view)
                else:
                    dist.send(view.contiguous(), dst=r, group=group)
        elif c0 < me.n:
            a, b = window_bounds(me, c0, min(chunk, me.n - c0))
            dist.recv(buf[:b - a], src=src, group=group)
        if c0 < me.n:
            nc = min(chunk, me.n - c0)
            process(buf[:nc + 2 * halo], me.first + c0, nc)
            received += nc + 2 * halo
        k += 1
    return received


def _distribute_cuda(shards, chunk, process, host_stream, stream_first, src, dev, dtype, group, rank, world):
    """GPU path: H2D copies and the NCCL point-to-point transfers run on a side stream `xs`; `process` runs
    on the caller's current stream `cs`. Two receive buffers: chunk k+1 moves while chunk k is processed;
    events order buffer reuse. On the source, two staging buffers alternate across destinations."""
    me = shards[rank]
    halo = me.halo
    n_max = max(s.n for s in shards)
    # gloo cannot move CUDA tensors point-to-point: stage through host memory (functional smoke runs of the
    # multi-rank path on fewer GPUs than ranks only — NCCL is the transport on a real multi-GPU node)
    via_host = dist.is_initialized() and dist.get_backend(group) == "gloo"
    cs = torch.cuda.current_stream(dev)
    xs = torch.cuda.Stream(device=dev)
    bufs = [torch.empty(chunk + 2 * halo, dtype=dtype, device=dev) for _ in range(2)]
    free = [None, None]                                  # event: process() finished reading bufs[i]
    stage = [torch.empty(chunk + 2 * halo, dtype=dtype, device=dev) for _ in range(2)] if rank == src else None
    stage_work = [None, None]
    si = 0
    received = 0
    k = 0
    for c0 in range(0, n_max, chunk):
        i = k & 1
        buf = bufs[i]
        ready = torch.cuda.Event()
        work = None
        with torch.cuda.stream(xs):
            if free[i] is not None:
                xs.wait_event(free[i])
            if rank == src:
                assert host_stream is not None
                for r, sh in enumerate(shards):
                    if c0 >= sh.n:
                        continue
                    a, b = window_bounds(sh, c0, min(chunk, sh.n - c0))
                    view = host_stream[a - stream_first:b - stream_first]
                    assert view.numel() == b - a, "host stream does not cover the window"
                    if r == rank:
                        buf[:b - a].copy_(view, non_blocking=True)
                        continue
                    if stage_work[si] is not None:
                        stage_work[si].wait()            # xs waits for the send that last used this buffer
                    st = stage[si]
                    if via_host:
                        dist.send(view.contiguous(), dst=r, group=group)
                        continue
                    st[:b - a].copy_(view, non_blocking=True)
                    stage_work[si] = dist.isend(st[:b - a], dst=r, group=group)
                    si ^= 1
            elif c0 < me.n:
                a, b = window_bounds(me, c0, min(chunk, me.n - c0))
                if via_host:
                    hb = torch.empty(b - a, dtype=dtype)
                    dist.recv(hb, src=src, group=group)
                    buf[:b - a].copy_(hb)
                else:
                    work = dist.irecv(buf[:b - a], src=src, group=group)
                    work.wait()                          # xs waits for the transfer
            ready.record(xs)
        if c0 < me.n:
            nc = min(chunk, me.n - c0)
            cs.wait_event(ready)
            process(buf[:nc + 2 * halo], me.first + c0, nc)
            ev = torch.cuda.Event()
            ev.record(cs)
            free[i] = ev
            received += nc + 2 * halo
        k += 1
    with torch.cuda.stream(xs):
        for w in stage_work:
            if w is not None:
                w.wait()
    cs.wait_stream(xs)
    return received
