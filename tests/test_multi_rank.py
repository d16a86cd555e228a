"""World-size-2 gloo tests of the multi-GPU host logic (shard plan, halos, counter allreduce, max-over-ranks)
on CPU. The per-rank data path here is the fp64 oracle (test infrastructure) standing in for one GPU's
kernels, so the test checks that the shard plan + halos + counter reduction reproduce the single-stream
counts exactly."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2104_06311_b200 import shard as S


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_plans_cover_stream_without_overlap():
    for world in (1, 2, 3, 4, 8):
        sh = S.plan_strong(37 * S.FRAME_SAMPLES, world, stream_first=5 * S.FRAME_SAMPLES)
        assert sh[0].first == 5 * S.FRAME_SAMPLES
        for a, b in zip(sh, sh[1:]):
            assert a.first + a.n == b.first
        assert sum(x.n for x in sh) == 37 * S.FRAME_SAMPLES
        assert max(x.n for x in sh) - min(x.n for x in sh) <= S.FRAME_SAMPLES
        w = S.plan_weak(4 * S.FRAME_SAMPLES, world)
        assert [x.first for x in w] == [r * 4 * S.FRAME_SAMPLES for r in range(world)]
        assert all(x.read_count == x.n + 2 * S.HALO for x in w)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import kkgen
    from oracle import receiver as R
    lc = kkgen.LinkConfig(formats=(16, 64), segment_frames=1, dl_ps_nm=32000.0, cspr_db=12.0, esn0_db=21.0, seed=77)
    cfg = R.OracleConfig(dispersion_ps_per_nm=32000.0, adc_scale=lc.adc_scale, ref_intensity=lc.i_ref,
                         formats=(16, 64), segment_frames=1)
    sh = S.plan_strong(6 * S.FRAME_SAMPLES, world, stream_first=2 * S.FRAME_SAMPLES)[rank]
    g = kkgen.generate(lc, sh.read_first, sh.read_first + sh.read_count)
    ref = g["labels"].numpy()[S.HALO // 4:(S.HALO + sh.n) // 4]
    out = R.receive(g["codes"].numpy(), sh.first, sh.n, cfg, ref=ref, keep=False)
    c = out["counts"]
    words = torch.tensor(list(c["sym"]) + list(c["sym_err"]) + list(c["bits"]) + list(c["bit_err"]) +
                         [c["clamped"], c["frames"], c["dead_frames"], c["bad_frames"]], dtype=torch.int64)
    S.allreduce_counters(words)
    t = S.max_over_ranks(float(rank + 1))
    if rank == 0:
        q.put((words.tolist(), t))
    dist.destroy_process_group()


def test_two_rank_counters_match_single_stream():
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    words, tmax = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert tmax == 2.0
    # the same six frames on one "rank"
    import kkgen
    from oracle import receiver as R
    lc = kkgen.LinkConfig(formats=(16, 64), segment_frames=1, dl_ps_nm=32000.0, cspr_db=12.0, esn0_db=21.0, seed=77)
    cfg = R.OracleConfig(dispersion_ps_per_nm=32000.0, adc_scale=lc.adc_scale, ref_intensity=lc.i_ref,
                         formats=(16, 64), segment_frames=1)
    sh = S.plan_strong(6 * S.FRAME_SAMPLES, 1, stream_first=2 * S.FRAME_SAMPLES)[0]
    g = kkgen.generate(lc, sh.read_first, sh.read_first + sh.read_count)
    out = R.receive(g["codes"].numpy(), sh.first, sh.n, cfg, ref=g["labels"].numpy()[S.HALO // 4:(S.HALO + sh.n) // 4],
                    keep=False)
    c = out["counts"]
    whole = list(c["sym"]) + list(c["sym_err"]) + list(c["bits"]) + list(c["bit_err"]) + \
        [c["clamped"], c["frames"], c["dead_frames"], c["bad_frames"]]
    assert words == [int(x) for x in whole]
    assert sum(words[5:10]) > 0          # non-trivial error counts were reduced


# ------------------------------------------------------------------ single-ingest distribution (NEXT-3)
def _ingest_worker(rank, world, port, q, weak):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import kkgen
    from paper_2104_06311_b200 import ingest
    lc = kkgen.LinkConfig(formats=(16,), dl_ps_nm=8000.0, cspr_db=12.0, esn0_db=20.0, seed=91)
    F = S.FRAME_SAMPLES
    halo = S.HALO_UP if weak else S.HALO
    shards = (S.plan_weak(3 * F, world, stream_first=F, halo=halo) if weak
              else S.plan_strong(7 * F, world, stream_first=F, halo=halo))
    lo = min(s.read_first for s in shards)
    hi = max(s.read_first + s.read_count for s in shards)
    full = kkgen.generate(lc, lo, hi)["codes"]        # every rank: the reference (rank 0: the ADC stream)
    host = full if rank == 0 else None
    got = []
    n = ingest.distribute(shards, 2 * F, lambda w, f0, nc: got.append((w.clone(), f0, nc)), host_stream=host,
                          stream_first=lo)
    # every window must be the stream's samples [f0 − halo, f0 + nc + halo) exactly, chunks tiling the core
    me = shards[rank]
    ok = sum(nc for _, _, nc in got) == me.n and n == sum(nc + 2 * halo for _, _, nc in got)
    cur = me.first
    for w, f0, nc in got:
        ref = full[f0 - halo - lo:f0 + nc + halo - lo]
        ok = ok and f0 == cur and torch.equal(w, ref)
        cur += nc
    flag = torch.tensor([int(ok)])
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if rank == 0:
        q.put(int(flag.item()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,weak", [(2, True), (3, False)])
def test_single_ingest_delivers_exact_windows(world, weak):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_ingest_worker, args=(r, world, port, q, weak)) for r in range(world)]
    for p in ps:
        p.start()
    res = q.get(timeout=300)
    for p in ps:
        p.join(timeout=60)
    assert res == 1
