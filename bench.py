#!/usr/bin/env python
"""bench.py — ADC GS/s of the B200 KK receive chain (BASELINE.json metric) on the C5 workload.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl kkrx|reference]
  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 --master-port P bench.py --gpus N

Workload (BASELINE.json configs[4], "C5"): "continuous 2^32-sample mixed 4/8/16/32/64-QAM stream sharded over
1/2/4/8 GPUs with halo overlap" — format cycling per 256-frame segment, 1 GBaud at 4 GS/s, 1600 km of accumulated
dispersion (32,000 ps/nm), CSPR 12 dB, nominal Es/N0 26 dB white noise, int16 ADC codes, generated on the device
from the seeded generator (kkgen). By default (--scaling strong) the ONE 2^32-sample stream (8 GiB of int16) is
split into N contiguous frame ranges (shard.plan_strong), each rank holding its range plus 16,640-sample halos:
total work is fixed as N grows. (--scaling weak: every rank owns --samples-per-gpu samples of the stream.) One
step = the whole hot path (K1 KK → K2 MF → K3 EQ/CPR/decisions, in ≤ 2^29-sample calls through the C ABI) over
the rank's samples, plus the NCCL allreduce of the 24 error counters — the only cross-GPU traffic. Inputs (≥ 1 GiB
per rank at N = 8) are far larger than the 126 MB L2, so no L2 flush is needed between steps.

value = total core samples of all ranks × K / (max over ranks of the CUDA-event time of K steps), in GS/s.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ADC GS/s processed (real-time factor vs 4 GS/s) at 1/2/4/8 B200; % HBM roofline"
F = 16384
HALO = 16640
FP32_LANES_PER_SM = 128
N_SMS = 148


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="kkrx", choices=["kkrx", "reference"])
    ap.add_argument("--workload", default="C5")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: one --samples stream split over the ranks (BASELINE configs[4]); "
                         "weak: --samples-per-gpu per rank")
    ap.add_argument("--samples", type=int, default=1 << 32, help="stream length for --scaling strong")
    ap.add_argument("--samples-per-gpu", type=int, default=1 << 32, help="per-rank samples for --scaling weak")
    ap.add_argument("--chunk", type=int, default=1 << 29,
                    help="samples per kk_process_frames call (2^29: launch gaps and the persistent kernels' tail "
                         "waves amortised; tools/chunk_sweep.sh: 2^28 90.9, 2^29 91.6, 2^30 91.7 GS/s)")
    ap.add_argument("--e2e-samples", type=int, default=1 << 30)
    ap.add_argument("--cpu-frames", type=int, default=64, help="oracle sample size (frames) for cpu_baseline")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--eq-mode", default="block_ls", choices=["block_ls", "ddlms"],
                    help="block_ls: north-star per-frame WL least squares + CPR (default); "
                         "ddlms: the paper's static CD filter + 4-tap WL DDLMS")
    ap.add_argument("--static-cd", action="store_true",
                    help="block LS after the paper's static RRC x CD-inverse filter in K2 (L = 5; SURVEY NEXT-2)")
    ap.add_argument("--upsample", type=int, default=1, choices=[1, 2],
                    help="2: KK at 8 sps (half-band interpolation/decimation, K1U; DESIGN.md §3)")
    ap.add_argument("--ingest", default="local", choices=["local", "single"],
                    help="e2e input path: every rank reads its own shard from host memory (local), or rank 0 "
                         "holds the whole stream and sends each rank its windows over NVLink (single; NEXT-3)")
    ap.add_argument("--e2e-ref", default="prbs", choices=["prbs", "buffer"],
                    help="e2e reference labels: generated in the receiver from the transmitter's known sequence "
                         "(kk_config.ref_prbs, default) or a host label buffer copied with the samples")
    ap.add_argument("--mf-n", type=int, default=4096, choices=[4096, 8192],
                    help="K2 overlap-save grid: FFT4096/hop 3072 or FFT8192/hop 7168 (same exact convolution)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process group for N > 1 (gloo only for functional smoke runs of the multi-rank path on "
                         "fewer GPUs than ranks; never for timing)")
    ap.add_argument("--ddlms-block", type=int, default=512)
    ap.add_argument("--ddlms-warmup", type=int, default=1024)
    ap.add_argument("--ddlms-mu-warm", type=float, default=2e-3)
    return ap.parse_args()


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# ----------------------------------------------------------------------------------------------- per-unit work
def k3_flops_per_symbol(L: int) -> float:
    """Real-form arithmetic of the widely-linear block-LS step: pass 1 (L complex MACs = 8L) +
    lag sums (2L − 1 (ρ, d) pairs × 4 FMA, the shared real products of conj(a)·b and a·b) + cross-correlations
    (L × 4 FMA for p1 and p2) + WL pass 2 (L × 4 FMA) = 40L − 8 flops, + ~40 (four slicers, unbias, CPR)."""
    return 40.0 * L + 32.0


def k2_tile_flops(n: int) -> float:
    """One MF tile: FFT_n + IFFT_{n/2} (5·N·log2 N each) + ×H and fold (6 per folded bin) + mixer (8 per input
    sample): 403,456 for n = 4096 (3072 new samples), 868,352 for n = 8192 (7168 new samples)."""
    import math
    return 5.0 * n * math.log2(n) + 5.0 * (n // 2) * math.log2(n // 2) + 6.0 * (n // 2) + 8.0 * n


def kernel_units(chunk: int, L: int, eq_mode: str = "block_ls", ddlms_block: int = 512, ddlms_warmup: int = 1024,
                 upsample: int = 1, mf_n: int = 4096, static_cd: bool = False):
    """Algorithmic flops and HBM bytes per launch of each kernel for one call of `chunk` samples."""
    K = (L - 1) // 2
    k1_samples = chunk + 2 * F
    y_first = -K
    keep = mf_n // 2 - 512
    n_tiles = (chunk // 2 + 2 * K + keep - 1) // keep + 1
    frames = chunk // F
    if eq_mode == "ddlms":
        # per processed symbol (kept + warm-up), real-form WL (DESIGN.md §5 K3′): output 4 taps × 4 FMA +
        # update 4 taps × 4 FMA = 64 flops + ~20 (slicer, error)
        sym = chunk // 4 * (ddlms_block + ddlms_warmup) / ddlms_block
        k3 = dict(flops=84.0 * sym, bytes=(8.0 * (ddlms_block + ddlms_warmup) / ddlms_block * 2 + 2.0) * (chunk // 4))
        k2_flops = k2_tile_flops(mf_n) + (mf_n // 2) * 8.0   # complex H: 8 more flops per folded bin
    else:
        k3 = dict(flops=k3_flops_per_symbol(L) * 4096 * frames, bytes=73728.0 * frames)
        k2_flops = k2_tile_flops(mf_n) + ((mf_n // 2) * 8.0 if static_cd else 0.0)   # complex H: +8 per folded bin
    # K1U (upsample 2), per output sample: FFT2048 pair 220 + decimation 50 + interpolation 27 + E₂ 13 + logs 7
    k1_flops = 317.0 if upsample == 2 else 107.0
    return {
        ("K1u_kk" if upsample == 2 else "K1_kk"): dict(flops=k1_flops * k1_samples, bytes=10.0 * k1_samples),
        "K2_mf": dict(flops=k2_flops * n_tiles, bytes=(8.0 * mf_n + 8.0 * keep) * n_tiles),
        "K3_eq": k3,
    }


# ----------------------------------------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.index = index
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            names = {
                "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
                "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
                "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100}

            def run():
                while not self._stop.is_set():
                    try:
                        self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        for k, v in names.items():
                            if r & v and k != "gpu_idle":
                                self.reasons.add(k)
                    except Exception:
                        pass
                    self._stop.wait(0.05)
            self._t = threading.Thread(target=run, daemon=True)
            self._t.start()
        except Exception:
            self._t = None
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ----------------------------------------------------------------------------------------------- oracle sample
def _oracle_run(args):
    """Worker: run the fp64 oracle (single-threaded) on one contiguous run of frames."""
    codes, first, n, ocfg_kw, ref = args
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass
    from oracle import receiver as R
    cfg = R.OracleConfig(**ocfg_kw)
    t = time.perf_counter()
    out = R.receive(codes, first, n, cfg, ref=ref, keep=False)
    return out["dec"], {k: (v.tolist() if hasattr(v, "tolist") else v) for k, v in out["counts"].items()}, \
        time.perf_counter() - t


def _warm(_):
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass
    import oracle.receiver  # noqa: F401  (imports numpy/scipy once per worker, outside the timed region)
    return 0


def make_pool(cores):
    import multiprocessing as mp
    pool = mp.get_context("fork").Pool(processes=cores)
    pool.map(_warm, range(cores * 2))
    return pool


def oracle_sample(runs, ocfg_kw, pool):
    """Time the oracle on `runs` = [(codes_with_halo, first, n, ref)] over a warmed process pool."""
    jobs = [(c, f, n, ocfg_kw, r) for (c, f, n, r) in runs]
    t0 = time.perf_counter()
    res = pool.map(_oracle_run, jobs, chunksize=1)
    wall = time.perf_counter() - t0
    return res, wall


def ocfg_kwargs(lc, eq_mode="block_ls", a=None):
    kw = dict(dispersion_ps_per_nm=lc.dl_ps_nm, adc_scale=lc.adc_scale, ref_intensity=lc.i_ref,
              formats=tuple(lc.formats), segment_frames=lc.segment_frames, eq_mode=eq_mode,
              upsample=(a.upsample if a is not None else 1),
              static_cd=bool(a.static_cd) if a is not None else False)
    if a is not None and eq_mode == "ddlms":
        kw.update(ddlms_block=a.ddlms_block, ddlms_warmup=a.ddlms_warmup, ddlms_mu_warm=a.ddlms_mu_warm)
    return kw


def halo_of(a) -> int:
    """kk_halo() of the configuration (the oracle's halo() is the same number)."""
    return 16656 if a.upsample == 2 else 16640


# ----------------------------------------------------------------------------------------------- reference arm
def run_reference(a, rank, world):
    """The fp64 oracle, as it stands, timed on the host cores on a bounded sample of the same workload."""
    if rank != 0:
        return 0
    import numpy as np
    import kkgen
    wl = kkgen.WORKLOADS[a.workload]
    lc = wl["cfg"]
    cores = max(1, min(len(os.sched_getaffinity(0)), 32))
    frames_per_run = 4
    n_runs = cores
    S = a.samples if a.scaling == "strong" else a.samples_per_gpu
    HALO = halo_of(a)
    # sample: n_runs runs of 4 frames spread over the rank-0 shard (generated on the CPU)
    runs = []
    stride = max(frames_per_run, (S // F) // n_runs)
    for i in range(n_runs):
        first = i * stride * F
        n = frames_per_run * F
        g = kkgen.generate(lc, first - HALO, first + n + HALO)
        runs.append((g["codes"].numpy(), first, n, g["labels"].numpy()[HALO // 4:(HALO + n) // 4]))
    samples = n_runs * frames_per_run * F
    times = []
    pool = make_pool(cores)
    for it in range(a.warmup + a.steps):
        _, wall = oracle_sample(runs, ocfg_kwargs(lc, a.eq_mode, a), pool)
        if it >= a.warmup:
            times.append(wall)
    pool.close()
    T = sum(times)
    value = samples * len(times) / T / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GS/s", "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": 1e3 * T / len(times), "higher_is_better": True, "scaling": a.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{a.workload}: mixed 4/8/16/32/64-QAM, 1600 km, CSPR 12 dB, Es/N0 26 dB; "
                               f"oracle sample of {n_runs} runs x {frames_per_run} frames per step"},
        "cpu_baseline": {"value": value, "unit": "GS/s", "cores": cores, "kind": "oracle",
                         "sample": f"{n_runs} runs x {frames_per_run} frames (16384 samples) of the {a.workload} "
                                   f"stream per step, one fp64 numpy process per core"},
        "e2e": {"value": value, "unit": "GS/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------------------------- 8-bit ADC e2e
def e2e_uint8(a, lc, HALO, chunk, first, En, world, dev, SH, kkrx, kkgen, torch, dist, Receiver):
    """Same end-to-end measurement with an 8-bit ADC stream of the same link (SPEC S:199's AdcConfig default;
    the paper does not state the ADC resolution): half the host→device bytes of the int16 headline."""
    import dataclasses
    lc8 = dataclasses.replace(lc, adc_bits=8)
    g = kkgen.generate(lc8, first - HALO, first + En + HALO, device=dev)
    h_codes = torch.empty(En + 2 * HALO, dtype=torch.uint8, pin_memory=True)
    h_codes.copy_(g["codes"])
    h_ref = None
    if a.e2e_ref == "buffer":
        h_ref = torch.empty(En // 4, dtype=torch.uint8, pin_memory=True)
        h_ref.copy_(g["labels"][HALO // 4:(HALO + En) // 4])
    del g
    h_dec = torch.empty(En // 4, dtype=torch.uint8, pin_memory=True)
    rx8 = Receiver(adc_scale=lc8.adc_scale, ref_intensity=lc8.i_ref, dispersion_ps_per_nm=lc8.dl_ps_nm,
                   formats=lc8.formats, segment_frames=lc8.segment_frames, max_samples_per_call=chunk, device=dev.index,
                   input_uint8=True, upsample=a.upsample, mf_fft_n=a.mf_n, static_cd=a.static_cd,
                   ref_prbs_seed=None if h_ref is not None else lc8.seed, ref_prbs_kind=lc8.label_source)
    rx8.process_host(h_codes, first, En, ref=h_ref, decisions=h_dec)          # warm-up
    if world > 1:
        dist.barrier()
    rx8.reset_stats()
    torch.cuda.synchronize()
    t_e = []
    for _ in range(max(1, a.steps)):
        t1 = time.perf_counter()
        rx8.process_host(h_codes, first, En, ref=h_ref, decisions=h_dec)
        st = rx8.stats()
        t_e.append(time.perf_counter() - t1)
    rx8.close()
    te = SH.max_over_ranks(sum(t_e), device=dev)
    n_chunks = (En + (1 << 26) - 1) // (1 << 26)
    be = {f"{M}QAM": st["bit_err"][i] / st["bits"][i] for i, M in enumerate((4, 8, 16, 32, 64)) if st["bits"][i]}
    return {"value": En * world * len(t_e) / te / 1e9, "unit": "GS/s",
            "h2d_bytes_per_step": int((En + 2 * HALO * n_chunks) * 1 + (En // 4 if h_ref is not None else 0)),
            "d2h_bytes_per_step": int(En // 4 + 8 * kkrx.KK_STATS_WORDS), "samples_per_gpu": En,
            "adc": "uint8 (adc_bits 8, same link)", "ber": be}


# ----------------------------------------------------------------------------------------------- single ingest
def e2e_single_ingest(a, rx, lc, HALO, chunk, rank, world, dev, SH, kkrx, kkgen, torch, dist):
    """e2e with ONE ingest point (paper_2104_06311_b200/ingest.py): rank 0 holds the whole
    stream in pinned host memory (the ADC's DMA target), copies each rank's windows to the device and sends
    them point-to-point (NCCL over NVLink); each rank runs kk_process_frames on what it receives. Timed per
    step: distribution + processing + the D2H read of the counters; max over ranks."""
    from paper_2104_06311_b200 import ingest
    En = min(a.e2e_samples, 1 << 28, a.samples // world if a.scaling == "strong" else a.samples_per_gpu)
    En -= En % F
    shards = SH.plan_weak(En, world, halo=HALO)
    lo, hi = shards[0].read_first, shards[-1].read_first + shards[-1].read_count
    host = None
    if rank == 0:
        g = kkgen.generate(lc, lo, hi, device=dev)
        host = torch.empty(hi - lo, dtype=torch.int16, pin_memory=True)
        host.copy_(g["codes"])
        del g
    me = shards[rank]
    k = torch.arange(me.first // 4, (me.first + me.n) // 4, dtype=torch.int64, device=dev)
    ref = kkgen.symbol_labels(lc, k)
    dec = torch.empty(me.n // 4, dtype=torch.uint8, device=dev)

    def process(w, f0, nc):
        o = (f0 - me.first) // 4
        rx.process(w, f0, nc, ref=ref[o:o + nc // 4], decisions=dec[o:o + nc // 4])

    def one():
        ingest.distribute(shards, chunk, process, host_stream=host, stream_first=lo, device=dev)
        _ = rx.stats()

    one()                                                   # warm-up (allocations, NCCL P2P setup)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t = []
    for _ in range(max(1, a.steps)):
        t1 = time.perf_counter()
        one()
        t.append(time.perf_counter() - t1)
    te = SH.max_over_ranks(sum(t), device=dev)
    n_chunks = (En + chunk - 1) // chunk
    return {"value": En * world * len(t) / te / 1e9, "unit": "GS/s",
            "h2d_bytes_per_step": int(world * (En + 2 * HALO * n_chunks) * 2) if rank == 0 else 0,
            "d2h_bytes_per_step": int(8 * kkrx.KK_STATS_WORDS),
            "nvlink_bytes_per_step": int((world - 1) * (En + 2 * HALO * n_chunks) * 2),
            "samples_per_gpu": En, "ingest": "single (rank 0 -> all, ingest.distribute)",
            "api": "kk_process_frames on received windows"}


# ----------------------------------------------------------------------------------------------- GPU arm
def main():
    a = parse()
    rank, world, local = env_rank()
    if a.impl == "reference":
        return run_reference(a, rank, world)
    import numpy as np
    import torch
    import torch.distributed as dist

    import kkgen
    from paper_2104_06311_b200 import Receiver, kkrx, stats_from_words
    from paper_2104_06311_b200 import shard as SH

    local = local % max(torch.cuda.device_count(), 1)    # = LOCAL_RANK on a node with one GPU per rank
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if a.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    wl = kkgen.WORKLOADS[a.workload]
    lc = wl["cfg"]
    HALO = halo_of(a)
    if a.scaling == "strong":                           # one stream, N contiguous frame ranges (configs[4])
        plan = SH.plan_strong(a.samples, world, halo=HALO)
    else:                                               # rank r owns [r·S, (r+1)·S)
        plan = SH.plan_weak(a.samples_per_gpu, world, halo=HALO)
    my = plan[rank]
    S = my.n
    first = my.first
    chunk = min(a.chunk, S)
    assert chunk % F == 0 and S % F == 0
    calls = [(c0, min(chunk, S - c0)) for c0 in range(0, S, chunk)]
    dist_info = None
    if world > 1:                                       # evidence of the process group the counters cross
        me = {"rank": rank, "local_rank": local, "device": torch.cuda.get_device_name(dev),
              "pci_bus_id": torch.cuda.get_device_properties(dev).pci_bus_id if hasattr(
                  torch.cuda.get_device_properties(dev), "pci_bus_id") else None,
              "host": os.uname().nodename, "shard_first": first, "shard_samples": S}
        allinfo = [None] * world
        dist.all_gather_object(allinfo, me)
        dist_info = {"backend": dist.get_backend(), "world_size": dist.get_world_size(),
                     "nccl_version": ".".join(map(str, torch.cuda.nccl.version())) if a.dist_backend == "nccl" else None,
                     "ranks": allinfo}

    t0 = time.perf_counter()
    g = kkgen.generate(lc, my.read_first, my.read_first + my.read_count, device=dev, chunk=1 << 24)
    codes = g["codes"]
    ref = g["labels"][HALO // 4:(HALO + S) // 4].clone()   # own allocation: 16-B aligned (K3 TMA-stages ref)
    del g
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t0

    rx = Receiver(adc_scale=lc.adc_scale, ref_intensity=lc.i_ref, dispersion_ps_per_nm=lc.dl_ps_nm,
                  formats=lc.formats, segment_frames=lc.segment_frames, max_samples_per_call=chunk, device=local,
                  eq_mode=a.eq_mode, static_cd=a.static_cd, ddlms_block=a.ddlms_block, ddlms_warmup=a.ddlms_warmup,
                  ddlms_mu_warm=a.ddlms_mu_warm, upsample=a.upsample, mf_fft_n=a.mf_n)
    assert rx.halo == HALO
    L = rx.taps
    dec = torch.empty(S // 4, dtype=torch.uint8, device=dev)
    counters = torch.zeros(kkrx.KK_STATS_WORDS, dtype=torch.int64, device=dev)
    stream = torch.cuda.current_stream(dev)
    calls_per_step = len(calls)

    def step():
        for c0, cn in calls:
            rx.process(codes, first + c0, cn, ref=ref[c0 // 4:(c0 + cn) // 4],
                       decisions=dec[c0 // 4:(c0 + cn) // 4], offset=c0, stream=stream)
        rx.stats_device(counters, stream)
        SH.allreduce_counters(counters)                 # the only cross-GPU data movement (24 × 8 B, NCCL)

    for _ in range(a.warmup):
        step()
    rx.reset_stats()
    torch.cuda.synchronize()
    kkrx.kk_kernel_times(rx.ctx, reset=True)
    kkrx.kk_enable_timing(rx.ctx, True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(a.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    kkrx.kk_enable_timing(rx.ctx, False)
    kt_ms, kt_n = kkrx.kk_kernel_times(rx.ctx, reset=True)
    ms_max = SH.max_over_ranks(ms, device=dev)
    total_samples = sum(x.n for x in plan) * a.steps
    value = total_samples / (ms_max * 1e-3) / 1e9
    st = stats_from_words(counters.cpu().tolist())

    # ---------------- per-kernel roofline (live CUDA-event durations over the timed region)
    peak_fp32 = N_SMS * FP32_LANES_PER_SM * 2 * 1965e6 / 1e12      # TFLOP/s at clocks.max.sm
    hbm_peak = 6453.1
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        hbm_peak = float(mp.get("hbm_gbs", hbm_peak))
        peak_fp32 = N_SMS * FP32_LANES_PER_SM * 2 * float(mp.get("sm_max_mhz", 1965.0)) * 1e6 / 1e12
    except Exception:
        pass
    units = kernel_units(chunk, L, a.eq_mode, a.ddlms_block, a.ddlms_warmup, a.upsample, a.mf_n, a.static_cd)
    traffic = {}
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            tj = json.load(open(tp))
            scale = chunk / float(tj.get("chunk_samples", chunk))      # per-launch bytes scale with the call size
            traffic = {k: v * scale for k, v in tj.get("bytes_per_launch", {}).items()}
        except Exception:
            traffic = {}
    kernels = {}
    for i, name in enumerate(("K1u_kk" if a.upsample == 2 else "K1_kk", "K2_mf", "K3_eq")):
        avg_ms = kt_ms[i] / max(kt_n[i], 1)
        u = units[name]
        kernels[name] = {
            "avg_ms": avg_ms, "launches": kt_n[i], "share": kt_ms[i] / max(sum(kt_ms), 1e-9),
            "tflops": u["flops"] / (avg_ms * 1e-3) / 1e12, "gbs": u["bytes"] / (avg_ms * 1e-3) / 1e9,
            "flops_per_launch": u["flops"], "bytes_per_launch": u["bytes"],
            "frac_alu": u["flops"] / (avg_ms * 1e-3) / 1e12 / peak_fp32,
            "frac_hbm": u["bytes"] / (avg_ms * 1e-3) / 1e9 / hbm_peak,
            # SURVEY §8(d)'s reading: fraction of the kernel's attainable roofline min(BW·AI, P_FP32)
            "attainable_tflops": min(hbm_peak * 1e-3 * u["flops"] / u["bytes"], peak_fp32),
            "frac_attainable": (u["flops"] / (avg_ms * 1e-3) / 1e12)
            / min(hbm_peak * 1e-3 * u["flops"] / u["bytes"], peak_fp32),
        }
    dom = max(kernels, key=lambda k: kernels[k]["share"])
    kd = kernels[dom]
    roofline = {"kernel": dom, "bound": "alu", "achieved": kd["tflops"], "peak": peak_fp32, "unit": "TFLOP/s",
                "frac": kd["tflops"] / peak_fp32, "traffic": traffic.get(dom),
                "peak_source": "148 SM x 128 FP32 lanes x 2 x clocks.max.sm (derived, DESIGN.md §6)",
                "hbm_gbs": kd["gbs"], "hbm_frac_of_measured": kd["frac_hbm"],
                "attainable": kd["attainable_tflops"], "frac_attainable": kd["frac_attainable"]}

    # ---------------- end to end through the host-buffer C-ABI call (pinned memory, copies inside)
    e2e = None
    e2e_u8 = None
    if not a.no_e2e and a.ingest == "single":
        e2e = e2e_single_ingest(a, rx, lc, HALO, chunk, rank, world, dev, SH, kkrx, kkgen, torch, dist)
    elif not a.no_e2e:
        En = min(a.e2e_samples, S)
        h_codes = torch.empty(En + 2 * HALO, dtype=torch.int16, pin_memory=True)
        h_codes.copy_(codes[:En + 2 * HALO])
        h_ref = None
        if a.e2e_ref == "buffer":                                            # labels cross PCIe with the samples
            h_ref = torch.empty(En // 4, dtype=torch.uint8, pin_memory=True)
            h_ref.copy_(ref[:En // 4])
            rxe = rx
        else:                                                                # the receiver knows the transmitter's
            rxe = Receiver(adc_scale=lc.adc_scale, ref_intensity=lc.i_ref, dispersion_ps_per_nm=lc.dl_ps_nm,
                           formats=lc.formats, segment_frames=lc.segment_frames, max_samples_per_call=chunk,
                           device=local, eq_mode=a.eq_mode, static_cd=a.static_cd, ddlms_block=a.ddlms_block, ddlms_warmup=a.ddlms_warmup,
                           ddlms_mu_warm=a.ddlms_mu_warm, upsample=a.upsample, mf_fft_n=a.mf_n,
                           ref_prbs_seed=lc.seed, ref_prbs_kind=lc.label_source)   # (kk_config.ref_prbs)
        h_dec = torch.empty(En // 4, dtype=torch.uint8, pin_memory=True)
        n_chunks = (En + min(chunk, 1 << 26) - 1) // min(chunk, 1 << 26)    # host path stages ≤ 2^26 per sub-call
        rxe.process_host(h_codes, first, En, ref=h_ref, decisions=h_dec)     # warm-up (allocates staging)
        if world > 1:
            dist.barrier()
        rxe.reset_stats()
        torch.cuda.synchronize()                                             # the host path runs on its own streams
        t_e = []
        for _ in range(max(1, a.steps)):
            t1 = time.perf_counter()
            rxe.process_host(h_codes, first, En, ref=h_ref, decisions=h_dec)
            st_e = rxe.stats()                                               # D2H of the step's result
            t_e.append(time.perf_counter() - t1)
        te = SH.max_over_ranks(sum(t_e), device=dev)
        e2e = {"value": En * world * len(t_e) / te / 1e9, "unit": "GS/s",
               "h2d_bytes_per_step": int((En + 2 * HALO * n_chunks) * 2 + (En // 4 if h_ref is not None else 0)),
               "d2h_bytes_per_step": int(En // 4 + 8 * kkrx.KK_STATS_WORDS),
               "samples_per_gpu": En, "api": "kk_process_frames_host (pinned host buffers, 2 streams)",
               "ref": ("host label buffer" if h_ref is not None else
                       f"transmitter label sequence generated on the GPU (kk_config.ref_prbs: {lc.label_source})"),
               "ber": {f"{M}QAM": st_e["bit_err"][i] / st_e["bits"][i]
                       for i, M in enumerate((4, 8, 16, 32, 64)) if st_e["bits"][i]}}
        if rxe is not rx:
            rxe.close()
        del h_codes, h_ref, h_dec
        e2e_u8 = e2e_uint8(a, lc, HALO, chunk, first, En, world, dev, SH, kkrx, kkgen, torch, dist, Receiver)

    # ---------------- oracle beside it (rank 0, N = 1 only): timing + sampled-frame parity
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cores = max(1, min(len(os.sched_getaffinity(0)), 32))
        fr_per_run = 4
        n_runs = max(1, min(cores * 2, a.cpu_frames // fr_per_run))
        total_frames = S // F
        runs, picks = [], []
        for i in range(n_runs):
            f0 = (i * (total_frames - fr_per_run)) // max(n_runs - 1, 1)
            s0 = f0 * F
            c = codes[s0: s0 + fr_per_run * F + 2 * HALO].cpu().numpy()
            r = ref[s0 // 4:(s0 + fr_per_run * F) // 4].cpu().numpy()
            runs.append((c, first + s0, fr_per_run * F, r))
            picks.append(s0 // 4)
        pool = make_pool(cores)
        oracle_sample(runs[:cores], ocfg_kwargs(lc, a.eq_mode, a), pool)   # warm-up pass (first-touch, caches)
        res, wall = oracle_sample(runs, ocfg_kwargs(lc, a.eq_mode, a), pool)
        pool.close()
        agree, nsym = 0, 0
        be_o = 0
        dec_h = dec.cpu().numpy()
        for (d_or, cnt, _), k0 in zip(res, picks):
            d_gpu = dec_h[k0:k0 + len(d_or)]
            agree += int(np.sum(d_gpu == d_or))
            nsym += len(d_or)
            be_o += sum(cnt["bit_err"])
        n_s = n_runs * fr_per_run * F
        cpu = {"value": n_s / wall / 1e9, "unit": "GS/s", "cores": cores, "kind": "oracle",
               "sample": f"{n_runs} runs x {fr_per_run} frames ({n_s} samples) spread over the {a.workload} shard, "
                         f"one fp64 numpy process per core",
               "parity_decisions_identical": agree / max(nsym, 1)}

    q = {}
    for i, M in enumerate((4, 8, 16, 32, 64)):
        if st["bits"][i]:
            ber = st["bit_err"][i] / st["bits"][i]
            q[f"{M}QAM"] = {"ber": ber, "q_db": (kkrx.kk_q_from_ber(ber) if 0 < ber < 0.5 else None)}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GS/s", "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": ms_max / a.steps, "higher_is_better": True, "scaling": a.scaling, "vs_baseline": None,
            "dtype": "f32", "data": "synthetic (kkgen seeded generator, generated on device)",
            "config": {"workload": f"{a.workload}: continuous mixed 4/8/16/32/64-QAM stream (256-frame segments), "
                                   f"1 GBaud @ 4 GS/s, 1600 km (32000 ps/nm), CSPR 12 dB, Es/N0 26 dB white, int16 ADC",
                       "stream_samples": (a.samples if a.scaling == "strong" else a.samples_per_gpu * world),
                       "samples_per_gpu": S, "chunk_samples": chunk, "eq_taps": L, "eq_mode": a.eq_mode,
                       "parallelism": f"{world} contiguous frame-range shards + halos, counters allreduced",
                       "kk_upsample": a.upsample, "mf_grid": f"FFT{a.mf_n}/hop {a.mf_n - 1024}",
                       "static_cd": bool(a.static_cd),
                       **({"ddlms_block": a.ddlms_block, "ddlms_warmup": a.ddlms_warmup,
                           "ddlms_mu_warm": a.ddlms_mu_warm} if a.eq_mode == "ddlms" else {}),
                       "l2": "inputs 8 GiB/GPU per step >> 126 MB L2, no flush needed", "seed": lc.seed},
            "rt_factor": value / 4.0,
            "clocks": clk.summary(),
            "e2e": e2e,
            "e2e_uint8": e2e_u8,
            "gpu_launches": (3 if a.eq_mode == "ddlms" else 5) * calls_per_step * a.steps,
            "roofline": roofline,
            "kernels": kernels,
            "cpu_baseline": cpu,
            "quality": {"per_format": q, "frames": st["frames"], "dead_frames": st["dead_frames"],
                        "bad_frames": st["bad_frames"], "clamped": st["clamped"],
                        "counts": {k: st[k] for k in ("sym", "sym_err", "bits", "bit_err")}},
            "dist": dist_info,
            "gen_seconds": t_gen,
        }
        print(json.dumps(line), flush=True)
    rx.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
