"""Probe: does running two contexts on two streams (alternate 2^27/2^28-sample calls) overlap K1/K2/K3 of
neighbouring calls on the SMs and raise throughput? Diagnostic only (C5 workload, 2^30 samples)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import kkgen  # noqa: E402
from paper_2104_06311_b200 import Receiver  # noqa: E402

HALO = 16640
S = 1 << 30
lc = kkgen.WORKLOADS["C5"]["cfg"]
dev = torch.device("cuda", 0)
g = kkgen.generate(lc, -HALO, S + HALO, device=dev, chunk=1 << 24)
codes = g["codes"]
ref = g["labels"][HALO // 4:(HALO + S) // 4].clone()
del g
dec = torch.empty(S // 4, dtype=torch.uint8, device=dev)
for chunk in (1 << 27, 1 << 28):
    rxs = [Receiver(adc_scale=lc.adc_scale, ref_intensity=lc.i_ref, dispersion_ps_per_nm=lc.dl_ps_nm,
                    formats=lc.formats, segment_frames=lc.segment_frames, max_samples_per_call=chunk, device=0)
           for _ in range(2)]
    streams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
    for nstreams in (1, 2, 1, 2):
        def step():
            for i, c0 in enumerate(range(0, S, chunk)):
                k = i % nstreams
                rxs[k].process(codes, c0, chunk, ref=ref[c0 // 4:(c0 + chunk) // 4],
                               decisions=dec[c0 // 4:(c0 + chunk) // 4], offset=c0 + HALO - HALO, stream=streams[k])
        torch.cuda.synchronize()
        step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for s_ in streams:
            s_.wait_event(e0)
        for _ in range(3):
            step()
        for s_ in streams:
            ev = torch.cuda.Event()
            ev.record(s_)
            torch.cuda.current_stream().wait_event(ev)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"chunk 2^{chunk.bit_length() - 1} streams {nstreams}: {3 * S / (ms * 1e-3) / 1e9:.2f} GS/s")
    for r in rxs:
        r.close()
