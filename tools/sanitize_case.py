"""Small end-to-end exercise of every kernel (both equalizer modes, int16/uint8/float inputs, device and host
paths, per-frame errors) for compute-sanitizer runs:  compute-sanitizer --tool memcheck python tools/sanitize_case.py"""
import dataclasses
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import kkgen  # noqa: E402
from paper_2104_06311_b200 import KK_STAGE_EQ, KK_STAGE_FIELD, KK_STAGE_MF, Receiver  # noqa: E402

F, H = 16384, 16640


def main():
    first, n = 2 * F, 3 * F
    for eq_mode, dl, bits in (("block_ls", 200000.0, 15), ("ddlms", 112000.0, 15), ("block_ls", 32000.0, 8)):
        lc = kkgen.LinkConfig(formats=(4, 16, 64), segment_frames=1, dl_ps_nm=dl, cspr_db=12.0, esn0_db=20.0,
                              seed=3, adc_bits=bits)
        g = kkgen.generate(lc, first - H, first + n + H)
        rx = Receiver(adc_scale=lc.adc_scale, ref_intensity=lc.i_ref, dispersion_ps_per_nm=dl, formats=lc.formats,
                      segment_frames=1, max_samples_per_call=n, keep_intermediate=True, eq_mode=eq_mode,
                      input_uint8=(bits <= 8))
        codes, ref = g["codes"].cuda(), g["labels"][H // 4:(H + n) // 4].cuda()
        dec = torch.zeros(n // 4, dtype=torch.uint8, device="cuda")
        fe = torch.zeros(2 * n // F, dtype=torch.int32, device="cuda")
        rx.process(codes, first, n, ref=ref, decisions=dec, frame_errors=fe)
        for st in (KK_STAGE_FIELD, KK_STAGE_MF, KK_STAGE_EQ):
            rx.intermediate(st)
        hc = g["codes"].pin_memory()
        hr = g["labels"][H // 4:(H + n) // 4].pin_memory()
        hd = torch.zeros(n // 4, dtype=torch.uint8).pin_memory()
        rx.process_host(hc, first, n, ref=hr, decisions=hd)
        s = rx.stats()
        print(eq_mode, bits, "frames", s["frames"], "bit_err", sum(s["bit_err"]))
        rx.close()
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
