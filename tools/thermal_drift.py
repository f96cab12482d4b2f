#!/usr/bin/env python3
"""Per-call throughput over consecutive calls (the GPU heating up under sw_power_cap):
K back-to-back [encode, decode] steps as bench.py times them, then K decode-only and K
encode-only calls; one CUDA event between calls, % of the MEASURED_PEAKS copy figure.
usage: python tools/thermal_drift.py [C3|C4|C5 ...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
import paper_1312_5155_b200 as rsp  # noqa: E402

PEAK = 6459.9


def run(cfg, K=10):
    c = synth.CONFIGS[cfg]
    k, m, w, B, S = c["k"], c["m"], c["w"], c["block_bytes"], c["stripes"]
    st = torch.empty((S, k + m, B), dtype=torch.uint8, device="cuda")
    rsp.synth_fill(st, k, seed=0)
    plan = rsp.Plan(k, m, w, c["poly"])
    er = synth.erasure_table(cfg, 0, S)
    plan.prepare(er)
    moved = S * (k + m) * B

    def frac(ms):
        return moved / ms / 1e6 / PEAK

    for _ in range(3):
        plan.encode_batch(st)
        plan.decode_batch(st, er)
    torch.cuda.synchronize()

    def timed(calls):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(calls) + 1)]
        ev[0].record()
        for i, fn in enumerate(calls):
            fn()
            ev[i + 1].record()
        torch.cuda.synchronize()
        return [frac(ev[i].elapsed_time(ev[i + 1])) for i in range(len(calls))]

    enc = lambda: plan.encode_batch(st)  # noqa: E731
    dec = lambda: plan.decode_batch(st, er)  # noqa: E731
    alt = timed([enc, dec] * K)
    print(cfg, "alternating encode", " ".join(f"{v:.3f}" for v in alt[0::2]))
    print(cfg, "alternating decode", " ".join(f"{v:.3f}" for v in alt[1::2]))
    print(cfg, "decode only       ", " ".join(f"{v:.3f}" for v in timed([dec] * K)))
    print(cfg, "encode only       ", " ".join(f"{v:.3f}" for v in timed([enc] * K)), flush=True)
    del st
    torch.cuda.empty_cache()


if __name__ == "__main__":
    for cfg in sys.argv[1:] or ["C3", "C5", "C4"]:
        run(cfg)
