#!/usr/bin/env python3
"""Decode call from an idle stream (synchronize before each call) vs the same call queued
behind a ~10 ms GPU sleep (the host is then ahead of the GPU): the difference is host work
before the GPU can start (RS_POLY_HOST_PROFILE=1 prints the phases on stderr).  Prints % of
the MEASURED_PEAKS copy figure and the host time of each call (h, ms).
usage: python tools/start_latency.py [C3|C4|C5 ...]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
import paper_1312_5155_b200 as rsp  # noqa: E402

PEAK = 6459.9


def run(cfg):
    c = synth.CONFIGS[cfg]
    k, m, w, B, S = c["k"], c["m"], c["w"], c["block_bytes"], c["stripes"]
    st = torch.empty((S, k + m, B), dtype=torch.uint8, device="cuda")
    rsp.synth_fill(st, k, seed=0)
    plan = rsp.Plan(k, m, w, c["poly"])
    er = synth.erasure_table(cfg, 0, S)
    plan.prepare(er)
    moved = S * (k + m) * B
    for _ in range(3):
        plan.decode_batch(st, er)
        plan.encode_batch(st)

    def one(cycles):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if cycles:
            torch.cuda._sleep(cycles)
        e0.record()
        t = time.perf_counter()
        plan.decode_batch(st, er)
        th = time.perf_counter() - t
        e1.record()
        torch.cuda.synchronize()
        return moved / e0.elapsed_time(e1) / 1e6 / PEAK, th * 1e3

    for name, cyc, n in (("idle stream", 0, 10), ("after sleep", 20_000_000, 4)):
        r = [one(cyc) for _ in range(n)]
        print(f"{cfg} decode, {name}:", " ".join(f"{a:.3f}(h{h:.1f})" for a, h in r), flush=True)
    del st
    torch.cuda.empty_cache()


if __name__ == "__main__":
    for cfg in sys.argv[1:] or ["C4", "C3", "C5"]:
        run(cfg)
