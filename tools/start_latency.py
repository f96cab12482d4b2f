#!/usr/bin/env python3
"""Decode call from an idle stream (synchronize before each call) vs the same call queued
behind a ~10 ms GPU sleep (the host is then ahead of the GPU): the difference is host work
before the GPU can start (RS_POLY_HOST_PROFILE=1 prints the phases on stderr).  Prints % of
the MEASURED_PEAKS copy figure and the host time of each call (h, ms).
usage: python tools/start_latency.py [C3|C4|C5 ...]
       python tools/start_latency.py cold [C5|C4 ...]   # first decode of a fresh plan:
         background JIT (new patterns on the table kernels) vs after rs_poly_prepare_all"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
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


def cold(cfg):
    """First decode call on never-seen erasure patterns vs the warm figure, in a process whose
    library is already warm (a storage node meeting a new failure pattern): a fresh plan
    without preparation (background JIT: the new patterns run on the table kernels until
    their kernels are compiled) and a fresh plan after rs_poly_prepare_all (every <= m
    pattern compiled and loaded up front; its time reported -- the on-disk cubin cache makes
    a second process fast)."""
    c = synth.CONFIGS[cfg]
    k, m, w, B, S = c["k"], c["m"], c["w"], c["block_bytes"], c["stripes"]
    st = torch.empty((S, k + m, B), dtype=torch.uint8, device="cuda")
    rsp.synth_fill(st, k, seed=0)
    er = synth.erasure_table(cfg, 0, S)
    moved = S * (k + m) * B
    # warm the process: library kernels, NVRTC, pools -- on a pattern outside the batch
    used = {tuple(r) for r in er.tolist()}
    other = next(p for p in (list(range(m)), list(range(k, k + m)), list(range(1, m + 1))) if tuple(p) not in used)
    warm_er = np.tile(np.array(other, dtype=np.int32), (S, 1))
    wp = rsp.Plan(k, m, w, c["poly"])
    wp.decode_batch(st, warm_er)
    wp.set_jit(rsp.RS_JIT_OFF)
    wp.decode_batch(st, warm_er)
    torch.cuda.synchronize()

    host_ms = []

    def call(plan):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        t = time.perf_counter()
        plan.decode_batch(st, er)
        host_ms.append((time.perf_counter() - t) * 1e3)
        e1.record()
        torch.cuda.synchronize()
        return moved / e0.elapsed_time(e1) / 1e6 / PEAK

    for mode in ("no preparation", "prepare_all"):
        plan = rsp.Plan(k, m, w, c["poly"])
        t0 = time.perf_counter()
        if mode == "prepare_all":
            plan.prepare_all()
        setup = time.perf_counter() - t0
        host_ms.clear()
        first = call(plan)
        second = call(plan)
        plan.prepare(er)
        warm = sorted(call(plan) for _ in range(5))[2]
        stt = plan.stats()
        print(f"{cfg} cold decode, {mode}: first {first:.3f} second {second:.3f} warm {warm:.3f} "
              f"first/warm {first / warm:.3f} host ms (first, second) {host_ms[0]:.2f} {host_ms[1]:.2f} "
              f"setup {setup:.1f} s patterns {stt['patterns']} "
              f"jit_ready {stt['jit_ready']} cache_hits {stt['jit_cache_hits']}", flush=True)
        plan.close()
    del st
    torch.cuda.empty_cache()


if __name__ == "__main__":
    if sys.argv[1:2] == ["cold"]:
        for cfg in sys.argv[2:] or ["C5"]:
            cold(cfg)
    else:
        for cfg in sys.argv[1:] or ["C4", "C3", "C5"]:
            run(cfg)
