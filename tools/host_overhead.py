#!/usr/bin/env python3
"""Host-side cost of one decode_batch call (enqueue only) vs its device time, for batches
with many erasure patterns (C3 shape, and 1 MiB blocks as in the paper's Fig. 1 sweep)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_1312_5155_b200 as rsp  # noqa: E402


def run(B, S, reps=10):
    k, m = 10, 4
    st = torch.empty((S, k + m, B), dtype=torch.uint8, device="cuda")
    rsp.synth_fill(st, k, seed=0)
    plan = rsp.Plan(k, m)
    plan.encode_batch(st)
    er = np.full((S, m), -1, dtype=np.int32)
    for s in range(S):
        er[s] = synth.erasure_draw(0, s, range(k + m), m)
    plan.prepare(er)
    plan.decode_batch(st, er)
    torch.cuda.synchronize()
    host = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        t = time.perf_counter()
        plan.decode_batch(st, er)
        host.append(time.perf_counter() - t)
    e1.record()
    torch.cuda.synchronize()
    dev = e0.elapsed_time(e1) / reps
    pats = len({tuple(r) for r in er.tolist()})
    print(f"B={B >> 20} MiB S={S} patterns={pats}: host {np.median(host) * 1e3:.3f} ms/call, device {dev:.3f} ms/call, "
          f"{pats / (np.median(host) * 1e3):.0f} launches/ms host")


if __name__ == "__main__":
    run(4 << 20, 512)
    run(1 << 20, 2048)
