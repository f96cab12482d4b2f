#!/usr/bin/env python3
"""Host-side cost of one decode_batch call (enqueue only) vs its device time, for the
bench workloads (per-stripe erasure patterns: one launch per pattern run) and for 1 MiB
blocks as in the paper's Fig. 1 sweep.  If the host needs longer to enqueue a call than
the device needs to run it, the device starves and the bench number is host-bound."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_1312_5155_b200 as rsp  # noqa: E402


def run(name, k, m, w, poly, B, S, er, reps=10):
    st = torch.empty((S, k + m, B), dtype=torch.uint8, device="cuda")
    rsp.synth_fill(st, k, seed=0)
    plan = rsp.Plan(k, m, w, poly)
    plan.encode_batch(st)
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
    launches = plan.stats()["jit_launches"]
    pats = len({tuple(r) for r in er.tolist()})
    h = float(np.median(host)) * 1e3
    print(f"{name}: B={B >> 10} KiB S={S} patterns={pats}: host {h:.3f} ms/call "
          f"({1e3 * h / max(pats, 1):.1f} us per pattern), device {dev:.3f} ms/call, "
          f"host/device {h / dev:.2f} (jit launches so far {launches})", flush=True)
    del st
    torch.cuda.empty_cache()


def main():
    for cfg in (sys.argv[1:] or ["C3", "C4", "C5"]):
        c = synth.CONFIGS[cfg]
        S = c["stripes"]
        er = synth.erasure_table(cfg, 0, S)
        run(cfg, c["k"], c["m"], c["w"], c["poly"], c["block_bytes"], S, er)
    er = np.full((2048, 4), -1, dtype=np.int32)
    for s in range(2048):
        er[s] = synth.erasure_draw(0, s, range(14), 4)
    run("fig1-1MiB", 10, 4, 8, 0x11D, 1 << 20, 2048, er)


if __name__ == "__main__":
    main()
