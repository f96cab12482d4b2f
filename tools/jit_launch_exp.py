#!/usr/bin/env python3
"""Decode throughput of the per-pattern JIT path vs the number of distinct patterns in
a batch (C4 / C5 shapes): one shared pattern (one launch) vs per-stripe patterns."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_1312_5155_b200 as rsp  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
    c = synth.CONFIGS[cfg]
    k, m, w, B, S = c["k"], c["m"], c["w"], c["block_bytes"], c["stripes"]
    n = k + m
    st = torch.empty((S, n, B), dtype=torch.uint8, device="cuda")
    rsp.synth_fill(st, k, seed=0)
    plan = rsp.Plan(k, m, w, c["poly"])
    plan.encode_batch(st)
    er_rand = synth.erasure_table(cfg if cfg != "C2" else "C5", 0, S)
    er_same = np.tile(er_rand[:1], (S, 1))
    moved = S * n * B
    cases = [("same", er_same)]
    for npat in (2, 8, 32):
        cases.append((f"{npat}-rr", er_rand[np.arange(S) % npat]))           # round-robin over stripes
        cases.append((f"{npat}-blk", er_rand[np.arange(S) * npat // S]))      # contiguous stripe ranges
    cases.append(("per-stripe", er_rand))
    for name, er in cases:
        plan.prepare(er)
        for _ in range(2):
            plan.decode_batch(st, er)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        reps = 5
        for _ in range(reps):
            plan.decode_batch(st, er)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print(f"{cfg} {name:10s} "
              f"patterns={len({tuple(r) for r in er.tolist()})} {ms:.3f} ms  {moved / ms / 1e6:.0f} GB/s moved")


if __name__ == "__main__":
    main()
