#!/usr/bin/env python3
"""Small driver for ncu captures: the bench's kernels on a reduced stripe count.

  ncu --set full -k regex:sliced_kernel -s 2 -c 2 python tools/profile_kernel.py --config C5 --stripes 8

Runs warm-up encode+decode once, then encode+decode once more (the captured
launches with -s 2).  Same kernels, block size and erasure recipe as bench.py.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
import paper_1312_5155_b200 as rsp  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--stripes", type=int, default=8)
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    c = synth.CONFIGS[a.config]
    k, m, w, B = c["k"], c["m"], c["w"], c["block_bytes"]
    S = a.stripes
    plan = rsp.Plan(k, m, w, c["poly"])
    st = torch.empty((S, k + m, B), dtype=torch.uint8, device="cuda")
    rsp.synth_fill(st, k, seed=0)
    er = synth.erasure_table(a.config, 0, S)
    plan.prepare(er)
    for _ in range(a.reps):
        plan.encode_batch(st)
        plan.decode_batch(st, er)
    torch.cuda.synchronize()
    print(f"ok {plan.kernel_kind} {a.config} S={S}")


if __name__ == "__main__":
    main()
