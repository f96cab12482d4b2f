#!/usr/bin/env python3
"""PCIe / host-path diagnostics for the e2e number: raw pinned H2D / D2H copy rates
(alone and concurrent) vs rs_poly_encode_host / rs_poly_decode_host on the C5 batch."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
import paper_1312_5155_b200 as rsp  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C5"
    c = synth.CONFIGS[cfg]
    k, m, w, B = c["k"], c["m"], c["w"], c["block_bytes"]
    S = c.get("stripes_per_gpu", c.get("stripes"))
    n = k + m
    dev = torch.empty((S, n, B), dtype=torch.uint8, device="cuda")
    rsp.synth_fill(dev, k, seed=0)
    host = torch.empty((S, n, B), dtype=torch.uint8, pin_memory=True)
    nb = 2 << 30
    h1 = host.view(-1)[:nb]
    d1 = dev.view(-1)[:nb]
    d2 = dev.view(-1)[nb:2 * nb]
    h2 = host.view(-1)[nb:2 * nb]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    t = timed(lambda: d1.copy_(h1, non_blocking=True))
    print(f"H2D pinned {nb / t / 1e9:.1f} GB/s")
    t = timed(lambda: h1.copy_(d1, non_blocking=True))
    print(f"D2H pinned {nb / t / 1e9:.1f} GB/s")

    def both():
        with torch.cuda.stream(s1):
            d1.copy_(h1, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
    t = timed(both)
    print(f"H2D+D2H concurrent {2 * nb / t / 1e9:.1f} GB/s total")
    plan = rsp.Plan(k, m, w, c["poly"])
    host.copy_(dev)
    er = synth.erasure_table(cfg, 0, S)
    plan.prepare(er)
    t = timed(lambda: plan.encode_host(host), reps=2)
    print(f"encode_host {t * 1e3:.1f} ms: H2D {S * k * B / t / 1e9:.1f} GB/s, user {S * k * B / t / 1e9:.1f} GB/s")
    t = timed(lambda: plan.decode_host(host, er), reps=2)
    print(f"decode_host {t * 1e3:.1f} ms: user {S * k * B / t / 1e9:.1f} GB/s")


if __name__ == "__main__":
    main()
