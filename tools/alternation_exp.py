#!/usr/bin/env python3
"""Why is a decode call slower inside bench.py's encode/decode alternation than alone?

Times the same decode_batch call of one config (default C4) in four schedules, sampling the SM
clock and power over each (NVML, as bench.py does):
  alone      decode, decode, ...
  enc+dec    encode, decode, encode, decode, ...        (bench.py's timed region)
  copy+dec   a device copy of the encode's bytes, then decode, ...
  idle+dec   a host sleep of the encode's duration, then decode, ...

  python tools/alternation_exp.py [config] [steps]

One JSON line per schedule: decode ms (mean / min / max), fraction of the copy peak, median SM
clock, mean power.
"""
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_1312_5155_b200 as rsp  # noqa: E402
from bench import hbm_peak, nvml_handle  # noqa: E402


class Sampler:
    def __init__(self):
        import pynvml
        pynvml.nvmlInit()
        self.nv, self.h = pynvml, nvml_handle(pynvml, 0)
        self.clk, self.pw = [], []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.clk.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.pw.append(self.nv.nvmlDeviceGetPowerUsage(self.h) / 1e3)
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join()


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
    K = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    c = synth.CONFIGS[cfg]
    k, m, w, B, S = c["k"], c["m"], c["w"], c["block_bytes"], c["stripes"]
    n = k + m
    st = torch.empty((S, n, B), dtype=torch.uint8, device="cuda")
    rsp.synth_fill(st, k, seed=0)
    plan = rsp.Plan(k, m, w, c["poly"])
    er = synth.erasure_table(cfg, 0, S)
    plan.prepare(er)
    plan.encode_batch(st)
    torch.cuda.synchronize()
    golden = st.clone()
    # the copy schedule moves what one encode moves: (k+m)*B per stripe, read + write
    half = S * n * B // 2
    src = golden.view(-1)[:half]
    dst = torch.empty_like(src)
    peak = hbm_peak()[0]
    moved = S * n * B
    stream = torch.cuda.current_stream()

    def timed(pre):
        for _ in range(5):
            pre()
            plan.decode_batch(st, er)
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        with Sampler() as sm:
            for a, b in ev:
                pre()
                a.record(stream)
                plan.decode_batch(st, er)
                b.record(stream)
            torch.cuda.synchronize()
        ms = [a.elapsed_time(b) for a, b in ev]
        return ms, sm

    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    plan.encode_batch(st)
    e1.record(stream)
    torch.cuda.synchronize()
    enc_s = e0.elapsed_time(e1) / 1e3

    def idle():
        torch.cuda.synchronize()
        time.sleep(enc_s)

    schedules = [("alone", lambda: None), ("enc+dec", lambda: plan.encode_batch(st)),
                 ("copy+dec", lambda: dst.copy_(src)), ("idle+dec", idle), ("alone-again", lambda: None)]
    for name, pre in schedules:
        ms, sm = timed(pre)
        mean = statistics.mean(ms)
        print(json.dumps({"cfg": cfg, "schedule": name, "steps": K, "decode_ms_mean": round(mean, 4),
                          "decode_ms_min": round(min(ms), 4), "decode_ms_max": round(max(ms), 4),
                          "frac_mean": round(moved / mean / 1e6 / peak, 4), "peak_gbs": peak,
                          "sm_mhz_median": statistics.median(sm.clk) if sm.clk else None,
                          "sm_mhz_min": min(sm.clk) if sm.clk else None,
                          "power_w_mean": round(statistics.mean(sm.pw), 1) if sm.pw else None,
                          "samples": len(sm.clk)}), flush=True)
    assert torch.equal(st, golden), "batch changed"


if __name__ == "__main__":
    main()
