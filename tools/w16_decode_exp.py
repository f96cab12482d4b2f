#!/usr/bin/env python3
"""GF(2^16) decode A/B harness (C4 shape): the per-stripe pattern chain that bench.py times,
and single erasure patterns shared by every stripe (one launch), per kernel form.

  python tools/w16_decode_exp.py [reps]      # the form is chosen by the environment

Prints one line per case: ms per decode call and the fraction of the copy peak
(S*(k+m)*B bytes moved per call).  Every case is checked to restore the batch exactly.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_1312_5155_b200 as rsp  # noqa: E402


def _peak() -> float:
    """Copy peak the fractions are quoted against: MEASURED_PEAKS.json (driver-written), else the
    round-1 figure."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6459.9


PEAK = _peak()


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    cfg = os.environ.get("EXP_CFG", "C4")
    c = synth.CONFIGS[cfg]
    k, m, w, B, S = c["k"], c["m"], c["w"], c["block_bytes"], c["stripes"]
    if os.environ.get("EXP_B"):  # other block sizes at the same batch bytes
        B2 = int(os.environ["EXP_B"])
        S, B = S * B // B2, B2
    n = k + m
    st = torch.empty((S, n, B), dtype=torch.uint8, device="cuda")
    rsp.synth_fill(st, k, seed=0)
    plan = rsp.Plan(k, m, w, c["poly"])
    plan.encode_batch(st)
    torch.cuda.synchronize()
    golden = st.clone()
    er_rand = synth.erasure_table(cfg, 0, S)
    cases = [("per-stripe", er_rand)]
    singles = {"data4": [0, 3, 7, 11], "par4": [12, 13, 14, 15], "mix": [2, 5, 12, 15],
               "low-data": [0, 1, 2, 3], "high-data": [8, 9, 10, 11]}
    if n != 16:
        singles = {"first": list(er_rand[0])}
    for name, p in singles.items():
        cases.append((name, np.tile(np.array(p, dtype=np.int32), (S, 1))))
    moved = S * n * B
    form = {kk: v for kk, v in os.environ.items() if kk.startswith("RS_POLY_")}
    for name, er in cases:
        plan.prepare(er)
        for s in range(S):
            st[s, torch.from_numpy(er[s][er[s] >= 0].astype(np.int64)).cuda()] = 0x5A
        plan.decode_batch(st, er)
        torch.cuda.synchronize()
        ok = torch.equal(st, golden)
        plan.decode_batch(st, er)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
        ev[0].record()
        for i in range(reps):
            plan.decode_batch(st, er)
            ev[i + 1].record()
        torch.cuda.synchronize()
        ms = sorted(ev[i].elapsed_time(ev[i + 1]) for i in range(reps))
        med = ms[len(ms) // 2]
        print(json.dumps({"cfg": cfg, "block_bytes": B, "case": name, "form": form, "ok": ok, "ms_med": round(med, 4),
                          "ms_min": round(ms[0], 4), "frac_med": round(moved / med / 1e6 / PEAK, 4),
                          "patterns": len({tuple(r) for r in er.tolist()})}), flush=True)
        if name == "per-stripe" and os.environ.get("EXP_GRAPH"):
            # the same call captured once into a CUDA graph and replayed (PDL edges kept)
            g = torch.cuda.CUDAGraph()
            s_ = torch.cuda.Stream()
            s_.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s_):
                plan.decode_batch(st, er)
                torch.cuda.synchronize()
                with torch.cuda.graph(g, stream=s_):
                    plan.decode_batch(st, er)
            torch.cuda.synchronize()
            g.replay()
            torch.cuda.synchronize()
            ev[0].record()
            for i in range(reps):
                g.replay()
                ev[i + 1].record()
            torch.cuda.synchronize()
            ms = sorted(ev[i].elapsed_time(ev[i + 1]) for i in range(reps))
            med = ms[len(ms) // 2]
            print(json.dumps({"cfg": cfg, "block_bytes": B, "case": "per-stripe graph", "ok": bool(torch.equal(st, golden)),
                              "ms_med": round(med, 4), "frac_med": round(moved / med / 1e6 / PEAK, 4)}), flush=True)


if __name__ == "__main__":
    main()
