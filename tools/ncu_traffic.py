#!/usr/bin/env python3
"""Whole-call DRAM traffic of bench.py's dominant calls, measured by ncu over a profiler range.

  # on the GPU box (app-range replay re-runs this script once per ncu pass):
  ncu --replay-mode app-range --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --csv --log-file gpurun_out/traffic_C5_decode.csv python tools/ncu_traffic.py run C5 decode
  # here: fold the captures into profiles/ncu_traffic.json (keyed by bench.code_hash())
  python tools/ncu_traffic.py summarize gpurun_out/traffic_*.csv

`run` sets up the bench workload exactly as bench.py does (same stripes, plan, prepare, warm
calls), then profiles two cudaProfilerStart/Stop ranges:
  range 1: one whole call (encode_batch: one launch; decode_batch: every per-pattern launch
           of the call) followed by a read of a 2 x L2 buffer, which evicts -- and so writes
           back and counts -- every line the call left dirty in L2;
  range 2: the same L2-sized read alone.
bytes per call = range 1 - range 2 (read + write); the call's duration likewise.  Range
replay measures the call as one unit, so write-backs that land during the next launch of
the chain are counted once (per-kernel captures miss the dirty lines at each launch end).
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(cfg: str, op: str) -> None:
    import numpy as np
    import torch

    import bench
    import synth
    import paper_1312_5155_b200 as rsp

    c = bench.workload(cfg, 0)
    k, m, n, w, B, S = c["k"], c["m"], c["n"], c["w"], c["block_bytes"], c["stripes"]
    torch.cuda.set_device(0)
    plan = rsp.Plan(k, m, w, c["poly"])
    st = torch.empty((S, n, B), dtype=torch.uint8, device="cuda")
    rsp.synth_fill(st, k, seed=c["seed"])
    er = synth.erasure_table(cfg, c["seed"], S)
    plan.prepare(er)
    plan.encode_batch(st)
    for s in range(S):
        st[s, torch.from_numpy(er[s][er[s] >= 0].astype(np.int64)).cuda()] = 0xEE
    plan.decode_batch(st, er)
    for _ in range(2):
        plan.encode_batch(st)
        plan.decode_batch(st, er)
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    flush = torch.ones(2 * l2 // 4, dtype=torch.int32, device="cuda")
    flush.sum()  # warm: the reduction's scratch comes from the caching allocator afterwards
    torch.cuda.synchronize()
    call = (lambda: plan.encode_batch(st)) if op == "encode" else (lambda: plan.decode_batch(st, er))
    # ranges 1-2 as documented; 3 (empty) and 4 (two flushes) are diagnostics of the method
    for calls, flushes in ((1, 1), (0, 1), (0, 0), (0, 2)):
        torch.cuda.profiler.start()
        for _ in range(calls):
            call()
        for _ in range(flushes):
            flush.sum()  # reads 2 x L2: evicts (writes back) what the call left dirty
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
    print(json.dumps({"cfg": cfg, "op": op, "algorithmic_bytes": S * n * B, "flush_bytes": flush.numel() * 4,
                      "code_hash": bench.code_hash()}), flush=True)


def parse(path: str) -> list[dict]:
    """Per range: {metric: value (base units)} from an ncu --csv log (range replay)."""
    rows = [r for r in csv.reader(open(path)) if r]
    hdr_i = next(i for i, r in enumerate(rows) if "Metric Name" in r)
    h = rows[hdr_i]
    ci, ni, ui, vi = (h.index("ID") if "ID" in h else 0), h.index("Metric Name"), h.index("Metric Unit"), \
        h.index("Metric Value")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
             "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6,
             "ms": 1e-3}
    out: dict = {}
    for r in rows[hdr_i + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        out.setdefault(r[ci], {})[r[ni]] = v * scale.get(r[ui], 1.0)
    return [out[key] for key in sorted(out, key=lambda x: int(x) if x.isdigit() else x)]


def summarize(paths: list[str]) -> None:
    import bench
    dst = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        db = json.load(open(dst))
    except Exception:
        db = {}
    db["_what"] = ("whole-call DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) of one bench.py call, "
                   "ncu --replay-mode app-range over cudaProfilerStart/Stop ranges (tools/ncu_traffic.py): "
                   "[call + 2xL2 read] minus [2xL2 read alone], so lines the call left dirty in L2 are counted; "
                   "valid only for the library source with this code_hash (bench.py refuses others)")
    lines = []
    for p in paths:
        name = os.path.basename(p)
        cfg, op = name.split("_")[1], name.split("_")[2].split(".")[0]
        rng = parse(p)
        if len(rng) < 2:
            raise SystemExit(f"{p}: expected 2 ranges, got {len(rng)}")
        a, b = rng[0], rng[1]
        rd = a["dram__bytes_read.sum"] - b["dram__bytes_read.sum"]
        wr = a["dram__bytes_write.sum"] - b["dram__bytes_write.sum"]
        dur = a["gpu__time_duration.sum"] - b["gpu__time_duration.sum"]
        c = bench.workload(cfg, 0)
        alg = c["stripes"] * (c["k"] + c["m"]) * c["block_bytes"]
        tot = int(round(rd + wr))
        db.setdefault(cfg, {})[op] = {
            "bytes_per_call": tot, "read_bytes": int(round(rd)), "write_bytes": int(round(wr)),
            "algorithmic_bytes": alg, "traffic_over_algorithmic": round(tot / alg, 4),
            "ncu_call_seconds": dur, "ncu_dram_gbs": round(tot / dur / 1e9, 1) if dur > 0 else None,
            "code_hash": bench.code_hash(),
            "source": f"gpurun_out/{name} (ncu app-range, flush-corrected), summarized in profiles/",
        }
        lines.append(f"{cfg} {op}: read {rd / 1e9:.4f} GB write {wr / 1e9:.4f} GB total {tot / 1e9:.4f} GB "
                     f"= {tot / alg:.4f} x algorithmic {alg / 1e9:.4f} GB; ncu range {dur * 1e3:.3f} ms "
                     f"-> {tot / dur / 1e9 if dur > 0 else 0:.1f} GB/s")
        for i, r in enumerate(rng):
            lines.append(f"    range {i + 1}: read {r['dram__bytes_read.sum'] / 1e9:.4f} GB write "
                         f"{r['dram__bytes_write.sum'] / 1e9:.4f} GB time {r['gpu__time_duration.sum'] * 1e3:.3f} ms")
    with open(dst, "w") as f:
        json.dump(db, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2], sys.argv[3])
    else:
        summarize(sys.argv[2:])
