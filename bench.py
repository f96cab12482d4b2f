#!/usr/bin/env python3
"""bench.py -- RS-poly encode + decode throughput on B200 (BASELINE.json metric).

One STEP = one pass of the whole hot path over the batch resident in HBM:
rs_poly_encode_batch (parity = d(x) x^m mod g(x)) followed by
rs_poly_decode_batch with a per-stripe erasure pattern.  Each pass
counts the batch's user data S*k*B once, so value = 2*S*k*B*N / max-rank time.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5|C3|C4]
  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...
  python bench.py --impl reference ...   # the CPU oracle, timed on this host's cores

Default workload: BASELINE.json configs[4] (C5): RS(10,4) over GF(2^8)/0x11D,
51 stripes x 10 x 16 MiB of synthetic data per GPU (seed = rank), 4 random erasures
per stripe -- the config the metric is quoted on ("per GPU and at 8xB200").
Stripes shard across ranks with no data exchange (weak scaling); NCCL only carries
the barrier and the max-over-ranks time / summed mismatch counts.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402  (seeded input generator shared by both sides)

MEASURED_PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback, used only if MEASURED_PEAKS.json is absent
METRIC = "RS poly encode/decode GB/s of data per GPU and at 8×B200; % of HBM roofline"

WORKLOADS = {
    "C5": "RS(10,4) GF(2^8)/0x11D, 51 stripes x 10 x 16 MiB per GPU (seed=rank), encode + 4-random-erasure decode",
    "C3": "RS(10,4) GF(2^8)/0x11D, 512 stripes x 10 x 4 MiB per GPU, encode + decode with 4 erasures "
          "(even stripes data-only)",
    "C4": "RS(12,4) GF(2^16)/0x1100B LE uint16, 256 stripes x 12 x 8 MiB per GPU, encode + 4-erasure decode",
}


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C5", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=None, help="end-to-end steps (default: min(steps, 5))")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="CPU baseline sample duration")
    ap.add_argument("--jit", default="on", choices=["on", "off"], help="per-pattern JIT decode kernels")
    ap.add_argument("--verify", default="full", choices=["full", "sampled"],
                    help="oracle check before timing: every stripe (default) or stripes 0, S/2, S-1")
    return ap.parse_args()


def hbm_peak():
    try:
        with open(MEASURED_PEAKS) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def copy_peak_in_run(dev) -> float:
    """GB/s of b.copy_(a) on 1 Gi bf16 elements (read + write bytes, best of 10, CUDA events):
    the MEASURED_PEAKS.json method, repeated in this run on this box."""
    import torch
    a = torch.empty(1 << 30, dtype=torch.bfloat16, device=dev)
    b = torch.empty_like(a)
    best = float("inf")
    for _ in range(11):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        b.copy_(a)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    torch.cuda.empty_cache()
    return 2 * (1 << 30) * 2 / (best / 1e3) / 1e9


LIB_SOURCES = ("paper_1312_5155_b200/csrc", "include")


def code_hash() -> str:
    """sha256 (16 hex digits) of the library's sources: kernels, planner, JIT generator and the
    ABI header -- the code an ncu traffic capture is valid for."""
    import hashlib
    h = hashlib.sha256()
    for d in LIB_SOURCES:
        base = os.path.join(ROOT, d)
        for name in sorted(os.listdir(base)):
            if name.endswith((".cu", ".cuh", ".cpp", ".hpp", ".h", ".py")):
                h.update(name.encode())
                with open(os.path.join(base, name), "rb") as f:
                    h.update(f.read())
    return h.hexdigest()[:16]


def ncu_traffic(cfg: str, op: str):
    """(DRAM bytes per call, ncu DRAM GB/s, source note) of one whole call from the committed ncu
    capture (tools/ncu_traffic.py); (None, None, why) unless taken on this exact library source."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            e = json.load(f)[cfg][op]
    except Exception:
        return None, None, "no capture for this config"
    if e.get("code_hash") != code_hash():
        return None, None, f"capture is of code {e.get('code_hash')}, not this build ({code_hash()}): refused"
    return int(e["bytes_per_call"]), e.get("ncu_dram_gbs"), e.get("source", "")


def allreduce(x: float, op: str, world: int, device) -> float:
    """Max/sum of a scalar over ranks (NCCL on the GPU box; gloo in tests/test_dist_gloo.py)."""
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op={"max": dist.ReduceOp.MAX, "sum": dist.ReduceOp.SUM}[op])
    return float(t.item())


def step_throughput(user_bytes_per_gpu: int, passes: int, world: int, max_step_ms: float) -> float:
    """Whole-job GB/s of user data: every rank processes its own stripes (weak scaling)."""
    return passes * user_bytes_per_gpu * world / (max_step_ms / 1e3) / 1e9


def workload(cfg: str, rank: int):
    c = dict(synth.CONFIGS[cfg])
    c["seed"] = rank  # C5: seed = rank (BASELINE.json); other configs: seed 0 on rank 0
    c["n"] = c["k"] + c["m"]
    c["name"] = cfg
    return c


# --------------------------------------------------------------------------------------
# CPU oracle leg (cpu_baseline and --impl reference)
# --------------------------------------------------------------------------------------
def oracle_sample(c, n_stripes: int, block_prefix: int):
    """Host copy of the first `block_prefix` bytes of every block of stripes 0..n_stripes-1
    (columns are independent codewords, so a column prefix is a valid sub-workload)."""
    st = synth.stripes_array(c["seed"], range(n_stripes), c["k"], c["m"], block_prefix)
    er = synth.erasure_table(c["name"], c["seed"], n_stripes)
    return st, er


def oracle_pass(oracle, st, er, c, threads):
    oracle.encode_bulk(st, c["k"], c["m"], c["w"], c["poly"], threads=threads)
    oracle.decode_bulk(st, er, c["k"], c["m"], c["w"], c["poly"], threads=threads)


def cpu_model() -> str:
    """The host CPU's model string (/proc/cpuinfo), for the baseline's context (P:361 states the paper's)."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def core_partition(local_rank: int, local_world: int) -> list[int]:
    """This rank's share of the node's host cores: the process affinity split into
    local_world contiguous slices (the ranks of one node share its cores)."""
    cpus = sorted(os.sched_getaffinity(0))
    per = max(1, len(cpus) // max(1, local_world))
    lo = min(local_rank * per, max(0, len(cpus) - per))
    return cpus[lo:lo + per]


def cpu_baseline(c, seconds: float, cpus: list[int] | None = None):
    """The oracle (as it stands) on host cores: `cpus` (default: all of this process's), one
    thread per core and per stripe, on a bounded prefix of the config's stripes."""
    import oracle
    old_aff = os.sched_getaffinity(0)
    if cpus:
        os.sched_setaffinity(0, cpus)
    try:
        cores = len(os.sched_getaffinity(0))
        threads = max(1, min(cores, c["stripes"]))
        prefix = min(c["block_bytes"], 2 << 20)
        st, er = oracle_sample(c, threads, prefix)
        oracle_pass(oracle, st, er, c, threads)  # warm
        passes, t0 = 0, time.perf_counter()
        while True:
            oracle_pass(oracle, st, er, c, threads)
            passes += 1
            el = time.perf_counter() - t0
            if el >= seconds:
                break
        user = threads * c["k"] * prefix
        # single thread, one stripe: the paper's per-core framing
        st1, er1 = oracle_sample(c, 1, prefix)
        p1, t1 = 0, time.perf_counter()
        while True:
            oracle_pass(oracle, st1, er1, c, 1)
            p1 += 1
            e1 = time.perf_counter() - t1
            if e1 >= seconds / 4:
                break
    finally:
        os.sched_setaffinity(0, old_aff)
    single = {"value": round(2 * c["k"] * prefix * p1 / e1 / 1e9, 4), "unit": "GB/s", "cores": 1,
              "sample": f"1 stripe x {c['k']} data blocks x first {prefix} B, {p1} passes in {e1:.1f} s"}
    return {"value": round(2 * user * passes / el / 1e9, 4), "unit": "GB/s", "cores": threads, "kind": "oracle",
            "threads": threads, "cpu_model": cpu_model(), "host_cpus": os.cpu_count(),
            "single_thread": single,
            "sample": f"{threads} stripes x {c['k']} data blocks x first {prefix} B of each block "
                      f"({user / 2**20:.0f} MiB user data), encode + decode with the config's erasure patterns, "
                      f"{passes} passes in {el:.1f} s, {threads} threads (one stripe each) on {cores} of "
                      f"{os.cpu_count()} host cores ({cpu_model()})"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    c = workload(args.config, 0)
    cores = os.cpu_count() or 1
    threads = max(1, min(cores, c["stripes"]))
    prefix = min(c["block_bytes"], 2 << 20)
    st, er = oracle_sample(c, threads, prefix)
    for _ in range(args.warmup):
        oracle_pass(oracle, st, er, c, threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle_pass(oracle, st, er, c, threads)
    el = time.perf_counter() - t0
    user = threads * c["k"] * prefix
    value = 2 * user * args.steps / el / 1e9
    sample = (f"per step: {threads} stripes x {c['k']} data blocks x first {prefix} B of each block of the "
              f"{args.config} workload, encode + decode; {threads} threads of {cores} host cores ({cpu_model()})")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(el / args.steps * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u8" if c["w"] == 8 else "u16", "data": "synthetic",
        "config": {"workload": f"{args.config}: {WORKLOADS[args.config]}", "k": c["k"], "m": c["m"], "w": c["w"],
                   "prim_poly": hex(c["poly"]), "block_bytes": c["block_bytes"], "stripes_per_gpu": c["stripes"],
                   "parallelism": f"dp{args.gpus}"},
        "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": threads, "kind": "oracle",
                         "threads": threads, "cpu_model": cpu_model(), "host_cpus": cores, "sample": sample},
        "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------------------
# clocks during the timed region (NVML)
# --------------------------------------------------------------------------------------
def nvml_handle(pynvml, cuda_index: int):
    """NVML handle of CUDA device `cuda_index`, matched by PCI address (NVML enumerates in its own
    order and ignores CUDA_VISIBLE_DEVICES); NVML index `cuda_index` if that fails."""
    try:
        import torch
        pr = torch.cuda.get_device_properties(cuda_index)
        bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
        return pynvml.nvmlDeviceGetHandleByPciBusId(bus)
    except Exception:
        return pynvml.nvmlDeviceGetHandleByIndex(cuda_index)


class ClockSampler:
    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
        "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
        "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100,
    }

    def __init__(self, index: int, period: float = 0.005):
        self.index, self.period = index, period
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._t = None
        self.ok = False

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = nvml_handle(pynvml, self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            return self
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for name, bit in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join()
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# --------------------------------------------------------------------------------------
# GPU leg
# --------------------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1312_5155_b200 as rsp

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # Harness self-test only (never set by the driver): RS_BENCH_HARNESS_TEST=1 runs every rank
    # on cuda:0 over gloo, to exercise the N > 1 code path on a one-GPU box.  The ranks'
    # kernels never wait on each other; the collectives are gloo's host-side ones.
    harness_test = os.environ.get("RS_BENCH_HARNESS_TEST") == "1"
    if harness_test:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if harness_test:
            dist.init_process_group("gloo")
        else:
            # NCCL's communicator-init lines on stderr (ranks, devices, transports) so that a
            # reader of the run's log can check nranks = N; not the data path (no collective on it)
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    c = workload(args.config, rank)
    k, m, n, w, B, S = c["k"], c["m"], c["n"], c["w"], c["block_bytes"], c["stripes"]
    plan = rsp.Plan(k, m, w, c["poly"])
    stream = torch.cuda.current_stream()
    stripes = torch.empty((S, n, B), dtype=torch.uint8, device=dev)
    rsp.synth_fill(stripes, k, seed=c["seed"], stripe0=0)
    er = synth.erasure_table(args.config, c["seed"], S)
    er_t = [torch.from_numpy(er[s][er[s] >= 0].astype(np.int64)).to(dev) for s in range(S)]
    if args.jit == "off":
        plan.set_jit(rsp.RS_JIT_OFF)
    # setup (outside the timed region, reported separately): the paper's Opt1/Opt3
    # per-pattern precomputation, here including the per-pattern JIT decode kernels
    t_setup = time.perf_counter()
    plan.prepare(er)
    setup_ms = (time.perf_counter() - t_setup) * 1e3

    # ---- correctness before any number: every byte of every stripe vs the CPU oracle ----
    # (outside the timed region, MDS uniqueness P:33).  At N > 1 the ranks
    # share the node's cores, so rank r checks its stripes s = r (mod N): S stripes of
    # host work in total, as at N = 1.
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", world))
    vcpus = core_partition(local, local_world) if world > 1 else sorted(os.sched_getaffinity(0))
    vids = list(range(S)) if world == 1 else [s for s in range(S) if s % world == rank % world]
    if args.verify == "sampled":
        vids = sorted({0, S // 2, S - 1})

    def fetch(ids):
        return np.stack([stripes[s_].cpu().numpy() for s_ in ids])

    plan.encode_batch(stripes)
    torch.cuda.synchronize()
    checks = verify_full(fetch, c, er, vids, vcpus, phase="encode")
    golden = stripes.clone()
    for s in range(S):
        stripes[s].index_fill_(0, er_t[s], 0xEE)
    plan.decode_batch(stripes, er)
    torch.cuda.synchronize()
    checks += verify_full(fetch, c, er, vids, vcpus, phase="decode")
    roundtrip_ok = torch.equal(stripes, golden)
    mismatches = sum(len(ch["mismatched_stripes"]) for ch in checks) + (0 if roundtrip_ok else 1)

    # ---- warm-up ----
    for _ in range(args.warmup):
        plan.encode_batch(stripes)
        plan.decode_batch(stripes, er)
    barrier()

    # ---- timed region: K steps, per-call CUDA events on the launching stream ----
    K = args.steps
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * K + 1)]
    clk = ClockSampler(local).start()
    launches0 = rsp.launch_count()
    barrier()
    ev[0].record(stream)
    for i in range(K):
        plan.encode_batch(stripes)
        ev[2 * i + 1].record(stream)
        plan.decode_batch(stripes, er)
        ev[2 * i + 2].record(stream)
    torch.cuda.synchronize()
    barrier()
    clocks = clk.stop()
    launches = rsp.launch_count() - launches0
    enc_ms = [ev[2 * i].elapsed_time(ev[2 * i + 1]) for i in range(K)]
    dec_ms = [ev[2 * i + 1].elapsed_time(ev[2 * i + 2]) for i in range(K)]
    total_ms = ev[0].elapsed_time(ev[2 * K])
    total_ms = allreduce(total_ms, "max", world, dev)
    enc_avg, dec_avg = statistics.mean(enc_ms), statistics.mean(dec_ms)

    # post-run check: the timed passes (ending with a decode) left exactly the verified batch
    after_ok = torch.equal(stripes, golden)
    del golden
    torch.cuda.empty_cache()
    mismatches += 0 if after_ok else 1
    mismatches = int(allreduce(float(mismatches), "sum", world, dev))
    verified_bytes = int(allreduce(float(sum(ch["bytes"] for ch in checks if ch["phase"] == "decode")), "sum",
                                   world, dev))

    user_bytes = S * k * B                      # per GPU per pass
    moved = S * (k + m) * B                     # HBM bytes per pass (read once or written once)
    value = step_throughput(user_bytes, 2, world, total_ms / K)
    peak, peak_src = hbm_peak()
    peak_run = copy_peak_in_run(dev)
    jst = plan.stats()
    dec_kernel = "rs_jit (per-pattern NVRTC XOR network)" if jst["jit_launches"] else "sliced_kernel decode (tables)"
    dom_ms, dom_name = (dec_avg, "decode: " + dec_kernel) if dec_avg >= enc_avg else (enc_avg, "encode: sliced_kernel")
    achieved = moved / (dom_ms / 1e3) / 1e9
    traffic, ncu_gbs, traffic_src = ncu_traffic(args.config, "decode" if dom_name.startswith("decode") else "encode")

    # ---- end to end through the public API from pinned host memory ----
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, plan, stripes, er, c, world, dev, barrier)

    cpu = None
    if not args.no_cpu_baseline:
        if world == 1:
            cpu = cpu_baseline(c, args.cpu_seconds)
        else:  # every rank on its own slice of the node's cores, concurrently
            part = core_partition(local, local_world)
            mine = cpu_baseline(c, args.cpu_seconds, cpus=part)
            mine.update(rank=rank, cpus=f"{part[0]}-{part[-1]}")
            per_rank = [None] * world
            dist.all_gather_object(per_rank, mine)
            cpu = {"value": round(sum(r_["value"] for r_ in per_rank), 4), "unit": "GB/s",
                   "cores": sum(r_["cores"] for r_ in per_rank), "kind": "oracle",
                   "threads": sum(r_["threads"] for r_ in per_rank), "cpu_model": cpu_model(),
                   "host_cpus": os.cpu_count(),
                   "sample": f"each of the {world} ranks ran the oracle on its own core slice at the same time "
                             f"({per_rank[0]['sample']}); value = sum over ranks",
                   "per_rank": [{k_: r_[k_] for k_ in ("rank", "cpus", "cores", "value", "single_thread")}
                                for r_ in per_rank]}

    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": round(total_ms / K, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8" if w == 8 else "u16", "data": "synthetic",
        "config": {"workload": f"{args.config}: {WORKLOADS[args.config]}", "k": k, "m": m, "w": w,
                   "prim_poly": hex(c["poly"]), "block_bytes": B, "stripes_per_gpu": S,
                   "bytes_per_gpu": S * n * B, "parallelism": f"dp{world}",
                   "kernels": plan.kernel_kind,
                   "l2": f"inputs {S * n * B / 2**30:.1f} GiB per GPU >> 126 MB L2: no flush needed"},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic, "traffic_source": traffic_src,
                     "traffic_over_algorithmic": round(traffic / moved, 4) if traffic else None,
                     "ncu_dram_gbs": ncu_gbs,
                     "dram_gbs_in_run": round(traffic / (dom_ms / 1e3) / 1e9, 1) if traffic else None,
                     "code_hash": code_hash(),
                     "kernel": f"{dom_name}; {moved} algorithmic bytes per call = S*(k+m)*B, avg {dom_ms:.4f} ms",
                     "peak_source": peak_src,
                     "peak_in_run": round(peak_run, 1), "frac_in_run": round(achieved / peak_run, 4),
                     "frac_nominal_8tbs": round(achieved / 8000.0, 4)},
        "encode": {"gbs_user": round(user_bytes / (enc_avg / 1e3) / 1e9, 2), "ms": round(enc_avg, 4),
                   "hbm_frac": round(moved / (enc_avg / 1e3) / 1e9 / peak, 4),
                   "ms_min_med_max": [round(min(enc_ms), 4), round(statistics.median(enc_ms), 4), round(max(enc_ms), 4)]},
        "decode": {"gbs_user": round(user_bytes / (dec_avg / 1e3) / 1e9, 2), "ms": round(dec_avg, 4),
                   "hbm_frac": round(moved / (dec_avg / 1e3) / 1e9 / peak, 4),
                   "ms_min_med_max": [round(min(dec_ms), 4), round(statistics.median(dec_ms), 4), round(max(dec_ms), 4)]},
        "verified": {"mismatches": mismatches,
                     "how": (f"all S*n*B bytes vs oracle: every byte of {'every stripe' if args.verify == 'full' else 'stripes ' + str(vids)}"
                             f"{' (rank r: stripes = r mod N)' if world > 1 and args.verify == 'full' else ''} "
                             "compared with the CPU oracle's encode (oracle/rs_oracle.c long division of the "
                             "synth data) after the device encode, and with the oracle's own decode of the same "
                             "erasures after the device decode; plus device round trip and the batch after "
                             "the timed passes equal to that verified state"),
                     "oracle_bytes_compared_per_phase": verified_bytes,
                     "checks": [{k_: v for k_, v in ch.items() if k_ != "mismatched_stripes"} |
                                {"mismatched": len(ch["mismatched_stripes"])} for ch in checks]},
        "gpu_launches": launches,
        "setup": {"ms": round(setup_ms, 1), "what": "rs_poly_prepare: decode constants + JIT kernels for the "
                  "batch's erasure patterns (once per pattern, outside the timed region)",
                  "stats": {k_: v for k_, v in jst.items()}},
        "clocks": clocks,
    }
    if e2e is not None:
        line["e2e"] = e2e
    if cpu is not None:
        line["cpu_baseline"] = cpu
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0 if mismatches == 0 else 1


def verify_full(fetch, c, er, ids, cpus, phase: str) -> list[dict]:
    """Bit-exact check of stripes `ids` against the oracle (oracle/fullcheck.py) on `cpus`."""
    from oracle import fullcheck
    old = os.sched_getaffinity(0)
    os.sched_setaffinity(0, cpus)
    try:
        if phase == "encode":
            r = fullcheck.check_encode(fetch, c, ids, threads=len(cpus))
        else:
            r = fullcheck.check_decode(fetch, c, er, ids, threads=len(cpus))
    finally:
        os.sched_setaffinity(0, old)
    r["phase"] = phase
    r["threads"] = len(cpus)
    return [r]


def gpu_local_cpus(index: int):
    """CPUs NVML reports as local to GPU `index` (its NUMA node), within our affinity; None if unknown."""
    try:
        import pynvml
        pynvml.nvmlInit()
        h = nvml_handle(pynvml, index)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
        cpus = {64 * i + b for i, mk in enumerate(words) for b in range(64) if (mk >> b) & 1}
        cpus &= os.sched_getaffinity(0)
        return cpus or None
    except Exception:
        return None


def run_e2e(args, plan, stripes, er, c, world, dev, barrier):
    import torch
    K = args.e2e_steps if args.e2e_steps is not None else min(args.steps, 5)
    K = max(1, K)
    S, k, B = c["stripes"], c["k"], c["block_bytes"]
    # pinned buffers and the copy-issuing thread on the GPU's own NUMA node: pages are
    # placed where they are first touched, and a remote node costs PCIe bandwidth
    old_aff = os.sched_getaffinity(0)
    local = gpu_local_cpus(dev.index if dev.index is not None else 0)
    if local:
        os.sched_setaffinity(0, local)
    try:
        return _run_e2e(K, plan, stripes, er, S, k, B, world, dev, barrier, local, len(old_aff))
    finally:
        os.sched_setaffinity(0, old_aff)


def host_budget_stripes(S, stripe_bytes, world):
    """Stripes whose pinned host copy fits in 40% of MemAvailable shared by the ranks of this
    node (8 ranks x the full 11 GiB batch would not fit every box)."""
    try:
        with open("/proc/meminfo") as f:
            avail = next(int(l.split()[1]) * 1024 for l in f if l.startswith("MemAvailable:"))
    except Exception:
        return S
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", world))
    return max(1, min(S, int(0.4 * avail / max(1, local_world) // stripe_bytes)))


def _run_e2e(K, plan, stripes, er, S, k, B, world, dev, barrier, local, n_all):
    import torch
    S = host_budget_stripes(S, stripes[0].numel(), world)
    stripes, er = stripes[:S], er[:S]
    host = torch.empty(tuple(stripes.shape), dtype=torch.uint8, pin_memory=True)
    host.copy_(stripes)
    plan.encode_host(host)  # warm
    plan.decode_host(host, er)
    barrier()
    t0 = time.perf_counter()
    h2d = d2h = 0
    t_enc, t_dec = [], []
    for _ in range(K):
        ta = time.perf_counter()
        a, b = plan.encode_host(host)
        tb = time.perf_counter()
        c2, d = plan.decode_host(host, er)
        t_enc.append(tb - ta)
        t_dec.append(time.perf_counter() - tb)
        h2d += a + c2
        d2h += b + d
    barrier()
    el = allreduce(time.perf_counter() - t0, "max", world, dev)
    ok = all(torch.equal(host[s], stripes[s].cpu()) for s in range(S))  # stripe by stripe: no 2nd full copy
    value = step_throughput(S * k * B, 2, world, el / K * 1e3)
    return {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": h2d // K, "d2h_bytes_per_step": d2h // K,
            "steps": K, "ms_per_step": round(el / K * 1e3, 3), "verified": bool(ok), "stripes": S,
            "encode_host_ms": round(statistics.median(t_enc) * 1e3, 2),
            "decode_host_ms": round(statistics.median(t_dec) * 1e3, 2),
            "host_cpus": (f"{len(local)} GPU-local CPUs of {n_all} (NVML affinity)" if local else "all"),
            "how": "rs_poly_encode_host + rs_poly_decode_host on pinned host stripes; host->device inputs, "
                   "device->host outputs inside the timed region (wall clock, max over ranks)"}


def free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def launch_ranks(args) -> int | None:
    """One process per GPU.  Under a launcher (WORLD_SIZE set) --gpus must match the world
    size; without one, --gpus N > 1 re-executes this command under torch.distributed.run
    (N ranks on this node, rendezvous on 127.0.0.1) and returns its exit code."""
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is not None:
        if int(env_world) != args.gpus:
            print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={env_world} (one rank per GPU): refusing to run",
                  file=sys.stderr, flush=True)
            return 2
        return None
    if args.gpus <= 1:
        return None
    import subprocess
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(sys.argv[0])] + sys.argv[1:]
    print("bench.py: launching", " ".join(cmd[1:]), file=sys.stderr, flush=True)
    return subprocess.call(cmd)


def main():
    args = parse_args()
    rc = launch_ranks(args)
    if rc is not None:
        return rc
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
