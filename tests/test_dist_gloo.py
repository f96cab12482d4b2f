"""The N>1 harness path of bench.py on CPU: world_size 2 over gloo.

The data path does not communicate (stripes shard by rank); the
process group only carries the barrier, the max-over-ranks time and the summed
mismatch count.  This checks those reductions, the per-rank sharding of the
synthetic workload, and that the reference arm runs on rank 0 only.
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    import bench
    import synth
    dist.init_process_group("gloo", rank=rank, world_size=world)
    t = bench.allreduce(10.0 + rank, "max", world, "cpu")
    mism = bench.allreduce(float(rank), "sum", world, "cpu")
    c = bench.workload("C5", rank)
    er = synth.erasure_table("C5", c["seed"], c["stripes"])
    first = synth.data_block(c["seed"], 0, 0, 64)
    dist.barrier()
    out[rank] = dict(t=t, mism=mism, seed=c["seed"], er=er.tolist(), first=first.tolist())
    dist.destroy_process_group()


def test_two_rank_reductions_and_sharding():
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    r0, r1 = out[0], out[1]
    assert r0["t"] == r1["t"] == 11.0          # max over ranks
    assert r0["mism"] == r1["mism"] == 1.0     # sum over ranks
    assert (r0["seed"], r1["seed"]) == (0, 1)  # C5: seed = rank
    assert r0["er"] != r1["er"] and r0["first"] != r1["first"]  # disjoint synthetic shards


def test_step_throughput_weak_scaling():
    import bench
    one = bench.step_throughput(10 << 20, 2, 1, 5.0)
    eight = bench.step_throughput(10 << 20, 2, 8, 5.0)
    assert abs(eight - 8 * one) < 1e-9
    assert abs(one - 2 * (10 << 20) / 5e-3 / 1e9) < 1e-9


def test_reference_arm_under_torchrun_prints_once():
    """--impl reference under the launcher: rank 0 prints one JSON line, rank 1 exits 0 silently."""
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0", "--config", "C5"]
    env = dict(os.environ, OMP_NUM_THREADS="1")
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert np.isfinite(d["ms_per_step"])


def test_bench_full_verification_catches_one_flipped_byte():
    """T6 negative test of the harness: bench.py's whole-batch oracle check (oracle/fullcheck.py)
    reports a single corrupted byte anywhere in a stripe, after encode and after decode (CPU
    arrays stand in for the device copies; the check itself is host-side)."""
    sys.path.insert(0, ROOT)
    import bench
    import oracle
    import synth
    c = bench.workload("C1", 0)
    c["stripes"] = 3
    c["block_bytes"] = 4096 + 40          # a ragged length
    er = synth.erasure_table("C1", 0, 3)
    good = synth.stripes_array(c["seed"], range(3), c["k"], c["m"], c["block_bytes"])
    oracle.encode_bulk(good, c["k"], c["m"], c["w"], c["poly"], threads=2)
    cpus = sorted(os.sched_getaffinity(0))
    ids = [0, 1, 2]
    for phase in ("encode", "decode"):
        dev = good.copy()
        r = bench.verify_full(lambda q: dev[q], c, er, ids, cpus, phase)[0]
        assert r["mismatched_stripes"] == [] and r["bytes"] == good.nbytes
        dev[1, c["k"] + 2, 4100] ^= 0x01      # one parity byte in the tail of stripe 1
        r = bench.verify_full(lambda q: dev[q], c, er, ids, cpus, phase)[0]
        assert r["mismatched_stripes"] == [1]


def test_bench_self_launches_ranks_for_gpus_n():
    """`bench.py --gpus 2` without an outside launcher re-executes itself under
    torch.distributed.run: one JSON line from rank 0 with n_gpus 2."""
    env = dict(os.environ, OMP_NUM_THREADS="1")
    env.pop("WORLD_SIZE", None)
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2", "--steps", "1",
           "--warmup", "0", "--config", "C5"]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "dp2"
    assert d["cpu_baseline"]["cpu_model"] and d["cpu_baseline"]["threads"] >= 1


def test_bench_refuses_gpus_world_size_mismatch():
    env = dict(os.environ, WORLD_SIZE="3", RANK="0")
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2", "--steps", "1"]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=120, env=env, cwd=ROOT)
    assert p.returncode != 0 and "WORLD_SIZE=3" in p.stderr and not p.stdout.strip()


def test_core_partition_slices_the_node():
    import bench
    cpus = sorted(os.sched_getaffinity(0))
    parts = [bench.core_partition(r, 2) for r in range(2)]
    if len(cpus) >= 2:
        assert set(parts[0]).isdisjoint(parts[1]) and len(parts[0]) == len(cpus) // 2
    assert all(p and set(p) <= set(cpus) for p in parts)
    assert bench.cpu_model()


def test_bench_traffic_capture_keyed_by_code_hash(tmp_path, monkeypatch):
    """bench.py reports an ncu traffic capture only for the library source it was taken on."""
    import bench
    prof = tmp_path / "profiles"
    prof.mkdir()
    entry = {"bytes_per_call": 12_000_000_000, "ncu_dram_gbs": 5000.0, "source": "x"}
    (prof / "ncu_traffic.json").write_text(json.dumps({"C5": {"decode": dict(entry, code_hash="0" * 16)}}))
    real_hash = bench.code_hash()
    monkeypatch.setattr(bench, "ROOT", str(tmp_path))
    monkeypatch.setattr(bench, "code_hash", lambda: real_hash)
    t, gbs, why = bench.ncu_traffic("C5", "decode")
    assert t is None and gbs is None and "refused" in why
    (prof / "ncu_traffic.json").write_text(json.dumps({"C5": {"decode": dict(entry, code_hash=real_hash)}}))
    assert bench.ncu_traffic("C5", "decode")[:2] == (12_000_000_000, 5000.0)
    assert bench.ncu_traffic("C4", "decode")[0] is None


def test_code_hash_tracks_library_sources():
    import bench
    h = bench.code_hash()
    assert len(h) == 16 and h == bench.code_hash()
