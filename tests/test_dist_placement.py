"""Cross-GPU stripe placement (NEXT-4): the host-side protocol with gloo ranks on CPU.

paper_1312_5155_b200/placement.py runs SPMD: local partial parities, an all_to_all of the
partials to the parity owners, XOR reduction.  Here the compute steps are CPU stand-ins
built from the oracle (test infrastructure; the product uses the CUDA kernels, checked in
tests/test_gpu_placement.py), so what is tested is the placement, the wire order and the
reduction bookkeeping: every owner's parity must equal the oracle's encoding of the stripe.
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth

from tests.placement_ops import P8, OracleOps  # noqa: E402


def _worker(rank, world, k, m, S, B, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1312_5155_b200.placement import Layout, encode_distributed
    lay = Layout(k, m, world)
    full = synth.stripes_array(3, range(S), k, m, B)
    store = {}
    for s in range(S):
        for b in lay.blocks_on(rank, s):
            store[(s, b)] = torch.from_numpy(full[s, b].copy()) if b < k else torch.full((B,), 0xCD, dtype=torch.uint8)

    def a2a(send, in_splits, out_splits):
        out = torch.empty((sum(out_splits), B), dtype=torch.uint8)
        dist.all_to_all_single(out.view(-1), send.reshape(-1).contiguous(),
                               [x * B for x in out_splits], [x * B for x in in_splits])
        return out

    stats = encode_distributed(lay, store, S, B, rank, a2a, OracleOps(k, m))
    ref = full.copy()
    oracle.encode_bulk(ref, k, m, 8, P8)
    bad = 0
    for (s, b), t in store.items():
        bad += int(not np.array_equal(t.numpy(), ref[s, b]))
    q.put((rank, bad, stats))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,k,m", [(2, 10, 4), (3, 6, 3), (4, 2, 2)])
def test_placement_protocol_gloo(world, k, m):
    S, B = 7, 96
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + world * 7 + k
    ps = [ctx.Process(target=_worker, args=(r, world, k, m, S, B, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    assert all(bad == 0 for _, bad, _ in res), res
    assert sum(st["sent_blocks"] for _, _, st in res) == sum(st["received_blocks"] for _, _, st in res)


def test_layout_owner_rotation():
    from paper_1312_5155_b200.placement import Layout
    lay = Layout(10, 4, 8)
    for s in range(8):
        assert sorted(b for r in range(8) for b in lay.blocks_on(r, s)) == list(range(14))
    owners = [lay.parity_owner(i, s) for s in range(8) for i in range(4)]
    assert sorted(set(owners)) == list(range(8))          # rotation spreads parity ownership


def _worker_p2p(rank, world, k, m, S, B, port, recv_bufs, q):
    """Fused variant: partials are stored straight into the owners' receive buffers (here
    shared-memory tensors standing in for NVLink-mapped peer memory)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1312_5155_b200.placement import Layout, encode_distributed_p2p
    lay = Layout(k, m, world)
    full = synth.stripes_array(4, range(S), k, m, B)
    store = {}
    for s in range(S):
        for b in lay.blocks_on(rank, s):
            store[(s, b)] = torch.from_numpy(full[s, b].copy()) if b < k else torch.full((B,), 0xCD, dtype=torch.uint8)
    stats = encode_distributed_p2p(lay, store, S, B, rank, recv_bufs, dist.barrier, OracleOps(k, m))
    ref = full.copy()
    oracle.encode_bulk(ref, k, m, 8, P8)
    bad = sum(int(not np.array_equal(t.numpy(), ref[s, b])) for (s, b), t in store.items())
    q.put((rank, bad, stats))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,k,m", [(2, 10, 4), (3, 6, 3), (4, 2, 2)])
def test_placement_p2p_protocol_gloo(world, k, m):
    from paper_1312_5155_b200.placement import Layout, recv_slots
    S, B = 7, 64
    lay = Layout(k, m, world)
    rows = max(1, max(len(recv_slots(lay, d, S)) for d in range(world)))
    bufs = [torch.zeros((rows, B), dtype=torch.uint8).share_memory_() for _ in range(world)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + world * 7 + k
    ps = [ctx.Process(target=_worker_p2p, args=(r, world, k, m, S, B, port, bufs, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    assert all(bad == 0 for _, bad, _ in res), res
    assert sum(st["sent_blocks"] for _, _, st in res) == sum(st["received_blocks"] for _, _, st in res)


def test_placement_launched_like_bench_gloo():
    """The SPMD job through bench.py's launcher path (`--gpus 2` re-executes under
    torch.distributed.run): gloo ranks, oracle compute steps, all_to_all exchange, two calls
    reusing the buffers, every owned block equal to the oracle's encoding."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, OMP_NUM_THREADS="1")
    env.pop("WORLD_SIZE", None)
    p = subprocess.run([sys.executable, os.path.join(root, "tests", "placement_worker.py"), "--gpus", "2",
                        "--backend", "gloo"], capture_output=True, text=True, timeout=600, env=env, cwd=root)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["world"] == 2 and d["mismatched_blocks"] == 0 and d["sent_blocks"] == d["received_blocks"] > 0


def _worker_peer_check(rank, world, port, allow, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1312_5155_b200.placement import check_peer_access
    try:
        check_peer_access(device=rank, can_access=lambda a, b: allow)
        q.put((rank, "ok"))
    except RuntimeError as e:
        q.put((rank, str(e)))
    dist.destroy_process_group()


@pytest.mark.parametrize("allow", [True, False])
def test_peer_access_guard_raises_on_every_rank(allow):
    """Without peer access the fused path refuses on every rank with a clear error (no hang)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29800 + int(allow)
    ps = [ctx.Process(target=_worker_peer_check, args=(r, 2, port, allow, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    if allow:
        assert res == {0: "ok", 1: "ok"}
    else:
        assert all("peer access" in v and "cuda:0 -> cuda:[1]" in v for v in res.values()), res
