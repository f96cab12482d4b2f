"""Cross-GPU stripe placement (NEXT-4) with the CUDA kernels: N ranks emulated by host threads
on one GPU (the exchange is a host-side rendezvous plus device copies -- no kernel waits on
another), every owner's parity block equal to the oracle's encoding of the stripe.  Also the
two kernels on their own: partial encoding of a split of the data sums to the full encoding,
and the XOR reduction."""
import threading

import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
P8, P16 = 0x11D, 0x1100B


def rs():
    import paper_1312_5155_b200 as m
    return m


@pytest.mark.parametrize("k,m,w,poly,B", [(10, 4, 8, P8, 65536), (12, 4, 16, P16, 8192 + 6), (6, 3, 8, P8, 1000)])
def test_partial_encodings_sum_to_encode(k, m, w, poly, B):
    S = 3
    ref = synth.stripes_array(5, range(S), k, m, B)
    oracle.encode_bulk(ref, k, m, w, poly, threads=4)
    m_ = rs()
    plan = m_.Plan(k, m, w, poly)
    plan.set_jit(m_.RS_JIT_SYNC)
    d = torch.from_numpy(ref).cuda()
    halves = [list(range(0, k, 2)), list(range(1, k, 2))]
    parts = [torch.empty((S, m, B), dtype=torch.uint8, device="cuda") for _ in halves]
    for idx, p in zip(halves, parts):
        plan.encode_partial(idx, [[d[s, j] for j in idx] for s in range(S)], [[p[s, i] for i in range(m)]
                                                                             for s in range(S)], B)
    out = torch.empty((S, m, B), dtype=torch.uint8, device="cuda")
    plan.xor_reduce([out[s, i] for s in range(S) for i in range(m)],
                    [[parts[0][s, i], parts[1][s, i]] for s in range(S) for i in range(m)], B)
    # accumulate mode: second half XORed onto the first half's partial
    acc = parts[0].clone()
    plan.encode_partial(halves[1], [[d[s, j] for j in halves[1]] for s in range(S)],
                        [[acc[s, i] for i in range(m)] for s in range(S)], B, accumulate=True)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), ref[:, k:])
    assert np.array_equal(acc.cpu().numpy(), ref[:, k:])


@pytest.mark.parametrize("world,k,m", [(4, 10, 4), (3, 12, 4), (8, 6, 3)])
def test_placement_protocol_on_gpu(world, k, m):
    from paper_1312_5155_b200.placement import CudaOps, Layout, encode_distributed
    S, B = 9, 64 * 1024 + 32
    lay = Layout(k, m, world)
    full = synth.stripes_array(6, range(S), k, m, B)
    ref = full.copy()
    oracle.encode_bulk(ref, k, m, 8, P8, threads=4)
    m_ = rs()
    plans = [m_.Plan(k, m) for _ in range(world)]
    stores = []
    for r in range(world):
        st = {}
        for s in range(S):
            for b in lay.blocks_on(r, s):
                st[(s, b)] = torch.from_numpy(full[s, b].copy()).cuda() if b < k else \
                    torch.full((B,), 0xCD, dtype=torch.uint8, device="cuda")
        stores.append(st)
    sends = [None] * world
    bar = threading.Barrier(world)

    def make_a2a(rank):
        def a2a(send, in_splits, out_splits):
            torch.cuda.synchronize()
            sends[rank] = (send, in_splits)
            bar.wait()
            rows = []
            for src in range(world):
                sb, sp = sends[src]
                off = sum(sp[:rank])
                rows.append(sb[off:off + sp[rank]])
            recv = torch.cat(rows) if rows else torch.empty((0, B), dtype=torch.uint8, device="cuda")
            torch.cuda.synchronize()
            bar.wait()
            return recv
        return a2a

    errs = []

    def run(r):
        try:
            encode_distributed(lay, stores[r], S, B, r, make_a2a(r), CudaOps(plans[r]))
            torch.cuda.synchronize()
        except Exception as e:  # surfaced below
            errs.append(e)
            bar.abort()

    ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for r in range(world):
        for (s, b), t in stores[r].items():
            assert np.array_equal(t.cpu().numpy(), ref[s, b]), (r, s, b)


@pytest.mark.parametrize("world,k,m", [(4, 10, 4), (8, 6, 3)])
def test_placement_p2p_on_gpu(world, k, m):
    """Fused variant with the CUDA kernels: the partial-encode kernel writes straight into the
    owners' receive buffers (device tensors standing in for peer-mapped memory)."""
    from paper_1312_5155_b200.placement import CudaOps, Layout, encode_distributed_p2p, recv_slots
    S, B = 9, 32 * 1024
    lay = Layout(k, m, world)
    full = synth.stripes_array(7, range(S), k, m, B)
    ref = full.copy()
    oracle.encode_bulk(ref, k, m, 8, P8, threads=4)
    m_ = rs()
    rows = max(1, max(len(recv_slots(lay, d, S)) for d in range(world)))
    bufs = [torch.zeros((rows, B), dtype=torch.uint8, device="cuda") for _ in range(world)]
    stores = [{(s, b): (torch.from_numpy(full[s, b].copy()).cuda() if b < k else
                        torch.full((B,), 0xCD, dtype=torch.uint8, device="cuda"))
               for s in range(S) for b in lay.blocks_on(r, s)} for r in range(world)]
    bar = threading.Barrier(world)

    def barrier():
        torch.cuda.synchronize()
        bar.wait()

    errs = []

    def run(r):
        try:
            encode_distributed_p2p(lay, stores[r], S, B, r, bufs, barrier, CudaOps(m_.Plan(k, m)))
            torch.cuda.synchronize()
        except Exception as e:  # noqa: BLE001
            errs.append(e)
            bar.abort()

    ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for r in range(world):
        for (s, b), t in stores[r].items():
            assert np.array_equal(t.cpu().numpy(), ref[s, b]), (r, s, b)


def test_symmetric_memory_path_one_rank():
    """encode_distributed_p2p over torch symmetric memory (one-rank NCCL group, in a
    subprocess so the process group does not leak into other tests)."""
    import os
    import random
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SYMM_PORT=str(random.randint(30000, 39000)))
    out = subprocess.run([sys.executable, os.path.join(root, "tools", "symm_smoke.py")], capture_output=True,
                         text=True, timeout=300, cwd=root, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    assert "bad 0" in out.stdout, out.stdout
