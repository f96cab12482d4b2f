"""GPU parity of the run-time specialised (NVRTC) kernels vs the CPU oracle."""
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


def encoded(k, m, w, poly, B, S, seed):
    st = synth.stripes_array(seed, range(S), k, m, B)
    oracle.encode_bulk(st, k, m, w, poly, threads=8)
    return st


@pytest.mark.parametrize("k,m,w,poly,B", [(10, 4, 8, P8, 64 * 1024 + 40), (12, 4, 16, P16, 32 * 1024 + 6),
                                          (6, 3, 8, P8, 8192), (5, 2, 8, P8, 4096 + 3), (10, 6, 8, P8, 2048)])
def test_jit_decode_matches_oracle(k, m, w, poly, B):
    S, n = 12, k + m
    ref = encoded(k, m, w, poly, B, S, seed=21)
    rng = np.random.default_rng(k + 100 * m)
    er = np.full((S, m), -1, dtype=np.int32)
    for s in range(S):
        t = [m, 1, m][s] if s < 3 else int(rng.integers(1, m + 1))
        er[s, :t] = rng.choice(n, t, replace=False)
    er[5] = er[4]  # two stripes sharing a pattern -> one launch covers both
    bad = ref.copy()
    for s in range(S):
        for b in er[s]:
            if b >= 0:
                bad[s, b] = 0x3C
    m_ = rs()
    plan = m_.Plan(k, m, w, poly)
    plan.set_jit(m_.RS_JIT_SYNC)
    d = torch.from_numpy(bad).cuda()
    plan.decode_batch(d, er)
    torch.cuda.synchronize()
    assert np.array_equal(d.cpu().numpy(), ref)
    st = plan.stats()
    assert st["jit_available"] == 1 and st["jit_failed"] == 0
    # the JIT body needs 32-byte aligned blocks (one unit = 32 columns of w/8 bytes)
    aligned = B % 32 == 0 and B >= 4 * w
    eligible = aligned and any((er[s] >= 0).sum() <= (8 if w == 8 else 4) for s in range(S))
    assert (st["jit_launches"] > 0) == eligible


def test_prepare_then_decode_uses_only_jit():
    k, m, B, S = 10, 4, 256 * 1024, 16
    ref = encoded(k, m, 8, P8, B, S, seed=22)
    er = synth.erasure_table("C5", 3, S)
    m_ = rs()
    plan = m_.Plan(k, m)
    plan.prepare(er)
    st = plan.stats()
    assert st["jit_ready"] == len({tuple(r) for r in er.tolist()}) and st["jit_pending"] == 0
    bad = ref.copy()
    for s in range(S):
        bad[s, er[s]] = 0
    d = torch.from_numpy(bad).cuda()
    plan.decode_batch(d, er)
    torch.cuda.synchronize()
    assert np.array_equal(d.cpu().numpy(), ref)
    st2 = plan.stats()
    # one launch per run of adjacent stripes sharing a pattern (nothing uploaded)
    rows = [tuple(r) for r in er.tolist()]
    runs = sum(1 for s in range(S) if s == 0 or rows[s] != rows[s - 1])
    assert st2["table_launches"] == 0 and st2["jit_launches"] == runs


def test_prepare_all_then_any_pattern_runs_jit_only():
    """rs_poly_prepare_all: every <= m pattern compiled up front; a batch of never-requested
    random patterns (all of 1..m erasures) then decodes on JIT kernels only, bit-exactly."""
    from math import comb
    k, m, B, S = 6, 3, 32 * 1024, 24
    ref = encoded(k, m, 8, P8, B, S, seed=27)
    rng = np.random.default_rng(5)
    er = np.full((S, m), -1, dtype=np.int32)
    for s in range(S):
        t = 1 + s % m
        er[s, :t] = rng.choice(k + m, t, replace=False)
    m_ = rs()
    plan = m_.Plan(k, m)
    plan.prepare_all()
    st = plan.stats()
    n_pat = sum(comb(k + m, t) for t in range(1, m + 1))
    assert st["patterns"] == n_pat and st["jit_ready"] == n_pat and st["jit_pending"] == 0
    bad = ref.copy()
    for s in range(S):
        bad[s, er[s][er[s] >= 0]] = 0x77
    d = torch.from_numpy(bad).cuda()
    plan.decode_batch(d, er)
    torch.cuda.synchronize()
    assert np.array_equal(d.cpu().numpy(), ref)
    st2 = plan.stats()
    assert st2["table_launches"] == 0 and st2["jit_launches"] > 0


def test_background_mode_converges():
    """Background JIT: first calls use tables, later ones the compiled kernels; always exact."""
    import time
    k, m, B, S = 6, 3, 64 * 1024, 4
    ref = encoded(k, m, 8, P8, B, S, seed=23)
    er = np.array([[0, 2, 7], [1, -1, -1], [6, 7, 8], [0, 2, 7]], dtype=np.int32)
    m_ = rs()
    plan = m_.Plan(k, m)
    d = torch.from_numpy(ref).cuda()
    for it in range(60):
        for s in range(S):
            d[s, torch.from_numpy(er[s][er[s] >= 0].astype(np.int64)).cuda()] = 0
        plan.decode_batch(d, er)
        torch.cuda.synchronize()
        assert np.array_equal(d.cpu().numpy(), ref)
        st = plan.stats()
        if st["jit_pending"] == 0 and st["jit_launches"] > 0:
            break
        time.sleep(0.1)
    assert st["jit_ready"] == 3 and st["jit_launches"] > 0


@pytest.mark.parametrize("k,m,w,poly", [(5, 2, 8, P8), (10, 4, 16, P16)])
def test_jit_encoder_for_codes_without_compiled_network(k, m, w, poly):
    B, S = 8192 + 64, 3
    ref = encoded(k, m, w, poly, B, S, seed=24)
    m_ = rs()
    plan = m_.Plan(k, m, w, poly)
    assert plan.kernel_kind == "generic"
    plan.set_jit(m_.RS_JIT_SYNC)
    d = torch.from_numpy(ref).cuda()
    d[:, k:] = 0
    plan.encode_batch(d)
    torch.cuda.synchronize()
    assert np.array_equal(d.cpu().numpy(), ref)
    assert plan.stats()["jit_launches"] == 1


@pytest.mark.parametrize("jit", [True, False])
@pytest.mark.parametrize("k,m,w,poly,B", [(10, 4, 8, P8, 64 * 1024 + 40), (12, 4, 16, P16, 32 * 1024 + 6),
                                          (6, 3, 8, P8, 8192), (10, 6, 8, P8, 4096)])
def test_k_survivor_read_policy(k, m, w, poly, B, jit):
    """RS_READ_K_SURVIVORS (NEXT-2): only k survivors are read when t < m; the unread
    survivors are overwritten with garbage first to prove they are not used."""
    S, n = 10, k + m
    ref = encoded(k, m, w, poly, B, S, seed=25)
    rng = np.random.default_rng(k * 7 + m)
    er = np.full((S, m), -1, dtype=np.int32)
    for s in range(S):
        t = 1 + (s % m)
        er[s, :t] = rng.choice(n, t, replace=False)
    m_ = rs()
    plan = m_.Plan(k, m, w, poly)
    plan.set_read_policy(m_.RS_READ_K_SURVIVORS)
    plan.set_jit(m_.RS_JIT_SYNC if jit else m_.RS_JIT_OFF)
    bad = ref.copy()
    for s in range(S):
        e = [b for b in er[s] if b >= 0]
        for b in e:
            bad[s, b] = 0x3C
        # the k survivors read are the first k non-erased blocks (data first); scribble the rest
        surv = [b for b in range(n) if b not in e]
        for b in surv[k:]:
            bad[s, b] = 0x77
    d = torch.from_numpy(bad).cuda()
    plan.decode_batch(d, er)
    torch.cuda.synchronize()
    got = d.cpu().numpy()
    for s in range(S):
        for b in er[s]:
            if b >= 0:
                assert np.array_equal(got[s, b], ref[s, b]), (s, b)


def test_concurrent_host_threads_share_a_plan():
    """One plan used from 4 host threads at once (own streams, different batches and patterns,
    background JIT compiling while calls run): every result exact."""
    import threading
    k, m, B, S = 10, 4, 64 * 1024, 6
    m_ = rs()
    plan = m_.Plan(k, m)
    refs = [encoded(k, m, 8, P8, B, S, seed=50 + t) for t in range(4)]
    errs = []

    def worker(t):
        try:
            stream = torch.cuda.Stream()
            rng = np.random.default_rng(t)
            with torch.cuda.stream(stream):
                for it in range(6):
                    er = np.full((S, m), -1, dtype=np.int32)
                    for s in range(S):
                        tt = int(rng.integers(1, m + 1))
                        er[s, :tt] = rng.choice(k + m, tt, replace=False)
                    d = torch.from_numpy(refs[t]).cuda()
                    for s in range(S):
                        for b in er[s]:
                            if b >= 0:
                                d[s, int(b)] = 0
                    plan.decode_batch(d, er, stream=stream)
                    d2 = torch.from_numpy(refs[t]).cuda()
                    d2[:, k:] = 0
                    plan.encode_batch(d2, stream=stream)
                    stream.synchronize()
                    if not (np.array_equal(d.cpu().numpy(), refs[t]) and np.array_equal(d2.cpu().numpy(), refs[t])):
                        errs.append((t, it))
        except Exception as e:  # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=worker, args=(t,)) for t in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs


def test_jit_disk_cache(tmp_path, monkeypatch):
    """Second plan, same patterns: kernels come from the on-disk cubin cache, same bytes."""
    import time
    monkeypatch.setenv("RS_POLY_JIT_CACHE", str(tmp_path))
    k, m, B, S = 12, 4, 16384, 6
    ref = encoded(k, m, 16, P16, B, S, seed=60)
    er = synth.erasure_table("C4", 9, S)
    m_ = rs()
    p1 = m_.Plan(k, m, 16, P16)
    t0 = time.perf_counter()
    p1.prepare(er)
    t_compile = time.perf_counter() - t0
    assert p1.stats()["jit_cache_hits"] == 0 and len(list(tmp_path.iterdir())) >= 1
    p2 = m_.Plan(k, m, 16, P16)
    t0 = time.perf_counter()
    p2.prepare(er)
    t_cached = time.perf_counter() - t0
    st = p2.stats()
    assert st["jit_cache_hits"] == st["jit_ready"] > 0
    assert t_cached < t_compile
    d = torch.from_numpy(ref).cuda()
    for s in range(S):
        d[s, torch.from_numpy(er[s].astype(np.int64)).cuda()] = 0
    p2.decode_batch(d, er)
    torch.cuda.synchronize()
    assert np.array_equal(d.cpu().numpy(), ref)


def test_stress_many_patterns_repeated():
    """30 decode calls over 256 stripes with fresh random per-stripe patterns each time (PDL
    chains over two streams, table fallback while kernels compile), interleaved with encodes
    and diff-updates on the same stream: every byte right every time."""
    k, m, B, S = 10, 4, 16 * 1024 + 32, 256
    m_ = rs()
    plan = m_.Plan(k, m)
    ref = encoded(k, m, 8, P8, B, S, seed=70)
    d = torch.from_numpy(ref).cuda()
    golden = d.clone()
    rng = np.random.default_rng(70)
    for it in range(30):
        er = np.full((S, m), -1, dtype=np.int32)
        for s in range(S):
            t = int(rng.integers(1, m + 1))
            er[s, :t] = np.sort(rng.choice(k + m, t, replace=False))
        mask = torch.zeros((S, k + m), dtype=torch.bool, device="cuda")
        for s in range(S):
            mask[s, torch.from_numpy(er[s][er[s] >= 0].astype(np.int64)).cuda()] = True
        d[mask] = 0x11
        plan.decode_batch(d, er)
        if it % 3 == 0:
            plan.encode_batch(d)
        if it % 5 == 0:
            old = d[:, [2]].clone()
            d[:, 2] ^= 0x3C
            plan.update_batch(d, [2], old)
            d[:, 2] ^= 0x3C
            plan.update_batch(d, [2], old ^ 0x3C)
        assert torch.equal(d, golden), f"iteration {it}"


@pytest.mark.parametrize("k,m,w,poly", [(10, 4, 8, P8), (12, 4, 16, P16)])
def test_jit_pointer_api(k, m, w, poly):
    """Single-stripe entry points (host arrays of device pointers, blocks in separate
    allocations) through the JIT kernels: pointer-mode addressing in the generated code."""
    B = 64 * 1024
    ref = encoded(k, m, w, poly, B, 1, seed=80)[0]
    m_ = rs()
    plan = m_.Plan(k, m, w, poly)
    plan.set_jit(m_.RS_JIT_SYNC)
    blocks = [torch.from_numpy(ref[b].copy()).cuda() for b in range(k + m)]
    for b in range(k, k + m):
        blocks[b].zero_()
    plan.encode(blocks[:k], blocks[k:], B)
    er = [1, 3, k, k + m - 1]
    for b in er:
        blocks[b].fill_(0x42)
    plan.decode(blocks, B, er)
    torch.cuda.synchronize()
    for b in range(k + m):
        assert np.array_equal(blocks[b].cpu().numpy(), ref[b]), b
    assert plan.stats()["jit_launches"] >= 1


def test_no_device_memory_growth_over_many_calls():
    """400 encode/decode/update/verify calls: the per-call blobs, pinned slots and staging are
    reused or freed (device free memory stays put once the JIT modules are loaded)."""
    k, m, B, S = 10, 4, 32 * 1024, 24
    m_ = rs()
    plan = m_.Plan(k, m)
    ref = encoded(k, m, 8, P8, B, S, seed=99)
    d = torch.from_numpy(ref).cuda()
    er = synth.erasure_table("C5", 4, S)
    plan.prepare(er)
    flags = torch.zeros(S, dtype=torch.int32, device="cuda")
    old = d[:, [3]].clone()

    def burst(n):
        for _ in range(n):
            plan.encode_batch(d)
            plan.decode_batch(d, er)
            plan.update_batch(d, [3], old)
            plan.verify_batch(d, flags)
        torch.cuda.synchronize()

    burst(20)
    free0 = torch.cuda.mem_get_info()[0]
    burst(100)
    free1 = torch.cuda.mem_get_info()[0]
    assert free0 - free1 < (64 << 20), (free0, free1)
    assert torch.equal(d.cpu(), torch.from_numpy(ref))


def test_cuda_graph_capture():
    """Calls that only launch kernels can be captured in a CUDA graph (replays are bit-exact);
    a call that would upload per-call constants refuses capture (RS_ERR_CUDA) instead of
    baking a reused host buffer into the graph."""
    k, m, B, S = 10, 4, 64 * 1024, 4
    m_ = rs()
    plan = m_.Plan(k, m)
    ref = encoded(k, m, 8, P8, B, S, seed=111)
    d = torch.from_numpy(ref).cuda()
    er_same = np.tile(np.array([[1, 4, 10, 13]], dtype=np.int32), (S, 1))   # one shared pattern
    plan.prepare(er_same)
    cap = torch.cuda.Stream()
    with torch.cuda.stream(cap):                      # run once on the device before capturing
        plan.encode_batch(d, stream=cap)
        plan.decode_batch(d, er_same, stream=cap)
    torch.cuda.synchronize()
    g_enc, g_dec = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_enc, stream=cap):
        plan.encode_batch(d, stream=cap)
    with torch.cuda.graph(g_dec, stream=cap):
        plan.decode_batch(d, er_same, stream=cap)
    d[:, k:] = 0
    g_enc.replay()
    torch.cuda.synchronize()
    assert np.array_equal(d.cpu().numpy(), ref)
    d[:, [1, 4, 10, 13]] = 0x77
    g_dec.replay()
    torch.cuda.synchronize()
    assert np.array_equal(d.cpu().numpy(), ref)
    # patterns A, B, A, B: one launch per run of adjacent stripes, still nothing uploaded
    er_mixed = np.array([[1, 4, 10, 13], [0, 2, 3, 5], [1, 4, 10, 13], [0, 2, 3, 5]], dtype=np.int32)
    plan.prepare(er_mixed)
    with torch.cuda.stream(cap):
        plan.decode_batch(d, er_mixed, stream=cap)
    torch.cuda.synchronize()
    g_mixed = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_mixed, stream=cap):
        plan.decode_batch(d, er_mixed, stream=cap)
    for s_, row in enumerate(er_mixed):
        d[s_, list(row)] = 0x5A
    g_mixed.replay()
    torch.cuda.synchronize()
    assert np.array_equal(d.cpu().numpy(), ref)
    # a ragged block length: the tail kernel reads per-call pattern records -> refused
    Br = B - 40
    rag = torch.from_numpy(np.ascontiguousarray(encoded(k, m, 8, P8, Br, S, seed=112))).cuda()
    plan.decode_batch(rag, er_mixed)
    torch.cuda.synchronize()
    g_bad = torch.cuda.CUDAGraph()
    with pytest.raises((m_.RSError, RuntimeError)):
        with torch.cuda.graph(g_bad, stream=cap):
            plan.decode_batch(rag, er_mixed, stream=cap)
    torch.cuda.synchronize()


def test_alternating_patterns_keep_one_launch_per_pattern():
    """Two patterns alternating over many small stripes: runs of adjacent stripes would be
    one launch per stripe, so the batch keeps one launch per pattern (stripe lists in the
    uploaded blob); three patterns in long runs split into one launch per run."""
    k, m, B, S = 10, 4, 4096, 64
    ref = encoded(k, m, 8, P8, B, S, seed=113)
    m_ = rs()
    plan = m_.Plan(k, m)
    A, Bp, Cp = [1, 4, 10, 13], [0, 2, 3, 5], [6, 7, 8, 9]
    for rows, want in (([A if s % 2 == 0 else Bp for s in range(S)], 2),
                       ([A] * 20 + [Bp] * 20 + [A] * 14 + [Cp] * 10, 4)):
        er = np.array(rows, dtype=np.int32)
        plan.prepare(er)
        bad = ref.copy()
        for s in range(S):
            bad[s, er[s]] = 0xEE
        d = torch.from_numpy(bad).cuda()
        n0 = plan.stats()["jit_launches"]
        plan.decode_batch(d, er)
        torch.cuda.synchronize()
        assert np.array_equal(d.cpu().numpy(), ref)
        assert plan.stats()["jit_launches"] - n0 == want


@pytest.mark.parametrize("w", [8, 16])
def test_pdl_chain_completes_in_stream_order(w):
    """A decode call is a chain of per-pattern launches in which only each kernel's last CTA
    waits for its predecessor.  Work queued after the call on the same stream (here an
    asynchronous copy to pinned host memory) must still see every kernel's output: repeated
    calls with short kernels and many patterns, each followed at once by the copy."""
    k, m, poly = (10, 4, P8) if w == 8 else (12, 4, P16)
    B, S = 16 * 1024, 96
    ref = encoded(k, m, w, poly, B, S, seed=120 + w)
    m_ = rs()
    plan = m_.Plan(k, m, w, poly)
    d = torch.from_numpy(ref).cuda()
    host = torch.empty(d.shape, dtype=torch.uint8).pin_memory()
    rng = np.random.default_rng(w)
    stream = torch.cuda.current_stream()
    pats = np.array([np.sort(rng.choice(k + m, m, replace=False)) for _ in range(S)], dtype=np.int32)
    plan.prepare(pats)                                 # compiled once; each rep reorders them
    for rep in range(8):
        er = np.ascontiguousarray(pats[rng.permutation(S)])
        for s in range(S):
            d[s, list(er[s])] = 0xEE                   # queued on the same stream
        plan.decode_batch(d, er)
        host.copy_(d, non_blocking=True)
        stream.synchronize()
        assert np.array_equal(host.numpy(), ref), rep
