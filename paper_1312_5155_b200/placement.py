"""Cross-GPU stripe placement: encode when a stripe's blocks live on different GPUs.

In a distributed store (the HDFS-RAID setting that motivates the paper) the n
blocks of a stripe sit on different nodes.  Here block b of stripe s lives on rank
``(b + s) % world`` (the rotation spreads parity ownership).  Because the code is linear
 and parity = sum_j P[:, j] d_j (the parity map of g), encoding splits into

1. **local partial parity**: every rank computes, for each stripe, the m partial parities of
   the data blocks it holds (``rs_poly_encode_partial``; the partial of a parity block the
   rank itself owns is written straight into that block);
2. **exchange**: each partial goes to the owner of its parity block, one ``all_to_all``
   over the process group (NCCL over NVLink/NVSwitch on GPUs);
3. **XOR reduction**: each owner adds (XORs, GF(2^w) addition) the partials it received into
   its parity block (``rs_poly_xor_reduce``).

The result equals rs_poly_encode of the whole stripe (tests/test_dist_placement.py checks it
against the oracle with gloo ranks; tests/test_gpu_placement.py runs the GPU kernels with
in-process ranks).  The byte traffic and the alternatives are discussed in DESIGN.md §8.

``encode_distributed_p2p`` is the fused variant: every rank's receive buffer is mapped into
its peers (torch symmetric memory over NVLink / NVSwitch), and the partial-encode kernel's
output pointers for a remote owner are the owner's receive slots -- the kernel's stores are
the transfer, overlapping the math tile by tile; one barrier, then the owners' XOR.

``ops`` supplies the compute steps; the default is the CUDA library (``Plan``).  Tests of the
host-side protocol inject CPU implementations -- the product path itself has no CPU fallback.
"""
from __future__ import annotations

from dataclasses import dataclass


def owner(block: int, stripe: int, world: int) -> int:
    """Rank holding API block `block` of stripe `stripe`."""
    return (block + stripe) % world


@dataclass
class Layout:
    k: int
    m: int
    world: int

    @property
    def n(self) -> int:
        return self.k + self.m

    def data_on(self, rank: int, s: int) -> list[int]:
        return [j for j in range(self.k) if owner(j, s, self.world) == rank]

    def parity_owner(self, i: int, s: int) -> int:
        return owner(self.k + i, s, self.world)

    def blocks_on(self, rank: int, s: int) -> list[int]:
        return [b for b in range(self.n) if owner(b, s, self.world) == rank]

    def sends(self, src: int, dst: int, S: int) -> list[tuple[int, int]]:
        """(stripe, parity index) partials rank `src` sends to rank `dst`, in wire order."""
        if src == dst:
            return []
        return [(s, i) for s in range(S) for i in range(self.m)
                if self.parity_owner(i, s) == dst and self.data_on(src, s)]


class CudaOps:
    """Compute steps on the GPU through the C ABI (the product path)."""

    def __init__(self, plan):
        self.plan = plan

    def encode_partial(self, idx, data, partial, nbytes):
        self.plan.encode_partial(idx, data, partial, nbytes, accumulate=False)

    def xor_reduce(self, dst, srcs, nbytes):
        self.plan.xor_reduce(dst, srcs, nbytes)

    def empty(self, nblocks, nbytes, like):
        import torch
        return torch.empty((nblocks, nbytes), dtype=torch.uint8, device=like.device)


def encode_distributed(lay: Layout, store: dict, S: int, nbytes: int, rank: int, all_to_all, ops) -> dict:
    """SPMD: run on every rank.  `store[(s, b)]` holds this rank's blocks (uint8 [nbytes]
    tensors; its parity blocks are overwritten).  `all_to_all(send, in_splits, out_splits)`
    moves a [rows, nbytes] buffer between ranks (rows per destination / source) and returns
    the received [rows, nbytes] buffer.  Returns counters for the caller's report."""
    k, m, N = lay.k, lay.m, lay.world
    like = next(iter(store.values()))
    # wire order of the send buffer: by destination rank, then (stripe, parity index)
    send_rows = {d: lay.sends(rank, d, S) for d in range(N)}
    row_of = {}
    for d in range(N):
        for si in send_rows[d]:
            row_of[si] = len(row_of)
    send = ops.empty(max(1, len(row_of)), nbytes, like)
    junk = ops.empty(1, nbytes, like)[0]  # target of partials nobody needs (rank without data in s)
    # 1. partial parities, batched by the set of local data blocks (N distinct sets under rotation)
    groups: dict[tuple, list[int]] = {}
    for s in range(S):
        groups.setdefault(tuple(lay.data_on(rank, s)), []).append(s)
    for idx, stripes in groups.items():
        data = [[store[(s, j)] for j in idx] for s in stripes]
        # owned parity blocks take this rank's partial directly; a rank without data in a
        # stripe writes zeros there (c = 0) and sends nothing
        partial = [[store[(s, k + i)] if lay.parity_owner(i, s) == rank
                    else (send[row_of[(s, i)]] if (s, i) in row_of else junk)
                    for i in range(m)] for s in stripes]
        ops.encode_partial(list(idx), data, partial, nbytes)
    # 2. exchange
    in_splits = [len(send_rows[d]) for d in range(N)]
    recv_rows = {r: lay.sends(r, rank, S) for r in range(N)}
    out_splits = [len(recv_rows[r]) for r in range(N)]
    recv = all_to_all(send[:sum(in_splits)], in_splits, out_splits)
    # 3. XOR the received partials into the owned parity blocks, batched by source count
    got: dict[tuple[int, int], list] = {}
    row = 0
    for r in range(N):
        for si in recv_rows[r]:
            got.setdefault(si, []).append(recv[row])
            row += 1
    by_n: dict[int, list] = {}
    for (s, i), parts in got.items():
        by_n.setdefault(len(parts), []).append((s, i, parts))
    for nsrc, items in by_n.items():
        dst = [store[(s, k + i)] for s, i, _ in items]
        srcs = [[store[(s, k + i)]] + parts for s, i, parts in items]
        ops.xor_reduce(dst, srcs, nbytes)
    return {"sent_blocks": sum(in_splits), "received_blocks": sum(out_splits),
            "local_partial_calls": len(groups), "xor_calls": len(by_n)}


def recv_slots(lay: Layout, dst: int, S: int) -> dict:
    """Row of every partial (src, stripe, parity index) in rank `dst`'s receive buffer
    (sources in rank order, then the wire order of Layout.sends)."""
    rows = {}
    for src in range(lay.world):
        for s, i in lay.sends(src, dst, S):
            rows[(src, s, i)] = len(rows)
    return rows


def encode_distributed_p2p(lay: Layout, store: dict, S: int, nbytes: int, rank: int, peer_recv: list,
                           barrier, ops) -> dict:
    """SPMD, fused compute + transfer.  `peer_recv[r]` is rank r's receive buffer ([rows,
    nbytes]; rows >= len(recv_slots(lay, r, S))) as seen from this rank -- a peer-mapped
    view (symmetric memory) on GPUs.  `barrier()` returns once every rank's partial stores
    are complete and visible.  Same result as encode_distributed.

    Reuse contract: the receive buffers may be reused by the next call.  A second barrier
    after the XOR reduction keeps a fast rank's next partial stores out of a peer's slots
    until that peer has read them."""
    k, m, N = lay.k, lay.m, lay.world
    like = next(iter(store.values()))
    slots = [recv_slots(lay, d, S) for d in range(N)]
    junk = ops.empty(1, nbytes, like)[0]
    groups: dict[tuple, list[int]] = {}
    for s in range(S):
        groups.setdefault(tuple(lay.data_on(rank, s)), []).append(s)
    sent = 0
    for idx, stripes in groups.items():
        data = [[store[(s, j)] for j in idx] for s in stripes]
        partial = []
        for s in stripes:
            row = []
            for i in range(m):
                d = lay.parity_owner(i, s)
                if d == rank:
                    row.append(store[(s, k + i)])
                elif idx:
                    row.append(peer_recv[d][slots[d][(rank, s, i)]])   # the store goes over NVLink
                    sent += 1
                else:
                    row.append(junk)
            partial.append(row)
        ops.encode_partial(list(idx), data, partial, nbytes)
    barrier()
    mine = peer_recv[rank]
    got: dict[tuple[int, int], list] = {}
    for (src, s, i), r in slots[rank].items():
        got.setdefault((s, i), []).append(mine[r])
    by_n: dict[int, list] = {}
    for (s, i), parts in got.items():
        by_n.setdefault(len(parts), []).append((s, i, parts))
    for nsrc, items in by_n.items():
        ops.xor_reduce([store[(s, k + i)] for s, i, _ in items],
                       [[store[(s, k + i)]] + parts for s, i, parts in items], nbytes)
    barrier()  # every rank has consumed its slots: the buffers may be written again
    return {"sent_blocks": sent, "received_blocks": len(slots[rank]), "local_partial_calls": len(groups),
            "xor_calls": len(by_n)}


def check_peer_access(group=None, can_access=None, device=None) -> None:
    """Raise on every rank (instead of hanging in the rendezvous or faulting in a kernel)
    unless each rank's GPU can map every other rank's GPU of the group
    (cudaDeviceCanAccessPeer; NVLink / NVSwitch).  Ranks on the same device need none."""
    import torch
    import torch.distributed as dist
    if can_access is None:
        can_access = torch.cuda.can_device_access_peer
    me = torch.cuda.current_device() if device is None else device
    devs = [None] * dist.get_world_size(group)
    dist.all_gather_object(devs, me, group=group)
    missing = sorted({d for d in devs if d != me and not can_access(me, d)})
    report = [None] * len(devs)
    dist.all_gather_object(report, (me, missing), group=group)
    bad = [(d, miss) for d, miss in report if miss]
    if bad:
        raise RuntimeError("no CUDA peer access (cudaDeviceCanAccessPeer) for "
                           + ", ".join(f"cuda:{d} -> cuda:{miss}" for d, miss in bad)
                           + ": the fused placement needs NVLink peer mappings; use encode_distributed "
                             "(all_to_all) instead")


def symmetric_recv_buffers(lay: Layout, S: int, nbytes: int, group=None):
    """Allocate this rank's receive buffer in symmetric memory and return (views of every
    rank's buffer as mapped here, device barrier).  Needs CUDA peer access (NVLink)."""
    import torch
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm_mem
    check_peer_access(group)
    rows = max(max(len(recv_slots(lay, d, S)) for d in range(lay.world)), 1)
    buf = symm_mem.empty((rows, nbytes), dtype=torch.uint8, device=torch.cuda.current_device())
    hdl = symm_mem.rendezvous(buf, group or dist.group.WORLD)
    views = [buf if r == hdl.rank else hdl.get_buffer(r, (rows, nbytes), torch.uint8) for r in range(lay.world)]

    def barrier():
        hdl.barrier(channel=0)   # every rank's stores issued before it on its stream are visible

    return views, barrier
