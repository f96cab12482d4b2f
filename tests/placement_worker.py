#!/usr/bin/env python3
"""Cross-GPU stripe placement (NEXT-4) as an SPMD job, launched like bench.py: `--gpus N`
without an outside launcher re-executes under torch.distributed.run (bench.launch_ranks).

  python tests/placement_worker.py --gpus 2 --backend gloo            # CPU ranks (oracle ops)
  python tests/placement_worker.py --gpus 8 --backend nccl --mode p2p  # one rank per GPU

gloo: the compute steps are the oracle stand-ins (tests/placement_ops.py), the exchange is
gloo's all_to_all.  nccl: the CUDA kernels (placement.CudaOps), NCCL all_to_all (a2a) or
the fused kernel storing into peer-mapped symmetric memory (p2p).  Every rank encodes the
same stripes twice (the second call reuses the buffers) and checks each block it owns
against the oracle; rank 0 prints one JSON line.  Test infrastructure (imports oracle/).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
import oracle  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=2)
    ap.add_argument("--backend", default="gloo", choices=["gloo", "nccl"])
    ap.add_argument("--mode", default="a2a", choices=["a2a", "p2p"])
    ap.add_argument("--k", type=int, default=10)
    ap.add_argument("--m", type=int, default=4)
    ap.add_argument("--stripes", type=int, default=6)
    ap.add_argument("--block-bytes", type=int, default=4096)
    args = ap.parse_args()
    rc = bench.launch_ranks(args)
    if rc is not None:
        return rc
    from paper_1312_5155_b200.placement import CudaOps, Layout, encode_distributed, encode_distributed_p2p
    if "WORLD_SIZE" not in os.environ:  # one process, no launcher: a world of one
        os.environ.update(WORLD_SIZE="1", RANK="0", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1",
                          MASTER_PORT=str(bench.free_port()))
    world, rank = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0"))
    k, m, S, B = args.k, args.m, args.stripes, args.block_bytes
    gpu = args.backend == "nccl"
    if gpu:
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        dev = torch.device("cuda", torch.cuda.current_device())
        dist.init_process_group("nccl", device_id=dev)
        import paper_1312_5155_b200 as rsp
        ops = CudaOps(rsp.Plan(k, m, 8, 0x11D))
    else:
        dev = torch.device("cpu")
        dist.init_process_group("gloo")
        from tests.placement_ops import OracleOps
        ops = OracleOps(k, m)
    lay = Layout(k, m, world)
    full = synth.stripes_array(5, range(S), k, m, B)
    ref = full.copy()
    oracle.encode_bulk(ref, k, m, 8, 0x11D)

    def a2a(send, in_splits, out_splits):
        out = torch.empty((sum(out_splits), B), dtype=torch.uint8, device=dev)
        dist.all_to_all_single(out.view(-1), send.reshape(-1).contiguous(),
                               [x * B for x in out_splits], [x * B for x in in_splits])
        return out

    views = barrier = None
    if args.mode == "p2p":
        if not gpu:
            raise SystemExit("--mode p2p needs --backend nccl (peer-mapped symmetric memory)")
        from paper_1312_5155_b200.placement import symmetric_recv_buffers
        views, barrier = symmetric_recv_buffers(lay, S, B)
    bad, stats, secs = 0, None, []
    for rep in range(2):  # the second call reuses the exchange buffers
        store = {}
        for s in range(S):
            for b in lay.blocks_on(rank, s):
                t = torch.from_numpy(full[s, b].copy()) if b < k else torch.full((B,), 0xCD, dtype=torch.uint8)
                store[(s, b)] = t.to(dev)
        dist.barrier()
        t0 = time.perf_counter()
        if args.mode == "a2a":
            stats = encode_distributed(lay, store, S, B, rank, a2a, ops)
        else:
            stats = encode_distributed_p2p(lay, store, S, B, rank, views, barrier, ops)
        if gpu:
            torch.cuda.synchronize()
        secs.append(time.perf_counter() - t0)
        bad += sum(int(not np.array_equal(t.cpu().numpy(), ref[s, b])) for (s, b), t in store.items())
    tot = torch.tensor([float(bad), float(stats["sent_blocks"]), float(stats["received_blocks"])],
                       dtype=torch.float64, device=dev)
    dist.all_reduce(tot)
    if rank == 0:
        print(json.dumps({"world": world, "backend": args.backend, "mode": args.mode, "k": k, "m": m,
                          "stripes": S, "block_bytes": B, "mismatched_blocks": int(tot[0].item()),
                          "sent_blocks": int(tot[1].item()), "received_blocks": int(tot[2].item()),
                          "rank0_seconds": [round(x, 4) for x in secs]}), flush=True)
    dist.destroy_process_group()
    return 0 if bad == 0 else 1


if __name__ == "__main__":
    sys.exit(main())
