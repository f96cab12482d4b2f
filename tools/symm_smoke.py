#!/usr/bin/env python3
"""The fused cross-GPU placement path (placement.encode_distributed_p2p) on torch symmetric
memory with a one-rank NCCL group: allocation, rendezvous, peer views, device barrier and the
kernels' stores into the receive buffer.  (The multi-rank exchange needs >= 2 GPUs.)"""
import os, sys
sys.path.insert(0, os.getcwd())
import torch, torch.distributed as dist
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=os.environ.get("SYMM_PORT", "29611"), RANK="0",
                  WORLD_SIZE="1", LOCAL_RANK="0")
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
import numpy as np, oracle, synth
from paper_1312_5155_b200 import Plan
from paper_1312_5155_b200.placement import Layout, CudaOps, encode_distributed_p2p, symmetric_recv_buffers
k, m, S, B = 10, 4, 5, 65536
lay = Layout(k, m, 1)
full = synth.stripes_array(3, range(S), k, m, B)
ref = full.copy(); oracle.encode_bulk(ref, k, m, 8, 0x11D, threads=4)
store = {(s, b): (torch.from_numpy(full[s, b].copy()).cuda() if b < k else torch.zeros(B, dtype=torch.uint8, device="cuda"))
         for s in range(S) for b in lay.blocks_on(0, s)}
views, barrier = symmetric_recv_buffers(lay, S, B)
print("views", [tuple(v.shape) for v in views])
st = encode_distributed_p2p(lay, store, S, B, 0, views, barrier, CudaOps(Plan(k, m)))
torch.cuda.synchronize()
bad = sum(int(not np.array_equal(t.cpu().numpy(), ref[s, b])) for (s, b), t in store.items())
print("p2p world=1 stats", st, "bad", bad)
dist.destroy_process_group()
