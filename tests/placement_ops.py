"""CPU stand-ins for the placement protocol's compute steps (test infrastructure: the oracle
does the GF arithmetic; the product path uses the CUDA kernels through placement.CudaOps)."""
import numpy as np
import torch

import oracle

P8 = 0x11D


class OracleOps:
    """partial = oracle encoding of the stripe with only blocks idx non-zero; XOR in numpy."""

    def __init__(self, k, m):
        self.k, self.m = k, m

    def encode_partial(self, idx, data, partial, nbytes):
        for drow, prow in zip(data, partial):
            st = np.zeros((1, self.k + self.m, nbytes), dtype=np.uint8)
            for j, d in zip(idx, drow):
                st[0, j] = d.numpy()
            oracle.encode_bulk(st, self.k, self.m, 8, P8)
            for i in range(self.m):
                prow[i].copy_(torch.from_numpy(st[0, self.k + i].copy()))

    def xor_reduce(self, dst, srcs, nbytes):
        for d, row in zip(dst, srcs):
            acc = np.zeros(nbytes, dtype=np.uint8)
            for x in row:
                acc ^= x.numpy()
            d.copy_(torch.from_numpy(acc))

    def empty(self, nblocks, nbytes, like):
        return torch.empty((nblocks, nbytes), dtype=torch.uint8)
