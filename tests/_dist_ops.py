"""CPU test double of dist.CudaOps -- TEST INFRASTRUCTURE ONLY.

Implements the same operations with torch CPU fp64 tensors and the CPU oracle
(reference-convention Householder QR and Jacobi SVD), so the multi-rank
gloo tests exercise the distributed schedule of paper_2104_05782_b200/dist.py
end to end on CPU.  The product never uses this (CudaOps has no fallback).
"""
import numpy as np
import torch
import torch.distributed as dist

import oracle
from paper_2104_05782_b200.dist import cm_empty


def _np(x):
    return np.asfortranarray(x.detach().numpy())


class _NoSide:
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


class TorchCpuOps:
    def begin(self):
        pass

    def side(self, on=True):
        return _NoSide()

    def keep(self, *tensors):
        pass

    def join(self):
        pass
    def copy(self, dst, src):
        dst.copy_(src)

    def copy_upper(self, dst, src):
        dst.copy_(torch.triu(src))

    def identity(self, a):
        a.copy_(torch.eye(a.shape[0], a.shape[1], dtype=torch.float64))

    def normal_fill(self, seed, pos, g):
        r, c = g.shape
        g.copy_(torch.from_numpy(oracle.normal_stream(seed, pos, r * c).reshape(c, r).T.copy()))

    def gemm(self, alpha, ta, a, tb, b, beta, c):
        A = a.T if ta else a
        B = b.T if tb else b
        prod = alpha * (A @ B)
        if beta == 0.0:
            c.copy_(prod)
        else:
            c.copy_(beta * c + prod)

    def hqr(self, a):
        qr, tau, _ = oracle.hqr(_np(a))
        a.copy_(torch.from_numpy(qr))
        return torch.from_numpy(tau.copy())

    def form_wy(self, qr, tau, p):
        q = _np(qr)
        s = q.shape[0]
        W = np.tril(q[:, :p], -1)
        W[np.arange(p), np.arange(p)] = 1.0
        twy = oracle.form_wy_t(q[:, :p], tau.numpy())
        M = W @ twy.T
        Wt, Mt = cm_empty(s, p), cm_empty(s, p)
        Wt.copy_(torch.from_numpy(W))
        Mt.copy_(torch.from_numpy(M))
        return Wt, Mt

    def rect_diag(self, block, sigma, p):
        block.zero_()
        k = min(p, block.shape[0], block.shape[1])
        idx = torch.arange(k)
        block[idx, idx] = sigma[:k]

    def block_rows(self, small, big, big_rows, b, first, stride, count, scatter):
        for t in range(count):
            r = (first + t * stride) * b
            w = min(b, big_rows - r)
            if w <= 0:
                continue
            if scatter:
                big[r:r + w, :] = small[t * b:t * b + w, :]
            else:
                small[t * b:t * b + w, :] = big[r:r + w, :]

    def svd_batch(self, mats):
        out = []
        for m in mats:
            u, s, v = oracle.svd_block(_np(m))
            U, V = cm_empty(*u.shape), cm_empty(*v.shape)
            U.copy_(torch.from_numpy(u))
            V.copy_(torch.from_numpy(v))
            out.append((U, torch.from_numpy(s.copy()), V))
        return out

    def all_reduce(self, x, comm):
        y = x.T.contiguous()
        dist.all_reduce(y, group=comm.group)
        x.copy_(y.T)

    def all_gather(self, x, comm):
        outs = [torch.zeros(x.shape[1], x.shape[0], dtype=torch.float64) for _ in range(comm.size)]
        dist.all_gather(outs, x.T.contiguous(), group=comm.group)
        return [o.T for o in outs]

    def broadcast(self, x, src, comm):
        y = x.T.contiguous() if x.dim() == 2 else x.contiguous()
        dist.broadcast(y, src, group=comm.group)
        x.copy_(y.T if x.dim() == 2 else y)

    def finish(self):
        pass
