"""Multi-GPU blocked randUTV over a 2D block-cyclic P x Q grid --
the Python model of the schedule.

The PRODUCT multi-GPU path is the C++ driver ``csrc/dist.cu`` behind the C ABI
(``rutv_b200_factorize_dist``, ``rutv_opts.grid_p/q``; ``bench.py --gpus N``), which
restates this algorithm with the single-GPU driver's overlap (panel-first look-ahead,
sketch hoisting, Twy/M on a side stream).  This module keeps the same algorithm over
torch.distributed with a pluggable ``ops`` object, so the distributed schedule itself
is testable on the CPU with gloo (tests/test_dist_cpu.py) and, through ``CudaOps``,
with NCCL (tests/test_gpu_dist.py); ``Grid`` is also the reference the C++ layout is
checked against (tests/test_capi.py).

One process per GPU (torch.distributed, NCCL on the GPU path).  The layout is
the paper's ScaLAPACK scheme with the distribution block
equal to the step width b: block (br, bc) lives on rank (br mod P) * Q +
(bc mod Q) (proj/src/block_cyclic.cpp:26-31), local index (br div P, bc div Q)
(:33-38).  T, U and V are distributed identically; every rank stores its row
blocks and its column blocks in global order, so "rows >= r0" and "columns >=
r0" of any of them are contiguous local suffixes.  P = 1 is the 1D column
layout (``Layout``).

Per step i of randutv_blocked.cpp:122-155 (s = n - i*b); "row comm" = the Q
ranks of my process row, "column comm" = the P ranks of my process column:

  sketch   G (s x b) is replicated -- the counter RNG (rng.hpp:9-17) lets every
           rank draw it with no communication.  Y = T22' G: local T22_loc' G[my
           rows] -> all-reduce over the column comm (Y rows = T22 columns).  Each
           power iteration: Z = T22 Y -> all-reduce over the row comm, then
           Y = T22' Z -> all-reduce over the column comm.
  QR(Y)    all-gather the Y slices over the row comm (s x b), factor
           redundantly on every rank (deterministic kernels: identical W_v,
           Twy_v everywhere, no broadcast).
  V-apply  [V; T](:, r0:) Q_v: Zx = X_loc W_v[my cols] -> all-reduce over the
           row comm, then the rank-b update X_loc -= Zx M_v[my cols]' is local.
  U-QR     the panel T22(:, 0:b) is block column i: its process column
           all-gathers it, the owner of the diagonal block (i, i) factors it and
           broadcasts the packed panel + tau (s x b); every rank forms W_u, M_u.
  Qu'      T22(:, b:) <- Q_u' T22(:, b:): Zl = W_u[my rows]' B_loc ->
           all-reduce over the column comm, local update.
  U-apply  like the V-apply (all-reduce over the row comm).
  beta     deferred exactly as the single-GPU driver (randutv.cu): each
           diagonal owner SVDs its R_i; [Us_i | Vs_i | sigma_i] are all-gathered
           once; diagonal writes, row strips (Us' from the left, process row of
           block i) and right-multiplies (Vs / Us, process column of block i)
           are then local.

Data-path collectives per step: 2q + 4 all-reduces of O((n + s) b / P or Q)
words, one all-gather of Y, one panel all-gather + broadcast; the s^2 b and
n s b flops stay local.

The compute is abstracted behind an ``ops`` object: ``CudaOps`` (this module)
runs our sm_100a kernels through the asynchronous C ABI on the caller's stream;
the CPU gloo tests plug a test double in to validate the distributed schedule
itself.  There is no CPU fallback in the product: CudaOps raises without the
library or a GPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import torch
import torch.distributed as dist


@dataclass
class Axis:
    """Block-cyclic distribution of n indices in blocks of b over p processes; my coordinate c."""
    n: int
    b: int
    p: int
    c: int

    @property
    def nblk(self) -> int:
        return (self.n + self.b - 1) // self.b

    def width(self, k: int) -> int:
        return min(self.b, self.n - k * self.b)

    def owned(self, c: int | None = None) -> list[int]:
        c = self.c if c is None else c
        return list(range(c, self.nblk, self.p))

    def loc(self, k: int) -> int:
        """Local offset of block k on its owner (blocks k mod p, k mod p + p, ... before it)."""
        return sum(self.width(j) for j in range(k % self.p, k, self.p))

    def length(self, c: int | None = None) -> int:
        return sum(self.width(k) for k in self.owned(c))

    def first_from(self, i: int, c: int | None = None) -> int | None:
        c = self.c if c is None else c
        k = i + ((c - i) % self.p)
        return k if k < self.nblk else None

    def suffix(self, i: int, c: int | None = None) -> tuple[int, int]:
        """(local offset, block count) of the owned blocks >= i."""
        k = self.first_from(i, c)
        if k is None:
            return self.length(c), 0
        return self.loc(k), (self.nblk - 1 - k) // self.p + 1


class Grid:
    """2D block-cyclic P x Q layout of an n x n matrix in b x b blocks (block_cyclic.cpp:26-38)."""

    def __init__(self, n: int, b: int, P: int, Q: int, rank: int):
        if P < 1 or Q < 1 or not 0 <= rank < P * Q:
            raise ValueError(f"bad process grid {P}x{Q} for rank {rank}")
        self.n, self.b, self.P, self.Q, self.rank = n, b, P, Q, rank
        self.pr, self.pc = divmod(rank, Q)
        self.rows = Axis(n, b, P, self.pr)
        self.cols = Axis(n, b, Q, self.pc)

    @property
    def nblk(self) -> int:
        return self.rows.nblk

    @property
    def world(self) -> int:
        return self.P * self.Q

    def width(self, k: int) -> int:
        return self.rows.width(k)

    def owner2(self, br: int, bc: int) -> int:
        return (br % self.P) * self.Q + (bc % self.Q)

    def local_shape(self, rank: int | None = None) -> tuple[int, int]:
        r = self.rank if rank is None else rank
        pr, pc = divmod(r, self.Q)
        return self.rows.length(pr), self.cols.length(pc)

    def row_ranks(self, pr: int | None = None) -> list[int]:
        pr = self.pr if pr is None else pr
        return [pr * self.Q + c for c in range(self.Q)]

    def col_ranks(self, pc: int | None = None) -> list[int]:
        pc = self.pc if pc is None else pc
        return [r * self.Q + pc for r in range(self.P)]


class Layout(Grid):
    """1D block-cyclic column layout (the P = 1 row of the grid): block column k on rank k mod world."""

    def __init__(self, n: int, b: int, world: int, rank: int):
        super().__init__(n, b, 1, world, rank)

    def owner(self, k: int) -> int:
        return k % self.Q

    def owned(self, rank: int | None = None) -> list[int]:
        return self.cols.owned(rank)

    def loc_off(self, k: int) -> int:
        return self.cols.loc(k)

    def ncols(self, rank: int | None = None) -> int:
        return self.cols.length(rank)

    def first_owned_from(self, i: int, rank: int | None = None) -> int | None:
        return self.cols.first_from(i, rank)

    def suffix(self, i: int, rank: int | None = None) -> tuple[int, int]:
        return self.cols.suffix(i, rank)


def grid_shape(world: int) -> tuple[int, int]:
    """Default process grid: P x Q with P <= Q, as square as possible (1x1, 1x2, 2x2, 2x4, ...)."""
    p = int(world ** 0.5)
    while world % p:
        p -= 1
    return p, world // p


@dataclass
class Comm:
    """A sub-communicator: global ranks in group order; ``group`` None means the default (world)."""
    ranks: list[int]
    group: object = None

    @property
    def size(self) -> int:
        return len(self.ranks)


@dataclass
class Comms:
    row: Comm
    col: Comm
    world: Comm
    row_side: Comm | None = None  # a second row communicator for the off-critical stream
    _all: list = field(default_factory=list)


def make_comms(grid: Grid) -> Comms:
    """Row and column communicators of the grid.  Every rank creates every group
    in the same order (a torch.distributed requirement); singleton groups are
    not created (their collectives are no-ops)."""
    W = grid.world
    world = Comm(list(range(W)), None)

    def mk(ranks):
        if len(ranks) == W:
            return Comm(ranks, None)
        if len(ranks) == 1:
            return Comm(ranks, None)
        return Comm(ranks, dist.new_group(ranks))

    def mk_side(ranks):  # always a separate group: its own NCCL stream, no coupling to the critical one
        return Comm(ranks, dist.new_group(ranks)) if len(ranks) > 1 else Comm(ranks, None)

    rows = [mk(grid.row_ranks(pr)) for pr in range(grid.P)]
    cols = [mk(grid.col_ranks(pc)) for pc in range(grid.Q)]
    sides = [mk_side(grid.row_ranks(pr)) for pr in range(grid.P)]
    return Comms(rows[grid.pr], cols[grid.pc], world, sides[grid.pr], rows + cols + sides)


def cm_empty(rows: int, cols: int, like: torch.Tensor | None = None, device=None) -> torch.Tensor:
    """Zero column-major fp64 matrix (a transposed contiguous tensor, stride (1, rows))."""
    dev = like.device if like is not None else device
    return torch.zeros((max(cols, 0), max(rows, 0)), dtype=torch.float64, device=dev).T


def _gather_blocks(ops, comm: Comm, axis: Axis, coord_of, loc: torch.Tensor, i: int, s: int, b: int,
                   like: torch.Tensor) -> torch.Tensor:
    """All-gather over ``comm`` the row slabs ``loc`` (my blocks >= i of ``axis``) and
    assemble the full s x b matrix in global block order."""
    maxcnt = (axis.nblk - 1 - i) // axis.p + 1
    slab = cm_empty(maxcnt * b, b, like=like)
    if loc.shape[0]:
        ops.copy(slab[:loc.shape[0], :], loc)
    parts = ops.all_gather(slab, comm) if comm.size > 1 else [slab]
    full = cm_empty(s, b, like=like)
    for rk, part in zip(comm.ranks, parts):
        c = coord_of(rk)
        k0 = axis.first_from(i, c)
        if k0 is None:
            continue
        cnt = (axis.nblk - 1 - k0) // axis.p + 1
        ops.block_rows(part[:cnt * b, :], full, s, b, k0 - i, axis.p, cnt, scatter=True)
    return full


def _pick_rows(ops, full: torch.Tensor, axis: Axis, i: int, s: int, b: int) -> torch.Tensor:
    """My blocks >= i (of ``axis``) of an s x w matrix indexed from block i."""
    off, cnt = axis.suffix(i)
    k0 = axis.first_from(i)
    m = axis.length() - off
    out = cm_empty(m, full.shape[1], like=full)
    if cnt:
        ops.block_rows(out, full, s, b, k0 - i, axis.p, cnt, scatter=False)
    return out


def _all_reduce(ops, x: torch.Tensor, comm: Comm) -> None:
    if comm.size > 1:
        ops.all_reduce(x, comm)


def factorize_dist(a_loc: torch.Tensor, grid: Grid, *, q: int, seed: int, ops, build_uv: bool = True,
                   g: torch.Tensor | None = None, comms: Comms | None = None):
    """Distributed randUTV (randutv_blocked.cpp:84-157) over the P x Q grid.
    ``a_loc``: this rank's blocks of A (local rows x local columns, column-major).
    ``g``: optional explicit Gaussian stream (the reference's per-step G blocks in
    stream order, rng.cpp:38-53); otherwise drawn from ``seed`` on the device.
    Returns this rank's blocks (T_loc, U_loc, V_loc)."""
    n, b, P, Q, me = grid.n, grid.b, grid.P, grid.Q, grid.rank
    if b < 1 or q < 0:
        raise ValueError("block size must be >= 1 and q >= 0")
    if comms is None:
        comms = make_comms(grid)
    if comms.row_side is None:
        comms.row_side = comms.row
    ops.begin()
    RA, CA = grid.rows, grid.cols
    mr, mc = grid.local_shape()
    if tuple(a_loc.shape) != (mr, mc):
        raise ValueError(f"a_loc is {tuple(a_loc.shape)}, rank {me} of the {P}x{Q} grid holds {(mr, mc)}")
    vr = mr if build_uv else 0
    VT = cm_empty(vr + mr, mc, like=a_loc)   # V on top of T, as the single-GPU driver
    U = cm_empty(mr, mc, like=a_loc) if build_uv else None
    T = VT[vr:, :]
    ops.copy(T, a_loc)
    nblk = grid.nblk
    if build_uv:  # V, U := I on my diagonal blocks (:114-120)
        for k in range(grid.pr, nblk, P):
            if k % Q == grid.pc:
                w, ro, co = grid.width(k), RA.loc(k), CA.loc(k)
                ops.identity(VT[ro:ro + w, co:co + w])
                ops.identity(U[ro:ro + w, co:co + w])
    pr_of = lambda r: r // Q  # noqa: E731
    pc_of = lambda r: r % Q   # noqa: E731
    pos = 0
    saved = {}   # diagonal block -> (R, w) kept by its owner for the deferred beta stage
    steps = 0
    for i in range(nblk):
        r0, s = i * b, n - i * b
        ri, _ = RA.suffix(i)
        ci, _ = CA.suffix(i)
        T22 = T[ri:, ci:]
        m_r, m_c = T22.shape
        downer = grid.owner2(i, i)
        steps = i + 1
        if s <= b:   # ragged tail: dense s x s block (:129-137), entirely on the diagonal owner
            if me == downer:
                R = cm_empty(s, s, like=a_loc)
                ops.copy(R, T22[:s, :s])
                saved[i] = (R, s)
            break
        # ---- sketch (build_v_alpha, :41-50): G replicated, reductions over row / column comms
        G = cm_empty(s, b, like=a_loc)
        if g is not None:
            ops.copy(G, g[pos:pos + s * b].reshape(b, s).T)
        else:
            ops.normal_fill(seed, pos, G)
        pos += s * b
        G_loc = _pick_rows(ops, G, RA, i, s, b)
        Y_loc = cm_empty(m_c, b, like=a_loc)
        if m_c and m_r:
            ops.gemm(1.0, 1, T22, 0, G_loc, 0.0, Y_loc)
        if m_c:
            _all_reduce(ops, Y_loc, comms.col)
        for _ in range(q):
            Z_loc = cm_empty(m_r, b, like=a_loc)
            if m_r and m_c:
                ops.gemm(1.0, 0, T22, 0, Y_loc, 0.0, Z_loc)
            if m_r:
                _all_reduce(ops, Z_loc, comms.row)
            if m_c:
                Y_loc = cm_empty(m_c, b, like=a_loc)
                if m_r:
                    ops.gemm(1.0, 1, T22, 0, Z_loc, 0.0, Y_loc)
                _all_reduce(ops, Y_loc, comms.col)
        # ---- QR(Y) redundantly on every rank (:52-53)
        Y = _gather_blocks(ops, comms.row, CA, pc_of, Y_loc, i, s, b, a_loc)
        tau_v = ops.hqr(Y)
        Wv, Mv = ops.form_wy(Y, tau_v, b)
        # ---- V-apply on [V; T](:, r0:) (:140-143): Zx = X_loc W_v[my cols] over the row comm.
        # The rows of T22 are the critical chain; V and the finished rows of T
        # (rows [0, vr + ri)) go to the side stream with their own row communicator.
        Wl = Ml = None
        if m_c:
            Wl, Ml = _pick_rows(ops, Wv, CA, i, s, b), _pick_rows(ops, Mv, CA, i, s, b)
        for crit in (True, False):
            X = VT[vr + ri:, ci:] if crit else VT[:vr + ri, ci:]
            if X.shape[0] == 0:
                continue
            with ops.side(not crit):
                if m_c:
                    ops.keep(Wl, Ml)
                Zx = cm_empty(X.shape[0], b, like=a_loc)
                if m_c:
                    ops.gemm(1.0, 0, X, 0, Wl, 0.0, Zx)
                _all_reduce(ops, Zx, comms.row if crit else comms.row_side)
                if m_c:
                    ops.gemm(-1.0, 0, Zx, 1, Ml, 1.0, X)
        # ---- U-side panel QR (build_u_alpha, :58-64): block column i gathered in its
        #      process column, factored by the diagonal owner, broadcast to all
        pan_pc = i % Q
        if grid.pc == pan_pc:
            pan = _gather_blocks(ops, comms.col, RA, pr_of, T22[:, :b], i, s, b, a_loc)
        else:
            pan = cm_empty(s, b, like=a_loc)
        tau_u = torch.zeros(b, dtype=torch.float64, device=a_loc.device)
        if me == downer:
            tau_u = ops.hqr(pan)
            R = cm_empty(b, b, like=a_loc)
            ops.copy_upper(R, pan[:b, :])      # beta_stage's R (:73-75)
            saved[i] = (R, b)
        if grid.world > 1:
            ops.broadcast(pan, downer, comms.world)
            ops.broadcast(tau_u, downer, comms.world)
        Wu, Mu = ops.form_wy(pan, tau_u, b)
        # ---- Q_u' on T22(:, b:) (:147): Zl = W_u[my rows]' B_loc over the column comm
        Bc = T22[:, b:] if grid.pc == pan_pc else T22
        if Bc.shape[1]:
            Zl = cm_empty(b, Bc.shape[1], like=a_loc)
            Wr, Mr = _pick_rows(ops, Wu, RA, i, s, b), _pick_rows(ops, Mu, RA, i, s, b)
            if m_r:
                ops.gemm(1.0, 1, Wr, 0, Bc, 0.0, Zl)
            _all_reduce(ops, Zl, comms.col)
            if m_r:
                ops.gemm(-1.0, 0, Mr, 0, Zl, 1.0, Bc)
        # ---- U accumulate (:148): like the V-apply, off the critical chain
        if build_uv and mr:
            Xu = U[:, ci:]
            if m_c:
                Wl, Ml = _pick_rows(ops, Wu, CA, i, s, b), _pick_rows(ops, Mu, CA, i, s, b)
            with ops.side(True):
                if m_c:
                    ops.keep(Wl, Ml)
                Zu = cm_empty(mr, b, like=a_loc)
                if m_c:
                    ops.gemm(1.0, 0, Xu, 0, Wl, 0.0, Zu)
                _all_reduce(ops, Zu, comms.row_side)
                if m_c:
                    ops.gemm(-1.0, 0, Zu, 1, Ml, 1.0, Xu)

    # ======== deferred beta stage (:66-82, :129-137, :150-154) ========
    ops.join()
    mine = sorted(saved)
    res = ops.svd_batch([saved[k][0] for k in mine])     # [(Us, sigma, Vs)]
    fac = {k: r for k, r in zip(mine, res)}
    # [Us | Vs | sigma] of every step on every rank: one all-gather of fixed slots
    diag = {r: [k for k in range(steps) if grid.owner2(k, k) == r] for r in range(grid.world)}
    slots = max(len(v) for v in diag.values()) if steps else 0
    width = 2 * b + 1
    allfac = {}
    if slots:
        mybuf = cm_empty(b, slots * width, like=a_loc)
        for t, k in enumerate(mine):
            Us, sig, Vs = fac[k]
            w = saved[k][1]
            c0 = t * width
            ops.copy(mybuf[:w, c0:c0 + w], Us)
            ops.copy(mybuf[:w, c0 + b:c0 + b + w], Vs)
            ops.copy(mybuf[:w, c0 + 2 * b:c0 + 2 * b + 1], sig[:w].reshape(w, 1))
        bufs = ops.all_gather(mybuf, comms.world) if grid.world > 1 else [mybuf]
        for r, buf in enumerate(bufs):
            for t, k in enumerate(diag[r]):
                w = grid.width(k)
                c0 = t * width
                allfac[k] = (buf[:w, c0:c0 + w], buf[:w, c0 + 2 * b], buf[:w, c0 + b:c0 + b + w])
    for k in range(steps):  # diagonal writes: rows >= r0 of block column k (finished panel)
        if k % Q != grid.pc:
            continue
        ro, _ = RA.suffix(k)
        w, co = grid.width(k), CA.loc(k)
        blk = T[ro:, co:co + w]
        if blk.shape[0] == 0:
            continue
        Us, sig, Vs = allfac[k]
        ops.rect_diag(blk, sig, w if grid.owner2(k, k) == me else 0)
    for k in range(steps):  # strips T(r0:r0+b, r0+b:) <- Us_k' (...): row block k, my columns > k
        if n - k * b <= b or k % P != grid.pr:
            continue
        c_k, _ = CA.suffix(k + 1)
        if c_k >= mc:
            continue
        Us = allfac[k][0]
        ro = RA.loc(k)
        strip = T[ro:ro + b, c_k:]
        tmp = cm_empty(b, strip.shape[1], like=a_loc)
        ops.gemm(1.0, 1, Us, 0, strip, 0.0, tmp)
        ops.copy(strip, tmp)
    for k in range(steps):  # right-multiplies of block column k: [V; T(0:r0)] Vs, U Us
        if k % Q != grid.pc:
            continue
        Us, sig, Vs = allfac[k]
        w, co = grid.width(k), CA.loc(k)
        rows_above = vr + RA.suffix(k)[0]
        if rows_above:
            Xb = VT[:rows_above, co:co + w]
            tmp = cm_empty(rows_above, w, like=a_loc)
            ops.gemm(1.0, 0, Xb, 0, Vs, 0.0, tmp)
            ops.copy(Xb, tmp)
        if build_uv and mr:
            Xb = U[:, co:co + w]
            tmp = cm_empty(mr, w, like=a_loc)
            ops.gemm(1.0, 0, Xb, 0, Us, 0.0, tmp)
            ops.copy(Xb, tmp)
    ops.finish()
    return T, U, (VT[:mr, :] if build_uv else None)


def scatter_grid(a: torch.Tensor, grid: Grid) -> torch.Tensor:
    """This rank's blocks of a full column-major matrix (host or device)."""
    b = grid.b
    rows = [a[k * b:k * b + grid.width(k), :] for k in grid.rows.owned()]
    mr, mc = grid.local_shape()
    out = cm_empty(mr, mc, like=a)
    if rows and mc:
        rsel = torch.cat(rows, dim=0)
        cols = [rsel[:, k * b:k * b + grid.width(k)] for k in grid.cols.owned()]
        out.copy_(torch.cat(cols, dim=1))
    return out


def gather_grid(x_loc: torch.Tensor, grid: Grid) -> torch.Tensor:
    """Reassemble the full n x n matrix on every rank from the grid blocks (test / bench helper)."""
    b, n = grid.b, grid.n
    shapes = [grid.local_shape(r) for r in range(grid.world)]
    maxr, maxc = max(s[0] for s in shapes), max(s[1] for s in shapes)
    buf = cm_empty(maxr, maxc, like=x_loc)
    buf[:x_loc.shape[0], :x_loc.shape[1]].copy_(x_loc)
    bufs = [cm_empty(maxr, maxc, like=x_loc) for _ in range(grid.world)]
    if grid.world > 1:
        dist.all_gather([t.T for t in bufs], buf.T.contiguous())
    else:
        bufs[0].copy_(buf)
    full = cm_empty(n, n, like=x_loc)
    for r in range(grid.world):
        pr, pc = divmod(r, grid.Q)
        for kr in grid.rows.owned(pr):
            ro, wr = grid.rows.loc(kr), grid.width(kr)
            for kc in grid.cols.owned(pc):
                co, wc = grid.cols.loc(kc), grid.width(kc)
                full[kr * b:kr * b + wr, kc * b:kc * b + wc].copy_(bufs[r][ro:ro + wr, co:co + wc])
    return full


# 1D names kept for callers of the column layout
scatter_columns = scatter_grid


def gather_columns(x_loc: torch.Tensor, lay: Grid, rows: int | None = None) -> torch.Tensor:
    return gather_grid(x_loc, lay)


# --------------------------------------------------------------------------- GPU ops
class CudaOps:
    """Our sm_100a kernels through the asynchronous C ABI, on torch's current stream;
    NCCL collectives through torch.distributed on the same stream."""

    def __init__(self, device: torch.device):
        from . import lib
        self.L = lib()
        self.dev = device
        self.caller = torch.cuda.current_stream(device)
        # critical chain on a high-priority stream, V/U accumulation on a
        # low-priority one (the single-GPU driver's schedule, randutv.cu)
        self.sA = torch.cuda.Stream(device, priority=-1)
        self.sB = torch.cuda.Stream(device, priority=0)
        self.stream = self.caller
        self._set(self.caller)
        self.status: list[torch.Tensor] = []

    def _set(self, st):
        self.stream = st
        torch.cuda.set_stream(st)
        self.L.rutv_b200_set_stream(C.c_uint64(st.cuda_stream))

    # stream schedule
    def begin(self):
        self.caller = torch.cuda.current_stream(self.dev)
        self.sA.wait_stream(self.caller)
        self._set(self.sA)

    def side(self, on: bool = True):
        ops = self

        class _Side:
            def __enter__(self_):
                if on:
                    ops.sB.wait_stream(ops.sA)
                    ops._set(ops.sB)

            def __exit__(self_, *exc):
                if on:
                    ops._set(ops.sA)
                return False
        return _Side()

    def keep(self, *tensors):
        """Tensors made on the critical stream and read on the side stream."""
        if self.stream is self.sB:
            for t in tensors:
                if t is not None:
                    t.record_stream(self.sB)

    def join(self):
        self.sA.wait_stream(self.sB)

    # helpers
    @staticmethod
    def _cm(x):
        r, c = x.shape
        ld = max(x.stride(1) if c > 1 else r, r, 1)
        return C.c_void_p(x.data_ptr()), r, c, ld

    def _chk(self, rc, st):
        from . import _raise
        _raise(st)

    def _call(self, fn, *args):
        from . import Status
        st = Status()
        fn(*args, C.byref(st))
        self._chk(0, st)

    # ops
    def copy(self, dst, src):
        if dst.numel() == 0:
            return
        pd, r, c, ldd = self._cm(dst)
        ps, _, _, lds = self._cm(src)
        self._call(self.L.rutv_b200_copy_async, pd, r, c, ldd, ps, lds)

    def copy_upper(self, dst, src):
        pd, r, c, ldd = self._cm(dst)
        ps, _, _, lds = self._cm(src)
        self._call(self.L.rutv_b200_copy_upper_async, pd, r, c, ldd, ps, lds)

    def identity(self, a):
        pa, r, c, lda = self._cm(a)
        self._call(self.L.rutv_b200_identity_async, pa, r, c, lda)

    def normal_fill(self, seed, pos, g):
        pg, r, c, ld = self._cm(g)
        self._call(self.L.rutv_b200_normal_fill_async, C.c_uint64(seed), C.c_uint64(pos), pg, r, c, ld)

    def gemm(self, alpha, ta, a, tb, b, beta, c):
        pa, ar, ac, lda = self._cm(a)
        pb, br, bc, ldb = self._cm(b)
        pc, m, n, ldc = self._cm(c)
        self._call(self.L.rutv_b200_gemm_async, C.c_double(alpha), ta, pa, ar, ac, lda, tb, pb, br, bc, ldb,
                   C.c_double(beta), pc, m, n, ldc)

    def hqr(self, a):
        pa, m, n, lda = self._cm(a)
        tau = torch.zeros(max(min(m, n), 1), dtype=torch.float64, device=self.dev)
        self._call(self.L.rutv_b200_hqr_async, pa, m, n, lda, C.c_void_p(tau.data_ptr()))
        return tau[:min(m, n)]

    def form_wy(self, qr, tau, p):
        s = qr.shape[0]
        W, M, Tw = cm_empty(s, p, like=qr), cm_empty(s, p, like=qr), cm_empty(p, p, like=qr)
        pq, _, _, ldq = self._cm(qr)
        self._call(self.L.rutv_b200_form_wy, pq, s, ldq, C.c_void_p(tau.data_ptr()), p, C.c_void_p(W.data_ptr()),
                   max(s, 1), C.c_void_p(M.data_ptr()), max(s, 1), C.c_void_p(Tw.data_ptr()), max(p, 1))
        return W, M

    def rect_diag(self, block, sigma, p):
        pb, r, c, ld = self._cm(block)
        self._call(self.L.rutv_b200_rect_diag_async, pb, r, c, ld, C.c_void_p(sigma.data_ptr()), p)

    def block_rows(self, small, big, big_rows, b, first, stride, count, scatter):
        ps, _, cols, lds = self._cm(small)
        pb, _, _, ldb = self._cm(big)
        self._call(self.L.rutv_b200_block_rows_async, ps, lds, pb, ldb, big_rows, cols, b, first, stride, count,
                   1 if scatter else 0)

    def svd_batch(self, mats):
        if not mats:
            return []
        k = len(mats)
        outs = [(cm_empty(m.shape[0], m.shape[0], like=m), torch.zeros(m.shape[0], dtype=torch.float64,
                                                                            device=self.dev),
                 cm_empty(m.shape[0], m.shape[0], like=m)) for m in mats]
        status = torch.zeros(4 * k, dtype=torch.float64, device=self.dev)
        arr = lambda vals, t: (t * k)(*vals)  # noqa: E731
        P = C.c_void_p
        self._call(self.L.rutv_b200_svd_batch_async, k, arr([m.shape[0] for m in mats], C.c_int64),
                   arr([m.data_ptr() for m in mats], P), arr([max(m.stride(1), m.shape[0], 1) for m in mats], C.c_int64),
                   arr([o[0].data_ptr() for o in outs], P), arr([o[1].data_ptr() for o in outs], P),
                   arr([o[2].data_ptr() for o in outs], P), P(status.data_ptr()))
        self.status.append(status)
        return outs

    # NCCL collectives on the caller's stream.  Column-major views are passed as
    # their row-major transposes; a non-contiguous slice is staged through a copy.
    def all_reduce(self, x, comm):
        t = x.T if x.dim() == 2 else x
        if t.is_contiguous():
            dist.all_reduce(t, group=comm.group)
        else:
            y = t.contiguous()
            dist.all_reduce(y, group=comm.group)
            t.copy_(y)

    def all_gather(self, x, comm):
        outs = [cm_empty(*x.shape, like=x) for _ in range(comm.size)]
        dist.all_gather([o.T for o in outs], x.T.contiguous(), group=comm.group)
        return outs

    def broadcast(self, x, src, comm):
        t = x.T if x.dim() == 2 else x
        if t.is_contiguous():
            dist.broadcast(t, src, group=comm.group)
        else:
            y = t.contiguous()
            dist.broadcast(y, src, group=comm.group)
            t.copy_(y)

    def finish(self):
        from . import ConvergenceError
        self.join()
        self.caller.wait_stream(self.sA)
        self._set(self.caller)
        torch.cuda.synchronize(self.dev)
        for st in self.status:
            h = st.cpu().view(-1, 4)
            bad = (h[:, 0] == 4).nonzero()
            if len(bad):
                raise ConvergenceError(4, "jacobi sweeps exhausted after 30 sweeps", float(h[bad[0, 0], 1]))
        self.status.clear()
