"""x-slab domain decomposition of the structured K.v and PCG across GPUs.

SURVEY 8e.  Rank r of P owns element layers ex in [x0_r, x1_r) and node planes
i in [x0_r, x1_r]; the plane i = x1_r is replicated on ranks r and r+1.  Each
rank stores its slab as an ordinary structured grid with LOCAL x-fastest
numbering, so the single-GPU kernels run unchanged on it.  One matvec is

    local kernel (masked input, no pass-through)
      -> exchange the two interface node planes' partial sums with the
         neighbours (torch.distributed P2P: NCCL over NVLink on B200, gloo on
         CPU in the tests)
      -> add them in a fixed order (left partial first, then right partial),
         so both replicas of an interface DOF hold bitwise-identical values
      -> fixed-DOF pass-through (after the exchange: a constrained DOF on an
         interface must not be counted twice).

CG dot products use owner-computes masks (the replicated plane is counted by
the lower rank) and one all-reduce per reduction point (FP64 partials).  On
the GPU the CG scalars live in device memory (`slab_pcg_device`,
csrc/tf_slab.cu): the host only enqueues and polls.

Transports: "p2p" (torch.distributed P2P + all-reduce: NCCL on GPUs) or
"peer" (peer.py: CUDA-IPC peer memory with stream-ordered flags; with it the
whole CG loop runs from the native runtime csrc/tf_slab_run.cu, in CUDA-graph
blocks of 10 iterations).

The local compute is pluggable (`local_apply`, `local_diag_partial`): the
product binds the sm_100a kernels; tests/test_slab.py binds the CPU oracle and
runs world_size 2 with gloo to cover the decomposition logic without a GPU.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .mesh import BoundaryConditions, StructuredMesh


@dataclass(frozen=True)
class SlabPartition:
    """Element layers [x0, x1) of a global mesh on rank `rank` of `world`."""

    mesh: StructuredMesh
    world: int
    rank: int

    def __post_init__(self):
        if not (0 <= self.rank < self.world):
            raise ValueError("rank out of range")
        if self.mesh.nelx < self.world:
            raise ValueError("fewer element layers than ranks")

    @staticmethod
    def bounds(nelx: int, world: int, rank: int) -> tuple[int, int]:
        return (rank * nelx) // world, ((rank + 1) * nelx) // world

    @property
    def x0(self) -> int:
        return self.bounds(self.mesh.nelx, self.world, self.rank)[0]

    @property
    def x1(self) -> int:
        return self.bounds(self.mesh.nelx, self.world, self.rank)[1]

    @property
    def local_mesh(self) -> StructuredMesh:
        return StructuredMesh(self.x1 - self.x0, self.mesh.nely, self.mesh.nelz)

    @property
    def has_left(self) -> bool:
        return self.rank > 0

    @property
    def has_right(self) -> bool:
        return self.rank < self.world - 1

    # -- index maps -------------------------------------------------------------
    def local_node_to_global(self) -> np.ndarray:
        lm = self.local_mesh
        g = self.mesh
        ids = np.arange(lm.n_nodes, dtype=np.int64)
        nx1 = lm.nelx + 1
        i = ids % nx1
        rest = ids // nx1
        j = rest % (lm.nely + 1)
        k = rest // (lm.nely + 1)
        return g.node_id(i + self.x0, j, k)

    def local_dof_to_global(self) -> np.ndarray:
        n = self.local_node_to_global()
        return (3 * n[:, None] + np.arange(3)).ravel()

    def local_elem_to_global(self) -> np.ndarray:
        lm = self.local_mesh
        e = np.arange(lm.n_elem, dtype=np.int64)
        ex = e % lm.nelx + self.x0
        ey = (e // lm.nelx) % lm.nely
        ez = e // (lm.nelx * lm.nely)
        return self.mesh.element_id(ex, ey, ez)

    def plane_dofs(self, i_local: int) -> np.ndarray:
        """Local DOF ids of node plane x = i_local, (j, k) row-major, 3 comps."""
        lm = self.local_mesh
        jj, kk = np.meshgrid(np.arange(lm.nely + 1), np.arange(lm.nelz + 1), indexing="xy")
        nodes = (i_local + (lm.nelx + 1) * (jj.ravel() + (lm.nely + 1) * kk.ravel())).astype(np.int64)
        return (3 * nodes[:, None] + np.arange(3)).ravel()

    def owned_dof_mask(self) -> np.ndarray:
        """True on DOFs this rank counts in global reductions (left plane
        belongs to the lower rank)."""
        m = np.ones(self.local_mesh.n_dof, dtype=bool)
        if self.has_left:
            m[self.plane_dofs(0)] = False
        return m

    def local_bcs(self, bcs: BoundaryConditions) -> BoundaryConditions:
        g2l = self.local_dof_to_global()
        is_fixed = np.zeros(self.mesh.n_dof, dtype=bool)
        is_fixed[bcs.fixed_dofs] = True
        fixed_local = np.flatnonzero(is_fixed[g2l])
        force = np.asarray(bcs.force)[g2l].copy()
        return BoundaryConditions(fixed_local, force)

    def scatter(self, global_vec: np.ndarray) -> np.ndarray:
        return np.asarray(global_vec)[self.local_dof_to_global()]

    def scatter_elem(self, global_elem_vec: np.ndarray) -> np.ndarray:
        return np.asarray(global_elem_vec)[self.local_elem_to_global()]


class SlabExchange:
    """Interface-plane partial-sum exchange with the x-neighbours.

    Works on torch tensors with any torch.distributed backend (NCCL on GPU,
    gloo on CPU).  The sum order at an interface is always
    (left rank's partial) + (right rank's partial).
    """

    def __init__(self, part: SlabPartition, device, group=None):
        import torch

        self.part = part
        self.group = group
        lm = part.local_mesh
        self.left_idx = torch.as_tensor(part.plane_dofs(0), device=device)
        self.right_idx = torch.as_tensor(part.plane_dofs(lm.nelx), device=device)

    def __call__(self, w):
        return self.finish(w, self.start(w))

    def start(self, w):
        """Post the interface-plane exchange (needs only the interface columns
        of w to be final); returns the state finish() completes."""
        import torch
        import torch.distributed as dist

        p = self.part
        # gloo moves host tensors only: stage device planes through the host
        # (used by the single-GPU multi-rank tests); NCCL exchanges in place
        host = (p.has_left or p.has_right) and w.is_cuda and dist.get_backend(self.group) == "gloo"
        ops = []
        send_l = recv_l = send_r = recv_r = None
        if p.has_left:
            send_l = w[self.left_idx].contiguous()
            recv_l = torch.empty_like(send_l, device="cpu" if host else w.device)
            sl = send_l.cpu() if host else send_l
            ops += [dist.P2POp(dist.isend, sl, p.rank - 1, self.group),
                    dist.P2POp(dist.irecv, recv_l, p.rank - 1, self.group)]
        if p.has_right:
            send_r = w[self.right_idx].contiguous()
            recv_r = torch.empty_like(send_r, device="cpu" if host else w.device)
            sr = send_r.cpu() if host else send_r
            ops += [dist.P2POp(dist.isend, sr, p.rank + 1, self.group),
                    dist.P2POp(dist.irecv, recv_r, p.rank + 1, self.group)]
        works = dist.batch_isend_irecv(ops) if ops else []
        return works, send_l, recv_l, send_r, recv_r

    def finish(self, w, state):
        works, send_l, recv_l, send_r, recv_r = state
        for r in works:
            r.wait()
        if recv_l is not None:  # my left plane: left partial first
            w[self.left_idx] = recv_l.to(w.device) + send_l
        if recv_r is not None:  # my right plane: my (left) partial first
            w[self.right_idx] = send_r + recv_r.to(w.device)
        return w


class SlabOperator:
    """Distributed K(rho) on one rank's slab.

    local_apply(x) must return the slab's own element contributions with the
    input masked on constrained DOFs and NO pass-through; the exchange and the
    pass-through are added here.
    """

    def __init__(self, part: SlabPartition, bcs_local: BoundaryConditions, local_apply,
                 local_diag_partial, device, dtype, group=None, transport: str | None = None):
        import os

        import torch

        self.part = part
        self.local_apply = local_apply
        self.local_diag_partial = local_diag_partial
        # "p2p": torch.distributed P2P + all_reduce (NCCL on GPUs, gloo with
        # host staging in the one-GPU tests); "peer": peer-memory puts and
        # stream-ordered flags (peer.py / csrc/tf_peer.cu)
        self.transport = transport or os.environ.get("TF_SLAB_TRANSPORT", "p2p")
        if self.transport == "peer":
            from .peer import PeerTransport

            self.exchange = PeerTransport(part, device, group)
        elif self.transport == "p2p":
            self.exchange = SlabExchange(part, device, group)
        else:
            raise ValueError(f"unknown slab transport {self.transport!r}")
        self.group = group
        self.device = device
        self.dtype = dtype
        self.fixed = torch.as_tensor(bcs_local.fixed_dofs, device=device, dtype=torch.int64)
        self.owned = torch.as_tensor(part.owned_dof_mask(), device=device)
        self.n_apply = 0

    def apply(self, x):
        nat = self.native()
        if nat is not None:  # the whole distributed product enqueued from C++
            self.n_apply += 1
            return nat.apply(x)
        split = getattr(self.local_apply, "split", None)
        if split is not None:
            # interface columns first, exchange in flight while the interior runs
            w = split(x, None, "boundary")
            state = self.exchange.start(w)
            split(x, w, "interior")
            w = self.exchange.finish(w, state)
        else:
            w = self.local_apply(x)
            w = self.exchange(w)
        if self.fixed.numel():
            w[self.fixed] = x[self.fixed]
        self.n_apply += 1
        return w

    def diagonal(self):
        """Jacobi diagonal: FP64 partial sums exchanged, cast, 1.0 on fixed."""
        d64 = self.exchange(self.local_diag_partial())
        d = d64.to(self.dtype)
        if self.fixed.numel():
            d[self.fixed] = 1.0
        return d

    def native(self):
        """The native slab runtime over the peer transport (tf_slab_run.cu),
        or None (other transports, or local compute that is not the tile
        kernels)."""
        import os

        if (self.transport != "peer" or getattr(self.local_apply, "op", None) is None
                or os.environ.get("TF_SLAB_NATIVE", "1") != "1"):
            return None
        if getattr(self, "_native", None) is None:
            self._native = NativeSlab(self)
        return self._native

    def allreduce_dev(self, t, lo: int, hi: int):
        """In place, no host round trip on NCCL/peer: t[lo:hi] (FP64 device
        tensor) summed over ranks; every rank gets the same values."""
        import torch.distributed as dist

        if not (dist.is_initialized() and dist.get_world_size(self.group) > 1):
            return t
        if self.transport == "peer":
            return self.exchange.allreduce_(t, lo, hi)
        if t.is_cuda and dist.get_backend(self.group) == "gloo":
            h = t[lo:hi].cpu()
            dist.all_reduce(h, group=self.group)
            t[lo:hi].copy_(h)
        else:
            dist.all_reduce(t[lo:hi], group=self.group)
        return t

    def allreduce(self, vals):
        """Sum of FP64 partials over ranks (owner-computes)."""
        import torch
        import torch.distributed as dist

        t = torch.tensor(vals, dtype=torch.float64, device=self.device)
        if dist.is_initialized() and dist.get_world_size(self.group) > 1:
            dist.all_reduce(t, group=self.group)
        return t.tolist()

    def dots(self, *pairs):
        """Global FP64 dots of (a, b) pairs over owned DOFs (one all_reduce)."""
        import torch

        vals = []
        for a, b in pairs:
            vals.append(float(torch.sum(a.double()[self.owned] * b.double()[self.owned])))
        return self.allreduce(vals)


def slab_pcg(op: SlabOperator, b, diag, rel_tol=1e-5, max_iter=1000, recompute_every=50, x0=None):
    """Distributed Jacobi-PCG, same recurrence and stop rule as solver.py:57-147.

    Vectors are the rank-local slabs (torch tensors); every scalar is a global
    FP64 all-reduced dot rounded to the working dtype like the single-GPU
    device solver, so all ranks take identical decisions.  CUDA vectors run
    the device-driven protocol (slab_pcg_device); CPU vectors (the oracle-
    bound decomposition tests) the host loop below.
    """
    import os

    import torch

    if b.is_cuda and os.environ.get("TF_SLAB_HOST_CG", "0") != "1":
        return slab_pcg_device(op, b, diag, rel_tol, max_iter, recompute_every, x0)

    f32 = b.dtype == torch.float32
    rnd = (lambda v: float(np.float32(v))) if f32 else (lambda v: float(v))
    nrm = (lambda v: float(np.sqrt(np.float32(v)))) if f32 else (lambda v: math.sqrt(v))
    bnorm = nrm(rnd(op.dots((b, b))[0]))
    if bnorm == 0.0:
        return torch.zeros_like(b), dict(iterations=0, termination="converged", rel=0.0,
                                         history=[0.0], matvecs=0)
    mv = 0
    if x0 is None:
        x = torch.zeros_like(b)
        r = b.clone()
    else:
        x = x0.clone()
        r = b - op.apply(x)
        mv += 1
    inv = 1.0 / diag
    z = r * inv
    p = z.clone()
    rr, rz = op.dots((r, r), (r, z))
    rz = rnd(rz)
    rel = nrm(rnd(rr)) / bnorm
    hist = [rel]
    term = "converged" if rel <= rel_tol else "max_iter"
    done = rel <= rel_tol
    it = 0
    while not done and it < max_iter:
        it += 1
        q = op.apply(p)
        mv += 1
        pq = rnd(op.dots((p, q))[0])
        if not (math.isfinite(pq) and math.isfinite(rz)):
            raise FloatingPointError(f"CG diverged at iteration {it}")
        if pq <= 0.0:
            term = "breakdown"
            break
        alpha = torch.tensor(rz / pq, dtype=b.dtype, device=b.device)
        x = x + alpha * p
        if recompute_every and it % recompute_every == 0:
            r = b - op.apply(x)
            mv += 1
        else:
            r = r - alpha * q
        z = r * inv
        rr, rz_new = op.dots((r, r), (r, z))
        rn = nrm(rnd(rr))
        if not math.isfinite(rn):
            raise FloatingPointError(f"CG diverged at iteration {it}")
        rel = rn / bnorm
        hist.append(rel)
        if rel <= rel_tol:
            term, done = "converged", True
            break
        rz_new = rnd(rz_new)
        beta = torch.tensor(rz_new / rz, dtype=b.dtype, device=b.device)
        p = z + beta * p
        rz = rz_new
    return x, dict(iterations=it, termination=term, rel=rel, history=hist, matvecs=mv)


class NativeSlab:
    """Handle of the native slab runtime bound to a SlabOperator with the
    peer transport: products, all-reduces and batches of CG iterations are
    enqueued from C++ (csrc/tf_slab_run.cu), sharing the transport's receive
    regions and epoch counters."""

    def __init__(self, sop: "SlabOperator"):
        import ctypes

        import torch

        from . import _device as D
        from . import _lib

        tr, la = sop.exchange, sop.local_apply
        op = la.op
        self.sop = sop
        self._keep = [np.ascontiguousarray(op.ke), sop.owned.to(torch.uint8)]
        self._peers = (ctypes.c_void_p * tr.world)(*[tr.peer[r] for r in range(tr.world)])
        d = _lib.tf_slab_desc()
        d.grid = op.dev.grid
        d.precision = 64 if op.precision.dtype == np.float64 else 32
        d.ke = self._keep[0].ctypes.data
        d.scale = D.ptr(op._scale_dev)
        d.node_fixed = D.ptr(op.dev.node_fixed)
        d.fixed = D.ptr(sop.fixed) if sop.fixed.numel() else None
        d.n_fixed = int(sop.fixed.numel())
        d.owned = D.ptr(self._keep[1])
        d.left_idx, d.right_idx = D.ptr(tr.left_idx), D.ptr(tr.right_idx)
        d.plane_len = tr.plane_len
        p = sop.part
        d.has_left, d.has_right, d.rank, d.world = int(p.has_left), int(p.has_right), tr.rank, tr.world
        d.peer_base = ctypes.cast(self._peers, ctypes.c_void_p)
        d.off_planes, d.plane_bytes, d.off_flags = tr.off_planes, tr.plane_bytes, tr.off_flags
        d.off_arflags, d.off_slots, d.max_scalars = tr.off_arflags, tr.off_slots, tr.max_scalars
        d.bl, d.br = int(la.bl), int(la.br)
        h = ctypes.c_void_p()
        _lib.call("tf_slab_create", ctypes.byref(h), ctypes.byref(d))
        self.h = h
        self.epochs = (ctypes.c_uint32 * 2)()

    def _sync_in(self):
        tr = self.sop.exchange
        self.epochs[0], self.epochs[1] = tr.epoch, tr.ar_epoch

    def _sync_out(self):
        tr = self.sop.exchange
        tr.epoch, tr.ar_epoch = int(self.epochs[0]), int(self.epochs[1])

    def apply(self, x, out=None):
        import torch

        from . import _device as D
        from . import _lib

        w = torch.empty_like(x) if out is None else out
        self._sync_in()
        _lib.call("tf_slab_apply", self.h, D.ptr(x), D.ptr(w), self.epochs, D.stream_ptr())
        self._sync_out()
        return w

    def iterate(self, b, inv, x, r, z, p, q, wtmp, state, red, work, it0, n, recompute_every, hist,
                graph: bool = False):
        """n CG iterations it0+1..it0+n enqueued from C++; graph=True replays
        them as one CUDA graph (aligned blocks, see tf_slab_pcg_graph)."""
        from . import _device as D
        from . import _lib

        self._sync_in()
        args = (self.h, D.ptr(b), D.ptr(inv), D.ptr(x), D.ptr(r), D.ptr(z), D.ptr(p), D.ptr(q), D.ptr(wtmp),
                D.ptr(state), D.ptr(red), D.ptr(work), int(it0), int(n), int(recompute_every), D.ptr(hist),
                int(hist.numel()), self.epochs)
        if graph:
            _lib.call("tf_slab_pcg_graph", *args, None, D.stream_ptr())
        else:
            _lib.call("tf_slab_pcg_iterate", *args, D.stream_ptr())
        self._sync_out()

    def take_error(self) -> bool:
        import ctypes

        from . import _lib

        e = ctypes.c_int(0)
        _lib.call("tf_slab_take_error", self.h, ctypes.byref(e))
        return bool(e.value)

    def __del__(self):
        try:
            from . import _lib

            _lib.load().tf_slab_destroy(self.h)
        except Exception:
            pass


_SLAB_TERMS = {1: "converged", 2: "breakdown", 3: "diverged"}


def slab_pcg_device(op: SlabOperator, b, diag, rel_tol=1e-5, max_iter=1000, recompute_every=50, x0=None,
                    poll: int = 8):
    """slab_pcg with every scalar on the device (csrc/tf_slab.cu).

    Per iteration the host only enqueues: q = K p (slab kernels + interface
    exchange), the owned p.q partial, an all-reduce of it, the alpha step
    (x, r, z and the (r.r, r.z) partials), a second all-reduce and the beta
    step.  Nothing waits for the GPU except a poll of the device state every
    `poll` iterations; the device freezes the solve at the exact stop
    iteration, so results do not depend on `poll`.
    """
    import os

    import torch

    from . import _device as D
    from . import _lib

    f32 = b.dtype == torch.float32
    sfx = "f32" if f32 else "f64"
    dev = b.device
    st = D.stream_ptr()
    n = b.numel()
    f64 = torch.float64
    owned = op.owned.to(torch.uint8)
    work = torch.zeros(int(_lib.load().tf_slab_work_doubles(n)), dtype=f64, device=dev)
    red = torch.zeros(8, dtype=f64, device=dev)  # [0..7]: the single-reduction iteration's sums
    state = torch.zeros(8, dtype=f64, device=dev)
    hist = torch.full((max_iter + 1,), float("nan"), dtype=f64, device=dev)

    def allreduce(lo, hi):
        op.allreduce_dev(red, lo, hi)

    _lib.call(f"tf_slab_dot_{sfx}", n, D.ptr(b), D.ptr(b), D.ptr(owned), D.ptr(red) + 24, D.ptr(work), st)
    allreduce(3, 4)
    if float(red[3]) == 0.0:
        return torch.zeros_like(b), dict(iterations=0, termination="converged", rel=0.0, history=[0.0],
                                         matvecs=0)
    mv = 0
    if x0 is None:
        x = torch.zeros_like(b)
        r = b.clone()
    else:
        x = x0.clone()
        r = b - op.apply(x)
        mv += 1
    inv = 1.0 / diag
    z = torch.empty_like(b)
    p = torch.empty_like(b)
    _lib.call(f"tf_slab_cg_begin_{sfx}", n, D.ptr(r), D.ptr(inv), D.ptr(z), D.ptr(p), D.ptr(owned), D.ptr(red),
              D.ptr(work), st)
    allreduce(1, 3)
    _lib.call("tf_slab_cg_start", D.ptr(state), D.ptr(red), float(rel_tol), int(f32), st)
    hist[0:1].copy_(state[2:3])
    native = op.native()
    if native is not None and float(state[4]) != 0.0:
        # the whole loop body enqueued from C++ in batches of `poll` iterations
        q = torch.empty_like(b)
        wtmp = torch.empty_like(b)
        # CUDA-graph blocks of G iterations (TF_SLAB_GRAPH=0: plain enqueue):
        # G divides recompute_every so every block's refresh pattern is one
        # of two captured graphs; the first block runs eagerly (autotune,
        # first-touch), partial tail blocks too
        G = 10
        use_graph = (os.environ.get("TF_SLAB_GRAPH", "1") == "1"
                     and (recompute_every == 0 or recompute_every % G == 0))
        it = 0
        while it < max_iter:
            k = min(G if use_graph else poll, max_iter - it)
            graph = use_graph and it > 0 and k == G
            native.iterate(b, inv, x, r, z, p, q, wtmp, state, red, work, it, k, recompute_every, hist,
                           graph=graph)
            it += k
            if float(state[4]) == 0.0:
                break
        if native.take_error():
            raise RuntimeError("slab exchange timed out: a peer rank stopped raising its flags")
    elif float(state[4]) != 0.0:
        for it in range(1, max_iter + 1):
            q = op.apply(p)
            _lib.call(f"tf_slab_cg_pq_{sfx}", n, D.ptr(p), D.ptr(q), D.ptr(owned), D.ptr(state), D.ptr(red),
                      D.ptr(work), st)
            allreduce(0, 1)
            refresh = bool(recompute_every) and it % recompute_every == 0
            _lib.call(f"tf_slab_cg_alpha_{sfx}", n, D.ptr(x), D.ptr(r), D.ptr(p), D.ptr(q), D.ptr(inv), D.ptr(z),
                      D.ptr(owned), D.ptr(state), D.ptr(red), int(refresh), D.ptr(work), st)
            if refresh:
                w = op.apply(x)
                _lib.call(f"tf_slab_cg_residual_{sfx}", n, D.ptr(b), D.ptr(w), D.ptr(r), D.ptr(inv), D.ptr(z),
                          D.ptr(owned), D.ptr(state), D.ptr(red), D.ptr(work), st)
            allreduce(1, 3)
            _lib.call(f"tf_slab_cg_beta_{sfx}", n, D.ptr(p), D.ptr(z), D.ptr(state), D.ptr(red), D.ptr(hist),
                      max_iter + 1, st)
            if (it % poll == 0 or it == max_iter) and float(state[4]) == 0.0:
                break
    s_h = state.cpu().numpy()
    its = int(s_h[3])
    term = _SLAB_TERMS.get(int(s_h[5]), "max_iter")
    if term == "diverged":
        raise FloatingPointError(f"CG diverged at iteration {its}")
    if x0 is not None:
        mv = 1
    refreshes = its // recompute_every if recompute_every else 0
    if term == "breakdown" and recompute_every and its % recompute_every == 0:
        refreshes -= 1
    mv += its + refreshes
    h = hist.cpu().numpy()
    n_hist = its if term == "breakdown" else its + 1
    history = [float(v) for v in h[:n_hist]]
    return x, dict(iterations=its, termination=term, rel=history[-1], history=history, matvecs=mv)


def gpu_local_kernels(part: SlabPartition, bcs_local: BoundaryConditions, rho_local, simp,
                      precision: str, nu: float = 0.3):
    """Bind the sm_100a kernels as the slab's local compute."""
    import torch

    from . import _device as D
    from . import _lib
    from .mesh import build_edof
    from .operator import MatFreeOperator, ctypes_ref

    lm = part.local_mesh
    op = MatFreeOperator(lm, build_edof(lm), bcs_local, rho_local, simp, precision, nu=nu)
    dt = op.precision.dtype
    sfx = "f64" if dt == np.float64 else "f32"

    def local_apply(x):
        out = torch.empty_like(x)
        _lib.call(f"tf_matvec_grid_{sfx}", ctypes_ref(op.dev.grid), op.ke.ctypes.data,
                  D.ptr(op._scale_dev), D.ptr(x), D.ptr(out), D.ptr(op.dev.node_fixed),
                  _lib.TF_MASK_INPUT, op.grid_variant, D.stream_ptr())
        return out

    nnx = lm.nelx + 1
    bl = min(31, nnx) if part.has_left else 0          # one tile of interface columns
    br = min(31, nnx - bl) if part.has_right else 0

    def split(x, out, phase):
        """phase "boundary": outputs of the interface tiles; "interior": the rest."""
        if out is None:
            out = torch.empty_like(x)
        ranges = [(0, bl), (nnx - br, nnx)] if phase == "boundary" else [(bl, nnx - br)]
        for lo, hi in ranges:
            if hi > lo:
                _lib.call(f"tf_matvec_grid_range_{sfx}", ctypes_ref(op.dev.grid), op.ke.ctypes.data,
                          D.ptr(op._scale_dev), D.ptr(x), D.ptr(out), D.ptr(op.dev.node_fixed),
                          _lib.TF_MASK_INPUT, int(lo), int(hi), D.stream_ptr())
        return out

    if op.grid_kernel == "tile":
        local_apply.split = split
        # what the native slab runtime (tf_slab_run.cu) needs to run this slab
        local_apply.op, local_apply.bl, local_apply.br = op, bl, br

    def local_diag_partial():
        # FP64 partial sums of s_e * Ke[l,l] on this slab (no fixed handling
        # yet), gathered per node in ascending element order: deterministic
        kd = np.ascontiguousarray(np.diag(op.ke), dtype=dt)
        acc = torch.empty(lm.n_dof, dtype=torch.float64, device=op._scale_dev.device)
        _lib.call(f"tf_jacobi_grid_partial_{sfx}", ctypes_ref(op.dev.grid), kd.ctypes.data,
                  D.ptr(op._scale_dev), D.ptr(acc), D.stream_ptr())
        return acc

    return op, local_apply, local_diag_partial
