"""Peer-memory transport for the x-slab decomposition (csrc/tf_peer.cu).

SURVEY 8e asks to measure NCCL against a custom peer-memory one-shot for the
slab's two exchange steps; this is that transport.  Every rank allocates one
receive region (cudaMalloc) and maps the other ranks' regions through CUDA
IPC (over NVLink on an NVSwitch box; the same-device mapping between
processes on a one-GPU box runs the tests):

  receive region of a rank, bytes
    planes  [parity 2][side 2][plane_len] x 8 B   side 0 = from the left
                                                  neighbour, 1 = from the right
    flags   [2] uint32 plane epochs (per side), then [world] uint32 all-reduce
            epochs (per source rank)
    slots   [parity 2][world][max_scalars] FP64   all-reduce contributions

Interface exchange (same contract as slab.SlabExchange): `start` puts this
rank's interface partials into the neighbours' plane slots with peer stores
and raises their flags (a stream write-value, which fences the puts); the
interior tiles run; `finish` waits on the local flags (stream wait-value, no
SM spin) and adds the received partial in the fixed order (left first).

One-shot all-reduce: each rank puts its k partials into slot [parity][rank]
of every rank, raises its flag there, waits for all ranks' flags and sums the
slots in rank order on the device -- every rank gets the bitwise-same
result, no host round trip.
"""

from __future__ import annotations

import ctypes

from . import _device as D
from . import _lib


class PeerTransport:
    def __init__(self, part, device, group=None, max_scalars: int = 8):
        import torch
        import torch.distributed as dist

        t = torch
        self.part = part
        self.group = group
        self.device = device
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        lm = part.local_mesh
        self.left_idx = t.as_tensor(part.plane_dofs(0), device=device)
        self.right_idx = t.as_tensor(part.plane_dofs(lm.nelx), device=device)
        self.plane_len = int(self.left_idx.numel())
        self.max_scalars = int(max_scalars)
        self.off_planes = 0
        self.plane_bytes = 8 * self.plane_len
        self.off_flags = 4 * self.plane_bytes
        self.off_arflags = self.off_flags + 8
        self.off_slots = ((self.off_arflags + 4 * self.world + 255) // 256) * 256
        self.bytes = self.off_slots + 2 * self.world * self.max_scalars * 8
        L = _lib.load()
        p = ctypes.c_void_p()
        _lib.check(L.tf_peer_alloc(ctypes.byref(p), ctypes.c_size_t(self.bytes)), "tf_peer_alloc")
        self.base = int(p.value)
        hb = int(L.tf_ipc_handle_bytes())
        handle = (ctypes.c_char * hb)()
        mine = bytes(handle) if L.tf_ipc_export(ctypes.c_void_p(self.base), handle) == _lib.TF_OK else None
        if mine is not None:
            mine = bytes(handle)
        handles = [mine] * self.world
        if self.world > 1:
            dist.all_gather_object(handles, mine, group=group)
        self.peer = {self.rank: self.base}
        err = None if all(h is not None for h in handles) else "cudaIpcGetMemHandle failed on a rank"
        for r in range(self.world):
            if r == self.rank or err:
                continue
            q = ctypes.c_void_p()
            hbuf = ctypes.create_string_buffer(handles[r], hb)
            rc = L.tf_ipc_open(hbuf, ctypes.byref(q))
            if rc != _lib.TF_OK:
                err = L.tf_last_error().decode(errors="replace")
                break
            self.peer[r] = int(q.value)
        if self.world > 1:
            # every rank learns whether all mappings exist (and none puts
            # before they do): one all-reduce instead of a bare barrier, so a
            # failing rank cannot leave the others waiting in a collective
            gloo = dist.get_backend(group) == "gloo"
            ok = t.tensor([0 if err else 1], dtype=t.int32, device="cpu" if gloo else device)
            dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
            if int(ok.item()) == 0:
                self.close()
                raise RuntimeError(f"peer transport unavailable: {err or 'a peer rank failed to map'}")
        self.epoch = 0
        self.ar_epoch = 0
        self.scalar_idx = t.arange(self.max_scalars, dtype=t.int64, device=device)
        self._acc = t.empty(self.max_scalars, dtype=t.float64, device=device)
        self._tickets = t.zeros(16, dtype=t.int32, device=device)  # tf_put_flags block counters

    # -- layout ------------------------------------------------------------------
    def _plane(self, base, parity, side):
        return base + self.off_planes + (2 * parity + side) * self.plane_bytes

    def _flag(self, base, side):
        return base + self.off_flags + 4 * side

    def _arflag(self, base, src):
        return base + self.off_arflags + 4 * src

    def _slot(self, base, parity, src):
        return base + self.off_slots + 8 * self.max_scalars * (self.world * parity + src)

    # -- interface exchange (SlabExchange contract) -----------------------------
    def __call__(self, w):
        return self.finish(w, self.start(w))

    @staticmethod
    def _arr(ctype, vals):
        return (ctype * max(1, len(vals)))(*vals)

    def start(self, w):
        """Both interface planes into the neighbours' slots and their flags
        raised, one launch (tf_put_flags)."""
        p = self.part
        self.epoch += 1
        e, par = self.epoch, self.epoch & 1
        sfx = "f64" if w.element_size() == 8 else "f32"
        idx, dst, flg = [], [], []
        if p.has_left:  # my left plane -> the left neighbour's "from right" slot
            nb = self.peer[p.rank - 1]
            idx.append(D.ptr(self.left_idx)), dst.append(self._plane(nb, par, 1)), flg.append(self._flag(nb, 1))
        if p.has_right:
            nb = self.peer[p.rank + 1]
            idx.append(D.ptr(self.right_idx)), dst.append(self._plane(nb, par, 0)), flg.append(self._flag(nb, 0))
        if idx:
            V = ctypes.c_void_p
            _lib.call(f"tf_put_flags_{sfx}", D.ptr(w), self._arr(V, idx), self._arr(V, dst), self._arr(V, flg),
                      len(idx), self.plane_len, e, D.ptr(self._tickets), D.stream_ptr())
        return e

    def finish(self, w, state):
        p = self.part
        e, par = state, state & 1
        sfx = "f64" if w.element_size() == 8 else "f32"
        st = D.stream_ptr()
        waits = ([self._flag(self.base, 0)] if p.has_left else []) + ([self._flag(self.base, 1)] if p.has_right else [])
        if waits:
            _lib.call("tf_stream_wait_many_u32", self._arr(ctypes.c_void_p, waits), len(waits), e, st)
            # left partial first on the left plane, own partial first on the right
            _lib.call(f"tf_plane_add2_{sfx}", D.ptr(w), D.ptr(self.left_idx) if p.has_left else None,
                      self._plane(self.base, par, 0), D.ptr(self.right_idx) if p.has_right else None,
                      self._plane(self.base, par, 1), self.plane_len, st)
        return w

    # -- one-shot all-reduce of FP64 scalars -------------------------------------
    def allreduce_(self, t, lo: int, hi: int):
        """In place: t[lo:hi] (FP64, device) = sum over ranks, rank order."""
        k = hi - lo
        if k > self.max_scalars:
            raise ValueError("too many scalars for the peer all-reduce")
        if self.world == 1:
            return t
        self.ar_epoch += 1
        e, par = self.ar_epoch, self.ar_epoch & 1
        st = D.stream_ptr()
        src = D.ptr(t) + 8 * lo
        V = ctypes.c_void_p
        dst = self._arr(V, [self._slot(self.peer[r], par, self.rank) for r in range(self.world)])
        flg = self._arr(V, [self._arflag(self.peer[r], self.rank) for r in range(self.world)])
        # own partials into every rank's slot + flags (one launch), one batched wait
        _lib.call("tf_put_flags_f64", src, None, dst, flg, self.world, k, e, D.ptr(self._tickets), st)
        waits = self._arr(V, [self._arflag(self.base, r) for r in range(self.world)])
        _lib.call("tf_stream_wait_many_u32", waits, self.world, e, st)
        # the slots of one parity are [world][max_scalars]: sum full rows in
        # rank order, keep the k used
        _lib.call("tf_rank_sum_f64", self._slot(self.base, par, 0), self.world, self.max_scalars,
                  D.ptr(self._acc), st)
        t[lo:hi].copy_(self._acc[:k])
        return t

    def close(self):
        """Unmap the peers' regions and free this rank's (idempotent).  Peers
        may still write into a freed region if they outlive this rank's
        transport: close all ranks' transports at the same point."""
        if getattr(self, "base", None) is None:
            return
        L = _lib.load()
        for r, ptr in self.peer.items():
            if r != self.rank:
                L.tf_ipc_close(ctypes.c_void_p(ptr))
        self.peer = {}
        L.tf_peer_free(ctypes.c_void_p(self.base))
        self.base = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown: the context may be gone
            pass


__all__ = ["PeerTransport"]
