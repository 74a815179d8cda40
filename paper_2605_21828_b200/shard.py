"""Sharded plans: one butterfly factorization across G GPUs.

Stages 0..ls are partitioned by the G frequency subtrees at height L - log2 G,
stages ls+1..L+1 by the G space subtrees at depth log2 G (§2,
P:241-271: a transfer block (tau, nu) reads only z(parent(tau), children(nu)),
so both partitions are closed under the recursion).  The one exchange step is
an all-to-all of z_ls; the library (``mht_apply_shard_begin`` / ``_end`` and
the adjoint pair, ``include/mht.h``) runs every stage, this module only moves
the exchange blocks:

* ``ShardPlan`` — one rank's shard, with ``apply`` / ``adjoint`` that do
  begin -> ``torch.distributed.all_to_all_single`` (NCCL on GPUs) -> end;
* ``exchange_sizes`` — the exchange layout computed on the host from the plan
  file alone (no GPU), the same layout the loader builds; the gloo CPU tests
  check the all-to-all moves every z_ls block to its owner with it;
* ``emulate`` — all G shards on ONE GPU with the exchange done by device
  copies (the single-GPU correctness check of the sharded path);
* the fused exchange (``ShardPlan.fuse`` / ``emulate_fuse``): the switch
  stage's kernels store z_ls straight into the destination ranks' receive
  buffers over peer memory (CUDA IPC mappings, ``mht_shard_open_peers``) and
  signal them; no all-to-all call is left between ``begin`` and ``end``.  The
  host side only exchanges the IPC handles and layouts (``peer_tables``,
  covered by gloo tests on CPU).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import mht
from .precompute.planfile import PlanView


# --------------------------------------------------------------- host logic
def default_switch_level(L: int, G: int) -> int:
    lg = G.bit_length() - 1
    return max(lg, L // 2)


def check_switch_level(L: int, G: int, ls: int):
    lg = G.bit_length() - 1
    if G < 1 or (G & (G - 1)) != 0:
        raise ValueError("number of shards must be a power of two")
    if not (lg <= ls <= L - lg):
        raise ValueError(f"switch level {ls} outside [log2 G, L - log2 G] = [{lg}, {L - lg}]")


def exchange_sizes(path: str, G: int, ls: int | None = None):
    """Exchange layout of every rank, from the plan file's block tables:
    ``sizes[g][h]`` = workspace entries rank g sends to rank h, and
    ``blocks[g][h]`` = the (tau, nu) pairs of those entries in send order
    (tau-major).  Rank h receives from g exactly ``sizes[g][h]`` entries, in
    the same order."""
    pv = PlanView(path)
    L = pv.L
    ls = default_switch_level(L, G) if ls is None else ls
    check_switch_level(L, G, ls)
    nl = 1 << L
    nf = nl >> ls
    r_out = np.asarray(pv.stages[ls].blocks["r_out"], dtype=np.int64)
    sizes = np.zeros((G, G), dtype=np.int64)
    blocks = [[[] for _ in range(G)] for _ in range(G)]
    for t in range(1 << ls):
        h = t // ((1 << ls) // G)
        for v in range(nf):
            g = v // (nf // G)
            sizes[g, h] += int(r_out[t * nf + v])
            blocks[g][h].append((t, v))
    return sizes, blocks, ls


IPC_HANDLE_BYTES = 64  # sizeof(cudaIpcMemHandle_t)


def peer_tables(exports):
    """The inputs of mht_shard_open_peers from every rank's mht_shard_export
    (rank order): (handles: G x 64 bytes, layouts: G x (2 G + 1) int64), after
    checking that each pair (g, h) agrees on the exchange size (rank g's send
    length to h is rank h's receive length from g, from the offsets)."""
    G = len(exports)
    handles = b"".join(bytes(h) if h is not None else bytes(IPC_HANDLE_BYTES) for h, _ in exports)
    lay = np.array([np.asarray(l, dtype=np.int64) for _, l in exports], dtype=np.int64)
    if lay.shape != (G, 2 * G + 1) or len(handles) != G * IPC_HANDLE_BYTES:
        raise ValueError("inconsistent exports")
    return handles, lay


def gather_exports(mine, G: int, group=None):
    """All-gather every rank's (IPC handle, layout) over `group` (host
    objects: gloo or NCCL) and return peer_tables of them."""
    import torch.distributed as dist

    allx = [None] * G
    dist.all_gather_object(allx, (mine[0], [int(x) for x in mine[1]]), group=group)
    return peer_tables(allx)


class _DevBuf:
    """A raw device range as a torch uint8 tensor (zero copy, via
    __cuda_array_interface__); the memory stays owned by the plan."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (int(nbytes),), "typestr": "|u1", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


# --------------------------------------------------------------- one rank
class ShardPlan:
    """Rank ``shard`` of a plan split over ``nshards`` GPUs."""

    def __init__(self, path: str, nshards: int, shard: int, device: int = 0, switch_level: int = -1):
        import torch

        L = mht.load_library()
        h = C.c_void_p()
        mht._check(L.mht_plan_load_shard(str(path).encode(), int(device), int(nshards), int(shard),
                                         int(switch_level), C.byref(h)), "mht_plan_load_shard")
        self._h = h.value
        self.device = torch.device("cuda", device)
        self.info = mht.mht_plan_info_get(self._h)
        self.n, self.m, self.L = self.info.n, self.info.m, self.info.L
        self.is_complex = self.info.dtype == mht.MHT_DTYPE_C128
        self.torch_dtype = torch.complex128 if self.is_complex else torch.float64
        self.scalar_bytes = 16 if self.is_complex else 8
        G, g, ls = C.c_int32(), C.c_int32(), C.c_int32()
        so, sl, ro, rl = ((C.c_int64 * nshards)() for _ in range(4))
        mht._check(L.mht_shard_info(self._h, C.byref(G), C.byref(g), C.byref(ls), so, sl, ro, rl), "mht_shard_info")
        self.G, self.g, self.ls = G.value, g.value, ls.value
        self.send_off, self.send_len = np.array(so[:]), np.array(sl[:])
        self.recv_off, self.recv_len = np.array(ro[:]), np.array(rl[:])

    def _stream(self):
        import torch

        mht.mht_plan_set_stream(self._h, torch.cuda.current_stream(self.device).cuda_stream)

    def _views(self, nrhs: int):
        """(send, recv) uint8 tensors over the workspace exchange ranges, and
        the per-rank split sizes in bytes."""
        import torch

        z = C.c_void_p()
        mht._check(mht.load_library().mht_shard_workspace(self._h, int(nrhs), C.byref(z)), "mht_shard_workspace")
        row = nrhs * self.scalar_bytes
        s0, s1 = int(self.send_off[0]), int(self.send_off[-1] + self.send_len[-1])
        r0, r1 = int(self.recv_off[0]), int(self.recv_off[-1] + self.recv_len[-1])
        send = torch.as_tensor(_DevBuf(z.value + s0 * row, (s1 - s0) * row), device=self.device)
        recv = torch.as_tensor(_DevBuf(z.value + r0 * row, (r1 - r0) * row), device=self.device)
        return send, recv, [int(x) * row for x in self.send_len], [int(x) * row for x in self.recv_len]

    def begin(self, c, nrhs: int):
        self._stream()
        mht._check(mht.load_library().mht_apply_shard_begin(self._h, C.c_void_p(c.data_ptr()), int(nrhs)),
                   "mht_apply_shard_begin")

    def end(self, f, nrhs: int):
        self._stream()
        mht._check(mht.load_library().mht_apply_shard_end(self._h, C.c_void_p(f.data_ptr()), int(nrhs)),
                   "mht_apply_shard_end")

    def adjoint_begin(self, f, nrhs: int):
        self._stream()
        mht._check(mht.load_library().mht_apply_adjoint_shard_begin(self._h, C.c_void_p(f.data_ptr()), int(nrhs)),
                   "mht_apply_adjoint_shard_begin")

    def adjoint_end(self, c, nrhs: int):
        self._stream()
        mht._check(mht.load_library().mht_apply_adjoint_shard_end(self._h, C.c_void_p(c.data_ptr()), int(nrhs)),
                   "mht_apply_adjoint_shard_end")

    fused = False

    def export(self, nrhs: int, ipc: bool = True):
        """(IPC handle bytes or None, layout (2 G + 1) int64) for the peers."""
        h = (C.c_char * IPC_HANDLE_BYTES)() if ipc else None
        lay = (C.c_int64 * (2 * self.G + 1))()
        mht._check(mht.load_library().mht_shard_export(self._h, int(nrhs), h, lay), "mht_shard_export")
        return (bytes(h) if ipc else None), np.array(lay[:], dtype=np.int64)

    def fuse(self, nrhs: int, group=None):
        """Switch to the fused exchange for applies of up to nrhs right-hand
        sides: every rank exports its workspace handle and layout, they are
        all-gathered over `group` (host objects: gloo or NCCL), and each rank
        maps its peers' workspaces (mht_shard_open_peers)."""
        handles, lay = gather_exports(self.export(nrhs), self.G, group)
        hb = C.create_string_buffer(handles, len(handles))
        lp = lay.ravel().ctypes.data_as(C.POINTER(C.c_int64))
        mht._check(mht.load_library().mht_shard_open_peers(self._h, int(nrhs), hb, lp), "mht_shard_open_peers")
        self.fused = True

    def unfuse(self):
        mht._check(mht.load_library().mht_shard_close_peers(self._h), "mht_shard_close_peers")
        self.fused = False

    def apply(self, c, f, group=None):
        """f[rows of this rank] = (Phi c)[rows]; c: (nrhs, m) full, f: (nrhs, n)."""
        import torch.distributed as dist

        nrhs = c.reshape(-1, self.m).shape[0]
        self.begin(c, nrhs)
        if not self.fused:
            send, recv, ssz, rsz = self._views(nrhs)
            dist.all_to_all_single(recv, send, output_split_sizes=rsz, input_split_sizes=ssz, group=group)
        self.end(f, nrhs)
        return f

    def adjoint(self, f, c, group=None):
        """c[frequency range of this rank] = (Phi^* f)[range]; f: (nrhs, n) full."""
        import torch.distributed as dist

        nrhs = f.reshape(-1, self.n).shape[0]
        self.adjoint_begin(f, nrhs)
        if not self.fused:
            send, recv, ssz, rsz = self._views(nrhs)
            dist.all_to_all_single(send, recv, output_split_sizes=ssz, input_split_sizes=rsz, group=group)
        self.adjoint_end(c, nrhs)
        return c

    def close(self):
        if getattr(self, "_h", None):
            mht.mht_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# --------------------------------------------------------------- one-GPU emulation
def _exchange_local(shards, nrhs: int, reverse: bool):
    """The all-to-all among shards living in one process, by device copies."""
    views = [s._views(nrhs) for s in shards]
    G = len(shards)
    for g in range(G):
        send, _, ssz, _ = views[g]
        so = np.concatenate([[0], np.cumsum(ssz)])
        for h in range(G):
            recv, rsz = views[h][1], views[h][3]
            ro = np.concatenate([[0], np.cumsum(rsz)])
            a = send[so[h]:so[h + 1]]
            b = recv[ro[g]:ro[g + 1]]
            if reverse:
                a.copy_(b)
            else:
                b.copy_(a)


def emulate_fuse(shards, nrhs: int):
    """The fused exchange among shards living in one process (one GPU): each
    shard gets the others' workspaces as plain device pointers
    (mht_shard_set_peers), so the switch stage stores into them and the
    arrival flags are set and waited on exactly as across GPUs.  The begins
    of all shards run before the ends (emulate_apply), so no wait spins."""
    ex = [s.export(nrhs, ipc=False) for s in shards]
    _, lay = peer_tables([(None, l) for _, l in ex])
    bases = []
    for s in shards:
        z = C.c_void_p()
        mht._check(mht.load_library().mht_shard_workspace(s._h, int(nrhs), C.byref(z)), "mht_shard_workspace")
        bases.append(z.value)
    arr = (C.c_void_p * len(shards))(*bases)
    lp = lay.ravel().ctypes.data_as(C.POINTER(C.c_int64))
    for s in shards:
        mht._check(mht.load_library().mht_shard_set_peers(s._h, int(nrhs), arr, lp), "mht_shard_set_peers")
        s.fused = True


def emulate_apply(shards, c, f):
    nrhs = c.reshape(-1, shards[0].m).shape[0]
    for s in shards:
        s.begin(c, nrhs)
    if not shards[0].fused:
        _exchange_local(shards, nrhs, reverse=False)
    for s in shards:
        s.end(f, nrhs)
    return f


def emulate_adjoint(shards, f, c):
    nrhs = f.reshape(-1, shards[0].n).shape[0]
    for s in shards:
        s.adjoint_begin(f, nrhs)
    if not shards[0].fused:
        _exchange_local(shards, nrhs, reverse=True)
    for s in shards:
        s.adjoint_end(c, nrhs)
    return c
