"""Plan file v1: the packed butterfly factorization handed to ``mht_plan_load``.

Layout (little-endian; DESIGN.md §4 is the normative description):

header, 256 bytes::

    0   char[8]  "BFMHTPLN"
    8   u32      version = 1, or 2 when the plan carries a frequency permutation
    12  u32      dtype   (1 = float64, 2 = complex128)
    16  i64      n       (spatial points, rows of Phi)
    24  i64      m       (eigenfunctions, columns of Phi)
    32  i32      L       (levels; both trees have 2^L leaves)
    36  i32      0
    40  f64      tol     (ID tolerance used to build the plan)
    48  i64      n_stages = L + 2
    56  u64      checksum: wrapping sum of the body's little-endian u64 words
    64  i64      body_bytes
    72.. zero

body::

    i32 perm_x[n]           tree position -> user point index (pad to 8 B)
    i64 sp_off[2^L + 1]     space-leaf row offsets (in tree positions)
    i64 fr_off[2^L + 1]     frequency-leaf column offsets (plan frequency order)
    i32 perm_k[m]           (version 2 only) plan frequency position -> user coefficient index,
                            pad to 8 B: c[perm_k[q]] feeds plan column q (the quadtree-frequency
                            plans keep the user's eigenvalue order of c, reading A18)
    stage s = 0 .. L+1:
        i64 s, i64 nblk (= 2^L), i64 nidx, i64 ncoef
        scalar coef[ncoef]                   (8 B real / 16 B complex)
        nblk x {i32 kind, i32 r_out, i32 r_in, i32 0, i64 idx_off, i64 coef_off}
        i32 idx[nidx]                        (pad to 8 B)

Blocks (§2; reading A2 of SURVEY.md §8(c)):

* stage 0 — frequency leaf v: in = c[fr_off[v]:fr_off[v+1]], out = z_0(v).
* stage l in 1..L — block b = t * 2^(L-l) + v (t a space node at depth l, v a
  frequency node at height l): in = [z_{l-1}(t>>1, 2v); z_{l-1}(t>>1, 2v+1)].
* stage L+1 — space leaf t: in = z_L(t), out = f rows perm_x[sp_off[t]:sp_off[t+1]].

kind 0 IDENTITY (r_out == r_in, nothing stored); kind 1 ID: idx[idx_off:+r_out]
= skeleton positions, idx[idx_off+r_out : +r_in] = redundant positions,
coef[coef_off : + r_out*(r_in-r_out)] = T column-major, out = in[skel] +
T in[red]; kind 2 DENSE: coef r_out x r_in column-major, out = D in.

The writer streams: coefficients are appended as blocks complete (in canonical
block order) and the block table + index pool of a stage follow its
coefficients, so a plan larger than host RAM can be written in one pass.
"""
from __future__ import annotations

import os
import struct
from dataclasses import dataclass

import numpy as np

MAGIC = b"BFMHTPLN"
VERSION = 1           # without a frequency permutation
VERSION_PERMK = 2     # with perm_k[m] after fr_off
HEADER_BYTES = 256
KIND_IDENTITY, KIND_ID, KIND_DENSE = 0, 1, 2
DT_REAL, DT_COMPLEX = 1, 2
BLOCK_REC = np.dtype([("kind", "<i4"), ("r_out", "<i4"), ("r_in", "<i4"), ("pad", "<i4"),
                      ("idx_off", "<i8"), ("coef_off", "<i8")])


def _sum64(buf: bytes | np.ndarray) -> int:
    a = np.frombuffer(buf, dtype="<u8") if not isinstance(buf, np.ndarray) else buf.view("<u8")
    return int(a.sum(dtype=np.uint64)) & 0xFFFFFFFFFFFFFFFF


def _pad8(b: bytes) -> bytes:
    r = (-len(b)) % 8
    return b + b"\0" * r


class PlanWriter:
    """Streaming writer.  Usage::

        w = PlanWriter(path, dtype, n, m, L, tol, perm, sp_off, fr_off)
        for s in range(L + 2):
            w.begin_stage(s)
            for each block in canonical order: w.add_block(kind, r_out, r_in, skel, red, coef)
            w.end_stage()
        w.close()
    """

    def __init__(self, path, dtype, n, m, L, tol, perm, sp_off, fr_off, perm_k=None):
        self.path = str(path)
        self.complex = np.dtype(dtype) == np.complex128
        self.sdt = np.dtype("<c16") if self.complex else np.dtype("<f8")
        self.n, self.m, self.L, self.tol = int(n), int(m), int(L), float(tol)
        self.f = open(self.path + ".part", "wb")
        self.f.write(b"\0" * HEADER_BYTES)
        self.csum = 0
        self.body = 0
        nl = 1 << self.L
        perm = np.asarray(perm, dtype="<i4")
        sp_off = np.asarray(sp_off, dtype="<i8")
        fr_off = np.asarray(fr_off, dtype="<i8")
        assert perm.shape == (self.n,) and sp_off.shape == (nl + 1,) and fr_off.shape == (nl + 1,)
        assert sp_off[0] == 0 and sp_off[-1] == self.n and fr_off[0] == 0 and fr_off[-1] == self.m
        assert np.array_equal(np.sort(perm), np.arange(self.n))
        self._write(_pad8(perm.tobytes()))
        self._write(sp_off.tobytes())
        self._write(fr_off.tobytes())
        self.version = VERSION
        if perm_k is not None:
            perm_k = np.asarray(perm_k, dtype="<i4")
            assert perm_k.shape == (self.m,) and np.array_equal(np.sort(perm_k), np.arange(self.m))
            self._write(_pad8(perm_k.tobytes()))
            self.version = VERSION_PERMK
        self.stage = None
        self.entries = 0
        self.stage_stats = []

    def _write(self, b):
        if isinstance(b, np.ndarray):
            b = np.ascontiguousarray(b)
            mv = memoryview(b).cast("B")
            self.f.write(mv)
            self.csum = (self.csum + _sum64(b.reshape(-1).view(np.uint8))) & 0xFFFFFFFFFFFFFFFF
            self.body += b.nbytes
        else:
            self.f.write(b)
            self.csum = (self.csum + _sum64(b)) & 0xFFFFFFFFFFFFFFFF
            self.body += len(b)

    def begin_stage(self, s):
        assert self.stage is None
        self.stage = s
        self.hdr_pos = self.f.tell()
        self._write(struct.pack("<qqqq", s, 0, 0, 0))  # patched in end_stage
        self.recs = []
        self.idx = []
        self.nidx = 0
        self.ncoef = 0

    def add_block(self, kind, r_out, r_in, skel=None, red=None, coef=None):
        idx_off = coef_off = 0
        if kind == KIND_IDENTITY:
            assert r_out == r_in
        elif kind == KIND_ID:
            skel = np.asarray(skel, dtype="<i4")
            red = np.asarray(red, dtype="<i4")
            assert skel.size == r_out and red.size == r_in - r_out
            idx_off = self.nidx
            self.idx.append(skel)
            self.idx.append(red)
            self.nidx += r_in
            coef = np.asarray(coef)
            assert coef.shape == (r_out, r_in - r_out), (coef.shape, r_out, r_in)
            coef_off = self.ncoef
            self._write(np.asfortranarray(coef).astype(self.sdt).T.reshape(-1))
            self.ncoef += coef.size
        elif kind == KIND_DENSE:
            coef = np.asarray(coef)
            assert coef.shape == (r_out, r_in)
            coef_off = self.ncoef
            self._write(np.asfortranarray(coef).astype(self.sdt).T.reshape(-1))
            self.ncoef += coef.size
        else:
            raise ValueError(kind)
        self.recs.append((kind, r_out, r_in, 0, idx_off, coef_off))

    def end_stage(self):
        rec = np.array(self.recs, dtype=BLOCK_REC)
        assert rec.shape[0] == (1 << self.L)
        self._write(rec.tobytes())
        idx = np.concatenate(self.idx) if self.idx else np.zeros(0, "<i4")
        self._write(_pad8(idx.astype("<i4").tobytes()))
        # patch the stage header (placeholders were zero, so add to the checksum)
        end = self.f.tell()
        self.f.seek(self.hdr_pos + 8)
        patch = struct.pack("<qqq", len(self.recs), self.nidx, self.ncoef)
        self.f.write(patch)
        self.csum = (self.csum + _sum64(patch)) & 0xFFFFFFFFFFFFFFFF
        self.f.seek(end)
        self.entries += self.ncoef
        kinds = rec["kind"]
        self.stage_stats.append(dict(stage=self.stage, ncoef=int(self.ncoef),
                                     n_identity=int((kinds == 0).sum()), n_id=int((kinds == 1).sum()),
                                     n_dense=int((kinds == 2).sum()),
                                     r_out_mean=float(rec["r_out"].mean()),
                                     r_out_max=int(rec["r_out"].max())))
        self.stage = None

    def add_stage_spooled(self, s, spool_path, ncoef, recs, idx_list):
        """Write stage s whose coefficients were spooled to ``spool_path`` in
        any block order (``recs`` = per block (kind, r_out, r_in, 0, idx_off,
        spool_off) in canonical order, ``idx_list`` the index arrays in idx_off
        order).  The coefficients are copied into canonical block order, so the
        stage is laid out exactly as the stage-order writer lays it out.  Used
        by the post-order builder (streaming.py)."""
        assert self.stage is None
        nl = 1 << self.L
        assert len(recs) == nl
        nidx = int(sum(a.size for a in idx_list))
        self._write(struct.pack("<qqqq", s, nl, nidx, int(ncoef)))
        out = []
        cur = 0
        isz = self.sdt.itemsize
        with open(spool_path, "rb") as f:
            for (kind, r_out, r_in, pad, idx_off, spool_off) in recs:
                cnt = r_out * (r_in - r_out) if kind == KIND_ID else (r_out * r_in if kind == KIND_DENSE else 0)
                if cnt:
                    f.seek(int(spool_off) * isz)
                    b = f.read(cnt * isz)
                    if len(b) != cnt * isz:
                        raise IOError("short spool")
                    self._write(b)
                out.append((kind, r_out, r_in, pad, idx_off, cur if cnt else 0))
                cur += cnt
        assert cur == int(ncoef)
        rec = np.array(out, dtype=BLOCK_REC)
        self._write(rec.tobytes())
        idx = np.concatenate(idx_list) if idx_list else np.zeros(0, "<i4")
        self._write(_pad8(idx.astype("<i4").tobytes()))
        self.entries += int(ncoef)
        kinds = rec["kind"]
        self.stage_stats.append(dict(stage=s, ncoef=int(ncoef), n_identity=int((kinds == 0).sum()),
                                     n_id=int((kinds == 1).sum()), n_dense=int((kinds == 2).sum()),
                                     r_out_mean=float(rec["r_out"].mean()), r_out_max=int(rec["r_out"].max())))

    def close(self):
        assert self.stage is None
        self.f.seek(0)
        hdr = bytearray(HEADER_BYTES)
        struct.pack_into("<8sIIqqiidqQq", hdr, 0, MAGIC, self.version,
                         DT_COMPLEX if self.complex else DT_REAL, self.n, self.m, self.L, 0,
                         self.tol, self.L + 2, self.csum, self.body)
        self.f.write(bytes(hdr))
        self.f.close()
        os.replace(self.path + ".part", self.path)


@dataclass
class StageView:
    nblk: int
    nidx: int
    ncoef: int
    blocks: np.ndarray   # BLOCK_REC
    idx: np.ndarray      # int32
    coef: np.ndarray     # scalar


class PlanView:
    """Read-only numpy view of a plan file (memory-mapped; product-side helper
    for statistics and invariants — the C loader in csrc/ is what the GPU path uses)."""

    def __init__(self, path):
        self.path = str(path)
        self.mm = np.memmap(self.path, dtype=np.uint8, mode="r")
        h = bytes(self.mm[:HEADER_BYTES])
        (magic, ver, dt, n, m, L, _z, tol, nst, csum, body) = struct.unpack_from("<8sIIqqiidqQq", h, 0)
        if magic != MAGIC or ver not in (VERSION, VERSION_PERMK):
            raise ValueError("not a v1 / v2 plan")
        self.complex = dt == DT_COMPLEX
        self.sdt = np.dtype("<c16") if self.complex else np.dtype("<f8")
        self.n, self.m, self.L, self.tol, self.checksum, self.body = n, m, L, tol, csum, body
        nl = 1 << L
        q = HEADER_BYTES
        self.perm = self.mm[q:q + 4 * n].view("<i4")
        q += ((4 * n + 7) // 8) * 8
        self.sp_off = self.mm[q:q + 8 * (nl + 1)].view("<i8")
        q += 8 * (nl + 1)
        self.fr_off = self.mm[q:q + 8 * (nl + 1)].view("<i8")
        q += 8 * (nl + 1)
        self.perm_k = None
        if ver == VERSION_PERMK:
            self.perm_k = self.mm[q:q + 4 * m].view("<i4")
            q += ((4 * m + 7) // 8) * 8
        self.stages = []
        for s in range(L + 2):
            sh = self.mm[q:q + 32].view("<i8")
            assert sh[0] == s
            nblk, nidx, ncoef = int(sh[1]), int(sh[2]), int(sh[3])
            q += 32
            coef = self.mm[q:q + ncoef * self.sdt.itemsize].view(self.sdt)
            q += ncoef * self.sdt.itemsize
            blocks = self.mm[q:q + 32 * nblk].view(BLOCK_REC)
            q += 32 * nblk
            idx = self.mm[q:q + 4 * nidx].view("<i4")
            q += ((4 * nidx + 7) // 8) * 8
            self.stages.append(StageView(nblk, nidx, ncoef, blocks, idx, coef))
        assert q == HEADER_BYTES + body

    def verify_checksum(self) -> bool:
        return _sum64(self.mm[HEADER_BYTES:]) == self.checksum

    @property
    def entries(self) -> int:
        return sum(s.ncoef for s in self.stages)

    @property
    def scalar_bytes(self) -> int:
        return self.sdt.itemsize

    def stage_entries(self):
        return [s.ncoef for s in self.stages]
