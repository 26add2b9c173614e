"""Plans for the shared-memory staged sweep (``mfg_sweep_staged``).

The staged sweep computes exactly what ``mfg_sweep`` computes -- the unit of
the BASELINE metric: R = P_Omega(W H^T) - A (``residual_on_omega``,
mfg/data.py:272-280), R.H and R^T.W (``grad.csr @ H``, ``grad.csr_t @ W``,
mfg/operators.py:108,117), sum r^2 (``loss_quad``, mfg/data.py:291-293) and
||W||^2, ||H||^2 (``FactorPair.frob_sq``, mfg/operators.py:53-55) -- but
reads the gathered factor rows from shared memory. This module builds the
reordered entry streams the kernel walks. Planning runs once per
(ObservationSet, k) with torch ops on the tensors' device; the layout it
produces:

* per orientation (pass 0 = CSR rows gathering H, pass 1 = CSC rows gathering
  W): the gathered rows ranked by degree (descending, ties by id) and cut into
  blocks of S rows; block b is *staged* while its entries per nonempty
  (output row, block) pair reach ``lmin`` (the Zipf head), the remaining
  entries form the *cold* segment that gathers from global memory;
* the entry stream: segments in block order then cold, each 32-entry aligned,
  entries in (output row, col) order inside a segment; per entry the block
  slot (cold: gathered row id), output row, value and CSR position;
* chunks (one 8-lane worker each, a multiple of 32 entries, never crossing a
  segment) grouped into tiles of <= 64 chunks, assigned contiguously to one
  CTA per SM balanced by entries;
* pieces: a worker's run of one output row inside its chunk. Piece ids are
  stream-ordered; the fold adds the pieces of each row in that order.
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib

NUM_SMS = 148


def workers(k: int) -> int:
    """8-lane workers per CTA for width k = chunks per tile (csrc/staged.cu)."""
    return int(_lib.lib().mfg_staged_workers(int(k)))


def block_rows(k: int) -> int:
    """Rows of one staged block for width k (0: unsupported)."""
    return int(_lib.lib().mfg_staged_block_rows(int(k)))


def _pack_bits(flags: torch.Tensor) -> torch.Tensor:
    """bool [32 w] -> int32 [w] with bit l of word i = flags[32 i + l]."""
    w = flags.view(-1, 32).to(torch.int64)
    shifts = torch.arange(32, device=flags.device, dtype=torch.int64)
    words = (w << shifts).sum(1)
    words = torch.where(words >= 2 ** 31, words - 2 ** 32, words)
    return words.to(torch.int32)


class _PassPlan:
    """Streams of one orientation (see the module docstring)."""

    def __init__(self, idx, rows, vals, nrows, ngath, S, lmin, want_pos, stage_min=4.0,
                 l1=False):
        dev = idx.device
        nnz = int(idx.numel())
        self.nrows, self.ngath, self.S = int(nrows), int(ngath), int(S)
        i64 = torch.int64
        idx64 = idx.to(i64)
        rows64 = rows.to(i64)
        deg = torch.bincount(idx64, minlength=ngath)
        order = torch.sort(-deg, stable=True).indices            # gathered rows by degree
        rank = torch.empty_like(order)
        rank[order] = torch.arange(ngath, device=dev, dtype=i64)
        nb_all = max(1, -(-ngath // S))
        blk = rank // S
        eb = blk[idx64]
        # entries per (block, output row) pair: only pairs with >= lmin
        # entries are staged (a piece shorter than that costs a self-row read
        # and a piece write+fold read per few gathers saved); a block is
        # staged when such entries amortise its S staged rows stage_min times
        key = eb * max(nrows, 1) + rows64
        _, inv, cnt = torch.unique(key, return_inverse=True, return_counts=True)
        longp = cnt[inv] >= lmin
        ent_long = torch.bincount(eb[longp], minlength=nb_all)
        stg = ent_long >= max(1.0, stage_min * S)
        nst = int(stg.sum().item())
        self.nblocks = nst
        seg_of_block = torch.where(stg, torch.cumsum(stg.to(i64), 0) - 1,
                                   torch.full_like(ent_long, nst))
        seg = torch.where(longp & stg[eb], seg_of_block[eb], torch.full_like(eb, nst))
        staged = nst
        perm = torch.sort(seg, stable=True).indices               # (row, col) order kept per segment
        seg_s = seg[perm]
        nseg = staged + 1
        cnt = torch.bincount(seg, minlength=nseg)
        aligned = (cnt + 31) // 32 * 32
        start = torch.cumsum(aligned, 0) - aligned
        first = torch.cumsum(cnt, 0) - cnt
        self.nstream = int(aligned.sum().item())
        within = torch.arange(nnz, device=dev, dtype=i64) - first[seg_s]
        at = start[seg_s] + within                                  # stream position of sorted entries
        L_ = self.nstream + 64
        gcol = idx64[perm]
        slot = gcol if l1 else torch.where(seg_s < staged, rank[gcol] % S, gcol)
        self.l1 = l1
        self.sidx = torch.zeros(L_, dtype=torch.int32, device=dev)
        self.srow = torch.zeros(L_, dtype=torch.int32, device=dev)
        self.svals = torch.zeros(L_, dtype=torch.float32, device=dev)
        self.sidx[at] = slot.to(torch.int32)
        rs = rows64[perm]
        self.srow[at] = rs.to(torch.int32)
        self.svals[at] = vals[:nnz][perm].to(torch.float32)
        self.spos = None
        if want_pos:
            self.spos = torch.zeros(L_, dtype=torch.int32, device=dev)
            self.spos[at] = perm.to(torch.int32)
        # row starts (bit per stream entry)
        chg = torch.ones(nnz, dtype=torch.bool, device=dev)
        if nnz > 1:
            chg[1:] = (rs[1:] != rs[:-1]) | (seg_s[1:] != seg_s[:-1])
        flags = torch.zeros(self.nstream + 32 * 2, dtype=torch.bool, device=dev)
        flags[at] = chg
        nwords = self.nstream // 32 + 2
        self.bmask = _pack_bits(flags[: nwords * 32])
        self._flags = flags
        # slot s of staged segment j holds gathered row order[b_j * S + s]
        padded = torch.zeros(nb_all * S, dtype=torch.int32, device=dev)
        padded[:ngath] = order.to(torch.int32)
        sb = torch.nonzero(stg, as_tuple=False).flatten()
        self.members = (padded.view(nb_all, S)[sb].reshape(-1) if nst else
                        torch.zeros(S, dtype=torch.int32, device=dev)).contiguous()
        self.seg_counts = cnt.cpu().tolist()
        self.seg_starts = start.cpu().tolist()
        self.entries_staged = int(cnt[:staged].sum().item())
        self.nnz = nnz

    def chunk(self, te: int, groups: int):
        """Chunks and tiles of this pass for target tile size te (entries)."""
        chunks, tiles = [], []
        for s, (n, e0) in enumerate(zip(self.seg_counts, self.seg_starts)):
            if n == 0:
                continue
            block = s if (s < self.nblocks and not self.l1) else -1
            t = max(1, round(n / te))
            per = -(-n // (groups * t))
            cb = max(32, -(-per // 32) * 32)
            nch = -(-n // cb)
            for c0 in range(0, nch, groups):
                c1 = min(nch, c0 + groups)
                tiles.append((block, len(chunks), len(chunks) + (c1 - c0), cb // 32,
                              min(n, c1 * cb) - c0 * cb))
                for c in range(c0, c1):
                    chunks.append((e0 + c * cb, e0 + min(n, (c + 1) * cb)))
        return chunks, tiles

    def pieces(self, chunks):
        """Piece ids: stream-ordered runs of one output row inside a chunk."""
        dev = self.sidx.device
        ps = self._flags.clone()
        if chunks:
            e0 = torch.tensor([c[0] for c in chunks], dtype=torch.int64, device=dev)
            ps[e0] = True
        cum = torch.cumsum(ps.to(torch.int64), 0)
        npieces = int(cum[-1].item()) if cum.numel() else 0
        piece0 = (cum[e0] - 1) if chunks else torch.zeros(0, dtype=torch.int64, device=dev)
        pos = torch.nonzero(ps[: self.nstream], as_tuple=False).flatten()
        prow = self.srow[pos].to(torch.int64)
        self.prow = torch.zeros(prow.numel() + 3, dtype=torch.int32, device=dev)
        self.prow[: prow.numel()] = prow.to(torch.int32)
        self.plist = torch.sort(prow, stable=True).indices.to(torch.int32)
        cnt = torch.bincount(prow, minlength=self.nrows)
        self.pptr = torch.zeros(self.nrows + 1, dtype=torch.int32, device=dev)
        self.pptr[1:] = torch.cumsum(cnt, 0).to(torch.int32)
        self.npieces = npieces
        if self.plist.numel() == 0:
            self.plist = torch.zeros(1, dtype=torch.int32, device=dev)
        return piece0

    def cstruct(self):
        return _lib.StagedPass(self.nrows, self.S, self.nstream, self.sidx.data_ptr(),
                               self.srow.data_ptr(), self.prow.data_ptr(), self.svals.data_ptr(),
                               _lib.ptr(self.spos) or 0, self.bmask.data_ptr(),
                               self.members.data_ptr(), self.nblocks, self.npieces,
                               self.pptr.data_ptr(), self.plist.data_ptr())


class StagedInput:
    """The arrays a plan is built from: both orientations of Omega (entry
    order of the layouts) and the fp32 values in each order."""

    def __init__(self, m, n, csr_idx, csr_row, vals, csc_idx, csc_row, vals_csc):
        self.m, self.n = int(m), int(n)
        self.nnz = int(csr_idx.numel())
        self.csr_idx, self.csr_row, self.vals = csr_idx, csr_row, vals[: self.nnz]
        self.csc_idx, self.csc_row, self.vals_csc = csc_idx, csc_row, vals_csc[: self.nnz]
        self.device = csr_idx.device

    @classmethod
    def of(cls, obs) -> "StagedInput":
        d = obs.dev
        nnz = obs.size
        return cls(obs.m, obs.n, d.csr.idx[:nnz], d.csr.row_of[:nnz], d.vals, d.csc.idx[:nnz],
                   d.csc.row_of[:nnz], d.vals_csc)


class StagedPlan:
    """Staged-sweep plan of one ObservationSet at width k (fp32 storage).

    ``S`` overrides the block rows (<= block_rows(k); tests use small blocks
    to exercise many blocks and cold segments); ``lmin`` is the staging
    threshold in entries per (output row, block) pair; ``tiles_per_cta``
    sets the balancing granularity."""

    def __init__(self, obs, k: int, *, S: int | None = None, lmin: float = 8.0,
                 stage_min: float = 4.0, grid: int = NUM_SMS, tiles_per_cta: int = 4,
                 want_r: bool = True, l1_bytes: int = 0):
        src = obs if isinstance(obs, StagedInput) else StagedInput.of(obs)
        if src.vals.dtype != torch.float32:
            raise ValueError("the staged sweep runs on fp32 storage")
        if src.nnz == 0:
            raise ValueError("the staged sweep needs a nonempty Omega (use mfg_sweep)")
        smax = block_rows(k)
        if smax <= 0:
            raise ValueError(f"the staged sweep supports 1 <= k <= 64 (got {k})")
        # l1_bytes > 0: "L1-blocked" mode -- the same block-ordered stream, but
        # nothing is staged: tiles of one block run back to back on an SM and
        # its L1 caches the block's rows (gathers stay global loads)
        l1 = l1_bytes > 0
        if l1:
            S = max(1, int(l1_bytes) // (((int(k) * 4 + 15) // 16) * 16)) if S is None else int(S)
        else:
            S = smax if S is None else int(S)
            if not 1 <= S <= smax:
                raise ValueError(f"block rows must be in [1, {smax}]")
        self.l1 = l1
        self.k, self.S, self.grid = int(k), S, int(grid)
        self.m, self.n = src.m, src.n
        nnz = src.nnz
        self.p = [
            _PassPlan(src.csr_idx, src.csr_row, src.vals, src.m, src.n, S, lmin, want_r, stage_min, l1),
            _PassPlan(src.csc_idx, src.csc_row, src.vals_csc, src.n, src.m, S, lmin, False, stage_min,
                      l1),
        ]
        total = 2 * nnz
        self.groups = G = workers(k)
        te = max(32 * G // 4, -(-total // (self.grid * max(1, tiles_per_cta))))
        chunks, tiles, nblk, costs = [], [], [], []
        for pi, pp in enumerate(self.p):
            ch, tl = pp.chunk(te, G)
            piece0 = pp.pieces(ch).cpu().tolist()
            base = len(chunks)
            for c, (e0, e1) in enumerate(ch):
                chunks.append((e0, e1, piece0[c], pi))
            for (block, c0, c1, nb, entries) in tl:
                tiles.append((pi, block, base + c0, base + c1))
                nblk.append(nb)
                costs.append(nb * 32 * min(1.0, (c1 - c0) / G) + 16.0)
        i32 = dict(dtype=torch.int32, device=src.device)
        self.chunks = torch.tensor(chunks or [(0, 0, 0, 0)], **i32).contiguous()
        self.tiles = torch.tensor(tiles or [(0, -1, 0, 0)], **i32).contiguous()
        self.tile_nblk = torch.tensor(nblk or [0], **i32)
        self.ntiles = len(tiles)
        self.costs = costs
        self.c = _lib.StagedPlanC((_lib.StagedPass * 2)(self.p[0].cstruct(), self.p[1].cstruct()),
                                  self.k, self.grid, len(chunks), len(tiles),
                                  self.chunks.data_ptr(), self.tiles.data_ptr(),
                                  self.tile_nblk.data_ptr(), 1 if self.l1 else 0)

    @property
    def ref(self):
        return ctypes.byref(self.c)

    def stats(self) -> dict:
        return {
            "S": self.S,
            "blocks": [pp.nblocks for pp in self.p],
            "staged_frac": [pp.entries_staged / max(pp.nnz, 1) for pp in self.p],
            "pieces": [pp.npieces for pp in self.p],
            "tiles": self.ntiles,
            "mode": "l1-blocked" if self.l1 else "smem-staged",
        }

    def workspace_bytes(self) -> int:
        return int(_lib.lib().mfg_sweep_staged_workspace(self.ref))

