"""Hybrid Omega sweep: hot entries from shared-memory panels, cold entries
through the gather kernel (csrc/panel.cu, csrc/sweep.cu).

The sweep computes R = W H^T - A on Omega, R.H, R^T.W and the fp64 sums
(mfg/data.py:253-293, mfg/operators.py:108,117). ``HybridSweepPlan`` has the
interface of ``mfsolver.SweepPlan`` (``run(w, h)`` -> ``R``, ``RH``, ``RtW``,
``sums``) and splits each pass's entries once per Omega and k:

* an entry is *hot* when its gathered factor row is among the most gathered
  rows (rank < n_panels * panel_rows) and the run of its self row inside its
  panel (a *piece*) has at least ``lmin`` entries; hot entries are reordered
  by (panel, self row) and walked by ``k_panel`` from shared memory;
* the remaining *cold* entries keep their order in two sub-layouts (CSR of
  the CSR pass's cold entries, CSC of the CSC pass's) and run through the
  grouped gather kernel (``mfg_sweep_sharded``);
* ``mfg_panel_fold`` adds the piece outputs to the cold part in a fixed
  order, and one gather puts R back in CSR order.

The layout build below is device-side sort/scan plumbing in torch (run once
per Omega); the arithmetic of every sweep is in libmfg_b200.
"""

from __future__ import annotations

import ctypes
import math
import os

import torch

from . import _lib
from .data import OMEGA_PAD, ObservationSet, _LayoutBuffers, _padded


def panel_ld(k: int, dtype) -> int:
    """Factor row stride the panel kernel takes for width k (0: unsupported)."""
    if dtype != torch.float32:
        return 0
    from .mfsolver import grouped_ld

    ld = grouped_ld(int(k), dtype) or 0
    return ld if ld and _lib.lib().mfg_panel_rows(ld) > 0 else 0


def _chunk_rows(n: int, nchunks: int, rho: float) -> list:
    """Boundaries of nchunks contiguous row ranges of n rows whose sizes shrink
    geometrically (ratio rho): the last chunk's work is not hidden behind a
    transfer, so it is the smallest."""
    nchunks = max(1, min(int(nchunks), max(n, 1)))
    wts = [rho ** c for c in range(nchunks)]
    acc, tot, out = 0.0, sum(wts), [0]
    for c in range(nchunks):
        acc += wts[c]
        out.append(n if c == nchunks - 1 else max(out[-1], min(n, int(round(n * acc / tot)))))
    return out


def _cut(lens, prow, ppan, lmax, dev):
    """Cut pieces into sub-pieces of at most lmax entries (balanced lengths).
    Returns (srow, span, slen, cstart): self row, panel, length and first
    compact entry of every sub-piece, in piece order."""
    npieces = int(lens.numel())
    nsub = (lens + lmax - 1) // lmax
    pid = torch.repeat_interleave(torch.arange(npieces, device=dev), nsub)
    ns = int(pid.numel())
    first_sub = torch.cumsum(nsub, 0) - nsub
    j = torch.arange(ns, device=dev) - first_sub[pid]
    base = lens[pid] // nsub[pid]
    rem = lens[pid] % nsub[pid]
    slen = base + (j < rem).long()
    cstart_piece = torch.cumsum(lens, 0) - lens          # compact start of each piece
    cstart = cstart_piece[pid] + j * base + torch.minimum(j, rem)
    return prow[pid], ppan[pid], slen, cstart


class _PanelPass:
    """One pass's layout (device arrays): the hot pieces of the panels with
    their ctypes ``mfg_panel_pass`` (``c``), and -- with ``cold_pieces`` --
    the cold entries cut into pieces for ``mfg_cold_sweep`` (``cc``)."""

    def __init__(self, lay: _LayoutBuffers, vals: torch.Tensor, n_self: int, n_gath: int, PR: int,
                 ld: int, pass_id: int, *, lmin: int, lmax: int,
                 max_panels: int, min_panel_entries: int, want_r: bool, want_sq: bool,
                 cold_pieces: bool = False, direct: bool = False, chunk_rows=None,
                 chunk_by: str = "self"):
        """``chunk_rows``: boundaries [0, .., n] of contiguous row ranges of one
        factor (the end-to-end path moves that factor chunk by chunk).
        ``chunk_by`` = "self": they cut this pass's self rows (the CSC pass and
        H): every list element, cold piece and fold range lies in one chunk.
        "gath": they cut the gathered table (the CSR pass and H): panels hold
        rows of one chunk and a cold piece gathers from one chunk, so the work
        that needs chunk c only needs chunk c."""
        dev = vals.device
        if chunk_rows is None or len(chunk_rows) < 3:
            chunk_rows = [0, n_self if chunk_by == "self" else n_gath]
        nchunks = len(chunk_rows) - 1
        self.nchunks = nchunks
        self.chunk_rows = list(chunk_rows)
        self.chunk_by = chunk_by
        bounds = torch.tensor(self.chunk_rows[1:], device=dev)

        def chunk_of(rows_t):
            return torch.bucketize(rows_t, bounds, right=True).clamp_(max=nchunks - 1)

        nnz = lay.nnz
        idx = lay.idx[:nnz].long()
        row_of = lay.row_of[:nnz].long()
        cnt = torch.bincount(idx, minlength=n_gath)
        # panels: gathered rows by decreasing gather count -- inside their chunk
        # when the gathered table is chunked -- PR rows per panel
        allg = torch.arange(n_gath, device=dev)
        gch = chunk_of(allg) if chunk_by == "gath" else torch.zeros(n_gath, dtype=torch.long, device=dev)
        ngc = nchunks if chunk_by == "gath" else 1
        cmax = int(cnt.max().item()) if n_gath else 0
        order = torch.argsort(gch * (cmax + 1) + (cmax - cnt), stable=True)
        gsize = torch.bincount(gch, minlength=ngc)
        gstart0 = torch.cumsum(gsize, 0) - gsize
        rank_in = torch.empty_like(order)
        rank_in[order] = allg - gstart0[gch[order]]
        del cnt
        sizes = gsize.cpu().tolist()
        npc_c = [max(1, min((sz + PR - 1) // PR, max(1, int(round(max_panels * sz / max(n_gath, 1))))))
                 if sz else 0 for sz in sizes]
        pbase = [0]
        for x in npc_c:
            pbase.append(pbase[-1] + x)
        npt = max(pbase[-1], 1)                       # panels over all chunks
        pbase_t = torch.tensor(pbase[:-1], device=dev)
        npc_t = torch.tensor(npc_c, device=dev)
        pan_g = torch.where(rank_in < npc_t[gch] * PR, pbase_t[gch] + rank_in // PR,
                            torch.full_like(rank_in, npt))
        local_g = rank_in % PR
        panel_chunk = torch.repeat_interleave(torch.arange(ngc, device=dev), npc_t) if pbase[-1] else \
            torch.zeros(1, dtype=torch.long, device=dev)
        pan_e = pan_g[idx]
        key = pan_e.to(torch.int16)
        del pan_e
        skey, perm = torch.sort(key, stable=True)
        del key
        nh = int((skey < npt).sum().item())
        perm = perm[:nh]
        pkey = skey[:nh].long()
        del skey
        rows_s = row_of[perm]
        k2 = pkey * n_self + rows_s
        flag = torch.ones(nh, dtype=torch.bool, device=dev)
        if nh > 1:
            flag[1:] = k2[1:] != k2[:-1]
        del k2
        pstart = torch.nonzero(flag).flatten()
        plen = torch.diff(pstart, append=torch.tensor([nh], device=dev))
        ppanel = pkey[pstart]
        keep_piece = plen >= lmin
        ent_panel = torch.zeros(npt, dtype=torch.long, device=dev)
        ent_panel.index_add_(0, ppanel, plen * keep_piece)
        ok_p = ent_panel >= min_panel_entries       # panels worth loading
        keep_piece &= ok_p[ppanel]
        piece_id = torch.cumsum(flag, 0) - 1
        keep_e = keep_piece[piece_id] if nh else flag
        del piece_id, flag
        hot_orig = perm[keep_e]                 # original positions, (panel, row, order)
        del perm, keep_e, pkey
        npk = npt
        self.n_panels = int(ok_p.sum().item())
        self.n_hot = int(hot_orig.numel())
        cold = torch.ones(nnz, dtype=torch.bool, device=dev)
        cold[hot_orig] = False
        self.cold_mask = cold
        # kept pieces -> sub-pieces of at most lmax entries
        srow, span, slen, cstart = _cut(plen[keep_piece], rows_s[pstart][keep_piece],
                                        ppanel[keep_piece], lmax, dev)
        del rows_s, pstart, plen, ppanel, keep_piece
        ns = int(srow.numel())
        nblk = (slen + 15) // 16                             # record blocks of each sub-piece
        bstart = torch.cumsum(nblk, 0) - nblk                # first block of each sub-piece
        n_blocks = int(nblk.sum().item()) if ns else 0
        self.n_blocks = n_blocks
        # records. Inside a sub-piece the entries are ordered so that the 4
        # entries of a batch fall into different 32-byte bank windows of the
        # panel's tail array (window = local row mod 4) where the piece allows:
        # the t-th entry of each window, for t = 0, 1, ...
        sub_of_e = torch.repeat_interleave(torch.arange(ns, device=dev), slen)
        local = local_g[idx[hot_orig]]
        if self.n_hot:
            key1 = sub_of_e * 4 + (local % 4)
            o1 = torch.argsort(key1, stable=True)
            k1s = key1[o1]
            f1 = torch.ones(self.n_hot, dtype=torch.bool, device=dev)
            f1[1:] = k1s[1:] != k1s[:-1]
            ar = torch.arange(self.n_hot, device=dev)
            gstart = torch.cummax(torch.where(f1, ar, torch.zeros_like(ar)), 0).values
            key2 = sub_of_e[o1] * 2048 + (ar - gstart) * 4 + (k1s % 4)
            del k1s, f1, gstart, key1
            o2 = torch.argsort(key2)
            del key2
            o12 = o1[o2]
            del o1, o2
            hot_orig = hot_orig[o12]
            local = local[o12]
            del o12
        ar = torch.arange(self.n_hot, device=dev)
        ppos = bstart[sub_of_e] * 16 + (ar - cstart[sub_of_e])   # record position
        del sub_of_e, ar
        recs = torch.zeros((n_blocks + 2, 24), dtype=torch.int32, device=dev)
        if self.n_hot:
            blk, off = ppos // 16, ppos % 16
            recs.view(torch.int16).view(n_blocks + 2, 48)[blk, off] = local.to(torch.int16)
            recs[blk, 8 + off] = vals[:nnz][hot_orig].contiguous().view(torch.int32)
            del blk, off
        self.recs = recs
        self.hot_orig = hot_orig
        self.hot_pos = ppos
        # panel row ids
        ids = torch.full((max(npk, 1) * PR,), -1, dtype=torch.int32, device=dev)
        hot_g = torch.nonzero(pan_g < npt).flatten()
        ids[pan_g[hot_g] * PR + local_g[hot_g]] = hot_g.to(torch.int32)
        self.panel_ids = ids
        del order, local, hot_g
        # cold pieces: a self row's cold entries in their order, cut at lmax;
        # record blocks of 16 x u32 gathered-row ids + 16 x f32 values
        nsc = 0
        if cold_pieces:
            cold_orig = torch.nonzero(cold).flatten()
            ncold = int(cold_orig.numel())
            crow = row_of[cold_orig]
            if chunk_by == "gath" and nchunks > 1:
                # a cold piece gathers from one chunk: entries by (chunk of the
                # gathered row, self row, original order)
                cg = gch[idx[cold_orig]]
                o_g = torch.argsort(cg, stable=True)
                cold_orig, crow, cg = cold_orig[o_g], crow[o_g], cg[o_g]
                ckey = cg * n_self + crow
                del o_g
            else:
                cg = None
                ckey = crow
            fc = torch.ones(ncold, dtype=torch.bool, device=dev)
            if ncold > 1:
                fc[1:] = ckey[1:] != ckey[:-1]
            cps = torch.nonzero(fc).flatten()
            cpl = torch.diff(cps, append=torch.tensor([ncold], device=dev))
            pchunk = cg[cps] if cg is not None else None
            del ckey
            # (the panel slot of a cold sub-piece carries its gathered chunk when there is one)
            srow_c, span_c, slen_c, cstart_c = _cut(cpl, crow[cps], pchunk if pchunk is not None else torch.full_like(cps, npk), lmax, dev)
            nsc = int(srow_c.numel())
            nblk_c = (slen_c + 15) // 16
            bstart_c = torch.cumsum(nblk_c, 0) - nblk_c
            nbc = int(nblk_c.sum().item()) if nsc else 0
            sub_c = torch.repeat_interleave(torch.arange(nsc, device=dev), slen_c)
            cpos = bstart_c[sub_c] * 16 + (torch.arange(ncold, device=dev) - cstart_c[sub_c])
            del sub_c, fc, crow
            crecs = torch.zeros((nbc + 2, 32), dtype=torch.int32, device=dev)
            if ncold:
                blk, off = cpos // 16, cpos % 16
                crecs[blk, off] = idx[cold_orig].to(torch.int32)
                crecs[blk, 16 + off] = vals[:nnz][cold_orig].contiguous().view(torch.int32)
                del blk, off
            self.cold_recs, self.cold_orig, self.cold_pos, self.n_cold_blocks = crecs, cold_orig, cpos, nbc
            srow_all = torch.cat([srow, srow_c])
        else:
            srow_all = srow
        del idx, row_of
        # slots in (self row, panel, run) order; the cold pieces of a row come last
        nsa = ns + nsc
        seq = torch.arange(nsa, device=dev)
        o_rs = torch.argsort(srow_all * max(nsa, 1) + seq)
        slot = torch.empty(nsa, dtype=torch.long, device=dev)
        slot[o_rs] = seq
        frows, counts = torch.unique_consecutive(srow_all[o_rs], return_counts=True)
        fbeg = torch.cumsum(counts, 0) - counts
        direct_c = None
        if cold_pieces and direct and nsc:
            # a self row whose only slot is a cold piece: the piece writes the
            # output row itself (bit 30 of its length) and the row needs no fold
            rowcount = torch.zeros(n_self, dtype=torch.long, device=dev)
            rowcount.index_add_(0, srow_all, torch.ones_like(srow_all))
            direct_c = rowcount[srow_c] == 1
            row_direct = torch.zeros(n_self, dtype=torch.bool, device=dev)
            row_direct[srow_c[direct_c]] = True
            keep_f = ~row_direct[frows]
            frows, counts, fbeg = frows[keep_f], counts[keep_f], fbeg[keep_f]
            del rowcount, row_direct, keep_f
        # light rows (<= 32 slots) first, heavy rows after them
        o_lh = torch.argsort((counts > 32).to(torch.int8), stable=True)
        self.n_light = int((counts <= 32).sum().item()) if counts.numel() else 0
        self.frows = frows[o_lh].to(torch.int32)
        self.fbeg = fbeg[o_lh].to(torch.int32)
        self.fcnt = counts[o_lh].to(torch.int32)
        # piece table: per panel by decreasing length
        echunk = panel_chunk[span.clamp(max=panel_chunk.numel() - 1)] if chunk_by == "gath" else chunk_of(srow)
        span2 = span * nchunks + echunk                     # (panel, chunk)
        o_pl = torch.argsort(span2 * (lmax + 1) + (lmax - slen), stable=True)
        pieces = torch.stack([srow[o_pl], bstart[o_pl], slen[o_pl], slot[:ns][o_pl]], dim=1).to(torch.int32)
        self.pieces = pieces.contiguous() if ns else torch.zeros((1, 4), dtype=torch.int32, device=dev)
        self.n_pieces = ns
        self.n_slots = nsa
        if cold_pieces:
            chunk_c = span_c if pchunk is not None else chunk_of(srow_c)
            o_c = torch.argsort(chunk_c * (lmax + 1) + (lmax - slen_c), stable=True)
            cc_cnt = torch.bincount(chunk_c, minlength=nchunks).cpu().tolist() if nsc else [0] * nchunks
            self.cold_chunk_ptr = [0]
            for x in cc_cnt:
                self.cold_chunk_ptr.append(self.cold_chunk_ptr[-1] + int(x))
            lenf = slen_c if direct_c is None else slen_c + direct_c.long() * (1 << 30)
            self.n_direct = 0 if direct_c is None else int(direct_c.sum().item())
            cp = torch.stack([srow_c[o_c], bstart_c[o_c], lenf[o_c], slot[ns:][o_c]], dim=1).to(torch.int32)
            self.cold_pieces = cp.contiguous() if nsc else torch.zeros((1, 4), dtype=torch.int32, device=dev)
            self.n_cold_pieces = nsc
        # panel list: {pass, panel, first piece, end piece}, one element per
        # (panel, chunk), + entries and chunk of each element
        span_s = span2[o_pl]
        if ns:
            f3 = torch.ones(ns, dtype=torch.bool, device=dev)
            f3[1:] = span_s[1:] != span_s[:-1]
            ist = torch.nonzero(f3).flatten()
            iend = torch.cat([ist[1:], torch.tensor([ns], device=dev)])
            self.plist = torch.stack([torch.full_like(ist, pass_id), span_s[ist] // nchunks, ist, iend],
                                     dim=1).to(torch.int32)
            cum = torch.cat([torch.zeros(1, dtype=torch.long, device=dev), torch.cumsum(slen[o_pl], 0)])
            self.plist_entries = (cum[iend] - cum[ist]).cpu()
            self.plist_chunk = (span_s[ist] % nchunks).cpu()
        else:
            self.plist = torch.zeros((0, 4), dtype=torch.int32, device=dev)
            self.plist_entries = torch.zeros(0, dtype=torch.long)
            self.plist_chunk = torch.zeros(0, dtype=torch.long)
        # fold lists per chunk (light rows, then heavy rows, inside each chunk)
        if nchunks > 1 and chunk_by == "self":
            fch = chunk_of(frows)
            o_cf = torch.argsort(fch * 2 + (counts > 32).long(), stable=True)
            self.cf_rows = frows[o_cf].to(torch.int32)
            self.cf_beg = fbeg[o_cf].to(torch.int32)
            self.cf_cnt = counts[o_cf].to(torch.int32)
            nr = torch.bincount(fch, minlength=nchunks).cpu().tolist() if frows.numel() else [0] * nchunks
            nlt = (torch.bincount(fch[counts <= 32], minlength=nchunks).cpu().tolist()
                   if frows.numel() else [0] * nchunks)
            self.cf_info, off = [], 0
            for c in range(nchunks):
                self.cf_info.append((off, int(nr[c]), int(nlt[c])))
                off += int(nr[c])
        # outputs / scratch (slots are shared by the hot and the cold pieces)
        self.r_hot = torch.zeros((n_blocks + 2) * 16, dtype=torch.float32, device=dev) if want_r else None
        self.piece_out = torch.empty((max(nsa, 1), ld), dtype=torch.float32, device=dev)
        self.piece_sq = torch.zeros(max(nsa, 1), dtype=torch.float64, device=dev) if want_sq else None
        self.c = _lib.PanelPass(nsa, int(self.frows.numel()), self.n_light, self.panel_ids.data_ptr(),
                                self.pieces.data_ptr(), self.recs.data_ptr(),
                                self.frows.data_ptr(), self.fbeg.data_ptr(), self.fcnt.data_ptr(),
                                _lib.ptr(self.r_hot),
                                self.piece_out.data_ptr(), _lib.ptr(self.piece_sq))
        if cold_pieces:
            self.cc = _lib.PanelPass(nsc, 0, 0, None, self.cold_pieces.data_ptr(),
                                     self.cold_recs.data_ptr(), None, None, None, None,
                                     self.piece_out.data_ptr(), _lib.ptr(self.piece_sq))

    @property
    def ref(self):
        return ctypes.byref(self.c)

    @property
    def cold_ref(self):
        return ctypes.byref(self.cc)

    def chunk_structs(self):
        """Per chunk: (fold struct, cold-piece struct) -- copies of ``c`` / ``cc``
        restricted to the chunk's self rows."""
        out = []
        for c in range(self.nchunks):
            f = _lib.PanelPass.from_buffer_copy(self.c)
            if self.chunk_by == "self":
                off, nr, nlt = self.cf_info[c]
                f.n_frows, f.n_light = nr, nlt
                f.frows = self.cf_rows.data_ptr() + 4 * off
                f.fbeg = self.cf_beg.data_ptr() + 4 * off
                f.fcnt = self.cf_cnt.data_ptr() + 4 * off
            g = _lib.PanelPass.from_buffer_copy(self.cc)
            c0, c1 = self.cold_chunk_ptr[c], self.cold_chunk_ptr[c + 1]
            g.n_pieces = c1 - c0
            g.pieces = self.cold_pieces.data_ptr() + 16 * c0
            out.append((f, g))
        return out


def _cold_layout(lay: _LayoutBuffers, vals: torch.Tensor, cold: torch.Tensor):
    """Sub-layout of the cold entries (their order kept) + their values."""
    nnz = lay.nnz
    dev = vals.device
    idx = lay.idx[:nnz][cold]
    row_of = lay.row_of[:nnz][cold]
    nc = int(idx.numel())
    cidx = _padded(nc, torch.int32, dev)
    cidx.copy_(idx)
    crow = _padded(nc, torch.int32, dev)
    crow.copy_(row_of)
    cvals = _padded(nc, vals.dtype, dev)
    cvals.copy_(vals[:nnz][cold])
    ptr = torch.zeros(lay.nrows + 1, dtype=torch.int32, device=dev)
    if nc:
        ptr[1:] = torch.cumsum(torch.bincount(row_of.long(), minlength=lay.nrows), 0).to(torch.int32)
    return _LayoutBuffers(lay.nrows, lay.ncols, nc, ptr, cidx, crow), cvals


class HybridSweepPlan:
    """The Omega sweep with hot entries from shared-memory panels.

    Same outputs as ``mfsolver.SweepPlan``: ``R`` (CSR order), ``RH``, ``RtW``
    and ``sums`` = [sum r^2, ||W||^2, ||H||^2] (fp64). ``run(w, h)`` takes the
    factors with row stride ``ld`` (``pad``). fp32 storage only."""

    def __init__(self, obs: ObservationSet, k: int, *, want_r: bool = True, out_scale: float = 1.0,
                 lmin: int | None = None, lmax: int | None = None,
                 max_panels: int | None = None, min_panel_entries: int | None = None,
                 cold: str | None = None):
        if obs.dtype != torch.float32:
            raise ValueError("HybridSweepPlan: fp32 storage only")
        self.obs, self.k = obs, int(k)
        self.dt = obs.dtype
        self.ld = panel_ld(self.k, obs.dtype)
        if not self.ld:
            raise ValueError(f"HybridSweepPlan: unsupported factor width k={k}")
        env = os.environ.get
        lmin = int(env("MFG_PANEL_LMIN", 16)) if lmin is None else lmin
        lmax = int(env("MFG_PANEL_LMAX", 256)) if lmax is None else lmax
        max_panels = int(env("MFG_PANEL_MAXP", 32)) if max_panels is None else max_panels
        if min_panel_entries is None:
            min_panel_entries = int(env("MFG_PANEL_MINE", min(100_000, max(1, obs.size // 256))))
        lib = _lib.lib()
        dev = obs.dev
        self.PR = lib.mfg_panel_rows(self.ld)
        self.out_scale = float(out_scale)
        if lmax > 511:
            raise ValueError("HybridSweepPlan: lmax must be <= 511")
        # cold entries: "pieces" walks them like panel pieces on global loads
        # (k_cold4; rows of one 32-dim block), "gather" runs the grouped gather
        # kernel on their sub-layouts
        cold = cold or env("MFG_PANEL_COLD", "pieces")
        if cold not in ("pieces", "gather"):
            raise ValueError("cold must be 'pieces' or 'gather'")
        if self.ld == 64:
            cold = "gather"
        self.cold = cold
        lean = cold == "pieces"
        kw = dict(lmin=lmin, lmax=lmax, max_panels=max_panels, min_panel_entries=min_panel_entries,
                  cold_pieces=lean, direct=lean and self.ld == self.k)
        # H in column chunks (cold="pieces" plans): the end-to-end path moves H, runs
        # the work that needs a chunk and returns R^T.W chunk by chunk. The CSC pass
        # is cut by its self rows, the CSR pass by the rows it gathers.
        self.nchunks = int(env("MFG_PANEL_CHUNKS", 4)) if lean else 1
        # relative chunk sizes: a small first chunk (the first work starts early), a
        # small last one (its R^T.W rows return after the last fold); the kernels,
        # not the transfers, bound the step, so the chunks in between are large
        sizes = env("MFG_PANEL_CHUNK_SIZES", "5,15,25,25,20,10" if "MFG_PANEL_CHUNKS" not in os.environ else "")
        if sizes and lean:
            wts = [float(x) for x in sizes.split(",")]
            acc, crows = 0.0, [0]
            for i, x in enumerate(wts):
                acc += x
                crows.append(obs.n if i == len(wts) - 1 else
                             max(crows[-1], min(obs.n, int(round(obs.n * acc / sum(wts))))))
        else:
            crows = _chunk_rows(obs.n, self.nchunks, float(env("MFG_PANEL_CHUNK_RATIO", 0.7)))
        self.nchunks = len(crows) - 1
        self.p0 = _PanelPass(dev.csr, dev.vals, obs.m, obs.n, self.PR, self.ld, 0, want_r=False,
                             want_sq=True, chunk_rows=crows, chunk_by="gath", **kw)
        self.p1 = _PanelPass(dev.csc, dev.vals_csc, obs.n, obs.m, self.PR, self.ld, 1,
                             want_r=False, want_sq=False, chunk_rows=crows, chunk_by="self", **kw)
        # one list over both passes; the CSC pass's piece indices are its own
        self.plist = torch.cat([self.p0.plist, self.p1.plist], 0).contiguous()
        self.n_list = int(self.plist.shape[0])
        ent = torch.cat([self.p0.plist_entries, self.p1.plist_entries]).double()
        nctas = lib.mfg_panel_ctas()
        if self.n_list:
            # CTA c starts at the element holding work offset c / nctas of the total
            edges = torch.cumsum(ent, 0)
            at = (torch.arange(nctas, dtype=torch.float64) + 0.5) * float(edges[-1]) / nctas
            start = torch.searchsorted(edges, at).clamp_(max=self.n_list - 1)
        else:
            self.plist = torch.zeros((1, 4), dtype=torch.int32, device=dev.device)
            start = torch.zeros(nctas, dtype=torch.long)
        self.cta_start = start.to(torch.int32).to(dev.device)
        # per-pass lists for the end-to-end path (CSC pass first, so that the D2H of
        # R^T.W overlaps the CSR pass): their own CTA starts and tickets
        self._pass_lists = []
        for pp in (self.p0, self.p1):
            nl = int(pp.plist.shape[0])
            if nl:
                ed = torch.cumsum(pp.plist_entries.double(), 0)
                at = (torch.arange(nctas, dtype=torch.float64) + 0.5) * float(ed[-1]) / nctas
                cs = torch.searchsorted(ed, at).clamp_(max=nl - 1).to(torch.int32).to(dev.device)
            else:
                cs = torch.zeros(nctas, dtype=torch.int32, device=dev.device)
            self._pass_lists.append((nl, pp.plist.contiguous(), cs,
                                     torch.zeros(nl + 2, dtype=torch.int32, device=dev.device)))
        self._chunk_lists = []
        if lean and self.nchunks > 1:
            for c in range(self.nchunks):
                parts, ents = [], []
                for pp in (self.p0, self.p1):
                    sel = torch.nonzero(pp.plist_chunk == c).flatten()
                    if sel.numel():
                        parts.append(pp.plist[sel.to(dev.device)])
                        ents.append(pp.plist_entries[sel].double())
                nl = int(sum(x.shape[0] for x in parts))
                if nl:
                    pl = torch.cat(parts, 0).contiguous()
                    ed = torch.cumsum(torch.cat(ents), 0)
                    at = (torch.arange(nctas, dtype=torch.float64) + 0.5) * float(ed[-1]) / nctas
                    cs = torch.searchsorted(ed, at).clamp_(max=nl - 1).to(torch.int32).to(dev.device)
                else:
                    pl = torch.zeros((1, 4), dtype=torch.int32, device=dev.device)
                    cs = torch.zeros(nctas, dtype=torch.int32, device=dev.device)
                self._chunk_lists.append((nl, pl, cs, torch.zeros(nl + 2, dtype=torch.int32,
                                                                  device=dev.device)))
        nnz = obs.size
        self.want_r = want_r
        nh_pad = (self.p0.n_blocks + 2) * 16
        if lean:
            ncold_r = (self.p0.n_cold_blocks + 2) * 16
        else:
            self.cold_csr, self.cold_vals = _cold_layout(dev.csr, dev.vals, self.p0.cold_mask)
            self.cold_csc, self.cold_vals_csc = _cold_layout(dev.csc, dev.vals_csc, self.p1.cold_mask)
            ncold_r = self.cold_csr.nnz + OMEGA_PAD
        if want_r:
            # R in CSR order = gather from [hot residuals | cold residuals], both in record order
            self._rcat = torch.zeros(nh_pad + ncold_r, dtype=self.dt, device=dev.device)
            self.p0.r_hot = self._rcat[:nh_pad]
            self.p0.c.r_hot = self.p0.r_hot.data_ptr()
            self._rcold = self._rcat[nh_pad:]
            src = torch.empty(nnz, dtype=torch.int32, device=dev.device)
            src[self.p0.hot_orig] = self.p0.hot_pos.to(torch.int32)
            if lean:
                self.p0.cc.r_hot = self._rcold.data_ptr()
                src[self.p0.cold_orig] = (nh_pad + self.p0.cold_pos).to(torch.int32)
            else:
                cold_pos = torch.nonzero(self.p0.cold_mask).flatten()
                src[cold_pos] = (nh_pad + torch.arange(cold_pos.numel(), device=dev.device)).to(torch.int32)
            self._rsrc = src
            self.R = torch.empty(nnz, dtype=self.dt, device=dev.device)
        else:
            self.R = None
        if lean:
            for p in (self.p0, self.p1):
                del p.cold_orig, p.cold_pos
        for p in (self.p0, self.p1):
            del p.hot_orig, p.hot_pos, p.cold_mask
        es = 4
        nb_rh = obs.m * self.k * es
        nb_rtw = obs.n * self.k * es
        self._out = torch.zeros(32 + nb_rh + nb_rtw, dtype=torch.uint8, device=dev.device)
        self.sums = self._out[:24].view(torch.float64)
        self.RH = self._out[32:32 + nb_rh].view(self.dt).view(obs.m, self.k)
        self.RtW = self._out[32 + nb_rh:].view(self.dt).view(obs.n, self.k)
        if lean:
            self.wsb = 1 << 16        # the two norms (mfg_dot)
            self.cold_counters = torch.zeros(4, dtype=torch.int32, device=dev.device)
            # a pass's cold pieces alone: the other pass's struct with no pieces
            self._no_cold = _lib.PanelPass(0, 0, 0, None, None, None, None, None, None, None, None, None)
        else:
            self.wsb = lib.mfg_sweep_workspace(self.cold_csr.ref, self.cold_csc.ref, self.k)
        self.ws = torch.zeros(self.wsb, dtype=torch.uint8, device=dev.device)
        self.counters = torch.zeros(self.n_list + 2, dtype=torch.int32, device=dev.device)
        self.sq_ws = torch.zeros(1024, dtype=torch.uint8, device=dev.device)
        self._side = torch.cuda.Stream(device=dev.device)
        self._ev_fork = torch.cuda.Event()
        self._ev_join = torch.cuda.Event()
        self._copy = torch.cuda.Stream(device=dev.device)
        self._ev_csc = torch.cuda.Event()
        self._ev_copy = torch.cuda.Event()
        self._cin = torch.cuda.Stream(device=dev.device)
        self._ev_start = torch.cuda.Event()
        self._ev_w = torch.cuda.Event()
        self._ev_h = [torch.cuda.Event() for _ in range(max(self.nchunks, 1) + 16)]
        self._ev_f = [torch.cuda.Event() for _ in range(max(self.nchunks, 1) + 16)]
        if self._chunk_lists:
            self._chunk_structs0 = self.p0.chunk_structs()
            self._chunk_structs1 = self.p1.chunk_structs()
        self.stats = {
            "panel_rows": self.PR, "csr_panels": self.p0.n_panels, "csc_panels": self.p1.n_panels,
            "csr_hot": self.p0.n_hot, "csc_hot": self.p1.n_hot, "nnz": nnz,
            "csr_pieces": self.p0.n_pieces, "csc_pieces": self.p1.n_pieces, "lmax": lmax,
            "cold": ("pieces on global loads (k_cold4)" if lean else "gather kernel (k_sweep_g8f)"),
        }

    def pad(self, f: torch.Tensor) -> torch.Tensor:
        if self.ld == self.k:
            return f.to(self.dt).contiguous()
        out = torch.zeros((f.shape[0], self.ld), dtype=self.dt, device=self.obs.dev.device)
        out[:, : f.shape[1]] = f
        return out

    kind = "hybrid"

    # ---- end to end from host factors (the interface of SweepPlan.run_host) ----
    def pinned_factors(self):
        """Pinned host buffers (W: m x k, H: n x k), adjacent in one allocation."""
        whh = torch.zeros((self.obs.m + self.obs.n) * self.k, dtype=self.dt).pin_memory()
        return (whh[: self.obs.m * self.k].view(self.obs.m, self.k),
                whh[self.obs.m * self.k:].view(self.obs.n, self.k))

    def run_host(self, w_host: torch.Tensor, h_host: torch.Tensor, *, graph: bool = True):
        """H2D of the host factors into resident device factors, the sweep, and
        one D2H of the packed results [sums | RH | RtW]; returns pinned host
        views (sums, RH, RtW), valid once the current stream reaches this
        point. With ``graph`` the sequence is captured once per (host buffers,
        stream) as a CUDA graph and replayed."""
        for t, rows in ((w_host, self.obs.m), (h_host, self.obs.n)):
            if t.device.type != "cpu" or t.dtype != self.dt or tuple(t.shape) != (rows, self.k) \
                    or not t.is_contiguous():
                raise ValueError(f"host factor must be a contiguous CPU ({rows} x {self.k}) {self.dt} tensor")
        m, n, k, ld = self.obs.m, self.obs.n, self.k, self.ld
        if getattr(self, "_host", None) is None:
            dev = self.obs.dev.device
            self._whd = torch.zeros((m + n) * ld, dtype=self.dt, device=dev)
            self._wd = self._whd[: m * ld].view(m, ld)
            self._hd = self._whd[m * ld:].view(n, ld)
            self._host = torch.empty(self._out.numel(), dtype=torch.uint8).pin_memory()
            nb_rh = self.RH.numel() * 4
            self._host_views = (self._host[:24].view(torch.float64),
                                self._host[32:32 + nb_rh].view(self.dt).view(m, k),
                                self._host[32 + nb_rh:].view(self.dt).view(n, k))
            self._graph_key = None
        stream = torch.cuda.current_stream()
        if not graph or getattr(self, "_no_graph", False):
            self._host_call(w_host, h_host)
            return self._host_views
        key = (w_host.data_ptr(), h_host.data_ptr(), stream.cuda_stream)
        if self._graph_key != key:
            self._host_call(w_host, h_host)          # warm-up, eager
            torch.cuda.synchronize()
            side = torch.cuda.Stream()
            side.wait_stream(stream)
            g = torch.cuda.CUDAGraph()
            try:
                with torch.cuda.graph(g, stream=side, capture_error_mode="thread_local"):
                    self._host_call(w_host, h_host)
            except RuntimeError:
                torch.cuda.synchronize()
                self._no_graph = True
                return self._host_views
            stream.wait_stream(side)
            self._graph, self._graph_key = g, key
        self._graph.replay()
        return self._host_views

    def _host_call(self, w_host, h_host):
        m, n, k, ld = self.obs.m, self.obs.n, self.k, self.ld
        if self.cold == "pieces" and self._chunk_lists:
            self._host_call_chunked(w_host, h_host)
            return
        adjacent = (ld == k and h_host.data_ptr() == w_host.data_ptr() + m * k * 4
                    and w_host.untyped_storage().data_ptr() == h_host.untyped_storage().data_ptr())
        if adjacent:
            flat = torch.as_strided(w_host, ((m + n) * k,), (1,))
            self._whd.copy_(flat, non_blocking=True)
        else:
            self._wd[:, :k].copy_(w_host, non_blocking=True)
            self._hd[:, :k].copy_(h_host, non_blocking=True)
        cur = torch.cuda.current_stream()
        if self.cold == "pieces":
            # CSC pass first: the D2H of R^T.W (the large output) runs on a copy
            # stream while the CSR pass computes
            self._enqueue_pass(self._wd, self._hd, 1)
            nb_head = 32 + self.RH.numel() * 4
            self._ev_csc.record(cur)
            self._copy.wait_event(self._ev_csc)
            with torch.cuda.stream(self._copy):
                self._host[nb_head:].copy_(self._out[nb_head:], non_blocking=True)
                self._ev_copy.record(self._copy)
            pending = self._enqueue_pass(self._wd, self._hd, 0)
            self._host[:nb_head].copy_(self._out[:nb_head], non_blocking=True)
            if pending:
                cur.wait_event(self._ev_join)
            cur.wait_event(self._ev_copy)
            return
        # the D2H of [sums | RH | RtW] does not wait for R (side stream)
        pending = self._enqueue(self._wd, self._hd)
        self._host.copy_(self._out, non_blocking=True)
        if pending:
            cur.wait_event(self._ev_join)

    def _host_call_chunked(self, w_host, h_host):
        """The end-to-end step as a pipeline over chunks of H (contiguous row
        ranges): W, then H chunk by chunk, move to the device on a copy-in
        stream. As soon as chunk c has arrived, the work that needs it runs: the
        CSC pass on the chunk's columns (their rows of R^T.W are folded and
        return on a copy-out stream) and the CSR pass's pieces that gather from
        the chunk (panels hold rows of one chunk; cold pieces gather from one
        chunk). The CSR fold, sum r^2, the norms, the R gather and
        [sums | R.H] follow the last chunk."""
        lib = _lib.lib()
        m, n, k, ld = self.obs.m, self.obs.n, self.k, self.ld
        cur = torch.cuda.current_stream()
        cin, cout = self._cin, self._copy
        nc = self.nchunks
        cr = self.p1.chunk_rows
        self._ev_start.record(cur)
        cin.wait_event(self._ev_start)
        cout.wait_event(self._ev_start)
        with torch.cuda.stream(cin):
            self._wd[:, :k].copy_(w_host, non_blocking=True)
            self._ev_w.record(cin)
            for c in range(nc):
                self._hd[cr[c]:cr[c + 1], :k].copy_(h_host[cr[c]:cr[c + 1]], non_blocking=True)
                self._ev_h[c].record(cin)
        cur.wait_event(self._ev_w)
        st = cur.cuda_stream
        nb_head = 32 + self.RH.numel() * 4
        self.sums[0:1].zero_()
        _lib.check(lib.mfg_dot(_lib.MFG_F32, m * ld, self._wd.data_ptr(), self._wd.data_ptr(),
                               self.sums.data_ptr() + 8, self.ws.data_ptr(), self.wsb, st), "norm")
        for c in range(nc):
            cur.wait_event(self._ev_h[c])
            cold0 = self._chunk_structs0[c][1]
            fold1, cold1 = self._chunk_structs1[c]
            _lib.check(lib.mfg_cold_sweep(ld, ctypes.byref(cold0), ctypes.byref(cold1),
                                          self._wd.data_ptr(), self._hd.data_ptr(), self.RH.data_ptr(),
                                          self.RtW.data_ptr(), self.out_scale,
                                          self.cold_counters.data_ptr(), st), "cold sweep")
            nl, plist, cs, cnt = self._chunk_lists[c]
            if nl:
                _lib.check(lib.mfg_panel_sweep(ld, nl, plist.data_ptr(), cs.data_ptr(), self.p0.ref,
                                               self.p1.ref, self._wd.data_ptr(), self._hd.data_ptr(),
                                               cnt.data_ptr(), st), "panel sweep")
            _lib.check(lib.mfg_panel_fold(ld, k, ctypes.byref(fold1), self.RtW.data_ptr(), k,
                                          self.out_scale, 1, None, None, st), "panel fold")
            self._ev_f[c].record(cur)
            cout.wait_event(self._ev_f[c])
            b0, b1 = nb_head + cr[c] * k * 4, nb_head + cr[c + 1] * k * 4
            with torch.cuda.stream(cout):
                self._host[b0:b1].copy_(self._out[b0:b1], non_blocking=True)
        self._ev_copy.record(cout)
        # all of H is here: its norm, the CSR pass's fold and sum r^2, R in CSR order
        _lib.check(lib.mfg_dot(_lib.MFG_F32, n * ld, self._hd.data_ptr(), self._hd.data_ptr(),
                               self.sums.data_ptr() + 16, self.ws.data_ptr(), self.wsb, st), "norm")
        pending = False
        if self.want_r:
            self._ev_fork.record(cur)
            self._side.wait_event(self._ev_fork)
            _lib.check(lib.mfg_gather(_lib.MFG_F32, self.obs.size, self._rsrc.data_ptr(),
                                      self._rcat.data_ptr(), self.R.data_ptr(), self._side.cuda_stream),
                       "R gather")
            self._ev_join.record(self._side)
            pending = True
        _lib.check(lib.mfg_panel_fold(ld, k, self.p0.ref, self.RH.data_ptr(), k, self.out_scale, 1,
                                      self.sums.data_ptr(), self.sq_ws.data_ptr(), st), "panel fold")
        self._host[:nb_head].copy_(self._out[:nb_head], non_blocking=True)
        if pending:
            cur.wait_event(self._ev_join)
        cur.wait_event(self._ev_copy)

    def _enqueue_pass(self, w: torch.Tensor, h: torch.Tensor, ps: int) -> bool:
        """One pass of the sweep (cold="pieces" plans): 0 = CSR (R, R.H, sum r^2,
        the norms), 1 = CSC (R^T.W). True when the R gather is pending on the
        side stream."""
        lib = _lib.lib()
        st = _lib.stream_ptr()
        pp = self.p0 if ps == 0 else self.p1
        none = ctypes.byref(self._no_cold)
        if ps == 0:
            self.sums[0:1].zero_()
            for x, o in ((w, 1), (h, 2)):
                _lib.check(lib.mfg_dot(_lib.MFG_F32, x.shape[0] * self.ld, x.data_ptr(), x.data_ptr(),
                                       self.sums.data_ptr() + 8 * o, self.ws.data_ptr(), self.wsb, st),
                           "norm")
        _lib.check(lib.mfg_cold_sweep(self.ld, pp.cold_ref if ps == 0 else none,
                                      pp.cold_ref if ps == 1 else none, w.data_ptr(), h.data_ptr(),
                                      self.RH.data_ptr(), self.RtW.data_ptr(), self.out_scale,
                                      self.cold_counters.data_ptr(), st), "cold sweep")
        nl, plist, cs, cnt = self._pass_lists[ps]
        if nl:
            _lib.check(lib.mfg_panel_sweep(self.ld, nl, plist.data_ptr(), cs.data_ptr(), self.p0.ref,
                                           self.p1.ref, w.data_ptr(), h.data_ptr(), cnt.data_ptr(), st),
                       "panel sweep")
        pending = False
        if ps == 0 and self.want_r:
            cur = torch.cuda.current_stream()
            self._ev_fork.record(cur)
            self._side.wait_event(self._ev_fork)
            _lib.check(lib.mfg_gather(_lib.MFG_F32, self.obs.size, self._rsrc.data_ptr(),
                                      self._rcat.data_ptr(), self.R.data_ptr(), self._side.cuda_stream),
                       "R gather")
            self._ev_join.record(self._side)
            pending = True
        out = self.RH if ps == 0 else self.RtW
        _lib.check(lib.mfg_panel_fold(self.ld, self.k, pp.ref, out.data_ptr(), self.k, self.out_scale, 1,
                                      self.sums.data_ptr() if ps == 0 else None,
                                      self.sq_ws.data_ptr() if ps == 0 else None, st), "panel fold")
        return pending

    def run(self, w: torch.Tensor, h: torch.Tensor) -> None:
        if self._enqueue(w, h):
            torch.cuda.current_stream().wait_event(self._ev_join)

    def _enqueue(self, w: torch.Tensor, h: torch.Tensor) -> bool:
        """Enqueue one sweep; True when the R gather runs on the side stream and
        the caller still has to wait for ``_ev_join``."""
        lib = _lib.lib()
        st = _lib.stream_ptr()
        if int(w.stride(0)) != self.ld or int(h.stride(0)) != self.ld:
            raise ValueError(f"factors must have row stride {self.ld}")
        lean = self.cold == "pieces"
        if lean:
            # Every row with entries is the fold of its slots (assigned, not added);
            # rows without entries are never written and stay zero. The norms.
            self.sums[0:1].zero_()
            for x, o in ((w, 1), (h, 2)):
                _lib.check(lib.mfg_dot(_lib.MFG_F32, x.shape[0] * self.ld, x.data_ptr(), x.data_ptr(),
                                       self.sums.data_ptr() + 8 * o, self.ws.data_ptr(), self.wsb, st),
                           "norm")
            _lib.check(lib.mfg_cold_sweep(self.ld, self.p0.cold_ref, self.p1.cold_ref, w.data_ptr(),
                                          h.data_ptr(), self.RH.data_ptr(), self.RtW.data_ptr(),
                                          self.out_scale, self.cold_counters.data_ptr(), st),
                       "cold sweep")
        else:
            # cold entries: grouped gather kernel; also the dense norms and the row zeroing
            _lib.check(lib.mfg_sweep_sharded(
                _lib.MFG_F32, 0, self.cold_csr.ref, self.cold_csc.ref, self.k,
                self.cold_vals.data_ptr(), self.cold_vals_csc.data_ptr(),
                w.data_ptr(), w.data_ptr(), self.ld, h.data_ptr(), h.data_ptr(), self.ld,
                self._rcold.data_ptr() if self.want_r else None, self.RH.data_ptr(),
                self.RtW.data_ptr(), self.out_scale, self.sums.data_ptr(), self.ws.data_ptr(),
                self.wsb, st), "hybrid sweep (cold)")
        if self.n_list:
            _lib.check(lib.mfg_panel_sweep(self.ld, self.n_list, self.plist.data_ptr(),
                                           self.cta_start.data_ptr(), self.p0.ref, self.p1.ref,
                                           w.data_ptr(), h.data_ptr(), self.counters.data_ptr(), st),
                       "panel sweep")
        # R back to CSR order on a side stream, next to the folds (both are short,
        # latency- and DRAM-bound kernels; in a captured graph: parallel branches)
        side = None
        if self.want_r:
            cur = torch.cuda.current_stream()
            side = self._side
            self._ev_fork.record(cur)
            side.wait_event(self._ev_fork)
            _lib.check(lib.mfg_gather(_lib.MFG_F32, self.obs.size, self._rsrc.data_ptr(),
                                      self._rcat.data_ptr(), self.R.data_ptr(), side.cuda_stream),
                       "R gather")
            self._ev_join.record(side)
        if self.n_list or lean:
            _lib.check(lib.mfg_panel_fold(self.ld, self.k, self.p0.ref, self.RH.data_ptr(), self.k,
                                          self.out_scale, 1 if lean else 0, self.sums.data_ptr(),
                                          self.sq_ws.data_ptr(), st), "panel fold")
            _lib.check(lib.mfg_panel_fold(self.ld, self.k, self.p1.ref, self.RtW.data_ptr(), self.k,
                                          self.out_scale, 1 if lean else 0, None, None, st),
                       "panel fold")
        return side is not None


def best_sweep_plan(obs: ObservationSet, k: int, *, want_r: bool = True, out_scale: float = 1.0,
                    mode: str | None = None):
    """The faster of the gather-only sweep (``mfsolver.SweepPlan``) and the
    hybrid panel sweep for this Omega and k, decided by timing both once
    (3 sweeps each on seeded factors). ``mode`` / ``MFG_SWEEP_PLAN``:
    "gather", "hybrid" or "auto" (default). The hybrid plan is considered for
    fp32 storage, a supported width and at least ``MFG_HYBRID_MIN_NNZ``
    (2e7) entries."""
    from .mfsolver import SweepPlan

    mode = mode or os.environ.get("MFG_SWEEP_PLAN", "auto")
    base = SweepPlan(obs, k, want_r=want_r, out_scale=out_scale)
    base.kind = "gather"
    eligible = (obs.dtype == torch.float32 and panel_ld(k, obs.dtype) > 0
                and (mode == "hybrid" or obs.size >= int(float(os.environ.get("MFG_HYBRID_MIN_NNZ", 2e7)))))
    if mode == "gather" or not eligible:
        return base
    hyb = HybridSweepPlan(obs, k, want_r=want_r, out_scale=out_scale)
    if mode == "hybrid":
        return hyb
    g = torch.Generator(device="cpu").manual_seed(1234)
    dev = obs.dev.device
    w = base.pad((torch.rand((obs.m, k), generator=g) * 0.5).to(dev))
    h = base.pad((torch.rand((obs.n, k), generator=g) * 0.5).to(dev))

    def t(plan):
        best = float("inf")
        for i in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            plan.run(w, h)
            e1.record()
            e1.synchronize()
            if i >= 2:
                best = min(best, e0.elapsed_time(e1))
        return best

    tb, th = t(base), t(hyb)
    pick = hyb if th < tb else base
    pick.trial_ms = {"gather": tb, "hybrid": th}
    return pick
