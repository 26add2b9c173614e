"""Host logic of the hybrid sweep's panel layout (paper_2204_14067_b200/panel.py):
the arrays the panel kernel walks, replayed in numpy, reproduce the reference's
R and R.H (mfg/data.py:253-263, mfg/operators.py:108) on the hot entries, and
hot + cold entries partition Omega. Runs on CPU tensors (no GPU)."""
import types

import numpy as np
import pytest
import torch

from paper_2204_14067_b200 import panel


def _case(seed, m, n, dens, decay):
    rng = np.random.default_rng(seed)
    mask = rng.random((m, n)) < (dens * (1.0 / (1 + np.arange(n))) ** decay)[None, :]
    rows, cols = np.nonzero(mask)
    vals = rng.standard_normal(len(rows)).astype(np.float32)
    return rng, rows, cols, vals


@pytest.mark.parametrize("cfg", [
    dict(PR=16, lmin=3, lmax=21, max_panels=6, min_panel_entries=10),
    dict(PR=8, lmin=1, lmax=5, max_panels=100, min_panel_entries=1),
    dict(PR=64, lmin=2, lmax=500, max_panels=2, min_panel_entries=1),
])
def test_panel_layout_replay(cfg):
    m, n, k = 60, 300, 40
    rng, rows, cols, vals = _case(0, m, n, 0.5, 0.4)
    nnz = len(rows)
    lay = types.SimpleNamespace(nnz=nnz, nrows=m, ncols=n, idx=torch.tensor(cols, dtype=torch.int32),
                                row_of=torch.tensor(rows, dtype=torch.int32))
    PR = cfg.pop("PR")
    pp = panel._PanelPass(lay, torch.tensor(vals), m, n, PR, k, 0, want_r=False, want_sq=True, **cfg)
    assert pp.n_hot > 0
    W = rng.standard_normal((m, k))
    H = rng.standard_normal((n, k))
    ids = pp.panel_ids.numpy()
    pieces = pp.pieces.numpy()
    recs = pp.recs.numpy()
    loc16 = recs.view(np.int16).reshape(-1, 48)
    po = np.zeros((pp.n_pieces, k))
    rhot = np.zeros((pp.n_blocks + 2) * 16)
    seen = np.zeros(pp.n_pieces, int)
    covered = np.zeros(pp.n_pieces, int)
    for _, p, a, b in pp.plist.numpy():
        prow = ids[p * PR:(p + 1) * PR]
        covered[a:b] += 1
        assert np.all(np.diff(pieces[a:b, 2]) <= 0)          # longest first inside a panel
        for t in range(a, b):
            row, blk0, ln, slot = pieces[t]
            assert 1 <= ln <= cfg["lmax"]
            seen[slot] += 1
            for e in range(ln):
                blk, off = blk0 + e // 16, e % 16
                g = prow[loc16[blk, off]]
                assert g >= 0
                a_e = float(recs[blk, 8 + off:9 + off].view(np.float32)[0])
                r = float(W[row] @ H[g]) - a_e
                rhot[blk * 16 + off] = r
                po[slot] += r * H[g]
    assert np.all(seen == 1) and np.all(covered == 1)
    assert int(pp.plist_entries.sum()) == pp.n_hot
    # fold in slot order + the cold entries = R.H of the whole Omega
    RH = np.zeros((m, k))
    fr, fb, fc = pp.frows.numpy(), pp.fbeg.numpy(), pp.fcnt.numpy()
    assert len(set(fr.tolist())) == len(fr)
    assert np.all(fc[:pp.n_light] <= 32) and np.all(fc[pp.n_light:] > 32)
    for f, row in enumerate(fr):
        RH[row] += po[fb[f]:fb[f] + fc[f]].sum(0)
    cold = pp.cold_mask.numpy()
    Rfull = (W[rows] * H[cols]).sum(1) - vals.astype(np.float64)
    np.add.at(RH, rows[cold], Rfull[cold, None] * H[cols[cold]])
    RHref = np.zeros((m, k))
    np.add.at(RHref, rows, Rfull[:, None] * H[cols])
    assert np.abs(RH - RHref).max() < 1e-11
    # the residual map back to CSR order
    ho, hp = pp.hot_orig.numpy(), pp.hot_pos.numpy()
    assert len(ho) + int(cold.sum()) == nnz and not cold[ho].any()
    assert np.abs(rhot[hp] - Rfull[ho]).max() < 1e-12


@pytest.mark.parametrize("cfg", [
    dict(PR=16, lmin=3, lmax=21, max_panels=6, min_panel_entries=10),
    dict(PR=8, lmin=10 ** 6, lmax=7, max_panels=3, min_panel_entries=1),     # everything cold
])
def test_panel_layout_cold_pieces_replay(cfg):
    """With cold_pieces the cold entries are pieces too (global row ids in
    128-byte record blocks) and every output row is the fold of its slots."""
    m, n, k = 60, 300, 40
    rng, rows, cols, vals = _case(1, m, n, 0.5, 0.4)
    nnz = len(rows)
    lay = types.SimpleNamespace(nnz=nnz, nrows=m, ncols=n, idx=torch.tensor(cols, dtype=torch.int32),
                                row_of=torch.tensor(rows, dtype=torch.int32))
    PR = cfg.pop("PR")
    pp = panel._PanelPass(lay, torch.tensor(vals), m, n, PR, k, 0, want_r=False, want_sq=True,
                          cold_pieces=True, direct=True, **cfg)
    W = rng.standard_normal((m, k))
    H = rng.standard_normal((n, k))
    po = np.zeros((pp.n_slots, k))
    seen = np.zeros(pp.n_slots, int)
    ids = pp.panel_ids.numpy()
    recs = pp.recs.numpy()
    loc16 = recs.view(np.int16).reshape(-1, 48)
    for _, p, a, b in pp.plist.numpy():
        prow = ids[p * PR:(p + 1) * PR]
        for row, blk0, ln, slot in pp.pieces.numpy()[a:b]:
            seen[slot] += 1
            for e in range(ln):
                blk, off = blk0 + e // 16, e % 16
                g = prow[loc16[blk, off]]
                a_e = float(recs[blk, 8 + off:9 + off].view(np.float32)[0])
                po[slot] += (float(W[row] @ H[g]) - a_e) * H[g]
    crecs = pp.cold_recs.numpy()
    rcold = np.zeros((pp.n_cold_blocks + 2) * 16)
    cp = pp.cold_pieces.numpy()[:pp.n_cold_pieces]
    assert np.all(np.diff(cp[:, 2] & 0x3fffffff) <= 0)
    RH = np.zeros((m, k))
    ndirect = 0
    for row, blk0, ln, slot in cp:
        is_direct = (ln >> 30) != 0
        ln &= 0x3fffffff
        ndirect += is_direct
        assert 1 <= ln <= cfg["lmax"]
        seen[slot] += 1
        for e in range(ln):
            blk, off = blk0 + e // 16, e % 16
            g = crecs[blk, off]
            a_e = float(crecs[blk, 16 + off:17 + off].view(np.float32)[0])
            r = float(W[row] @ H[g]) - a_e
            rcold[blk * 16 + off] = r
            if is_direct:
                RH[row] += r * H[g]           # the piece writes its row itself
            else:
                po[slot] += r * H[g]
    assert np.all(seen == 1) and ndirect == pp.n_direct
    fr, fb, fc = pp.frows.numpy(), pp.fbeg.numpy(), pp.fcnt.numpy()
    for f, row in enumerate(fr):
        assert not RH[row].any()              # direct rows are not folded
        RH[row] += po[fb[f]:fb[f] + fc[f]].sum(0)
    Rfull = (W[rows] * H[cols]).sum(1) - vals.astype(np.float64)
    RHref = np.zeros((m, k))
    np.add.at(RHref, rows, Rfull[:, None] * H[cols])
    assert np.abs(RH - RHref).max() < 1e-11
    co, cpos = pp.cold_orig.numpy(), pp.cold_pos.numpy()
    assert len(co) + pp.n_hot == nnz
    assert np.abs(rcold[cpos] - Rfull[co]).max() < 1e-12


def test_panel_layout_no_hot_entries():
    m, n, k = 10, 40, 40
    rng, rows, cols, vals = _case(3, m, n, 0.3, 0.0)
    lay = types.SimpleNamespace(nnz=len(rows), nrows=m, ncols=n, idx=torch.tensor(cols, dtype=torch.int32),
                                row_of=torch.tensor(rows, dtype=torch.int32))
    pp = panel._PanelPass(lay, torch.tensor(vals), m, n, 16, k, 1, lmin=10 ** 6, lmax=256, max_panels=4,
                          min_panel_entries=1, want_r=False, want_sq=False)
    assert pp.n_hot == 0 and pp.n_pieces == 0 and pp.plist.shape[0] == 0
    assert bool(pp.cold_mask.all())


def test_panel_layout_chunks():
    """nchunks > 1 (the end-to-end path's CSC pass): every list element, cold
    piece range and fold range stays inside one contiguous range of self rows."""
    m, n, k = 60, 300, 40
    rng, rows, cols, vals = _case(2, m, n, 0.5, 0.4)
    lay = types.SimpleNamespace(nnz=len(rows), nrows=m, ncols=n, idx=torch.tensor(cols, dtype=torch.int32),
                                row_of=torch.tensor(rows, dtype=torch.int32))
    nc = 3
    crows = panel._chunk_rows(m, nc, 0.7)
    pp = panel._PanelPass(lay, torch.tensor(vals), m, n, 16, k, 1, lmin=3, lmax=21, max_panels=6,
                          min_panel_entries=10, want_r=False, want_sq=False, cold_pieces=True,
                          direct=True, chunk_rows=crows, chunk_by="self")
    cr = pp.chunk_rows
    assert cr[0] == 0 and cr[-1] == m and len(cr) == nc + 1 and cr[1] - cr[0] > cr[3] - cr[2]
    pieces = pp.pieces.numpy()
    panels = []
    for (_, p, a, b), c in zip(pp.plist.numpy(), pp.plist_chunk.numpy()):
        panels.append(p)
        r = pieces[a:b, 0]
        assert np.all((r >= cr[c]) & (r < cr[c + 1]))
        assert np.all(np.diff(pieces[a:b, 2]) <= 0)
    assert panels == sorted(panels)            # panel-major: consecutive elements share a panel
    cp = pp.cold_pieces.numpy()
    ptr = pp.cold_chunk_ptr
    assert ptr[0] == 0 and ptr[-1] == pp.n_cold_pieces
    for c in range(nc):
        r = cp[ptr[c]:ptr[c + 1], 0]
        assert np.all((r >= cr[c]) & (r < cr[c + 1]))
    tot = 0
    for c, (off, nr, nlt) in enumerate(pp.cf_info):
        r = pp.cf_rows.numpy()[off:off + nr]
        cnt = pp.cf_cnt.numpy()[off:off + nr]
        assert np.all((r >= cr[c]) & (r < cr[c + 1]))
        assert np.all(cnt[:nlt] <= 32) and np.all(cnt[nlt:] > 32)
        tot += nr
    assert tot == pp.frows.numel()
    assert sorted(pp.cf_rows.numpy().tolist()) == sorted(pp.frows.numpy().tolist())


def test_panel_layout_gathered_chunks():
    """chunk_by="gath" (the end-to-end path's CSR pass): a panel holds gathered
    rows of one chunk, a cold piece gathers from one chunk, and the replay
    still reproduces R.H."""
    m, n, k = 60, 300, 40
    rng, rows, cols, vals = _case(4, m, n, 0.5, 0.4)
    nnz = len(rows)
    lay = types.SimpleNamespace(nnz=nnz, nrows=m, ncols=n, idx=torch.tensor(cols, dtype=torch.int32),
                                row_of=torch.tensor(rows, dtype=torch.int32))
    nc, PR = 3, 16
    crows = panel._chunk_rows(n, nc, 0.7)
    pp = panel._PanelPass(lay, torch.tensor(vals), m, n, PR, k, 0, lmin=3, lmax=21, max_panels=9,
                          min_panel_entries=10, want_r=False, want_sq=True, cold_pieces=True,
                          direct=True, chunk_rows=crows, chunk_by="gath")
    assert pp.n_hot > 0 and pp.n_cold_pieces > 0
    W = rng.standard_normal((m, k))
    H = rng.standard_normal((n, k))
    ids = pp.panel_ids.numpy()
    recs = pp.recs.numpy()
    loc16 = recs.view(np.int16).reshape(-1, 48)
    po = np.zeros((pp.n_slots, k))
    RH = np.zeros((m, k))
    pieces = pp.pieces.numpy()
    for (_, p, a, b), c in zip(pp.plist.numpy(), pp.plist_chunk.numpy()):
        prow = ids[p * PR:(p + 1) * PR]
        live = prow[prow >= 0]
        assert np.all((live >= crows[c]) & (live < crows[c + 1]))    # the panel's rows: one chunk
        for row, blk0, ln, slot in pieces[a:b]:
            for e in range(ln):
                blk, off = blk0 + e // 16, e % 16
                g = prow[loc16[blk, off]]
                assert g >= 0
                a_e = float(recs[blk, 8 + off:9 + off].view(np.float32)[0])
                po[slot] += (float(W[row] @ H[g]) - a_e) * H[g]
    crecs = pp.cold_recs.numpy()
    cp = pp.cold_pieces.numpy()
    ptr = pp.cold_chunk_ptr
    assert ptr[-1] == pp.n_cold_pieces
    for c in range(nc):
        for row, blk0, ln, slot in cp[ptr[c]:ptr[c + 1]]:
            is_direct = (ln >> 30) != 0
            ln &= 0x3fffffff
            for e in range(ln):
                blk, off = blk0 + e // 16, e % 16
                g = crecs[blk, off]
                assert crows[c] <= g < crows[c + 1]                    # gathers from its chunk only
                a_e = float(crecs[blk, 16 + off:17 + off].view(np.float32)[0])
                r = float(W[row] @ H[g]) - a_e
                if is_direct:
                    RH[row] += r * H[g]
                else:
                    po[slot] += r * H[g]
    fr, fb, fc = pp.frows.numpy(), pp.fbeg.numpy(), pp.fcnt.numpy()
    for f, row in enumerate(fr):
        RH[row] += po[fb[f]:fb[f] + fc[f]].sum(0)
    Rfull = (W[rows] * H[cols]).sum(1) - vals.astype(np.float64)
    RHref = np.zeros((m, k))
    np.add.at(RHref, rows, Rfull[:, None] * H[cols])
    assert np.abs(RH - RHref).max() < 1e-11
    assert len(pp.cold_orig) + pp.n_hot == nnz
