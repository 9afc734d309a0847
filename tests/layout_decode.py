"""Test-side decoding of the documented HBM layouts (DESIGN.md "HBM layout",
csrc/layout.cuh comment) and of the oracle's complex values into the 46
plane order.  Pure indexing -- no method arithmetic beyond the trivial
Karatsuba sum re+im that defines the third plane of each pair."""
import numpy as np

R = [0, 1, 2, 5]
REAL_POS = [r * 6 + c for r in R for c in R]
CPX_POS = [0 * 6 + 3, 1 * 6 + 3, 2 * 6 + 3, 5 * 6 + 3, 3 * 6 + 0, 3 * 6 + 1, 3 * 6 + 2, 3 * 6 + 5, 3 * 6 + 3,
           3 * 6 + 4]


def tiled_offset(r, k, R_rows):
    r = np.asarray(r, np.int64); k = np.asarray(k, np.int64)
    return (k >> 5) * R_rows * 32 + (r >> 3) * 256 + ((k >> 4) & 1) * 128 + (r & 7) * 16 + (k & 15)


def decode_w_staged(buf: np.ndarray, cout_pad: int, nblk: int, ksteps: int, cin: int, nplanes: int = 46):
    """W' image [plane][cout block][K step][W hi rows | W lo rows] (balanced s8 pieces) ->
    int [nplanes][cout_pad][cin] of hi*256 + lo."""
    co = np.arange(cout_pad)[:, None]; k = np.arange(cin)[None, :]
    nblocks = cout_pad // nblk
    b = buf.astype(np.int64)
    out = np.zeros((nplanes, cout_pad, cin), np.int64)
    for pl in range(nplanes):
        base = ((pl * nblocks + co // nblk) * ksteps + (k >> 5)) * (2 * nblk * 32)
        hi = b[base + tiled_offset(co % nblk, k & 31, 2 * nblk)]
        lo = b[base + tiled_offset(nblk + co % nblk, k & 31, 2 * nblk)]
        out[pl] = hi * 256 + lo
    return out


def decode_w1(buf: np.ndarray, cout_pad: int, nblk: int, ksteps: int, cin: int, nplanes: int = 46):
    """Single-piece W' image of the int8-native target (f3) [plane][cout block][K step][n_block rows]
    -> int [nplanes][cout_pad][cin]."""
    co = np.arange(cout_pad)[:, None]; k = np.arange(cin)[None, :]
    nblocks = cout_pad // nblk
    b = buf.astype(np.int64)
    out = np.zeros((nplanes, cout_pad, cin), np.int64)
    for pl in range(nplanes):
        base = ((pl * nblocks + co // nblk) * ksteps + (k >> 5)) * (nblk * 32)
        out[pl] = b[base + tiled_offset(co % nblk, k & 31, nblk)]
    return out


def decode_v(buf: np.ndarray, tiles: int, ksteps: int, cin: int, nplanes: int = 46):
    """V image [tile_block][plane][K step][hi, lo][4 KB] (balanced s8 pieces) -> int [nplanes][tiles][cin]."""
    t = np.arange(tiles)[:, None]; k = np.arange(cin)[None, :]
    within = tiled_offset(t % 128, k & 31, 128)
    b = buf.astype(np.int64)
    out = np.zeros((nplanes, tiles, cin), np.int64)
    for pl in range(nplanes):
        blk = (((t // 128) * nplanes + pl) * ksteps + (k >> 5)) * 2
        out[pl] = b[blk * 4096 + within] * 256 + b[(blk + 1) * 4096 + within]
    return out


def complex_to_planes(Z: np.ndarray) -> np.ndarray:
    """Z [..., 36, 2] (re, im per position) -> [46, ...] plane values."""
    planes = [Z[..., p, 0] for p in REAL_POS]
    for p in CPX_POS:
        re, im = Z[..., p, 0], Z[..., p, 1]
        planes += [re, im, re + im]
    return np.stack(planes, 0)


def karatsuba_planes_to_complex(Mp: np.ndarray):
    """GPU per-plane int32 results [46, ...] -> (real [16, ...], re [10, ...], im [10, ...]) as int32 wrap."""
    Mp = Mp.astype(np.int64)
    real = Mp[:16]
    p0, p1, p2 = Mp[16::3], Mp[17::3], Mp[18::3]
    wrap = lambda v: ((v + 2 ** 31) % 2 ** 32) - 2 ** 31
    return wrap(real), wrap(p0 - p1), wrap(p2 - p0 - p1)


def decode_m(buf: np.ndarray, tiles: int, cout: int, cout_pad: int, nblk: int, tiles_pad: int, slots=36):
    """M (int32 [slots][tile_block][cout_block][128][nblk], 16-byte chunks
    XOR-swizzled by row) -> [slots][tiles][cout]."""
    t = np.arange(tiles)[:, None]; c = np.arange(cout)[None, :]
    r = t % 128; cc = c % nblk; nb = c // nblk
    cpr = nblk // 4; swz = min(cpr, 8) - 1
    off = ((t // 128) * (cout_pad // nblk) + nb) * (128 * nblk) + r * nblk + (((cc >> 2) ^ (r & swz)) << 2) + (cc & 3)
    buf = buf.reshape(slots, tiles_pad * cout_pad)
    return np.stack([buf[p][off] for p in range(slots)], 0)


# ------------------------------------------------------------------ fused-path layouts (layout.cuh)
# Groups in processing order gi: gi = 5k + s for k = 0..3 over rows R[FROW[k]] (rows 0, 5, 1, 2):
# s < 4 real (R[ri], R[s]), s = 4 the primary (R[ri], 3); gi = 20..25 primaries 4..9.
FROW = [0, 3, 1, 2]


def fused_groups():
    """[(kind, index)] per gi: ("real", plane s = ri*4 + c) or ("cpx", primary k)."""
    out = []
    for k in range(4):
        ri = FROW[k]
        out += [("real", ri * 4 + s) for s in range(4)] + [("cpx", ri)]
    return out + [("cpx", k) for k in range(4, 10)]


def _prefixes(sizes):
    pre, acc = [], 0
    for s in sizes:
        pre.append(acc); acc += s
    return pre, acc


def decode_v_fused(buf: np.ndarray, tiles: int, ksteps: int, cin: int):
    """V image [tile_block][group][kstep][piece][4 KB], pieces hi (s8) and lo (u8) -> (real [16][T][cin],
    re [10][T][cin], im [10][T][cin]) as hi * 256 + lo."""
    groups = fused_groups()
    pcs = [4 if g[0] == "cpx" else 2 for g in groups]
    pre, total = _prefixes(pcs)
    assert total == 72
    t = np.arange(tiles)[:, None]; k = np.arange(cin)[None, :]
    within = tiled_offset(t % 128, k & 31, 128)
    real = np.zeros((16, tiles, cin), np.int64); re = np.zeros((10, tiles, cin), np.int64); im = re.copy()
    b = buf.astype(np.int64)   # int8 buffer: signed pieces
    for gi, (kind, idx) in enumerate(groups):
        base = ((t // 128) * 72 + pre[gi]) * ksteps + (k >> 5) * pcs[gi]
        val = lambda p: b[(base + p) * 4096 + within] * 256 + (b[(base + p + 1) * 4096 + within] & 255)
        if kind == "real":
            real[idx] = val(0)
        else:
            re[idx], im[idx] = val(0), val(2)
    return real, re, im


def decode_w_fused(buf: np.ndarray, cout_pad: int, ksteps: int, cin_pad: int):
    """W' image [cout block of 16][group][kstep][rows x 32 B] -> (real [16][cout][cin], re, im [10][cout][cin],
    consistency flag of the duplicated B1 rows: -Wi and Wr)."""
    groups = fused_groups()
    wu = [4 if g[0] == "cpx" else 1 for g in groups]
    pre, total = _prefixes(wu)
    assert total == 56
    co = np.arange(cout_pad)[:, None]; k = np.arange(cin_pad)[None, :]
    nb, cr = co // 16, co % 16
    b = buf.astype(np.int64)
    real = np.zeros((16, cout_pad, cin_pad), np.int64); re = np.zeros((10, cout_pad, cin_pad), np.int64)
    im = re.copy(); ok = True
    for gi, (kind, idx) in enumerate(groups):
        base = ((nb * 56 + pre[gi]) * ksteps + (k >> 5) * wu[gi]) * 1024
        rowv = lambda r: b[base + tiled_offset(r, k & 31, 32 * wu[gi])]
        if kind == "real":
            real[idx] = rowv(cr) * 256 + rowv(16 + cr)
        else:
            re[idx] = rowv(cr) * 256 + rowv(32 + cr)
            im[idx] = rowv(16 + cr) * 256 + rowv(48 + cr)
            ok &= bool(np.array_equal(rowv(64 + cr) * 256 + rowv(96 + cr), -im[idx]))
            ok &= bool(np.array_equal(rowv(80 + cr) * 256 + rowv(112 + cr), re[idx]))
    return real, re, im, ok


def complex_to_values(Z: np.ndarray):
    """Z [..., 36, 2] -> (real [16, ...], re [10, ...], im [10, ...]) in plane / primary order."""
    real = np.stack([Z[..., p, 0] for p in REAL_POS], 0)
    re = np.stack([Z[..., p, 0] for p in CPX_POS], 0)
    im = np.stack([Z[..., p, 1] for p in CPX_POS], 0)
    return real, re, im


# ---------------------------------------------------------------- quarter-K packing (c_in <= 8, layout.cuh)
def qk_sg_of(gi):
    return (gi // 5) * 3 + ((gi % 5) // 2 if gi % 5 < 4 else 2) if gi < 20 else 12 + gi - 20


def qk_sg_first(sg):
    return (sg // 3) * 5 + (sg % 3) * 2 if sg < 12 else 20 + sg - 12


def decode_w_qk(buf: np.ndarray, cout_pad: int, cin: int):
    """Packed W' [16-cout block][pack 0..8][160 rows x 32 B] -> (real [16][cout][cin], re, im, ok) as
    hi * 256 + lo; ok: the -Wi / Wr duplicates, the zero rows and the other slot's K half are as specified."""
    groups = fused_groups()
    b = buf.astype(np.int64)
    co = np.arange(cout_pad)[:, None]; ch = np.arange(cin)[None, :]
    nb, cr = co // 16, co % 16
    real = np.zeros((16, cout_pad, cin), np.int64); re = np.zeros((10, cout_pad, cin), np.int64)
    im = re.copy(); ok = True

    def at(pack, row, kbyte):
        return b[(nb * 9 + pack) * 5120 + tiled_offset(row, kbyte, 160)]

    for gi, (kind, idx) in enumerate(groups):
        sg = qk_sg_of(gi); pack, sp = sg // 2, sg % 2
        base = 96 * sp
        if kind == "real":
            vp = gi - qk_sg_first(sg)
            kb = sp * 16 + vp * 8 + ch
            real[idx] = at(pack, base + 16 * vp + cr, kb) * 256 + at(pack, base + 32 + 16 * vp + cr, kb)
            ok &= not at(pack, base + 16 * (1 - vp) + cr, kb).any()     # the other group's rows: 0 here
        else:
            k0, k1 = sp * 16 + ch, sp * 16 + 8 + ch
            re[idx] = at(pack, base + cr, k0) * 256 + at(pack, base + 32 + cr, k0)
            im[idx] = at(pack, base + 16 + cr, k0) * 256 + at(pack, base + 48 + cr, k0)
            ok &= bool(np.array_equal(at(pack, base + cr, k1) * 256 + at(pack, base + 32 + cr, k1), -im[idx]))
            ok &= bool(np.array_equal(at(pack, base + 16 + cr, k1) * 256 + at(pack, base + 48 + cr, k1), re[idx]))
        other = (1 - sp) * 16 + ch            # the other slot's K half of this slot's rows
        for r in range(4):
            ok &= not at(pack, base + 16 * r + cr, other).any() and not at(pack, base + 16 * r + cr, other + 8).any()
    for pack in range(9):
        for r in (64, 80):
            for kb in range(32):
                ok &= not at(pack, r + cr, np.full_like(ch, kb)).any()
    return real, re, im, ok


def decode_v_qk(buf: np.ndarray, tiles: int, cin: int):
    """Packed V [tile block][pack][piece hi (s8), lo (u8)][4 KB] -> (real [16][T][cin], re, im)."""
    groups = fused_groups()
    b = buf.astype(np.int64)
    t = np.arange(tiles)[:, None]; ch = np.arange(cin)[None, :]
    real = np.zeros((16, tiles, cin), np.int64); re = np.zeros((10, tiles, cin), np.int64); im = re.copy()

    def val(pack, kbyte):
        off = ((t // 128) * 9 + pack) * 8192 + tiled_offset(t % 128, kbyte, 128)
        return b[off] * 256 + (b[off + 4096] & 255)

    for gi, (kind, idx) in enumerate(groups):
        sg = qk_sg_of(gi); pack, sp = sg // 2, sg % 2
        if kind == "real":
            real[idx] = val(pack, sp * 16 + (gi - qk_sg_first(sg)) * 8 + ch)
        else:
            re[idx], im[idx] = val(pack, sp * 16 + ch), val(pack, sp * 16 + 8 + ch)
    return real, re, im
