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


def decode_pieces(buf: np.ndarray, rows: int, R_rows: int, ksteps: int, cin: int, pp_stride: int):
    """buf: int8 image.  Returns int array [46][rows][cin] of hi*256 + lo."""
    r = np.arange(rows)[:, None]; k = np.arange(cin)[None, :]
    off = (r // R_rows) * ksteps * R_rows * 32 + tiled_offset(r % R_rows, k, R_rows)
    out = np.zeros((46, rows, cin), np.int64)
    for pl in range(46):
        hi = buf[2 * pl * pp_stride + off].astype(np.int64)
        lo = buf[(2 * pl + 1) * pp_stride + off].astype(np.int64) & 255
        out[pl] = hi * 256 + lo
    return out


def decode_v(buf: np.ndarray, tiles: int, ksteps: int, cin: int):
    """V image [tile_block][kstep][92 plane-pieces][4 KB] -> int [46][tiles][cin] (hi*256 + lo)."""
    t = np.arange(tiles)[:, None]; k = np.arange(cin)[None, :]
    blk = ((t // 128) * ksteps + (k >> 5)) * 92
    within = tiled_offset(t % 128, k & 31, 128)
    out = np.zeros((46, tiles, cin), np.int64)
    for pl in range(46):
        hi = buf[(blk + 2 * pl) * 4096 + within].astype(np.int64)
        lo = buf[(blk + 2 * pl + 1) * 4096 + within].astype(np.int64) & 255
        out[pl] = hi * 256 + lo
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
