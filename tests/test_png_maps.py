"""PNG map ingest (occupancy_map.cpp:148-165 + image_png.cpp:37-100):
load_map decodes PNG like the reference's libpng path — 8-bit grayscale,
1/2/4-bit grayscale expanded to 8 bits (x255/x85/x17, as
png_set_expand_gray_1_2_4_to_8), 8-bit gray+alpha with the alpha stripped,
Adam7 interlacing, all five row filters — and rejects 16-bit, colour,
truncated and CRC-corrupt streams with MapParseError. libpng is not in this
image, so the reference's own PNG path cannot run here; the test PNGs are
written by an independent encoder below and every case is checked against
the same image saved as PGM (whose parity with the reference is pinned in
test_capi.py). Host code only: runs on the CPU."""
import ctypes as C
import struct
import zlib

import numpy as np
import pytest

from paper_1910_00572_b200 import _lib
from paper_1910_00572_b200.floorplan import make_floorplan

ADAM7 = [(0, 0, 8, 8), (4, 0, 8, 8), (0, 4, 4, 8), (2, 0, 4, 4), (0, 2, 2, 4), (1, 0, 2, 2), (0, 1, 1, 2)]


def _chunk(typ, data, corrupt=False):
    crc = zlib.crc32(typ + data) & 0xFFFFFFFF
    if corrupt:
        crc ^= 1
    return struct.pack(">I", len(data)) + typ + data + struct.pack(">I", crc)


def _pack_row(vals, depth):
    if depth == 8:
        return bytes(vals)
    per = 8 / depth
    out = bytearray((len(vals) * depth + 7) // 8)
    for i, v in enumerate(vals):
        out[int(i // per)] |= v << (8 - depth * (1 + i % int(per)))
    return bytes(out)


def _filter(raw, prev, bpp, ftype):
    out = bytearray(len(raw))
    for i, x in enumerate(raw):
        a = raw[i - bpp] if i >= bpp else 0
        b = prev[i] if prev is not None else 0
        c = prev[i - bpp] if (prev is not None and i >= bpp) else 0
        if ftype == 0:
            p = 0
        elif ftype == 1:
            p = a
        elif ftype == 2:
            p = b
        elif ftype == 3:
            p = (a + b) >> 1
        else:
            pa, pb, pc = abs(b - c), abs(a - c), abs(a + b - 2 * c)
            p = a if (pa <= pb and pa <= pc) else (b if pb <= pc else c)
        out[i] = (x - p) & 0xFF
    return bytes([ftype]) + bytes(out)


def encode_png(samples, depth=8, alpha=None, interlace=False, color=None, bitdepth=None, extra=b"",
               corrupt_idat=False, truncate=0):
    """samples: (H, W) uint array of depth-bit gray values."""
    h, w = samples.shape
    color = (4 if alpha is not None else 0) if color is None else color
    channels = 2 if color == 4 else 1
    bpp = max(1, channels * depth // 8)
    passes = ADAM7 if interlace else [(0, 0, 1, 1)]
    raw = bytearray()
    ftype = 0
    for (x0, y0, dx, dy) in passes:
        sub = samples[y0::dy, x0::dx]
        if sub.size == 0:
            continue
        asub = alpha[y0::dy, x0::dx] if alpha is not None else None
        prev = None
        for r in range(sub.shape[0]):
            if channels == 2:
                vals = [int(v) for pair in zip(sub[r], asub[r]) for v in pair]
            else:
                vals = [int(v) for v in sub[r]]
            row = _pack_row(vals, depth)
            raw += _filter(row, prev, bpp, ftype % 5)
            ftype += 1
            prev = row
    ihdr = struct.pack(">IIBBBBB", w, h, bitdepth or depth, color, 0, 0, 1 if interlace else 0)
    z = zlib.compress(bytes(raw), 9)
    png = b"\x89PNG\r\n\x1a\n" + _chunk(b"IHDR", ihdr) + extra
    png += _chunk(b"IDAT", z[: len(z) // 2]) + _chunk(b"IDAT", z[len(z) // 2:], corrupt=corrupt_idat)
    png += _chunk(b"IEND", b"")
    return png[: len(png) - truncate] if truncate else png


def _load(data, threshold):
    lib = _lib.load()
    buf = np.frombuffer(data, np.uint8).copy()
    w, h = C.c_int(), C.c_int()
    rc = lib.gl_load_map(buf.ctypes.data_as(C.POINTER(C.c_uint8)), len(buf), threshold, C.byref(w), C.byref(h),
                         None)
    if rc != 0:
        return rc, None
    out = np.empty((h.value, w.value), np.uint8)
    rc = lib.gl_load_map(buf.ctypes.data_as(C.POINTER(C.c_uint8)), len(buf), threshold, C.byref(w), C.byref(h),
                         out.ctypes.data_as(C.POINTER(C.c_uint8)))
    return rc, out


def _pgm(gray8):
    h, w = gray8.shape
    return b"P5\n%d %d\n255\n" % (w, h) + gray8.astype(np.uint8).tobytes()


CASES = [  # (H, W, depth, gray+alpha, interlaced)
    (60, 90, 8, False, False), (61, 37, 8, False, True), (5, 3, 8, True, False), (17, 9, 8, True, True),
    (1, 1, 8, False, False), (2, 1, 8, False, True), (23, 31, 4, False, False), (23, 31, 4, False, True),
    (13, 29, 2, False, False), (13, 29, 2, False, True), (9, 33, 1, False, False), (9, 33, 1, False, True),
]


@pytest.mark.parametrize("H,W,depth,ga,il", CASES)
def test_png_decodes_like_the_pgm_of_the_same_image(H, W, depth, ga, il):
    rng = np.random.default_rng(H * 100 + W + depth)
    top = (1 << depth) - 1
    samples = rng.integers(0, top + 1, size=(H, W))
    if depth == 8 and H >= 40:  # a real floor plan for the big case
        samples = np.where(make_floorplan(W, H, seed=2) == 0, 254, rng.integers(0, 60, size=(H, W)))
    alpha = rng.integers(0, 256, size=(H, W)) if ga else None
    gray8 = samples * (255 // top)
    png = encode_png(samples, depth, alpha=alpha, interlace=il)
    for thr in (1, 60, 128, 200, 254):
        rc, occ = _load(png, thr)
        assert rc == 0, (thr, _lib.load().gl_last_error())
        rc2, occ_pgm = _load(_pgm(gray8), thr)
        assert rc2 == 0
        assert np.array_equal(occ, occ_pgm), thr


def test_png_ancillary_chunks_and_bad_ancillary_crc_are_ignored():
    s = np.random.default_rng(1).integers(0, 256, size=(7, 11))
    extra = _chunk(b"tEXt", b"Comment\x00hi") + _chunk(b"gAMA", b"\x00\x00\xb1\x8f", corrupt=True)
    rc, occ = _load(encode_png(s, extra=extra), 128)
    assert rc == 0
    assert np.array_equal(occ, _load(_pgm(s), 128)[1])


@pytest.mark.parametrize("kw", [dict(bitdepth=16), dict(color=2), dict(color=3), dict(corrupt_idat=True),
                                dict(truncate=30), dict(bitdepth=3)])
def test_png_rejections_are_map_parse_errors(kw):
    s = np.random.default_rng(2).integers(0, 256, size=(6, 6))
    rc, _ = _load(encode_png(s, **kw), 128)
    assert rc == _lib.GL_E_MAP_PARSE, kw
