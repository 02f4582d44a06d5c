"""8-bit grayscale image I/O for frames and typ=3 inputs (reference
proj/include/rdcnn/image.hpp).

* PGM P5, maxval 255: the bit-exact interchange format (image.hpp:96-138).
* PNG: 8-bit gray out with filter 0 per row and one zlib stream at level 6,
  which is byte-identical to the reference's write_png (image.hpp:144-174)
  because both use the system zlib.  In: 8-bit gray or RGB (luma-reduced),
  all five row filters, no interlace (image.hpp:176-253).
* load_grayscale: PGM or PNG to a [0,1] float64 raster, optional
  nearest-neighbour square resample (image.hpp:259-290).

Host-side codecs only; frames are normalised to 8 bits on the device
(Simulator.frame_normalize) before they are downloaded.
"""
from __future__ import annotations

import struct
import zlib
from typing import Optional, Tuple

import numpy as np


class DecodeError(ValueError):
    pass


class UnsupportedFormat(ValueError):
    pass


def write_pgm(path: str, img: np.ndarray):
    img = np.ascontiguousarray(img, np.uint8)
    rows, cols = img.shape
    with open(path, "wb") as f:
        f.write(f"P5\n{cols} {rows}\n255\n".encode())
        f.write(img.tobytes())


def read_pgm(path: str) -> np.ndarray:
    data = open(path, "rb").read()
    pos = 0

    def token():
        nonlocal pos
        while pos < len(data):
            if data[pos:pos + 1] == b"#":
                while pos < len(data) and data[pos:pos + 1] != b"\n":
                    pos += 1
            elif data[pos:pos + 1].isspace():
                pos += 1
            else:
                break
        start = pos
        while pos < len(data) and not data[pos:pos + 1].isspace():
            pos += 1
        return data[start:pos].decode("ascii", "replace")

    if token() != "P5":
        raise DecodeError(f"{path}: not a P5 PGM")
    try:
        cols, rows, maxval = int(token()), int(token()), int(token())
    except ValueError:
        raise DecodeError(f"{path}: malformed PGM header")
    if maxval != 255:
        raise UnsupportedFormat(f"{path}: PGM maxval must be 255")
    if rows <= 0 or cols <= 0:
        raise DecodeError(f"{path}: bad PGM size")
    pos += 1
    need = rows * cols
    if len(data) - pos < need:
        raise DecodeError(f"{path}: truncated PGM data")
    return np.frombuffer(data, np.uint8, need, pos).reshape(rows, cols).copy()


def _chunk(kind: bytes, body: bytes) -> bytes:
    return struct.pack(">I", len(body)) + kind + body + struct.pack(">I", zlib.crc32(kind + body) & 0xFFFFFFFF)


def png_bytes(img: np.ndarray) -> bytes:
    img = np.ascontiguousarray(img, np.uint8)
    rows, cols = img.shape
    ihdr = struct.pack(">IIBBBBB", cols, rows, 8, 0, 0, 0, 0)
    raw = np.concatenate([np.zeros((rows, 1), np.uint8), img], axis=1).tobytes()
    return (b"\x89PNG\r\n\x1a\n" + _chunk(b"IHDR", ihdr) + _chunk(b"IDAT", zlib.compress(raw, 6))
            + _chunk(b"IEND", b""))


def write_png(path: str, img: np.ndarray):
    with open(path, "wb") as f:
        f.write(png_bytes(img))


def _paeth(a: int, b: int, c: int) -> int:
    p = a + b - c
    pa, pb, pc = abs(p - a), abs(p - b), abs(p - c)
    if pa <= pb and pa <= pc:
        return a
    return b if pb <= pc else c


def read_png(path: str) -> np.ndarray:
    data = open(path, "rb").read()
    if data[:8] != b"\x89PNG\r\n\x1a\n":
        raise DecodeError(f"{path}: not a PNG")
    pos, z, ihdr = 8, bytearray(), None
    while pos + 8 <= len(data):
        (length,) = struct.unpack(">I", data[pos:pos + 4])
        kind = data[pos + 4:pos + 8]
        if pos + 12 + length > len(data):
            raise DecodeError(f"{path}: truncated chunk")
        body = data[pos + 8:pos + 8 + length]
        if kind == b"IHDR":
            ihdr = struct.unpack(">IIBBBBB", body[:13])
            if ihdr[6] != 0:
                raise UnsupportedFormat(f"{path}: interlaced PNG")
        elif kind == b"IDAT":
            z += body
        elif kind == b"IEND":
            break
        pos += 12 + length
    if ihdr is None or ihdr[0] <= 0 or ihdr[1] <= 0:
        raise DecodeError(f"{path}: no IHDR")
    width, height, depth, ctype = ihdr[0], ihdr[1], ihdr[2], ihdr[3]
    if depth != 8 or ctype not in (0, 2):
        raise UnsupportedFormat(f"{path}: only 8-bit gray or RGB PNG supported")
    bpp = 1 if ctype == 0 else 3
    stride = width * bpp
    try:
        raw = zlib.decompress(bytes(z))
    except zlib.error:
        raise DecodeError(f"{path}: inflate failed")
    if len(raw) != height * (stride + 1):
        raise DecodeError(f"{path}: inflate failed")
    prev = [0] * stride
    out = np.zeros((height, width), np.uint8)
    for i in range(height):
        row = raw[i * (stride + 1):(i + 1) * (stride + 1)]
        f, s = row[0], row[1:]
        line = [0] * stride
        for x in range(stride):
            a = line[x - bpp] if x >= bpp else 0
            b = prev[x]
            c = prev[x - bpp] if x >= bpp else 0
            v = s[x]
            if f == 1:
                v += a
            elif f == 2:
                v += b
            elif f == 3:
                v += (a + b) // 2
            elif f == 4:
                v += _paeth(a, b, c)
            elif f != 0:
                raise DecodeError(f"{path}: bad filter type")
            line[x] = v & 0xFF
        prev = line
        arr = np.asarray(line, np.float64)
        if ctype == 0:
            out[i] = arr.astype(np.uint8)
        else:
            y = 0.299 * arr[0::3] + 0.587 * arr[1::3] + 0.114 * arr[2::3]
            out[i] = lround(y).astype(np.uint8)
    return out


def lround(y: np.ndarray) -> np.ndarray:
    """std::lround: round half away from zero, exactly (no y + 0.5 rounding)."""
    y = np.asarray(y, np.float64)
    a = np.abs(y)
    r = np.floor(a)
    r = r + ((a - r) >= 0.5)
    return np.copysign(r, y).astype(np.int64)


def load_grayscale(path: str, target_size: Optional[int] = None) -> np.ndarray:
    """[0,1] float64 raster (image.hpp:273-290)."""
    head = open(path, "rb").read(2)
    if len(head) < 2:
        raise DecodeError(f"{path}: empty file")
    if head == b"P5":
        img = read_pgm(path)
    elif head[0] == 137 and head[1:2] == b"P":
        img = read_png(path)
    else:
        raise UnsupportedFormat(f"{path}: expected PGM (P5) or PNG")
    g = img.astype(np.float64) / 255.0
    if target_size and (target_size != g.shape[0] or target_size != g.shape[1]):
        g = resize_nearest(g, target_size, target_size)
    return g


def load_image_u8(path: str, target_size: Optional[int] = None) -> np.ndarray:
    """The 8-bit raster load_grayscale scales by 1/255 (same pixel selection),
    for the device-side typ=3 init (Simulator.init_image)."""
    head = open(path, "rb").read(2)
    if len(head) < 2:
        raise DecodeError(f"{path}: empty file")
    if head == b"P5":
        img = read_pgm(path)
    elif head[0] == 137 and head[1:2] == b"P":
        img = read_png(path)
    else:
        raise UnsupportedFormat(f"{path}: expected PGM (P5) or PNG")
    if target_size and (target_size != img.shape[0] or target_size != img.shape[1]):
        img = resize_nearest(img, target_size, target_size)
    return np.ascontiguousarray(img)


def resize_nearest(src: np.ndarray, rows: int, cols: int) -> np.ndarray:
    si = (np.arange(rows, dtype=np.int64) * src.shape[0]) // rows
    sj = (np.arange(cols, dtype=np.int64) * src.shape[1]) // cols
    return src[si][:, sj]


def normalize_frame(layer: np.ndarray, lo: Optional[float] = None, hi: Optional[float] = None
                    ) -> Tuple[np.ndarray, float, float]:
    """Host form of normalize_frame(_fixed) (frame.hpp:28-66), for host data."""
    x = np.asarray(layer, np.float64)
    if lo is None or hi is None:
        lo, hi = float(x.min()), float(x.max())
    if not hi > lo:
        return np.full(x.shape, 128, np.uint8), lo, hi
    scale = 255.0 / (hi - lo)
    return np.clip(lround((x - lo) * scale), 0, 255).astype(np.uint8), lo, hi
