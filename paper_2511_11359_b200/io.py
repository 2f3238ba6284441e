"""Instance file formats -- drop-in for leanot.io (data formats only).

Same names, arguments, return values and ValueError cases as
/root/reference/pkg/src/leanot/io.py:
  read_pgm / write_pgm           P2 (ASCII) and P5 (binary, 8- or 16-bit big-endian) PGM,
                                 header comments, row-major pixels (io.py:21-80)
  read_histogram_csv /           one value per line, optional non-numeric first line
  write_histogram_csv            (io.py:83-105)
  write_matrix_csv               one row per line, comma separated (io.py:108-112)
  block_mean_downsample          mean over non-overlapping f x f blocks (io.py:115-123)
Host code: these parse and write files; the histograms they produce feed the solvers.
"""

from __future__ import annotations

import numpy as np

__all__ = ["read_pgm", "write_pgm", "read_histogram_csv", "write_histogram_csv", "write_matrix_csv",
           "block_mean_downsample"]

_WS = b" \t\n\r\x0b\x0c"


def _header(buf: bytes):
    """(magic, width, height, maxval, offset of the first pixel byte) -- io.py:41-67."""
    magic = buf[:2]
    if magic not in (b"P2", b"P5"):
        raise ValueError("not a P2/P5 PGM file")
    vals: list[bytes] = []
    pos, end = 2, len(buf)
    while pos < end and len(vals) < 3:
        c = buf[pos]
        if c == 0x23:                                    # '#': comment to end of line
            nl = [k for k in (buf.find(b"\n", pos), buf.find(b"\r", pos)) if k >= 0]
            pos = min(nl) if nl else end
        elif c in _WS:
            pos += 1
        else:
            stop = pos
            while stop < end and buf[stop] not in _WS:
                stop += 1
            vals.append(buf[pos:stop])
            pos = stop
    if len(vals) < 3:
        raise ValueError("truncated PGM header")
    width, height, maxval = map(int, vals)
    if min(width, height) <= 0 or maxval <= 0 or maxval >= 65536:
        raise ValueError("invalid PGM dimensions")
    return magic, width, height, maxval, pos + 1       # exactly one separator byte after maxval


def read_pgm(path) -> np.ndarray:
    """Grayscale PGM as a float (height, width) array."""
    with open(path, "rb") as fh:
        buf = fh.read()
    magic, width, height, maxval, off = _header(buf)
    count = width * height
    if magic == b"P5":
        px = np.frombuffer(buf, dtype=">u2" if maxval > 255 else "u1", count=count, offset=off).astype(float)
    else:
        words = buf[off:].split()
        if len(words) < count:
            raise ValueError("truncated P2 image")
        px = np.array(words[:count], dtype=float)
    if count and px.max() > maxval:
        raise ValueError("pixel value exceeds declared maxval")
    return px.reshape(height, width)


def write_pgm(path, pixels, maxval: int = 255, rescale: bool = True) -> None:
    """Binary P5, [0, max(pixels)] mapped linearly to [0, maxval] and rounded half-to-even.

    rescale=False writes the values as they are (rounded, clipped to [0, maxval]): the
    reference CLI's `downsample` passes it (cli.py:397) but its write_pgm lacks the
    parameter; the default keeps the reference behaviour."""
    img = np.asarray(pixels, dtype=float)
    if img.ndim != 2:
        raise ValueError("expected a 2-D image")
    peak = img.max()
    if not rescale:
        q = img
    else:
        q = np.zeros(img.shape) if peak <= 0 else img / peak * maxval
    q = np.clip(np.rint(q), 0, maxval).astype(">u2" if maxval >= 256 else "u1")
    head = b"P5\n%d %d\n%d\n" % (img.shape[1], img.shape[0], maxval)
    with open(path, "wb") as fh:
        fh.write(head + q.tobytes())


def read_histogram_csv(path) -> np.ndarray:
    """One float per line; blank lines skipped; a non-numeric FIRST line is a header."""
    out = []
    with open(path) as fh:                       # text mode: \r\n and \r arrive as \n
        lines = fh.read().split("\n")
    for k, raw in enumerate(lines):
        item = raw.strip()
        if item == "":
            continue
        try:
            out.append(float(item))
        except ValueError:
            if k != 0:
                raise ValueError(f"{path}: bad value on line {k + 1}: {item!r}") from None
    if len(out) == 0:
        raise ValueError(f"{path}: no histogram values")
    return np.array(out)


def write_histogram_csv(path, weights) -> None:
    flat = np.asarray(weights, dtype=float).reshape(-1)
    with open(path, "w") as fh:
        fh.write("".join("%.17g\n" % v for v in flat))


def write_matrix_csv(path, matrix) -> None:
    rows = np.asarray(matrix, dtype=float)
    with open(path, "w") as fh:
        for row in rows:
            fh.write(",".join("%.17g" % v for v in row) + "\n")


def block_mean_downsample(pixels, factor: int) -> np.ndarray:
    """Mean of each non-overlapping factor x factor block; factor must divide both sides."""
    img = np.asarray(pixels, dtype=float)
    if factor < 1:
        raise ValueError("factor must be >= 1")
    h, w = img.shape
    if h % factor or w % factor:
        raise ValueError(f"factor {factor} does not divide image dimensions {h}x{w}")
    return img.reshape(h // factor, factor, w // factor, factor).mean(axis=(1, 3))
