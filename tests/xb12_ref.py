"""numpy restatement of the XB12 tile record (paper_2408_10284_b200/csrc/kernels/xb12.hpp) — test
infrastructure: encodes a bf16 tile the way the GPU encoder must (window = first of the best 15
consecutive exponents, lowest on ties; escapes ascending) and decodes records."""
import numpy as np


def align(v, a=16):
    return (v + a - 1) // a * a


def encode(bits: np.ndarray):
    """bits: uint16 [n] (n % 16 == 0) -> (record bytes, meta dict); meta['format'] 0 if not worth it."""
    v = np.ascontiguousarray(bits, dtype=np.uint16).astype(np.uint32)
    n = v.size
    e = (v >> 7) & 0xFF
    hist = np.bincount(e, minlength=256)
    win = np.array([hist[b:b + 15].sum() for b in range(242)])
    base = int(np.argmax(win))  # first maximum
    c = e.astype(np.int64) - base
    esc = (c < 0) | (c >= 15)
    c = np.where(esc, 15, c).astype(np.uint8)
    n_exc = int(esc.sum())
    if n_exc > n // 64:
        return bits.tobytes(), {"format": 0, "base": base, "n_exc": n_exc, "bytes": 2 * n}
    lo = (((v >> 8) & 0x80) | (v & 0x7F)).astype(np.uint8)
    nib = (c[0::2] | (c[1::2] << 4)).astype(np.uint8)
    idx = np.nonzero(esc)[0].astype(np.uint64)
    exc = (idx << np.uint64(16)) | v[esc].astype(np.uint64)
    nib_off = align(n)
    exc_off = align(nib_off + n // 2)
    total = align(exc_off + 8 * n_exc, 256)
    rec = np.zeros(total, dtype=np.uint8)
    rec[:n] = lo
    rec[nib_off:nib_off + n // 2] = nib
    rec[exc_off:exc_off + 8 * n_exc] = exc.view(np.uint8)
    return rec.tobytes(), {"format": 1, "base": base, "n_exc": n_exc, "nib_off": nib_off, "exc_off": exc_off,
                           "bytes": total}


def decode(rec: bytes, meta: dict, n: int) -> np.ndarray:
    r = np.frombuffer(rec, dtype=np.uint8)
    if meta["format"] == 0:
        return r[:2 * n].view(np.uint16).copy()
    lo = r[:n].astype(np.uint32)
    nib = r[meta["nib_off"]:meta["nib_off"] + n // 2]
    c = np.empty(n, dtype=np.uint32)
    c[0::2] = nib & 15
    c[1::2] = nib >> 4
    ex = (meta["base"] + c) & 0xFF
    out = (((lo & 0x80) << 8) | (ex << 7) | (lo & 0x7F)).astype(np.uint16)
    m = meta["n_exc"]
    exc = r[meta["exc_off"]:meta["exc_off"] + 8 * m].view(np.uint64)
    out[(exc >> np.uint64(16)).astype(np.int64)] = (exc & np.uint64(0xFFFF)).astype(np.uint16)
    return out
