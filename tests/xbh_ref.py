"""numpy restatement of the XBH tile record (paper_2408_10284_b200/csrc/kernels/xbh.hpp) — test
infrastructure: encodes a bf16 tile the way the store's encoder must (XB12's 15-exponent window,
package-merge code lengths <= 12 over the 16 symbol counts with leaves before packages on equal
weight, canonical codes by (length, symbol), 512-value segments, escapes ascending) and decodes
records."""
import numpy as np

MAX_LEN = 12
SEG = 512


def align(v, a=16):
    return (v + a - 1) // a * a


def lut_off(n):
    return align(n)


def seg_off(n):
    return lut_off(n) + 2 * (1 << MAX_LEN)


def segments(n):
    return (n + SEG - 1) // SEG


def bits_off(n):
    return align(seg_off(n) + 4 * (segments(n) + 1))


def words(total_bits):
    return (total_bits + 31) // 32 + 2


def build_code(hist):
    """hist[256] exponent counts -> (base, len[16], code[16], lut[4096])."""
    hist = [int(h) for h in hist]
    total = sum(hist)
    best, base = 0, 0
    for b in range(242):
        s = sum(hist[b:b + 15])
        if s > best:
            best, base = s, b
    cnt = hist[base:base + 15] + [total - best]
    leaves = sorted(((cnt[s], s) for s in range(16) if cnt[s]), key=lambda t: t[0])  # stable: (count, symbol)
    leaves = [(w, {s: 1}) for w, s in leaves]
    ln = [0] * 16
    m = len(leaves)
    if m == 1:
        for s in leaves[0][1]:
            ln[s] = 1
    elif m > 1:
        lst = list(leaves)
        for _ in range(MAX_LEN - 1):
            pk = []
            for i in range(0, len(lst) - 1, 2):
                c = dict(lst[i][1])
                for s, k in lst[i + 1][1].items():
                    c[s] = c.get(s, 0) + k
                pk.append((lst[i][0] + lst[i + 1][0], c))
            merged, i, j = [], 0, 0
            while i < len(leaves) or j < len(pk):
                if j >= len(pk) or (i < len(leaves) and leaves[i][0] <= pk[j][0]):
                    merged.append(leaves[i])
                    i += 1
                else:
                    merged.append(pk[j])
                    j += 1
            lst = merged
        for w, c in lst[:2 * m - 2]:
            for s, k in c.items():
                ln[s] += k
    code = [0] * 16
    cur, prev, first = 0, 0, True
    for L in range(1, MAX_LEN + 1):
        for s in range(16):
            if ln[s] != L:
                continue
            if not first:
                cur = (cur + 1) << (L - prev)
            first, prev = False, L
            code[s] = cur
    lut = np.zeros(1 << MAX_LEN, dtype=np.uint16)
    for s in range(16):
        if ln[s]:
            sh = MAX_LEN - ln[s]
            lut[code[s] << sh:(code[s] + 1) << sh] = (((base + s) if s < 15 else 0) & 0xFF) | (ln[s] << 8)
    return base, ln, code, lut


def encode(bits: np.ndarray):
    """bits: uint16 [n] (n % 16 == 0) -> (record bytes, meta dict); meta['format'] 0 if not worth it."""
    v = np.ascontiguousarray(bits, dtype=np.uint16).astype(np.uint32)
    n = v.size
    e = (v >> 7) & 0xFF
    base, ln, code, lut = build_code(np.bincount(e, minlength=256))
    s = e.astype(np.int64) - base
    esc = (s < 0) | (s >= 15)
    sym = np.where(esc, 15, s)
    n_exc = int(esc.sum())
    L = np.asarray(ln, dtype=np.int64)[sym]
    C = np.asarray(code, dtype=np.int64)[sym]
    del s, sym
    end = np.cumsum(L)
    pos = end - L
    total = int(end[-1])
    seg = np.append(pos[::SEG], total).astype(np.uint32)
    nw = words(total)
    exc_off = align(bits_off(n) + 4 * nw)
    nbytes = align(exc_off + 8 * n_exc, 256)
    if n_exc > n // 64 or nbytes >= 2 * n:
        return bits.tobytes(), {"format": 0, "base": base, "n_exc": n_exc, "bytes": 2 * n}
    bitarr = np.zeros(32 * nw, dtype=np.uint8)
    for j in range(MAX_LEN):
        m = L > j
        bitarr[pos[m] + j] = (C[m] >> (L[m] - 1 - j)) & 1
    wbytes = np.packbits(bitarr)  # MSB first; a word's 4 bytes big-endian
    wds = wbytes.view(">u4").astype("<u4")
    lo = (((v >> 8) & 0x80) | (v & 0x7F)).astype(np.uint8)
    idx = np.nonzero(esc)[0].astype(np.uint64)
    exc = (idx << np.uint64(16)) | v[esc].astype(np.uint64)
    rec = np.zeros(nbytes, dtype=np.uint8)
    rec[:n] = lo
    rec[lut_off(n):lut_off(n) + 2 * lut.size] = lut.view(np.uint8)
    rec[seg_off(n):seg_off(n) + 4 * seg.size] = seg.view(np.uint8)
    rec[bits_off(n):bits_off(n) + 4 * nw] = wds.view(np.uint8)
    rec[exc_off:exc_off + 8 * n_exc] = exc.view(np.uint8)
    return rec.tobytes(), {"format": 2, "base": base, "n_exc": n_exc, "nib_off": seg_off(n), "exc_off": exc_off,
                           "bytes": nbytes, "total_bits": total, "len": ln}


def decode(rec: bytes, meta: dict, n: int) -> np.ndarray:
    r = np.frombuffer(rec, dtype=np.uint8)
    if meta["format"] == 0:
        return r[:2 * n].view(np.uint16).copy()
    lut = r[lut_off(n):lut_off(n) + 2 * (1 << MAX_LEN)].view(np.uint16)
    seg = r[seg_off(n):seg_off(n) + 4 * (segments(n) + 1)].view(np.uint32)
    total = int(seg[-1])
    nw = words(total)
    wds = r[bits_off(n):bits_off(n) + 4 * nw].view(np.uint32).astype(">u4")
    bitarr = np.unpackbits(wds.view(np.uint8))
    # walk the codes value by value (vectorised over segments: each segment's position advances
    # independently, one value per step)
    nseg = segments(n)
    p = seg[:-1].astype(np.int64)
    ex = np.zeros(nseg * SEG, dtype=np.uint32)
    weights = (1 << np.arange(MAX_LEN - 1, -1, -1)).astype(np.int64)
    for k in range(SEG):
        idx = p[:, None] + np.arange(MAX_LEN)[None, :]
        peek = (bitarr[np.minimum(idx, bitarr.size - 1)].astype(np.int64) * weights).sum(axis=1)
        ent = lut[peek]
        ex[np.arange(nseg) * SEG + k] = ent & 0xFF
        p += ent >> 8
    ex = ex[:n]
    lo = r[:n].astype(np.uint32)
    out = (((lo & 0x80) << 8) | (ex << 7) | (lo & 0x7F)).astype(np.uint16)
    m = meta["n_exc"]
    exc = r[meta["exc_off"]:meta["exc_off"] + 8 * m].view(np.uint64)
    out[(exc >> np.uint64(16)).astype(np.int64)] = (exc & np.uint64(0xFFFF)).astype(np.uint16)
    return out
