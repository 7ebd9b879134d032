"""numpy restatement of the XBH tile record (paper_2408_10284_b200/csrc/kernels/xbh.hpp) — test
infrastructure: encodes a bf16 tile the way the store's encoder must (XB12's 15-exponent window,
package-merge code lengths <= 12 over the 16 symbol counts with leaves before packages on equal
weight, canonical codes by (length, symbol), single- and multi-code tables, 128-bit chunk gaps and
per-block value bases, escapes ascending) and decodes records."""
import numpy as np

MAX_LEN = 12
MULTI = 5             # codes per multi-code table entry
CHUNK = 128           # bits per independently decodable chunk
BLOCK = 256 * CHUNK   # bits per output-base entry


def align(v, a=16):
    return (v + a - 1) // a * a


def lut_off(n):
    return align(n)


def mlut_off(n):
    return lut_off(n) + 2 * (1 << MAX_LEN)


def hdr_off(n):
    return mlut_off(n) + 4 * (1 << MAX_LEN)


def bits_off(n):
    return hdr_off(n) + 16


def words(total_bits):
    return (total_bits + 31) // 32 + 8


def chunks(bits):
    return (bits + CHUNK - 1) // CHUNK


def blocks(bits):
    return (bits + BLOCK - 1) // BLOCK


def gap_off(n, bits):
    return align(bits_off(n) + 4 * words(bits))


def base_off(n, bits):
    return align(gap_off(n, bits) + 4 * ((chunks(bits) + 7) // 8))


def build_code(hist):
    """hist[256] exponent counts -> (base, len[16], code[16], lut[4096], mlut[4096])."""
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
    sym_lut = np.zeros(1 << MAX_LEN, dtype=np.int64)  # symbol | length << 8
    for s in range(16):
        if ln[s]:
            sh = MAX_LEN - ln[s]
            sym_lut[code[s] << sh:(code[s] + 1) << sh] = s | (ln[s] << 8)
    # multi-code table: up to 5 consecutive codes ending inside the 12-bit peek: symbols (4 bits
    # each) | count << 20 | first length << 23 | total length << 27
    mlut = np.zeros(1 << MAX_LEN, dtype=np.uint32)
    for i in range(1 << MAX_LEN):
        L = syms = first = cnt = 0
        for k in range(MULTI):
            if L >= MAX_LEN:
                break
            e = int(sym_lut[(i << L) & ((1 << MAX_LEN) - 1)])
            l2 = e >> 8
            if l2 == 0 or L + l2 > MAX_LEN:
                break
            syms |= (e & 15) << (4 * k)
            if k == 0:
                first = l2
            cnt += 1
            L += l2
        mlut[i] = syms | (cnt << 20) | (first << 23) | (L << 27)
    return base, ln, code, lut, mlut


def encode(bits: np.ndarray):
    """bits: uint16 [n] (n % 16 == 0) -> (record bytes, meta dict); meta['format'] 0 if not worth it."""
    v = np.ascontiguousarray(bits, dtype=np.uint16).astype(np.uint32)
    n = v.size
    e = (v >> 7) & 0xFF
    base, ln, code, lut, mlut = build_code(np.bincount(e, minlength=256))
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
    nw = words(total)
    nb = blocks(total)
    exc_off = align(base_off(n, total) + 4 * (nb + 1))
    nbytes = align(exc_off + 8 * n_exc, 256)
    if n_exc > n // 64 or nbytes >= 2 * n:
        return bits.tobytes(), {"format": 0, "base": base, "n_exc": n_exc, "bytes": 2 * n}
    # chunk gaps: the first code starting in each 128-bit chunk; block bases: its value index
    c = pos // CHUNK
    first = np.ones(n, dtype=bool)
    first[1:] = c[1:] != c[:-1]
    gaps = np.zeros(chunks(total), dtype=np.uint32)
    gaps[c[first]] = (pos[first] - c[first] * CHUNK).astype(np.uint32)
    gw = np.zeros((chunks(total) + 7) // 8, dtype=np.uint32)
    for k in range(8):
        part = gaps[k::8]
        gw[:part.size] |= part << np.uint32(4 * k)
    idx_first = np.nonzero(first)[0]
    blk_first = (c[first] % 256) == 0
    bases = list(idx_first[blk_first])
    cl = chunks(total) - 1
    if c[-1] != cl:  # the last code runs into a final chunk where no code starts
        gaps[cl] = total - cl * CHUNK
        gw[cl >> 3] |= np.uint32(gaps[cl]) << np.uint32(4 * (cl & 7))
        if cl % 256 == 0:
            bases.append(n)
    bases = np.array(bases + [n], dtype=np.uint32)
    assert bases.size == nb + 1
    bitarr = np.zeros(32 * nw, dtype=np.uint8)
    for j in range(MAX_LEN):
        m = L > j
        bitarr[pos[m] + j] = (C[m] >> (L[m] - 1 - j)) & 1
    wds = np.packbits(bitarr).view(">u4").astype("<u4")  # MSB first; a word's 4 bytes big-endian
    lo = (((v >> 8) & 0x80) | (v & 0x7F)).astype(np.uint8)
    idx = np.nonzero(esc)[0].astype(np.uint64)
    exc = (idx << np.uint64(16)) | v[esc].astype(np.uint64)
    rec = np.zeros(nbytes, dtype=np.uint8)
    rec[:n] = lo
    rec[lut_off(n):lut_off(n) + 2 * lut.size] = lut.view(np.uint8)
    rec[mlut_off(n):mlut_off(n) + 4 * mlut.size] = mlut.view(np.uint8)
    rec[hdr_off(n):hdr_off(n) + 16] = np.array([total, n_exc], dtype=np.uint64).view(np.uint8)
    rec[bits_off(n):bits_off(n) + 4 * nw] = wds.view(np.uint8)
    rec[gap_off(n, total):gap_off(n, total) + 4 * gw.size] = gw.view(np.uint8)
    rec[base_off(n, total):base_off(n, total) + 4 * bases.size] = bases.view(np.uint8)
    rec[exc_off:exc_off + 8 * n_exc] = exc.view(np.uint8)
    return rec.tobytes(), {"format": 2, "base": base, "n_exc": n_exc, "nib_off": hdr_off(n), "exc_off": exc_off,
                           "bytes": nbytes, "total_bits": total, "len": ln}


def decode(rec: bytes, meta: dict, n: int) -> np.ndarray:
    """The GPU decoder's scheme: every chunk walks the multi-code table from its gap, keeping the
    codes that start inside it; chunk outputs are concatenated in order (value positions = prefix
    sums of the chunk counts, checked against the block bases)."""
    r = np.frombuffer(rec, dtype=np.uint8)
    if meta["format"] == 0:
        return r[:2 * n].view(np.uint16).copy()
    mlut = r[mlut_off(n):mlut_off(n) + 4 * (1 << MAX_LEN)].view(np.uint32).astype(np.int64)
    total, n_exc = (int(x) for x in r[hdr_off(n):hdr_off(n) + 16].view(np.uint64))
    nw = words(total)
    bitarr = np.unpackbits(r[bits_off(n):bits_off(n) + 4 * nw].view(np.uint32).astype(">u4").view(np.uint8))
    nc = chunks(total)
    gw = r[gap_off(n, total):gap_off(n, total) + 4 * ((nc + 7) // 8)].view(np.uint32)
    gaps = np.array([(int(gw[c >> 3]) >> (4 * (c & 7))) & 15 for c in range(nc)], dtype=np.int64)
    bases = r[base_off(n, total):base_off(n, total) + 4 * (blocks(total) + 1)].view(np.uint32)
    base = meta["base"]
    cid = np.arange(nc, dtype=np.int64)
    pos = cid * CHUNK + gaps
    stop = np.minimum((cid + 1) * CHUNK, total)
    weights = (1 << np.arange(MAX_LEN - 1, -1, -1)).astype(np.int64)
    out_syms = [[] for _ in range(nc)]
    active = pos < stop
    while active.any():
        ids = np.nonzero(active)[0]
        p = pos[ids]
        peek = (bitarr[p[:, None] + np.arange(MAX_LEN)[None, :]].astype(np.int64) * weights).sum(axis=1)
        e = mlut[peek]
        whole = p + MAX_LEN <= stop[ids]  # every code of the entry starts inside the chunk
        k = np.where(whole, (e >> 20) & 7, 1)
        adv = np.where(whole, e >> 27, (e >> 23) & 15)
        for j, i in enumerate(ids):
            for q in range(int(k[j])):
                out_syms[i].append((int(e[j]) >> (4 * q)) & 15)
        pos[ids] = p + adv
        active = pos < stop
    counts = np.array([len(x) for x in out_syms], dtype=np.int64)
    starts = np.concatenate([[0], np.cumsum(counts)])
    assert starts[-1] == n
    assert np.array_equal(starts[::256][: bases.size - 1], bases[:-1].astype(np.int64))
    syms = np.concatenate([np.array(x, dtype=np.uint32) for x in out_syms])
    ex = (base + syms) & 0xFF
    lo = r[:n].astype(np.uint32)
    out = (((lo & 0x80) << 8) | (ex << 7) | (lo & 0x7F)).astype(np.uint16)
    exc = r[meta["exc_off"]:meta["exc_off"] + 8 * n_exc].view(np.uint64)
    out[(exc >> np.uint64(16)).astype(np.int64)] = (exc & np.uint64(0xFFFF)).astype(np.uint16)
    return out
