"""The paper's dataset statistics (host arithmetic on a build's outputs; no device work).

Definitions (Sec. 6.2, Table 2; Sec. 6.4, Table 4):
  full sort key        = the key + its 8-byte record id, in 8-byte words:
                         8*ceil(key_bytes/8) + 8 bytes (for variable-length keys the
                         longest key);
  compressed sort key  = the distinction bits of the key + the variant bits of the record id,
                         in 8-byte words: 8*ceil((|D| + rid_bits)/64) bytes;
                         "either the whole or only the variant bits of a record ID can be used"
                         (P:555): with the whole 8-byte record id 8*ceil(|D|/64) + 8 bytes.
                         Reading R18: Table 2 uses the variant bits (all six rows
                         agree), Table 4 the whole record id (its rows 10-20 need it: Zipf(1.5,40,4)
                         has at most 20 x 5 = 100 distinction bits, and 100 + ~25 variant bits fit
                         16 B, not the printed 24 B);
  compression ratio    = full key bits / |D|;
  sort key ratio       = full sort key size / compressed sort key size;
  word comparison ratio = wcc_full / wcc_comp, the average number of 8-byte word comparisons
                         of one full-key comparison over that of one compressed-key
                         comparison. Reading R19: averaged over the
                         comparisons that decide the final order, i.e. the pairs adjacent in
                         sorted order; a pair differing first at key bit d compares
                         d//64 + 1 full-key words and t//64 + 1 compressed words, t = the
                         rank of d in D; an equal pair compares every word including the
                         record id's.
Row ids here are the dense input indices 0..n-1, so rid_bits = bit length of n - 1.
"""
from __future__ import annotations

import numpy as np

DBIT_NONE = 0xFFFF


def rid_bits(n: int) -> int:
    """Variant bits of dense row ids 0..n-1."""
    return max(1, (int(n) - 1).bit_length())


def full_sort_key_bytes(key_bytes: int) -> int:
    return 8 * ((int(key_bytes) + 7) // 8) + 8


def compressed_sort_key_bytes(d_bits: int, rid_variant_bits: int) -> int:
    return 8 * ((int(d_bits) + int(rid_variant_bits) + 63) // 64)


def compressed_sort_key_bytes_whole_rid(d_bits: int) -> int:
    return 8 * ((int(d_bits) + 63) // 64) + 8


def table_stats(key_bytes: int, d_bits: int, rid_variant_bits: int) -> dict:
    """Table 2's rows for one column: full key bits, |D|, rid bits, ratios, sort key sizes."""
    full_bits = 8 * int(key_bytes)
    fs = full_sort_key_bytes(key_bytes)
    cs = compressed_sort_key_bytes(d_bits, rid_variant_bits)
    cw = compressed_sort_key_bytes_whole_rid(d_bits)
    return {"full_key_bits": full_bits, "d_bits": int(d_bits), "rid_variant_bits": int(rid_variant_bits),
            "compression_ratio": full_bits / d_bits if d_bits else None,
            "full_sort_key_bytes": fs, "compressed_sort_key_bytes": cs, "sort_key_ratio": fs / cs,
            "compressed_sort_key_bytes_whole_rid": cw, "sort_key_ratio_whole_rid": fs / cw}


def word_comparisons(dbit: np.ndarray, mask: np.ndarray, key_bytes: int, rid_variant_bits: int) -> dict:
    """Average 8-byte word comparisons per key comparison over the adjacent pairs of the sorted
    order (reading R19): dbit = D_i of positions 1..n-1 (u16, DBIT_NONE for equal keys),
    mask = the exact D-bitmap (u8[key_bytes], bit p = MSB-first position p)."""
    db = np.asarray(dbit, dtype=np.uint16)[1:]
    B = int(key_bytes)
    bits = np.unpackbits(np.asarray(mask, dtype=np.uint8))[:8 * B]
    d = int(bits.sum())
    if db.size == 0:
        return {"wcc_full": None, "wcc_comp": None, "word_comparison_ratio": None}
    rank = np.cumsum(bits) - 1                        # rank[p] = index of position p within D
    eq = db == DBIT_NONE
    pos = db.astype(np.int64)
    pos[eq] = 0
    full = np.where(eq, (B + 7) // 8 + 1, pos // 64 + 1)
    comp = np.where(eq, (d + int(rid_variant_bits) + 63) // 64, rank[pos] // 64 + 1)
    wf, wc = float(full.mean()), float(comp.mean())
    return {"wcc_full": wf, "wcc_comp": wc, "word_comparison_ratio": wf / wc}
