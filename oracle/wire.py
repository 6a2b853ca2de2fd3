"""CPU ORACLE for the SLC1 wire format (NEXT row f2) — TEST INFRASTRUCTURE ONLY.

Plain, bit-string implementation of SPEC's serialize / deserialize (
"the paper does not fix a byte layout", so SPEC's format is the reference)
and of pack_indices (12 bits per index, big-endian bit order,
concatenated, zero-padded to a byte boundary; "12 bits/value").  Also the
conversion from this repo's device record layout (R#6) to SPEC's
CompressedChunk (indices, codes, scale-lo, scale-hi).  Reading R#27:
a 2-bit code symbol is (sign bit, bucket bit) written sign first, i.e. the
symbol value is sign*2 + bucket, packed big-endian like the indices.
Only tests/ may import this module.
"""
from __future__ import annotations

import struct
from typing import List, Sequence, Tuple

MAGIC = b"SLC1"
VERSION = 1
HEADER_BYTES = 4 + 1 + 8 + 16 + 32 + 4  # = 65


class FormatError(ValueError):
    """SPEC format-error: bad magic / version, truncated or trailing bytes."""


class InvalidData(ValueError):
    """SPEC invalid-data: a parsed chunk violates the CompressedChunk invariants."""


def _bits_to_bytes(bits: str) -> bytes:
    bits += "0" * (-len(bits) % 8)
    return bytes(int(bits[i:i + 8], 2) for i in range(0, len(bits), 8))


def _bytes_to_bits(b: bytes) -> str:
    return "".join(format(x, "08b") for x in b)


def pack_indices(indices: Sequence[int], ib: int = 12) -> bytes:
    for i in indices:
        if not 0 <= int(i) < (1 << ib):
            raise ValueError(f"index {i} out of range")  # SPEC invalid-argument
    return _bits_to_bytes("".join(format(int(i), f"0{ib}b") for i in indices))


def unpack_indices(b: bytes, count: int, ib: int = 12) -> List[int]:
    bits = _bytes_to_bits(b)
    return [int(bits[ib * j:ib * j + ib], 2) for j in range(count)]


def pack_codes(codes: Sequence[int]) -> bytes:
    return _bits_to_bytes("".join(format(int(c), "02b") for c in codes))


def unpack_codes(b: bytes, count: int) -> List[int]:
    bits = _bytes_to_bits(b)
    return [int(bits[2 * j:2 * j + 2], 2) for j in range(count)]


def chunk_wire_bytes(count: int, ib: int = 12) -> int:
    return 2 + 2 + 2 + (count * ib + 7) // 8 + (2 * count + 7) // 8


def record_to_chunk(rec, k_eff: int, k: int = 64, ib: int = 12) -> Tuple[List[int], List[int], int, int]:
    """Device record (R#6: index stream bits [ib*j, ib*j+ib) little-endian over
    u32 words, code stream bit 2j = sign and 2j+1 = bucket, last word
    s_lo | s_hi << 16) -> (indices, SPEC code symbols sign*2 + bucket, s_lo bits, s_hi bits)."""
    words = [int(w) for w in rec]
    iw = (k * ib + 31) // 32
    stream = 0
    for i, w in enumerate(words[:iw]):
        stream |= w << (32 * i)
    cstream = 0
    cw = (2 * k + 31) // 32
    for i, w in enumerate(words[iw:iw + cw]):
        cstream |= w << (32 * i)
    idx = [(stream >> (ib * j)) & ((1 << ib) - 1) for j in range(k_eff)]
    codes = [(((cstream >> (2 * j)) & 1) << 1) | ((cstream >> (2 * j + 1)) & 1) for j in range(k_eff)]
    last = words[-1]
    return idx, codes, last & 0xFFFF, last >> 16


def chunk_to_record(idx, codes, lo, hi, k: int = 64, ib: int = 12) -> List[int]:
    iw = (k * ib + 31) // 32
    cw = (2 * k + 31) // 32
    stream = 0
    cstream = 0
    for j, (p, c) in enumerate(zip(idx, codes)):
        stream |= int(p) << (ib * j)
        cstream |= ((int(c) >> 1) & 1) << (2 * j) | (int(c) & 1) << (2 * j + 1)
    words = [(stream >> (32 * i)) & 0xFFFFFFFF for i in range(iw)]
    words += [(cstream >> (32 * i)) & 0xFFFFFFFF for i in range(cw)]
    words.append(int(lo) | int(hi) << 16)
    return words


def encode_chunk(idx, codes, lo: int, hi: int, ib: int = 12) -> bytes:
    return struct.pack(">HHH", len(idx), lo, hi) + pack_indices(idx, ib) + pack_codes(codes)


def _f16_ok(h: int) -> bool:
    return ((h >> 10) & 0x1F) != 0x1F and not (h >> 15)  # finite and >= 0 (+0 allowed)


def _f16_val(h: int) -> float:
    e, m = (h >> 10) & 0x1F, h & 0x3FF
    return m * 2.0 ** -24 if e == 0 else (1024 + m) * 2.0 ** (e - 25)


def serialize(base_round: int, peer_id: bytes, layout_digest: bytes, chunks) -> bytes:
    """magic, version, base-round, peer-id, layout-digest, chunk count,
    then per chunk count, scale-lo, scale-hi, packed indices, packed codes;
    multi-byte integers big-endian."""
    out = [MAGIC, struct.pack(">B", VERSION), struct.pack(">Q", base_round), bytes(peer_id).ljust(16, b"\0")[:16],
           bytes(layout_digest)[:32].ljust(32, b"\0"), struct.pack(">I", len(chunks))]
    for idx, codes, lo, hi in chunks:
        out.append(encode_chunk(idx, codes, lo, hi))
    return b"".join(out)


def deserialize(buf: bytes, chunk_lens: Sequence[int], k_effs: Sequence[int]):
    """Inverse of serialize with SPEC's error classes: bad magic /
    version, truncated or trailing bytes -> FormatError; a chunk whose count is
    not k_eff, indices not strictly increasing or >= the chunk length, or
    scales non-finite / negative / lo > hi -> InvalidData."""
    if len(buf) < HEADER_BYTES:
        raise FormatError("truncated header")
    if buf[:4] != MAGIC:
        raise FormatError("bad magic")
    if buf[4] != VERSION:
        raise FormatError("bad version")
    base_round, = struct.unpack(">Q", buf[5:13])
    peer_id = buf[13:29]
    digest = buf[29:61]
    n, = struct.unpack(">I", buf[61:65])
    if n != len(chunk_lens):
        raise InvalidData("chunk count does not match the layout")
    off = HEADER_BYTES
    chunks = []
    for c in range(n):
        if off + 6 > len(buf):
            raise FormatError("truncated chunk header")
        cnt, lo, hi = struct.unpack(">HHH", buf[off:off + 6])
        if cnt != k_effs[c]:
            raise InvalidData("count != k_eff")
        size = chunk_wire_bytes(cnt)
        if off + size > len(buf):
            raise FormatError("truncated chunk")
        ib_bytes = (cnt * 12 + 7) // 8
        idx = unpack_indices(buf[off + 6:off + 6 + ib_bytes], cnt)
        codes = unpack_codes(buf[off + 6 + ib_bytes:off + size], cnt)
        # padding bits must be zero
        if _bytes_to_bits(buf[off + 6:off + 6 + ib_bytes])[12 * cnt:].strip("0") or \
                _bytes_to_bits(buf[off + 6 + ib_bytes:off + size])[2 * cnt:].strip("0"):
            raise InvalidData("nonzero padding bits")
        if any(b <= a for a, b in zip(idx, idx[1:])) or any(i >= chunk_lens[c] for i in idx):
            raise InvalidData("indices not strictly increasing / out of range")
        if not (_f16_ok(lo) and _f16_ok(hi)) or _f16_val(lo) > _f16_val(hi):
            raise InvalidData("bad scales")
        chunks.append((idx, codes, lo, hi))
        off += size
    if off != len(buf):
        raise FormatError("trailing bytes")
    return base_round, peer_id, digest, chunks
