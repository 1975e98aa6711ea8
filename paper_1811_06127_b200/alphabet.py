"""2-bit DNA alphabet: symbol codes, pattern gate and packing.

Mirrors the reference's alphabet module (alphabet.py:8-95): codes A<C<G<T =
0..3, lowercase accepted (13-14), character j of a packed sequence in bits
2(j%4).. of byte j//4 (53-56).  Adds vectorised numpy forms used by the
batched GPU entry points (pattern gate a9 of SURVEY §8a).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Iterable, Sequence

import numpy as np

SYMBOLS = "ACGT"
A, C, G, T = 0, 1, 2, 3

CODE_OF = {ch: i for i, ch in enumerate(SYMBOLS)}
CODE_OF.update({ch.lower(): i for i, ch in enumerate(SYMBOLS)})

TERMINATOR = "$"
CHARS_PER_BYTE = 4

# byte -> code, 255 for anything outside ACGT/acgt
_LUT = np.full(256, 255, dtype=np.uint8)
for _ch, _code in CODE_OF.items():
    _LUT[ord(_ch)] = _code


class AlphabetError(ValueError):
    """A character outside A/C/G/T (either case) was encountered."""


def encode(text: str) -> list[int]:
    """Map a DNA string to symbol codes, rejecting anything outside ACGT."""
    return encode_array(text).tolist()


def encode_array(text: str | bytes) -> np.ndarray:
    """Vectorised encode: uint8 codes, AlphabetError on the first bad character."""
    if isinstance(text, str):
        try:
            raw = text.encode("ascii")
        except UnicodeEncodeError:
            for i, ch in enumerate(text):
                if ch not in CODE_OF:
                    raise AlphabetError(
                        f"invalid character {ch!r} at position {i}; expected one of ACGT"
                    ) from None
            raise
    else:
        raw = bytes(text)
    codes = _LUT[np.frombuffer(raw, dtype=np.uint8)]
    bad = np.flatnonzero(codes == 255)
    if bad.size:
        i = int(bad[0])
        ch = text[i] if isinstance(text, str) else chr(raw[i])
        raise AlphabetError(f"invalid character {ch!r} at position {i}; expected one of ACGT")
    return codes


def decode(codes: Iterable[int]) -> str:
    return "".join(SYMBOLS[c] for c in codes)


def is_dna(text: str) -> bool:
    """True when every character of `text` is A/C/G/T (either case)."""
    try:
        raw = text.encode("ascii")
    except UnicodeEncodeError:
        return False
    return bool((_LUT[np.frombuffer(raw, dtype=np.uint8)] != 255).all())


@dataclass(frozen=True)
class PackedText:
    """2-bit packed character sequence, four characters per byte."""

    data: bytes
    length: int

    def __post_init__(self) -> None:
        expected = (self.length + CHARS_PER_BYTE - 1) // CHARS_PER_BYTE
        if len(self.data) != expected:
            raise ValueError(f"packed size {len(self.data)} does not match length {self.length}")

    def char_code(self, j: int) -> int:
        if not 0 <= j < self.length:
            raise IndexError(f"position {j} out of range for length {self.length}")
        return (self.data[j >> 2] >> ((j & 3) << 1)) & 3


def pack_codes(codes: Sequence[int], pad_to: int | None = None) -> bytes:
    """Pack 2-bit codes into bytes, low-order fields first; zero-pad to `pad_to`."""
    arr = np.asarray(codes, dtype=np.uint8) & 3
    nbytes = (arr.size + CHARS_PER_BYTE - 1) // CHARS_PER_BYTE
    padded = np.zeros(nbytes * CHARS_PER_BYTE, dtype=np.uint8)
    padded[: arr.size] = arr
    quads = padded.reshape(-1, 4)
    out = (quads[:, 0] | (quads[:, 1] << 2) | (quads[:, 2] << 4) | (quads[:, 3] << 6)).tobytes()
    if pad_to is not None:
        if len(out) > pad_to:
            raise ValueError(f"{arr.size} characters do not fit in {pad_to} bytes")
        out += b"\x00" * (pad_to - len(out))
    return out


def pack_2bit(chars: str) -> PackedText:
    return PackedText(data=pack_codes(encode_array(chars)), length=len(chars))


def unpack_2bit(packed: PackedText) -> str:
    return "".join(SYMBOLS[packed.char_code(j)] for j in range(packed.length))


def pack_patterns_u64(codes: np.ndarray) -> np.ndarray:
    """(N, m) uint8 codes with m <= 32 -> N uint64, character j in bits 2j..2j+1."""
    codes = np.ascontiguousarray(codes, dtype=np.uint8)
    n, m = codes.shape
    if not 1 <= m <= 32:
        raise ValueError("packed patterns need 1 <= m <= 32")
    out = np.zeros(n, dtype=np.uint64)
    for j in range(m):
        out |= (codes[:, j].astype(np.uint64) & np.uint64(3)) << np.uint64(2 * j)
    return out


def patterns_to_csr(patterns) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """Patterns (list of str, or 2-D uint8 code array) -> (codes, offsets, degenerate).

    Degenerate patterns (characters outside ACGT, search.py:85-86, 117-118) are
    flagged and their bad characters replaced by A so the batch stays
    well-formed; callers overwrite their results.  Empty patterns raise
    ValueError (search.py:83-84, 115-116).
    """
    if isinstance(patterns, np.ndarray):
        if patterns.ndim != 2 or patterns.shape[1] == 0:
            raise ValueError("pattern is empty")
        codes = np.ascontiguousarray(patterns, dtype=np.uint8)
        if codes.size and codes.max() > 3:
            raise ValueError("symbol code outside [0, 4)")
        n, m = codes.shape
        offsets = np.arange(0, (n + 1) * m, m, dtype=np.uint64)
        return codes.reshape(-1), offsets, np.zeros(n, dtype=bool)
    pats = list(patterns)
    lengths = np.fromiter((len(p) for p in pats), dtype=np.int64, count=len(pats))
    if (lengths == 0).any():
        raise ValueError("pattern is empty")
    joined = "".join(pats)
    raw = np.frombuffer(joined.encode("ascii", "replace"), dtype=np.uint8)
    if raw.size != int(lengths.sum()):  # non-ASCII: fall back to per-pattern bytes
        raw = np.frombuffer(b"".join(p.encode("ascii", "replace") for p in pats), dtype=np.uint8)
    codes = _LUT[raw]
    offsets = np.zeros(len(pats) + 1, dtype=np.uint64)
    np.cumsum(lengths, out=offsets[1:])
    bad = codes == 255
    degenerate = np.zeros(len(pats), dtype=bool)
    if bad.any():
        idx = np.searchsorted(offsets[1:], np.flatnonzero(bad), side="right")
        degenerate[idx] = True
        codes = codes.copy()
        codes[bad] = 0
    return codes, offsets, degenerate
