"""Independent string oracles for the acceptance criteria (test helpers only).

Direct scanning, Hamming windows and a banded anchored edit distance, written
from their definitions (the reference keeps its own in tests/oracles.py)."""

from __future__ import annotations

import numpy as np


def scan_positions(text: np.ndarray, pat: np.ndarray) -> np.ndarray:
    """Every start position of pat in text (codes), by comparing all windows."""
    m = pat.size
    if m > text.size:
        return np.zeros(0, dtype=np.int64)
    win = np.lib.stride_tricks.sliding_window_view(text, m)
    return np.flatnonzero((win == pat[None, :]).all(axis=1))


def hamming_positions(text: np.ndarray, pat: np.ndarray, z: int) -> np.ndarray:
    """Starts whose equal-length window differs from pat in at most z places."""
    m = pat.size
    if m > text.size:
        return np.zeros(0, dtype=np.int64)
    win = np.lib.stride_tricks.sliding_window_view(text, m)
    return np.flatnonzero((win != pat[None, :]).sum(axis=1) <= z)


def anchored_edit_distance(pat: np.ndarray, window: np.ndarray, band: int) -> int:
    """min over prefix lengths L in [m - band, m + band] of edit(pat, window[:L]),
    both strings anchored at their starts; values above band come back as band + 1."""
    m, w = pat.size, window.size
    big = band + 1
    # D[i][j] = edit distance of pat[:i] and window[:j]
    prev = np.minimum(np.arange(w + 1), big)
    for i in range(1, m + 1):
        cur = np.full(w + 1, big, dtype=np.int64)
        cur[0] = min(i, big)
        for j in range(max(1, i - band), min(w, i + band) + 1):
            cur[j] = min(prev[j - 1] + (pat[i - 1] != window[j - 1]), prev[j] + 1, cur[j - 1] + 1, big)
        prev = cur
    lo, hi = max(0, m - band), min(w, m + band)
    return int(prev[lo:hi + 1].min()) if hi >= lo else big
