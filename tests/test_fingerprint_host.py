"""The library's blake2b-16 (csrc/fingerprint.cu, host build) equals hashlib's: CPU only."""

import hashlib

import numpy as np
import pytest

from paper_2303_17503_b200 import _native as nat


@pytest.mark.parametrize("n", [0, 1, 64, 127, 128, 129, 256, 257, 3343, 10000])
def test_blake2b16_matches_hashlib(n):
    L = nat.lib()
    m = np.random.default_rng(n).integers(0, 256, n, dtype=np.uint8)
    out = np.zeros(16, np.uint8)
    assert L.bbk_blake2b16_host(m.ctypes.data, n, out.ctypes.data) == 0
    assert out.tobytes() == hashlib.blake2b(m.tobytes(), digest_size=16).digest()


def test_fingerprint_stride_bounds():
    L = nat.lib()
    # prefix (game id <= 16, scalars 10, p2r 2, rewards 8, packed mask) + encode upper bounds
    assert L.bbk_fingerprint_stride(0, 19) >= 16 + 20 + 46 + 361 * 9 + 20
    assert L.bbk_fingerprint_stride(2, 0) >= 16 + 20 + 584 + 69
    assert all(L.bbk_fingerprint_stride(g, 9) % 16 == 0 for g in range(4))
