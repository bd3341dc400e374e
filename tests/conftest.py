import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: multi-second CPU work")


def load_hex_keys(name: str) -> np.ndarray:
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            rows.append(bytes.fromhex(line))
    return np.array([list(r) for r in rows], dtype=np.uint8)


def load_bit_rows(name: str) -> np.ndarray:
    bits = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            for tok in line.split():
                bits.append(int(tok, 2))
    return np.array(bits, dtype=np.uint8)


def positions(mask) -> set:
    """Set bit positions of a key-layout mask (bit 0 = MSB of byte 0)."""
    m = np.unpackbits(np.asarray(mask, dtype=np.uint8))
    return set(int(i) for i in np.nonzero(m)[0])


def mask_from(pos, B: int) -> np.ndarray:
    bits = np.zeros(8 * B, np.uint8)
    for p in pos:
        bits[p] = 1
    return np.packbits(bits)


@pytest.fixture(scope="session", autouse=True)
def _cpu_libs():
    import cksgen
    import oracle
    cksgen.build()
    oracle.build()
