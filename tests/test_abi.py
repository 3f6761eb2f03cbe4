"""The C-ABI library builds, loads without a GPU and exports every symbol
declared in include/splatstream_b200.h (no compute calls here)."""

import ctypes
import re

from conftest import ROOT


def declared_symbols():
    text = (ROOT / "include" / "splatstream_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ss_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_header():
    from paper_2604_02851_b200 import _lib
    lib = _lib.load_library()
    names = declared_symbols()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    assert lib.ss_abi_version() == 1
    offs = (ctypes.c_int64 * 5)()
    assert lib.ss_grad_layout(1000, 3, offs) == 1000 * 59
    assert list(offs) == [0, 3000, 6000, 10000, 11000]


def test_bounds_and_host_zlib_match_python():
    import zlib
    import numpy as np
    from paper_2604_02851_b200 import _lib
    from paper_2604_02851_b200.protocol import host_zlib
    lib = _lib.load_library()
    assert lib.ss_delta_bound(0, 10, 3) >= 24 + 60
    assert lib.ss_snapshot_bound(10, 3, 1) == 40 + (52 + 12 * 16) * 10
    rng = np.random.default_rng(0)
    for n in (0, 1, 1000, 100000):
        blk = rng.integers(0, 40, n).astype(np.uint8).tobytes()
        assert host_zlib(blk) == zlib.compress(blk, 6)


def test_parallel_host_zlib_is_byte_identical():
    """blocks deflated on parallel threads equal Python's
    zlib.compress(block, 6), the reference's compression stage."""
    import os
    import zlib
    from paper_2604_02851_b200.protocol import compress_blocks, host_zlib
    blocks = [os.urandom(5000) * 40 + bytes(100000), b"", b"\x00", os.urandom(70000)]
    assert compress_blocks(blocks) == [zlib.compress(b, 6) for b in blocks]
    assert host_zlib(blocks[0]) == zlib.compress(blocks[0], 6)
