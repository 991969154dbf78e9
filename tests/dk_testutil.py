"""Shared constants for the test modules (imported as a top-level module)."""

import os

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden", "reference_golden.npz")
FAMILIES = ("gaussian", "exponential", "laplacian")


def malformed_files(raw: bytes):
    """(name, bytes) cases for the loader's error paths; shared by tests/test_loader.py and golden/make_golden.py."""
    hdr = raw[:16]
    u32 = lambda v: int(v).to_bytes(4, "little")  # noqa: E731
    return [
        ("empty", b""),
        ("short_header", raw[:11]),
        ("bad_magic", b"DEANN2\x00\x00" + hdr[8:] + raw[16:]),
        ("bad_magic_quote", b"DE'NN1\x00\n" + hdr[8:] + raw[16:]),
        ("zero_rows", hdr[:8] + u32(0) + hdr[12:16]),
        ("zero_dims", hdr[:8] + hdr[8:12] + u32(0)),
        ("short_payload", raw[:-4]),
        ("long_payload", raw + b"\x00"),
        ("huge_shape", hdr[:8] + u32(4294967295) + u32(4294967295) + raw[16:64]),
    ]
