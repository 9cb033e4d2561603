"""TEST INFRASTRUCTURE ONLY — independent numpy reader of the TSFSNAP1 snapshot
format (layout documented in paper_1607_02904_b200/csrc/tsf_snapshot.cpp).

Used where the product must not be loaded: the oracle side of the parity
tests and ``bench.py --impl reference`` (the reference arm reads the same
fixture bytes the GPU arm evaluates).  It also cross-checks the product's
reader and writer (tests/test_host.py).
"""
from __future__ import annotations

import hashlib

import numpy as np

MAGIC = b"TSFSNAP1"
F32_COORDS, VELOCITIES = 0x1, 0x2


def read(path: str) -> dict:
    raw = open(path, "rb").read()
    if len(raw) < 56 + 32 or raw[:8] != MAGIC:
        raise ValueError(f"{path}: not a TSFSNAP1 snapshot")
    body, sha = raw[:-32], raw[-32:]
    if hashlib.sha256(body).digest() != sha:
        raise ValueError(f"{path}: SHA-256 mismatch")
    flags = int(np.frombuffer(body, "<u4", 1, 8)[0])
    ns = int(np.frombuffer(body, "<i4", 1, 12)[0])
    n = int(np.frombuffer(body, "<i8", 1, 16)[0])
    box = np.frombuffer(body, "<f8", 3, 24).copy()
    per = np.frombuffer(body, np.uint8, 3, 48).copy()
    at = 56
    masses = np.frombuffer(body, "<f8", ns, at).copy()
    at += 8 * ns
    if flags & F32_COORDS:
        xyz = np.frombuffer(body, "<f4", 3 * n, at).astype(np.float64).reshape(n, 3)
        at += 12 * n
    else:
        xyz = np.frombuffer(body, "<f8", 3 * n, at).copy().reshape(n, 3)
        at += 24 * n
    species = np.frombuffer(body, np.uint8, n, at).astype(np.int32)
    at += n
    vel = None
    if flags & VELOCITIES:
        vel = np.frombuffer(body, "<f8", 3 * n, at).copy().reshape(n, 3)
        at += 24 * n
    if at != len(body):
        raise ValueError(f"{path}: size does not match header")
    return {"positions": xyz, "species": species, "masses": masses, "box": box,
            "periodic": per, "velocities": vel, "flags": flags, "sha256": sha.hex()}
