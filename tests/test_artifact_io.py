"""Artifact I/O from device buffers: the reference's TPA1
file format (persistence.hpp; persistence.cpp:69-125) with the CRC-32 on the
GPU.  The format is restated here with struct + zlib.crc32 (the same IEEE
CRC-32 as persistence.cpp:16-32); the reference's own persistence tests
(persistence_test.cpp) run against the unchanged host code in
tests/test_reference_suite.py."""
from __future__ import annotations

import os
import struct
import zlib

import numpy as np
import pytest

import paper_1708_02574_b200 as P


def restated_file(scores, fp, c, eps, T) -> bytes:
    body = b"TPA1" + struct.pack("<IQddIQ", 1, len(scores), c, eps, T, fp) + \
        np.ascontiguousarray(scores, "<f8").tobytes()
    return body + struct.pack("<I", zlib.crc32(body))


@pytest.mark.gpu
@pytest.mark.parametrize("size", [0, 1, 15, 16, 4095, 4096, 4097, 1 << 20, (1 << 20) * 3 + 77])
def test_gpu_crc32_matches_zlib(size):
    data = np.random.default_rng(size).integers(0, 256, size, dtype=np.uint8).tobytes()
    assert P.crc32(data) == zlib.crc32(data)


@pytest.mark.gpu
def test_save_is_the_reference_format_and_round_trips(tmp_path):
    g = P.generate_rmat(12, 8, rng_seed=4, policy="uniform")
    art = P.preprocess(g, 0.15, 1e-9, 10)
    f = tmp_path / "a.tpa"
    P.save_artifact(art, f, g)
    raw = f.read_bytes()
    assert len(raw) == 48 + 8 * g.node_count()
    assert raw == restated_file(art.stranger_scores, g.fingerprint(), 0.15, 1e-9, 10)
    back = P.load_artifact(f, g)
    assert np.array_equal(back.stranger_scores, art.stranger_scores)
    assert (back.graph_fingerprint, back.restart_prob, back.tolerance, back.stranger_start) == \
        (g.fingerprint(), 0.15, 1e-9, 10)
    # the loaded artifact answers queries like the original, bit for bit
    s = P.sample_seeds(g, 8, 2)
    assert np.array_equal(P.query_batch(g, back, s, 5), P.query_batch(g, art, s, 5))
    f2 = tmp_path / "b.tpa"
    P.save_artifact(back, f2, g)
    assert f2.read_bytes() == raw


@pytest.mark.gpu
def test_load_errors_in_reference_order(tmp_path):
    g = P.generate_rmat(10, 8, rng_seed=1)
    art = P.preprocess(g, 0.15, 1e-9, 10)
    good = tmp_path / "good.tpa"
    P.save_artifact(art, good, g)
    raw = good.read_bytes()

    def load(data: bytes):
        p = tmp_path / "x.tpa"
        p.write_bytes(data)
        with pytest.raises(RuntimeError) as e:
            P.load_artifact(p, g)
        return str(e.value)

    with pytest.raises(RuntimeError, match="cannot open artifact"):
        P.load_artifact(tmp_path / "missing.tpa", g)
    assert load(raw[:47]).startswith("artifact truncated: ")
    assert load(b"TPA2" + raw[4:]).startswith("bad artifact magic: ")
    assert load(raw[:4] + struct.pack("<I", 2) + raw[8:]) == "unsupported artifact version 2"
    assert load(raw + b"\0") == f"artifact truncated or oversized: expected {len(raw)} bytes, got {len(raw) + 1}"
    flipped = bytearray(raw)
    flipped[100] ^= 1
    assert load(bytes(flipped)).startswith("artifact checksum mismatch: ")
    # a stale artifact (other graph) loads, and the query refuses it (tpa.cpp:63-64)
    g2 = P.generate_rmat(10, 8, rng_seed=2)
    other = P.load_artifact(good, g2)
    with pytest.raises(RuntimeError, match="fingerprint"):
        P.query(g2, other, 0, 5)
