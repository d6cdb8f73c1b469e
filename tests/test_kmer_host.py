"""k-mer ingestion, host side (no GPU): packing and FASTA structure.

Restates the reference's kmer tests (pkg/tests/test_kmer.py:53-124) for the
parts that run on the host: ``pack_kmer`` and the FASTA parse that feeds the
device (record separators, stripping, the headerless-sequence error).
"""

from __future__ import annotations

import itertools

import numpy as np
import pytest

from paper_2603_15486_b200.errors import FastaError
from paper_2603_15486_b200.kmer import pack_kmer, sequence_buffer, stream_kmers


def naive_pack(window):
    return int("".join("0123"["ACGT".index(c)] for c in window), 4)


def test_pack_pinned_examples():
    assert pack_kmer("ACGT") == 27
    assert pack_kmer("AAAA") == 0
    assert pack_kmer("TTTT") == 255
    assert pack_kmer("A") == 0 and pack_kmer("T") == 3
    assert pack_kmer("ACGN") is None
    assert pack_kmer("acgt") == 27


def test_pack_rejects_bad_lengths():
    with pytest.raises(ValueError):
        pack_kmer("")
    with pytest.raises(ValueError):
        pack_kmer("A" * 32)
    assert pack_kmer("A" * 31) == 0


def test_pack_matches_naive_and_is_injective():
    seen = set()
    for bases in itertools.product("ACGT", repeat=4):
        v = pack_kmer("".join(bases))
        assert v == naive_pack("".join(bases)) and v not in seen
        seen.add(v)
    rng = np.random.default_rng(6)
    for _ in range(200):
        word = "".join("ACGT"[d] for d in rng.integers(0, 4, size=21))
        assert pack_kmer(word) == naive_pack(word)


def test_sequence_buffer_structure():
    # records separated, lines of one record joined, blank lines and whitespace dropped
    assert sequence_buffer([">a", "ACG", " TT ", "", ">b", "gg"]) == b"\nACGTT\ngg"
    assert sequence_buffer([]) == b""
    assert sequence_buffer([">only header"]) == b"\n"


def test_headerless_sequence_raises_with_line_number():
    with pytest.raises(FastaError) as exc:
        sequence_buffer(["", "  ", "ACGT"])
    assert exc.value.line_number == 3 and "line 3" in str(exc.value)


def test_stream_k_validation_happens_before_any_device_work():
    # a lazy iterator like the reference's generator: checked on first next()
    it = stream_kmers([">r", "ACGT"], 0)
    with pytest.raises(ValueError):
        list(it)
    with pytest.raises(ValueError):
        list(stream_kmers([">r", "ACGT"], 32))
    with pytest.raises(ValueError):
        stream_kmers([">r", "ACGT"], 32, as_tensor=True)
    with pytest.raises(FastaError):
        list(stream_kmers(["", "  ", "ACGT"], 2))


def test_kmer_golden_fixture_is_the_reference_stream():
    """The fixture's tiny.fasta windows, re-packed on the host with pack_kmer,
    equal the reference stream stored next to it (pins the fixture itself)."""
    from pathlib import Path

    z = np.load(Path(__file__).parent / "golden" / "kmer_golden.npz")
    for name in ("tiny", "synth"):
        text = bytes(z[f"{name}_fasta"]).decode()
        for k in (5, 31):
            want = []
            for rec in text.split(">")[1:]:
                seq = "".join(ln.strip() for ln in rec.splitlines()[1:])
                for i in range(len(seq) - k + 1):
                    v = pack_kmer(seq[i:i + k])
                    if v is not None:
                        want.append(v)
            assert np.array_equal(np.array(want, dtype=np.uint64), z[f"{name}_k{k}"]), (name, k)
