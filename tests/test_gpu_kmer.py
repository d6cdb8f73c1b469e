"""GPU k-mer extraction (ckf_kmers) against a naive re-parse oracle.

The oracle restates the reference's own test oracle (pkg/tests/test_kmer.py
naive_parse: base-4 digit strings over whole records); the cases follow
pkg/tests/test_kmer.py:92-175 plus long records whose ambiguous bases and
record breaks sit on the device's 1024-base chunk boundaries.
"""

from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

from paper_2603_15486_b200 import CuckooFilter, FilterConfig
from paper_2603_15486_b200.bench_harness import RunSpec
from paper_2603_15486_b200.kmer import kmer_array, kmer_bench, stream_kmers

pytestmark = pytest.mark.gpu


def naive_pack(window):
    return int("".join("0123"["ACGT".index(c)] for c in window), 4)


def naive_parse(lines, k):
    records, current = [], None
    for line in lines:
        line = line.strip()
        if not line:
            continue
        if line.startswith(">"):
            if current is not None:
                records.append(current)
            current = ""
        else:
            current += line
    if current is not None:
        records.append(current)
    out = []
    for rec in records:
        seq = rec.upper()
        for i in range(len(seq) - k + 1):
            win = seq[i:i + k]
            if set(win) <= set("ACGT"):
                out.append(naive_pack(win))
    return out


def fast_naive(seq: str, k: int) -> np.ndarray:
    """Vectorised naive windows of one record (long-sequence cases)."""
    code = np.full(256, 4, np.uint64)
    for c, v in zip("ACGTacgt", [0, 1, 2, 3, 0, 1, 2, 3]):
        code[ord(c)] = v
    b = code[np.frombuffer(seq.encode(), np.uint8)]
    n = len(b) - k + 1
    if n <= 0:
        return np.zeros(0, np.uint64)
    vals = np.zeros(n, np.uint64)
    bad = np.zeros(n, bool)
    for j in range(k):
        w = b[j:j + n]
        bad |= w > 3
        vals = (vals << np.uint64(2)) | (w & np.uint64(3))
    return vals[~bad]


def test_stream_pinned_windows():
    assert list(stream_kmers([">r1", "ACGTA"], 4)) == [naive_pack("ACGT"), naive_pack("CGTA")]
    assert list(stream_kmers([">r", "ACNGT"], 2)) == [naive_pack("AC"), naive_pack("GT")]
    assert list(stream_kmers([">short", "ACG"], 4)) == []


def test_stream_windows_never_span_records():
    assert list(stream_kmers([">a", "ACG", ">b", "TAC"], 3)) == [naive_pack("ACG"), naive_pack("TAC")]


def test_stream_handles_wrapped_lines_and_case():
    lines = [">wrapped", "acGT", "ACgt"]
    assert list(stream_kmers(lines, 5)) == naive_parse(lines, 5)


def test_stream_matches_naive_on_random_fasta():
    rng = np.random.default_rng(9)
    alphabet = "ACGTacgtN"
    lines = []
    for rec in range(8):
        lines.append(f">record_{rec}")
        length = int(rng.integers(5, 220))
        seq = "".join(alphabet[d] for d in rng.integers(0, len(alphabet), size=length))
        for i in range(0, length, 37):
            lines.append(seq[i:i + 37])
        if rec % 3 == 0:
            lines.append("")
    for k in (1, 2, 7, 31):
        assert list(stream_kmers(lines, k)) == naive_parse(lines, k)


def test_stream_from_path(tmp_path):
    rng = np.random.default_rng(3)
    text = []
    for r in range(5):
        text.append(f">chr{r} some description")
        seq = "".join("ACGTN"[d] for d in rng.choice(5, size=int(rng.integers(50, 400)), p=[.24, .24, .24, .24, .04]))
        text += [seq[i:i + 60] for i in range(0, len(seq), 60)]
    p = tmp_path / "x.fasta"
    p.write_text("\n".join(text) + "\n")
    for k in (4, 31):
        assert list(stream_kmers(p, k)) == naive_parse(text, k)


@pytest.mark.parametrize("k", [1, 15, 31])
def test_long_records_across_chunk_boundaries(k):
    rng = np.random.default_rng(k)
    recs = []
    for length in (1023, 1024, 1025, 5000, 70_000):
        s = np.array(list("ACGTacgt"))[rng.integers(0, 8, size=length)]
        for pos in (1023, 1024, 2047, 3000):  # ambiguous bases on / next to chunk edges
            if pos < length:
                s[pos] = "N"
        recs.append("".join(s))
    lines = []
    for i, r in enumerate(recs):
        lines.append(f">r{i}")
        lines += [r[j:j + 80] for j in range(0, len(r), 80)]
    want = np.concatenate([fast_naive(r, k) for r in recs])
    got = kmer_array(lines, k)
    assert got.dtype == np.uint64 and np.array_equal(got, want)


def test_kmer_pipeline_insert_query_delete(tmp_path):
    rng = np.random.default_rng(8)
    seq = "".join("ACGT"[d] for d in rng.integers(0, 4, size=200_000))
    p = tmp_path / "g.fasta"
    p.write_text(">g\n" + "\n".join(seq[i:i + 70] for i in range(0, len(seq), 70)) + "\n")
    keys = stream_kmers(p, 31, as_tensor=True)
    assert keys.numel() == len(seq) - 30
    filt = CuckooFilter(FilterConfig(bucket_count=1 << 14))
    res = filt.insert_batch(keys)
    assert res.n_failed == 0 and bool(filt.query_batch(keys).all())
    filt.delete_batch(keys)
    assert len(filt) == 0


def test_kmer_bench_reports_three_phases(tmp_path):
    rng = np.random.default_rng(1)
    seq = "".join("ACGT"[d] for d in rng.integers(0, 4, size=30_000))
    p = tmp_path / "t.fasta"
    p.write_text(">t\n" + seq + "\n")
    reports = kmer_bench(p, 31, RunSpec(bucket_count=1 << 12))
    assert [r.op for r in reports] == ["insert", "query_pos", "delete"]
    assert all(r.n_keys == len(seq) - 30 for r in reports)
    assert reports[0].insert_failures == 0 and all(r.throughput > 0 for r in reports)


# ---- pinned to the reference's own output (tests/golden/make_kmer_golden.py) ----

@pytest.mark.parametrize("name", ["tiny", "synth"])
@pytest.mark.parametrize("k", [1, 2, 5, 15, 21, 31])
def test_stream_matches_reference_golden(name, k):
    z = np.load(Path(__file__).parent / "golden" / "kmer_golden.npz")
    text = bytes(z[f"{name}_fasta"]).decode()
    want = z[f"{name}_k{k}"]
    got = kmer_array(text.splitlines(keepends=True), k)
    assert np.array_equal(got, want)
    if name == "tiny" and k == 31:
        assert len(got) == 332  # reference pkg/tests/test_cli.py:97
    it = stream_kmers(text.splitlines(keepends=True), k)
    assert iter(it) is it and [next(it) for _ in range(min(3, len(want)))] == [int(v) for v in want[:3]]
