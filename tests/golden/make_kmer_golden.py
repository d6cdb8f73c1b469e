"""Golden k-mer streams produced by the REFERENCE (swarcuckoo.kmer.stream_kmers).

Run in the build container (where /root/reference exists):

    python tests/golden/make_kmer_golden.py

Inputs: the reference's own test FASTA (pkg/tests/data/tiny.fasta, stored
byte-for-byte in the fixture because the GPU box has no /root/reference) and
a synthetic FASTA exercising what the parse must get right: blank lines,
lower case, N runs, records shorter than k, lines of mixed widths, a record
longer than the device chunk (1024 bases).  Output: tests/golden/kmer_golden.npz
with, per (input, k), the reference's packed stream as uint64.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))
from swarcuckoo.kmer import stream_kmers  # noqa: E402

HERE = Path(__file__).resolve().parent
KS = (1, 2, 5, 15, 21, 31)


def synthetic() -> bytes:
    rng = np.random.default_rng(2603)
    lines = [">s0 blank lines and case", "", "acgtACGTnnACGT", "   ", "TTTTGGGGCCCCAAAA"]
    lines += [">s1 shorter than most k", "ACG"]
    seq = "".join("ACGTNacgt"[d] for d in rng.choice(9, size=3000, p=[.2, .2, .2, .2, .02, .045, .045, .045, .045]))
    lines += [">s2 long record, mixed widths"] + [seq[i:i + w] for i, w in zip(range(0, 3000, 70), [70, 61, 80] * 100)]
    lines += [">s3 empty record", ">s4", "N" * 40 + "ACGTACGTACGTACGTACGTACGTACGTACGTAC"]
    return ("\n".join(lines) + "\n").encode()


def main() -> None:
    tiny = (REF.parent / "tests" / "data" / "tiny.fasta").read_bytes()
    out = {"tiny_fasta": np.frombuffer(tiny, np.uint8), "synth_fasta": np.frombuffer(synthetic(), np.uint8)}
    for name in ("tiny", "synth"):
        text = bytes(out[f"{name}_fasta"]).decode()
        for k in KS:
            out[f"{name}_k{k}"] = np.fromiter(stream_kmers(text.splitlines(keepends=True), k), dtype=np.uint64)
    np.savez_compressed(HERE / "kmer_golden.npz", **out)
    print({k: v.shape for k, v in out.items()})


if __name__ == "__main__":
    main()
